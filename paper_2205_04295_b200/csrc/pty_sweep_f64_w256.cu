// explicit instantiation of the sweep for double, W = 256
#include "pty_sweep_host.cuh"
namespace pty {
template int run_sweep<double, 256>(const PtySweepArgs*, cudaStream_t);
}
