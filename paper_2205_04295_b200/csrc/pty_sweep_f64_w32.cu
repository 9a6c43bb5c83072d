// explicit instantiation of the sweep for double, W = 32
#include "pty_sweep_host.cuh"
namespace pty {
template int run_sweep<double, 32>(const PtySweepArgs*, cudaStream_t);
}
