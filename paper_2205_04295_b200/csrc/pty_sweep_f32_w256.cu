// explicit instantiation of the sweep for float, W = 256
#include "pty_sweep_host.cuh"
namespace pty {
template int run_sweep<float, 256>(const PtySweepArgs*, cudaStream_t);
}
