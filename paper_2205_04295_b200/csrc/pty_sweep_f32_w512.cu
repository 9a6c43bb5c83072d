// explicit instantiation of the sweep for float, W = 512
#include "pty_sweep_host.cuh"
namespace pty {
template int run_sweep<float, 512>(const PtySweepArgs*, cudaStream_t);
template int run_sweep_batched<float, 512>(const BatchedSweepIO&, cudaStream_t);
template int sweep_batched_fits<float, 512>(int, int);
}
