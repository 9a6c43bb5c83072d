// explicit instantiation of the sweep for float, W = 64
#include "pty_sweep_host.cuh"
namespace pty {
template int run_sweep<float, 64>(const PtySweepArgs*, cudaStream_t);
template int run_sweep_batched<float, 64>(const BatchedSweepIO&, cudaStream_t);
template int sweep_batched_fits<float, 64>(int, int);
}
