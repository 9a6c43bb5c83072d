// explicit instantiation of the sweep for double, W = 32
#include "pty_sweep_host.cuh"
namespace pty {
template int run_sweep<double, 32>(const PtySweepArgs*, cudaStream_t);
template int run_sweep_batched<double, 32>(const BatchedSweepIO&, cudaStream_t);
template int sweep_batched_fits<double, 32>(int, int);
}
