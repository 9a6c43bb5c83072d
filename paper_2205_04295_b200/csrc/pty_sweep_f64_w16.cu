// explicit instantiation of the sweep for double, W = 16
#include "pty_sweep_host.cuh"
namespace pty {
template int run_sweep<double, 16>(const PtySweepArgs*, cudaStream_t);
template int run_sweep_batched<double, 16>(const BatchedSweepIO&, cudaStream_t);
template int sweep_batched_fits<double, 16>(int, int);
}
