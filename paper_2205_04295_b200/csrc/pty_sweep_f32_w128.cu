// explicit instantiation of the sweep for float, W = 128
#include "pty_sweep_host.cuh"
namespace pty {
template int run_sweep<float, 128>(const PtySweepArgs*, cudaStream_t);
template int run_sweep_batched<float, 128>(const BatchedSweepIO&, cudaStream_t);
template int sweep_batched_fits<float, 128>(int, int);
}
