// explicit instantiation of the sweep for float, W = 256
#include "pty_sweep_host.cuh"
namespace pty {
template int run_sweep<float, 256>(const PtySweepArgs*, cudaStream_t);
template int run_sweep_batched<float, 256>(const BatchedSweepIO&, cudaStream_t);
template int sweep_batched_fits<float, 256>(int, int);
}

#ifdef PTY_PROBE
// debug: the probe stamps of the last sweep (64 steps x 32 slots)
extern "C" __attribute__((visibility("default"))) int pty_probe_read(unsigned long long* out) {
    return cudaMemcpyFromSymbol(out, pty::pty_probe_buf, sizeof(pty::pty_probe_buf)) == cudaSuccess ? 0 : 1;
}
#endif
