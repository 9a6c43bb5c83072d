// Narrow-line build of the fp32 W = 256 line-task sweep: every W = 256 line is
// transformed by a whole warp, 8 points per lane (pty_fft.cuh narrow_fft256),
// so a CTA of 512 threads holds the same 4 teams / 16 groups as the 256-thread
// default and the SM runs 32 warps instead of 16 at the same shared-memory
// footprint (64 registers per thread).  The headers are compiled here with
// Shape<256> = {8, 32} inside namespace pty_n (so no template of the default
// build is redefined); pty_sweep_host.cuh dispatches to this translation unit
// when PTY_NARROW=1.
//
// Opt-in build (PTY_NVCC_DEFS=-DPTY_BUILD_NARROW): measured 32.9 ms per sweep
// against 21.9 ms for the default at 18 replicas (profiles/r2_ab.txt).  The
// two exchanges per line double the shared-memory traffic of the transforms
// and the 64-register cap of 2 x 512 threads per SM spills the per-CTA state.
#ifdef PTY_BUILD_NARROW
#define PTY_NARROW256 1
#define pty pty_n
#include "pty_sweep_host.cuh"
#undef pty

namespace pty_n {
std::atomic<long long> g_launches{0};
std::vector<unsigned long long> g_timeline;
int g_timeline_grid = 0;
}  // namespace pty_n

namespace pty {
extern std::atomic<long long> g_launches;
extern std::vector<unsigned long long> g_timeline;
extern int g_timeline_grid;
}  // namespace pty

extern "C" int pty_internal_sweep_narrow_f32_w256(const PtySweepArgs* a, void* stream) {
    const long long before = pty_n::g_launches.load();
    const int rc = pty_n::run_sweep_lines<float, 256>(a, static_cast<cudaStream_t>(stream));
    pty::g_launches.fetch_add(pty_n::g_launches.load() - before);
    if (!pty_n::g_timeline.empty()) {
        pty::g_timeline = pty_n::g_timeline;
        pty::g_timeline_grid = pty_n::g_timeline_grid;
        pty_n::g_timeline.clear();
    }
    return rc;
}
#endif  // PTY_BUILD_NARROW
