// pty_sweep_tiles_host.cuh -- host side of the latency variant of pty_sweep: workspace layout, tile-size
// choice and the cooperative launch of sweep_kernel<T, W>.  Explicitly
// instantiated per (dtype, window) in pty_sweep_*.cu so the kernels compile in
// parallel translation units.
#pragma once
#include "pty_host.cuh"
#include "pty_sweep_tiles.cuh"

namespace pty {
namespace tiles {

// ------------------------------------------------------------- sweep ------
constexpr int kMinTC = 1;   // narrowest column tile: one column per item keeps every CTA busy for one reconstruction (measured: 4 -> 1 cut the single-reconstruction visit from 26.6 to 22.6 us)
constexpr int kTilesNoFit = -1;   // internal: resident tiles exceed shared memory   // column tiles are >= 4 complex (32-byte sectors)

struct SweepLayout {
    unsigned int* barrier;
    int* anchors;
    void* scratch;
    void* omax;
    void* peak;
    void* tmax;
    double* err_part;
    size_t bytes;
};

template <typename T>
inline SweepLayout carve_sweep(void* ws, int W, int M, int N, int S) {
    Carver c(ws);
    SweepLayout L{};
    L.barrier = c.take<unsigned int>(sizeof(unsigned int));
    L.anchors = c.take<int>((size_t)S * N * 2 * sizeof(int));
    L.scratch = c.take<void>((size_t)S * M * W * W * sizeof(cplx<T>));
    L.omax = c.take<void>((size_t)S * W * sizeof(T));
    L.peak = c.take<void>((size_t)2 * S * W * sizeof(T));
    L.tmax = c.take<void>((size_t)S * W * sizeof(T));
    L.err_part = c.take<double>((size_t)S * N * (W / kMinTC) * 3 * sizeof(double));
    L.bytes = c.off;
    return L;
}

template <typename T, int W>
int run_sweep(const PtySweepArgs* a, cudaStream_t st) {
    const int M = a->modes, N = a->n_positions, S = a->n_slots;
    SweepLayout L = carve_sweep<T>(a->workspace, W, M, N, S);
    if (!a->workspace || a->workspace_bytes < (int64_t)L.bytes) return PTY_ERR_ARGUMENT;
    const cplx<T>* tw = twiddles<T, W>(st);
    if (!tw) return PTY_ERR_CUDA;

    SweepDev P{};
    P.W = W; P.M = M; P.N = N; P.nslots = S;
    P.alpha_o = a->alpha_obj; P.alpha_p = a->alpha_probe; P.beta = a->beta; P.gamma = a->gamma;
    P.eps_rel = a->epsilon_rel;
    P.update_probe = a->update_probe; P.track_mod = a->track_modulus; P.sense = a->sense;
    P.barrier = L.barrier; P.anchors = L.anchors; P.scratch = L.scratch;
    P.omax_part = L.omax; P.peak_part = L.peak; P.tmax_part = L.tmax;
    P.err_part = L.err_part; P.twiddles = tw;
    ErrOut outs{};
    for (int s = 0; s < S; ++s) {
        const PtySlot& h = a->slots[s];
        if (!h.obj || !h.probes || !h.patterns || !h.positions || !h.order || !h.status || !h.err_out)
            return PTY_ERR_ARGUMENT;
        if (a->sense != PTY_SENSE_NONE && !h.stage) return PTY_ERR_ARGUMENT;
        if (h.H < W || h.Wc < W) return PTY_ERR_ARGUMENT;
        P.slot[s] = SlotDev{h.obj, h.H, h.Wc, h.r0, h.c0, h.probes, h.patterns, h.positions,
                            h.order, h.stage, h.err_out, h.status};
        outs.p[s] = h.err_out;
    }

    // launch geometry: kSweepThreads-thread CTAs, `per_sm` of them per SM
    // (default 2 so one CTA's loads overlap the other's FFTs), cooperative.
    // Tiles: the smallest power-of-two rows/columns per item that keep the
    // item count <= the CTA count (every CTA busy even for one reconstruction),
    // bounded by the per-CTA shared-memory budget.  PTY_TR / PTY_TC /
    // PTY_CTAS_PER_SM override (tuning).
    const int sms = sm_count();
    const int want_per_sm = std::max(1, env_int("PTY_CTAS_PER_SM", kSweepMinCtasPerSm));
    const size_t smem_sm = max_smem_per_sm();
    const size_t fixed = sweep_smem_fixed<T, W>();
    constexpr int LS = line_stride<W>();
    const size_t line_bytes = (size_t)LS * sizeof(cplx<T>);
    int per_sm = 0, grid = 0, TR = 0, TC = 0, nRT = 0, nCT = 0, K = 0;
    size_t tile_bytes = 0;
    // fewer CTAs per SM (bigger shared-memory budget) until the resident
    // tiles fit; kTilesNoFit sends the caller to the line-task kernel.
    for (per_sm = want_per_sm; per_sm >= 1; --per_sm) {
        const size_t budget = std::min(max_dyn_smem(), smem_sm / per_sm - 1024 - 512) - fixed;
        grid = sms * per_sm;
        TR = env_int("PTY_TR", 0);
        if (TR <= 0) {
            TR = 1;
            while (TR < W && (long)S * (W / TR) > grid && (size_t)2 * TR * M * line_bytes <= budget) TR *= 2;
        }
        TC = env_int("PTY_TC", 0);
        if (TC <= 0) {
            TC = kMinTC;
            while (TC < W && (long)S * (W / TC) > grid && (size_t)2 * TC * M * line_bytes <= budget) TC *= 2;
        }
        if (TR < 1 || TR > W || (W % TR) || TC < kMinTC || TC > W || (W % TC)) return PTY_ERR_ARGUMENT;
        nRT = W / TR;
        nCT = W / TC;
        K = (S * nCT + grid - 1) / grid;
        tile_bytes = std::max((size_t)TR * M * line_bytes, (size_t)K * M * TC * line_bytes);
        if (tile_bytes <= budget) break;
    }
    if (per_sm < 1) return kTilesNoFit;
    P.TR = TR; P.TC = TC; P.nRT = nRT; P.nCT = nCT; P.K = K;
    P.lgTR = 0; while ((1 << P.lgTR) < TR) ++P.lgTR;
    P.lgTC = 0; while ((1 << P.lgTC) < TC) ++P.lgTC;
    const size_t smem = fixed + tile_bytes;

    auto kern = sweep_kernel<T, W>;
    if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess)
        return PTY_ERR_CUDA;
    int fit = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&fit, kern, kSweepThreads, smem) != cudaSuccess || fit < per_sm)
        return PTY_ERR_CUDA;   // the cooperative grid must be co-resident

    // debug timeline (PTY_TIMELINE=<steps>): per-CTA phase completion stamps
    const int tl_steps = std::min(env_int("PTY_TIMELINE", 0), N);
    unsigned long long* tl = nullptr;
    if (tl_steps > 0) {
        if (cudaMalloc(&tl, (size_t)tl_steps * 9 * grid * sizeof(unsigned long long)) != cudaSuccess) return PTY_ERR_CUDA;
        P.timeline = tl;
        P.timeline_steps = tl_steps;
    }
    if (cudaMemsetAsync(L.barrier, 0, sizeof(unsigned int), st) != cudaSuccess) return PTY_ERR_CUDA;
    if (cudaMemsetAsync(L.err_part, 0, (size_t)S * N * nCT * 3 * sizeof(double), st) != cudaSuccess)
        return PTY_ERR_CUDA;
    void* args[] = {&P};
    cudaError_t e = cudaLaunchCooperativeKernel((const void*)kern, dim3(grid), dim3(kSweepThreads), args, smem, st);
    if (e != cudaSuccess) return PTY_ERR_CUDA;
    sweep_finalize_kernel<<<S, 256, 0, st>>>(L.err_part, N, nCT, S, outs);
    count(2);
    if (tl) {
        g_timeline.assign((size_t)tl_steps * 9 * grid, 0ull);
        cudaMemcpyAsync(g_timeline.data(), tl, g_timeline.size() * sizeof(unsigned long long),
                        cudaMemcpyDeviceToHost, st);
        cudaStreamSynchronize(st);
        cudaFree(tl);
        g_timeline_grid = grid;
    }
    return last_status();
}


}  // namespace tiles
}  // namespace pty
