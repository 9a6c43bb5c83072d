// pty_sweep_host.cuh -- host side of pty_sweep: workspace layout, tile-size
// choice and the cooperative launch of sweep_kernel<T, W>.  Explicitly
// instantiated per (dtype, window) in pty_sweep_*.cu so the kernels compile in
// parallel translation units.
#pragma once
#include "pty_host.cuh"
#include "pty_sweep.cuh"
#include "pty_sweep_tiles_host.cuh"

namespace pty {

// ------------------------------------------------------------- sweep ------
struct SweepLayout {
    unsigned int* barrier;
    int* anchors;
    int4* steptab;
    void* scratch;
    void* totT;
    void* omax;
    void* peak;
    void* tmax;
    double* err_part;
    double* visit_sum;
    void* ppg;
    unsigned int* slot_bar;
    unsigned int* sm_pair;
    size_t bytes;
};

template <typename T>
inline SweepLayout carve_sweep(void* ws, int W, int M, int N, int S) {
    Carver c(ws);
    SweepLayout L{};
    L.barrier = c.take<unsigned int>(sizeof(unsigned int));
    L.anchors = c.take<int>((size_t)S * N * 2 * sizeof(int));
    L.steptab = c.take<int4>((size_t)S * N * sizeof(int4));
    L.scratch = c.take<void>((size_t)S * M * W * W * sizeof(cplx<T>));
    L.totT = c.take<void>((size_t)S * W * W * sizeof(T));
    L.omax = c.take<void>((size_t)2 * S * (W / 4) * sizeof(T));
    L.peak = c.take<void>((size_t)2 * S * (W / 4) * sizeof(T));
    L.tmax = c.take<void>((size_t)S * W * sizeof(T));
    L.err_part = c.take<double>((size_t)S * N * W * 3 * sizeof(double));
    L.visit_sum = c.take<double>((size_t)S * N * 3 * sizeof(double));
    L.ppg = c.take<void>((size_t)S * W * W * sizeof(T));
    L.slot_bar = c.take<unsigned int>((size_t)S * 32 * sizeof(unsigned int));
    L.sm_pair = c.take<unsigned int>((8 + 256) * sizeof(unsigned int));
    L.bytes = c.off;
    return L;
}

// few slots (latency): the tile kernel; many slots (throughput): line tasks.
inline int tiles_max_slots() { return env_int("PTY_SWEEP_TILES_MAX", 4); }   // measured crossover: lines win from 5 slots

template <typename T>
inline size_t sweep_workspace(int W, int M, int N, int S) {
    return std::max(carve_sweep<T>(nullptr, W, M, N, S).bytes, tiles::carve_sweep<T>(nullptr, W, M, N, S).bytes);
}

template <typename T, int W>
int run_sweep_lines(const PtySweepArgs* a, cudaStream_t st);

}  // namespace pty
// the narrow-line fp32 W = 256 build (pty_sweep_f32_w256n.cu)
extern "C" int pty_internal_sweep_narrow_f32_w256(const PtySweepArgs* a, void* stream);
namespace pty {

inline bool narrow_lines() { return env_int("PTY_NARROW", 0) != 0; }

template <typename T, int W>
int run_sweep(const PtySweepArgs* a, cudaStream_t st) {
    if (a->n_slots <= tiles_max_slots()) {
        const int rc = tiles::run_sweep<T, W>(a, st);
        if (rc != tiles::kTilesNoFit) return rc;
    }
#ifdef PTY_BUILD_NARROW
    if constexpr (std::is_same<T, float>::value && W == 256) {
        if (narrow_lines()) return pty_internal_sweep_narrow_f32_w256(a, st);
    }
#endif
    return run_sweep_lines<T, W>(a, st);
}

// Grid-flavour launch plan of the line-task kernel for S slots (the part of
// run_sweep_lines below that the batched flavour shares): shared memory,
// residency, staged row blocks, slot-local barriers, SM pairing.
template <typename T, int W, bool BAT = false>
int plan_lines_grid(int M, int S, SweepDev& P, const SweepLayout& L, int& grid, size_t& smem) {
    constexpr int NGRP = kSweepThreads / Shape<W>::B;
    const size_t res_bytes = (size_t)NGRP * M * xch_size<W>() * sizeof(cplx<T>);
    const size_t base_phase = sweep_smem_phase<T, W>(kSweepThreads);
    const size_t res_phase = std::max(base_phase, res_bytes);
    const bool res_fit = 2 * (sweep_smem_fixed<T, W>() + res_phase + 1024) <= max_smem_per_sm();
    const int grid_ctas = sm_count() * kSweepMaxCtasPerSm;
    P.resident = (env_int("PTY_RESIDENT", 1) && res_fit && (long)S * W <= (long)grid_ctas * NGRP) ? 1 : 0;
    constexpr int NTEAM4 = kSweepThreads / (4 * Shape<W>::B);
    constexpr int RTS = kStagedRows, NTEAM_S = kSweepThreads / (RTS * Shape<W>::B);
    const size_t p4s_bytes = (size_t)NTEAM_S * M * RTS * block_line_stride<W, RTS>() * sizeof(cplx<T>) +
                             (size_t)NTEAM_S * RTS * sizeof(T);
    size_t phase = P.resident ? res_phase : base_phase;
    const bool p4s_fit = 2 * (sweep_smem_fixed<T, W>() + std::max(phase, p4s_bytes) + 1024) <= max_smem_per_sm();
    P.p4_staged = (env_int("PTY_P4_STAGED", 1) && M <= 4 && p4s_fit) ? 1 : 0;
    if (P.p4_staged) phase = std::max(phase, p4s_bytes);
    P.p1_staged = P.p4_staged;
    smem = sweep_smem_fixed<T, W>() + phase;
    if (smem > max_dyn_smem()) return PTY_ERR_ARGUMENT;
    auto kern = sweep_kernel<T, W, false, BAT>;
    if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess)
        return PTY_ERR_CUDA;
    int fit = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&fit, kern, kSweepThreads, smem) != cudaSuccess || fit < 1)
        return PTY_ERR_CUDA;
    int per_sm = std::min(fit, kSweepMaxCtasPerSm);
    const int want = env_int("PTY_CTAS_PER_SM", 0);
    if (want > 0) per_sm = std::min(per_sm, want);
    grid = sm_count() * per_sm;
    if ((long)S * W > (long)grid * NGRP) P.resident = 0;   // more than one column task per group
    const int cps_rows = P.p4_staged ? (W / RTS) / NTEAM_S : (W / 4) / NTEAM4, cps_cols = W / NGRP;
    const bool rows_even = P.p4_staged ? (W / RTS) % NTEAM_S == 0 : (W / 4) % NTEAM4 == 0;
    P.cps = cps_rows;
    P.slot_local = (env_int("PTY_SLOT_BARRIER", 1) && P.p1_staged && P.p4_staged && P.resident &&
                    cps_rows == cps_cols && cps_rows >= 1 && (long)S * cps_rows <= grid &&
                    rows_even && W % NGRP == 0) ? 1 : 0;
    P.slot_bar = L.slot_bar;
    const int spp = (grid / 2) / std::max(1, cps_rows);
    P.pair = (P.slot_local && per_sm == 2 && S > spp && S <= 2 * spp && env_int("PTY_SLOT_PAIR", 1)) ? spp * cps_rows : 0;
    P.pair_offset = P.pair > 0 ? std::max(0, env_int("PTY_PAIR_OFFSET", 2)) : 0;
    P.sm_pair = L.sm_pair;
    return PTY_OK;
}

// most slots the batched flavour can run at once (slot-local: one row block
// and one column per CTA / group of a slot, 2 CTAs per SM)
template <int W> inline int batched_max_slots() {
    constexpr int NGRP = kSweepThreads / Shape<W>::B;
    const int cps = W / NGRP;
    return std::max(1, std::min(kMaxSlots, (sm_count() * kSweepMaxCtasPerSm) / std::max(1, cps)));
}

// workspace of the batched flavour for cnt positions per launch
template <typename T>
inline size_t sweep_batched_workspace(int W, int M, int S, int cnt) {
    const int steps = (cnt + S - 1) / S;
    return carve_sweep<T>(nullptr, W, M, steps, S).bytes;
}

template <typename T, int W>
int run_sweep_lines(const PtySweepArgs* a, cudaStream_t st) {
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
    P.barrier = L.barrier; P.anchors = L.anchors; P.steptab = L.steptab; P.scratch = L.scratch; P.totT = L.totT;
    P.omax_part = L.omax; P.peak_part = L.peak; P.tmax_part = L.tmax;
    P.err_part = L.err_part; P.twiddles = tw; P.ppg = L.ppg;
    ErrOut outs{};
    for (int s = 0; s < S; ++s) {
        const PtySlot& h = a->slots[s];
        if (!h.obj || !h.probes || !h.patterns || !h.patterns_t || !h.positions || !h.order || !h.status || !h.err_out)
            return PTY_ERR_ARGUMENT;
        if (a->sense != PTY_SENSE_NONE && !h.stage) return PTY_ERR_ARGUMENT;
        if (h.H < W || h.Wc < W) return PTY_ERR_ARGUMENT;
        P.slot[s] = SlotDev{h.obj, h.H, h.Wc, h.r0, h.c0, h.probes, h.patterns, h.patterns_t, h.positions,
                            h.order, h.stage, h.err_out, h.status};
        outs.p[s] = h.err_out;
    }

    // launch geometry.  Grid flavour (default): kSweepThreads-thread CTAs, as
    // many per SM as fit (<= 2), cooperative, all slots in lock-step;
    // PTY_CTAS_PER_SM overrides downwards.  Cluster flavour (PTY_CLUSTER=K):
    // one cluster of K CTAs per slot, slots scheduled independently (measured
    // slower at 16 replicas: 8 clusters of 16 fit the GPCs at once).
    // P2 -> P3 residency: every group owns at most one column task per step and
    // its M transformed lines fit next to the phase region with 2 CTAs per SM
    constexpr int NGRP = kSweepThreads / Shape<W>::B;
    const size_t res_bytes = (size_t)NGRP * M * xch_size<W>() * sizeof(cplx<T>);
    const size_t base_phase = sweep_smem_phase<T, W>(kSweepThreads);
    const int want_res = env_int("PTY_RESIDENT", 1);
    const size_t res_phase = std::max(base_phase, res_bytes);
    const bool res_fit = 2 * (sweep_smem_fixed<T, W>() + res_phase + 1024) <= max_smem_per_sm();
    const int grid_ctas = sm_count() * kSweepMaxCtasPerSm;
    P.resident = (want_res && res_fit && (long)S * W <= (long)grid_ctas * NGRP && env_int("PTY_CLUSTER", 0) == 0) ? 1 : 0;
    // P4 staged: M*4 padded lines per team (M <= 4)
    constexpr int NTEAM4 = kSweepThreads / (4 * Shape<W>::B);
    constexpr int RTS = kStagedRows, NTEAM_S = kSweepThreads / (RTS * Shape<W>::B);
    const size_t p4s_bytes = (size_t)NTEAM_S * M * RTS * block_line_stride<W, RTS>() * sizeof(cplx<T>) +
                             (size_t)NTEAM_S * RTS * sizeof(T);
    size_t phase = P.resident ? res_phase : base_phase;
    const bool p4s_fit = 2 * (sweep_smem_fixed<T, W>() + std::max(phase, p4s_bytes) + 1024) <= max_smem_per_sm();
    P.p4_staged = (env_int("PTY_P4_STAGED", 1) && M <= 4 && p4s_fit) ? 1 : 0;
    if (P.p4_staged) phase = std::max(phase, p4s_bytes);
    P.p1_staged = P.p4_staged;                 // staged P1 and P4 share the row-block task layout
    size_t smem = sweep_smem_fixed<T, W>() + phase;
    if (smem > max_dyn_smem()) return PTY_ERR_ARGUMENT;
    int K = std::max(0, env_int("PTY_CLUSTER", 0));
    int grid = 0;
    if (K > 0) {
        auto kern = sweep_kernel<T, W, true>;
        if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess)
            return PTY_ERR_CUDA;
        if (K > 8 && cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1) != cudaSuccess)
            K = 8;
        // largest power of two <= K with at least one co-resident cluster
        for (; K >= 1; K /= 2) {
            cudaLaunchConfig_t cfg{};
            cudaLaunchAttribute at[1];
            cfg.gridDim = dim3(K * S);
            cfg.blockDim = dim3(kSweepThreads);
            cfg.dynamicSmemBytes = smem;
            cfg.stream = st;
            at[0].id = cudaLaunchAttributeClusterDimension;
            at[0].val.clusterDim.x = K;
            at[0].val.clusterDim.y = 1;
            at[0].val.clusterDim.z = 1;
            cfg.attrs = at;
            cfg.numAttrs = 1;
            int nclusters = 0;
            if (cudaOccupancyMaxActiveClusters(&nclusters, kern, &cfg) == cudaSuccess && nclusters > 0) break;
            cudaGetLastError();
        }
        if (K < 1) return PTY_ERR_CUDA;
        grid = K * S;
    } else {
        const int rc = plan_lines_grid<T, W>(M, S, P, L, grid, smem);
        if (rc) return rc;
    }

    // debug timeline (PTY_TIMELINE=<steps>): per-CTA phase completion stamps
    const int tl_steps = std::min(env_int("PTY_TIMELINE", 0), N);
    unsigned long long* tl = nullptr;
    if (tl_steps > 0) {
        if (cudaMalloc(&tl, (size_t)tl_steps * 9 * grid * sizeof(unsigned long long)) != cudaSuccess) return PTY_ERR_CUDA;
        P.timeline = tl;
        P.timeline_steps = tl_steps;
    }
    if (cudaMemsetAsync(L.barrier, 0, sizeof(unsigned int), st) != cudaSuccess) return PTY_ERR_CUDA;
    if (cudaMemsetAsync(L.slot_bar, 0, (size_t)S * 32 * sizeof(unsigned int), st) != cudaSuccess) return PTY_ERR_CUDA;
    if (cudaMemsetAsync(L.sm_pair, 0, (8 + 256) * sizeof(unsigned int), st) != cudaSuccess) return PTY_ERR_CUDA;
    if (cudaMemsetAsync(L.err_part, 0, (size_t)S * N * W * 3 * sizeof(double), st) != cudaSuccess)
        return PTY_ERR_CUDA;
    cudaError_t e;
    if (K > 0) {
        cudaLaunchConfig_t cfg{};
        cudaLaunchAttribute at[1];
        cfg.gridDim = dim3(grid);
        cfg.blockDim = dim3(kSweepThreads);
        cfg.dynamicSmemBytes = smem;
        cfg.stream = st;
        at[0].id = cudaLaunchAttributeClusterDimension;
        at[0].val.clusterDim.x = K;
        at[0].val.clusterDim.y = 1;
        at[0].val.clusterDim.z = 1;
        cfg.attrs = at;
        cfg.numAttrs = 1;
        e = cudaLaunchKernelEx(&cfg, sweep_kernel<T, W, true>, P);
    } else {
        void* args[] = {&P};
        const bool win = l2_window_set(st, L.scratch, (size_t)S * M * W * W * sizeof(cplx<T>) + (size_t)S * W * W * sizeof(T));
        e = cudaLaunchCooperativeKernel((const void*)sweep_kernel<T, W, false>, dim3(grid), dim3(kSweepThreads), args,
                                        smem, st);
        if (win) l2_window_clear(st);
    }
    if (e != cudaSuccess) return PTY_ERR_CUDA;
    err_visit_kernel<<<S * N, 256, 0, st>>>(L.err_part, W, L.visit_sum);
    err_slot_kernel<<<S, 256, 0, st>>>(L.visit_sum, N, S, outs);
    count(3);
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

// ------------------------------------------------- batched flavour -------
// The batched extension's contribution pass (pty_batch_contrib, oracle/
// batched.py contrib) on the line-task kernel: S slots each take every S-th
// position of the launch's range, so S positions are in flight at once with
// their scratch in L2, and the per-slot probe accumulators form S fixed
// groups (summed in slot order by bk_probe_reduce).
constexpr int kBatchedNoFit = -100;

struct BatchedSweepIO {
    const PtyBatchArgs* a;
    int off, cnt;                 // positions [off, off + cnt) of the batch
    int S;                        // slots
    void* onum;                   // [cnt][W][W] complex
    void* pgroup;                 // [S][2M+1][W][W] real, zeroed per batch by the caller
    void* ws;                     // sweep_batched_workspace bytes
    size_t ws_bytes;
};

// steptab of the batched flavour: slot s, step t -> batch position k = s + S t
// (j, anchor row, anchor column, k), or j = -1 past the range; bounds check
// (engine.py:192-195 anchors, round half to even)
static __global__ void batched_steptab_kernel(int4* steptab, int S, int steps, const int* batch, int cnt,
                                              const double* positions, int r0, int c0, int H, int Wc, int W,
                                              int* status) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= S * steps) return;
    const int s = i / steps, t = i % steps, k = s + S * t;
    if (k >= cnt) {
        steptab[i] = make_int4(-1, 0, 0, -1);
        return;
    }
    const int j = batch[k];
    const int ar = (int)rint(positions[2 * j + 1]) - r0;
    const int ac = (int)rint(positions[2 * j]) - c0;
    if (ar < 0 || ac < 0 || ar + W > H || ac + W > Wc) atomicOr(status, PTY_ERR_BOUNDS);
    steptab[i] = make_int4(j, ar, ac, k);
}

// 1 if the batched flavour runs for (T, W, M) with S slots on this device
template <typename T, int W>
int sweep_batched_fits(int M, int S) {
    SweepDev P{};
    SweepLayout L{};
    int grid = 0;
    size_t smem = 0;
    if (S < 1 || S > kMaxSlots || plan_lines_grid<T, W, true>(M, S, P, L, grid, smem) != PTY_OK) return 0;
    return (P.slot_local && P.p4_staged && P.resident) ? 1 : 0;
}

template <typename T, int W>
int run_sweep_batched(const BatchedSweepIO& io, cudaStream_t st) {
    const PtyBatchArgs* a = io.a;
    const int M = a->modes, S = io.S, steps = (io.cnt + S - 1) / S;
    if (S < 1 || S > kMaxSlots || io.cnt < 1) return kBatchedNoFit;
    SweepLayout L = carve_sweep<T>(io.ws, W, M, steps, S);
    if (!io.ws || io.ws_bytes < L.bytes) return PTY_ERR_ARGUMENT;
    const cplx<T>* tw = twiddles<T, W>(st);
    if (!tw) return PTY_ERR_CUDA;
    SweepDev P{};
    P.W = W; P.M = M; P.N = steps; P.nslots = S;
    P.alpha_o = a->alpha_obj; P.alpha_p = a->alpha_probe; P.beta = a->beta; P.gamma = a->gamma;
    P.eps_rel = a->epsilon_rel;
    P.update_probe = a->update_probe; P.track_mod = a->track_modulus; P.sense = a->sense;
    P.barrier = L.barrier; P.anchors = L.anchors; P.steptab = L.steptab; P.scratch = L.scratch; P.totT = L.totT;
    P.omax_part = L.omax; P.peak_part = L.peak; P.tmax_part = L.tmax;
    P.err_part = L.err_part; P.twiddles = tw; P.ppg = L.ppg;
    P.batched = 1;
    P.visit0 = a->visit0 + io.off;
    P.onum = io.onum;
    P.pgroup = io.pgroup;
    P.err_batch = a->err_part;
    for (int s = 0; s < S; ++s)
        P.slot[s] = SlotDev{a->obj, a->H, a->Wc, a->r0, a->c0, a->probes, a->patterns, a->patterns_t, a->positions,
                            nullptr, a->stage, nullptr, a->status};
    int grid = 0;
    size_t smem = 0;
    int rc = plan_lines_grid<T, W, true>(M, S, P, L, grid, smem);
    if (rc) return rc;
    if (!P.slot_local || !P.p4_staged || !P.resident) return kBatchedNoFit;
    // no SM pairing here: with three slot barriers per step the paired
    // anti-phase start measured slower (config 5: 18.80-18.94 vs 18.42-18.45
    // ms per sweep unpaired); PTY_BATCH_SLOT_PAIR=1 restores it
    if (!env_int("PTY_BATCH_SLOT_PAIR", 0)) {
        P.pair = 0;
        P.pair_offset = 0;
    }
    if (cudaMemsetAsync(L.barrier, 0, sizeof(unsigned int), st) != cudaSuccess) return PTY_ERR_CUDA;
    if (cudaMemsetAsync(L.slot_bar, 0, (size_t)S * 32 * sizeof(unsigned int), st) != cudaSuccess) return PTY_ERR_CUDA;
    if (cudaMemsetAsync(L.sm_pair, 0, (8 + 256) * sizeof(unsigned int), st) != cudaSuccess) return PTY_ERR_CUDA;
    batched_steptab_kernel<<<(S * steps + 255) / 256, 256, 0, st>>>(L.steptab, S, steps, a->batch + io.off, io.cnt,
                                                                    a->positions, a->r0, a->c0, a->H, a->Wc, W,
                                                                    a->status);
    // debug timeline (PTY_TIMELINE=<steps>), as in run_sweep_lines
    const int tl_steps = std::min(env_int("PTY_TIMELINE", 0), steps);
    unsigned long long* tl = nullptr;
    if (tl_steps > 0) {
        if (cudaMalloc(&tl, (size_t)tl_steps * 9 * grid * sizeof(unsigned long long)) != cudaSuccess) return PTY_ERR_CUDA;
        P.timeline = tl;
        P.timeline_steps = tl_steps;
    }
    void* args[] = {&P};
    const bool win = l2_window_set(st, L.scratch, (size_t)S * M * W * W * sizeof(cplx<T>) + (size_t)S * W * W * sizeof(T));
    const cudaError_t e = cudaLaunchCooperativeKernel((const void*)sweep_kernel<T, W, false, true>, dim3(grid),
                                                      dim3(kSweepThreads), args, smem, st);
    if (win) l2_window_clear(st);
    if (e != cudaSuccess) return PTY_ERR_CUDA;
    if (tl) {
        g_timeline.assign((size_t)tl_steps * 9 * grid, 0ull);
        cudaMemcpyAsync(g_timeline.data(), tl, g_timeline.size() * sizeof(unsigned long long), cudaMemcpyDeviceToHost, st);
        cudaStreamSynchronize(st);
        cudaFree(tl);
        g_timeline_grid = grid;
    }
    count(2);
    return last_status();
}

}  // namespace pty
