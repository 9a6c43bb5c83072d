// pty_batched_host.cuh -- host side of the batched extension: workspace
// layout, tile choice and the kernel sequence of pty_batch_contrib /
// pty_batch_apply.  Instantiated per (dtype, window) in pty_batch_*.cu.
#pragma once
#include "pty_batched.cuh"
#include "pty_host.cuh"
#include "pty_sweep_host.cuh"

namespace pty {

// the contribution pass on the line-task sweep kernel (pty_sweep_host.cuh),
// instantiated in the pty_sweep_*.cu units
template <typename T, int W> int run_sweep_batched(const BatchedSweepIO& io, cudaStream_t st);
template <typename T, int W> int sweep_batched_fits(int M, int S);

// Which contribution pass runs (PTY_BATCH_FUSED=0 forces the five-kernel
// chain): the line-task flavour when the sweep kernel runs slot-local with
// staged row blocks for this (dtype, W, M) -- S positions in flight, scratch
// L2-resident, one object-numerator plane per position.
template <typename T, int W> inline int fused_slots(int M, int chunk) {
    if (!env_int("PTY_BATCH_FUSED", 1) || M > 4) return 0;
    const int S = std::min(batched_max_slots<W>(), chunk);
    return sweep_batched_fits<T, W>(M, S) ? S : 0;
}

struct BatchLayout {
    int* anchors;
    void *scratch, *onum, *totT, *pp, *pp_part, *omax_part, *tmax_part, *pgroup, *tile_max, *upd;
    void* sweep_ws;                    // line-task flavour: the sweep kernel's workspace
    size_t sweep_ws_bytes;
    size_t bytes;
};

struct BatchShape {
    int nRT, G, ntiles, chunk;
};

// Positions per chunk (PTY_BATCH_CHUNK overrides).  Default: the whole batch,
// capped by a device-memory budget for the per-position scratch and object
// numerators (2 M W^2 complex each, PTY_BATCH_BUDGET_MB, default 8 GB) and by
// the gather kernel's shared-memory position list (12 bytes per position), so
// a large batch_size runs in chunks instead of failing.
inline int batch_chunk(int b, size_t per_pos_bytes = 0) {
    const int c = env_int("PTY_BATCH_CHUNK", 0);
    if (c > 0) return std::min(c, b);
    int chunk = b;
    if (per_pos_bytes > 0) {
        const size_t budget = (size_t)std::max(1, env_int("PTY_BATCH_BUDGET_MB", 8192)) << 20;
        chunk = (int)std::max<size_t>(1, std::min<size_t>((size_t)chunk, budget / per_pos_bytes));
    }
    const size_t smem = max_dyn_smem();
    if (smem > 1024) chunk = std::min(chunk, (int)((smem - 1024) / (3 * sizeof(int))));
    return std::max(1, chunk);
}
// bk_obj_gather's shared memory: position list + anchors (int + int2 each)
inline size_t gather_smem(int chunk) { return (size_t)((chunk + 1) & ~1) * sizeof(int) + (size_t)chunk * sizeof(int2); }
template <typename T> inline size_t batch_pos_bytes(int W, int M) { return (size_t)2 * M * W * W * sizeof(cplx<T>); }

template <int W> inline int k4_groups(int chunk) {
    const int g = env_int("PTY_K4_GROUPS", 0);
    if (g > 0) return std::min(g, chunk);
    const int want = 24 * sm_count();                         // K4 team tasks (x modes) in flight
    return std::max(1, std::min(chunk, (want + W / 4 - 1) / (W / 4)));
}

inline BatchShape batch_shape(int W, int b, int H, int Wc, int G, int chunk) {
    BatchShape s;
    s.chunk = chunk;
    s.nRT = W / 4;                                            // pp_part: 4-row tiles
    s.G = G;
    s.ntiles = ((H + kObjTile - 1) / kObjTile) * ((Wc + kObjTile - 1) / kObjTile);
    return s;
}

template <typename T>
inline BatchLayout carve_batch(void* ws, int W, int M, int b, const BatchShape& sh, int H, int Wc, bool upd,
                               int fused_S = 0) {
    Carver c(ws);
    BatchLayout L{};
    const size_t WW = (size_t)W * W;
    const size_t per = fused_S ? 0 : (size_t)sh.chunk;       // five-kernel chain only
    L.anchors = c.take<int>((size_t)b * 2 * sizeof(int));
    L.scratch = c.take<void>(per * M * WW * sizeof(cplx<T>));
    L.onum = c.take<void>((size_t)sh.chunk * (fused_S ? 1 : M) * WW * sizeof(cplx<T>));
    L.totT = c.take<void>(per * WW * sizeof(T));
    L.pp = c.take<void>(WW * sizeof(T));
    L.pp_part = c.take<void>((size_t)sh.nRT * sizeof(T));
    L.omax_part = c.take<void>(per * (W / 4) * sizeof(T));
    L.tmax_part = c.take<void>(per * W * sizeof(T));
    L.pgroup = c.take<void>((size_t)sh.G * (2 * M + 1) * WW * sizeof(T));
    L.sweep_ws_bytes = fused_S ? sweep_batched_workspace<T>(W, M, fused_S, sh.chunk) : 0;
    L.sweep_ws = c.take<void>(L.sweep_ws_bytes);
    L.tile_max = c.take<void>((size_t)sh.ntiles * sizeof(T));
    L.upd = upd ? c.take<void>((size_t)H * Wc * sizeof(cplx<T>)) : nullptr;
    L.bytes = c.off;
    return L;
}

// chunking, groups and contribution flavour of a batch (the same answer for
// the workspace query and the run)
template <typename T, int W>
BatchShape batch_plan(int M, int b, int H, int Wc, int& fused_S) {
    const int chunk_f = batch_chunk(b, (size_t)W * W * sizeof(cplx<T>));
    fused_S = fused_slots<T, W>(M, chunk_f);
    const int chunk = fused_S ? chunk_f : batch_chunk(b, batch_pos_bytes<T>(W, M));
    return batch_shape(W, b, H, Wc, fused_S ? fused_S : k4_groups<W>(chunk), chunk);
}

template <typename T, int W>
int fill_batch(const PtyBatchArgs* a, BatchDev& P, BatchShape& sh, cudaStream_t st, BatchLayout* Lout = nullptr,
               int* fused_out = nullptr) {
    const int M = a->modes, b = a->n_batch;
    int fused_S = 0;
    sh = batch_plan<T, W>(M, b, a->H, a->Wc, fused_S);
    const bool upd = a->sense == PTY_SENSE_XCORR_A;
    BatchLayout L = carve_batch<T>(a->workspace, W, M, b, sh, a->H, a->Wc, upd, fused_S);
    if (Lout) *Lout = L;
    if (fused_out) *fused_out = fused_S;
    if (!a->workspace || a->workspace_bytes < (int64_t)L.bytes) return PTY_ERR_ARGUMENT;
    P = BatchDev{};
    P.W = W; P.M = M; P.N = a->n_positions; P.b = b;
    P.TR = 4; P.lgTR = 2; P.nRT = sh.nRT; P.G = sh.G;
    P.obj = a->obj; P.H = a->H; P.Wc = a->Wc; P.r0 = a->r0; P.c0 = a->c0;
    P.probes = a->probes; P.patterns = a->patterns; P.patternsT = a->patterns_t; P.positions = a->positions;
    P.batch = a->batch; P.visit0 = a->visit0;
    P.alpha_o = a->alpha_obj; P.alpha_p = a->alpha_probe; P.beta = a->beta; P.gamma = a->gamma;
    P.eps_rel = a->epsilon_rel;
    P.update_probe = a->update_probe; P.track_mod = a->track_modulus; P.sense = a->sense;
    P.stage = a->stage; P.obj_acc = a->obj_acc; P.probe_acc = a->probe_acc;
    P.err_part = a->err_part; P.status = a->status;
    P.anchors = L.anchors; P.scratch = L.scratch; P.onum = L.onum; P.totT = L.totT; P.pp = L.pp;
    P.onum_planes = fused_S ? 1 : M;
    P.pp_part = L.pp_part; P.omax_part = L.omax_part; P.tmax_part = L.tmax_part; P.pgroup = L.pgroup;
    P.tile_max = L.tile_max; P.upd = L.upd;
    P.twiddles = twiddles<T, W>(st);
    if (!P.twiddles) return PTY_ERR_CUDA;
    return PTY_OK;
}

template <typename K> inline int set_smem(K kern, size_t bytes) {
    return cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes) == cudaSuccess
               ? PTY_OK : PTY_ERR_CUDA;
}

// persistent grid: every resident CTA slot, capped by the task count
template <typename K> inline int persistent_grid(K kern, int threads, size_t smem, long tasks_ctas) {
    int per_sm = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, threads, smem);
    const long cap = (long)std::max(1, per_sm) * sm_count();
    return (int)std::max(1L, std::min(cap, tasks_ctas));
}

template <typename T, int W>
int run_batch_contrib_fused(const PtyBatchArgs* a, BatchDev& P, const BatchShape& sh, const BatchLayout& L, int S,
                            cudaStream_t st) {
    const int M = a->modes, b = a->n_batch;
    const size_t s_gather = gather_smem(sh.chunk);
    if (s_gather > max_dyn_smem()) return PTY_ERR_ARGUMENT;
    int rc = set_smem(bk_obj_gather<T, W, true>, s_gather);
    if (rc) return rc;
    const size_t HW = (size_t)a->H * a->Wc, WW = (size_t)W * W;
    cudaMemsetAsync(a->obj_acc, 0, 3 * HW * sizeof(T), st);
    cudaMemsetAsync(a->probe_acc, 0, (size_t)(2 * M + 1) * WW * sizeof(T), st);
    cudaMemsetAsync(L.pgroup, 0, (size_t)S * (2 * M + 1) * WW * sizeof(T), st);
    bk_probe_power<T, W><<<std::max(sh.nRT, (b + kBatThreads - 1) / kBatThreads), kBatThreads, 0, st>>>(P);
    int launches = 1;
    for (int off = 0; off < b; off += sh.chunk) {   // the batch in chunks, in order
        BatchedSweepIO io{a, off, std::min(sh.chunk, b - off), S, L.onum, L.pgroup, L.sweep_ws, L.sweep_ws_bytes};
        rc = run_sweep_batched<T, W>(io, st);
        if (rc) return rc == kBatchedNoFit ? PTY_ERR_ARGUMENT : rc;
        BatchDev Q = P;
        Q.b = io.cnt;
        Q.batch = P.batch + off;
        Q.anchors = P.anchors + 2 * off;
        Q.visit0 = P.visit0 + off;
        bk_obj_gather<T, W, true><<<sh.ntiles, 256, s_gather, st>>>(Q);
        launches += 1;
    }
    P.G = S;
    bk_probe_reduce<T, W><<<std::min<size_t>(4096, ((2 * M + 1) * WW + 255) / 256), 256, 0, st>>>(P);
    count(launches + 1);
    return last_status();
}

template <typename T, int W>
int run_batch_contrib(const PtyBatchArgs* a, cudaStream_t st) {
    BatchDev P;
    BatchShape sh;
    BatchLayout L;
    int fused_S = 0;
    int rc = fill_batch<T, W>(a, P, sh, st, &L, &fused_S);
    if (rc) return rc;
    if (!a->patterns_t) return PTY_ERR_ARGUMENT;
    if (fused_S) return run_batch_contrib_fused<T, W>(a, P, sh, L, fused_S, st);
    const int M = a->modes, b = a->n_batch;
    constexpr int B = Shape<W>::B, TEAM = 4 * B, NTEAM = kLineThreads / TEAM, XS = xch_size<W>();
    constexpr int LS4 = team_line_stride<W>();
    using C = cplx<T>;
    const size_t s_k1 = W * sizeof(C) + (kLineThreads / B) * XS * sizeof(C) + NTEAM * W * 5 * sizeof(C) + 64 * sizeof(T);
    const size_t s_k23 = W * sizeof(C) + (kLineThreads / B) * XS * sizeof(C);
    const size_t s_k4 = W * sizeof(C) + 4 * LS4 * sizeof(C) + 4 * W * sizeof(C) + 4 * W * sizeof(T);
    const size_t s_gather = gather_smem(sh.chunk);
    if (s_gather > max_dyn_smem() || s_k4 > max_dyn_smem()) return PTY_ERR_ARGUMENT;
    if ((rc = set_smem(bk_rows_fwd<T, W>, s_k1)) || (rc = set_smem(bk_cols_fwd<T, W>, s_k23)) ||
        (rc = set_smem(bk_cols_mod<T, W>, s_k23)) || (rc = set_smem(bk_rows_inv<T, W>, s_k4)) ||
        (rc = set_smem(bk_obj_gather<T, W>, s_gather)))
        return rc;
    const size_t HW = (size_t)a->H * a->Wc, WW = (size_t)W * W;
    cudaMemsetAsync(a->obj_acc, 0, 3 * HW * sizeof(T), st);
    cudaMemsetAsync(a->probe_acc, 0, (size_t)(2 * M + 1) * WW * sizeof(T), st);
    bk_probe_power<T, W><<<std::max(sh.nRT, (b + kBatThreads - 1) / kBatThreads), kBatThreads, 0, st>>>(P);
    int launches = 1;
    for (int off = 0; off < b; off += sh.chunk) {   // the batch in chunks, in order
        BatchDev Q = P;
        Q.b = std::min(sh.chunk, b - off);
        Q.batch = P.batch + off;
        Q.anchors = P.anchors + 2 * off;
        Q.visit0 = P.visit0 + off;
        Q.accumulate = off > 0;
        Q.G = std::min(sh.G, Q.b);
        const long t1 = (long)Q.b * M * (W / 4), t23 = (long)Q.b * W;
        bk_rows_fwd<T, W><<<persistent_grid(bk_rows_fwd<T, W>, kLineThreads, s_k1, (t1 + NTEAM - 1) / NTEAM),
                            kLineThreads, s_k1, st>>>(Q);
        bk_cols_fwd<T, W><<<persistent_grid(bk_cols_fwd<T, W>, kLineThreads, s_k23, (t23 * B + kLineThreads - 1) / kLineThreads),
                            kLineThreads, s_k23, st>>>(Q);
        bk_cols_mod<T, W><<<persistent_grid(bk_cols_mod<T, W>, kLineThreads, s_k23, (t23 * B + kLineThreads - 1) / kLineThreads),
                            kLineThreads, s_k23, st>>>(Q);
        // a short last chunk has fewer groups: the missing groups' partials
        // keep their earlier values (bk_probe_reduce sums P.G groups)
        bk_rows_inv<T, W><<<persistent_grid(bk_rows_inv<T, W>, TEAM, s_k4, (long)(W / 4) * M * Q.G), TEAM, s_k4, st>>>(Q);
        bk_obj_gather<T, W><<<sh.ntiles, 256, s_gather, st>>>(Q);
        launches += 5;
    }
    P.G = std::min(sh.G, b);
    bk_probe_reduce<T, W><<<std::min<size_t>(4096, ((2 * M + 1) * WW + 255) / 256), 256, 0, st>>>(P);
    count(launches + 1);
    return last_status();
}

template <typename T, int W>
int run_batch_apply(const PtyBatchArgs* a, cudaStream_t st) {
    BatchDev P;
    BatchShape sh;
    int rc = fill_batch<T, W>(a, P, sh, st);
    if (rc) return rc;
    const size_t HW = (size_t)a->H * a->Wc, WW = (size_t)W * W;
    bk_obj_tile_max<T, W><<<sh.ntiles, 256, 0, st>>>(P);
    bk_obj_apply<T, W><<<(unsigned)std::min<size_t>(8 * sm_count(), (HW + 255) / 256), 256, 0, st>>>(P, sh.ntiles);
    int n = 2;
    if (a->update_probe) {
        bk_probe_apply<T, W><<<(unsigned)std::min<size_t>(2 * sm_count(), (WW + 255) / 256), 256, 0, st>>>(P);
        ++n;
    }
    if (a->sense == PTY_SENSE_XCORR_A) {
        bk_stage_after<T, W><<<a->n_batch * sh.nRT, 256, 0, st>>>(P);
        ++n;
    }
    count(n);
    return last_status();
}

template <typename T, int W>
int64_t batch_workspace(int M, int b, int H, int Wc, bool upd) {
    int fused_S = 0;
    BatchShape sh = batch_plan<T, W>(M, b, H, Wc, fused_S);
    return (int64_t)carve_batch<T>(nullptr, W, M, b, sh, H, Wc, upd, fused_S).bytes;
}

}  // namespace pty
