// pty_batched.cuh -- batched (semi-parallel) rPIE: the extension the reference
// does not have, stated on the CPU in oracle/batched.py.  Every
// position of a batch sees the batch-start object and probes; their object and
// probe numerators/denominators are accumulated and applied once per batch.
// Batch size 1 reproduces the reference sweep (engine.py:173-243).
//
// Throughput design (no grid barrier, no cooperative launch): many small CTAs
// per SM so load latency of one CTA overlaps the DFTs of another.
//   bk_probe_power : pp = sum_m |P_m|^2 map and its max (engine.py:129-132)
//   bk_rows_fwd    : exit waves, row DFTs -> scratch[k]; max|o_k|^2 partials
//   bk_cols_fwd    : column DFTs -> total^T and max(total) partials (Psi is
//                    not written back: one scratch write pass saved)
//   bk_cols_mod    : column DFTs recomputed, modulus constraint, error terms,
//                    inverse column DFTs
//   bk_rows_inv    : inverse row DFTs -> psi'; object numerator per position
//                    (onum[k]); probe numerator/denominator summed over a fixed
//                    group of positions per CTA (deterministic)
//   bk_probe_reduce: groups -> probe accumulator (fixed order)
//   bk_obj_gather  : owner-computes canvas tiles: object numerator/denominator
//                    summed over the covering positions in batch order
//   -- accumulators may be all-reduced across ranks here (NCCL) --
//   bk_obj_tile_max, bk_obj_apply, bk_probe_apply, bk_stage_after
#pragma once
#include "pty_tasks.cuh"

namespace pty {

constexpr int kBatThreads = 128;
#ifndef PTY_GATHER_U
#define PTY_GATHER_U 1          // covering positions per round in the one-plane gather (1 / 2 / 4 / 8: 18.86 / 18.92 / 19.37 / 21.13 ms per config-5 sweep)
#endif
constexpr int kObjTile = 32;           // owner tile edge (canvas pixels)
constexpr int kMaxBatchModes = 8;

struct BatchDev {
    int W, M, N, b;                    // window, modes, positions in dataset, positions in batch
    int TR, TC, lgTR, lgTC, nRT, nCT, G;
    int accumulate;                    // chunks after the first add into pgroup
    void* obj;
    int H, Wc, r0, c0;
    void* probes;
    const void* patterns;
    const void* patternsT;             // [N][W][W] real, transposed (I^T[j][kc][u])
    const double* positions;
    const int* batch;                  // [b] position ids
    int visit0;                        // index of batch[0] in the sweep's visit order
    double alpha_o, alpha_p, beta, gamma, eps_rel;
    int update_probe, track_mod, sense;
    void* stage;                       // [N][2][W][W] complex or null
    void* obj_acc;                     // [H][3][Wc] real: num.re, num.im, den (planes interleaved per row)
    void* probe_acc;                   // [2M+1][W][W] real: pnum (re, im) per mode, pden
    double* err_part;                  // [N][W][3] by visit rank (visit0 + k)
    int* status;
    // workspace
    int* anchors;                      // [b][2]
    void* scratch;                     // [b][M][W][W] complex
    void* onum;                        // [b][onum_planes][W][W] complex: object numerators
    int onum_planes;                   // M (per-mode, bk_rows_inv) or 1 (mode sum, the line-task flavour)
    void* pp;                          // [W][W] real (probe power)
    void* pp_part;                     // [nRT] real
    void* omax_part;                   // [b][W/4] real (per row quad)
    void* tmax_part;                   // [b][W] real (per column)
    void* totT;                        // [b][W][W] real: total^T
    void* pgroup;                      // [G][2M+1][W][W] real
    void* tile_max;                    // [ntiles] real
    void* upd;                         // [H][Wc] complex (posref staging only) or null
    const void* twiddles;
};

template <typename T>
__device__ __forceinline__ T bk_max_of(const T* p, int n) {
    T m = T(0);
    for (int i = 0; i < n; ++i) m = fmax(m, p[i]);
    return m;
}

// pp map and per-row-tile maxima; anchors of the batch and bounds check
template <typename T, int W>
__global__ void __launch_bounds__(kBatThreads) bk_probe_power(const __grid_constant__ BatchDev P) {
    using C = cplx<T>;
    __shared__ T red[32];
    const C* probes = reinterpret_cast<const C*>(P.probes);
    T* pp = reinterpret_cast<T*>(P.pp);
    const size_t WW = (size_t)W * W;
    const int rt = blockIdx.x;
    if (rt < P.nRT) {
        T mx = T(0);
        for (int i = threadIdx.x; i < P.TR * W; i += blockDim.x) {
            const size_t off = (size_t)rt * P.TR * W + i;
            T v = T(0);
            for (int m = 0; m < P.M; ++m) v += norm2(probes[m * WW + off]);
            pp[off] = v;
            mx = fmax(mx, v);
        }
        mx = block_max(mx, red);
        if (threadIdx.x == 0) reinterpret_cast<T*>(P.pp_part)[rt] = mx;
    }
    for (int k = blockIdx.x * blockDim.x + threadIdx.x; k < P.b; k += gridDim.x * blockDim.x) {
        const int j = P.batch[k];
        const int ar = (int)rint(P.positions[2 * j + 1]) - P.r0;
        const int ac = (int)rint(P.positions[2 * j]) - P.c0;
        P.anchors[2 * k] = ar;
        P.anchors[2 * k + 1] = ac;
        if (ar < 0 || ac < 0 || ar + W > P.H || ac + W > P.Wc) atomicOr(P.status, PTY_ERR_BOUNDS);
    }
}

// ---------------------------------------------------------------------------
// Line-task kernels.  A "group" is B threads transforming one line with the
// fused-I/O group_fft; a "team" is 4 groups that own 4 consecutive rows, so a
// transposed scratch access moves 4 consecutive complex values (one 32-byte
// sector) per column.  Scratch layout after the row pass: [k][m][kc][r]
// (row-DFT output transposed), so column passes read contiguous lines.
// CTAs are persistent over tasks; no CTA-wide barrier inside a task.

constexpr int kLineThreads = 128;

// K1: exit waves C * P_m * o_j and row DFTs (engine.py:113, fields.py:81).
// Team task (k, m, row quad); output transposed into scratch.
template <typename T, int W>
#ifndef PTY_BK_ROWS_MINB
#define PTY_BK_ROWS_MINB 4      // 128 registers: measured best (6 -> 85 registers spills: 242 K vs 294 K pos/s)
#endif
__global__ void __launch_bounds__(kLineThreads, PTY_BK_ROWS_MINB) bk_rows_fwd(const __grid_constant__ BatchDev P) {
    using C = cplx<T>;
    constexpr int B = Shape<W>::B, TEAM = 4 * B, NTEAM = kLineThreads / TEAM, XS = xch_size<W>();
    extern __shared__ __align__(16) unsigned char smem_raw[];
    C* tw = reinterpret_cast<C*>(smem_raw);
    C* xch_all = tw + W;
    C* tt_all = xch_all + (kLineThreads / B) * XS;
    T* red = reinterpret_cast<T*>(tt_all + NTEAM * W * 5);
    load_twiddles<T, W>(tw, reinterpret_cast<const C*>(P.twiddles));
    __syncthreads();
    if (*(volatile const int*)P.status) return;
    const int team = threadIdx.x / TEAM, tl = threadIdx.x % TEAM, gi = tl / B, b = tl % B;
    const unsigned gmask = group_mask<W>();
    C* xch = xch_all + (threadIdx.x / B) * XS;
    C* tt = tt_all + team * W * 5;
    const int M = P.M, nq = W / 4, ntasks = P.b * M * nq;
    const size_t WW = (size_t)W * W;
    const C* obj = reinterpret_cast<const C*>(P.obj);
    const C* probes = reinterpret_cast<const C*>(P.probes);
    C* scratch = reinterpret_cast<C*>(P.scratch);
    for (int task = blockIdx.x * NTEAM + team; task < ntasks; task += gridDim.x * NTEAM) {
        const int k = task / (M * nq), rem = task % (M * nq), m = rem / nq, rq = rem % nq;
        const int j = P.batch[k];
        C* stg = (P.sense == PTY_SENSE_XCORR_A && m == 0) ? reinterpret_cast<C*>(P.stage) + (size_t)j * 2 * WW : nullptr;
        const T om = task_row_fwd<T, W>(tw, xch, tt, red + team * 4, team, tl, gi, b, gmask, obj, P.Wc,
                                        P.anchors[2 * k], P.anchors[2 * k + 1], probes, m, rq,
                                        scratch + (size_t)k * M * WW, stg);
        if (m == 0 && tl == 0) reinterpret_cast<T*>(P.omax_part)[(size_t)k * nq + rq] = om;
    }
}

// K2: column DFTs of every mode, total^T and max(total) partial per column
// (engine.py:114-117); Psi stays on chip (K3 recomputes it: the grid-wide
// max(total) of the position must be known before the modulus scale, and a
// second DFT costs less than a scratch write + read).  Group task (k, kc).
template <typename T, int W>
__global__ void __launch_bounds__(kLineThreads) bk_cols_fwd(const __grid_constant__ BatchDev P) {
    using C = cplx<T>;
    constexpr int A = Shape<W>::A, B = Shape<W>::B, NG = kLineThreads / B, XS = xch_size<W>();
    extern __shared__ __align__(16) unsigned char smem_raw[];
    C* tw = reinterpret_cast<C*>(smem_raw);
    C* xch = tw + W + (threadIdx.x / B) * XS;
    load_twiddles<T, W>(tw, reinterpret_cast<const C*>(P.twiddles));
    __syncthreads();
    if (*(volatile const int*)P.status) return;
    const int grp = threadIdx.x / B, b = threadIdx.x % B;
    const unsigned gmask = group_mask<W>();
    const int M = P.M;
    const size_t WW = (size_t)W * W;
    const T invW2 = T(1) / (T(W) * T(W));
    C* scratch = reinterpret_cast<C*>(P.scratch);
    T* totT = reinterpret_cast<T*>(P.totT);
    for (int task = blockIdx.x * NG + grp; task < P.b * W; task += gridDim.x * NG) {
        const int k = task / W, kc = task % W;
        const T tm = task_col_fwd<T, W, false, false>(tw, xch, b, gmask, scratch + (size_t)k * M * WW, M, kc, totT + (size_t)k * WW);
        if (b == 0) reinterpret_cast<T*>(P.tmax_part)[(size_t)k * W + kc] = tm;
    }
}

// K3: forward column DFTs recomputed from the row-DFT output, modulus constraint scale = sqrt(I)/sqrt(total + eps) (engine.py:117-118),
// error terms (engine.py:198-214), inverse column DFTs.  Group task (k, kc).
template <typename T, int W>
__global__ void __launch_bounds__(kLineThreads) bk_cols_mod(const __grid_constant__ BatchDev P) {
    using C = cplx<T>;
    constexpr int A = Shape<W>::A, B = Shape<W>::B, NG = kLineThreads / B, XS = xch_size<W>();
    extern __shared__ __align__(16) unsigned char smem_raw[];
    C* tw = reinterpret_cast<C*>(smem_raw);
    C* xch = tw + W + (threadIdx.x / B) * XS;
    load_twiddles<T, W>(tw, reinterpret_cast<const C*>(P.twiddles));
    __syncthreads();
    if (*(volatile const int*)P.status) return;
    const int grp = threadIdx.x / B, b = threadIdx.x % B;
    const unsigned gmask = group_mask<W>();
    const int M = P.M;
    const size_t WW = (size_t)W * W;
    const T invW2 = T(1) / (T(W) * T(W));
    C* scratch = reinterpret_cast<C*>(P.scratch);
    const T* totT = reinterpret_cast<const T*>(P.totT);
    for (int task = blockIdx.x * NG + grp; task < P.b * W; task += gridDim.x * NG) {
        const int k = task / W, kc = task % W, j = P.batch[k];
        C* stg = P.sense == PTY_SENSE_XCORR_B ? reinterpret_cast<C*>(P.stage) + (size_t)j * 2 * WW : nullptr;
        task_col_mod<T, W, false, true>(tw, xch, b, gmask, scratch + (size_t)k * M * WW, M, kc, totT + (size_t)k * WW,
                           reinterpret_cast<const T*>(P.tmax_part) + (size_t)k * W,
                           reinterpret_cast<const T*>(P.patternsT) + (size_t)j * WW, T(P.eps_rel), P.track_mod, stg,
                           P.err_part + ((size_t)(P.visit0 + k) * W + kc) * 3);
    }
}

// K4: inverse row DFTs and the update terms.  Team task (row quad, mode m,
// position group g): the team walks positions k = g, g+G, ... of the chunk in
// order, writes the per-mode object numerator onum[k][m] and keeps mode m's
// probe numerator (and, for m = 0, the probe denominator) in shared memory --
// a fixed-order, atomic-free reduction.
template <typename T, int W>
__global__ void __launch_bounds__(64, 2 * PTY_BK_ROWS_MINB) bk_rows_inv(const __grid_constant__ BatchDev P) {
    using C = cplx<T>;
    constexpr int A = Shape<W>::A, B = Shape<W>::B, TEAM = 4 * B, LS4 = team_line_stride<W>();
    extern __shared__ __align__(16) unsigned char smem_raw[];
    const int M = P.M;
    C* tw = reinterpret_cast<C*>(smem_raw);
    C* lines = tw + W;                                         // [4][LS4]
    C* pnum = lines + 4 * LS4;                                 // [4][W] (mode m)
    T* pden = reinterpret_cast<T*>(pnum + 4 * W);             // [4][W]
    load_twiddles<T, W>(tw, reinterpret_cast<const C*>(P.twiddles));
    __syncthreads();
    if (*(volatile const int*)P.status) return;
    const int tl = threadIdx.x, gi = tl / B, b = tl % B;
    const unsigned gmask = group_mask<W>();
    const int nq = W / 4;
    const size_t WW = (size_t)W * W;
    const T invW2 = T(1) / (T(W) * T(W));
    const T alpha_p = T(P.alpha_p), beta = T(P.beta);
    const C* obj = reinterpret_cast<const C*>(P.obj);
    const C* probes = reinterpret_cast<const C*>(P.probes);
    const C* scratch = reinterpret_cast<const C*>(P.scratch);
    C* myline = lines + gi * LS4;
    for (int task = blockIdx.x; task < nq * M * P.G; task += gridDim.x) {
        const int rq = task % nq, m = (task / nq) % M, g = task / (nq * M), r = 4 * rq + gi;
        T* pg = reinterpret_cast<T*>(P.pgroup) + (size_t)g * (2 * M + 1) * WW + (size_t)4 * rq * W;
        const bool den_owner = P.update_probe && m == 0;
        for (int i = tl; i < 4 * W; i += TEAM) {
            pnum[i] = P.accumulate ? C{pg[(size_t)(2 * m) * WW + i], pg[(size_t)(2 * m + 1) * WW + i]} : C{T(0), T(0)};
            if (den_owner) pden[i] = P.accumulate ? pg[(size_t)(2 * M) * WW + i] : T(0);
        }
        C pv[A];                                               // P_m(r, c) for my output columns
        const C* prow = probes + m * WW + (size_t)r * W;
#pragma unroll
        for (int q = 0; q < A; ++q) pv[q] = prow[b + B * (q / B) + A * (q % B)];
        int arn = g < P.b ? P.anchors[2 * g] : 0, acn = g < P.b ? P.anchors[2 * g + 1] : 0;
        for (int k = g; k < P.b; k += P.G) {
            const int ar = arn, ac = acn;                      // the next position's anchors load during this one
            if (k + P.G < P.b) {
                arn = P.anchors[2 * (k + P.G)];
                acn = P.anchors[2 * (k + P.G) + 1];
            }
            const T* op = reinterpret_cast<const T*>(P.omax_part) + (size_t)k * nq;
            T omax = T(0);
            for (int q = b; q < nq; q += B) omax = fmax(omax, op[q]);
            omax = group_max<B>(omax);
            if (P.update_probe && omax == T(0)) {              // engine.py:145-147
                if (tl == 0) atomicOr(P.status, PTY_ERR_OBJECT_ZERO);
                continue;
            }
            const C* src = scratch + ((size_t)k * M + m) * WW + 4 * rq;
            const C* orow = obj + (size_t)(ar + r) * P.Wc + ac;
            team_sync<TEAM>(0);                                // previous FFT done with `lines`
            for (int e = tl; e < 4 * W; e += TEAM) lines[(e & 3) * LS4 + pad<W>(e >> 2)] = src[(size_t)(e >> 2) * W + (e & 3)];
            C ov[A];
#pragma unroll
            for (int q = 0; q < A; ++q) ov[q] = orow[b + B * (q / B) + A * (q % B)];
            team_sync<TEAM>(0);
            C* on = reinterpret_cast<C*>(P.onum) + ((size_t)k * M + m) * WW + (size_t)r * W;
            group_fft<T, W, true>(
                myline, tw, b, gmask, [&](int n, int) { return myline[pad<W>(n)]; },
                [&](int c, int slot, C X) {
                    const C o = ov[slot];
                    const C d = scale(X, checker<T>(r, c) * invW2) - pv[slot] * o;
                    on[c] = mulc(d, pv[slot]);                             // engine.py:130-131
                    if (P.update_probe) {
                        C& acc = pnum[gi * W + c];
                        acc = acc + mulc(scale(d, alpha_p), o);            // engine.py:150
                        if (m == 0) pden[gi * W + c] += beta * omax + (T(1) - beta) * norm2(o);   // engine.py:148
                    }
                });
        }
        team_sync<TEAM>(0);
        for (int i = tl; i < 4 * W; i += TEAM) {
            pg[(size_t)(2 * m) * WW + i] = pnum[i].re;
            pg[(size_t)(2 * m + 1) * WW + i] = pnum[i].im;
            if (den_owner) pg[(size_t)(2 * M) * WW + i] = pden[i];
        }
        team_sync<TEAM>(0);
    }
}

// groups -> probe accumulator, fixed order g = 0..G-1
template <typename T, int W>
__global__ void bk_probe_reduce(const __grid_constant__ BatchDev P) {
    const size_t WW = (size_t)W * W, n = (size_t)(2 * P.M + 1) * WW;
    const T* pg = reinterpret_cast<const T*>(P.pgroup);
    T* acc = reinterpret_cast<T*>(P.probe_acc);
    for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
        T s = T(0);
        for (int g = 0; g < P.G; ++g) s += pg[(size_t)g * n + i];
        acc[i] = s;
    }
}

// Owner-computes object accumulation: CTA = one kObjTile x kObjTile canvas tile;
// it lists the batch positions covering the tile in batch order (block scan)
// and sums their numerators and denominators (engine.py:130-136) in that order.
template <typename T, int W, bool ONE_PLANE = false>
__global__ void __launch_bounds__(256) bk_obj_gather(const __grid_constant__ BatchDev P) {
    using C = cplx<T>;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    int* list = reinterpret_cast<int*>(smem_raw);            // [b] covering positions, batch order
    int2* lanc = reinterpret_cast<int2*>(list + ((P.b + 1) & ~1));   // [b] their anchors
    __shared__ int wcount[8], total;
    const int tiles_x = (P.Wc + kObjTile - 1) / kObjTile;
    const int ty = blockIdx.x / tiles_x, tx = blockIdx.x % tiles_x;
    const int R0 = ty * kObjTile, C0 = tx * kObjTile;
    // a failed batch (bounds / zero probe) raises; never read its numerators
    if (*(volatile const int*)P.status) return;
    if (threadIdx.x == 0) total = 0;
    __syncthreads();
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    constexpr int LR = 8;                                     // list rounds whose anchor loads fly together
    for (int base0 = 0; base0 < P.b; base0 += LR * blockDim.x) {
        bool covr[LR];
        int2 anc[LR];
#pragma unroll
        for (int u = 0; u < LR; ++u) {
            const int k = base0 + u * blockDim.x + threadIdx.x;
            covr[u] = false;
            anc[u] = make_int2(0, 0);
            if (k < P.b) {
                const int ar = P.anchors[2 * k], ac = P.anchors[2 * k + 1];
                anc[u] = make_int2(ar, ac);
                covr[u] = ar < R0 + kObjTile && ar + W > R0 && ac < C0 + kObjTile && ac + W > C0;
            }
        }
#pragma unroll
        for (int u = 0; u < LR; ++u) {
            const int base = base0 + u * blockDim.x;
            if (base >= P.b) break;                           // block-uniform
            const int k = base + threadIdx.x;
            const bool cov = covr[u];
            const unsigned bal = __ballot_sync(0xffffffffu, cov);
            if (lane == 0) wcount[wid] = __popc(bal);
            __syncthreads();
            int off = total;
            for (int w = 0; w < wid; ++w) off += wcount[w];
            if (cov) {
                const int slot = off + __popc(bal & ((1u << lane) - 1u));
                list[slot] = k;
                lanc[slot] = anc[u];
            }
            __syncthreads();
            if (threadIdx.x == 0) for (int w = 0; w < (int)(blockDim.x >> 5); ++w) total += wcount[w];
            __syncthreads();
        }
    }
    if (total == 0) return;
    const T* pp = reinterpret_cast<const T*>(P.pp);
    const T peak = bk_max_of(reinterpret_cast<const T*>(P.pp_part), P.nRT);
    if (peak == T(0)) {                                       // engine.py:132-134
        if (threadIdx.x == 0) atomicOr(P.status, PTY_ERR_PROBE_ZERO);
        return;
    }
    const T gamma = T(P.gamma);
    const C* onum = reinterpret_cast<const C*>(P.onum);      // [k][onum_planes][W][W]
    T* acc = reinterpret_cast<T*>(P.obj_acc);
    const size_t HW = (size_t)P.H * P.Wc;
    const size_t WW = (size_t)W * W;
    constexpr int PX = kObjTile * kObjTile / 256;             // pixels per thread
    C num[PX];
    T den[PX];
#pragma unroll
    for (int q = 0; q < PX; ++q) { num[q] = C{T(0), T(0)}; den[q] = T(0); }
    // one numerator plane per position (the line-task pass): covering positions
    // in batch order, U at a time (their numerator and sum|P|^2 loads fly
    // together; more than one per round costs occupancy), added in list order
    auto accumulate = [&](auto u_const) {
        constexpr int U = decltype(u_const)::value;
        for (int t0 = 0; t0 < total; t0 += U) {
            C v[U][PX];
            T pw[U][PX];
            bool ok[U][PX];
#pragma unroll
            for (int u = 0; u < U; ++u) {
                const int t = t0 + u;
                const int k = t < total ? list[t] : 0;
                const int2 an = t < total ? lanc[t] : make_int2(0, 0);
#pragma unroll
                for (int q = 0; q < PX; ++q) {
                    const int p = threadIdx.x + q * 256, R = R0 + p / kObjTile, Cc = C0 + p % kObjTile;
                    const int r = R - an.x, c = Cc - an.y;
                    ok[u][q] = t < total && R < P.H && Cc < P.Wc && r >= 0 && r < W && c >= 0 && c < W;
                    if (ok[u][q]) {
                        const C* src = onum + (size_t)k * P.onum_planes * WW + (size_t)r * W + c;
                        v[u][q] = src[0];
                        pw[u][q] = pp[(size_t)r * W + c];
                    }
                }
            }
#pragma unroll
            for (int u = 0; u < U; ++u)
#pragma unroll
                for (int q = 0; q < PX; ++q)
                    if (ok[u][q]) {
                        num[q] = num[q] + v[u][q];
                        den[q] += gamma * peak + (T(1) - gamma) * pw[u][q];
                    }
        }
    };
    if constexpr (ONE_PLANE) {
        accumulate(std::integral_constant<int, PTY_GATHER_U>{});
    } else {                                                  // per-mode planes (bk_rows_inv)
        int k = list[0];
        int2 an = lanc[0];
        for (int t = 0; t < total; ++t) {
            const int kn = t + 1 < total ? list[t + 1] : k;  // the next position's entry read ahead
            const int2 ann = t + 1 < total ? lanc[t + 1] : an;
#pragma unroll
            for (int q = 0; q < PX; ++q) {
                const int p = threadIdx.x + q * 256, R = R0 + p / kObjTile, Cc = C0 + p % kObjTile;
                const int r = R - an.x, c = Cc - an.y;
                if (R < P.H && Cc < P.Wc && r >= 0 && r < W && c >= 0 && c < W) {
                    const C* src = onum + (size_t)k * P.onum_planes * WW + (size_t)r * W + c;
                    C v[kMaxBatchModes];                      // every plane's load in flight at once
#pragma unroll
                    for (int m = 0; m < kMaxBatchModes; ++m)
                        if (m < P.onum_planes) v[m] = src[(size_t)m * WW];
                    C sm = v[0];
#pragma unroll
                    for (int m = 1; m < kMaxBatchModes; ++m)
                        if (m < P.onum_planes) sm = sm + v[m];   // mode order
                    num[q] = num[q] + sm;
                    den[q] += gamma * peak + (T(1) - gamma) * pp[(size_t)r * W + c];
                }
            }
            k = kn;
            an = ann;
        }
    }
#pragma unroll
    for (int q = 0; q < PX; ++q) {
        const int p = threadIdx.x + q * 256, R = R0 + p / kObjTile, Cc = C0 + p % kObjTile;
        if (R < P.H && Cc < P.Wc) {
            const size_t o = (size_t)R * 3 * P.Wc + Cc;
            acc[o] += num[q].re;                      // chunks add in a fixed order
            acc[P.Wc + o] += num[q].im;
            acc[2 * P.Wc + o] += den[q];
        }
    }
}

// per-tile maxima of the accumulated object denominator (after any all-reduce)
template <typename T, int W>
__global__ void __launch_bounds__(256) bk_obj_tile_max(const __grid_constant__ BatchDev P) {
    __shared__ T red[32];
    const int tiles_x = (P.Wc + kObjTile - 1) / kObjTile;
    const int ty = blockIdx.x / tiles_x, tx = blockIdx.x % tiles_x;
    const T* den = reinterpret_cast<const T*>(P.obj_acc) + 2 * (size_t)P.Wc;
    T m = T(0);
    for (int p = threadIdx.x; p < kObjTile * kObjTile; p += blockDim.x) {
        const int R = ty * kObjTile + p / kObjTile, Cc = tx * kObjTile + p % kObjTile;
        if (R < P.H && Cc < P.Wc) m = fmax(m, den[(size_t)R * 3 * P.Wc + Cc]);
    }
    m = block_max(m, red);
    if (threadIdx.x == 0) reinterpret_cast<T*>(P.tile_max)[blockIdx.x] = m;
}

// o <- o + ((o + alpha num/(den + eps max den)) - o) on covered pixels
template <typename T, int W>
__global__ void __launch_bounds__(256) bk_obj_apply(const __grid_constant__ BatchDev P, int ntiles) {
    using C = cplx<T>;
    __shared__ T s_max;
    if (*(volatile const int*)P.status) return;
    if (threadIdx.x < 32) {
        T m = T(0);
        for (int i = threadIdx.x; i < ntiles; i += 32) m = fmax(m, reinterpret_cast<const T*>(P.tile_max)[i]);
        m = warp_max(m);
        if (threadIdx.x == 0) s_max = m;
    }
    __syncthreads();
    const T dmax = s_max;
    const size_t HW = (size_t)P.H * P.Wc;
    const T* acc = reinterpret_cast<const T*>(P.obj_acc);
    C* obj = reinterpret_cast<C*>(P.obj);
    C* upd = reinterpret_cast<C*>(P.upd);
    const T alpha_o = T(P.alpha_o), eps_rel = T(P.eps_rel);
    for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < HW; i += (size_t)gridDim.x * blockDim.x) {
        const size_t a = (i / P.Wc) * 3 * P.Wc + i % P.Wc;          // [R][plane][C]
        const T den = acc[a + 2 * P.Wc];
        const C o = obj[i];
        C u = o;
        if (den > T(0)) {
            u = o + divr(scale(C{acc[a], acc[a + P.Wc]}, alpha_o), den + eps_rel * dmax);
            obj[i] = o + (u - o);
        }
        if (upd) upd[i] = u;
    }
}

// P <- P + pnum / (pden + eps max pden); also the next batch's pp map is
// recomputed by bk_probe_power at the next call.
template <typename T, int W>
__global__ void __launch_bounds__(256) bk_probe_apply(const __grid_constant__ BatchDev P) {
    using C = cplx<T>;
    __shared__ T red[32];
    if (*(volatile const int*)P.status) return;
    const size_t WW = (size_t)W * W;
    const T* acc = reinterpret_cast<const T*>(P.probe_acc);
    const T* pden = acc + (size_t)(2 * P.M) * WW;
    T m = T(0);
    for (size_t i = threadIdx.x; i < WW; i += blockDim.x) m = fmax(m, pden[i]);
    m = block_max(m, red);
    const T eps = T(P.eps_rel) * m;
    C* probes = reinterpret_cast<C*>(P.probes);
    for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < WW; i += (size_t)gridDim.x * blockDim.x) {
        const T d = pden[i] + eps;
        for (int mm = 0; mm < P.M; ++mm) {
            const C q{acc[(size_t)(2 * mm) * WW + i], acc[(size_t)(2 * mm + 1) * WW + i]};
            probes[mm * WW + i] = probes[mm * WW + i] + divr(q, d);
        }
    }
}

// posref.py:66-76 for the batch: second sensor input = the updated crop before
// the paste rounding (oracle/batched.py).  CTA = (position k, row tile).
template <typename T, int W>
__global__ void bk_stage_after(const __grid_constant__ BatchDev P) {
    using C = cplx<T>;
    if (*(volatile const int*)P.status) return;        // e.g. an out-of-canvas anchor
    const int k = blockIdx.x / P.nRT, rt = blockIdx.x % P.nRT;
    const int j = P.batch[k], ar = P.anchors[2 * k], ac = P.anchors[2 * k + 1];
    const size_t WW = (size_t)W * W;
    C* stg = reinterpret_cast<C*>(P.stage) + (size_t)j * 2 * WW + WW;
    const C* upd = reinterpret_cast<const C*>(P.upd);
    for (int i = threadIdx.x; i < P.TR * W; i += blockDim.x) {
        const int rr = rt * P.TR + i / W, c = i % W;
        stg[(size_t)rr * W + c] = upd[(size_t)(ar + rr) * P.Wc + ac + c];
    }
}

}  // namespace pty
