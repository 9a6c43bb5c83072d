// pty_tasks.cuh -- the per-line task bodies shared by the reference-order
// sweep kernel (pty_sweep.cuh) and the batched kernels (pty_batched.cuh).
//
// Vocabulary: a "group" is B threads that transform one W-line with the
// fused-I/O group_fft (stage-1 loads straight from global memory, stage-2
// outputs straight into the epilogue); a "team" is 4 groups owning 4
// consecutive rows, so transposed accesses move 4 consecutive complex values
// (one 32-byte sector) per column.  Scratch layout per position:
//   [m][kc][r]  after the row pass (row-DFT output transposed), so the column
//   passes read and write contiguous lines; totT[kc][u] = total detector
//   intensity transposed.
#pragma once
#include "pty_fft.cuh"

namespace pty {

#ifdef PTY_PROBE
// debug build (-DPTY_PROBE): globaltimer stamps of CTA 0 / thread 0 inside
// the P1 and P4 task bodies, per step ([step][32]); read back with
// cudaMemcpyFromSymbol by the host (pty_probe_read)
__device__ unsigned long long pty_probe_buf[64][32];
__device__ int pty_probe_step;
__device__ __forceinline__ void probe_stamp(int k) {
    if (blockIdx.x == 0 && threadIdx.x == 0 && pty_probe_step < 64) {
        unsigned long long t;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
        pty_probe_buf[pty_probe_step][k] = t;
    }
}
#define PTY_PROBE_STAMP(k) probe_stamp(k)
#else
#define PTY_PROBE_STAMP(k)
#endif

template <int TEAM>
__device__ __forceinline__ void team_sync(int team) {
    if constexpr (TEAM <= 32) {
        const unsigned lane = threadIdx.x & 31;
        const unsigned m = TEAM == 32 ? 0xffffffffu : (((1u << TEAM) - 1u) << (lane & ~(unsigned)(TEAM - 1)));
        __syncwarp(m);
    } else {
        asm volatile("bar.sync %0, %1;" ::"r"(team + 1), "r"(TEAM) : "memory");
    }
}

// max / sum over the B lanes of a group (B divides 32)
template <int B, typename T>
__device__ __forceinline__ T group_max(T v) {
#pragma unroll
    for (int o = B / 2; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
    return v;
}
template <int B, typename T>
__device__ __forceinline__ T group_sum(T v) {
#pragma unroll
    for (int o = B / 2; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

template <int W> __device__ __forceinline__ unsigned group_mask() {
    constexpr int B = Shape<W>::B;
    const unsigned lane = threadIdx.x & 31;
    return B == 32 ? 0xffffffffu : (((1u << B) - 1u) << (lane & ~(unsigned)(B - 1)));
}

// line stride of the team lines: >= W + W/B + 1 and = 4 (mod 16) so that the
// 4-row transposed stores hit distinct banks
template <int W> __host__ __device__ constexpr int team_line_stride() {
    return ((W + W / Shape<W>::B + 1 + 11) / 16) * 16 + 4;
}

// transposed staging tile tt[kc][4]: the row slot is XOR-swizzled with
// (kc / 4) % 4 so both the column-wise writes (16 consecutive kc of one row)
// and the row-quad reads (4 consecutive kc, all rows) are bank-conflict free
__device__ __forceinline__ int tt_swz(int kc) { return (kc >> 2) & 3; }

// row stride of the team's real [4][.] accumulators: +16 words puts the two
// groups of a warp on different banks
template <int W> __host__ __device__ constexpr int acc_stride() { return W + 16; }

// output column of stage-2 slot q for group lane b
template <int W> __device__ __forceinline__ int slot_col(int b, int q) {
    constexpr int A = Shape<W>::A, B = Shape<W>::B;
    if constexpr (A < B)                       // narrow_fft256: lane (k1, d2), slot p*4 + f
        return (b >> 2) + 8 * (2 * (b & 3) + (q >> 2)) + 64 * (q & 3);
    else
        return b + B * (q / B) + A * (q % B);
}

// Line stride of the staged lines of an RT-row block: >= W + W/B + 1 (the
// padded line plus the exchange) and = 1 (mod 16) for RT = 16 (the 16 rows of
// one column land in 16 different 8-byte bank pairs: conflict-free transposes),
// = 4 (mod 16) for RT = 4 (team_line_stride).
template <int W, int RT> __host__ __device__ constexpr int block_line_stride() {
    return RT == 4 ? team_line_stride<W>() : ((W + W / Shape<W>::B + 1 + 14) / 16) * 16 + 1;
}

// Team-level max of one value per group over RT groups; red = RT shared slots of the team.
template <int W, int RT, typename T>
__device__ __forceinline__ T team_maxn(T v, T* red, int team, int gi, int b) {
    constexpr int B = Shape<W>::B, TEAM = RT * B;
    v = group_max<B>(v);
    if (b == 0) red[gi] = v;
    team_sync<TEAM>(team);
    T r = red[0];
#pragma unroll
    for (int g = 1; g < RT; ++g) r = fmax(r, red[g]);
    team_sync<TEAM>(team);
    return r;
}

// Team-level max of one value per group (4 groups); red4 = 4 shared slots of the team.
template <int W, typename T>
__device__ __forceinline__ T team_max4(T v, T* red4, int team, int gi, int b) {
    constexpr int B = Shape<W>::B, TEAM = 4 * B;
    v = group_max<B>(v);
    if (b == 0) red4[gi] = v;
    team_sync<TEAM>(team);
    const T r = fmax(fmax(red4[0], red4[1]), fmax(red4[2], red4[3]));
    team_sync<TEAM>(team);
    return r;
}

// Row pass, team task (mode m, row quad rq) of one position (engine.py:113,
// fields.py:81): exit waves C * P_m * o_j, row DFTs, output transposed into
// dst = the position's scratch.  Returns the team's max|o|^2 when m == 0
// (engine.py:145); stg_o (row-major o_j, XCORR_A sensor input) may be null.
template <typename T, int W>
__device__ __forceinline__ T task_row_fwd(const cplx<T>* tw, cplx<T>* xch, cplx<T>* tt, T* red4, int team, int tl,
                                          int gi, int b, unsigned gmask, const cplx<T>* obj, int Wc, int ar, int ac,
                                          const cplx<T>* probes, int m, int rq, cplx<T>* dst_pos, cplx<T>* stg_o) {
    using C = cplx<T>;
    constexpr int B = Shape<W>::B, TEAM = 4 * B;
    const size_t WW = (size_t)W * W;
    const int r = 4 * rq + gi;
    const C* orow = obj + (size_t)(ar + r) * Wc + ac;
    const C* prow = probes + m * WW + (size_t)r * W;
    constexpr int A = Shape<W>::A;
    C* stg = stg_o ? stg_o + (size_t)r * W : nullptr;
    // all 2A loads in flight before any use or store (a store between them
    // would serialise the loads behind it: the pointers may alias)
    C ov[A], pv[A];
#pragma unroll
    for (int a = 0; a < A; ++a) {
        ov[a] = orow[B * a + b];
        pv[a] = prow[B * a + b];
    }
    T om = T(0);
    if (m == 0) {
#pragma unroll
        for (int a = 0; a < A; ++a) {
            om = fmax(om, norm2(ov[a]));
            if (stg) stg[B * a + b] = ov[a];
        }
    }
    group_fft<T, W, false>(
        xch, tw, b, gmask, [&](int n, int a) { return scale(pv[a] * ov[a], checker<T>(r, n)); },
        [&](int kc, int, C v) { tt[kc * 4 + (gi ^ tt_swz(kc))] = v; });
    team_sync<TEAM>(team);
    C* dst = dst_pos + m * WW + 4 * rq;
#pragma unroll
    for (int i = 0; i < 4 * W / TEAM; ++i) {
        const int e = tl + i * TEAM;
        dst[(size_t)(e >> 2) * W + (e & 3)] = tt[(e >> 2) * 4 + ((e & 3) ^ tt_swz(e >> 2))];
    }
    T res = T(0);
    if (m == 0) res = team_max4<W>(om, red4, team, gi, b);
    team_sync<TEAM>(team);
    return res;
}

// Row pass, staged: team task (block blk of RT consecutive rows, ALL modes)
// of one position.  A team is RT line groups; group gi owns row r = RT*blk +
// gi.  The object row is loaded once into registers; every mode's exit wave
// C * P_m * o_j enters the line transform from registers (no staging pass)
// and the spectrum lands in the team's lines (lines[(m*RT + gi)*LS +
// pad(k)]); the block is then written transposed ([m][kc][r]) from the lines.
// With RT = 16 one column of the block is 16 consecutive rows = one 128-byte
// line of scratch, so the transposed stores are full-line writes (with RT = 4
// they were 32-byte pieces of four lines).  Same arithmetic as task_row_fwd.
// Returns the team's max|o|^2.
template <typename T, int W, int MODES, int RT>
__device__ __forceinline__ T task_rows_fwd_block(const cplx<T>* tw, cplx<T>* lines, T* red, int team, int tl, int gi,
                                                 int b, unsigned gmask, const cplx<T>* obj, int Wc, int ar, int ac,
                                                 const cplx<T>* probes, int blk, cplx<T>* dst_pos, cplx<T>* stg_o) {
    using C = cplx<T>;
    constexpr int A = Shape<W>::A, B = Shape<W>::B, TEAM = RT * B, LS = block_line_stride<W, RT>();
    const size_t WW = (size_t)W * W;
    const int r = RT * blk + gi;
    const C* orow = obj + (size_t)(ar + r) * Wc + ac;
    const C* prow = probes + (size_t)r * W;
    PTY_PROBE_STAMP(0);
    C ov[A], pv[A];
#pragma unroll
    for (int a = 0; a < A; ++a) {
        ov[a] = orow[B * a + b];
        pv[a] = prow[B * a + b];
    }
    T om = T(0);
#pragma unroll
    for (int a = 0; a < A; ++a) om = fmax(om, norm2(ov[a]));
    if (stg_o) {
        C* stg = stg_o + (size_t)r * W;
#pragma unroll
        for (int a = 0; a < A; ++a) stg[B * a + b] = ov[a];
    }
    PTY_PROBE_STAMP(1);
    PTY_PROBE_STAMP(2);
    // exit wave C * P_m * o_j straight from registers into the transform's
    // first stage (lane b holds n = B*a + b, the stage-1 input order); the
    // line only serves as the exchange buffer and receives the spectrum in
    // natural (padded) order; mode m+1's probe row loads are in flight during
    // mode m's transform
#pragma unroll
    for (int m = 0; m < MODES; ++m) {
        C pn[A];
        if (m + 1 < MODES) {
#pragma unroll
            for (int a = 0; a < A; ++a) pn[a] = prow[(m + 1) * WW + B * a + b];
        }
        C* line = lines + (m * RT + gi) * LS;
        group_fft<T, W, false>(
            line, tw, b, gmask, [&](int n, int a) { return scale(pv[a] * ov[a], checker<T>(r, n)); },
            [&](int k, int, C v) { line[pad<W>(k)] = v; });
        if (m + 1 < MODES) {
#pragma unroll
            for (int a = 0; a < A; ++a) pv[a] = pn[a];
        }
    }
    PTY_PROBE_STAMP(3);
    PTY_PROBE_STAMP(4);
    team_sync<TEAM>(team);
    PTY_PROBE_STAMP(5);
#pragma unroll
    for (int m = 0; m < MODES; ++m) {
        C* dst = dst_pos + m * WW + RT * blk;
        const C* lm = lines + m * RT * LS;
#pragma unroll
        for (int i = 0; i < RT * W / TEAM; ++i) {
            const int e = tl + i * TEAM;
            dst[(size_t)(e / RT) * W + (e % RT)] = lm[(e % RT) * LS + pad<W>(e / RT)];
        }
    }
    PTY_PROBE_STAMP(6);
    return team_maxn<W, RT>(om, red, team, gi, b);
}

// Column pass, group task (column kc) of one position: forward column DFTs of
// every mode written back in place (Psi), total = sum_m |Psi_m|^2 (engine.py:
// 114-116) stored transposed; returns the column's max(total).  STORE = false
// keeps Psi off HBM (the batched column pass 2 recomputes it, REFWD below).
// RES: the M column lines are brought into the group's resident shared-memory
// lines by bulk copies (one elected lane, one mbarrier per group: every mode's
// line in flight at once, no registers), then transformed in place.
template <typename T, int W, bool RES = false, bool STORE = true>
__device__ __forceinline__ T task_col_fwd(const cplx<T>* tw, cplx<T>* xch, int b, unsigned gmask, cplx<T>* pos, int M,
                                          int kc, T* totT_pos, cplx<T>* res = nullptr,
                                          unsigned long long* mbar = nullptr, unsigned* mphase = nullptr) {
    using C = cplx<T>;
    constexpr int A = Shape<W>::A, B = Shape<W>::B;
    const size_t WW = (size_t)W * W;
    const T invW2 = T(1) / (T(W) * T(W));
    T tot[A];
#pragma unroll
    for (int q = 0; q < A; ++q) tot[q] = T(0);
#ifdef PTY_TMA_LINES
    if constexpr (RES) {
        if (b == 0) {
            fence_proxy_async();
            mbar_expect_tx(mbar, (unsigned)(M * W * sizeof(C)));
            for (int m = 0; m < M; ++m)
                bulk_g2s(res + m * xch_size<W>(), pos + m * WW + (size_t)kc * W, (unsigned)(W * sizeof(C)), mbar);
        }
        mbar_wait(mbar, *mphase);
        *mphase ^= 1u;
    }
#endif
#if defined(PTY_P2_ASYNC) && !defined(PTY_TMA_LINES)
    if constexpr (RES) {   // every mode's column line in flight at once: 16-byte cp.async, no registers
        constexpr int NCH = W * (int)sizeof(C) / 16;
        for (int m = 0; m < M; ++m) {
            const char* src = reinterpret_cast<const char*>(pos + m * WW + (size_t)kc * W);
            char* dst = reinterpret_cast<char*>(res + m * xch_size<W>());
#pragma unroll
            for (int q = b; q < NCH; q += B) cp_async<16>(dst + 16 * q, src + 16 * q);
        }
        cp_async_wait_all();
        __syncwarp(gmask);
    }
#endif
#if defined(PTY_P2_PREFETCH) && !defined(PTY_TMA_LINES)
    C nxt[A];
    if constexpr (RES) {
#pragma unroll
        for (int a = 0; a < A; ++a) nxt[a] = pos[(size_t)kc * W + B * a + b];
    }
#endif
    for (int m = 0; m < M;++m) {
        C* line = pos + m * WW + (size_t)kc * W;
#if defined(PTY_P2_PREFETCH) && !defined(PTY_TMA_LINES)
        if constexpr (RES) {   // mode m+1's column loads fly during mode m's transform
            C cur[A];
#pragma unroll
            for (int a = 0; a < A; ++a) cur[a] = nxt[a];
            if (m + 1 < M) {
#pragma unroll
                for (int a = 0; a < A; ++a) nxt[a] = line[WW + B * a + b];
            }
            C* rl = res + m * xch_size<W>();
            group_fft<T, W, false>(
                rl, tw, b, gmask, [&](int, int a) { return cur[a]; },
                [&](int u, int slot, C v) {
                    rl[pad<W>(u)] = v;
                    tot[slot] += norm2(v) * invW2;
                });
            continue;
        }
#endif
        if constexpr (RES) {   // Psi_m stays in this group's shared-memory line for P3
            C* rl = res + m * xch_size<W>();
            group_fft<T, W, false>(
#if defined(PTY_TMA_LINES) || defined(PTY_P2_ASYNC)
                rl, tw, b, gmask, [&](int n, int) { return rl[n]; },
#else
                rl, tw, b, gmask, [&](int n, int) { return line[n]; },
#endif
                [&](int u, int slot, C v) {
                    rl[pad<W>(u)] = v;
                    tot[slot] += norm2(v) * invW2;
                });
        } else {
            group_fft<T, W, false>(
                xch, tw, b, gmask, [&](int n, int) { return line[n]; },
                [&](int u, int slot, C v) {
                    if constexpr (STORE) line[u] = v;
                    tot[slot] += norm2(v) * invW2;
                });
        }
    }
    T tm = T(0);
    T* trow = totT_pos + (size_t)kc * W;
#pragma unroll
    for (int q = 0; q < A; ++q) {
        trow[slot_col<W>(b, q)] = tot[q];
        tm = fmax(tm, tot[q]);
    }
    return group_max<B>(tm);
}

// Column pass 2, group task (column kc): modulus constraint
// scale = sqrt(I)/sqrt(total + eps) (engine.py:117-118), error terms
// (engine.py:198-214) and inverse column DFTs of every mode.
// tmax_pos: the position's W column maxima; It: the transposed pattern.
// stg (XCORR_B sensor planes, row-major total and I) may be null.
// Writes err[0..2] = (sum (sqrt(total)-sqrt(I))^2, sum I, worst modulus error).
// REFWD: `pos` holds the row-DFT output, not Psi; each mode's forward column
// DFT is recomputed into the group's exchange line (same code as
// task_col_fwd) instead of being read back from HBM.
template <typename T, int W, bool RES = false, bool REFWD = false>
__device__ __forceinline__ void task_col_mod(const cplx<T>* tw, cplx<T>* xch, int b, unsigned gmask, cplx<T>* pos,
                                             int M, int kc, const T* totT_pos, const T* tmax_pos, const T* It_pos,
                                             T eps_rel, int track, cplx<T>* stg, double* err,
                                             cplx<T>* res = nullptr) {
    using C = cplx<T>;
    constexpr int A = Shape<W>::A, B = Shape<W>::B;
    const size_t WW = (size_t)W * W;
    const T invW2 = T(1) / (T(W) * T(W));
    const T* It = It_pos + (size_t)kc * W;
    const T* tt = totT_pos + (size_t)kc * W;
    // the column maxima, I and total of this column: one round trip
    T tmax = T(0), Ia[A], ta[A];
#pragma unroll
    for (int i = 0; i < W / B; ++i) tmax = fmax(tmax, tmax_pos[b + i * B]);
#pragma unroll
    for (int a = 0; a < A; ++a) {
        Ia[a] = It[B * a + b];
        ta[a] = tt[B * a + b];
    }
    tmax = group_max<B>(tmax);
    const T eps = eps_rel * fmax(tmax, real_limits<T>::tiny());
    T sc[A];
    double en = 0.0, ed = 0.0;
#pragma unroll
    for (int a = 0; a < A; ++a) {
        const int u = B * a + b;
        const T Iv = Ia[a], tv = ta[a];
        const T sI = sqrt_fast(Iv);
        sc[a] = modulus_scale(sI, tv + eps);
        const T d = sqrt_fast(tv) - sI;
        en += (double)(d * d);
        ed += (double)Iv;
        if (stg) {
            stg[(size_t)u * W + kc] = C{tv, T(0)};
            stg[WW + (size_t)u * W + kc] = C{Iv, T(0)};
        }
    }
    // I and total are dead here (reloaded below for the diagnostic): only the
    // A scales stay live across the mode loop
    auto inverse_cols = [&](auto&& on_input) {
        for (int m = 0; m < M; ++m) {
            C* line = pos + m * WW + (size_t)kc * W;
            C* rl = RES ? res + m * xch_size<W>() : xch;      // resident Psi_m from P2
            if constexpr (REFWD) {
                group_fft<T, W, false>(
                    xch, tw, b, gmask, [&](int n, int) { return line[n]; },
                    [&](int u, int, C v) { xch[pad<W>(u)] = v; });
                __syncwarp(gmask);
            }
            group_fft<T, W, true>(
                rl, tw, b, gmask,
                [&](int n, int a) {
                    const C v = scale((RES || REFWD) ? rl[pad<W>(n)] : line[n], sc[a]);
                    on_input(a, v);
                    return v;
                },
                [&](int r, int, C v) { line[r] = v; });
        }
    };
    T worst = T(0);
    if (!track) {
        inverse_cols([](int, C) {});
    } else {                                           // modulus diagnostic (engine.py:204-214)
        T after[A];
#pragma unroll
        for (int a = 0; a < A; ++a) after[a] = T(0);
        inverse_cols([&](int a, C v) { after[a] += norm2(v) * invW2; });
#pragma unroll
        for (int a = 0; a < A; ++a) {
            const T Iv = It[B * a + b], tv = tt[B * a + b];
            if (tv > T(1e-3) * tmax) worst = fmax(worst, fabs(after[a] - Iv) / fmax(Iv, real_limits<T>::tiny()));
        }
    }
    en = group_sum<B>(en);
    ed = group_sum<B>(ed);
    worst = group_max<B>(worst);
    if (b == 0) {
        err[0] = en;
        err[1] = ed;
        err[2] = (double)worst;
    }
}

// Team load of one mode's 4 rows from the transposed scratch into the team's
// padded lines (natural order along kc).
template <typename T, int W>
__device__ __forceinline__ void team_load_rows(cplx<T>* lines, const cplx<T>* src_mode, int rq, int tl) {
    constexpr int B = Shape<W>::B, TEAM = 4 * B, LS4 = team_line_stride<W>();
    constexpr int NE = 4 * W / TEAM;   // elements per thread, all loads in flight before the stores
    const cplx<T>* src = src_mode + 4 * rq;
    cplx<T> v[NE];
#pragma unroll
    for (int i = 0; i < NE; ++i) {
        const int e = tl + i * TEAM;
        v[i] = src[(size_t)(e >> 2) * W + (e & 3)];
    }
#pragma unroll
    for (int i = 0; i < NE; ++i) {
        const int e = tl + i * TEAM;
        lines[(e & 3) * LS4 + pad<W>(e >> 2)] = v[i];
    }
}

struct UpdateParams {
    double alpha_o, alpha_p, beta, gamma, eps_rel;
    int update_probe;
};

// Row pass 2 of the reference-order sweep, team task (row quad rq) of one
// position: inverse row DFTs of every mode -> corrected exit waves psi'
// (engine.py:119); object update with the paste-add rounding (engine.py:123-137,
// fields.py:101-107) and in-place probe update with the pre-update o_j and
// probes (engine.py:140-150, 218-223).  numer/pp/nppacc: the team's [4][W]
// shared accumulators (owner-only access).  Returns the team's max of the next
// visit's sum_m |P_m|^2 (engine.py:129-132).  stg (XCORR_A planes) may be null.
template <typename T, int W>
__device__ __forceinline__ T task_row_inv_update(const cplx<T>* tw, cplx<T>* lines, cplx<T>* __restrict__ numer,
                                                 T* __restrict__ invdp, T* __restrict__ nppacc,
                                                 T* red4,
                                                 int team, int tl, int gi, int b, unsigned gmask, const cplx<T>* pos,
                                                 int M, int rq, cplx<T>* obj, T* ppg, int Wc, int ar, int ac,
                                                 cplx<T>* probes, T peak, T omax, const UpdateParams& U,
                                                 cplx<T>* stg) {
    using C = cplx<T>;
    constexpr int A = Shape<W>::A, B = Shape<W>::B, TEAM = 4 * B, LS4 = team_line_stride<W>();
    const size_t WW = (size_t)W * W;
    const T invW2 = T(1) / (T(W) * T(W));
    const T alpha_o = T(U.alpha_o), alpha_p = T(U.alpha_p), beta = T(U.beta), gamma = T(U.gamma),
            eps_rel = T(U.eps_rel);
    const int r = 4 * rq + gi;
    C* orow = obj + (size_t)(ar + r) * Wc + ac;
    T* pprow = ppg + (size_t)r * W;
    C* myline = lines + gi * LS4;
    C* nrow = numer + gi * W;
    T* idp = invdp + gi * acc_stride<W>();
    T* npp = nppacc + gi * acc_stride<W>();
    const T dmax_p = beta * omax + (T(1) - beta) * omax;
    C ov[A];
#pragma unroll
    for (int q = 0; q < A; ++q) ov[q] = orow[slot_col<W>(b, q)];
#pragma unroll
    for (int q = 0; q < A; ++q) {
        const int c = slot_col<W>(b, q);
        nrow[c] = C{T(0), T(0)};
        npp[c] = T(0);
        // the probe-update denominator (engine.py:148-150) is mode-invariant:
        // one reciprocal per element (divr multiplies by it, numpy's complex/real)
        T dp = beta * omax + (T(1) - beta) * norm2(ov[q]);
        dp = dp + eps_rel * dmax_p;
        idp[c] = rcp_fast(dp);
    }
    for (int m = 0; m < M; ++m) {
        team_sync<TEAM>(team);
        // scratch rows and probe row in flight together (one L2 round trip)
        constexpr int NE = 4 * W / TEAM;
        const C* src = pos + m * WW + 4 * rq;
        C sv[NE];
#pragma unroll
        for (int i = 0; i < NE; ++i) {
            const int e = tl + i * TEAM;
            sv[i] = src[(size_t)(e >> 2) * W + (e & 3)];
        }
        C* pr = probes + m * WW + (size_t)r * W;
        C pv[A];
#pragma unroll
        for (int q = 0; q < A; ++q) pv[q] = pr[slot_col<W>(b, q)];
#pragma unroll
        for (int i = 0; i < NE; ++i) {
            const int e = tl + i * TEAM;
            lines[(e & 3) * LS4 + pad<W>(e >> 2)] = sv[i];
        }
        team_sync<TEAM>(team);
        group_fft<T, W, true>(
            myline, tw, b, gmask, [&](int n, int) { return myline[pad<W>(n)]; },
            [&](int c, int q, C X) {
                const C o = ov[q];
                const C d = scale(X, checker<T>(r, c) * invW2) - pv[q] * o;
                nrow[c] = nrow[c] + mulc(d, pv[q]);
                if (U.update_probe) {
                    const C np_ = pv[q] + scale(mulc(scale(d, alpha_p), o), idp[c]);
                    pr[c] = np_;
                    npp[c] += norm2(np_);
                }
            });
    }
    // sum_m |P_m|^2 of this visit's probes: kept from the previous visit's
    // update (same values, same mode order) or phase 0.  All loads first.
    T ppv[A];
#pragma unroll
    for (int q = 0; q < A; ++q) ppv[q] = pprow[slot_col<W>(b, q)];
    const T dmax_o = gamma * peak + (T(1) - gamma) * peak;
    T pk = T(0);
#pragma unroll
    for (int q = 0; q < A; ++q) {
        const int c = slot_col<W>(b, q);
        const C o = ov[q];
        T den = gamma * peak + (T(1) - gamma) * ppv[q];
        den = den + eps_rel * dmax_o;
        const C no = o + scale(scale(nrow[c], alpha_o), rcp_fast(den));
        orow[c] = o + (no - o);                                // paste_add_inplace
        if (stg) {
            stg[(size_t)r * W + c] = o;
            stg[WW + (size_t)r * W + c] = no;
        }
        if (U.update_probe) {
            const T nv = npp[c];
            pprow[c] = nv;
            pk = fmax(pk, nv);
        } else {
            pk = fmax(pk, ppv[q]);
        }
    }
    return team_max4<W>(pk, red4, team, gi, b);
}

// This visit's max sum_m |P_m|^2 and max |o_j|^2 from their per-block partials
// (every group reduces all of them: the result is uniform over the team).
// false (and the error bit in `bad`) if the update is degenerate
// (engine.py:132-134, 145-147).
template <typename T, int B>
__device__ __forceinline__ bool block_maxima(const T* peak_part, const T* omax_part, int n, int b, int update_probe,
                                             T& peak, T& omax, int& bad) {
    peak = T(0);
    omax = T(0);
    for (int q = b; q < n; q += B) {
        peak = fmax(peak, peak_part[q]);
        omax = fmax(omax, omax_part[q]);
    }
    peak = group_max<B>(peak);
    omax = group_max<B>(omax);
    if (peak == T(0)) {
        bad = PTY_ERR_PROBE_ZERO;
        return false;
    }
    if (update_probe && omax == T(0)) {
        bad = PTY_ERR_OBJECT_ZERO;
        return false;
    }
    return true;
}

// The block's scratch rows ([m][kc][RT*blk + row]: RT consecutive complex
// values per column -- a 128-byte line for RT = 16) of every mode into the
// team's lines (lines[(m*RT + row)*LS + pad(kc)]) and their inverse row
// transforms in place; this visit's maxima come from their per-block partials
// while the rows are in flight.  false (and the error bit in `bad`) if the
// update is degenerate -- uniform over the team, no shared memory touched.
template <typename T, int W, int MODES, int RT>
__device__ __forceinline__ bool stage_inverse_rows(const cplx<T>* tw, cplx<T>* lines, int team, int tl, int gi, int b,
                                                   unsigned gmask, const cplx<T>* pos, int blk, const T* peak_part,
                                                   const T* omax_part, int nparts, int update_probe, T& peak, T& omax,
                                                   int& bad) {
    using C = cplx<T>;
    constexpr int B = Shape<W>::B, TEAM = RT * B, LS = block_line_stride<W, RT>(), NE = RT * W / TEAM;
    const size_t WW = (size_t)W * W;
#ifndef PTY_P4_REGS
    // every mode's rows in flight at once (cp.async, no register staging;
    // PTY_P4_REGS: the register-staged loads, mode m+1 in flight while mode m
    // is stored -- measured 1.2 % slower)
    team_sync<TEAM>(team);                                     // lines free
#pragma unroll
    for (int m = 0; m < MODES; ++m) {
#pragma unroll
        for (int i = 0; i < NE; ++i) {
            const int e = tl + i * TEAM;
            cp_async<sizeof(C)>(lines + (m * RT + (e % RT)) * LS + pad<W>(e / RT),
                                pos + m * WW + (size_t)(e / RT) * W + RT * blk + (e % RT));
        }
    }
    if (!block_maxima<T, B>(peak_part, omax_part, nparts, b, update_probe, peak, omax, bad)) {
        cp_async_wait_all();
        return false;
    }
    cp_async_wait_all();
#else
    C cur[NE], nxt[NE];
#pragma unroll
    for (int i = 0; i < NE; ++i) {
        const int e = tl + i * TEAM;
        cur[i] = pos[(size_t)(e / RT) * W + RT * blk + (e % RT)];
    }
    if (!block_maxima<T, B>(peak_part, omax_part, nparts, b, update_probe, peak, omax, bad)) return false;
    team_sync<TEAM>(team);                                     // lines free
#pragma unroll
    for (int m = 0; m < MODES; ++m) {
        if (m + 1 < MODES) {
#pragma unroll
            for (int i = 0; i < NE; ++i) {
                const int e = tl + i * TEAM;
                nxt[i] = pos[(m + 1) * WW + (size_t)(e / RT) * W + RT * blk + (e % RT)];
            }
        }
#pragma unroll
        for (int i = 0; i < NE; ++i) {
            const int e = tl + i * TEAM;
            lines[(m * RT + (e % RT)) * LS + pad<W>(e / RT)] = cur[i];
        }
        if (m + 1 < MODES) {
#pragma unroll
            for (int i = 0; i < NE; ++i) cur[i] = nxt[i];
        }
    }
#endif
    team_sync<TEAM>(team);
    PTY_PROBE_STAMP(11);
#pragma unroll 1
    for (int m = 0; m < MODES; ++m) line_fft<T, W, true>(lines + (m * RT + gi) * LS, tw, b, gmask);
    PTY_PROBE_STAMP(12);
    team_sync<TEAM>(team);
    PTY_PROBE_STAMP(13);
    return true;
}

// Row pass 2, staged variant (shared memory for all modes): team task (block
// blk of RT rows) of one position.  (1) stage_inverse_rows brings every mode's
// rows into the team's lines and inverse-transforms them in place, (2) the
// update epilogue runs element-linear over the team with all of an element's
// inputs (o, sum|P|^2, P_m, psi'_m) gathered first and its accumulators in
// registers.  Same expressions and mode order as task_row_inv_update
// (engine.py:119-150, 218-224, fields.py:101-107).  Returns the team max of
// the next visit's sum_m |P_m|^2.
template <typename T, int W, int MODES, int RT>
__device__ __forceinline__ T task_rows_inv_block(const cplx<T>* tw, cplx<T>* lines, T* red, int team,
                                                 int tl, int gi, int b, unsigned gmask, const cplx<T>* pos,
                                                 int blk, cplx<T>* obj, T* ppg, int Wc, int ar, int ac,
                                                 cplx<T>* probes, const T* peak_part, const T* omax_part, int nparts,
                                                 const UpdateParams& U, cplx<T>* stg, int& bad) {
    using C = cplx<T>;
    constexpr int B = Shape<W>::B, TEAM = RT * B, LS = block_line_stride<W, RT>(), NE = RT * W / TEAM;
#ifdef PTY_P4_CH
    constexpr int CH = MODES <= 3 ? PTY_P4_CH : (MODES <= 6 ? 2 : 1);
#else
    constexpr int CH = MODES <= 3 ? 4 : (MODES <= 6 ? 2 : 1);
#endif
    const size_t WW = (size_t)W * W;
    const T invW2 = T(1) / (T(W) * T(W));
    const T alpha_o = T(U.alpha_o), alpha_p = T(U.alpha_p), beta = T(U.beta), gamma = T(U.gamma),
            eps_rel = T(U.eps_rel);
    T peak, omax;
    PTY_PROBE_STAMP(10);
    // the block's scratch rows ([m][kc][RT*blk + row]: RT consecutive complex
    // values per column -- a 128-byte line for RT = 16) into the team's lines;
    // mode m+1's loads are in flight while mode m is stored to shared memory
    if (!stage_inverse_rows<T, W, MODES, RT>(tw, lines, team, tl, gi, b, gmask, pos, blk, peak_part, omax_part, nparts,
                                             U.update_probe, peak, omax, bad))
        return T(0);
    const T dmax_p = beta * omax + (T(1) - beta) * omax;
    const T dmax_o = gamma * peak + (T(1) - gamma) * peak;
    T pk = T(0);
    // element-linear epilogue in chunks of CH elements per thread (all of a
    // chunk's o_j and P_m loads in flight together; issuing them a chunk ahead
    // measured 1-5 % slower)
    auto load_chunk = [&](int h, C* ov, C (*pv)[CH]) {
#pragma unroll
        for (int k = 0; k < CH; ++k) {
            const int e = tl + (h + k) * TEAM, rr = e / W, c = e % W, r = RT * blk + rr;
            ov[k] = obj[(size_t)(ar + r) * Wc + ac + c];
#pragma unroll
            for (int m = 0; m < MODES; ++m) pv[m][k] = probes[m * WW + (size_t)r * W + c];
        }
    };
    auto update_chunk = [&](int h, const C* ov, C (*pv)[CH]) {
#pragma unroll
        for (int k = 0; k < CH; ++k) {
            const int e = tl + (h + k) * TEAM, rr = e / W, c = e % W, r = RT * blk + rr;
            const C o = ov[k];
            T dp = beta * omax + (T(1) - beta) * norm2(o);
            dp = dp + eps_rel * dmax_p;
            const T idp = rcp_fast(dp);
            const OMul<T> om(o);
            C numer{T(0), T(0)};
            T npp = T(0);
#pragma unroll
            for (int m = 0; m < MODES; ++m) {
                const C X = lines[(m * RT + rr) * LS + pad<W>(c)];
                const C d = scale(X, checker<T>(r, c) * invW2) - om.mul(pv[m][k]);
                numer = numer + mulc(d, pv[m][k]);
                if (U.update_probe) {
                    const C np_ = pv[m][k] + scale(om.mulconj(scale(d, alpha_p)), idp);
                    probes[m * WW + (size_t)r * W + c] = np_;
                    npp += norm2(np_);
                }
            }
            // sum_m |P_m|^2 of this visit's probes, in mode order (engine.py:129)
            T ppk = T(0);
#pragma unroll
            for (int m = 0; m < MODES; ++m) ppk += norm2(pv[m][k]);
            T den = gamma * peak + (T(1) - gamma) * ppk;
            den = den + eps_rel * dmax_o;
            const C no = o + scale(scale(numer, alpha_o), rcp_fast(den));
            obj[(size_t)(ar + r) * Wc + ac + c] = o + (no - o);          // paste_add_inplace
            if (stg) {
                stg[(size_t)r * W + c] = o;
                stg[WW + (size_t)r * W + c] = no;
            }
            pk = fmax(pk, U.update_probe ? npp : ppk);
        }
    };
#ifndef PTY_P4_NO_PAIRS
    if constexpr (std::is_same<T, float>::value && W % 2 == 0) {
        // fp32: a thread takes column pairs (c, c+1) of a row, so the probe
        // (and staging) accesses are 16-byte loads / stores; the object patch
        // sits at an arbitrary anchor, its accesses stay 8-byte
        constexpr int HW2 = W / 2, NP = NE / 2, CP = CH / 2 > 0 ? CH / 2 : 1;
#pragma unroll 1
        for (int h = 0; h < NP; h += CP) {
            C ov[2 * CP], pv[MODES][2 * CP];
#pragma unroll
            for (int k = 0; k < CP; ++k) {
                const int q = tl + (h + k) * TEAM, rr = q / HW2, c = 2 * (q % HW2), r = RT * blk + rr;
                const C* orow = obj + (size_t)(ar + r) * Wc + ac + c;
                ov[2 * k] = orow[0];
                ov[2 * k + 1] = orow[1];
#pragma unroll
                for (int m = 0; m < MODES; ++m) {
                    const float4 v = *reinterpret_cast<const float4*>(probes + m * WW + (size_t)r * W + c);
                    pv[m][2 * k] = C{v.x, v.y};
                    pv[m][2 * k + 1] = C{v.z, v.w};
                }
            }
#pragma unroll
            for (int k = 0; k < CP; ++k) {
                const int q = tl + (h + k) * TEAM, rr = q / HW2, c0 = 2 * (q % HW2), r = RT * blk + rr;
                C np2[MODES][2], no2[2];
#pragma unroll
                for (int u = 0; u < 2; ++u) {
                    const int c = c0 + u;
                    const C o = ov[2 * k + u];
                    T dp = beta * omax + (T(1) - beta) * norm2(o);
                    dp = dp + eps_rel * dmax_p;
                    const T idp = rcp_fast(dp);
                    const OMul<T> om(o);
                    C numer{T(0), T(0)};
                    T npp = T(0);
#pragma unroll
                    for (int m = 0; m < MODES; ++m) {
                        const C pm = pv[m][2 * k + u];
                        const C X = lines[(m * RT + rr) * LS + pad<W>(c)];
                        const C d = scale(X, checker<T>(r, c) * invW2) - om.mul(pm);
                        numer = numer + mulc(d, pm);
                        np2[m][u] = pm;
                        if (U.update_probe) {
                            const C np_ = pm + scale(om.mulconj(scale(d, alpha_p)), idp);
                            np2[m][u] = np_;
                            npp += norm2(np_);
                        }
                    }
                    T ppk = T(0);
#pragma unroll
                    for (int m = 0; m < MODES; ++m) ppk += norm2(pv[m][2 * k + u]);
                    T den = gamma * peak + (T(1) - gamma) * ppk;
                    den = den + eps_rel * dmax_o;
                    const C no = o + scale(scale(numer, alpha_o), rcp_fast(den));
                    obj[(size_t)(ar + r) * Wc + ac + c] = o + (no - o);      // paste_add_inplace
                    no2[u] = no;
                    pk = fmax(pk, U.update_probe ? npp : ppk);
                }
                if (U.update_probe) {
#pragma unroll
                    for (int m = 0; m < MODES; ++m)
                        *reinterpret_cast<float4*>(probes + m * WW + (size_t)r * W + c0) =
                            make_float4(np2[m][0].re, np2[m][0].im, np2[m][1].re, np2[m][1].im);
                }
                if (stg) {
                    *reinterpret_cast<float4*>(stg + (size_t)r * W + c0) =
                        make_float4(ov[2 * k].re, ov[2 * k].im, ov[2 * k + 1].re, ov[2 * k + 1].im);
                    *reinterpret_cast<float4*>(stg + WW + (size_t)r * W + c0) =
                        make_float4(no2[0].re, no2[0].im, no2[1].re, no2[1].im);
                }
            }
        }
    } else
#endif
    {
#pragma unroll 1
    for (int h = 0; h < NE; h += CH) {
        C ov[CH], pv[MODES][CH];
        load_chunk(h, ov, pv);
        update_chunk(h, ov, pv);
    }
    }
    PTY_PROBE_STAMP(14);
    pk = group_max<B>(pk);
    return team_maxn<W, RT>(pk, red, team, gi, b);
}

// Row pass 2 of the batched extension (oracle/batched.py contrib; the
// reference has no batched mode): same staging and inverse
// transforms as task_rows_inv_block, but nothing is written back -- every
// position of a batch sees the batch-start object and probes.  Per element the
// position's object numerator sum_m (psi'_m - P_m o) conj(P_m) (engine.py:
// 130-131) goes to its own plane onum_k, and the probe numerators alpha_P
// (psi'_m - P_m o) conj(o) (engine.py:150) and denominator beta max|o|^2 +
// (1 - beta)|o|^2 (engine.py:148) are added into this slot's group
// accumulator pg ([2M+1][W][W] real: re/im per mode, then the denominator,
// zeroed per batch).  The rows of block blk of pg are added to by this team
// alone, position after position, with fire-and-forget reductions (red.add:
// no load round trip; same-thread same-address order = the slot's batch
// order, so the sums are deterministic and equal the load-add-store ones).
template <typename T, int W, int MODES, int RT>
__device__ __forceinline__ void task_rows_acc_block(const cplx<T>* tw, cplx<T>* lines, int team, int tl, int gi, int b,
                                                    unsigned gmask, const cplx<T>* pos, int blk, const cplx<T>* obj,
                                                    int Wc, int ar, int ac, const cplx<T>* probes, const T* peak_part,
                                                    const T* omax_part, int nparts, const UpdateParams& U,
                                                    cplx<T>* onum_k, T* pg, int& bad) {
    using C = cplx<T>;
    constexpr int B = Shape<W>::B, TEAM = RT * B, LS = block_line_stride<W, RT>(), NE = RT * W / TEAM;
    constexpr int CH = MODES <= 3 ? 4 : (MODES <= 6 ? 2 : 1);
    const size_t WW = (size_t)W * W;
    const T invW2 = T(1) / (T(W) * T(W));
    const T alpha_p = T(U.alpha_p), beta = T(U.beta);
    T peak, omax;
    if (!stage_inverse_rows<T, W, MODES, RT>(tw, lines, team, tl, gi, b, gmask, pos, blk, peak_part, omax_part, nparts,
                                             U.update_probe, peak, omax, bad))
        return;
#pragma unroll 1
    for (int h = 0; h < NE; h += CH) {
        C ov[CH], pv[MODES][CH];
#pragma unroll
        for (int k = 0; k < CH; ++k) {
            const int e = tl + (h + k) * TEAM, rr = e / W, c = e % W, r = RT * blk + rr;
            ov[k] = obj[(size_t)(ar + r) * Wc + ac + c];
#pragma unroll
            for (int m = 0; m < MODES; ++m) pv[m][k] = probes[m * WW + (size_t)r * W + c];
        }
#pragma unroll
        for (int k = 0; k < CH; ++k) {
            const int e = tl + (h + k) * TEAM, rr = e / W, c = e % W, r = RT * blk + rr;
            const size_t off = (size_t)r * W + c;
            const C o = ov[k];
            const OMul<T> om(o);
            C numer{T(0), T(0)};
#pragma unroll
            for (int m = 0; m < MODES; ++m) {
                const C X = lines[(m * RT + rr) * LS + pad<W>(c)];
                const C d = scale(X, checker<T>(r, c) * invW2) - om.mul(pv[m][k]);
                numer = numer + mulc(d, pv[m][k]);
                if (U.update_probe) {
                    const C pn = om.mulconj(scale(d, alpha_p));
                    atomicAdd(pg + (2 * m) * WW + off, pn.re);
                    atomicAdd(pg + (2 * m + 1) * WW + off, pn.im);
                }
            }
            onum_k[off] = numer;
            if (U.update_probe) atomicAdd(pg + (2 * MODES) * WW + off, beta * omax + (T(1) - beta) * norm2(o));
        }
    }
    team_sync<TEAM>(team);                                     // lines free for the next task
}

}  // namespace pty
