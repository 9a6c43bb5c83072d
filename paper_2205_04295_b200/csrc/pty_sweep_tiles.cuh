// pty_sweep_tiles.cuh -- the latency variant of the fused rPIE sweep (one
// cooperative persistent kernel per sweep, engine.py:173-243), used for few
// slots (the reference's single reconstruction): every phase spreads small
// row / column tiles of all modes over all CTAs so one visit finishes fast.
// pty_sweep.cuh holds the throughput variant (line tasks) for many slots.
//
// Per visit step s (every slot advances to its position order[s]):
//   P1 rows  : gather o_j rows at the integer anchor (engine.py:192-195),
//              exit waves C*P_m*o_j for every mode (engine.py:113, C = (-1)^(r+c)),
//              forward row DFTs -> scratch;  max|o_j|^2 partials (engine.py:145)
//   P2 cols  : forward column DFTs (tile stays resident in shared memory),
//              max of total = sum_m |Psi_m|^2 partials (engine.py:114-117)
//   P3 cols  : modulus constraint scale = sqrt(I)/sqrt(total+eps) (engine.py:118),
//              error partials (engine.py:198-202), inverse column DFTs -> scratch
//   P4 rows  : inverse row DFTs -> corrected exit waves (engine.py:119),
//              rPIE object update (engine.py:123-137) written back with the
//              paste-add rounding (fields.py:101-107), rPIE probe update for every
//              mode with the pre-update crop (engine.py:140-150, 218-223), next
//              visit's max sum|P|^2 partials, posref staging (engine.py:226-230)
// separated by a software grid barrier.  The centered DFT of fields.py:71-84 is
// C * DFT(C * x) / W for even W, so no fftshift is materialised.
#pragma once
#include "pty_fft.cuh"
#include "../../include/ptycho_b200.h"

namespace pty {
namespace tiles {

constexpr int kSweepThreads = 256;
constexpr int kSweepMinCtasPerSm = 2;
constexpr int kMaxSlots = 24;
constexpr int kMaxModes = 8;

struct SlotDev {
    void* obj;
    int H, Wc, r0, c0;
    void* probes;
    const void* patterns;
    const double* positions;
    const int* order;
    void* stage;
    double* err_out;
    int* status;
};

struct SweepDev {
    int W, M, N, nslots;
    int TR, TC, nRT, nCT, K;      // row tile, col tile, tile counts, col items held per CTA
    int lgTR, lgTC;               // log2 of the (power-of-two) tile sizes
    double alpha_o, alpha_p, beta, gamma, eps_rel;
    int update_probe, track_mod, sense;
    // workspace
    unsigned int* barrier;
    int* anchors;                 // [nslots][N][2]
    void* scratch;                // [nslots][M][W][W] complex
    void* omax_part;              // [nslots][nRT] real
    void* peak_part;              // [2][nslots][nRT] real
    void* tmax_part;              // [nslots][nCT] real
    double* err_part;             // [nslots][N][nCT][3] per-visit error partials
    const void* twiddles;         // [W] complex, global
    unsigned long long* timeline; // debug: [steps][9][gridDim] globaltimer stamps (phase ends at 1,3,5,7) or null
    int timeline_steps;
    SlotDev slot[kMaxSlots];
};

// shared-memory carve-up (bytes): twiddles | reduction scratch | tile region
template <typename T, int W>
__host__ __device__ constexpr size_t sweep_smem_fixed() {
    return (size_t)W * sizeof(cplx<T>) + 64 * sizeof(double);
}
template <typename T, int W>
__host__ __device__ inline size_t sweep_smem_rows(int TR, int M) {
    return (size_t)TR * M * line_stride<W>() * sizeof(cplx<T>);
}
template <typename T, int W>
__host__ __device__ inline size_t sweep_smem_cols(int TC, int M, int K) {
    return (size_t)K * M * TC * line_stride<W>() * sizeof(cplx<T>);
}

template <typename T>
__device__ __forceinline__ T t_reduce_max_global(const T* p, int n) {
    T m = T(0);
    for (int i = 0; i < n; ++i) m = fmax(m, p[i]);
    return m;
}

// Prefetch [base, base + bytes) into L2 (or L1 when to_l1), one request per
// 128-byte line, spread over the CTA's threads.
__device__ __forceinline__ void t_prefetch_span(const void* base, size_t bytes, bool to_l1) {
    const char* p = static_cast<const char*>(base);
    const size_t lines = (bytes + 127) / 128;
    for (size_t k = threadIdx.x; k < lines; k += blockDim.x) {
        if (to_l1) asm volatile("prefetch.global.L1 [%0];" ::"l"(p + k * 128));
        else asm volatile("prefetch.global.L2 [%0];" ::"l"(p + k * 128));
    }
}

// Batched element copy: U independent loads in flight per thread before the
// stores (memory-level parallelism for L2-latency-bound tile moves).
template <int U, typename F>
__device__ __forceinline__ void t_batched(int n, F&& body) {
    for (int i0 = threadIdx.x; i0 < n; i0 += blockDim.x * U) body(i0);
}

__device__ __forceinline__ unsigned long long gtimer_t() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}

// max over n partials, loaded by warp 0 in parallel and broadcast through
// shared memory.  Every thread of the CTA must call it.
// Two maxima in one pass (both partial arrays loaded together: one L2 round
// trip and one pair of barriers instead of two).  cell: 2 shared slots.
template <typename T>
__device__ __forceinline__ void t_cta_max2_of(const T* p, const T* q, int n, T* cell, T& a, T& b) {
    if (threadIdx.x < 32) {
        T ma = T(0), mb = T(0);
        for (int i = threadIdx.x; i < n; i += 32) {
            ma = fmax(ma, p[i]);
            mb = fmax(mb, q[i]);
        }
        ma = warp_max(ma);
        mb = warp_max(mb);
        if (threadIdx.x == 0) {
            cell[0] = ma;
            cell[1] = mb;
        }
    }
    __syncthreads();
    a = cell[0];
    b = cell[1];
    __syncthreads();
}

template <typename T>
__device__ __forceinline__ T t_cta_max_of(const T* p, int n, T* cell) {
    if (threadIdx.x < 32) {
        T m = T(0);
        for (int i = threadIdx.x; i < n; i += 32) m = fmax(m, p[i]);
        m = warp_max(m);
        if (threadIdx.x == 0) *cell = m;
    }
    __syncthreads();
    const T v = *cell;
    __syncthreads();
    return v;
}

// One CTA's view of the sweep: shared-memory carve-up, per-thread constants
// and the four phases, one method per
// phase body; they are inlined (non-inlined member calls spill the CTA state
// to local memory, measured 2x slower).
template <typename T, int W>
struct SweepCta {
    using C = cplx<T>;
    static constexpr int LS = line_stride<W>();
    const SweepDev& P;
    C* tw;
    T* red;
    C* tile;
    int* s_dead;
    int* s_j;
    int* s_ar;
    int* s_ac;
    T* cellT;
    C* scratch;
    T* omax_part;
    T* peak_part;
    T* tmax_part;
    int tid, NT, M, N, S;
    size_t WW;
    T invW2, alpha_o, alpha_p, beta, gamma, eps_rel;

    __device__ __forceinline__ void phase1(int step) {
    // ------------------------------------------------------------ P1 rows
    for (int item = blockIdx.x; item < S * P.nRT; item += gridDim.x) {
        const int s = item / P.nRT, rt = item % P.nRT;
        const SlotDev& sl = P.slot[s];
        if (s_dead[s]) continue;
        const int ar = s_ar[s], ac = s_ac[s];
        const C* obj = reinterpret_cast<const C*>(sl.obj);
        const C* probes = reinterpret_cast<const C*>(sl.probes);
        // the pattern rows P3 will read: HBM -> L2 while P1/P2 run
        t_prefetch_span(reinterpret_cast<const T*>(sl.patterns) + (size_t)s_j[s] * WW + (size_t)rt * P.TR * W,
                      (size_t)P.TR * W * sizeof(T), false);
        T om = T(0);
        constexpr int U = 8;
        const int nel = P.TR * M * W;          // element = (row, mode, column)
        t_batched<U>(nel, [&](int i0) {
            C o[U], p[U];
#pragma unroll
            for (int u = 0; u < U; ++u) {
                const int i = i0 + u * NT;
                if (i < nel) {
                    const int l = i / W, c = i % W, m = l >> P.lgTR, r = l & (P.TR - 1), rr = rt * P.TR + r;
                    o[u] = obj[(size_t)(ar + rr) * sl.Wc + ac + c];
                    p[u] = probes[m * WW + (size_t)rr * W + c];
                }
            }
#pragma unroll
            for (int u = 0; u < U; ++u) {
                const int i = i0 + u * NT;
                if (i < nel) {
                    const int l = i / W, c = i % W, m = l >> P.lgTR, rr = rt * P.TR + (l & (P.TR - 1));
                    if (m == 0) om = fmax(om, norm2(o[u]));
                    tile[(size_t)l * LS + pad<W>(c)] = scale(p[u] * o[u], checker<T>(rr, c));
                }
            }
        });
        om = block_max(om, red);
        if (tid == 0) omax_part[(size_t)s * P.nRT + rt] = om;
        __syncthreads();
        lines_fft<T, W, false>(tile, P.TR * M, LS, tw);
        __syncthreads();
        C* scr = scratch + (size_t)s * M * WW;
        for (int i = tid; i < P.TR * M * W; i += NT) {   // lines are mode-major: contiguous rows
            const int l = i / W, c = i % W;
            scr[(l >> P.lgTR) * WW + (size_t)(rt * P.TR + (l & (P.TR - 1))) * W + c] = tile[(size_t)l * LS + pad<W>(c)];
        }
        __syncthreads();
    }
    }

    __device__ __forceinline__ void phase2(int step) {
    // ------------------------------------------------- P2 cols (forward)
    int held = 0;
    for (int item = blockIdx.x; item < S * P.nCT; item += gridDim.x, ++held) {
        const int s = item / P.nCT, ct = item % P.nCT;
        if (s_dead[s]) continue;
        C* my = tile + (size_t)held * M * P.TC * LS;
        const C* scr = scratch + (size_t)s * M * WW;
        {
            constexpr int U = 8;
            const int nel = M * W * P.TC;
            t_batched<U>(nel, [&](int i0) {
                C v[U];
#pragma unroll
                for (int u = 0; u < U; ++u) {
                    const int i = i0 + u * NT;
                    if (i < nel) {
                        const int rem = i & ((W << P.lgTC) - 1), m = i >> (P.lgTC + Log2<W>::value);
                        v[u] = scr[m * WW + (size_t)(rem >> P.lgTC) * W + ct * P.TC + (rem & (P.TC - 1))];
                    }
                }
#pragma unroll
                for (int u = 0; u < U; ++u) {
                    const int i = i0 + u * NT;
                    if (i < nel) {
                        const int rem = i & ((W << P.lgTC) - 1), m = i >> (P.lgTC + Log2<W>::value);
                        my[(size_t)((m << P.lgTC) + (rem & (P.TC - 1))) * LS + pad<W>(rem >> P.lgTC)] = v[u];
                    }
                }
            });
        }
        __syncthreads();
        lines_fft<T, W, false>(my, M * P.TC, LS, tw);
        __syncthreads();
        T tm = T(0);
        for (int i = tid; i < W * P.TC; i += NT) {
            const int cc = i / W, r = i % W;   // W is a compile-time power of two
            T tot = T(0);
            for (int m = 0; m < M; ++m) tot += norm2(my[(size_t)(m * P.TC + cc) * LS + pad<W>(r)]) * invW2;
            tm = fmax(tm, tot);
        }
        tm = block_max(tm, red);
        if (tid == 0) tmax_part[(size_t)s * P.nCT + ct] = tm;
    }
    }

    __device__ __forceinline__ void phase3(int step) {
    // ------------------------------------- P3 modulus + cols (inverse)
    int held = 0;
    for (int item = blockIdx.x; item < S * P.nCT; item += gridDim.x, ++held) {
        const int s = item / P.nCT, ct = item % P.nCT;
        const SlotDev& sl = P.slot[s];
        if (s_dead[s]) continue;
        C* my = tile + (size_t)held * M * P.TC * LS;
        const int j = s_j[s];
        const T tmax = t_cta_max_of(tmax_part + (size_t)s * P.nCT, P.nCT, cellT);
        const T eps = eps_rel * fmax(tmax, real_limits<T>::tiny());
        const T* I = reinterpret_cast<const T*>(sl.patterns) + (size_t)j * WW;
        C* stg = P.sense == PTY_SENSE_XCORR_B ? reinterpret_cast<C*>(sl.stage) + (size_t)j * 2 * WW : nullptr;
        double enum_ = 0.0, eden = 0.0;
        T worst = T(0);
        constexpr int UI = 8;
        const int npx = W * P.TC;
        t_batched<UI>(npx, [&](int i0) {
          T Ib[UI];
#pragma unroll
          for (int u = 0; u < UI; ++u) {
            const int i = i0 + u * NT;
            if (i < npx) Ib[u] = I[(size_t)(i >> P.lgTC) * W + ct * P.TC + (i & (P.TC - 1))];
          }
#pragma unroll
          for (int u = 0; u < UI; ++u) {
            const int i = i0 + u * NT;
            if (i >= npx) continue;
            const int r = i >> P.lgTC, cc = i & (P.TC - 1), c = ct * P.TC + cc;
            T tot = T(0);
            for (int m = 0; m < M; ++m) tot += norm2(my[(size_t)(m * P.TC + cc) * LS + pad<W>(r)]) * invW2;
            const T Iv = Ib[u];
            const T sI = sqrt_fast(Iv);
            const T sc = modulus_scale(sI, tot + eps);
            const T d = sqrt_fast(tot) - sI;
            enum_ += (double)(d * d);
            eden += (double)Iv;
            T after = T(0);
            for (int m = 0; m < M; ++m) {
                C& a = my[(size_t)(m * P.TC + cc) * LS + pad<W>(r)];
                a = scale(a, sc);
                after += norm2(a) * invW2;
            }
            if (P.track_mod && tot > T(1e-3) * tmax) {
                worst = fmax(worst, fabs(after - Iv) / fmax(Iv, real_limits<T>::tiny()));
            }
            if (stg) {
                stg[(size_t)r * W + c] = C{tot, T(0)};
                stg[WW + (size_t)r * W + c] = C{Iv, T(0)};
            }
          }
        });
        __syncthreads();
        lines_fft<T, W, true>(my, M * P.TC, LS, tw);
        __syncthreads();
        block_err3(enum_, eden, worst, reinterpret_cast<double*>(red));
        if (tid == 0) {
            double* e = P.err_part + (((size_t)s * N + step) * P.nCT + ct) * 3;
            e[0] = enum_;
            e[1] = eden;
            e[2] = (double)worst;
        }
        C* scr = scratch + (size_t)s * M * WW;
        for (int i = tid; i < M * W * P.TC; i += NT) {
            const int rem = i & ((W << P.lgTC) - 1), m = i >> (P.lgTC + Log2<W>::value);
            const int r = rem >> P.lgTC, cc = rem & (P.TC - 1);
            scr[m * WW + (size_t)r * W + ct * P.TC + cc] = my[(size_t)((m << P.lgTC) + cc) * LS + pad<W>(r)];
        }
        __syncthreads();
    }
    }

    __device__ __forceinline__ void phase4(int step) {
    // ------------------------------------------ P4 rows (inverse) + update
    for (int item = blockIdx.x; item < S * P.nRT; item += gridDim.x) {
        const int s = item / P.nRT, rt = item % P.nRT;
        const SlotDev& sl = P.slot[s];
        if (s_dead[s]) continue;
        const int j = s_j[s];
        const int ar = s_ar[s], ac = s_ac[s];   // the row loads below do not need the maxima: issued first
        {   // obj / probe rows of the update: into L1 while the inverse DFTs run
            const bool l1 = (size_t)P.TR * (M + 1) * W * sizeof(C) <= 16 * 1024;
            for (int r = 0; r < P.TR; ++r) {
                const int rr = rt * P.TR + r;
                t_prefetch_span(reinterpret_cast<const C*>(sl.obj) + (size_t)(ar + rr) * sl.Wc + ac, W * sizeof(C), l1);
                for (int m = 0; m < M; ++m)
                    t_prefetch_span(reinterpret_cast<const C*>(sl.probes) + m * WW + (size_t)rr * W, W * sizeof(C), l1);
            }
        }
        const C* scr = scratch + (size_t)s * M * WW;
        {
            constexpr int U = 8;
            const int nel = P.TR * M * W;
            t_batched<U>(nel, [&](int i0) {
                C v[U];
#pragma unroll
                for (int u = 0; u < U; ++u) {
                    const int i = i0 + u * NT;
                    if (i < nel) {
                        const int l = i / W, c = i % W;
                        v[u] = scr[(l >> P.lgTR) * WW + (size_t)(rt * P.TR + (l & (P.TR - 1))) * W + c];
                    }
                }
#pragma unroll
                for (int u = 0; u < U; ++u) {
                    const int i = i0 + u * NT;
                    if (i < nel) tile[(size_t)(i / W) * LS + pad<W>(i % W)] = v[u];
                }
            });
        }
        T peak, omax;
        t_cta_max2_of(peak_part + ((size_t)(step & 1) * S + s) * P.nRT, omax_part + (size_t)s * P.nRT, P.nRT, cellT,
                      peak, omax);
        if (peak == T(0)) {                      // engine.py:132-134
            if (tid == 0) atomicOr(sl.status, PTY_ERR_PROBE_ZERO);
            continue;
        }
        if (P.update_probe && omax == T(0)) {    // engine.py:145-147
            if (tid == 0) atomicOr(sl.status, PTY_ERR_OBJECT_ZERO);
            continue;
        }
        __syncthreads();
        lines_fft<T, W, true>(tile, P.TR * M, LS, tw);
        __syncthreads();
        C* obj = reinterpret_cast<C*>(sl.obj);
        C* probes = reinterpret_cast<C*>(sl.probes);
        C* stg = P.sense == PTY_SENSE_XCORR_A ? reinterpret_cast<C*>(sl.stage) + (size_t)j * 2 * WW : nullptr;
        const T dmax_o = gamma * peak + (T(1) - gamma) * peak;   // = max of the object denominator
        const T dmax_p = beta * omax + (T(1) - beta) * omax;
        T pk = T(0);
        for (int i = tid; i < P.TR * W; i += NT) {
            const int r = i / W, c = i % W, rr = rt * P.TR + r;
            const size_t oi = (size_t)(ar + rr) * sl.Wc + ac + c;
            const C o = obj[oi];
            const T sg = checker<T>(rr, c) * invW2;
            C numer{T(0), T(0)};
            T pp = T(0);
            for (int m = 0; m < M; ++m) {
                const C pv = probes[m * WW + (size_t)rr * W + c];
                const C psi = scale(tile[(size_t)((m << P.lgTR) + r) * LS + pad<W>(c)], sg);
                numer = numer + mulc(psi - pv * o, pv);
                pp += norm2(pv);
            }
            T den = gamma * peak + (T(1) - gamma) * pp;
            den = den + eps_rel * dmax_o;
            const C no = o + scale(scale(numer, alpha_o), rcp_fast(den));
            obj[oi] = o + (no - o);                              // paste_add_inplace
            if (stg) {
                stg[(size_t)rr * W + c] = o;
                stg[WW + (size_t)rr * W + c] = no;
            }
            if (P.update_probe) {
                const T op = norm2(o);
                T dp = beta * omax + (T(1) - beta) * op;
                dp = dp + eps_rel * dmax_p;
                const T idp = rcp_fast(dp);                          // divr multiplies by 1/dp
                T npp = T(0);
                for (int m = 0; m < M; ++m) {   // pre-update probes and o_j (engine.py:218-223)
                    const size_t pi = m * WW + (size_t)rr * W + c;
                    const C pv = probes[pi];
                    const C psi = scale(tile[(size_t)((m << P.lgTR) + r) * LS + pad<W>(c)], sg);
                    const C np_ = pv + scale(mulc(scale(psi - pv * o, alpha_p), o), idp);
                    probes[pi] = np_;
                    npp += norm2(np_);
                }
                pk = fmax(pk, npp);
            } else {
                pk = fmax(pk, pp);
            }
        }
        pk = block_max(pk, red);
        if (tid == 0) peak_part[((size_t)((step + 1) & 1) * S + s) * P.nRT + rt] = pk;
        __syncthreads();
    }
    }
};

template <typename T, int W>
__global__ void __launch_bounds__(kSweepThreads, kSweepMinCtasPerSm) sweep_kernel(const __grid_constant__ SweepDev P) {
    using C = cplx<T>;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    // per-step snapshot of every slot: dead flag, position index, anchor
    __shared__ int s_dead[kMaxSlots], s_j[kMaxSlots], s_ar[kMaxSlots], s_ac[kMaxSlots];
    __shared__ double s_cell[2];
    SweepCta<T, W> X{P};
    X.tw = reinterpret_cast<C*>(smem_raw);
    X.red = reinterpret_cast<T*>(smem_raw + (size_t)W * sizeof(C));
    X.tile = reinterpret_cast<C*>(smem_raw + sweep_smem_fixed<T, W>());
    X.s_dead = s_dead;
    X.s_j = s_j;
    X.s_ar = s_ar;
    X.s_ac = s_ac;
    X.cellT = reinterpret_cast<T*>(s_cell);
    X.scratch = reinterpret_cast<C*>(P.scratch);
    X.omax_part = reinterpret_cast<T*>(P.omax_part);
    X.peak_part = reinterpret_cast<T*>(P.peak_part);
    X.tmax_part = reinterpret_cast<T*>(P.tmax_part);
    X.tid = threadIdx.x;
    X.NT = blockDim.x;
    X.M = P.M;
    X.N = P.N;
    X.S = P.nslots;
    X.WW = (size_t)W * W;
    X.invW2 = T(1) / (T(W) * T(W));
    X.alpha_o = T(P.alpha_o);
    X.alpha_p = T(P.alpha_p);
    X.beta = T(P.beta);
    X.gamma = T(P.gamma);
    X.eps_rel = T(P.eps_rel);
    const int tid = threadIdx.x, NT = blockDim.x, M = P.M, N = P.N, S = P.nslots;
    const size_t WW = (size_t)W * W;
    T* red = X.red;
    T* peak_part = X.peak_part;

    GridBarrier bar{P.barrier, 0u};
    load_twiddles<T, W>(X.tw, reinterpret_cast<const C*>(P.twiddles));

    // ---- phase 0: anchors (engine.py:69-70, 192-195) + bounds, initial probe peak
    for (int idx = blockIdx.x * NT + tid; idx < S * N; idx += gridDim.x * NT) {
        const int s = idx / N, j = idx % N;
        const SlotDev& sl = P.slot[s];
        const double x = sl.positions[2 * j], y = sl.positions[2 * j + 1];
        const int ar = (int)rint(y) - sl.r0;   // round half to even == Python round()
        const int ac = (int)rint(x) - sl.c0;
        P.anchors[2 * idx] = ar;
        P.anchors[2 * idx + 1] = ac;
        if (ar < 0 || ac < 0 || ar + W > sl.H || ac + W > sl.Wc) atomicOr(sl.status, PTY_ERR_BOUNDS);
    }
    for (int item = blockIdx.x; item < S * P.nRT; item += gridDim.x) {
        const int s = item / P.nRT, rt = item % P.nRT;
        const C* probes = reinterpret_cast<const C*>(P.slot[s].probes);
        T pk = T(0);
        for (int i = tid; i < P.TR * W; i += NT) {
            const size_t off = (size_t)(rt * P.TR) * W + i;
            T pp = T(0);
            for (int m = 0; m < M; ++m) pp += norm2(probes[m * WW + off]);
            pk = fmax(pk, pp);
        }
        pk = block_max(pk, red);
        if (tid == 0) peak_part[(size_t)s * P.nRT + rt] = pk;
    }
    bar.sync();

    auto stamp = [&](int step, int k) {
        if (P.timeline && step < P.timeline_steps) {
            __syncthreads();
            if (tid == 0) P.timeline[((size_t)step * 9 + (k ? 2 * k - 1 : 0)) * gridDim.x + blockIdx.x] = gtimer_t();
        }
    };
    for (int step = 0; step < N; ++step) {
        stamp(step, 0);
        if (tid < S) {   // status only changes in P4 / phase 0, both behind a barrier
            const SlotDev& sl = P.slot[tid];
            const int j = sl.order[step];
            s_dead[tid] = *(volatile const int*)sl.status;
            s_j[tid] = j;
            s_ar[tid] = P.anchors[2 * (tid * N + j)];
            s_ac[tid] = P.anchors[2 * (tid * N + j) + 1];
        }
        __syncthreads();
        X.phase1(step);
        stamp(step, 1);
        bar.sync();
        X.phase2(step);
        stamp(step, 2);
        bar.sync();
        X.phase3(step);
        stamp(step, 3);
        bar.sync();
        X.phase4(step);
        stamp(step, 4);
        bar.sync();
    }
}

// Deterministic end-of-sweep reduction of the per-visit error partials
// (engine.py:198-202, 239-241): one CTA per slot, thread t sums visits
// t, t+256, ... in order, then a fixed shuffle tree -- same order every run.
struct ErrOut {
    double* p[kMaxSlots];
};
static __global__ void __launch_bounds__(256) sweep_finalize_kernel(const double* err_part, int N, int nCT,
                                                                    int nslots, ErrOut outs) {
    __shared__ double red[32];
    const int s = blockIdx.x;
    if (s >= nslots) return;
    double num = 0.0, den = 0.0, worst = 0.0;
    for (int k = threadIdx.x; k < N; k += blockDim.x) {
        for (int ct = 0; ct < nCT; ++ct) {
            const double* e = err_part + (((size_t)s * N + k) * nCT + ct) * 3;
            num += e[0];
            den += e[1];
            worst = fmax(worst, e[2]);
        }
    }
    num = block_sum(num, red);
    den = block_sum(den, red);
    worst = block_max(worst, red);
    if (threadIdx.x == 0) {
        outs.p[s][0] = num;
        outs.p[s][1] = den;
        outs.p[s][2] = worst;
    }
}

}  // namespace tiles
}  // namespace pty
