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
//   bk_cols_fwd    : column DFTs, Psi -> scratch[k]; max(total) partials
//   bk_cols_mod    : modulus constraint, error terms, inverse column DFTs
//   bk_rows_inv    : inverse row DFTs -> psi'; object numerator per position
//                    (onum[k]); probe numerator/denominator summed over a fixed
//                    group of positions per CTA (deterministic)
//   bk_probe_reduce: groups -> probe accumulator (fixed order)
//   bk_obj_gather  : owner-computes canvas tiles: object numerator/denominator
//                    summed over the covering positions in batch order
//   -- accumulators may be all-reduced across ranks here (NCCL) --
//   bk_obj_tile_max, bk_obj_apply, bk_probe_apply, bk_stage_after
#pragma once
#include "pty_fft.cuh"

namespace pty {

constexpr int kBatThreads = 128;
constexpr int kObjTile = 32;           // owner tile edge (canvas pixels)
constexpr int kMaxBatchModes = 8;

struct BatchDev {
    int W, M, N, b;                    // window, modes, positions in dataset, positions in batch
    int TR, TC, lgTR, lgTC, nRT, nCT, G;
    void* obj;
    int H, Wc, r0, c0;
    void* probes;
    const void* patterns;
    const double* positions;
    const int* batch;                  // [b] position ids
    int visit0;                        // index of batch[0] in the sweep's visit order
    double alpha_o, alpha_p, beta, gamma, eps_rel;
    int update_probe, track_mod, sense;
    void* stage;                       // [N][2][W][W] complex or null
    void* obj_acc;                     // [3][H][Wc] real: num.re, num.im, den
    void* probe_acc;                   // [2M+1][W][W] real: pnum (re, im) per mode, pden
    double* err_part;                  // [N][nCT][3] by visit rank (visit0 + k)
    int* status;
    // workspace
    int* anchors;                      // [b][2]
    void* scratch;                     // [b][M][W][W] complex
    void* onum;                        // [b][W][W] complex
    void* pp;                          // [W][W] real (probe power)
    void* pp_part;                     // [nRT] real
    void* omax_part;                   // [b][nRT] real
    void* tmax_part;                   // [b][nCT] real
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

// K1: gather + exit waves + row DFTs.  CTA = (position k, row tile).
template <typename T, int W>
__global__ void __launch_bounds__(kBatThreads) bk_rows_fwd(const __grid_constant__ BatchDev P) {
    using C = cplx<T>;
    constexpr int LS = line_stride<W>();
    extern __shared__ __align__(16) unsigned char smem_raw[];
    C* tw = reinterpret_cast<C*>(smem_raw);
    T* red = reinterpret_cast<T*>(tw + W);
    C* tile = reinterpret_cast<C*>(red + 64);
    load_twiddles<T, W>(tw, reinterpret_cast<const C*>(P.twiddles));
    const int k = blockIdx.x / P.nRT, rt = blockIdx.x % P.nRT;
    if (*(volatile const int*)P.status) return;
    const int M = P.M, NT = blockDim.x;
    const size_t WW = (size_t)W * W;
    const int j = P.batch[k], ar = P.anchors[2 * k], ac = P.anchors[2 * k + 1];
    const C* obj = reinterpret_cast<const C*>(P.obj);
    const C* probes = reinterpret_cast<const C*>(P.probes);
    const T* I = reinterpret_cast<const T*>(P.patterns) + (size_t)j * WW;
    for (size_t q = threadIdx.x; q < (size_t)P.TR * W * sizeof(T) / 128; q += NT)   // pattern rows -> L2
        asm volatile("prefetch.global.L2 [%0];" ::"l"(reinterpret_cast<const char*>(I + (size_t)rt * P.TR * W) + q * 128));
    C* stg = P.sense == PTY_SENSE_XCORR_A ? reinterpret_cast<C*>(P.stage) + (size_t)j * 2 * WW : nullptr;
    T om = T(0);
    constexpr int U = 4;
    const int nel = P.TR * M * W;
    for (int i0 = threadIdx.x; i0 < nel; i0 += NT * U) {
        C o[U], p[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const int i = i0 + u * NT;
            if (i < nel) {
                const int l = i / W, c = i % W, m = l >> P.lgTR, rr = rt * P.TR + (l & (P.TR - 1));
                o[u] = obj[(size_t)(ar + rr) * P.Wc + ac + c];
                p[u] = probes[m * WW + (size_t)rr * W + c];
            }
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const int i = i0 + u * NT;
            if (i < nel) {
                const int l = i / W, c = i % W, m = l >> P.lgTR, rr = rt * P.TR + (l & (P.TR - 1));
                if (m == 0) {
                    om = fmax(om, norm2(o[u]));
                    if (stg) stg[(size_t)rr * W + c] = o[u];          // sensor input o_j (posref.py:66)
                }
                tile[(size_t)l * LS + pad<W>(c)] = scale(p[u] * o[u], checker<T>(rr, c));
            }
        }
    }
    om = block_max(om, red);
    if (threadIdx.x == 0) reinterpret_cast<T*>(P.omax_part)[(size_t)k * P.nRT + rt] = om;
    __syncthreads();
    lines_fft<T, W, false>(tile, P.TR * M, LS, tw);
    __syncthreads();
    C* scr = reinterpret_cast<C*>(P.scratch) + (size_t)k * M * WW;
    for (int i = threadIdx.x; i < P.TR * M * W; i += NT) {
        const int l = i / W, c = i % W;
        scr[(l >> P.lgTR) * WW + (size_t)(rt * P.TR + (l & (P.TR - 1))) * W + c] = tile[(size_t)l * LS + pad<W>(c)];
    }
}

// column tile <-> padded lines (mode-major lines m*TC + cc)
template <typename T, int W>
__device__ __forceinline__ void bk_load_cols(cplx<T>* tile, const cplx<T>* scr, int M, int TC, int lgTC, int ct) {
    constexpr int LS = line_stride<W>(), U = 8;
    const size_t WW = (size_t)W * W;
    const int nel = M * W * TC;
    for (int i0 = threadIdx.x; i0 < nel; i0 += blockDim.x * U) {
        cplx<T> v[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const int i = i0 + u * blockDim.x;
            if (i < nel) {
                const int rem = i & ((W << lgTC) - 1), m = i >> (lgTC + Log2<W>::value);
                v[u] = scr[m * WW + (size_t)(rem >> lgTC) * W + ct * TC + (rem & (TC - 1))];
            }
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const int i = i0 + u * blockDim.x;
            if (i < nel) {
                const int rem = i & ((W << lgTC) - 1), m = i >> (lgTC + Log2<W>::value);
                tile[(size_t)((m << lgTC) + (rem & (TC - 1))) * LS + pad<W>(rem >> lgTC)] = v[u];
            }
        }
    }
}
template <typename T, int W>
__device__ __forceinline__ void bk_store_cols(const cplx<T>* tile, cplx<T>* scr, int M, int TC, int lgTC, int ct) {
    constexpr int LS = line_stride<W>();
    const size_t WW = (size_t)W * W;
    for (int i = threadIdx.x; i < M * W * TC; i += blockDim.x) {
        const int rem = i & ((W << lgTC) - 1), m = i >> (lgTC + Log2<W>::value);
        const int r = rem >> lgTC, cc = rem & (TC - 1);
        scr[m * WW + (size_t)r * W + ct * TC + cc] = tile[(size_t)((m << lgTC) + cc) * LS + pad<W>(r)];
    }
}

// K2: column DFTs; Psi stored back; max(total) partials (engine.py:114-117)
template <typename T, int W>
__global__ void __launch_bounds__(kBatThreads) bk_cols_fwd(const __grid_constant__ BatchDev P) {
    using C = cplx<T>;
    constexpr int LS = line_stride<W>();
    extern __shared__ __align__(16) unsigned char smem_raw[];
    C* tw = reinterpret_cast<C*>(smem_raw);
    T* red = reinterpret_cast<T*>(tw + W);
    C* tile = reinterpret_cast<C*>(red + 64);
    load_twiddles<T, W>(tw, reinterpret_cast<const C*>(P.twiddles));
    if (*(volatile const int*)P.status) return;
    const int k = blockIdx.x / P.nCT, ct = blockIdx.x % P.nCT, M = P.M;
    C* scr = reinterpret_cast<C*>(P.scratch) + (size_t)k * M * W * W;
    bk_load_cols<T, W>(tile, scr, M, P.TC, P.lgTC, ct);
    __syncthreads();
    lines_fft<T, W, false>(tile, M * P.TC, LS, tw);
    __syncthreads();
    const T invW2 = T(1) / (T(W) * T(W));
    T tm = T(0);
    for (int i = threadIdx.x; i < W * P.TC; i += blockDim.x) {
        const int cc = i / W, r = i % W;
        T tot = T(0);
        for (int m = 0; m < M; ++m) tot += norm2(tile[(size_t)(m * P.TC + cc) * LS + pad<W>(r)]) * invW2;
        tm = fmax(tm, tot);
    }
    tm = block_max(tm, red);
    if (threadIdx.x == 0) reinterpret_cast<T*>(P.tmax_part)[(size_t)k * P.nCT + ct] = tm;
    bk_store_cols<T, W>(tile, scr, M, P.TC, P.lgTC, ct);
}

// K3: modulus constraint (engine.py:117-119), error terms (engine.py:198-202),
// inverse column DFTs
template <typename T, int W>
__global__ void __launch_bounds__(kBatThreads) bk_cols_mod(const __grid_constant__ BatchDev P) {
    using C = cplx<T>;
    constexpr int LS = line_stride<W>();
    extern __shared__ __align__(16) unsigned char smem_raw[];
    C* tw = reinterpret_cast<C*>(smem_raw);
    T* red = reinterpret_cast<T*>(tw + W);
    C* tile = reinterpret_cast<C*>(red + 64);
    load_twiddles<T, W>(tw, reinterpret_cast<const C*>(P.twiddles));
    if (*(volatile const int*)P.status) return;
    const int k = blockIdx.x / P.nCT, ct = blockIdx.x % P.nCT, M = P.M;
    const size_t WW = (size_t)W * W;
    const int j = P.batch[k];
    C* scr = reinterpret_cast<C*>(P.scratch) + (size_t)k * M * WW;
    bk_load_cols<T, W>(tile, scr, M, P.TC, P.lgTC, ct);
    const T tmax = bk_max_of(reinterpret_cast<const T*>(P.tmax_part) + (size_t)k * P.nCT, P.nCT);
    const T eps = T(P.eps_rel) * fmax(tmax, real_limits<T>::tiny());
    const T* I = reinterpret_cast<const T*>(P.patterns) + (size_t)j * WW;
    C* stg = P.sense == PTY_SENSE_XCORR_B ? reinterpret_cast<C*>(P.stage) + (size_t)j * 2 * WW : nullptr;
    const T invW2 = T(1) / (T(W) * T(W));
    __syncthreads();
    double en = 0.0, ed = 0.0;
    T worst = T(0);
    for (int i = threadIdx.x; i < W * P.TC; i += blockDim.x) {
        const int r = i >> P.lgTC, cc = i & (P.TC - 1), c = ct * P.TC + cc;
        T tot = T(0);
        for (int m = 0; m < M; ++m) tot += norm2(tile[(size_t)(m * P.TC + cc) * LS + pad<W>(r)]) * invW2;
        const T Iv = I[(size_t)r * W + c];
        const T sI = sqrt_rn(Iv);
        const T sc = sI / sqrt_rn(tot + eps);
        const T d = sqrt_rn(tot) - sI;
        en += (double)(d * d);
        ed += (double)Iv;
        T after = T(0);
        for (int m = 0; m < M; ++m) {
            C& a = tile[(size_t)(m * P.TC + cc) * LS + pad<W>(r)];
            a = scale(a, sc);
            after += norm2(a) * invW2;
        }
        if (P.track_mod && tot > T(1e-3) * tmax) worst = fmax(worst, fabs(after - Iv) / fmax(Iv, real_limits<T>::tiny()));
        if (stg) {
            stg[(size_t)r * W + c] = C{tot, T(0)};
            stg[WW + (size_t)r * W + c] = C{Iv, T(0)};
        }
    }
    __syncthreads();
    lines_fft<T, W, true>(tile, M * P.TC, LS, tw);
    __syncthreads();
    double* dred = reinterpret_cast<double*>(red);
    en = block_sum(en, dred);
    ed = block_sum(ed, dred);
    worst = block_max(worst, red);
    if (threadIdx.x == 0) {
        double* e = P.err_part + ((size_t)(P.visit0 + k) * P.nCT + ct) * 3;
        e[0] = en;
        e[1] = ed;
        e[2] = (double)worst;
    }
    bk_store_cols<T, W>(tile, scr, M, P.TC, P.lgTC, ct);
}

// K4: inverse row DFTs and the update contributions.  CTA = (row tile, group g);
// it walks the positions k = g, g + G, ... in order, so its probe partial is a
// fixed-order sum.  Probe accumulators for the tile rows live in shared memory.
template <typename T, int W>
__global__ void __launch_bounds__(kBatThreads) bk_rows_inv(const __grid_constant__ BatchDev P) {
    using C = cplx<T>;
    constexpr int LS = line_stride<W>();
    extern __shared__ __align__(16) unsigned char smem_raw[];
    C* tw = reinterpret_cast<C*>(smem_raw);
    T* red = reinterpret_cast<T*>(tw + W);
    C* tile = reinterpret_cast<C*>(red + 64);
    const int M = P.M, NT = blockDim.x;
    C* pnum = tile + (size_t)P.TR * M * LS;                  // [M][TR*W]
    T* pden = reinterpret_cast<T*>(pnum + (size_t)M * P.TR * W);   // [TR*W]
    load_twiddles<T, W>(tw, reinterpret_cast<const C*>(P.twiddles));
    if (*(volatile const int*)P.status) return;
    const int rt = blockIdx.x % P.nRT, g = blockIdx.x / P.nRT;
    const size_t WW = (size_t)W * W;
    const int npx = P.TR * W;
    for (int i = threadIdx.x; i < M * npx; i += NT) pnum[i] = C{T(0), T(0)};
    for (int i = threadIdx.x; i < npx; i += NT) pden[i] = T(0);
    const C* obj = reinterpret_cast<const C*>(P.obj);
    const C* probes = reinterpret_cast<const C*>(P.probes);
    const T invW2 = T(1) / (T(W) * T(W));
    const T alpha_p = T(P.alpha_p), beta = T(P.beta);
    for (int k = g; k < P.b; k += P.G) {
        const C* scr = reinterpret_cast<const C*>(P.scratch) + (size_t)k * M * WW;
        __syncthreads();
        constexpr int U = 8;
        const int nel = P.TR * M * W;
        for (int i0 = threadIdx.x; i0 < nel; i0 += NT * U) {
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
        }
        __syncthreads();
        lines_fft<T, W, true>(tile, P.TR * M, LS, tw);
        __syncthreads();
        const int ar = P.anchors[2 * k], ac = P.anchors[2 * k + 1];
        const T omax = bk_max_of(reinterpret_cast<const T*>(P.omax_part) + (size_t)k * P.nRT, P.nRT);
        if (P.update_probe && omax == T(0)) {            // engine.py:145-147
            if (threadIdx.x == 0) atomicOr(P.status, PTY_ERR_OBJECT_ZERO);
            continue;
        }
        C* onum = reinterpret_cast<C*>(P.onum) + (size_t)k * WW;
        for (int i = threadIdx.x; i < npx; i += NT) {
            const int r = i / W, c = i % W, rr = rt * P.TR + r;
            const C o = obj[(size_t)(ar + rr) * P.Wc + ac + c];
            const T sg = checker<T>(rr, c) * invW2;
            C numer{T(0), T(0)};
            for (int m = 0; m < M; ++m) {
                const C pv = probes[m * WW + (size_t)rr * W + c];
                const C d = scale(tile[(size_t)((m << P.lgTR) + r) * LS + pad<W>(c)], sg) - pv * o;
                numer = numer + mulc(d, pv);                                   // engine.py:130-131
                if (P.update_probe) pnum[(size_t)m * npx + i] = pnum[(size_t)m * npx + i] + mulc(scale(d, alpha_p), o);
            }
            onum[(size_t)rr * W + c] = numer;
            if (P.update_probe) pden[i] += beta * omax + (T(1) - beta) * norm2(o);   // engine.py:148
        }
    }
    __syncthreads();
    T* pg = reinterpret_cast<T*>(P.pgroup) + (size_t)g * (2 * M + 1) * WW;
    for (int i = threadIdx.x; i < npx; i += NT) {
        const size_t off = (size_t)rt * npx + i;
        for (int m = 0; m < M; ++m) {
            pg[(size_t)(2 * m) * WW + off] = pnum[(size_t)m * npx + i].re;
            pg[(size_t)(2 * m + 1) * WW + off] = pnum[(size_t)m * npx + i].im;
        }
        pg[(size_t)(2 * M) * WW + off] = pden[i];
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
template <typename T, int W>
__global__ void __launch_bounds__(256) bk_obj_gather(const __grid_constant__ BatchDev P) {
    using C = cplx<T>;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    int* list = reinterpret_cast<int*>(smem_raw);            // [b]
    __shared__ int wcount[8], total;
    const int tiles_x = (P.Wc + kObjTile - 1) / kObjTile;
    const int ty = blockIdx.x / tiles_x, tx = blockIdx.x % tiles_x;
    const int R0 = ty * kObjTile, C0 = tx * kObjTile;
    if (threadIdx.x == 0) total = 0;
    __syncthreads();
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    for (int base = 0; base < P.b; base += blockDim.x) {
        const int k = base + threadIdx.x;
        bool cov = false;
        if (k < P.b) {
            const int ar = P.anchors[2 * k], ac = P.anchors[2 * k + 1];
            cov = ar < R0 + kObjTile && ar + W > R0 && ac < C0 + kObjTile && ac + W > C0;
        }
        const unsigned bal = __ballot_sync(0xffffffffu, cov);
        if (lane == 0) wcount[wid] = __popc(bal);
        __syncthreads();
        int off = total;
        for (int w = 0; w < wid; ++w) off += wcount[w];
        if (cov) list[off + __popc(bal & ((1u << lane) - 1u))] = k;
        __syncthreads();
        if (threadIdx.x == 0) for (int w = 0; w < (int)(blockDim.x >> 5); ++w) total += wcount[w];
        __syncthreads();
    }
    const T* pp = reinterpret_cast<const T*>(P.pp);
    const T peak = bk_max_of(reinterpret_cast<const T*>(P.pp_part), P.nRT);
    if (peak == T(0)) {                                       // engine.py:132-134
        if (threadIdx.x == 0) atomicOr(P.status, PTY_ERR_PROBE_ZERO);
        return;
    }
    const T gamma = T(P.gamma);
    const C* onum = reinterpret_cast<const C*>(P.onum);
    T* acc = reinterpret_cast<T*>(P.obj_acc);
    const size_t HW = (size_t)P.H * P.Wc;
    const size_t WW = (size_t)W * W;
    constexpr int PX = kObjTile * kObjTile / 256;             // pixels per thread
    C num[PX];
    T den[PX];
#pragma unroll
    for (int q = 0; q < PX; ++q) { num[q] = C{T(0), T(0)}; den[q] = T(0); }
    for (int t = 0; t < total; ++t) {
        const int k = list[t];
        const int ar = P.anchors[2 * k], ac = P.anchors[2 * k + 1];
#pragma unroll
        for (int q = 0; q < PX; ++q) {
            const int p = threadIdx.x + q * 256, R = R0 + p / kObjTile, Cc = C0 + p % kObjTile;
            const int r = R - ar, c = Cc - ac;
            if (R < P.H && Cc < P.Wc && r >= 0 && r < W && c >= 0 && c < W) {
                num[q] = num[q] + onum[(size_t)k * WW + (size_t)r * W + c];
                den[q] += gamma * peak + (T(1) - gamma) * pp[(size_t)r * W + c];
            }
        }
    }
#pragma unroll
    for (int q = 0; q < PX; ++q) {
        const int p = threadIdx.x + q * 256, R = R0 + p / kObjTile, Cc = C0 + p % kObjTile;
        if (R < P.H && Cc < P.Wc) {
            const size_t o = (size_t)R * P.Wc + Cc;
            acc[o] = num[q].re;
            acc[HW + o] = num[q].im;
            acc[2 * HW + o] = den[q];
        }
    }
}

// per-tile maxima of the accumulated object denominator (after any all-reduce)
template <typename T, int W>
__global__ void __launch_bounds__(256) bk_obj_tile_max(const __grid_constant__ BatchDev P) {
    __shared__ T red[32];
    const int tiles_x = (P.Wc + kObjTile - 1) / kObjTile;
    const int ty = blockIdx.x / tiles_x, tx = blockIdx.x % tiles_x;
    const T* den = reinterpret_cast<const T*>(P.obj_acc) + 2 * (size_t)P.H * P.Wc;
    T m = T(0);
    for (int p = threadIdx.x; p < kObjTile * kObjTile; p += blockDim.x) {
        const int R = ty * kObjTile + p / kObjTile, Cc = tx * kObjTile + p % kObjTile;
        if (R < P.H && Cc < P.Wc) m = fmax(m, den[(size_t)R * P.Wc + Cc]);
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
        const T den = acc[2 * HW + i];
        const C o = obj[i];
        C u = o;
        if (den > T(0)) {
            u = o + divr(scale(C{acc[i], acc[HW + i]}, alpha_o), den + eps_rel * dmax);
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
