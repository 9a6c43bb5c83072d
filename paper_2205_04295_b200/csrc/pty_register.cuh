// pty_register.cuh -- batched Guizar-Sicairos subpixel registration
// (registration.py:43-128) and the per-position Adam controller
// (posref.py:87-113).
//
// Pipeline for n pairs (ref = plane 0, mov = plane 1 of `work`):
//   reg_rows_fwd   : row DFTs of both planes (uncentered np.fft.fft2)
//   reg_cols       : column DFTs, xps = F(ref) conj(F(mov)) -> plane 0,
//                    max|xps| partials (DegenerateInputError test,
//                    registration.py:49-52); for "raw" weighting also the
//                    inverse column DFT of xps -> plane 1
//   reg_whiten     : ("phase" only) xps / (|xps| + 1e-12 max) then inverse cols
//   reg_rows_inv   : inverse row DFTs, |ifft2(xps)| and the coarse argmax with
//                    the reference tie-break (registration.py:67-81)
//   reg_refine     : upsampled DFT on the floor(1.5 kappa)|odd grid around the
//                    coarse peak (registration.py:84-120); the phases
//                    2 pi rows fy / W are reduced exactly in integers
//   reg_finalize   : first max in row-major order -> (dy, dx, peak, ok)
#pragma once
#include "pty_fft.cuh"

namespace pty {

constexpr int kRegThreads = 256;
// rows of the upsampled grid per CTA (keeps 2 * rows * W complex in shared memory)
// 64 KB of shared memory per CTA (several CTAs per SM): 4..16 rows
template <typename T, int W> __host__ __device__ constexpr int refine_rows() {
    return 32768 / (W * (int)sizeof(cplx<T>)) < 4 ? 4 : (32768 / (W * (int)sizeof(cplx<T>)) > 16 ? 16 : 32768 / (W * (int)sizeof(cplx<T>)));
}
template <typename T, int W> __host__ __device__ constexpr size_t refine_smem() {
    return (size_t)2 * refine_rows<T, W>() * W * sizeof(cplx<T>);
}

struct ArgPart {        // coarse partial: max value and tie-break key
    double val;
    long long key;
};
struct RefPart {        // refine partial: max value and flat row-major index
    double val;
    long long idx;
};

// signed lag of an unshifted correlation index, (-W/2, W/2] (registration.py:59-64)
__device__ __forceinline__ int lag_of(int u, int W) { return u <= W / 2 ? u : u - W; }
// DFT frequency of index u, np.fft.fftfreq(W) * W: [-W/2, W/2) (registration.py:92-93)
__device__ __forceinline__ int freq_of(int u, int W) { return u < W / 2 ? u : u - W; }

template <typename T, int W>
__global__ void __launch_bounds__(kRegThreads) reg_rows_fwd(cplx<T>* work, const T* ref_real, const T* mov_real,
                                                            int real_inputs, int n, int TR, const cplx<T>* twg) {
    using C = cplx<T>;
    constexpr int LS = line_stride<W>();
    extern __shared__ __align__(16) unsigned char smem_raw[];
    C* tw = reinterpret_cast<C*>(smem_raw);
    C* tile = tw + W;
    load_twiddles<T, W>(tw, twg);
    const int nRT = W / TR;
    const int pr = blockIdx.x / nRT, rt = blockIdx.x % nRT;
    if (pr >= n) return;
    const size_t WW = (size_t)W * W;
    for (int i = threadIdx.x; i < 2 * TR * W; i += blockDim.x) {
        const int pl = i / (TR * W), rem = i % (TR * W), r = rem / W, c = rem % W;
        const size_t off = (size_t)(rt * TR + r) * W + c;
        C v;
        if (real_inputs == 2) {            // complex64 pairs [n][2][W][W] (ref_real), widened on load
            const float2 x = reinterpret_cast<const float2*>(ref_real)[((size_t)pr * 2 + pl) * WW + off];
            v = C{T(x.x), T(x.y)};
        } else if (real_inputs) {
            v = C{(pl ? mov_real : ref_real)[(size_t)pr * WW + off], T(0)};
        } else {
            v = work[((size_t)pr * 2 + pl) * WW + off];
        }
        tile[(size_t)(pl * TR + r) * LS + pad<W>(c)] = v;
    }
    __syncthreads();
    lines_fft<T, W, false>(tile, 2 * TR, LS, tw);
    __syncthreads();
    for (int i = threadIdx.x; i < 2 * TR * W; i += blockDim.x) {
        const int pl = i / (TR * W), rem = i % (TR * W), r = rem / W, c = rem % W;
        work[((size_t)pr * 2 + pl) * WW + (size_t)(rt * TR + r) * W + c] = tile[(size_t)(pl * TR + r) * LS + pad<W>(c)];
    }
}

// xps and (raw) its inverse column DFT.  mx_part[pr][ct] = max |xps| on the tile.
template <typename T, int W>
__global__ void __launch_bounds__(kRegThreads) reg_cols(cplx<T>* work, int n, int TC, int raw, T* mx_part,
                                                        const cplx<T>* twg) {
    using C = cplx<T>;
    constexpr int LS = line_stride<W>();
    extern __shared__ __align__(16) unsigned char smem_raw[];
    C* tw = reinterpret_cast<C*>(smem_raw);
    T* red = reinterpret_cast<T*>(tw + W);
    C* tile = reinterpret_cast<C*>(red + 64);
    load_twiddles<T, W>(tw, twg);
    const int nCT = W / TC;
    const int pr = blockIdx.x / nCT, ct = blockIdx.x % nCT;
    if (pr >= n) return;
    const size_t WW = (size_t)W * W;
    C* p0 = work + (size_t)pr * 2 * WW;
    for (int i = threadIdx.x; i < 2 * W * TC; i += blockDim.x) {
        const int pl = i / (W * TC), rem = i % (W * TC), r = rem / TC, cc = rem % TC;
        tile[(size_t)(pl * TC + cc) * LS + pad<W>(r)] = p0[pl * WW + (size_t)r * W + ct * TC + cc];
    }
    __syncthreads();
    lines_fft<T, W, false>(tile, 2 * TC, LS, tw);
    __syncthreads();
    T mx = T(0);
    for (int i = threadIdx.x; i < W * TC; i += blockDim.x) {
        const int r = i / TC, cc = i % TC;
        C& a = tile[(size_t)cc * LS + pad<W>(r)];
        const C b = tile[(size_t)(TC + cc) * LS + pad<W>(r)];
        a = mulc(a, b);                                   // F(ref) * conj(F(mov))
        mx = fmax(mx, sqrt(norm2(a)));
        p0[(size_t)r * W + ct * TC + cc] = a;             // plane 0 <- xps
    }
    mx = block_max(mx, red);
    if (threadIdx.x == 0) mx_part[(size_t)pr * nCT + ct] = mx;
    if (!raw) return;
    __syncthreads();
    lines_fft<T, W, true>(tile, TC, LS, tw);
    __syncthreads();
    for (int i = threadIdx.x; i < W * TC; i += blockDim.x) {
        const int r = i / TC, cc = i % TC;
        p0[WW + (size_t)r * W + ct * TC + cc] = tile[(size_t)cc * LS + pad<W>(r)];
    }
}

// "phase" weighting (registration.py:55): xps / (|xps| + 1e-12 * max|xps|)
template <typename T, int W>
__global__ void __launch_bounds__(kRegThreads) reg_whiten(cplx<T>* work, int n, int TC, const T* mx_part,
                                                          const cplx<T>* twg) {
    using C = cplx<T>;
    constexpr int LS = line_stride<W>();
    extern __shared__ __align__(16) unsigned char smem_raw[];
    C* tw = reinterpret_cast<C*>(smem_raw);
    C* tile = tw + W;
    load_twiddles<T, W>(tw, twg);
    const int nCT = W / TC;
    const int pr = blockIdx.x / nCT, ct = blockIdx.x % nCT;
    if (pr >= n) return;
    T mx = T(0);
    for (int k = 0; k < nCT; ++k) mx = fmax(mx, mx_part[(size_t)pr * nCT + k]);
    const T guard = T(1e-12) * mx;
    const size_t WW = (size_t)W * W;
    C* p0 = work + (size_t)pr * 2 * WW;
    for (int i = threadIdx.x; i < W * TC; i += blockDim.x) {
        const int r = i / TC, cc = i % TC;
        const size_t off = (size_t)r * W + ct * TC + cc;
        C a = p0[off];
        const T mag = sqrt(norm2(a));
        a = divr(a, mag + guard);
        p0[off] = a;
        tile[(size_t)cc * LS + pad<W>(r)] = a;
    }
    __syncthreads();
    lines_fft<T, W, true>(tile, TC, LS, tw);
    __syncthreads();
    for (int i = threadIdx.x; i < W * TC; i += blockDim.x) {
        const int r = i / TC, cc = i % TC;
        p0[WW + (size_t)r * W + ct * TC + cc] = tile[(size_t)cc * LS + pad<W>(r)];
    }
}

__device__ __forceinline__ bool arg_better(double v, long long k, double bv, long long bk) {
    return v > bv || (v == bv && k < bk);
}

// inverse row DFTs of plane 1 and the coarse argmax partial per (pair, row tile)
template <typename T, int W>
__global__ void __launch_bounds__(kRegThreads) reg_rows_inv(cplx<T>* work, int n, int TR, ArgPart* part,
                                                            const cplx<T>* twg) {
    using C = cplx<T>;
    constexpr int LS = line_stride<W>();
    extern __shared__ __align__(16) unsigned char smem_raw[];
    C* tw = reinterpret_cast<C*>(smem_raw);
    C* tile = tw + W;
    __shared__ double sv[kRegThreads / 32];
    __shared__ long long sk[kRegThreads / 32];
    load_twiddles<T, W>(tw, twg);
    const int nRT = W / TR;
    const int pr = blockIdx.x / nRT, rt = blockIdx.x % nRT;
    if (pr >= n) return;
    const size_t WW = (size_t)W * W;
    C* p1 = work + ((size_t)pr * 2 + 1) * WW + (size_t)rt * TR * W;
    for (int i = threadIdx.x; i < TR * W; i += blockDim.x) {
        const int r = i / W, c = i % W;
        tile[(size_t)r * LS + pad<W>(c)] = p1[i];
    }
    __syncthreads();
    lines_fft<T, W, true>(tile, TR, LS, tw);
    __syncthreads();
    const T invW2 = T(1) / (T(W) * T(W));
    double bv = -1.0;
    long long bk = 0x7fffffffffffffffLL;
    for (int i = threadIdx.x; i < TR * W; i += blockDim.x) {
        const int r = i / W, c = i % W;
        const C a = tile[(size_t)r * LS + pad<W>(c)];
        const double v = (double)(sqrt(norm2(a)) * invW2);
        const int dy = lag_of(rt * TR + r, W), dx = lag_of(c, W);
        const long long s = (long long)(abs(dy) + abs(dx));
        const long long key = (s * (W + 1) + (dy + W / 2)) * (W + 1) + (dx + W / 2);
        if (arg_better(v, key, bv, bk)) { bv = v; bk = key; }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        const double ov = __shfl_xor_sync(0xffffffffu, bv, o);
        const long long ok = __shfl_xor_sync(0xffffffffu, bk, o);
        if (arg_better(ov, ok, bv, bk)) { bv = ov; bk = ok; }
    }
    if ((threadIdx.x & 31) == 0) { sv[threadIdx.x >> 5] = bv; sk[threadIdx.x >> 5] = bk; }
    __syncthreads();
    if (threadIdx.x == 0) {
        bv = sv[0];
        bk = sk[0];
        for (int w = 1; w < (int)(blockDim.x >> 5); ++w)
            if (arg_better(sv[w], sk[w], bv, bk)) { bv = sv[w]; bk = sk[w]; }
        part[(size_t)pr * nRT + rt] = ArgPart{bv, bk};
    }
}

__device__ __forceinline__ void coarse_of(const ArgPart* part, int nRT, int W, double* peak, int* cdy, int* cdx) {
    double bv = -1.0;
    long long bk = 0x7fffffffffffffffLL;
    for (int k = 0; k < nRT; ++k)
        if (arg_better(part[k].val, part[k].key, bv, bk)) { bv = part[k].val; bk = part[k].key; }
    const long long dxs = bk % (W + 1), dys = (bk / (W + 1)) % (W + 1);
    *peak = bv;
    *cdy = (int)dys - W / 2;
    *cdx = (int)dxs - W / 2;
}

// Upsampled DFT around the coarse peak.  CTA = (pair, block of kRefineRows grid rows).
//   U[i][v] = sum_u exp(2 pi i rows_i fy_u / W) xps[u][v]
//   R[i][k] = sum_v U[i][v] exp(2 pi i fx_v cols_k / W) / W^2
// With rows_i = dy + (i - h)/kappa, the phase in turns is
//   ((dy*kappa + i - h) * fy_u mod kappa W) / (kappa W)  -- exact integer reduction.
template <typename T, int W>
__global__ void __launch_bounds__(kRegThreads) reg_refine(const cplx<T>* work, int n, int kappa, int npts,
                                                          const ArgPart* cpart, int nRT, RefPart* rpart) {
    using C = cplx<T>;
    constexpr int VPT = (W + kRegThreads - 1) / kRegThreads;   // columns v per thread
    constexpr int kRefineRows = refine_rows<T, W>();
    constexpr int kRefineCols = kRefineRows;                   // grid columns per chunk: ec fits in er
    static_assert(W * kRefineCols <= 2 * kRefineRows * W, "ec overruns the refine shared memory");
    extern __shared__ __align__(16) unsigned char smem_raw[];
    C* er = reinterpret_cast<C*>(smem_raw);                    // [kRefineRows][W]
    C* U = er + kRefineRows * W;                               // [kRefineRows][W]
    C* ec = er;                                                // [W][kRefineCols], after er is dead
    __shared__ double sv[kRegThreads / 32];
    __shared__ long long sk[kRegThreads / 32];
    const int nIB = (npts + kRefineRows - 1) / kRefineRows;
    const int pr = blockIdx.x / nIB, ib = blockIdx.x % nIB;
    if (pr >= n) return;
    double cpeak;
    int cdy, cdx;
    coarse_of(cpart + (size_t)pr * nRT, nRT, W, &cpeak, &cdy, &cdx);
    const int h = npts / 2;
    const long long KW = (long long)kappa * W;
    const int i0 = ib * kRefineRows;
    for (int t = threadIdx.x; t < kRefineRows * W; t += blockDim.x) {
        const int i = t / W, u = t % W;
        const long long q = (long long)cdy * kappa + (i0 + i) - h;
        long long ph = (q * freq_of(u, W)) % KW;
        if (ph < 0) ph += KW;
        T s, c;
        sincospi(T(2.0 * (double)ph / (double)KW), &s, &c);
        er[t] = C{c, s};
    }
    __syncthreads();
    const size_t WW = (size_t)W * W;
    const C* xps = work + (size_t)pr * 2 * WW;
    C acc[VPT][kRefineRows];
#pragma unroll
    for (int q = 0; q < VPT; ++q)
#pragma unroll
        for (int i = 0; i < kRefineRows; ++i) acc[q][i] = C{T(0), T(0)};
#pragma unroll 4
    for (int u = 0; u < W; ++u) {                              // 4 rows of xps in flight per thread
#pragma unroll
        for (int q = 0; q < VPT; ++q) {
            const int v = threadIdx.x + q * kRegThreads;
            if (v < W) {
                const C x = xps[(size_t)u * W + v];
#pragma unroll
                for (int i = 0; i < kRefineRows; ++i) acc[q][i] = acc[q][i] + er[i * W + u] * x;
            }
        }
    }
#pragma unroll
    for (int q = 0; q < VPT; ++q) {
        const int v = threadIdx.x + q * kRegThreads;
        if (v < W)
#pragma unroll
            for (int i = 0; i < kRefineRows; ++i) U[i * W + v] = acc[q][i];
    }
    const T invW2 = T(1) / (T(W) * T(W));
    double bv = -1.0;
    long long bk = 0x7fffffffffffffffLL;
    for (int k0 = 0; k0 < npts; k0 += kRefineCols) {
        __syncthreads();
        for (int t = threadIdx.x; t < W * kRefineCols; t += blockDim.x) {
            const int v = t / kRefineCols, kk = t % kRefineCols;
            const long long q = (long long)cdx * kappa + (k0 + kk) - h;
            long long ph = (q * freq_of(v, W)) % KW;
            if (ph < 0) ph += KW;
            T s, c;
            sincospi(T(2.0 * (double)ph / (double)KW), &s, &c);
            ec[t] = C{c, s};
        }
        __syncthreads();
        for (int t = threadIdx.x; t < kRefineRows * kRefineCols; t += blockDim.x) {
            const int i = t / kRefineCols, kk = t % kRefineCols;
            if (i0 + i >= npts || k0 + kk >= npts) continue;
            C r{T(0), T(0)};
            for (int v = 0; v < W; ++v) r = r + U[i * W + v] * ec[v * kRefineCols + kk];
            const double val = (double)(sqrt(norm2(r)) * invW2);
            const long long idx = (long long)(i0 + i) * npts + (k0 + kk);
            if (arg_better(val, idx, bv, bk)) { bv = val; bk = idx; }
        }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        const double ov = __shfl_xor_sync(0xffffffffu, bv, o);
        const long long ok = __shfl_xor_sync(0xffffffffu, bk, o);
        if (arg_better(ov, ok, bv, bk)) { bv = ov; bk = ok; }
    }
    if ((threadIdx.x & 31) == 0) { sv[threadIdx.x >> 5] = bv; sk[threadIdx.x >> 5] = bk; }
    __syncthreads();
    if (threadIdx.x == 0) {
        bv = sv[0];
        bk = sk[0];
        for (int w = 1; w < (int)(blockDim.x >> 5); ++w)
            if (arg_better(sv[w], sk[w], bv, bk)) { bv = sv[w]; bk = sk[w]; }
        rpart[(size_t)pr * nIB + ib] = RefPart{bv, bk};
    }
}

template <typename T>
__global__ void reg_finalize(int n, int W, int kappa, int npts, int kRefineRows, const T* mx_part, int nCT,
                             const ArgPart* cpart, int nRT, const RefPart* rpart,
                             double* dy, double* dx, double* peak, int* ok) {
    const int pr = blockIdx.x * blockDim.x + threadIdx.x;
    if (pr >= n) return;
    T mx = T(0);
    for (int k = 0; k < nCT; ++k) mx = fmax(mx, mx_part[(size_t)pr * nCT + k]);
    ok[pr] = mx > T(0);
    double cpeak;
    int cdy, cdx;
    coarse_of(cpart + (size_t)pr * nRT, nRT, W, &cpeak, &cdy, &cdx);
    if (kappa == 1) {
        dy[pr] = (double)cdy;
        dx[pr] = (double)cdx;
        peak[pr] = cpeak;
        return;
    }
    const int nIB = (npts + kRefineRows - 1) / kRefineRows;
    double bv = -1.0;
    long long bk = 0x7fffffffffffffffLL;
    for (int b = 0; b < nIB; ++b) {
        const RefPart p = rpart[(size_t)pr * nIB + b];
        if (arg_better(p.val, p.idx, bv, bk)) { bv = p.val; bk = p.idx; }
    }
    const int h = npts / 2;
    const int iy = (int)(bk / npts), ix = (int)(bk % npts);
    // rows = coarse.dy + arange(-h, h+1)/kappa  (registration.py:104,115-116), float64
    dy[pr] = (double)cdy + (double)(iy - h) / (double)kappa;
    dx[pr] = (double)cdx + (double)(ix - h) / (double)kappa;
    peak[pr] = bv;
}

// posref.py:87-113: Adam recurrence in float64 and clamp, one thread per sensed entry
static __global__ void adam_kernel(double* pos, double* m, double* v, long long* t, const double* gx,
                            const double* gy, const int* ok, const int* index, int n, double step,
                            double b1, double b2, double eps, double clip, double xmin, double ymin,
                            double xmax, double ymax) {
    const int k = blockIdx.x * blockDim.x + threadIdx.x;
    if (k >= n || !ok[k]) return;
    const int j = index ? index[k] : k;
    const long long tj = ++t[j];
    const double g[2] = {gx[k], gy[k]};
    double d[2];
    const double c1 = 1.0 - pow(b1, (double)tj), c2 = 1.0 - pow(b2, (double)tj);
#pragma unroll
    for (int a = 0; a < 2; ++a) {
        // no FMA contraction: same rounding sequence as numpy
        const double mm = __dadd_rn(__dmul_rn(b1, m[2 * j + a]), __dmul_rn(1.0 - b1, g[a]));
        const double vv = __dadd_rn(__dmul_rn(b2, v[2 * j + a]), __dmul_rn(__dmul_rn(1.0 - b2, g[a]), g[a]));
        m[2 * j + a] = mm;
        v[2 * j + a] = vv;
        const double mh = mm / c1, vh = vv / c2;
        const double dd = __dmul_rn(step, mh) / __dadd_rn(sqrt(vh), eps);
        d[a] = fmin(fmax(dd, -clip), clip);
    }
    const double x = __dadd_rn(pos[2 * j], d[0]), y = __dadd_rn(pos[2 * j + 1], d[1]);
    pos[2 * j] = fmin(fmax(x, xmin), xmax);
    pos[2 * j + 1] = fmin(fmax(y, ymin), ymax);
}

}  // namespace pty
