// pty_visit.cu -- the reference's per-visit and per-pair public functions as
// C-ABI entry points (include/ptycho_b200.h), for callers that drive single
// visits themselves (the reference's own tests do: pkg/tests/test_engine.py:
// 98-133, test_registration.py:41-113, test_posref.py:67-133).  The fused
// sweep (pty_sweep) evaluates the same expressions inside one launch; these
// entry points compose the building blocks instead:
//
//   pty_magnitude_correct  engine.py:104-120   exit waves, centered FFTs, modulus scale
//   pty_update_object      engine.py:123-137   rPIE object update of one crop
//   pty_update_probe       engine.py:140-150   rPIE probe update of one mode
//   pty_cross_power_spectrum registration.py:43-56
//   pty_coarse_argmax      registration.py:67-81  (argmax + tie-break of |ifft2(xps)|)
//   pty_upsampled_idft     registration.py:84-96
//   pty_argmax_abs         registration.py:117-119 (first maximum, row-major)
//   pty_adam_step          posref.py:87-99
//   pty_apply_correction   posref.py:102-113
//
// Reductions (max over a field) are two-level and deterministic: per-CTA
// partials, then every consumer CTA folds the partials in index order.
// fp64 evaluates numpy's expression order (complex / real = multiply by the
// reciprocal, numpy loops_arithm_fp); fp32 uses IEEE square roots and
// divisions here (no MUFU approximations: these are reference-facing calls).
#include <cuda_runtime.h>

#include "pty_host.cuh"
#include "pty_register.cuh"

namespace pty {

constexpr int kVisThreads = 256;

inline unsigned vis_blocks(long long n) { return (unsigned)std::min<long long>((n + kVisThreads - 1) / kVisThreads, 1024); }

template <typename T>
__device__ __forceinline__ T fold_max(const T* part, int nparts) {
    T m = T(0);
    for (int k = 0; k < nparts; ++k) m = fmax(m, part[k]);
    return m;
}

template <typename T>
__device__ __forceinline__ void store_block_max(T v, T* part) {
    __shared__ T red[32];
    v = block_max(v, red);
    if (threadIdx.x == 0) part[blockIdx.x] = v;
}

// psi[m] = P_m * o (engine.py:113) and the I < 0 check (engine.py:111-112)
template <typename T>
__global__ void __launch_bounds__(kVisThreads) vis_exit_kernel(const cplx<T>* probes, const cplx<T>* o, const T* I,
                                                               int M, long long WW, cplx<T>* psi, int* status) {
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < WW; i += (long long)gridDim.x * blockDim.x) {
        if (I[i] < T(0)) atomicOr(status, PTY_ERR_NEGATIVE_I);
        const cplx<T> ov = o[i];
        for (int m = 0; m < M; ++m) psi[m * WW + i] = probes[m * WW + i] * ov;
    }
}

// total = sum_m |psi_m|^2 in mode order (engine.py:114-116), per-CTA max
template <typename T>
__global__ void __launch_bounds__(kVisThreads) vis_total_kernel(const cplx<T>* psi, int M, long long WW, T* total,
                                                                T* part) {
    T mx = T(0);
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < WW; i += (long long)gridDim.x * blockDim.x) {
        T t = T(0);
        for (int m = 0; m < M; ++m) {
            const T a = sqrt_rn(norm2(psi[m * WW + i]));      // np.abs(psi) ** 2
            t += a * a;
        }
        total[i] = t;
        mx = fmax(mx, t);
    }
    store_block_max(mx, part);
}

// scale = sqrt(I) / sqrt(total + eps), corrected_m = scale * psi_m (engine.py:117-119, before the inverse FFT)
template <typename T>
__global__ void __launch_bounds__(kVisThreads) vis_scale_kernel(const cplx<T>* psi, const T* total, const T* I,
                                                                const T* part, int nparts, int M, long long WW,
                                                                double eps_rel, cplx<T>* out, const int* status) {
    if (*(volatile const int*)status) return;
    const T eps = T(eps_rel) * fmax(fold_max(part, nparts), real_limits<T>::tiny());
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < WW; i += (long long)gridDim.x * blockDim.x) {
        const T s = sqrt_rn(I[i]) / sqrt_rn(total[i] + eps);
        for (int m = 0; m < M; ++m) out[m * WW + i] = scale(psi[m * WW + i], s);
    }
}

// sum_m |P_m|^2 (engine.py:129) or |o|^2 (engine.py:145) and per-CTA maxima
template <typename T>
__global__ void __launch_bounds__(kVisThreads) vis_power_kernel(const cplx<T>* f, int M, long long WW, T* power,
                                                                T* part) {
    T mx = T(0);
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < WW; i += (long long)gridDim.x * blockDim.x) {
        T t = T(0);
        for (int m = 0; m < M; ++m) {
            const T a = sqrt_rn(norm2(f[m * WW + i]));        // np.abs(.) ** 2
            t += a * a;
        }
        power[i] = t;
        mx = fmax(mx, t);
    }
    store_block_max(mx, part);
}

// engine.py:123-137: o + alpha numer / (gamma peak + (1 - gamma) pp + eps max(denom))
template <typename T>
__global__ void __launch_bounds__(kVisThreads) vis_update_object_kernel(
    const cplx<T>* o, const cplx<T>* probes, const cplx<T>* corrected, const T* pp, const T* part, int nparts, int M,
    long long WW, double alpha, double gamma, double eps_rel, cplx<T>* out, int* status) {
    const T peak = fold_max(part, nparts);
    if (peak == T(0)) {                                       // engine.py:132-134
        if (blockIdx.x == 0 && threadIdx.x == 0) atomicOr(status, PTY_ERR_PROBE_ZERO);
        return;
    }
    const T g = T(gamma), a = T(alpha);
    const T dmax = g * peak + (T(1) - g) * peak;              // denom.max(): denom is monotone in pp
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < WW; i += (long long)gridDim.x * blockDim.x) {
        const cplx<T> ov = o[i];
        cplx<T> numer{T(0), T(0)};
        for (int m = 0; m < M; ++m) {
            const cplx<T> p = probes[m * WW + i];
            numer = numer + mulc(corrected[m * WW + i] - p * ov, p);
        }
        T den = g * peak + (T(1) - g) * pp[i];
        den = den + T(eps_rel) * dmax;
        out[i] = ov + divr(scale(numer, a), den);
    }
}

// engine.py:140-150 for one mode: P + alpha (psi - P o) conj(o) / (beta peak + (1 - beta)|o|^2 + eps max)
template <typename T>
__global__ void __launch_bounds__(kVisThreads) vis_update_probe_kernel(
    const cplx<T>* probe, const cplx<T>* o, const cplx<T>* corrected, const T* op, const T* part, int nparts,
    long long WW, double alpha, double beta, double eps_rel, cplx<T>* out, int* status) {
    const T peak = fold_max(part, nparts);
    if (peak == T(0)) {                                       // engine.py:145-147
        if (blockIdx.x == 0 && threadIdx.x == 0) atomicOr(status, PTY_ERR_OBJECT_ZERO);
        return;
    }
    const T b = T(beta), a = T(alpha);
    const T dmax = b * peak + (T(1) - b) * peak;
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < WW; i += (long long)gridDim.x * blockDim.x) {
        const cplx<T> ov = o[i], p = probe[i];
        T den = b * peak + (T(1) - b) * op[i];
        den = den + T(eps_rel) * dmax;
        out[i] = p + divr(mulc(scale(corrected[i] - p * ov, a), ov), den);
    }
}

// plane 0 of every (ref, mov) pair after reg_cols / reg_whiten -> xps[n][W][W]; ok = max|xps| > 0
template <typename T>
__global__ void vis_xps_out_kernel(const cplx<T>* work, long long WW, int n, const T* mx_part, int nCT,
                                   cplx<T>* xps, int* ok) {
    const long long total = (long long)n * WW;
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < total; i += (long long)gridDim.x * blockDim.x) {
        const long long pr = i / WW, e = i % WW;
        xps[i] = work[pr * 2 * WW + e];
        if (e == 0) ok[pr] = fold_max(mx_part + pr * nCT, nCT) > T(0);
    }
}

// argmax of |corr| over the fftshifted lags with the reference tie-break
// (min |dy| + |dx|, then dy, then dx; registration.py:67-81); CTA = one field
template <typename T>
__global__ void __launch_bounds__(kVisThreads) vis_coarse_argmax_kernel(const cplx<T>* corr, int W, double* dy,
                                                                        double* dx, double* peak) {
    __shared__ double sv[kVisThreads / 32];
    __shared__ long long sk[kVisThreads / 32];
    const long long WW = (long long)W * W;
    const cplx<T>* f = corr + blockIdx.x * WW;
    double bv = -1.0;
    long long bk = 0x7fffffffffffffffLL;
    for (long long i = threadIdx.x; i < WW; i += blockDim.x) {
        const int u = (int)(i / W), c = (int)(i % W);
        const double v = (double)sqrt_rn(norm2(f[i]));
        const int ly = lag_of(u, W), lx = lag_of(c, W);
        const long long s = (long long)(abs(ly) + abs(lx));
        const long long key = (s * (W + 1) + (ly + W / 2)) * (W + 1) + (lx + W / 2);
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
        dx[blockIdx.x] = (double)(bk % (W + 1) - W / 2);
        dy[blockIdx.x] = (double)((bk / (W + 1)) % (W + 1) - W / 2);
        peak[blockIdx.x] = bv;
    }
}

// upsampled_idft (registration.py:84-96): er[i][u] = exp(2 pi i rows_i fy_u / W),
// ec[v][k] = exp(2 pi i fx_v cols_k / W); out = er @ xps @ ec / W^2.
// Pass 1: U[i][v] = sum_u er[i][u] xps[u][v]; CTA = row i.
template <typename T>
__global__ void __launch_bounds__(kVisThreads) vis_updft_rows_kernel(const cplx<T>* xps, int W, const double* rows,
                                                                     cplx<T>* U) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    cplx<T>* er = reinterpret_cast<cplx<T>*>(smem_raw);
    const int i = blockIdx.x;
    for (int u = threadIdx.x; u < W; u += blockDim.x) {
        double s, c;
        sincospi(2.0 * (rows[i] * (double)freq_of(u, W)) / (double)W, &s, &c);
        er[u] = cplx<T>{T(c), T(s)};
    }
    __syncthreads();
    for (int v = threadIdx.x; v < W; v += blockDim.x) {
        cplx<T> acc{T(0), T(0)};
        for (int u = 0; u < W; ++u) acc = acc + er[u] * xps[(size_t)u * W + v];
        U[(size_t)i * W + v] = acc;
    }
}
// Pass 2: out[i][k] = sum_v U[i][v] ec[v][k] / W^2; CTA = row i, thread = column k.
template <typename T>
__global__ void __launch_bounds__(kVisThreads) vis_updft_cols_kernel(const cplx<T>* U, int W, const double* cols,
                                                                     int nc, cplx<T>* out) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    cplx<T>* urow = reinterpret_cast<cplx<T>*>(smem_raw);
    const int i = blockIdx.x;
    for (int v = threadIdx.x; v < W; v += blockDim.x) urow[v] = U[(size_t)i * W + v];
    __syncthreads();
    const T inv = T(1) / (T(W) * T(W));
    for (int k = threadIdx.x; k < nc; k += blockDim.x) {
        cplx<T> acc{T(0), T(0)};
        for (int v = 0; v < W; ++v) {
            double s, c;
            sincospi(2.0 * ((double)freq_of(v, W) * cols[k]) / (double)W, &s, &c);
            acc = acc + urow[v] * cplx<T>{T(c), T(s)};
        }
        out[(size_t)i * nc + k] = scale(acc, inv);
    }
}

// first maximum of |x| in index order (np.argmax of np.abs), one CTA
template <typename T>
__global__ void __launch_bounds__(kVisThreads) vis_argmax_abs_kernel(const cplx<T>* x, long long n, long long* idx,
                                                                     double* val) {
    __shared__ double sv[kVisThreads / 32];
    __shared__ long long sk[kVisThreads / 32];
    double bv = -1.0;
    long long bk = 0x7fffffffffffffffLL;
    for (long long i = threadIdx.x; i < n; i += blockDim.x) {
        const double v = (double)sqrt_rn(norm2(x[i]));
        if (arg_better(v, i, bv, bk)) { bv = v; bk = i; }
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
        *idx = bk;
        *val = bv;
    }
}

// posref.py:87-99 for one position j (no contraction: numpy's rounding sequence)
__global__ void vis_adam_step_kernel(double* m, double* v, long long* t, int j, double gx, double gy, double step,
                                     double b1, double b2, double eps, double clip, double* delta) {
    if (threadIdx.x != 0) return;
    const long long tj = ++t[j];
    const double g[2] = {gx, gy};
    const double c1 = 1.0 - pow(b1, (double)tj), c2 = 1.0 - pow(b2, (double)tj);
    for (int a = 0; a < 2; ++a) {
        const double mm = __dadd_rn(__dmul_rn(b1, m[2 * j + a]), __dmul_rn(1.0 - b1, g[a]));
        const double vv = __dadd_rn(__dmul_rn(b2, v[2 * j + a]), __dmul_rn(__dmul_rn(1.0 - b2, g[a]), g[a]));
        m[2 * j + a] = mm;
        v[2 * j + a] = vv;
        const double mh = mm / c1, vh = vv / c2;
        const double dd = __dmul_rn(step, mh) / __dadd_rn(sqrt(vh), eps);
        delta[a] = fmin(fmax(dd, -clip), clip);
    }
}

// posref.py:102-113: add and clamp; *inside = no clamping happened
__global__ void vis_apply_correction_kernel(double* pos, int j, double dx, double dy, double xmin, double ymin,
                                            double xmax, double ymax, int* inside) {
    if (threadIdx.x != 0) return;
    const double x = __dadd_rn(pos[2 * j], dx), y = __dadd_rn(pos[2 * j + 1], dy);
    const double cx = fmin(fmax(x, xmin), xmax), cy = fmin(fmax(y, ymin), ymax);
    pos[2 * j] = cx;
    pos[2 * j + 1] = cy;
    *inside = (cx == x && cy == y) ? 1 : 0;
}

// dst[i] += src[i] over n real values (batched mode: an owner adds the halo
// rows of the object accumulator received from another rank, in rank order)
template <typename T>
__global__ void __launch_bounds__(kVisThreads) vis_accumulate_kernel(T* dst, const T* src, long long n) {
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
        dst[i] += src[i];
}

}  // namespace pty

using namespace pty;

extern "C" {

int pty_accumulate(void* dst, const void* src, int64_t n, int32_t dtype, void* stream) {
    if (!dst || !src || n < 0) return PTY_ERR_ARGUMENT;
    if (n == 0) return PTY_OK;
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    return with_dtype(dtype, [&](auto t) {
        using T = decltype(t);
        vis_accumulate_kernel<T><<<vis_blocks(n), kVisThreads, 0, st>>>(static_cast<T*>(dst), static_cast<const T*>(src), n);
        count();
        return last_status();
    });
}

int64_t pty_visit_scratch_bytes(int32_t dtype, int32_t W, int32_t M) {
    if (!valid_window(W) || M < 1 || M > 8) return -1;
    const size_t real = dtype == PTY_DTYPE_C128 ? 8 : 4;
    return (int64_t)((size_t)W * W * real + 1024 * real + 1024);
}

int pty_magnitude_correct(int32_t dtype, int32_t W, int32_t M, const void* probes, const void* o_j, const void* I,
                          double epsilon_rel, void* corrected, void* psi_det, int32_t* status, void* scratch,
                          int64_t scratch_bytes, void* stream) {
    if (!probes || !o_j || !I || !corrected || !psi_det || !status || !scratch) return PTY_ERR_ARGUMENT;
    if (scratch_bytes < pty_visit_scratch_bytes(dtype, W, M)) return PTY_ERR_ARGUMENT;
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    const long long WW = (long long)W * W;
    const unsigned nb = vis_blocks(WW);
    int rc = with_dtype(dtype, [&](auto t) {
        using T = decltype(t);
        vis_exit_kernel<T><<<nb, kVisThreads, 0, st>>>(static_cast<const cplx<T>*>(probes),
                                                       static_cast<const cplx<T>*>(o_j), static_cast<const T*>(I), M,
                                                       WW, static_cast<cplx<T>*>(psi_det), status);
        count();
        return last_status();
    });
    if (rc) return rc;
    if ((rc = pty_fft2(psi_det, dtype, W, M, 0, 1, stream))) return rc;         // propagate(p * o_j)
    rc = with_dtype(dtype, [&](auto t) {
        using T = decltype(t);
        T* total = static_cast<T*>(scratch);
        T* part = total + WW;
        vis_total_kernel<T><<<nb, kVisThreads, 0, st>>>(static_cast<const cplx<T>*>(psi_det), M, WW, total, part);
        vis_scale_kernel<T><<<nb, kVisThreads, 0, st>>>(static_cast<const cplx<T>*>(psi_det), total,
                                                        static_cast<const T*>(I), part, (int)nb, M, WW, epsilon_rel,
                                                        static_cast<cplx<T>*>(corrected), status);
        count(2);
        return last_status();
    });
    if (rc) return rc;
    return pty_fft2(corrected, dtype, W, M, 1, 1, stream);                      // propagate(., "backward")
}

int pty_update_object(int32_t dtype, int32_t W, int32_t M, const void* o_j, const void* probes,
                      const void* corrected, double alpha_obj, double gamma, double epsilon_rel, void* out,
                      int32_t* status, void* scratch, int64_t scratch_bytes, void* stream) {
    if (!o_j || !probes || !corrected || !out || !status || !scratch) return PTY_ERR_ARGUMENT;
    if (scratch_bytes < pty_visit_scratch_bytes(dtype, W, M)) return PTY_ERR_ARGUMENT;
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    const long long WW = (long long)W * W;
    const unsigned nb = vis_blocks(WW);
    return with_dtype(dtype, [&](auto t) {
        using T = decltype(t);
        T* pp = static_cast<T*>(scratch);
        T* part = pp + WW;
        vis_power_kernel<T><<<nb, kVisThreads, 0, st>>>(static_cast<const cplx<T>*>(probes), M, WW, pp, part);
        vis_update_object_kernel<T><<<nb, kVisThreads, 0, st>>>(
            static_cast<const cplx<T>*>(o_j), static_cast<const cplx<T>*>(probes),
            static_cast<const cplx<T>*>(corrected), pp, part, (int)nb, M, WW, alpha_obj, gamma, epsilon_rel,
            static_cast<cplx<T>*>(out), status);
        count(2);
        return last_status();
    });
}

int pty_update_probe(int32_t dtype, int32_t W, const void* probe, const void* o_j, const void* corrected,
                     double alpha_probe, double beta, double epsilon_rel, void* out, int32_t* status, void* scratch,
                     int64_t scratch_bytes, void* stream) {
    if (!probe || !o_j || !corrected || !out || !status || !scratch) return PTY_ERR_ARGUMENT;
    if (scratch_bytes < pty_visit_scratch_bytes(dtype, W, 1)) return PTY_ERR_ARGUMENT;
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    const long long WW = (long long)W * W;
    const unsigned nb = vis_blocks(WW);
    return with_dtype(dtype, [&](auto t) {
        using T = decltype(t);
        T* op = static_cast<T*>(scratch);
        T* part = op + WW;
        vis_power_kernel<T><<<nb, kVisThreads, 0, st>>>(static_cast<const cplx<T>*>(o_j), 1, WW, op, part);
        vis_update_probe_kernel<T><<<nb, kVisThreads, 0, st>>>(
            static_cast<const cplx<T>*>(probe), static_cast<const cplx<T>*>(o_j),
            static_cast<const cplx<T>*>(corrected), op, part, (int)nb, WW, alpha_probe, beta, epsilon_rel,
            static_cast<cplx<T>*>(out), status);
        count(2);
        return last_status();
    });
}

int pty_cross_power_spectrum(void* work, const void* ref_real, const void* mov_real, int32_t real_inputs,
                             int32_t dtype, int32_t W, int32_t n, int32_t weighting, void* xps, int32_t* ok,
                             void* scratch, int64_t scratch_bytes, void* stream) {
    if (!work || !xps || !ok || !valid_window(W) || n < 0) return PTY_ERR_ARGUMENT;
    if (weighting != 0 && weighting != 1) return PTY_ERR_ARGUMENT;
    if (real_inputs && (!ref_real || !mov_real)) return PTY_ERR_ARGUMENT;
    if (scratch_bytes < pty_register_scratch_bytes(W, n, 1)) return PTY_ERR_ARGUMENT;
    if (n == 0) return PTY_OK;
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    return with_dtype(dtype, [&](auto t) {
        using T = decltype(t);
        return with_window(W, [&](auto w) {
            constexpr int WW = decltype(w)::value;
            const cplx<T>* tw = twiddles<T, WW>(st);
            if (!tw) return PTY_ERR_CUDA;
            const int TR = std::min(WW, 8), TC = std::min(WW, 8);
            const int nRT = WW / TR, nCT = WW / TC;
            T* mx = static_cast<T*>(scratch);
            cplx<T>* wk = static_cast<cplx<T>*>(work);
            const size_t line = (size_t)line_stride<WW>() * sizeof(cplx<T>);
            const size_t fix = (size_t)WW * sizeof(cplx<T>) + 64 * sizeof(double);
            const size_t s_rows = fix + 2 * TR * line, s_cols = fix + 2 * TC * line;
            auto k1 = reg_rows_fwd<T, WW>;
            auto k2 = reg_cols<T, WW>;
            auto k3 = reg_whiten<T, WW>;
            cudaFuncSetAttribute(k1, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)s_rows);
            cudaFuncSetAttribute(k2, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)s_cols);
            cudaFuncSetAttribute(k3, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)s_cols);
            k1<<<n * nRT, kRegThreads, s_rows, st>>>(wk, static_cast<const T*>(ref_real),
                                                     static_cast<const T*>(mov_real), real_inputs, n, TR, tw);
            k2<<<n * nCT, kRegThreads, s_cols, st>>>(wk, n, TC, 0, mx, tw);
            if (weighting == 0) k3<<<n * nCT, kRegThreads, s_cols, st>>>(wk, n, TC, mx, tw);
            const long long tot = (long long)n * WW * WW;
            vis_xps_out_kernel<T><<<vis_blocks(tot), kVisThreads, 0, st>>>(wk, (long long)WW * WW, n, mx, nCT,
                                                                          static_cast<cplx<T>*>(xps), ok);
            count(3 + (weighting == 0));
            (void)nRT;
            return last_status();
        });
    });
}

int pty_coarse_argmax(const void* corr, int32_t dtype, int32_t W, int32_t n, double* dy, double* dx, double* peak,
                      void* stream) {
    if (!corr || !dy || !dx || !peak || W < 2 || n < 0) return PTY_ERR_ARGUMENT;
    if (n == 0) return PTY_OK;
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    return with_dtype(dtype, [&](auto t) {
        using T = decltype(t);
        vis_coarse_argmax_kernel<T><<<n, kVisThreads, 0, st>>>(static_cast<const cplx<T>*>(corr), W, dy, dx, peak);
        count();
        return last_status();
    });
}

int64_t pty_upsampled_idft_scratch_bytes(int32_t dtype, int32_t W, int32_t n_rows) {
    if (W < 1 || n_rows < 1) return -1;
    return (int64_t)n_rows * W * (dtype == PTY_DTYPE_C128 ? 16 : 8);
}

int pty_upsampled_idft(const void* xps, int32_t dtype, int32_t W, const double* rows, int32_t n_rows,
                       const double* cols, int32_t n_cols, void* out, void* scratch, int64_t scratch_bytes,
                       void* stream) {
    if (!xps || !rows || !cols || !out || !scratch || W < 1 || n_rows < 1 || n_cols < 1) return PTY_ERR_ARGUMENT;
    if (scratch_bytes < pty_upsampled_idft_scratch_bytes(dtype, W, n_rows)) return PTY_ERR_ARGUMENT;
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    return with_dtype(dtype, [&](auto t) {
        using T = decltype(t);
        const size_t smem = (size_t)W * sizeof(cplx<T>);
        if (smem > max_dyn_smem()) return PTY_ERR_ARGUMENT;
        cudaFuncSetAttribute(vis_updft_rows_kernel<T>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        cudaFuncSetAttribute(vis_updft_cols_kernel<T>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        cplx<T>* U = static_cast<cplx<T>*>(scratch);
        vis_updft_rows_kernel<T><<<n_rows, kVisThreads, smem, st>>>(static_cast<const cplx<T>*>(xps), W, rows, U);
        vis_updft_cols_kernel<T><<<n_rows, kVisThreads, smem, st>>>(U, W, cols, n_cols, static_cast<cplx<T>*>(out));
        count(2);
        return last_status();
    });
}

int pty_argmax_abs(const void* x, int32_t dtype, int64_t n, int64_t* idx, double* val, void* stream) {
    if (!x || !idx || !val || n < 1) return PTY_ERR_ARGUMENT;
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    return with_dtype(dtype, [&](auto t) {
        using T = decltype(t);
        vis_argmax_abs_kernel<T><<<1, kVisThreads, 0, st>>>(static_cast<const cplx<T>*>(x), n,
                                                             reinterpret_cast<long long*>(idx), val);
        count();
        return last_status();
    });
}

int pty_adam_step(double* m, double* v, int64_t* t, int32_t j, double gx, double gy, double step_size,
                  double beta1, double beta2, double eps_adam, double max_correction, double* delta, void* stream) {
    if (!m || !v || !t || !delta || j < 0) return PTY_ERR_ARGUMENT;
    vis_adam_step_kernel<<<1, 32, 0, static_cast<cudaStream_t>(stream)>>>(
        m, v, reinterpret_cast<long long*>(t), j, gx, gy, step_size, beta1, beta2, eps_adam, max_correction, delta);
    count();
    return last_status();
}

int pty_apply_correction(double* positions, int32_t j, double dx, double dy, double xmin, double ymin, double xmax,
                         double ymax, int32_t* inside, void* stream) {
    if (!positions || !inside || j < 0) return PTY_ERR_ARGUMENT;
    vis_apply_correction_kernel<<<1, 32, 0, static_cast<cudaStream_t>(stream)>>>(positions, j, dx, dy, xmin, ymin,
                                                                                xmax, ymax, inside);
    count();
    return last_status();
}

}  // extern "C"
