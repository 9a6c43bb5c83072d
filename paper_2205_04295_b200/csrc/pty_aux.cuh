// pty_aux.cuh -- batched 2D FFT (fields.py:71-84 propagate and the uncentered
// np.fft.fft2/ifft2 of registration.py), probe initialisation
// (engine.py:83-95), Gram-Schmidt orthogonalisation (engine.py:153-164),
// the non-negative-intensity check (engine.py:111-112) and twiddle tables.
#pragma once
#include "pty_fft.cuh"

namespace pty {

constexpr int kAuxThreads = 256;

// tw[k1*B + b] = exp(-2 pi i b k1 / W), computed in float64 then rounded.
template <typename T, int W>
__global__ void twiddle_kernel(cplx<T>* tw) {
    constexpr int B = Shape<W>::B;
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= W) return;
    const int k1 = i / B, b = i % B;
    double s, c;
    sincospi(-2.0 * (double)(b * k1) / (double)W, &s, &c);
    tw[i] = cplx<T>{T(c), T(s)};
}

// Row pass of a batched 2D DFT: TR rows per CTA, in place.  centered: the
// input is pre-multiplied by (-1)^(r+c) (the ifftshift of fields.py:81,83).
template <typename T, int W, bool INV>
__global__ void __launch_bounds__(kAuxThreads) fft2_rows_kernel(cplx<T>* data, int batch, int TR,
                                                                 int centered, const cplx<T>* twg) {
    using C = cplx<T>;
    constexpr int LS = line_stride<W>();
    extern __shared__ __align__(16) unsigned char smem_raw[];
    C* tw = reinterpret_cast<C*>(smem_raw);
    C* tile = tw + W;
    load_twiddles<T, W>(tw, twg);
    const int nRT = W / TR;
    const int f = blockIdx.x / nRT, rt = blockIdx.x % nRT;
    if (f >= batch) return;
    C* base = data + (size_t)f * W * W + (size_t)rt * TR * W;
    for (int i = threadIdx.x; i < TR * W; i += blockDim.x) {
        const int r = i / W, c = i % W;
        C v = base[i];
        if (centered) v = scale(v, checker<T>(rt * TR + r, c));
        tile[(size_t)r * LS + pad<W>(c)] = v;
    }
    __syncthreads();
    lines_fft<T, W, INV>(tile, TR, LS, tw);
    __syncthreads();
    for (int i = threadIdx.x; i < TR * W; i += blockDim.x) {
        const int r = i / W, c = i % W;
        base[i] = tile[(size_t)r * LS + pad<W>(c)];
    }
}

// Column pass: TC columns per CTA; post-multiplies by (-1)^(r+c) when
// centered (the fftshift) and by `post` (the norm).
template <typename T, int W, bool INV>
__global__ void __launch_bounds__(kAuxThreads) fft2_cols_kernel(cplx<T>* data, int batch, int TC,
                                                                 int centered, T post, const cplx<T>* twg) {
    using C = cplx<T>;
    constexpr int LS = line_stride<W>();
    extern __shared__ __align__(16) unsigned char smem_raw[];
    C* tw = reinterpret_cast<C*>(smem_raw);
    C* tile = tw + W;
    load_twiddles<T, W>(tw, twg);
    const int nCT = W / TC;
    const int f = blockIdx.x / nCT, ct = blockIdx.x % nCT;
    if (f >= batch) return;
    C* base = data + (size_t)f * W * W + (size_t)ct * TC;
    for (int i = threadIdx.x; i < TC * W; i += blockDim.x) {
        const int r = i / TC, cc = i % TC;
        tile[(size_t)cc * LS + pad<W>(r)] = base[(size_t)r * W + cc];
    }
    __syncthreads();
    lines_fft<T, W, INV>(tile, TC, LS, tw);
    __syncthreads();
    for (int i = threadIdx.x; i < TC * W; i += blockDim.x) {
        const int r = i / TC, cc = i % TC;
        T s = post;
        if (centered) s *= checker<T>(r, ct * TC + cc);
        base[(size_t)r * W + cc] = scale(tile[(size_t)cc * LS + pad<W>(r)], s);
    }
}

// mean over patterns in float64 with numpy's axis-0 summation order
// (sequential over j), then sqrt(max(mean, 0)) as a complex128 field.
template <typename T>
__global__ void mean_amplitude_kernel(const T* patterns, int n, int WW, cplx<double>* out) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= WW) return;
    double acc = 0.0;
    for (int j = 0; j < n; ++j) acc += (double)patterns[(size_t)j * WW + i];
    const double mean = acc / (double)n;
    out[i] = cplx<double>{sqrt(fmax(mean, 0.0)), 0.0};
}

// Block reduction of a complex128 value.
__device__ inline cplx<double> block_csum(cplx<double> v, double* red) {
    v.re = block_sum(v.re, red);
    v.im = block_sum(v.im, red);
    return v;
}

// Gram-Schmidt in float64 over `modes` fields of WW pixels held in `work`,
// single CTA, in place.
// init = 1: engine.py:87-94 -- mode p := mode0 * noise[p-1], projected against
//   every previous mode, scaled to 1% of mode-0 power;
// init = 0: engine.py:153-164 -- power-preserving GS of every mode.
static __global__ void __launch_bounds__(1024) gram_schmidt_kernel(cplx<double>* work, int modes, int WW,
                                                            const cplx<double>* noise, int init) {
    __shared__ double red[64];
    __shared__ cplx<double> coef;
    const int tid = threadIdx.x, NT = blockDim.x;
    double acc = 0.0;
    for (int i = tid; i < (init ? WW : modes * WW); i += NT) acc += norm2(work[i]);
    const double power_before = block_sum(acc, red);   // mode-0 power (init) or total power
    for (int p = 1; p < modes; ++p) {
        cplx<double>* cand = work + (size_t)p * WW;
        if (init) {
            for (int i = tid; i < WW; i += NT) cand[i] = work[i] * noise[(size_t)(p - 1) * WW + i];
            __syncthreads();
        }
        for (int q = 0; q < p; ++q) {
            const cplx<double>* prev = work + (size_t)q * WW;
            cplx<double> a{0.0, 0.0};
            double b = 0.0;
            for (int i = tid; i < WW; i += NT) {
                a = a + mulc(cand[i], prev[i]);          // vdot(prev, cand) = sum conj(prev) cand
                b += norm2(prev[i]);
            }
            a = block_csum(a, red);
            b = block_sum(b, red);
            if (tid == 0) coef = cplx<double>{a.re / b, a.im / b};
            __syncthreads();
            const cplx<double> k = coef;
            for (int i = tid; i < WW; i += NT) cand[i] = cand[i] - prev[i] * k;
            __syncthreads();
        }
        if (init) {
            double pw = 0.0;
            for (int i = tid; i < WW; i += NT) pw += norm2(cand[i]);
            pw = block_sum(pw, red);
            const double s = sqrt(0.01 * power_before / pw);
            for (int i = tid; i < WW; i += NT) cand[i] = scale(cand[i], s);
            __syncthreads();
        }
    }
    if (!init) {
        double a2 = 0.0;
        for (int i = tid; i < modes * WW; i += NT) a2 += norm2(work[i]);
        a2 = block_sum(a2, red);
        const double s = a2 > 0.0 ? sqrt(power_before / a2) : 1.0;
        for (int i = tid; i < modes * WW; i += NT) work[i] = scale(work[i], s);
    }
}

template <typename T>
__global__ void check_nonneg_kernel(const T* x, long long n, int* status) {
    long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    const long long stride = (long long)gridDim.x * blockDim.x;
    bool bad = false;
    for (; i < n; i += stride) bad |= x[i] < T(0);   // engine.py:111 (NaN passes, as np.any(i < 0))
    if (__syncthreads_or(bad) && threadIdx.x == 0) atomicOr(status, PTY_ERR_NEGATIVE_I);
}

template <typename TO, typename TI>
__global__ void convert_kernel(const cplx<TI>* in, cplx<TO>* out, long long n) {
    long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) out[i] = cplx<TO>{TO(in[i].re), TO(in[i].im)};
}

}  // namespace pty
