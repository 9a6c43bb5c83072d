// pty_fft.cuh -- shared-memory-staged radix FFT building blocks (sm_100a).
//
// A length-W line (W = A*B, both powers of two, A >= B) is transformed by a
// group of B threads ("line group", <= one warp):
//   stage 1: thread b loads x[B*a + b] (a < A) into registers, runs an
//            in-register DFT_A, multiplies by the inter-stage twiddles
//            w_W^(b*k1) and writes the A partial spectra to the padded line;
//   stage 2: thread t reads the B values of column k1 = t + B*i, runs DFT_B and
//            writes X[k1 + A*k2] back in natural order.
// Lines live in shared memory with one pad slot every B elements
// (pad(i) = i + i/B) so both stages are bank-conflict free; the group
// synchronises with __syncwarp(mask).  Output order is natural, so the
// centered/uncentered conventions are applied purely elementwise outside.
//
// Forward = exp(-2 pi i k n / W) unnormalised (np.fft.fft), inverse =
// exp(+2 pi i k n / W) unnormalised (np.fft.ifft * W); callers scale.
#pragma once
#include <type_traits>
#include "pty_common.cuh"

namespace pty {

template <int W> struct Shape;
template <> struct Shape<16>   { static constexpr int A = 4,  B = 4;  };
template <> struct Shape<32>   { static constexpr int A = 8,  B = 4;  };
template <> struct Shape<64>   { static constexpr int A = 8,  B = 8;  };
template <> struct Shape<128>  { static constexpr int A = 16, B = 8;  };
#ifdef PTY_NARROW256
// narrow W = 256 lines (pty_sweep_f32_w256n.cu, compiled in namespace pty_n):
// a whole warp per line, 8 points per thread, 256 = 8 x 8 x 4 (group_fft below)
template <> struct Shape<256>  { static constexpr int A = 8, B = 32; };
#else
template <> struct Shape<256>  { static constexpr int A = 16, B = 16; };
#endif
template <> struct Shape<512>  { static constexpr int A = 32, B = 16; };

template <int N> struct Log2 { static constexpr int value = 1 + Log2<N / 2>::value; };
template <> struct Log2<1> { static constexpr int value = 0; };

template <int W> __device__ __forceinline__ int pad(int i) { return i + i / Shape<W>::B; }
// line stride in complex elements: padded length + 1 so that lines indexed by
// a column number land on different banks when tiles are transposed
template <int W> __host__ __device__ constexpr int line_stride() { return W + W / Shape<W>::B + 1; }

// cos(2 pi j / 32), j in [0, 8]
__host__ __device__ constexpr double kCos32(int j) {
    return j == 0 ? 1.0
         : j == 1 ? 0.98078528040323044912618223613424
         : j == 2 ? 0.92387953251128675612818318939679
         : j == 3 ? 0.83146961230254523707878837761791
         : j == 4 ? 0.70710678118654752440084436210485
         : j == 5 ? 0.55557023301960222474283081394853
         : j == 6 ? 0.38268343236508977172845998403040
         : j == 7 ? 0.19509032201612826784828486847702
         : 0.0;
}
// cos / sin of 2 pi j / 32 for any j (folded by the compiler for constant j)
__host__ __device__ constexpr double cos32(int j) {
    j &= 31;
    if (j > 16) j = 32 - j;
    return j <= 8 ? kCos32(j) : -kCos32(16 - j);
}
__host__ __device__ constexpr double sin32(int j) { return cos32(j - 8); }

// x * exp(-/+ 2 pi i j / 32): constant j, special angles exact
template <typename T, bool INV>
__device__ __forceinline__ cplx<T> twiddle32(cplx<T> x, int j) {
    j &= 31;
    if (j == 0) return x;
    if (j == 16) return {-x.re, -x.im};
    if (j == 8) return INV ? cplx<T>{-x.im, x.re} : cplx<T>{x.im, -x.re};
    if (j == 24) return INV ? cplx<T>{x.im, -x.re} : cplx<T>{-x.im, x.re};
    const T c = T(cos32(j));
    const T s = INV ? T(sin32(j)) : T(-sin32(j));
    return rot_const(x, c, s);      // float: the packed overload
}

// In-register DFT of N <= 32 points, natural order in and out (radix-2 DIT).
template <typename T, int N, bool INV>
struct DFT {
    static __device__ __forceinline__ void run(cplx<T>* v) {
        cplx<T> e[N / 2], o[N / 2];
#pragma unroll
        for (int i = 0; i < N / 2; ++i) { e[i] = v[2 * i]; o[i] = v[2 * i + 1]; }
        DFT<T, N / 2, INV>::run(e);
        DFT<T, N / 2, INV>::run(o);
#pragma unroll
        for (int k = 0; k < N / 2; ++k) {
            const cplx<T> t = twiddle32<T, INV>(o[k], k * (32 / N));
            v[k] = e[k] + t;
            v[k + N / 2] = e[k] - t;
        }
    }
};
template <typename T, bool INV>
struct DFT<T, 2, INV> {
    static __device__ __forceinline__ void run(cplx<T>* v) {
        const cplx<T> a = v[0], b = v[1];
        v[0] = a + b;
        v[1] = a - b;
    }
};
template <typename T, bool INV>
struct DFT<T, 4, INV> {
    static __device__ __forceinline__ void run(cplx<T>* v) {
        const cplx<T> s0 = v[0] + v[2], d0 = v[0] - v[2];
        const cplx<T> s1 = v[1] + v[3], d1 = v[1] - v[3];
        // d1 * (-i) forward, d1 * (+i) inverse
        const cplx<T> r = INV ? cplx<T>{-d1.im, d1.re} : cplx<T>{d1.im, -d1.re};
        v[0] = s0 + s1;
        v[2] = s0 - s1;
        v[1] = d0 + r;
        v[3] = d0 - r;
    }
};

// Inter-stage twiddle table for a W-line: tw[k1*B + b] = exp(-2 pi i b k1 / W).
// Filled once per CTA from a global table built on the host in float64.
template <typename T, int W>
__device__ __forceinline__ void load_twiddles(cplx<T>* tw_smem, const cplx<T>* tw_global) {
    for (int i = threadIdx.x; i < W; i += blockDim.x) tw_smem[i] = tw_global[i];
}

// Inter-stage twiddles v[k1] *= w^(b k1) (conjugate for the inverse).
// float: w(4q + r) = w(4q) * w(r) from 3 + A/4 - 1 table reads instead of
// A - 1 (the twiddle reads were 14 % of all shared-memory wavefronts of the
// sweep); the product adds ~1 ulp.  double: straight table reads.
template <typename T, int W, bool INV>
__device__ __forceinline__ void apply_twiddles(cplx<T>* v, const cplx<T>* tw, int b) {
    constexpr int A = Shape<W>::A, B = Shape<W>::B;
    if constexpr (std::is_same<T, float>::value && A >= 8 && A >= B) {
        cplx<T> wr[4], wq[A / 4];
        wr[0] = cplx<T>{T(1), T(0)};
        wq[0] = cplx<T>{T(1), T(0)};
#pragma unroll
        for (int r = 1; r < 4; ++r) wr[r] = tw[r * B + b];
#pragma unroll
        for (int q = 1; q < A / 4; ++q) wq[q] = tw[4 * q * B + b];
#pragma unroll
        for (int k1 = 1; k1 < A; ++k1) {
            const int q = k1 / 4, r = k1 % 4;
            const cplx<T> w = r == 0 ? wq[q] : (q == 0 ? wr[r] : wq[q] * wr[r]);
            v[k1] = INV ? mulc(v[k1], w) : v[k1] * w;
        }
    } else {
#pragma unroll
        for (int k1 = 1; k1 < A; ++k1) {
            const cplx<T> w = tw[k1 * B + b];
            v[k1] = INV ? mulc(v[k1], w) : v[k1] * w;
        }
    }
}

// Narrow line DFT (A = 8 points per lane, B = 32 lanes, W = 256 = 8 x 8 x 4),
// used when A < B.  Lane b holds x[32a + b]; stage 1 is a DFT8 over a with
// the inter-stage twiddles w256^(b k1); the DFT32 over b that remains for
// every k1 is split as b = 4c + d, k2 = e + 8f:
//   X[k1 + 8e + 64f] = sum_d w4^(df) w32^(de) sum_c Y_{4c+d}[k1] w8^(ce),
// stage 2a = DFT8 over c on lane (k1 = b/4, d = b%4) after exchange 1,
// twiddle w32^(de) = tw[e*32 + 8d], stage 2b = DFT4 over d on lane
// (k1, d2) for e in {2 d2, 2 d2 + 1} after exchange 2.  Both exchanges use a
// 256-slot XOR-swizzled layout that is bank-conflict free for 8-byte values
// on writes and reads.  Lane (k1, d2) outputs k = k1 + 8(2 d2 + p) + 64 f at
// slot p*4 + f.
template <typename T, bool INV, typename LD, typename ST>
__device__ __forceinline__ void narrow_fft256(cplx<T>* xch, const cplx<T>* tw, int b, unsigned mask, LD&& load,
                                              ST&& store) {
    constexpr int B = 32;
    cplx<T> v[8];
#pragma unroll
    for (int a = 0; a < 8; ++a) v[a] = load(B * a + b, a);
    DFT<T, 8, INV>::run(v);
    apply_twiddles<T, 256, INV>(v, tw, b);
    __syncwarp(mask);
#pragma unroll
    for (int k1 = 0; k1 < 8; ++k1) xch[32 * k1 + (b ^ (4 * k1))] = v[k1];
    __syncwarp(mask);
    const int k1s = b >> 2, d = b & 3, sw = 4 * (k1s & 3);
#pragma unroll
    for (int c = 0; c < 8; ++c) v[c] = xch[32 * k1s + ((4 * c + d) ^ (4 * k1s))];
    __syncwarp(mask);
    DFT<T, 8, INV>::run(v);
#pragma unroll
    for (int e = 1; e < 8; ++e) {
        const cplx<T> w = tw[e * 32 + 8 * d];                  // w32^(d e) = w256^(8 d e)
        v[e] = INV ? mulc(v[e], w) : v[e] * w;
    }
#pragma unroll
    for (int e = 0; e < 8; ++e) xch[32 * k1s + ((4 * e + ((d + (e >> 1)) & 3)) ^ sw)] = v[e];
    __syncwarp(mask);
#pragma unroll
    for (int p = 0; p < 2; ++p)
#pragma unroll
        for (int q = 0; q < 4; ++q) v[p * 4 + q] = xch[32 * k1s + ((4 * (2 * d + p) + ((q + d) & 3)) ^ sw)];
    __syncwarp(mask);
    DFT<T, 4, INV>::run(&v[0]);
    DFT<T, 4, INV>::run(&v[4]);
#pragma unroll
    for (int p = 0; p < 2; ++p)
#pragma unroll
        for (int f = 0; f < 4; ++f) store(k1s + 8 * (2 * d + p) + 64 * f, p * 4 + f, v[p * 4 + f]);
}

// Transform one padded line in shared memory with a group of B threads.
// b = thread index in the group, mask = the group's lanes.
template <typename T, int W, bool INV>
__device__ __forceinline__ void line_fft(cplx<T>* line, const cplx<T>* tw, int b, unsigned mask) {
    constexpr int A = Shape<W>::A, B = Shape<W>::B;
    if constexpr (A < B) {
        static_assert(W == 256 && A == 8 && B == 32, "narrow lines: W = 256 only");
        narrow_fft256<T, INV>(
            line, tw, b, mask, [&](int n, int) { return line[n + n / B]; },
            [&](int k, int, cplx<T> x) { line[k + k / B] = x; });
        __syncwarp(mask);
        return;
    } else {
    constexpr int Q = A / B;
    cplx<T> v[A];
#pragma unroll
    for (int a = 0; a < A; ++a) v[a] = line[a * (B + 1) + b];
    DFT<T, A, INV>::run(v);
    apply_twiddles<T, W, INV>(v, tw, b);
    __syncwarp(mask);
#pragma unroll
    for (int k1 = 0; k1 < A; ++k1) line[k1 * (B + 1) + b] = v[k1];
    __syncwarp(mask);
#pragma unroll
    for (int i = 0; i < Q; ++i)
#pragma unroll
        for (int j = 0; j < B; ++j) v[i * B + j] = line[(b + B * i) * (B + 1) + j];
    __syncwarp(mask);
#pragma unroll
    for (int i = 0; i < Q; ++i) {
        DFT<T, B, INV>::run(&v[i * B]);
#pragma unroll
        for (int k2 = 0; k2 < B; ++k2) {
            const int k = b + B * i + A * k2;
            line[k + k / B] = v[i * B + k2];
        }
    }
    __syncwarp(mask);
    }
}

// Fused-I/O line FFT by a group of B threads.  Stage 1 takes its A inputs from
// load(n, a) with n = B*a + b (for fixed a the group reads B consecutive
// elements: coalesced from global memory); stage 2 hands each output to
// store(k, slot, value) with k = b + B*i + A*k2 and slot = i*B + k2 (a thread's
// output set is fixed, so per-thread accumulators can be indexed by slot).
// xch: the group's exchange buffer, A*(B+1) complex, may alias the input when
// the input is shared memory (all stage-1 reads precede the first write).
template <typename T, int W, bool INV, typename LD, typename ST>
__device__ __forceinline__ void group_fft(cplx<T>* xch, const cplx<T>* tw, int b, unsigned mask, LD&& load,
                                          ST&& store) {
    constexpr int A = Shape<W>::A, B = Shape<W>::B;
    if constexpr (A < B) {
        static_assert(W == 256 && A == 8 && B == 32, "narrow lines: W = 256 only");
        narrow_fft256<T, INV>(xch, tw, b, mask, load, store);
        return;
    } else {
    constexpr int Q = A / B;
    cplx<T> v[A];
#pragma unroll
    for (int a = 0; a < A; ++a) v[a] = load(B * a + b, a);
    DFT<T, A, INV>::run(v);
    apply_twiddles<T, W, INV>(v, tw, b);
    __syncwarp(mask);
#pragma unroll
    for (int k1 = 0; k1 < A; ++k1) xch[k1 * (B + 1) + b] = v[k1];
    __syncwarp(mask);
#pragma unroll
    for (int i = 0; i < Q; ++i)
#pragma unroll
        for (int j = 0; j < B; ++j) v[i * B + j] = xch[(b + B * i) * (B + 1) + j];
    __syncwarp(mask);
#pragma unroll
    for (int i = 0; i < Q; ++i) {
        DFT<T, B, INV>::run(&v[i * B]);
#pragma unroll
        for (int k2 = 0; k2 < B; ++k2) store(b + B * i + A * k2, i * B + k2, v[i * B + k2]);
    }
    }
}

template <int W> __host__ __device__ constexpr int xch_size() { return Shape<W>::A * (Shape<W>::B + 1); }

// Run `nlines` line FFTs (lines at base + l * stride) with every line group of
// the CTA.  Caller synchronises the block before and after.
template <typename T, int W, bool INV>
__device__ __forceinline__ void lines_fft(cplx<T>* base, int nlines, int stride, const cplx<T>* tw) {
    constexpr int B = Shape<W>::B;
    const int groups = blockDim.x / B;
    const int g = threadIdx.x / B, b = threadIdx.x % B;
    const int lane = threadIdx.x & 31;
    const unsigned mask = (B == 32) ? 0xffffffffu : (((1u << B) - 1u) << (lane & ~(B - 1)));
    for (int l = g; l < nlines; l += groups) line_fft<T, W, INV>(base + (size_t)l * stride, tw, b, mask);
}

}  // namespace pty
