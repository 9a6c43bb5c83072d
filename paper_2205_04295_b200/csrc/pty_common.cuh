// pty_common.cuh -- complex arithmetic, reductions and the grid barrier shared
// by every kernel of libptycho_b200.so (sm_100a).
//
// Complex values are interleaved (re, im) pairs, float2 / double2 compatible,
// so a complex64 torch tensor is read with 8-byte (and 16-byte vector) loads.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/ptycho_b200.h"

namespace pty {

template <typename T>
struct __align__(2 * sizeof(T)) cplx {
    T re, im;
};

template <typename T> __device__ __forceinline__ cplx<T> mk(T a, T b) { return {a, b}; }
template <typename T> __device__ __forceinline__ cplx<T> operator+(cplx<T> a, cplx<T> b) { return {a.re + b.re, a.im + b.im}; }
template <typename T> __device__ __forceinline__ cplx<T> operator-(cplx<T> a, cplx<T> b) { return {a.re - b.re, a.im - b.im}; }
template <typename T> __device__ __forceinline__ cplx<T> operator*(cplx<T> a, cplx<T> b) {
    return {a.re * b.re - a.im * b.im, a.re * b.im + a.im * b.re};
}
// a * conj(b)
template <typename T> __device__ __forceinline__ cplx<T> mulc(cplx<T> a, cplx<T> b) {
    return {a.re * b.re + a.im * b.im, a.im * b.re - a.re * b.im};
}
template <typename T> __device__ __forceinline__ cplx<T> scale(cplx<T> a, T s) { return {a.re * s, a.im * s}; }
template <typename T> __device__ __forceinline__ cplx<T> conjg(cplx<T> a) { return {a.re, -a.im}; }

// complex<float> on the sm_100 packed-fp32 pipe: one FADD2 / FMUL2 / FFMA2
// per complex add, sub and real scale instead of two scalar instructions
// (same IEEE round-to-nearest result per component, no contraction).
__device__ __forceinline__ unsigned long long f2pack(float a, float b) {
    unsigned long long r;
    asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(a), "f"(b));
    return r;
}
__device__ __forceinline__ cplx<float> f2unpack(unsigned long long r) {
    cplx<float> a;
    asm("mov.b64 {%0, %1}, %2;" : "=f"(a.re), "=f"(a.im) : "l"(r));
    return a;
}
__device__ __forceinline__ cplx<float> operator+(cplx<float> a, cplx<float> b) {
    unsigned long long z;
    asm("add.rn.f32x2 %0, %1, %2;" : "=l"(z) : "l"(f2pack(a.re, a.im)), "l"(f2pack(b.re, b.im)));
    return f2unpack(z);
}
__device__ __forceinline__ cplx<float> operator-(cplx<float> a, cplx<float> b) {
    unsigned long long z;
    asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(z) : "l"(f2pack(a.re, a.im)), "l"(f2pack(b.re, b.im)));
    return f2unpack(z);
}
__device__ __forceinline__ cplx<float> scale(cplx<float> a, float s) {
    unsigned long long z;
    asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(z) : "l"(f2pack(a.re, a.im)), "l"(f2pack(s, s)));
    return f2unpack(z);
}
// General complex products on the packed pipe.  x * w = wr*(xr, xi) +
// wi*(-xi, xr): one FMUL2 with a broadcast operand and one FFMA2 whose
// swapped / negated operand ptxas folds into the .F32x2.LO_HI modifiers (2
// instructions instead of 2 FMUL + 2 FFMA).
__device__ __forceinline__ cplx<float> operator*(cplx<float> x, cplx<float> w) {
    unsigned long long t, z;
    asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(t) : "l"(f2pack(x.re, x.im)), "l"(f2pack(w.re, w.re)));
    asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(z) : "l"(f2pack(x.im, x.re)), "l"(f2pack(-w.im, w.im)), "l"(t));
    return f2unpack(z);
}
// x * conj(w) = wr*(xr, xi) + wi*(xi, -xr)
__device__ __forceinline__ cplx<float> mulc(cplx<float> x, cplx<float> w) {
    unsigned long long t, z;
    asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(t) : "l"(f2pack(x.re, x.im)), "l"(f2pack(w.re, w.re)));
    asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(z) : "l"(f2pack(x.im, x.re)), "l"(f2pack(w.im, -w.im)), "l"(t));
    return f2unpack(z);
}
// x * (c + i s) for a compile-time twiddle: c*(xr, xi) + (xi, xr)*(-s, s)
__device__ __forceinline__ cplx<float> rot_const(cplx<float> x, float c, float s) {
    unsigned long long t, z;
    asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(t) : "l"(f2pack(x.re, x.im)), "l"(f2pack(c, c)));
    asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(z) : "l"(f2pack(x.im, x.re)), "l"(f2pack(-s, s)), "l"(t));
    return f2unpack(z);
}
// Repeated multiplication by one complex factor o (x * o and x * conj(o)),
// e.g. the pre-update object value in the update epilogue.  float: the sign
// pairs are formed once, each product is one FMUL2 + one FFMA2.
template <typename T> struct OMul {
    cplx<T> o;
    __device__ __forceinline__ explicit OMul(cplx<T> o_) : o(o_) {}
    __device__ __forceinline__ cplx<T> mul(cplx<T> x) const { return x * o; }
    __device__ __forceinline__ cplx<T> mulconj(cplx<T> x) const { return mulc(x, o); }
};
template <> struct OMul<float> {
    unsigned long long rr, pn, pc;     // (o.re, o.re), (-o.im, o.im), (o.im, -o.im)
    __device__ __forceinline__ explicit OMul(cplx<float> o) {
        rr = f2pack(o.re, o.re);
        pn = f2pack(-o.im, o.im);
        pc = f2pack(o.im, -o.im);
    }
    __device__ __forceinline__ cplx<float> mul(cplx<float> x) const {   // x * o
        unsigned long long t, z;
        asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(t) : "l"(f2pack(x.re, x.im)), "l"(rr));
        asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(z) : "l"(f2pack(x.im, x.re)), "l"(pn), "l"(t));
        return f2unpack(z);
    }
    __device__ __forceinline__ cplx<float> mulconj(cplx<float> x) const {   // x * conj(o)
        unsigned long long t, z;
        asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(t) : "l"(f2pack(x.re, x.im)), "l"(rr));
        asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(z) : "l"(f2pack(x.im, x.re)), "l"(pc), "l"(t));
        return f2unpack(z);
    }
};

template <typename T> __device__ __forceinline__ cplx<T> rot_const(cplx<T> x, T c, T s) {
    return {x.re * c - x.im * s, x.re * s + x.im * c};
}
template <typename T> __device__ __forceinline__ T norm2(cplx<T> a) { return a.re * a.re + a.im * a.im; }
// numpy's complex / real: Smith's rule with a zero imaginary divisor reduces
// to a multiply by the reciprocal (numpy loops_arithm_fp complex divide).
template <typename T> __device__ __forceinline__ cplx<T> divr(cplx<T> a, T d) {
    T inv = T(1) / d;
    return {a.re * inv, a.im * inv};
}

template <typename T> struct real_limits;
template <> struct real_limits<float>  { static __device__ __forceinline__ float tiny() { return 1.17549435e-38f; } };
template <> struct real_limits<double> { static __device__ __forceinline__ double tiny() { return 2.2250738585072014e-308; } };

__device__ __forceinline__ float  sqrt_rn(float x)  { return __fsqrt_rn(x); }
__device__ __forceinline__ double sqrt_rn(double x) { return __dsqrt_rn(x); }

// Throughput forms for the fp32 path (the fp64 instantiation stays
// correctly rounded, it is the parity path): MUFU square root / reciprocal
// square root / reciprocal, a few ulp, no IEEE slow-path branches.
__device__ __forceinline__ float sqrt_fast(float x) {
    float y;
    asm("sqrt.approx.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}
__device__ __forceinline__ double sqrt_fast(double x) { return __dsqrt_rn(x); }
__device__ __forceinline__ float rsqrt_fast(float x) {
    float y;
    asm("rsqrt.approx.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}
__device__ __forceinline__ double rsqrt_fast(double x) { return 1.0 / __dsqrt_rn(x); }
// the modulus-constraint scale sqrt(I) / sqrt(total + eps) (engine.py:118):
// fp32 multiplies by the MUFU reciprocal square root, fp64 keeps numpy's
// correctly rounded quotient
__device__ __forceinline__ float  modulus_scale(float sI, float x)   { return sI * rsqrt_fast(x); }
__device__ __forceinline__ double modulus_scale(double sI, double x) { return sI / __dsqrt_rn(x); }
__device__ __forceinline__ float rcp_fast(float x) {
    float y;
    asm("rcp.approx.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}
__device__ __forceinline__ double rcp_fast(double x) { return 1.0 / x; }

template <typename T> __device__ __forceinline__ T warp_max(T v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
    return v;
}
template <typename T> __device__ __forceinline__ T warp_sum(T v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

// Block-wide max / sum; `red` is >= 32 entries of shared scratch.  Every
// thread returns the result.  Must be called by all threads of the block.
// The three per-visit error terms (sum, sum, max) reduced over the block in
// one pass: two barriers instead of six.  red: >= 48 doubles, blocks of at
// most 16 warps.  Every thread returns the results.
template <typename T> __device__ void block_err3(double& a, double& b, T& c, double* red) {
    a = warp_sum(a);
    b = warp_sum(b);
    c = warp_max(c);
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
    __syncthreads();
    if (lane == 0) {
        red[wid] = a;
        red[16 + wid] = b;
        red[32 + wid] = (double)c;
    }
    __syncthreads();
    a = warp_sum(lane < nw ? red[lane] : 0.0);
    b = warp_sum(lane < nw ? red[16 + lane] : 0.0);
    c = (T)warp_max(lane < nw ? red[32 + lane] : 0.0);
}

template <typename T> __device__ T block_max(T v, T* red) {
    v = warp_max(v);
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
    __syncthreads();
    if (lane == 0) red[wid] = v;
    __syncthreads();
    T r = lane < nw ? red[lane] : red[0];
    r = warp_max(r);
    return r;
}
template <typename T> __device__ T block_sum(T v, T* red) {
    v = warp_sum(v);
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
    __syncthreads();
    if (lane == 0) red[wid] = v;
    __syncthreads();
    T r = lane < nw ? red[lane] : T(0);
    r = warp_sum(r);
    return r;
}

// Software grid barrier for a cooperative launch (all CTAs co-resident).
// `counter` is zeroed before the launch; each barrier raises the target by
// gridDim.x.  bar.sync orders the CTA's writes before thread 0's release
// atomic; the acquire spin + bar.sync make every other CTA's writes visible.
struct GridBarrier {
    unsigned int* counter;
    unsigned int target;
    __device__ __forceinline__ void sync() {
        __syncthreads();
        target += gridDim.x;
        if (threadIdx.x == 0) {
            unsigned int one = 1u, seen;
            asm volatile("atom.add.release.gpu.global.u32 %0, [%1], %2;"
                         : "=r"(seen) : "l"(counter), "r"(one) : "memory");
            while (true) {
                asm volatile("ld.acquire.gpu.global.u32 %0, [%1];"
                             : "=r"(seen) : "l"(counter) : "memory");
                if ((int)(seen - target) >= 0) break;
                __nanosleep(20);
            }
        }
        __syncthreads();
    }
};

// cp.async (LDGSTS): global -> shared without register staging, so a thread
// can have all its tile elements in flight at once.  Element sizes 4/8/16 B.
template <int BYTES>
__device__ __forceinline__ void cp_async(void* smem, const void* gmem) {
    const unsigned s = (unsigned)__cvta_generic_to_shared(smem);
    if constexpr (BYTES == 16)
        asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(s), "l"(gmem) : "memory");
    else
        asm volatile("cp.async.ca.shared.global [%0], [%1], %2;" ::"r"(s), "l"(gmem), "n"(BYTES) : "memory");
}
__device__ __forceinline__ void cp_async_wait_all() {
    asm volatile("cp.async.commit_group;\ncp.async.wait_group 0;" ::: "memory");
}

// ---------------------------------------------------------------- TMA ----
// 1-D bulk copies global -> shared (cp.async.bulk, SASS UBLKCP) completing on an
// mbarrier: one elected lane issues whole 2 KB lines, the data lands without
// registers or per-element instructions, and every lane of the consumer group
// waits on the barrier's phase parity.  16-byte aligned addresses and sizes.
__device__ __forceinline__ unsigned smem_u32(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(unsigned long long* bar, unsigned count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(unsigned long long* bar, unsigned bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void mbar_wait(unsigned long long* bar, unsigned parity) {
    asm volatile(
        "{\n\t.reg .pred p;\n"
        "WAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
        "@!p bra WAIT_%=;\n}" ::"r"(smem_u32(bar)), "r"(parity) : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, unsigned bytes, unsigned long long* bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                 ::"r"(smem_u32(dst)), "l"(src), "r"(bytes), "r"(smem_u32(bar)) : "memory");
}
// order this thread's earlier generic-proxy accesses (and the global data other
// CTAs released to it) before its async-proxy (bulk copy) accesses
__device__ __forceinline__ void fence_proxy_async() { asm volatile("fence.proxy.async;" ::: "memory"); }

// (-1)^(r+c) checkerboard: the fftshift/ifftshift pair of a centered DFT of
// even size becomes a sign flip on load and store.
template <typename T> __device__ __forceinline__ T checker(int r, int c) {
    return ((r + c) & 1) ? T(-1) : T(1);
}

}  // namespace pty
