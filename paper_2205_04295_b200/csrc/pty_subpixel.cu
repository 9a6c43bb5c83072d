// pty_subpixel.cu -- the opt-in subpixel reconstruction gather (extension;
// SolverConfig.subpixel_gather).  The reference crops every visit at the
// rounded anchor (engine.py:69-70, 192-195); the simulator alone
// extracts views at float positions: integer crop plus the residual Fourier
// phase-ramp shift (simulate.py:157-166, fields.py:110-122).  This mode applies
// the simulator's gather to reconstruction:
//
//   o_j   = subpixel_shift(crop(obj, anchor_j), -rx, -ry)        rx = x - ac, ry = y - ar
//   visit = magnitude_correct / update_object / update_probe on o_j (engine.py:104-150)
//   obj[box] += subpixel_shift(new_o_j - o_j, rx, ry)            (the inverse shift)
//
// with o_j = crop exactly (no FFT round trip) when rx = ry = 0, so a scan on
// the integer grid reproduces the default path.  Parity is unpinned against
// the reference (it has no such mode); the CPU statement is
// oracle/rpie.py sweep(subpixel=True).
//
// The visit sequence is stream-ordered launches driven from this C++ loop (no
// host synchronisation inside a sweep): every kernel reads the step's
// position id order[step] and its float position on the device.
#include <cuda_runtime.h>

#include "pty_host.cuh"
#include "pty_sweep.cuh"

namespace pty {

constexpr int kSpThreads = 256;
// DFT frequency index of u, np.fft.fftfreq(W) * W (fields.py:119-120)
__device__ __forceinline__ int freq_of_sp(int u, int W) { return u < W / 2 ? u : u - W; }
constexpr int kSpBlocks = 64;                 // blocks of the element-wise kernels (fixed: reduction order)

struct SpVisit {                              // per-slot device view for one step
    const int* order;
    int step;
    const double* positions;
    int r0, c0, H, Wc;
};

__device__ __forceinline__ void sp_anchor(const SpVisit& v, int& j, int& ar, int& ac, double& rx, double& ry) {
    j = v.order[v.step];
    const double x = v.positions[2 * j], y = v.positions[2 * j + 1];
    const double ay = rint(y), ax = rint(x);                  // Python round(): half to even
    ar = (int)ay - v.r0;
    ac = (int)ax - v.c0;
    ry = y - ay;
    rx = x - ax;
}

// crop o_j at the integer anchor into o (and a copy into c for the shift); bounds -> status
template <typename T>
__global__ void __launch_bounds__(kSpThreads) sp_gather_kernel(const cplx<T>* obj, SpVisit v, int W, cplx<T>* o,
                                                               cplx<T>* c, int* status) {
    int j, ar, ac;
    double rx, ry;
    sp_anchor(v, j, ar, ac, rx, ry);
    if (ar < 0 || ac < 0 || ar + W > v.H || ac + W > v.Wc) {
        if (blockIdx.x == 0 && threadIdx.x == 0) atomicOr(status, PTY_ERR_BOUNDS);
        return;
    }
    const long long WW = (long long)W * W;
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < WW; i += (long long)gridDim.x * blockDim.x) {
        const cplx<T> x = obj[(size_t)(ar + i / W) * v.Wc + ac + i % W];
        o[i] = x;
        c[i] = x;
    }
}

// multiply a spectrum (np.fft.fft2 layout) by exp(-2 pi i (fy dy + fx dx)) with
// (dx, dy) = sign * (rx, ry): sign = -1 is the gather's subpixel_shift(crop, -rx, -ry)
template <typename T>
__global__ void __launch_bounds__(kSpThreads) sp_ramp_kernel(cplx<T>* f, SpVisit v, int W, double sign) {
    int j, ar, ac;
    double rx, ry;
    sp_anchor(v, j, ar, ac, rx, ry);
    if (rx == 0.0 && ry == 0.0) return;
    const double dx = sign * rx, dy = sign * ry;
    const long long WW = (long long)W * W;
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < WW; i += (long long)gridDim.x * blockDim.x) {
        const int u = (int)(i / W), c = (int)(i % W);
        const double fy = (double)freq_of_sp(u, W) / W, fx = (double)freq_of_sp(c, W) / W;
        double s, co;
        sincospi(-2.0 * (fy * dy + fx * dx), &s, &co);
        f[i] = f[i] * cplx<T>{T(co), T(s)};
    }
}

// o_j = shifted crop when the residual is non-zero (else the exact crop stays)
template <typename T>
__global__ void __launch_bounds__(kSpThreads) sp_select_kernel(cplx<T>* o, const cplx<T>* c, SpVisit v, int W) {
    int j, ar, ac;
    double rx, ry;
    sp_anchor(v, j, ar, ac, rx, ry);
    if (rx == 0.0 && ry == 0.0) return;
    const long long WW = (long long)W * W;
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < WW; i += (long long)gridDim.x * blockDim.x)
        o[i] = c[i];
}

// psi_m = P_m * o_j (engine.py:113)
template <typename T>
__global__ void __launch_bounds__(kSpThreads) sp_exit_kernel(const cplx<T>* probes, const cplx<T>* o, int M,
                                                             long long WW, cplx<T>* psi) {
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < WW; i += (long long)gridDim.x * blockDim.x) {
        const cplx<T> ov = o[i];
        for (int m = 0; m < M; ++m) psi[m * WW + i] = probes[m * WW + i] * ov;
    }
}

// total = sum_m |Psi_m|^2 (engine.py:114-116), per-block max, and the visit's
// error terms (engine.py:198-202) as per-block double partials [kSpBlocks][3]
template <typename T>
__global__ void __launch_bounds__(kSpThreads) sp_total_kernel(const cplx<T>* psi, const T* patterns, SpVisit v, int M,
                                                              long long WW, T* total, T* part, double* err_part) {
    __shared__ double red[32];
    const int j = v.order[v.step];
    const T* I = patterns + (size_t)j * WW;
    T mx = T(0);
    double en = 0.0, ed = 0.0;
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < WW; i += (long long)gridDim.x * blockDim.x) {
        T t = T(0);
        for (int m = 0; m < M; ++m) t += norm2(psi[m * WW + i]);
        total[i] = t;
        mx = fmax(mx, t);
        const T d = sqrt_rn(t) - sqrt_rn(I[i]);
        en += (double)(d * d);
        ed += (double)I[i];
    }
    mx = block_max(mx, reinterpret_cast<T*>(red));
    if (threadIdx.x == 0) part[blockIdx.x] = mx;
    en = block_sum(en, red);
    ed = block_sum(ed, red);
    if (threadIdx.x == 0) {
        double* e = err_part + ((size_t)v.step * kSpBlocks + blockIdx.x) * 3;
        e[0] = en;
        e[1] = ed;
        e[2] = 0.0;
    }
}

// corrected_m = sqrt(I) / sqrt(total + eps) * Psi_m (engine.py:117-118); XCORR_B staging
template <typename T>
__global__ void __launch_bounds__(kSpThreads) sp_scale_kernel(const cplx<T>* psi, const T* total, const T* patterns,
                                                              SpVisit v, const T* part, int M, long long WW,
                                                              double eps_rel, cplx<T>* out, cplx<T>* stage_b) {
    const int j = v.order[v.step];
    const T* I = patterns + (size_t)j * WW;
    T tmax = T(0);
    for (int k = 0; k < kSpBlocks; ++k) tmax = fmax(tmax, part[k]);
    const T eps = T(eps_rel) * fmax(tmax, real_limits<T>::tiny());
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < WW; i += (long long)gridDim.x * blockDim.x) {
        const T s = sqrt_rn(I[i]) / sqrt_rn(total[i] + eps);
        for (int m = 0; m < M; ++m) out[m * WW + i] = scale(psi[m * WW + i], s);
        if (stage_b) {
            cplx<T>* sb = stage_b + (size_t)j * 2 * WW;
            sb[i] = cplx<T>{total[i], T(0)};
            sb[WW + i] = cplx<T>{I[i], T(0)};
        }
    }
}

// sum_m |P_m|^2 and |o_j|^2 maps with per-block maxima (engine.py:129, 145)
template <typename T>
__global__ void __launch_bounds__(kSpThreads) sp_power_kernel(const cplx<T>* probes, const cplx<T>* o, int M,
                                                              long long WW, T* pp, T* op, T* part) {
    __shared__ T red[32];
    T mp = T(0), mo = T(0);
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < WW; i += (long long)gridDim.x * blockDim.x) {
        T t = T(0);
        for (int m = 0; m < M; ++m) t += norm2(probes[m * WW + i]);
        pp[i] = t;
        mp = fmax(mp, t);
        const T q = norm2(o[i]);
        op[i] = q;
        mo = fmax(mo, q);
    }
    mp = block_max(mp, red);
    if (threadIdx.x == 0) part[blockIdx.x] = mp;
    mo = block_max(mo, red);
    if (threadIdx.x == 0) part[kSpBlocks + blockIdx.x] = mo;
}

// engine.py:123-150 for one crop: new_o (object update), the probe updates with
// the pre-update o_j and probes into probes_new, and delta = new_o - o_j;
// XCORR_A staging (o_j, new_o)
template <typename T>
__global__ void __launch_bounds__(kSpThreads) sp_update_kernel(
    const cplx<T>* o, const cplx<T>* probes, const cplx<T>* corrected, const T* pp, const T* op, const T* part,
    SpVisit v, int M, long long WW, double alpha_o, double alpha_p, double beta, double gamma, double eps_rel,
    int update_probe, cplx<T>* probes_new, cplx<T>* delta, cplx<T>* stage_a, int* status) {
    T peak = T(0), omax = T(0);
    for (int k = 0; k < kSpBlocks; ++k) {
        peak = fmax(peak, part[k]);
        omax = fmax(omax, part[kSpBlocks + k]);
    }
    if (peak == T(0)) {                                                        // engine.py:132-134
        if (blockIdx.x == 0 && threadIdx.x == 0) atomicOr(status, PTY_ERR_PROBE_ZERO);
        return;
    }
    if (update_probe && omax == T(0)) {                                        // engine.py:145-147
        if (blockIdx.x == 0 && threadIdx.x == 0) atomicOr(status, PTY_ERR_OBJECT_ZERO);
        return;
    }
    const int j = v.order[v.step];
    const T g = T(gamma), b = T(beta), ao = T(alpha_o), ap = T(alpha_p);
    const T dmax_o = g * peak + (T(1) - g) * peak, dmax_p = b * omax + (T(1) - b) * omax;
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < WW; i += (long long)gridDim.x * blockDim.x) {
        const cplx<T> ov = o[i];
        cplx<T> numer{T(0), T(0)};
        T dp = b * omax + (T(1) - b) * op[i];
        dp = dp + T(eps_rel) * dmax_p;
        for (int m = 0; m < M; ++m) {
            const cplx<T> p = probes[m * WW + i];
            const cplx<T> d = corrected[m * WW + i] - p * ov;
            numer = numer + mulc(d, p);
            if (update_probe) probes_new[m * WW + i] = p + divr(mulc(scale(d, ap), ov), dp);
        }
        T den = g * peak + (T(1) - g) * pp[i];
        den = den + T(eps_rel) * dmax_o;
        const cplx<T> no = ov + divr(scale(numer, ao), den);
        delta[i] = no - ov;
        if (stage_a) {
            cplx<T>* sa = stage_a + (size_t)j * 2 * WW;
            sa[i] = ov;
            sa[WW + i] = no;
        }
    }
}

// probes <- probes_new (update_probe), element-wise
template <typename T>
__global__ void __launch_bounds__(kSpThreads) sp_copy_kernel(cplx<T>* dst, const cplx<T>* src, long long n) {
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
        dst[i] = src[i];
}

// paste: obj[box] += delta (fields.py:101-107; delta already shifted back)
template <typename T>
__global__ void __launch_bounds__(kSpThreads) sp_paste_kernel(cplx<T>* obj, const cplx<T>* delta, SpVisit v, int W,
                                                              const int* status) {
    if (*(volatile const int*)status) return;
    int j, ar, ac;
    double rx, ry;
    sp_anchor(v, j, ar, ac, rx, ry);
    const long long WW = (long long)W * W;
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < WW; i += (long long)gridDim.x * blockDim.x) {
        cplx<T>& x = obj[(size_t)(ar + i / W) * v.Wc + ac + i % W];
        x = x + delta[i];
    }
}

template <typename T>
int run_sweep_subpixel(const PtySweepArgs* a, cudaStream_t st) {
    const int W = a->window, M = a->modes, N = a->n_positions, S = a->n_slots;
    const long long WW = (long long)W * W;
    using C = cplx<T>;
    // scratch per call: o, c, delta (W^2); psi, corrected, probes_new (M W^2); total, pp, op (W^2 real);
    // partials; error partials [N][kSpBlocks][3]; visit sums [N][3]
    const size_t cbytes = (size_t)(3 + 3 * M) * WW * sizeof(C), rbytes = (size_t)3 * WW * sizeof(T);
    const size_t pbytes = 2 * kSpBlocks * sizeof(T) + 256;
    const size_t ebytes = (size_t)N * kSpBlocks * 3 * sizeof(double), vbytes = (size_t)N * 3 * sizeof(double);
    keep_pool_memory();
    char* mem = nullptr;
    const size_t total_bytes = cbytes + rbytes + pbytes + ebytes + vbytes + 1024;
    if (cudaMallocAsync(reinterpret_cast<void**>(&mem), total_bytes, st) != cudaSuccess) return PTY_ERR_CUDA;
    Carver cv(mem);
    C* o = cv.take<C>(WW * sizeof(C));
    C* c = cv.take<C>(WW * sizeof(C));
    C* delta = cv.take<C>(WW * sizeof(C));
    C* psi = cv.take<C>(M * WW * sizeof(C));
    C* corr = cv.take<C>(M * WW * sizeof(C));
    C* pnew = cv.take<C>(M * WW * sizeof(C));
    T* total = cv.take<T>(WW * sizeof(T));
    T* pp = cv.take<T>(WW * sizeof(T));
    T* op = cv.take<T>(WW * sizeof(T));
    T* part = cv.take<T>(2 * kSpBlocks * sizeof(T));
    double* err_part = cv.take<double>(ebytes);
    double* visit_sum = cv.take<double>(vbytes);
    const int dt = std::is_same<T, float>::value ? PTY_DTYPE_C64 : PTY_DTYPE_C128;
    const dim3 g(kSpBlocks), b(kSpThreads);
    int rc = PTY_OK;
    for (int s = 0; s < S && rc == PTY_OK; ++s) {
        const PtySlot& h = a->slots[s];
        C* obj = static_cast<C*>(h.obj);
        C* probes = static_cast<C*>(h.probes);
        const T* pats = static_cast<const T*>(h.patterns);
        C* stage_a = a->sense == PTY_SENSE_XCORR_A ? static_cast<C*>(h.stage) : nullptr;
        C* stage_b = a->sense == PTY_SENSE_XCORR_B ? static_cast<C*>(h.stage) : nullptr;
        for (int step = 0; step < N && rc == PTY_OK; ++step) {
            const SpVisit v{h.order, step, h.positions, h.r0, h.c0, h.H, h.Wc};
            sp_gather_kernel<T><<<g, b, 0, st>>>(obj, v, W, o, c, h.status);
            if ((rc = pty_fft2(c, dt, W, 1, 0, 0, st))) break;                     // fft2(crop)
            sp_ramp_kernel<T><<<g, b, 0, st>>>(c, v, W, -1.0);                     // shift by (-rx, -ry)
            if ((rc = pty_fft2(c, dt, W, 1, 1, 0, st))) break;                     // ifft2
            sp_select_kernel<T><<<g, b, 0, st>>>(o, c, v, W);
            sp_exit_kernel<T><<<g, b, 0, st>>>(probes, o, M, WW, psi);
            if ((rc = pty_fft2(psi, dt, W, M, 0, 1, st))) break;                   // propagate(P_m o_j)
            sp_total_kernel<T><<<g, b, 0, st>>>(psi, pats, v, M, WW, total, part, err_part);
            sp_scale_kernel<T><<<g, b, 0, st>>>(psi, total, pats, v, part, M, WW, a->epsilon_rel, corr, stage_b);
            if ((rc = pty_fft2(corr, dt, W, M, 1, 1, st))) break;                  // propagate(., backward)
            sp_power_kernel<T><<<g, b, 0, st>>>(probes, o, M, WW, pp, op, part);
            sp_update_kernel<T><<<g, b, 0, st>>>(o, probes, corr, pp, op, part, v, M, WW, a->alpha_obj,
                                                 a->alpha_probe, a->beta, a->gamma, a->epsilon_rel,
                                                 a->update_probe, pnew, delta, stage_a, h.status);
            if (a->update_probe) sp_copy_kernel<T><<<g, b, 0, st>>>(probes, pnew, (long long)M * WW);
            if ((rc = pty_fft2(delta, dt, W, 1, 0, 0, st))) break;                 // shift back by (rx, ry)
            sp_ramp_kernel<T><<<g, b, 0, st>>>(delta, v, W, 1.0);
            if ((rc = pty_fft2(delta, dt, W, 1, 1, 0, st))) break;
            sp_paste_kernel<T><<<g, b, 0, st>>>(obj, delta, v, W, h.status);
            count(11 + (a->update_probe ? 1 : 0));
            rc = last_status();
        }
        if (rc) break;
        ErrOut outs{};
        outs.p[0] = h.err_out;
        err_visit_kernel<<<N, 256, 0, st>>>(err_part, kSpBlocks, visit_sum);
        err_slot_kernel<<<1, 256, 0, st>>>(visit_sum, N, 1, outs);
        count(2);
        rc = last_status();
    }
    cudaFreeAsync(mem, st);
    return rc;
}

}  // namespace pty

using namespace pty;

extern "C" int pty_sweep_subpixel(const PtySweepArgs* a, void* stream) {
    if (!a || !a->slots || !valid_window(a->window) || a->modes < 1 || a->modes > kMaxModes ||
        a->n_positions < 1 || a->n_slots < 1 || a->n_slots > kMaxSlots || a->track_modulus)
        return PTY_ERR_ARGUMENT;
    for (int s = 0; s < a->n_slots; ++s) {
        const PtySlot& h = a->slots[s];
        if (!h.obj || !h.probes || !h.patterns || !h.positions || !h.order || !h.status || !h.err_out)
            return PTY_ERR_ARGUMENT;
        if (a->sense != PTY_SENSE_NONE && !h.stage) return PTY_ERR_ARGUMENT;
    }
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    if (a->dtype == PTY_DTYPE_C64) return run_sweep_subpixel<float>(a, st);
    if (a->dtype == PTY_DTYPE_C128) return run_sweep_subpixel<double>(a, st);
    return PTY_ERR_ARGUMENT;
}
