// pty_capi.cu -- extern "C" entry points of libptycho_b200.so
// (declared in include/ptycho_b200.h).  Host-side only: argument checks,
// workspace carving and dtype/window dispatch onto the sm_100a kernels in
// pty_sweep.cuh (instantiated in pty_sweep_*.cu), pty_aux.cuh and
// pty_register.cuh.
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <cstdlib>
#include <cstring>
#include <type_traits>
#include <vector>

#include "pty_register.cuh"
#include "pty_sweep_host.cuh"
#include "pty_batched_host.cuh"

namespace pty {
std::atomic<long long> g_launches{0};
std::vector<unsigned long long> g_timeline;
int g_timeline_grid = 0;
extern template int run_sweep<float, 16>(const PtySweepArgs*, cudaStream_t);
extern template int run_sweep<float, 32>(const PtySweepArgs*, cudaStream_t);
extern template int run_sweep<float, 64>(const PtySweepArgs*, cudaStream_t);
extern template int run_sweep<float, 128>(const PtySweepArgs*, cudaStream_t);
extern template int run_sweep<float, 256>(const PtySweepArgs*, cudaStream_t);
extern template int run_sweep<float, 512>(const PtySweepArgs*, cudaStream_t);
extern template int run_sweep<double, 16>(const PtySweepArgs*, cudaStream_t);
extern template int run_sweep<double, 32>(const PtySweepArgs*, cudaStream_t);
extern template int run_sweep<double, 64>(const PtySweepArgs*, cudaStream_t);
extern template int run_sweep<double, 128>(const PtySweepArgs*, cudaStream_t);
extern template int run_sweep<double, 256>(const PtySweepArgs*, cudaStream_t);
extern template int run_sweep<double, 512>(const PtySweepArgs*, cudaStream_t);
extern template int run_batch_contrib<float, 16>(const PtyBatchArgs*, cudaStream_t);
extern template int run_batch_apply<float, 16>(const PtyBatchArgs*, cudaStream_t);
extern template int64_t batch_workspace<float, 16>(int, int, int, int, bool);
extern template int run_batch_contrib<float, 32>(const PtyBatchArgs*, cudaStream_t);
extern template int run_batch_apply<float, 32>(const PtyBatchArgs*, cudaStream_t);
extern template int64_t batch_workspace<float, 32>(int, int, int, int, bool);
extern template int run_batch_contrib<float, 64>(const PtyBatchArgs*, cudaStream_t);
extern template int run_batch_apply<float, 64>(const PtyBatchArgs*, cudaStream_t);
extern template int64_t batch_workspace<float, 64>(int, int, int, int, bool);
extern template int run_batch_contrib<float, 128>(const PtyBatchArgs*, cudaStream_t);
extern template int run_batch_apply<float, 128>(const PtyBatchArgs*, cudaStream_t);
extern template int64_t batch_workspace<float, 128>(int, int, int, int, bool);
extern template int run_batch_contrib<float, 256>(const PtyBatchArgs*, cudaStream_t);
extern template int run_batch_apply<float, 256>(const PtyBatchArgs*, cudaStream_t);
extern template int64_t batch_workspace<float, 256>(int, int, int, int, bool);
extern template int run_batch_contrib<float, 512>(const PtyBatchArgs*, cudaStream_t);
extern template int run_batch_apply<float, 512>(const PtyBatchArgs*, cudaStream_t);
extern template int64_t batch_workspace<float, 512>(int, int, int, int, bool);
extern template int run_batch_contrib<double, 16>(const PtyBatchArgs*, cudaStream_t);
extern template int run_batch_apply<double, 16>(const PtyBatchArgs*, cudaStream_t);
extern template int64_t batch_workspace<double, 16>(int, int, int, int, bool);
extern template int run_batch_contrib<double, 32>(const PtyBatchArgs*, cudaStream_t);
extern template int run_batch_apply<double, 32>(const PtyBatchArgs*, cudaStream_t);
extern template int64_t batch_workspace<double, 32>(int, int, int, int, bool);
extern template int run_batch_contrib<double, 64>(const PtyBatchArgs*, cudaStream_t);
extern template int run_batch_apply<double, 64>(const PtyBatchArgs*, cudaStream_t);
extern template int64_t batch_workspace<double, 64>(int, int, int, int, bool);
extern template int run_batch_contrib<double, 128>(const PtyBatchArgs*, cudaStream_t);
extern template int run_batch_apply<double, 128>(const PtyBatchArgs*, cudaStream_t);
extern template int64_t batch_workspace<double, 128>(int, int, int, int, bool);
extern template int run_batch_contrib<double, 256>(const PtyBatchArgs*, cudaStream_t);
extern template int run_batch_apply<double, 256>(const PtyBatchArgs*, cudaStream_t);
extern template int64_t batch_workspace<double, 256>(int, int, int, int, bool);
extern template int run_batch_contrib<double, 512>(const PtyBatchArgs*, cudaStream_t);
extern template int run_batch_apply<double, 512>(const PtyBatchArgs*, cudaStream_t);
extern template int64_t batch_workspace<double, 512>(int, int, int, int, bool);
}  // namespace pty

using namespace pty;

namespace {

__global__ void barrier_bench_kernel(unsigned int* counter, int iters, unsigned long long* ns) {
    GridBarrier bar{counter, 0u};
    bar.sync();
    unsigned long long t0 = 0;
    if (blockIdx.x == 0 && threadIdx.x == 0) asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
    for (int i = 0; i < iters; ++i) bar.sync();
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        unsigned long long t1;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t1));
        *ns = t1 - t0;
    }
}

}  // namespace

// =================================================================== C ABI ==
extern "C" {

int pty_abi_version(void) { return PTY_ABI_VERSION; }

int64_t pty_launch_count(void) { return (int64_t)g_launches.load(); }

int64_t pty_timeline(uint64_t* out, int64_t cap, int32_t* grid) {
    const int64_t n = (int64_t)g_timeline.size();
    if (out) std::memcpy(out, g_timeline.data(), (size_t)std::min(n, cap) * sizeof(uint64_t));
    if (grid) *grid = g_timeline_grid;
    return n;
}

int pty_barrier_bench(int32_t iters, int32_t ctas, double* ns_per_barrier) {
    if (iters < 1 || !ns_per_barrier) return PTY_ERR_ARGUMENT;
    if (ctas <= 0) ctas = sm_count();
    unsigned int* counter = nullptr;
    unsigned long long* ns = nullptr;
    if (cudaMalloc(&counter, sizeof(unsigned int)) != cudaSuccess) return PTY_ERR_CUDA;
    if (cudaMalloc(&ns, sizeof(unsigned long long)) != cudaSuccess) return PTY_ERR_CUDA;
    cudaMemset(counter, 0, sizeof(unsigned int));
    void* args[] = {&counter, &iters, &ns};
    cudaError_t e = cudaLaunchCooperativeKernel((const void*)barrier_bench_kernel, dim3(ctas), dim3(kSweepThreads),
                                                args, 0, 0);
    count();
    unsigned long long h = 0;
    if (e == cudaSuccess) e = cudaMemcpy(&h, ns, sizeof(h), cudaMemcpyDeviceToHost);
    cudaFree(counter);
    cudaFree(ns);
    *ns_per_barrier = (double)h / iters;
    return cuda_status(e);
}

int pty_device_info(int32_t* sm, int32_t* coop, int32_t* major, int32_t* minor) {
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess) return PTY_ERR_CUDA;
    cudaDeviceProp p;
    if (cudaGetDeviceProperties(&p, dev) != cudaSuccess) return PTY_ERR_CUDA;
    if (sm) *sm = p.multiProcessorCount;
    if (coop) *coop = p.cooperativeLaunch ? p.multiProcessorCount : 0;
    if (major) *major = p.major;
    if (minor) *minor = p.minor;
    return PTY_OK;
}

int64_t pty_sweep_workspace_bytes(int32_t dtype, int32_t W, int32_t M, int32_t N, int32_t S) {
    if (!valid_window(W) || M < 1 || M > kMaxModes || N < 1 || S < 1 || S > kMaxSlots) return -1;
    if (dtype == PTY_DTYPE_C64) return (int64_t)sweep_workspace<float>(W, M, N, S);
    if (dtype == PTY_DTYPE_C128) return (int64_t)sweep_workspace<double>(W, M, N, S);
    return -1;
}

int pty_sweep(const PtySweepArgs* a, void* stream) {
    if (!a || !a->slots || !valid_window(a->window) || a->modes < 1 || a->modes > kMaxModes ||
        a->n_positions < 1 || a->n_slots < 1 || a->n_slots > kMaxSlots)
        return PTY_ERR_ARGUMENT;
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    return with_dtype(a->dtype, [&](auto t) {
        using T = decltype(t);
        return with_window(a->window, [&](auto w) { return run_sweep<T, decltype(w)::value>(a, st); });
    });
}

int pty_fft2(void* data, int32_t dtype, int32_t W, int32_t batch, int32_t inverse, int32_t centered,
             void* stream) {
    if (!data || batch < 0 || !valid_window(W)) return PTY_ERR_ARGUMENT;
    if (batch == 0) return PTY_OK;
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    return with_dtype(dtype, [&](auto t) {
        using T = decltype(t);
        return with_window(W, [&](auto w) {
            constexpr int WW = decltype(w)::value;
            const cplx<T>* tw = twiddles<T, WW>(st);
            if (!tw) return PTY_ERR_CUDA;
            const int TR = std::min(WW, 16);
            const size_t smem = (size_t)WW * sizeof(cplx<T>) + (size_t)TR * line_stride<WW>() * sizeof(cplx<T>);
            // centered: C * DFT(C * x) / W (both directions, norm="ortho");
            // uncentered: np.fft.fft2 (1) or np.fft.ifft2 (1/W^2)
            const T post = centered ? T(1) / T(WW) : (inverse ? T(1) / (T(WW) * T(WW)) : T(1));
            cplx<T>* d = static_cast<cplx<T>*>(data);
            const dim3 grid((unsigned)batch * (WW / TR));
            if (inverse) {
                auto kr = fft2_rows_kernel<T, WW, true>;
                auto kc = fft2_cols_kernel<T, WW, true>;
                cudaFuncSetAttribute(kr, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
                cudaFuncSetAttribute(kc, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
                kr<<<grid, kAuxThreads, smem, st>>>(d, batch, TR, centered, tw);
                kc<<<grid, kAuxThreads, smem, st>>>(d, batch, TR, centered, post, tw);
                count(2);
            } else {
                auto kr = fft2_rows_kernel<T, WW, false>;
                auto kc = fft2_cols_kernel<T, WW, false>;
                cudaFuncSetAttribute(kr, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
                cudaFuncSetAttribute(kc, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
                kr<<<grid, kAuxThreads, smem, st>>>(d, batch, TR, centered, tw);
                kc<<<grid, kAuxThreads, smem, st>>>(d, batch, TR, centered, post, tw);
                count(2);
            }
            return last_status();
        });
    });
}

int64_t pty_register_scratch_bytes(int32_t W, int32_t n, int32_t kappa) {
    if (!valid_window(W) || n < 0) return -1;
    const int npts = kappa <= 1 ? 1 : ((int)(1.5 * kappa) | 1);
    const size_t nIB = (size_t)(npts + 3) / 4;               // refine_rows() >= 4
    Carver c(nullptr);
    c.take<void>((size_t)n * W * sizeof(double));          // max|xps| partials (<= W col tiles)
    c.take<ArgPart>((size_t)n * W * sizeof(ArgPart));       // coarse partials
    c.take<RefPart>((size_t)n * nIB * sizeof(RefPart));     // refine partials
    return (int64_t)c.off;
}

int pty_register_batch(void* work, const void* ref_real, const void* mov_real, int32_t real_inputs,
                       int32_t dtype, int32_t W, int32_t n, int32_t weighting, int32_t kappa,
                       double* dy, double* dx, double* peak, int32_t* ok, void* scratch,
                       int64_t scratch_bytes, void* stream) {
    if (!work || !valid_window(W) || n < 0 || !dy || !dx || !peak || !ok) return PTY_ERR_ARGUMENT;
    if (!(kappa == 1 || (kappa >= 2 && kappa <= 1000))) return PTY_ERR_ARGUMENT;
    if (weighting != 0 && weighting != 1) return PTY_ERR_ARGUMENT;
    if (real_inputs == 1 && (!ref_real || !mov_real)) return PTY_ERR_ARGUMENT;
    if (real_inputs == 2 && (!ref_real || dtype != PTY_DTYPE_C128)) return PTY_ERR_ARGUMENT;
    if (real_inputs < 0 || real_inputs > 2) return PTY_ERR_ARGUMENT;
    if (scratch_bytes < pty_register_scratch_bytes(W, n, kappa)) return PTY_ERR_ARGUMENT;
    if (n == 0) return PTY_OK;
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    const int npts = kappa <= 1 ? 1 : ((int)(1.5 * kappa) | 1);   // registration.py:101-104
    return with_dtype(dtype, [&](auto t) {
        using T = decltype(t);
        return with_window(W, [&](auto w) {
            constexpr int WW = decltype(w)::value;
            const cplx<T>* tw = twiddles<T, WW>(st);
            if (!tw) return PTY_ERR_CUDA;
            const int TR = std::min(WW, 8), TC = std::min(WW, 8);
            const int nRT = WW / TR, nCT = WW / TC;
            Carver c(scratch);
            T* mx = c.take<T>((size_t)n * WW * sizeof(double));
            ArgPart* cpart = c.take<ArgPart>((size_t)n * WW * sizeof(ArgPart));
            RefPart* rpart = c.take<RefPart>((size_t)n * ((npts + 3) / 4) * sizeof(RefPart));
            cplx<T>* wk = static_cast<cplx<T>*>(work);
            const size_t line = (size_t)line_stride<WW>() * sizeof(cplx<T>);
            const size_t fix = (size_t)WW * sizeof(cplx<T>) + 64 * sizeof(double);
            const size_t s_rows = fix + 2 * TR * line, s_cols = fix + 2 * TC * line;
            auto k1 = reg_rows_fwd<T, WW>;
            auto k2 = reg_cols<T, WW>;
            auto k3 = reg_whiten<T, WW>;
            auto k4 = reg_rows_inv<T, WW>;
            auto k5 = reg_refine<T, WW>;
            cudaFuncSetAttribute(k1, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)s_rows);
            cudaFuncSetAttribute(k2, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)s_cols);
            cudaFuncSetAttribute(k3, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)s_cols);
            cudaFuncSetAttribute(k4, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)s_rows);
            cudaFuncSetAttribute(k5, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)refine_smem<T, WW>());
            k1<<<n * nRT, kRegThreads, s_rows, st>>>(wk, static_cast<const T*>(ref_real),
                                                     static_cast<const T*>(mov_real), real_inputs, n, TR, tw);
            k2<<<n * nCT, kRegThreads, s_cols, st>>>(wk, n, TC, weighting == 1, mx, tw);
            if (weighting == 0) k3<<<n * nCT, kRegThreads, s_cols, st>>>(wk, n, TC, mx, tw);
            k4<<<n * nRT, kRegThreads, s_rows, st>>>(wk, n, TR, cpart, tw);
            constexpr int IB = refine_rows<T, WW>();
            if (kappa > 1) {
                const int nIB = (npts + IB - 1) / IB;
                k5<<<n * nIB, kRegThreads, refine_smem<T, WW>(), st>>>(wk, n, kappa, npts, cpart, nRT, rpart);
            }
            reg_finalize<T><<<(n + 127) / 128, 128, 0, st>>>(n, WW, kappa, npts, IB, mx, nCT, cpart, nRT, rpart,
                                                             dy, dx, peak, ok);
            count(4 + (weighting == 0) + (kappa > 1));
            return last_status();
        });
    });
}

int pty_adam_apply(double* positions, double* m, double* v, int64_t* t, const double* gx, const double* gy,
                   const int32_t* ok, const int32_t* index, int32_t n, double step_size, double beta1,
                   double beta2, double eps_adam, double max_correction, double xmin, double ymin, double xmax,
                   double ymax, void* stream) {
    if (!positions || !m || !v || !t || !gx || !gy || !ok || n < 0) return PTY_ERR_ARGUMENT;
    if (n == 0) return PTY_OK;
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    adam_kernel<<<(n + 127) / 128, 128, 0, st>>>(positions, m, v, reinterpret_cast<long long*>(t), gx, gy, ok, index,
                                                 n, step_size, beta1, beta2, eps_adam, max_correction, xmin, ymin,
                                                 xmax, ymax);
    count();
    return last_status();
}

int pty_init_probes(void* probes, int32_t dtype, const void* patterns, int32_t n_patterns, const double* noise,
                    int32_t W, int32_t M, void* scratch, int64_t scratch_bytes, void* stream) {
    if (!probes || !patterns || n_patterns < 1 || !valid_window(W) || M < 1 || M > kMaxModes) return PTY_ERR_ARGUMENT;
    if (M > 1 && !noise) return PTY_ERR_ARGUMENT;
    const size_t WW = (size_t)W * W;
    if (!scratch || scratch_bytes < (int64_t)(M * WW * sizeof(cplx<double>))) return PTY_ERR_ARGUMENT;
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    cplx<double>* work = static_cast<cplx<double>*>(scratch);
    int rc = with_dtype(dtype, [&](auto t) {
        using T = decltype(t);
        mean_amplitude_kernel<T><<<(unsigned)((WW + 255) / 256), 256, 0, st>>>(static_cast<const T*>(patterns),
                                                                              n_patterns, (int)WW, work);
        count();
        return last_status();
    });
    if (rc) return rc;
    rc = pty_fft2(work, PTY_DTYPE_C128, W, 1, 1, 1, stream);   // propagate(..., "backward")
    if (rc) return rc;
    if (M > 1) {
        gram_schmidt_kernel<<<1, 1024, 0, st>>>(work, M, (int)WW, reinterpret_cast<const cplx<double>*>(noise), 1);
        count();
        rc = last_status();
        if (rc) return rc;
    }
    return with_dtype(dtype, [&](auto t) {
        using T = decltype(t);
        const long long n = (long long)M * WW;
        convert_kernel<T, double><<<(unsigned)((n + 255) / 256), 256, 0, st>>>(work, static_cast<cplx<T>*>(probes), n);
        count();
        return last_status();
    });
}

int pty_orthogonalize(void* probes, int32_t dtype, int32_t W, int32_t M, void* stream) {
    if (!probes || !valid_window(W) || M < 1 || M > kMaxModes) return PTY_ERR_ARGUMENT;
    if (M == 1) return PTY_OK;
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    const long long n = (long long)M * W * W;
    cplx<double>* work = nullptr;
    keep_pool_memory();
    if (cudaMallocAsync(&work, n * sizeof(cplx<double>), st) != cudaSuccess) return PTY_ERR_CUDA;
    int rc = with_dtype(dtype, [&](auto t) {
        using T = decltype(t);
        cplx<T>* p = static_cast<cplx<T>*>(probes);
        convert_kernel<double, T><<<(unsigned)((n + 255) / 256), 256, 0, st>>>(p, work, n);
        gram_schmidt_kernel<<<1, 1024, 0, st>>>(work, M, W * W, nullptr, 0);
        convert_kernel<T, double><<<(unsigned)((n + 255) / 256), 256, 0, st>>>(work, p, n);
        count(3);
        return last_status();
    });
    cudaFreeAsync(work, st);
    return rc;
}

int64_t pty_batch_workspace_bytes(int32_t dtype, int32_t W, int32_t M, int32_t b, int32_t H, int32_t Wc) {
    if (!valid_window(W) || M < 1 || M > kMaxBatchModes || b < 1 || H < W || Wc < W) return -1;
    int64_t out = -1;
    with_dtype(dtype, [&](auto t) {
        using T = decltype(t);
        return with_window(W, [&](auto w) {
            out = batch_workspace<T, decltype(w)::value>(M, b, H, Wc, true);
            return PTY_OK;
        });
    });
    return out;
}

static int batch_check(const PtyBatchArgs* a) {
    if (!a || !valid_window(a->window) || a->modes < 1 || a->modes > kMaxBatchModes || a->n_batch < 1 ||
        !a->obj || !a->probes || !a->patterns || !a->patterns_t || !a->positions || !a->batch || !a->obj_acc ||
        !a->probe_acc || !a->err_part || !a->status || a->H < a->window || a->Wc < a->window ||
        a->visit0 < 0 || a->visit0 + a->n_batch > a->n_positions)
        return PTY_ERR_ARGUMENT;
    if (a->sense != PTY_SENSE_NONE && !a->stage) return PTY_ERR_ARGUMENT;
    return PTY_OK;
}

int pty_batch_contrib(const PtyBatchArgs* a, void* stream) {
    if (int rc = batch_check(a)) return rc;
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    return with_dtype(a->dtype, [&](auto t) {
        using T = decltype(t);
        return with_window(a->window, [&](auto w) { return run_batch_contrib<T, decltype(w)::value>(a, st); });
    });
}

int pty_batch_apply(const PtyBatchArgs* a, void* stream) {
    if (int rc = batch_check(a)) return rc;
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    return with_dtype(a->dtype, [&](auto t) {
        using T = decltype(t);
        return with_window(a->window, [&](auto w) { return run_batch_apply<T, decltype(w)::value>(a, st); });
    });
}

int pty_batch_finalize(const double* err_part, int32_t n_visits, int32_t W, double* err_out, void* stream) {
    if (!err_part || !err_out || n_visits < 1 || !valid_window(W)) return PTY_ERR_ARGUMENT;
    ErrOut outs{};
    outs.p[0] = err_out;
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    double* vs = nullptr;
    keep_pool_memory();
    if (cudaMallocAsync(&vs, (size_t)n_visits * 3 * sizeof(double), st) != cudaSuccess) return PTY_ERR_CUDA;
    err_visit_kernel<<<n_visits, 256, 0, st>>>(err_part, W, vs);
    err_slot_kernel<<<1, 256, 0, st>>>(vs, n_visits, 1, outs);
    cudaFreeAsync(vs, st);
    count(2);
    return last_status();
}

int pty_check_patterns(const void* patterns, int32_t dtype, int64_t count, int32_t* status, void* stream) {
    if (!patterns || !status || count < 0) return PTY_ERR_ARGUMENT;
    if (count == 0) return PTY_OK;
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    const unsigned blocks = (unsigned)std::min<int64_t>((count + 255) / 256, 4096);
    return with_dtype(dtype, [&](auto t) {
        using T = decltype(t);
        check_nonneg_kernel<T><<<blocks, 256, 0, st>>>(static_cast<const T*>(patterns), count, status);
        g_launches.fetch_add(1);
        return last_status();
    });
}

}  // extern "C"
