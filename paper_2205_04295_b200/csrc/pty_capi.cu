// pty_capi.cu -- extern "C" entry points of libptycho_b200.so
// (declared in include/ptycho_b200.h).  Host-side only: argument checks,
// workspace carving, tile-size choice and dtype/window dispatch onto the
// sm_100a kernels in pty_sweep.cuh, pty_aux.cuh and pty_register.cuh.
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <cstdlib>
#include <cstring>
#include <type_traits>
#include <vector>

#include "pty_aux.cuh"
#include "pty_register.cuh"
#include "pty_sweep.cuh"

using namespace pty;

namespace {

std::atomic<long long> g_launches{0};
std::vector<unsigned long long> g_timeline;   // debug: last sweep's phase stamps
int g_timeline_grid = 0;
inline void count(int k = 1) { g_launches.fetch_add(k, std::memory_order_relaxed); }

constexpr size_t kAlign = 256;
inline size_t align_up(size_t x) { return (x + kAlign - 1) / kAlign * kAlign; }

struct Carver {
    char* base;
    size_t off = 0;
    explicit Carver(void* b) : base(static_cast<char*>(b)) {}
    template <typename P> P* take(size_t bytes) {
        P* p = reinterpret_cast<P*>(base ? base + off : nullptr);
        off += align_up(bytes);
        return p;
    }
};

inline bool valid_window(int W) { return W == 16 || W == 32 || W == 64 || W == 128 || W == 256 || W == 512; }

// Call f(std::integral_constant<int, W>) for the supported windows.
template <typename F> int with_window(int W, F&& f) {
    switch (W) {
        case 16: return f(std::integral_constant<int, 16>{});
        case 32: return f(std::integral_constant<int, 32>{});
        case 64: return f(std::integral_constant<int, 64>{});
        case 128: return f(std::integral_constant<int, 128>{});
        case 256: return f(std::integral_constant<int, 256>{});
        case 512: return f(std::integral_constant<int, 512>{});
        default: return PTY_ERR_ARGUMENT;
    }
}
template <typename F> int with_dtype(int dtype, F&& f) {
    if (dtype == PTY_DTYPE_C64) return f(float{});
    if (dtype == PTY_DTYPE_C128) return f(double{});
    return PTY_ERR_ARGUMENT;
}

inline int cuda_status(cudaError_t e) { return e == cudaSuccess ? PTY_OK : PTY_ERR_CUDA; }
inline int last_status() { return cuda_status(cudaGetLastError()); }

int env_int(const char* name, int dflt) {
    const char* v = std::getenv(name);
    return v ? std::atoi(v) : dflt;
}

inline int pow2_floor(int x) {
    int p = 1;
    while (p * 2 <= x) p *= 2;
    return p;
}

int sm_count() {
    int dev = 0, n = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    return n;
}

size_t max_smem_per_sm() {
    int dev = 0, n = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&n, cudaDevAttrMaxSharedMemoryPerMultiprocessor, dev);
    return (size_t)n;
}

size_t max_dyn_smem() {
    int dev = 0, n = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&n, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
    return (size_t)n;
}

// ------------------------------------------------------------- twiddles --
// Twiddle tables live in one static device buffer per (dtype, W), built once.
template <typename T, int W> const cplx<T>* twiddles(cudaStream_t st) {
    static cplx<T>* table = nullptr;
    if (!table) {
        if (cudaMalloc(&table, W * sizeof(cplx<T>)) != cudaSuccess) return nullptr;
        twiddle_kernel<T, W><<<(W + 255) / 256, 256, 0, st>>>(table);
        count();
    }
    return table;
}

// ------------------------------------------------------------- sweep ------
constexpr int kMinTC = 4;   // column tiles are >= 4 complex (32-byte sectors)

struct SweepLayout {
    unsigned int* barrier;
    int* anchors;
    void* scratch;
    void* omax;
    void* peak;
    void* tmax;
    double* err_part;
    size_t bytes;
};

template <typename T>
SweepLayout carve_sweep(void* ws, int W, int M, int N, int S) {
    Carver c(ws);
    SweepLayout L{};
    L.barrier = c.take<unsigned int>(sizeof(unsigned int));
    L.anchors = c.take<int>((size_t)S * N * 2 * sizeof(int));
    L.scratch = c.take<void>((size_t)S * M * W * W * sizeof(cplx<T>));
    L.omax = c.take<void>((size_t)S * W * sizeof(T));
    L.peak = c.take<void>((size_t)2 * S * W * sizeof(T));
    L.tmax = c.take<void>((size_t)S * W * sizeof(T));
    L.err_part = c.take<double>((size_t)S * N * (W / kMinTC) * 3 * sizeof(double));
    L.bytes = c.off;
    return L;
}

template <typename T, int W>
int run_sweep(const PtySweepArgs* a, cudaStream_t st) {
    const int M = a->modes, N = a->n_positions, S = a->n_slots;
    SweepLayout L = carve_sweep<T>(a->workspace, W, M, N, S);
    if (!a->workspace || a->workspace_bytes < (int64_t)L.bytes) return PTY_ERR_ARGUMENT;
    const cplx<T>* tw = twiddles<T, W>(st);
    if (!tw) return PTY_ERR_CUDA;

    SweepDev P{};
    P.W = W; P.M = M; P.N = N; P.nslots = S;
    P.alpha_o = a->alpha_obj; P.alpha_p = a->alpha_probe; P.beta = a->beta; P.gamma = a->gamma;
    P.eps_rel = a->epsilon_rel;
    P.update_probe = a->update_probe; P.track_mod = a->track_modulus; P.sense = a->sense;
    P.barrier = L.barrier; P.anchors = L.anchors; P.scratch = L.scratch;
    P.omax_part = L.omax; P.peak_part = L.peak; P.tmax_part = L.tmax;
    P.err_part = L.err_part; P.twiddles = tw;
    ErrOut outs{};
    for (int s = 0; s < S; ++s) {
        const PtySlot& h = a->slots[s];
        if (!h.obj || !h.probes || !h.patterns || !h.positions || !h.order || !h.status || !h.err_out)
            return PTY_ERR_ARGUMENT;
        if (a->sense != PTY_SENSE_NONE && !h.stage) return PTY_ERR_ARGUMENT;
        if (h.H < W || h.Wc < W) return PTY_ERR_ARGUMENT;
        P.slot[s] = SlotDev{h.obj, h.H, h.Wc, h.r0, h.c0, h.probes, h.patterns, h.positions,
                            h.order, h.stage, h.err_out, h.status};
        outs.p[s] = h.err_out;
    }

    // launch geometry: kSweepThreads-thread CTAs, `per_sm` of them per SM
    // (default 2 so one CTA's loads overlap the other's FFTs), cooperative.
    // Tiles: the smallest power-of-two rows/columns per item that keep the
    // item count <= the CTA count (every CTA busy even for one reconstruction),
    // bounded by the per-CTA shared-memory budget.  PTY_TR / PTY_TC /
    // PTY_CTAS_PER_SM override (tuning).
    const int sms = sm_count();
    int per_sm = std::max(1, env_int("PTY_CTAS_PER_SM", kSweepMinCtasPerSm));
    const size_t smem_sm = max_smem_per_sm();
    const size_t fixed = sweep_smem_fixed<T, W>();
    const size_t budget = std::min(max_dyn_smem(), smem_sm / per_sm - 1024 - 512) - fixed;
    const int grid = sms * per_sm;
    constexpr int LS = line_stride<W>();
    const size_t line_bytes = (size_t)LS * sizeof(cplx<T>);
    int TR = env_int("PTY_TR", 0);
    if (TR <= 0) {
        TR = 1;
        while (TR < W && (long)S * (W / TR) > grid && (size_t)2 * TR * M * line_bytes <= budget) TR *= 2;
    }
    int TC = env_int("PTY_TC", 0);
    if (TC <= 0) {
        TC = kMinTC;
        while (TC < W && (long)S * (W / TC) > grid && (size_t)2 * TC * M * line_bytes <= budget) TC *= 2;
    }
    if (TR < 1 || TR > W || (W % TR) || TC < kMinTC || TC > W || (W % TC)) return PTY_ERR_ARGUMENT;
    const int nRT = W / TR, nCT = W / TC;
    const int K = (S * nCT + grid - 1) / grid;
    const size_t tile_bytes = std::max((size_t)TR * M * line_bytes, (size_t)K * M * TC * line_bytes);
    if (tile_bytes > budget) return PTY_ERR_ARGUMENT;   // too many replicas for the resident column tiles
    P.TR = TR; P.TC = TC; P.nRT = nRT; P.nCT = nCT; P.K = K;
    P.lgTR = 0; while ((1 << P.lgTR) < TR) ++P.lgTR;
    P.lgTC = 0; while ((1 << P.lgTC) < TC) ++P.lgTC;
    const size_t smem = fixed + tile_bytes;

    auto kern = sweep_kernel<T, W>;
    if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess)
        return PTY_ERR_CUDA;
    int fit = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&fit, kern, kSweepThreads, smem) != cudaSuccess || fit < per_sm)
        return PTY_ERR_CUDA;   // the cooperative grid must be co-resident

    // debug timeline (PTY_TIMELINE=<steps>): per-CTA phase completion stamps
    const int tl_steps = std::min(env_int("PTY_TIMELINE", 0), N);
    unsigned long long* tl = nullptr;
    if (tl_steps > 0) {
        if (cudaMalloc(&tl, (size_t)tl_steps * 5 * grid * sizeof(unsigned long long)) != cudaSuccess) return PTY_ERR_CUDA;
        P.timeline = tl;
        P.timeline_steps = tl_steps;
    }
    if (cudaMemsetAsync(L.barrier, 0, sizeof(unsigned int), st) != cudaSuccess) return PTY_ERR_CUDA;
    if (cudaMemsetAsync(L.err_part, 0, (size_t)S * N * nCT * 3 * sizeof(double), st) != cudaSuccess)
        return PTY_ERR_CUDA;
    void* args[] = {&P};
    cudaError_t e = cudaLaunchCooperativeKernel((const void*)kern, dim3(grid), dim3(kSweepThreads), args, smem, st);
    if (e != cudaSuccess) return PTY_ERR_CUDA;
    sweep_finalize_kernel<<<S, 32, 0, st>>>(L.err_part, N, nCT, S, outs);
    count(2);
    if (tl) {
        g_timeline.assign((size_t)tl_steps * 5 * grid, 0ull);
        cudaMemcpyAsync(g_timeline.data(), tl, g_timeline.size() * sizeof(unsigned long long),
                        cudaMemcpyDeviceToHost, st);
        cudaStreamSynchronize(st);
        cudaFree(tl);
        g_timeline_grid = grid;
    }
    return last_status();
}

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
    if (dtype == PTY_DTYPE_C64) return (int64_t)carve_sweep<float>(nullptr, W, M, N, S).bytes;
    if (dtype == PTY_DTYPE_C128) return (int64_t)carve_sweep<double>(nullptr, W, M, N, S).bytes;
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
    const size_t nIB = (size_t)(npts + 7) / 8;
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
    if (real_inputs && (!ref_real || !mov_real)) return PTY_ERR_ARGUMENT;
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
            RefPart* rpart = c.take<RefPart>((size_t)n * ((npts + 7) / 8) * sizeof(RefPart));
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
