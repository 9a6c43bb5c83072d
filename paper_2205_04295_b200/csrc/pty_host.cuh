// pty_host.cuh -- host-side helpers shared by the translation units of
// libptycho_b200.so: launch counter, workspace carving, device queries,
// twiddle tables and dtype/window dispatch.
#pragma once
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <type_traits>
#include <vector>

#include "pty_aux.cuh"

namespace pty {

extern std::atomic<long long> g_launches;            // defined in pty_capi.cu
extern std::vector<unsigned long long> g_timeline;   // debug: last sweep's phase stamps
extern int g_timeline_grid;
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

inline int env_int(const char* name, int dflt) {
    const char* v = std::getenv(name);
    return v ? std::atoi(v) : dflt;
}

// L2 persistence window over a kernel's scratch (PTY_L2_PERSIST_MB > 0): the
// line-task kernels rewrite their scratch every phase; streaming inputs and
// outputs (patterns, object patches, numerator planes) would otherwise evict
// it between the write and the read.  Returns whether a window was set.
inline bool l2_window_set(cudaStream_t st, void* base, size_t bytes) {
    const int mb = env_int("PTY_L2_PERSIST_MB", 0);
    if (mb <= 0 || !base || !bytes) return false;
    static size_t limit = 0;
    const size_t want = (size_t)mb << 20;
    if (limit != want) {
        if (cudaDeviceSetLimit(cudaLimitPersistingL2CacheSize, want) != cudaSuccess) {
            cudaGetLastError();
            return false;
        }
        limit = want;
    }
    cudaStreamAttrValue v{};
    v.accessPolicyWindow.base_ptr = base;
    v.accessPolicyWindow.num_bytes = std::min(bytes, want);
    v.accessPolicyWindow.hitRatio = 1.0f;
    v.accessPolicyWindow.hitProp = cudaAccessPropertyPersisting;
    v.accessPolicyWindow.missProp = cudaAccessPropertyStreaming;
    if (cudaStreamSetAttribute(st, cudaStreamAttributeAccessPolicyWindow, &v) != cudaSuccess) {
        cudaGetLastError();
        return false;
    }
    return true;
}
inline void l2_window_clear(cudaStream_t st) {
    cudaStreamAttrValue v{};
    v.accessPolicyWindow.num_bytes = 0;
    cudaStreamSetAttribute(st, cudaStreamAttributeAccessPolicyWindow, &v);
    cudaGetLastError();
}

inline int pow2_floor(int x) {
    int p = 1;
    while (p * 2 <= x) p *= 2;
    return p;
}

inline int sm_count() {
    int dev = 0, n = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    return n;
}

inline size_t max_smem_per_sm() {
    int dev = 0, n = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&n, cudaDevAttrMaxSharedMemoryPerMultiprocessor, dev);
    return (size_t)n;
}

inline size_t max_dyn_smem() {
    int dev = 0, n = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&n, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
    return (size_t)n;
}

// Stream-ordered allocations (small per-call temporaries): keep the device's
// default pool's memory cached.  With the default release threshold of 0 the
// pool returns its memory to the driver at every synchronisation and the next
// cudaMallocAsync re-maps it (measured: 1-600 ms stalls per call).
inline void keep_pool_memory() {
    static bool done[64] = {};
    static std::mutex mu;
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64) return;
    std::lock_guard<std::mutex> lock(mu);
    if (done[dev]) return;
    cudaMemPool_t pool;
    if (cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
        unsigned long long threshold = ~0ull;
        cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &threshold);
    }
    done[dev] = true;
}

// ------------------------------------------------------------- twiddles --
// Twiddle tables: one device buffer per (device, dtype, W), built once on
// first use (float64 twiddle_kernel, then rounded); guarded for callers on
// several host threads / devices.
constexpr int kMaxDevices = 64;
template <typename T, int W> inline const cplx<T>* twiddles(cudaStream_t st) {
    static cplx<T>* table[kMaxDevices] = {};
    static std::mutex mu;
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= kMaxDevices) return nullptr;
    std::lock_guard<std::mutex> lock(mu);
    if (!table[dev]) {
        cplx<T>* t = nullptr;
        if (cudaMalloc(&t, W * sizeof(cplx<T>)) != cudaSuccess) return nullptr;
        twiddle_kernel<T, W><<<(W + 255) / 256, 256, 0, st>>>(t);
        count();
        table[dev] = t;
    }
    return table[dev];
}

}  // namespace pty
