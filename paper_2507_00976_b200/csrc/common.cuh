// common.cuh — shared plumbing of the BQRRP CUDA library (no method arithmetic here).
#pragma once
#include <cuda_runtime.h>
#include <atomic>
#include <cstdint>
#include <cstdio>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

namespace bqrrp {

// Error carried from a failing CUDA call up to the C-ABI, which maps it to BQRRP_ECUDA.
struct CudaError : std::runtime_error {
    explicit CudaError(const std::string& s) : std::runtime_error(s) {}
};

#define BQ_CUDA(x)                                                                                      \
    do {                                                                                                \
        cudaError_t e_ = (x);                                                                           \
        if (e_ != cudaSuccess)                                                                          \
            throw ::bqrrp::CudaError(std::string(#x) + " @ " + __FILE__ + ":" + std::to_string(__LINE__) + \
                                     ": " + cudaGetErrorString(e_));                                    \
    } while (0)

// Every kernel launch of the library is followed by BQ_LAUNCH_CHECK (or counted explicitly for
// cooperative launches): g_launches is the count bqrrp_launch_count() reports (atomic: calls on
// several host threads / streams are allowed).
extern std::atomic<unsigned long long> g_launches;
#define BQ_LAUNCH_CHECK()                \
    do {                                 \
        ++::bqrrp::g_launches;           \
        BQ_CUDA(cudaGetLastError());     \
    } while (0)

// Kernel attributes (dynamic shared memory above 48 KB, non-portable cluster sizes) are per DEVICE: each
// call site keeps one bit per device that has been configured (a race only repeats the idempotent call).
struct AttrOnce {
    std::atomic<unsigned long long> done{0};
};
template <typename K>
inline void ensure_attr(AttrOnce& o, K* kernel, cudaFuncAttribute attr, int value)
{
    int dev = 0;
    BQ_CUDA(cudaGetDevice(&dev));
    const unsigned long long bit = 1ull << (dev & 63);
    if (o.done.load(std::memory_order_acquire) & bit) return;
    BQ_CUDA(cudaFuncSetAttribute((const void*)kernel, attr, value));
    o.done.fetch_or(bit, std::memory_order_release);
}

inline int64_t cdiv(int64_t a, int64_t b) { return (a + b - 1) / b; }
inline int64_t imin(int64_t a, int64_t b) { return a < b ? a : b; }
inline int64_t imax(int64_t a, int64_t b) { return a > b ? a : b; }

// A column-major matrix view on the device.
struct Mat {
    double* p;
    int64_t ld;
    __host__ __device__ double* at(int64_t i, int64_t j) const { return p + i + j * ld; }
    __host__ __device__ Mat sub(int64_t i, int64_t j) const { return Mat{p + i + j * ld, ld}; }
};

// Optional per-phase timer: mark(p) closes the running phase and opens phase p.
enum Phase {
    PH_QRCP_WIDE = 0, PH_TRI_RANK, PH_COL_PERM, PH_QR_TALL, PH_APPLY_QT, PH_SAMPLE_UPDATE, PH_OTHER, PH_TOTAL,
    PH_APPLY_QT_BULK,  // the overlapped bulk GEMM of a5 (its own stream), not part of the sequential sum
    PH_COUNT
};
struct Timer {
    bool on = false;
    cudaStream_t st = 0;
    std::vector<std::pair<int, cudaEvent_t>> ev;
    struct Interval { int phase; cudaEvent_t a, b; };
    std::vector<Interval> iv;
    void begin_interval(cudaStream_t s, int phase)
    {
        if (!on) return;
        Interval x{phase, nullptr, nullptr};
        cudaEventCreate(&x.a);
        cudaEventCreate(&x.b);
        cudaEventRecord(x.a, s);
        iv.push_back(x);
    }
    void end_interval(cudaStream_t s)
    {
        if (!on || iv.empty()) return;
        cudaEventRecord(iv.back().b, s);
    }
    void mark(int phase)
    {
        if (!on) return;
        cudaEvent_t e;
        if (cudaEventCreate(&e) != cudaSuccess) return;
        cudaEventRecord(e, st);
        ev.push_back({phase, e});
    }
    void finish(float* out)
    {
        if (!on) return;
        for (int i = 0; i < PH_COUNT; ++i) out[i] = 0.f;
        if (!ev.empty()) {
            cudaEventSynchronize(ev.back().second);
            for (size_t i = 0; i + 1 < ev.size(); ++i) {
                float ms = 0.f;
                cudaEventElapsedTime(&ms, ev[i].second, ev[i + 1].second);
                out[ev[i].first] += ms;
            }
            float tot = 0.f;
            cudaEventElapsedTime(&tot, ev.front().second, ev.back().second);
            out[PH_TOTAL] = tot;
        }
        for (auto& x : iv) {
            float ms = 0.f;
            cudaEventSynchronize(x.b);
            cudaEventElapsedTime(&ms, x.a, x.b);
            out[x.phase] += ms;
            cudaEventDestroy(x.a);
            cudaEventDestroy(x.b);
        }
        iv.clear();
        for (auto& p : ev) cudaEventDestroy(p.second);
        ev.clear();
    }
};

// Execution context: stream + a bump allocator over one workspace buffer + split-K scratch.
// Device memory the library allocates itself (workspace when the caller passes none, the host entry's
// device copies, debug scratch) comes from a library-owned stream-ordered pool per device whose release
// threshold is unlimited: freed blocks stay mapped for the next call instead of being unmapped at every
// synchronisation (the default pool's threshold is 0, which made each bqrrp_factor_host call re-map ~40 GB
// at C3).  bqrrp_trim_memory() returns the cached blocks to the driver.
cudaMemPool_t lib_pool();
inline cudaError_t lib_malloc_async(void** p, size_t bytes, cudaStream_t st)
{
    return cudaMallocFromPoolAsync(p, bytes, lib_pool(), st);
}
template <typename T>
inline cudaError_t lib_malloc_async(T** p, size_t bytes, cudaStream_t st)
{
    return lib_malloc_async(reinterpret_cast<void**>(p), bytes, st);
}

// A low-priority stream confined to a partition of about `sms` SMs of the current device (a driver green
// context, created once per device and size and kept for the process).  The bulk trailing GEMM
// runs there when it is shorter than the latency-bound chain it overlaps, leaving whole SM groups to the chain's
// kernels.  nullptr when the driver has no green contexts; *got = the partition's SM count.
cudaStream_t green_stream(int sms, int* got);

struct Ctx {
    cudaStream_t stream = 0;
    int num_sms = 148;
    char* ws = nullptr;
    size_t ws_bytes = 0, ws_used = 0;
    double* splitk = nullptr;
    size_t splitk_elems = 0;
    int* flags = nullptr;  // device int[8]: see Flags
    Timer* timer = nullptr;
    bool force_breakdown = false;  // test hook (bqrrp_options.debug_flags): report a POTRF breakdown per panel
    int lu_gpref = 16;             // K-LU register leaf: preferred largest cluster (bqrrp_options.lu_leaf_cluster)
    int lu_grid_max = 0;           // K-LU cooperative grid leaf: at most this many CTAs (0 = num_sms)
    void mark(int phase) { if (timer) timer->mark(phase); }

    double* alloc(size_t n_doubles)
    {
        size_t bytes = ((n_doubles * sizeof(double)) + 255) & ~size_t(255);
        if (ws_used + bytes > ws_bytes) throw std::runtime_error("bqrrp workspace exhausted");
        double* p = reinterpret_cast<double*>(ws + ws_used);
        ws_used += bytes;
        return p;
    }
    template <typename T>
    T* alloc_as(size_t n)
    {
        return reinterpret_cast<T*>(alloc((n * sizeof(T) + 7) / 8));
    }
};

// A context for work queued on a second stream.  Its bump allocator is an arena reserved on the main
// context (later main-stream allocations cannot overlap it); it has no split-K slices (those belong to the
// main stream) and no timer.  The main context releases the arena (resets ws_used below it) only after its
// stream has waited for the side stream's work.
inline Ctx side_ctx(Ctx& main, const Ctx& side, size_t arena_doubles)
{
    Ctx sc = side;
    sc.splitk = nullptr;
    sc.splitk_elems = 0;
    sc.timer = nullptr;
    sc.ws = arena_doubles ? reinterpret_cast<char*>(main.alloc(arena_doubles)) : nullptr;
    sc.ws_bytes = arena_doubles * sizeof(double);
    sc.ws_used = 0;
    return sc;
}

// Device flag slots (int) written by kernels and read back once per iteration.
enum Flags { F_K = 0, F_ZERO_COL = 1, F_POTRF_INFO = 2, F_NONFINITE = 3, F_NT = 4, F_NFLAGS = 8 };

// ---- device helpers shared by the small kernels -------------------------------------------------
// 8-byte global -> shared async copy; src-size 0 (zero-fill) when !pred
__device__ __forceinline__ void cp_async8z(void* smem, const void* gmem, bool pred)
{
    unsigned s = (unsigned)__cvta_generic_to_shared(smem);
    int sz = pred ? 8 : 0;
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(s), "l"(gmem), "r"(sz));
}
__device__ __forceinline__ void cp_async_wait_all()
{
    asm volatile("cp.async.commit_group;\n" ::);
    asm volatile("cp.async.wait_group 0;\n" ::);
}

// Column-major slab -> shared, all copies in flight at once: dst[c*ldd + r] = src[r + c*lds] for
// r < rows_valid, zero for rows_valid <= r < rows_pad; c < cols.  Ends with a block barrier.
__device__ __forceinline__ void slab_load_async(double* dst, int ldd, const double* src, int64_t lds, int rows_valid,
                                                int rows_pad, int cols)
{
    for (int c = 0; c < cols; ++c)
        for (int r = threadIdx.x; r < rows_pad; r += blockDim.x) {
            bool ok = r < rows_valid;
            cp_async8z(dst + (size_t)c * ldd + r, ok ? (const void*)(src + r + c * lds) : (const void*)src, ok);
        }
    cp_async_wait_all();
    __syncthreads();
}

}  // namespace bqrrp
