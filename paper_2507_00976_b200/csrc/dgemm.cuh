// dgemm.cuh — FP64 tensor-core GEMM engine for sm_100a (DMMA via mma.sync.m8n8k4.f64).
//
// sm_100a has no f64 tcgen05.mma kind (ptxas rejects .kind::f64); the FP64 tensor path is the
// warp-synchronous DMMA.8x8x4 with register accumulators.  This engine serves every
// dense contraction of the BQRRP iteration: the sketch (a1), the sketch LU / QR trailing updates (a2),
// SYRK / TRSM of the CholQR panel (a4), the compact-WY trailing update (a5) and the sketch update (a6).
//
//   C(MxN) = alpha * op(A)(MxK) * op(B)(KxN) + beta * C,   column-major, op = identity or transpose.
//
// Tiling is a template: CTA tile BM x BN x 16, WARPS_M x WARPS_N warps, each warp (BM/WARPS_M) x
// (BN/WARPS_N) = MI x NI DMMA tiles; STAGES-deep cp.async pipeline; 8-byte cp.async with zero-fill
// handles every ragged edge and any alignment (sub-matrix views start at arbitrary rows).  Shared
// tiles keep the operand's contiguous axis contiguous ("MN-major" [k][mn] or "K-major" [mn][k]) with a
// pad (row stride = 4 mod 16 doubles) that makes every fragment load conflict-free.
// Summation over K is in a fixed order (k-tiles ascending, DMMA-internal order inside a k4 step):
// results are deterministic and independent of the launch grid.  Optional split-K writes fixed slices
// that a second kernel sums in slice order.  `tri` = 1 skips tiles strictly above the diagonal (SYRK).
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace bqrrp {

constexpr int GEMM_BK = 16;
#ifndef BQRRP_GROUP_M
#define BQRRP_GROUP_M 32
#endif
constexpr int GROUP_M = BQRRP_GROUP_M;  // tile-rows per rasterisation group (experiments: -DBQRRP_GROUP_M=…)

__device__ __forceinline__ void dmma_884(double& c0, double& c1, double a, double b)
{
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                 : "+d"(c0), "+d"(c1)
                 : "d"(a), "d"(b));
}

__device__ __forceinline__ void cp_async8(void* smem, const void* gmem, bool pred)
{
    unsigned s = (unsigned)__cvta_generic_to_shared(smem);
    int sz = pred ? 8 : 0;
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(s), "l"(gmem), "r"(sz));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N)); }

// Shared-memory tile of one operand, MN x 16.  MNMAJOR: s[k][mn] (row stride MN+4); else s[mn][k]
// (row stride 20).  Both strides are 4 mod 16 doubles: the 16 lanes of a half-warp fragment load
// (4 consecutive mn x 4 consecutive k) hit 16 distinct 8-byte bank pairs.
template <bool MNMAJOR, int MN>
struct TileLayout {
    static constexpr int LD = MNMAJOR ? (MN + 4) : (GEMM_BK + 4);
    static constexpr int SIZE = MNMAJOR ? GEMM_BK * LD : MN * LD;  // doubles
    __device__ static __forceinline__ int off(int mn, int k) { return MNMAJOR ? k * LD + mn : mn * LD + k; }
};

// Per-thread loader of one operand: element e = it * THREADS + tid of the MN x 16 slice.
//   MNMAJOR (X[mn + k*ld]):  mn = tid % MN (fixed), k = it * (THREADS/MN) + tid / MN
//   K-major (X[k + mn*ld]):  k = tid % 16 (fixed),  mn = it * (THREADS/16) + tid / 16
// Addresses advance by a constant per `it` and per k-tile; interior tiles skip all predicates.
template <bool MNMAJOR, int MN, int THREADS>
struct Loader {
    using L = TileLayout<MNMAJOR, MN>;
    static constexpr int PER = (MN * GEMM_BK) / THREADS;
    static_assert((MN * GEMM_BK) % THREADS == 0, "tile / thread mismatch");
    static_assert(MNMAJOR ? (THREADS % MN == 0) : (THREADS % GEMM_BK == 0), "thread layout");
    static constexpr int STEP_FIXED = MNMAJOR ? THREADS / MN : THREADS / GEMM_BK;  // k (or mn) per `it`
    const double* p;    // element it = 0 of the current k-tile
    int64_t it_stride;  // pointer delta between consecutive `it`
    int64_t kt_stride;  // pointer delta per k-tile
    int soff;           // shared offset of element it = 0
    int kfix;           // this thread's k (K-major) or k of it = 0 (MN-major), relative to k0
    unsigned mn_ok;     // bit it: mn in range

    __device__ __forceinline__ Loader(const double* X, int64_t ld, int64_t mn0, int64_t k0, int64_t MNtot, int tid)
    {
        if (MNMAJOR) {
            int mn = tid % MN, k = tid / MN;
            p = X + (mn0 + mn) + (k0 + k) * ld;
            it_stride = (int64_t)STEP_FIXED * ld;
            kt_stride = (int64_t)GEMM_BK * ld;
            soff = L::off(mn, k);
            kfix = k;
            mn_ok = (mn0 + mn < MNtot) ? 0xffffffffu : 0u;
        } else {
            int k = tid % GEMM_BK, mn = tid / GEMM_BK;
            p = X + (k0 + k) + (mn0 + mn) * ld;
            it_stride = (int64_t)STEP_FIXED * ld;
            kt_stride = GEMM_BK;
            soff = L::off(mn, k);
            kfix = k;
            mn_ok = 0;
#pragma unroll
            for (int it = 0; it < PER; ++it)
                if (mn0 + mn + it * STEP_FIXED < MNtot) mn_ok |= 1u << it;
        }
    }
    static constexpr int SOFF_STEP = STEP_FIXED * L::LD;  // shared offset between consecutive `it`
    // load the k-tile whose first k is k0 (krem = valid k count remaining from k0) into buffer s
    __device__ __forceinline__ void load(double* s, int krem, bool interior) const
    {
        if (interior && krem >= GEMM_BK) {
#pragma unroll
            for (int it = 0; it < PER; ++it) cp_async8(s + soff + it * SOFF_STEP, p + it * it_stride, true);
        } else {
#pragma unroll
            for (int it = 0; it < PER; ++it) {
                int k = MNMAJOR ? kfix + it * STEP_FIXED : kfix;
                bool ok = ((mn_ok >> it) & 1u) && (k < krem);
                cp_async8(s + soff + it * SOFF_STEP, ok ? (const void*)(p + it * it_stride) : (const void*)p, ok);
            }
        }
    }
    __device__ __forceinline__ void advance() { p += kt_stride; }
};

struct GemmArgs {
    int64_t M, N, K;
    double alpha, beta;
    const double* A; int64_t lda;
    const double* B; int64_t ldb;
    double* C; int64_t ldc;
    double* ws;      // split-K slices (M x N each, ld M) or nullptr
    int64_t kchunk;  // K range per split (multiple of BK)
    int tri;         // 1: only tiles touching the lower triangle (m >= n) are computed
    int a_lower;     // 1: op(A) is lower triangular (TRMM): the K range of row tile m0 ends at m0 + BM (v2)
    // Tile handshake with a concurrent reader of C (v2, the pivot-aware lookahead).  Per
    // output tile (tile_m * tiles_n + tile_n): hs_state 0 = not started, 1 = started, 2 = written;
    // hs_readers = readers currently copying the tile's PRE-update values.  A CTA publishes 1 (SC fence)
    // before anything else, waits for hs_readers == 0 before its epilogue stores, and publishes 2 after.
    int* hs_state;
    int* hs_readers;
};

__device__ __forceinline__ int ld_acquire_gpu(const int* p)
{
    int v;
    asm volatile("ld.acquire.gpu.global.b32 %0, [%1];\n" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void st_release_gpu(int* p, int v)
{
    asm volatile("st.release.gpu.global.b32 [%0], %1;\n" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ void fence_sc_gpu() { asm volatile("fence.sc.gpu;\n" ::: "memory"); }

template <int BM_, int BN_, int WARPS_M_, int WARPS_N_, int STAGES_>
struct GemmCfg {
    static constexpr int BM = BM_, BN = BN_, WARPS_M = WARPS_M_, WARPS_N = WARPS_N_, STAGES = STAGES_;
    static constexpr int THREADS = 32 * WARPS_M * WARPS_N;
    static constexpr int MI = BM / WARPS_M / 8, NI = BN / WARPS_N / 8;
    static constexpr int MIN_BLOCKS = (THREADS <= 128 && MI * NI <= 16) ? 4 : 1;
};

// TA: op(A) = A^T.  TB: op(B) = B^T.
// A operand (op(A) is M x K): stored m-contiguous unless TA.  B operand (op(B) is K x N): stored
// n-contiguous only if TB.
template <class Cfg, bool TA, bool TB>
__global__ void __launch_bounds__(Cfg::THREADS, Cfg::MIN_BLOCKS) dgemm_kernel(GemmArgs g)
{
    constexpr int BM = Cfg::BM, BN = Cfg::BN, THREADS = Cfg::THREADS, STAGES = Cfg::STAGES;
    constexpr int MI = Cfg::MI, NI = Cfg::NI, WM = BM / Cfg::WARPS_M, WN = BN / Cfg::WARPS_N;
    constexpr bool A_MN = !TA;
    constexpr bool B_MN = TB;
    using LA = TileLayout<A_MN, BM>;
    using LB = TileLayout<B_MN, BN>;
    extern __shared__ __align__(16) double smem[];
    double* sA = smem;
    double* sB = smem + STAGES * LA::SIZE;

    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int wm = warp % Cfg::WARPS_M, wn = warp / Cfg::WARPS_M;
    // grouped rasterisation of the 1-D tile index (GROUP_M tile-rows per group) for L2 reuse of the
    // operand tiles among the CTAs resident at the same time
    int64_t tile_m, tile_n;
    {
        const int64_t tiles_m = (g.M + BM - 1) / BM, tiles_n = (g.N + BN - 1) / BN;
        const int64_t pid = blockIdx.x, in_group = (int64_t)GROUP_M * tiles_n;
        const int64_t first_m = (pid / in_group) * GROUP_M;
        const int64_t gsize = (tiles_m - first_m < GROUP_M) ? tiles_m - first_m : GROUP_M;
        tile_m = first_m + (pid % in_group) % gsize;
        tile_n = (pid % in_group) / gsize;
    }
    const int64_t m0 = tile_m * BM, n0 = tile_n * BN;
    if (g.tri && m0 + BM <= n0) return;  // tile strictly above the diagonal
    const int64_t kbeg = (int64_t)blockIdx.z * g.kchunk;
    const int64_t kend = (kbeg + g.kchunk < g.K) ? kbeg + g.kchunk : g.K;
    const int nk = (int)((kend - kbeg + GEMM_BK - 1) / GEMM_BK);

    const int gid = lane >> 2, tig = lane & 3;
    // C as the accumulator's initial value when alpha = +-1 (C = alpha (AB + alpha beta C)): the C read
    // is issued before the main loop and overlaps it instead of stalling the epilogue.
    const bool preload = (g.ws == nullptr) && (g.beta != 0.0) && (g.alpha == 1.0 || g.alpha == -1.0);
    const double cscale = g.alpha * g.beta;
    double acc[MI][NI][2];
#pragma unroll
    for (int i = 0; i < MI; ++i)
#pragma unroll
        for (int j = 0; j < NI; ++j)
#pragma unroll
            for (int h = 0; h < 2; ++h) {
                double v = 0.0;
                if (preload) {
                    int64_t r = m0 + wm * WM + i * 8 + gid, c = n0 + wn * WN + j * 8 + 2 * tig + h;
                    if (r < g.M && c < g.N) v = cscale * g.C[r + c * g.ldc];
                }
                acc[i][j][h] = v;
            }

    Loader<A_MN, BM, THREADS> ldA(g.A, g.lda, m0, kbeg, g.M, tid);
    Loader<B_MN, BN, THREADS> ldB(g.B, g.ldb, n0, kbeg, g.N, tid);
    const bool interior = (m0 + BM <= g.M) && (n0 + BN <= g.N);
#pragma unroll
    for (int st = 0; st < STAGES - 1; ++st) {
        if (st < nk) {
            int krem = (int)(kend - (kbeg + (int64_t)st * GEMM_BK));
            ldA.load(sA + st * LA::SIZE, krem, interior);
            ldB.load(sB + st * LB::SIZE, krem, interior);
            ldA.advance();
            ldB.advance();
        }
        cp_async_commit();
    }

    for (int kt = 0; kt < nk; ++kt) {
        cp_async_wait<STAGES - 2>();
        __syncthreads();
        {   // prefetch stage kt + STAGES - 1 (its buffer was consumed at iteration kt-1)
            int nt = kt + STAGES - 1;
            if (nt < nk) {
                int buf = nt % STAGES;
                int krem = (int)(kend - (kbeg + (int64_t)nt * GEMM_BK));
                ldA.load(sA + buf * LA::SIZE, krem, interior);
                ldB.load(sB + buf * LB::SIZE, krem, interior);
                ldA.advance();
                ldB.advance();
            }
            cp_async_commit();
        }
        const double* tA = sA + (kt % STAGES) * LA::SIZE;
        const double* tB = sB + (kt % STAGES) * LB::SIZE;
#pragma unroll
        for (int kk = 0; kk < GEMM_BK; kk += 4) {
            double af[MI], bf[NI];
#pragma unroll
            for (int i = 0; i < MI; ++i) af[i] = tA[LA::off(wm * WM + i * 8 + gid, kk + tig)];
#pragma unroll
            for (int j = 0; j < NI; ++j) bf[j] = tB[LB::off(wn * WN + j * 8 + gid, kk + tig)];
#pragma unroll
            for (int i = 0; i < MI; ++i)
#pragma unroll
                for (int j = 0; j < NI; ++j) dmma_884(acc[i][j][0], acc[i][j][1], af[i], bf[j]);
        }
    }
    cp_async_wait<0>();

    // epilogue: C fragment (row gid, cols 2*tig + {0,1}) of each 8x8 tile
    if (g.ws) {  // split-K slice, plain store
        double* W = g.ws + (int64_t)blockIdx.z * g.M * g.N;
#pragma unroll
        for (int i = 0; i < MI; ++i)
#pragma unroll
            for (int j = 0; j < NI; ++j)
#pragma unroll
                for (int h = 0; h < 2; ++h) {
                    int64_t r = m0 + wm * WM + i * 8 + gid, c = n0 + wn * WN + j * 8 + 2 * tig + h;
                    if (r < g.M && c < g.N) W[r + c * g.M] = acc[i][j][h];
                }
        return;
    }
#pragma unroll
    for (int i = 0; i < MI; ++i)
#pragma unroll
        for (int j = 0; j < NI; ++j)
#pragma unroll
            for (int h = 0; h < 2; ++h) {
                int64_t r = m0 + wm * WM + i * 8 + gid, c = n0 + wn * WN + j * 8 + 2 * tig + h;
                if (r < g.M && c < g.N) {
                    double* p = g.C + r + c * g.ldc;
                    double v = g.alpha * acc[i][j][h];
                    if (!preload && g.beta != 0.0) v = fma(g.beta, *p, v);
                    *p = v;
                }
            }
}

// Fixed-order split-K reduction: C = alpha * sum_{z ascending} ws[z] + beta * C.
static __global__ void dgemm_splitk_reduce(int64_t M, int64_t N, int nsplit, const double* ws, double alpha,
                                           double beta, double* C, int64_t ldc, int tri)
{
    int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    int64_t total = M * N;
    for (; idx < total; idx += (int64_t)gridDim.x * blockDim.x) {
        int64_t r = idx % M, c = idx / M;
        if (tri && r < c) continue;
        double s = 0.0;
        for (int z = 0; z < nsplit; ++z) s += ws[(int64_t)z * total + idx];
        double* p = C + r + c * ldc;
        double v = alpha * s;
        if (beta != 0.0) v = fma(beta, *p, v);
        *p = v;
    }
}

template <class Cfg, bool TA, bool TB>
constexpr size_t dgemm_smem_bytes()
{
    return (size_t)Cfg::STAGES *
           (TileLayout<!TA, Cfg::BM>::SIZE + TileLayout<TB, Cfg::BN>::SIZE) * sizeof(double);
}

// ------------------------------------------------------------------------------------------------
// v2 engine: 16-byte shared-memory fragment loads and 16-byte cp.async.
//
// DMMA.8x8x4 takes one A value (row gid, k slot tig) and one B value (k slot tig, col gid) per lane.
// The k values a DMMA step consumes can be ANY four of the k-tile as long as A and B agree, so k is
// processed in groups of 8 as two steps e = 0, 1 with lane tig taking k = 8 g + 2 tig + e.  A K-major
// operand tile (s[mn][k]) then serves both steps with ONE 16-byte load per 8x8 tile.  For an MN-major
// operand (s[k][mn]) the mn axis is paired instead: tiles 2p and 2p+1 of a warp take the interleaved
// rows (or columns) 16 p + 2 gid + {0, 1}, so one 16-byte load serves two tiles; the epilogue maps
// fragments back with the same interleave.  Half the shared-load instructions of v1; the K order is
// still fixed (deterministic, grid-independent).
//   MN-major tile: s[k][mn], row stride MN + 2 (= 2 mod 8 doubles: the 8 lanes of each 16-byte phase,
//                  (gid in {0,1}) x (tig in 0..3), hit 8 distinct 16-byte bank groups)
//   K-major tile:  s[mn][k], row stride BK, 16-byte unit u = k/2 stored at u ^ ((mn & 1) << 2)
//                  (XOR swizzle: rows gid = 0 / 1 of a phase land on bank groups 0-3 / 4-7)
template <bool MNMAJOR, int MN, int BK>
struct Tile2 {
    static constexpr int LD = MNMAJOR ? MN + 2 : BK;
    static constexpr int SIZE = MNMAJOR ? BK * LD : MN * BK;  // doubles
    __device__ static __forceinline__ int off(int mn, int k)
    {
        return MNMAJOR ? k * LD + mn : mn * BK + ((((k >> 1) ^ ((mn & 1) << 2))) << 1) + (k & 1);
    }
};

__device__ __forceinline__ void cp_async16(void* smem, const void* gmem, bool pred)
{
    unsigned s = (unsigned)__cvta_generic_to_shared(smem);
    int sz = pred ? 16 : 0;
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(s), "l"(gmem), "r"(sz));
}

__device__ __forceinline__ double2 lds128(const double* p)
{
    double2 v;
    unsigned a = (unsigned)__cvta_generic_to_shared(p);
    asm volatile("ld.shared.v2.f64 {%0, %1}, [%2];\n" : "=d"(v.x), "=d"(v.y) : "r"(a));
    return v;
}

// Loader of one operand in element pairs (2 consecutive doubles along the contiguous axis):
//   MNMAJOR (X[mn + k*ld]): pair index pp = tid % (MN/2) (fixed), k = it * STEP + tid / (MN/2)
//   K-major (X[k + mn*ld]): kp = tid % (BK/2) (fixed),  mn = it * STEP + tid / (BK/2)
// vec: X and ld allow 16-byte copies (X 16-byte aligned, ld even); interior + vec tiles use them.
template <bool MNMAJOR, int MN, int BK, int THREADS>
struct Loader2 {
    using L = Tile2<MNMAJOR, MN, BK>;
    static constexpr int PAIRS_FIXED = MNMAJOR ? MN / 2 : BK / 2;
    static constexpr int STEP = THREADS / PAIRS_FIXED;
    static constexpr int PER = (MN * BK / 2) / THREADS;
    static_assert((MN * BK / 2) % THREADS == 0 && THREADS % PAIRS_FIXED == 0, "tile / thread mismatch");
    static_assert(PER <= 32, "mask width");
    const double* p;
    int64_t it_stride, kt_stride, ld;
    int soff;   // shared offset of it = 0
    int kfix;   // k of it = 0 (MN-major) or this thread's first k (K-major), relative to the k-tile
    unsigned mn_ok0, mn_ok1;  // bit it: first / second element of the pair in range (MN-major: same k)

    __device__ __forceinline__ Loader2(const double* X, int64_t ld_, int64_t mn0, int64_t k0, int64_t MNtot, int tid)
    {
        ld = ld_;
        if (MNMAJOR) {
            int mn = 2 * (tid % PAIRS_FIXED), k = tid / PAIRS_FIXED;
            p = X + (mn0 + mn) + (k0 + k) * ld;
            it_stride = (int64_t)STEP * ld;
            kt_stride = (int64_t)BK * ld;
            soff = L::off(mn, k);
            kfix = k;
            mn_ok0 = (mn0 + mn < MNtot) ? 0xffffffffu : 0u;
            mn_ok1 = (mn0 + mn + 1 < MNtot) ? 0xffffffffu : 0u;
        } else {
            int k = 2 * (tid % PAIRS_FIXED), mn = tid / PAIRS_FIXED;
            p = X + (k0 + k) + (mn0 + mn) * ld;
            it_stride = (int64_t)STEP * ld;
            kt_stride = BK;
            soff = L::off(mn, k);
            kfix = k;
            mn_ok0 = 0;
#pragma unroll
            for (int it = 0; it < PER; ++it)
                if (mn0 + mn + it * STEP < MNtot) mn_ok0 |= 1u << it;
            mn_ok1 = mn_ok0;
        }
    }
    // shared offset of pair `it` (STEP rows further along the fixed-step axis)
    __device__ __forceinline__ int soff_it(int it) const
    {
        if (MNMAJOR) return soff + it * STEP * L::LD;
        // K-major: mn advances by STEP (even: the XOR swizzle term is unchanged)
        return soff + it * STEP * BK;
    }
    __device__ __forceinline__ void load(double* s, int krem, bool fast) const
    {
        if (fast && krem >= BK) {
#pragma unroll
            for (int it = 0; it < PER; ++it) cp_async16(s + soff_it(it), p + it * it_stride, true);
        } else {
#pragma unroll
            for (int it = 0; it < PER; ++it) {
                const double* q = p + it * it_stride;
                if (MNMAJOR) {
                    bool kok = kfix + it * STEP < krem;
                    bool ok0 = kok && ((mn_ok0 >> it) & 1u), ok1 = kok && ((mn_ok1 >> it) & 1u);
                    cp_async8(s + soff_it(it), ok0 ? (const void*)q : (const void*)p, ok0);
                    cp_async8(s + soff_it(it) + 1, ok1 ? (const void*)(q + 1) : (const void*)p, ok1);
                } else {
                    bool mok = (mn_ok0 >> it) & 1u;
                    bool ok0 = mok && (kfix < krem), ok1 = mok && (kfix + 1 < krem);
                    cp_async8(s + soff_it(it), ok0 ? (const void*)q : (const void*)p, ok0);
                    cp_async8(s + soff_it(it) + 1, ok1 ? (const void*)(q + 1) : (const void*)p, ok1);
                }
            }
        }
    }
    __device__ __forceinline__ void advance() { p += kt_stride; }
};

template <int BM_, int BN_, int BK_, int WARPS_M_, int WARPS_N_, int STAGES_, int MINB_>
struct Gemm2Cfg {
    static constexpr int BM = BM_, BN = BN_, BK = BK_, WARPS_M = WARPS_M_, WARPS_N = WARPS_N_, STAGES = STAGES_;
    static constexpr int THREADS = 32 * WARPS_M * WARPS_N;
    static constexpr int MI = BM / WARPS_M / 8, NI = BN / WARPS_N / 8;
    static constexpr int MIN_BLOCKS = MINB_;
    static_assert(BK % 8 == 0, "BK multiple of 8");
    static_assert(MI % 2 == 0 && NI % 2 == 0, "paired tiles");
};

template <class Cfg, bool TA, bool TB>
__global__ void __launch_bounds__(Cfg::THREADS, Cfg::MIN_BLOCKS) dgemm2_kernel(GemmArgs g, int vec)
{
    constexpr int BM = Cfg::BM, BN = Cfg::BN, BK = Cfg::BK, THREADS = Cfg::THREADS, STAGES = Cfg::STAGES;
    constexpr int MI = Cfg::MI, NI = Cfg::NI, WM = BM / Cfg::WARPS_M, WN = BN / Cfg::WARPS_N;
    constexpr bool A_MN = !TA;
    constexpr bool B_MN = TB;
    using LA = Tile2<A_MN, BM, BK>;
    using LB = Tile2<B_MN, BN, BK>;
    extern __shared__ __align__(16) double smem[];
    double* sA = smem;
    double* sB = smem + STAGES * LA::SIZE;

    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int wm = warp % Cfg::WARPS_M, wn = warp / Cfg::WARPS_M;
    const int64_t tiles_m = (g.M + BM - 1) / BM, tiles_n = (g.N + BN - 1) / BN;
    // persistent when the grid is smaller than the tile count (the bulk trailing update leaves SM slots
    // free for the concurrent critical-path kernels): tiles pid, pid + gridDim.x, ...
  for (int64_t pid = blockIdx.x; pid < tiles_m * tiles_n; pid += gridDim.x) {
    int64_t tile_m, tile_n;
    {
        const int64_t in_group = (int64_t)GROUP_M * tiles_n;
        const int64_t first_m = (pid / in_group) * GROUP_M;
        const int64_t gsize = (tiles_m - first_m < GROUP_M) ? tiles_m - first_m : GROUP_M;
        tile_m = first_m + (pid % in_group) % gsize;
        tile_n = (pid % in_group) / gsize;
    }
    const int64_t m0 = tile_m * BM, n0 = tile_n * BN;
    if (g.tri && m0 + BM <= n0) continue;
    const int64_t kbeg = (int64_t)blockIdx.z * g.kchunk;
    int64_t kend = (kbeg + g.kchunk < g.K) ? kbeg + g.kchunk : g.K;
    if (g.a_lower && kend > m0 + BM) kend = (m0 + BM > kbeg) ? m0 + BM : kbeg;  // op(A)(r, k) = 0 for k > r
    const int nk = (int)((kend - kbeg + BK - 1) / BK);
    int* const hs_st = g.hs_state ? g.hs_state + (tile_m * tiles_n + tile_n) : nullptr;
    if (hs_st && tid == 0) {
        atomicExch(hs_st, 1);
        fence_sc_gpu();  // Dekker with the reader: its (readers++, fence.sc, read state) vs (state = 1, fence.sc)
    }

    const int gid = lane >> 2, tig = lane & 3;
    // fragment -> matrix index maps (interleaved for MN-major operands, see above)
    auto row_of = [&](int i) -> int { return A_MN ? wm * WM + 16 * (i >> 1) + 2 * gid + (i & 1) : wm * WM + 8 * i + gid; };
    auto col_of = [&](int j, int slot) -> int {
        return B_MN ? wn * WN + 16 * (j >> 1) + 2 * slot + (j & 1) : wn * WN + 8 * j + slot;
    };
    const bool preload = (g.ws == nullptr) && (g.beta != 0.0) && (g.alpha == 1.0 || g.alpha == -1.0);
    const double cscale = g.alpha * g.beta;
    double acc[MI][NI][2];
#pragma unroll
    for (int i = 0; i < MI; ++i)
#pragma unroll
        for (int j = 0; j < NI; ++j)
#pragma unroll
            for (int h = 0; h < 2; ++h) {
                double v = 0.0;
                if (preload) {
                    int64_t r = m0 + row_of(i), c = n0 + col_of(j, 2 * tig + h);
                    if (r < g.M && c < g.N) v = cscale * g.C[r + c * g.ldc];
                }
                acc[i][j][h] = v;
            }

    Loader2<A_MN, BM, BK, THREADS> ldA(g.A, g.lda, m0, kbeg, g.M, tid);
    Loader2<B_MN, BN, BK, THREADS> ldB(g.B, g.ldb, n0, kbeg, g.N, tid);
    const bool fast = vec && (m0 + BM <= g.M) && (n0 + BN <= g.N);
#pragma unroll
    for (int st = 0; st < STAGES - 1; ++st) {
        if (st < nk) {
            int krem = (int)(kend - (kbeg + (int64_t)st * BK));
            ldA.load(sA + st * LA::SIZE, krem, fast);
            ldB.load(sB + st * LB::SIZE, krem, fast);
            ldA.advance();
            ldB.advance();
        }
        cp_async_commit();
    }

    for (int kt = 0; kt < nk; ++kt) {
        cp_async_wait<STAGES - 2>();
        __syncthreads();
        {
            int nt = kt + STAGES - 1;
            if (nt < nk) {
                int buf = nt % STAGES;
                int krem = (int)(kend - (kbeg + (int64_t)nt * BK));
                ldA.load(sA + buf * LA::SIZE, krem, fast);
                ldB.load(sB + buf * LB::SIZE, krem, fast);
                ldA.advance();
                ldB.advance();
            }
            cp_async_commit();
        }
        const double* tA = sA + (kt % STAGES) * LA::SIZE;
        const double* tB = sB + (kt % STAGES) * LB::SIZE;
#pragma unroll
        for (int kg = 0; kg < BK; kg += 8) {
            double af[2][MI], bf[2][NI];
            if (A_MN) {
#pragma unroll
                for (int e = 0; e < 2; ++e)
#pragma unroll
                    for (int ip = 0; ip < MI / 2; ++ip) {
                        double2 v = lds128(tA + LA::off(wm * WM + 16 * ip + 2 * gid, kg + 2 * tig + e));
                        af[e][2 * ip] = v.x;
                        af[e][2 * ip + 1] = v.y;
                    }
            } else {
#pragma unroll
                for (int i = 0; i < MI; ++i) {
                    double2 v = lds128(tA + LA::off(wm * WM + 8 * i + gid, kg + 2 * tig));
                    af[0][i] = v.x;
                    af[1][i] = v.y;
                }
            }
            if (B_MN) {
#pragma unroll
                for (int e = 0; e < 2; ++e)
#pragma unroll
                    for (int jp = 0; jp < NI / 2; ++jp) {
                        double2 v = lds128(tB + LB::off(wn * WN + 16 * jp + 2 * gid, kg + 2 * tig + e));
                        bf[e][2 * jp] = v.x;
                        bf[e][2 * jp + 1] = v.y;
                    }
            } else {
#pragma unroll
                for (int j = 0; j < NI; ++j) {
                    double2 v = lds128(tB + LB::off(wn * WN + 8 * j + gid, kg + 2 * tig));
                    bf[0][j] = v.x;
                    bf[1][j] = v.y;
                }
            }
#pragma unroll
            for (int e = 0; e < 2; ++e)
#pragma unroll
                for (int i = 0; i < MI; ++i)
#pragma unroll
                    for (int j = 0; j < NI; ++j) dmma_884(acc[i][j][0], acc[i][j][1], af[e][i], bf[e][j]);
        }
    }
    cp_async_wait<0>();

    if (g.ws) {
        double* W = g.ws + (int64_t)blockIdx.z * g.M * g.N;
#pragma unroll
        for (int i = 0; i < MI; ++i)
#pragma unroll
            for (int j = 0; j < NI; ++j)
#pragma unroll
                for (int h = 0; h < 2; ++h) {
                    int64_t r = m0 + row_of(i), c = n0 + col_of(j, 2 * tig + h);
                    if (r < g.M && c < g.N) W[r + c * g.M] = acc[i][j][h];
                }
    } else {
    if (hs_st) {  // no store while a reader is copying this tile's pre-update values
        if (tid == 0)
            while (ld_acquire_gpu(g.hs_readers + (hs_st - g.hs_state)) != 0) __nanosleep(64);
        __syncthreads();
    }
#pragma unroll
    for (int i = 0; i < MI; ++i)
#pragma unroll
        for (int j = 0; j < NI; ++j)
#pragma unroll
            for (int h = 0; h < 2; ++h) {
                int64_t r = m0 + row_of(i), c = n0 + col_of(j, 2 * tig + h);
                if (r < g.M && c < g.N) {
                    double* p = g.C + r + c * g.ldc;
                    double v = g.alpha * acc[i][j][h];
                    if (!preload && g.beta != 0.0) v = fma(g.beta, *p, v);
                    *p = v;
                }
            }
    }
    __syncthreads();  // the next tile's prologue overwrites stages other warps may still be reading
    if (hs_st && tid == 0) {
        __threadfence();
        st_release_gpu(hs_st, 2);
    }
  }
}

template <class Cfg, bool TA, bool TB>
constexpr size_t dgemm2_smem_bytes()
{
    return (size_t)Cfg::STAGES *
           (Tile2<!TA, Cfg::BM, Cfg::BK>::SIZE + Tile2<TB, Cfg::BN, Cfg::BK>::SIZE) * sizeof(double);
}

// 16-byte copies allowed for both operands
__host__ __forceinline__ int dgemm2_vec_ok(const GemmArgs& g)
{
    return ((((uintptr_t)g.A) & 15) == 0 && (g.lda % 2) == 0 && (((uintptr_t)g.B) & 15) == 0 && (g.ldb % 2) == 0) ? 1
                                                                                                                  : 0;
}

// The configurations the launcher chooses from (tools/gemm_tune.cu on B200, profiles/gemm_tune_r01.json:
// 8192^3 and the C3 trailing shapes; cuBLAS DGEMM reaches 35.7-36.4 TFLOP/s there).
// v1 (8-byte fragment loads; kept as the A/B baseline of tools/gemm_tune.cu, not used by the library):
using CfgWide = GemmCfg<128, 64, 2, 2, 4>;   // NN / NT, large: 33.3-33.7 TFLOP/s
using CfgMid = GemmCfg<64, 64, 2, 2, 3>;     // TN / TT, large: 33.6-34.0 TFLOP/s; medium shapes
using CfgSmall = GemmCfg<64, 32, 2, 2, 3>;   // small / skinny: most CTAs, 33 TFLOP/s when large
// v2 (the library's engine; profiles/gemm_tune_r01d_v2.json, cuBLAS 35.5-36.3 on the same shapes):
using Cfg2Mid = Gemm2Cfg<64, 64, 16, 2, 2, 3, 4>;    // every large GEMM: 35.3-36.0 TFLOP/s
using Cfg2Small = Gemm2Cfg<64, 32, 16, 2, 2, 3, 4>;  // small / skinny: 34.4-35.0 TFLOP/s when large

}  // namespace bqrrp
