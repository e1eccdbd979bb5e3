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
constexpr int GROUP_M = 8;  // tile-rows per rasterisation group

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
};

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

// The configurations the launcher chooses from (tools/gemm_tune.cu on B200, profiles/gemm_tune_r01.json:
// 8192^3 and the C3 trailing shapes; cuBLAS DGEMM reaches 35.7-36.4 TFLOP/s there).
using CfgWide = GemmCfg<128, 64, 2, 2, 4>;   // NN / NT, large: 33.3-33.7 TFLOP/s
using CfgMid = GemmCfg<64, 64, 2, 2, 3>;     // TN / TT, large: 33.6-34.0 TFLOP/s; medium shapes
using CfgSmall = GemmCfg<64, 32, 2, 2, 3>;   // small / skinny: most CTAs, 33 TFLOP/s when large

}  // namespace bqrrp
