// dgemm.cuh — FP64 tensor-core GEMM engine for sm_100a (DMMA via mma.sync.m8n8k4.f64).
//
// sm_100a has no f64 tcgen05.mma kind (ptxas rejects .kind::f64); the FP64 tensor path is the
// warp-synchronous DMMA.8x8x4 with register accumulators.  This engine serves every
// dense contraction of the BQRRP iteration: the sketch (a1), the sketch LU / QR trailing updates (a2),
// SYRK / TRSM of the CholQR panel (a4), the compact-WY trailing update (a5) and the sketch update (a6).
//
//   C(MxN) = alpha * op(A)(MxK) * op(B)(KxN) + beta * C,   column-major, op = identity or transpose.
//
// CTA tile BM x BN x BK = 128 x 128 x 16, 256 threads = 8 warps (2 x 4), warp tile 64 x 32 = 8 x 4
// DMMA tiles; STAGES-deep cp.async pipeline; 8-byte cp.async with zero-fill handles every ragged edge
// and any alignment (sub-matrix views start at arbitrary rows).  Shared tiles keep the operand's
// contiguous axis contiguous ("MN-major" [k][mn] or "K-major" [mn][k]) with a 4-double pad that
// makes every fragment load conflict-free.  Summation over K is in a fixed order
// (k-tiles ascending, DMMA-internal order inside a k4 step): results are deterministic and
// independent of the launch grid.  Optional split-K writes fixed slices that a second kernel sums
// in slice order.  `tri` = 1 computes only tiles intersecting the lower triangle (SYRK).
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace bqrrp {

constexpr int GEMM_BM = 128, GEMM_BN = 128, GEMM_BK = 16, GEMM_THREADS = 256, GEMM_STAGES = 4;
constexpr int GEMM_PAD = 4;

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

// Shared-memory tile of one operand.  MNMAJOR: s[k][mn] (row stride 128+PAD); else s[mn][k] (16+PAD).
template <bool MNMAJOR>
struct TileLayout {
    static constexpr int LD = MNMAJOR ? (GEMM_BM + GEMM_PAD) : (GEMM_BK + GEMM_PAD);
    static constexpr int SIZE = MNMAJOR ? GEMM_BK * LD : GEMM_BM * LD;  // doubles
    __device__ static __forceinline__ int off(int mn, int k) { return MNMAJOR ? k * LD + mn : mn * LD + k; }
};

// Load one BK-slice of an operand tile: rows mn0..mn0+127 of op(X), k0..k0+15.
//   op(X)(mn, k) = X[mn + k*ld] when X is stored mn-contiguous (MNMAJOR), else X[k + mn*ld].
template <bool MNMAJOR>
__device__ __forceinline__ void load_tile(double* s, const double* X, int64_t ld, int64_t mn0, int64_t k0,
                                          int64_t MN, int64_t K, int tid)
{
    using L = TileLayout<MNMAJOR>;
#pragma unroll
    for (int it = 0; it < (GEMM_BM * GEMM_BK) / GEMM_THREADS; ++it) {
        int e = it * GEMM_THREADS + tid;
        int mn, k;
        if (MNMAJOR) { mn = e % GEMM_BM; k = e / GEMM_BM; }
        else { k = e % GEMM_BK; mn = e / GEMM_BK; }
        int64_t gmn = mn0 + mn, gk = k0 + k;
        bool ok = (gmn < MN) && (gk < K);
        const double* src = ok ? (MNMAJOR ? X + gmn + gk * ld : X + gk + gmn * ld) : X;
        cp_async8(s + L::off(mn, k), src, ok);
    }
}

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

// TA: op(A) = A^T.  TB: op(B) = B^T.
// A operand (op(A) is M x K): stored m-contiguous unless TA.   B operand (op(B) is K x N): stored
// n-contiguous only if TB.
template <bool TA, bool TB>
__global__ void __launch_bounds__(GEMM_THREADS, 1) dgemm_kernel(GemmArgs g)
{
    constexpr bool A_MN = !TA;
    constexpr bool B_MN = TB;
    using LA = TileLayout<A_MN>;
    using LB = TileLayout<B_MN>;
    extern __shared__ __align__(16) double smem[];
    double* sA = smem;
    double* sB = smem + GEMM_STAGES * LA::SIZE;

    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int wm = warp & 1, wn = warp >> 1;  // 2 x 4 warps
    const int64_t m0 = (int64_t)blockIdx.x * GEMM_BM, n0 = (int64_t)blockIdx.y * GEMM_BN;
    if (g.tri && m0 + GEMM_BM <= n0) return;  // tile strictly above the diagonal
    const int64_t kbeg = (int64_t)blockIdx.z * g.kchunk;
    const int64_t kend = (kbeg + g.kchunk < g.K) ? kbeg + g.kchunk : g.K;
    const int nk = (int)((kend - kbeg + GEMM_BK - 1) / GEMM_BK);

    const double* Ap = g.A;
    const double* Bp = g.B;
    // op(A) as an (M x K) operand: A_MN => element (m,k) at A[m + k*lda]; else at A[k + m*lda]
    // op(B) as an (N x K) operand: B_MN => element (n,k) at B[n + k*ldb]; else at B[k + n*ldb]

    double acc[8][4][2];
#pragma unroll
    for (int i = 0; i < 8; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;

#pragma unroll
    for (int st = 0; st < GEMM_STAGES - 1; ++st) {
        if (st < nk) {
            int64_t k0 = kbeg + (int64_t)st * GEMM_BK;
            load_tile<A_MN>(sA + st * LA::SIZE, Ap, g.lda, m0, k0, g.M, kend, tid);
            load_tile<B_MN>(sB + st * LB::SIZE, Bp, g.ldb, n0, k0, g.N, kend, tid);
        }
        cp_async_commit();
    }

    const int gid = lane >> 2, tig = lane & 3;
    for (int kt = 0; kt < nk; ++kt) {
        cp_async_wait<GEMM_STAGES - 2>();
        __syncthreads();
        {   // prefetch stage kt + STAGES - 1 (its buffer was consumed at iteration kt-1)
            int nt = kt + GEMM_STAGES - 1;
            if (nt < nk) {
                int buf = nt % GEMM_STAGES;
                int64_t k0 = kbeg + (int64_t)nt * GEMM_BK;
                load_tile<A_MN>(sA + buf * LA::SIZE, Ap, g.lda, m0, k0, g.M, kend, tid);
                load_tile<B_MN>(sB + buf * LB::SIZE, Bp, g.ldb, n0, k0, g.N, kend, tid);
            }
            cp_async_commit();
        }
        const double* tA = sA + (kt % GEMM_STAGES) * LA::SIZE;
        const double* tB = sB + (kt % GEMM_STAGES) * LB::SIZE;
#pragma unroll
        for (int kk = 0; kk < GEMM_BK; kk += 4) {
            double af[8], bf[4];
#pragma unroll
            for (int i = 0; i < 8; ++i) af[i] = tA[LA::off(wm * 64 + i * 8 + gid, kk + tig)];
#pragma unroll
            for (int j = 0; j < 4; ++j) bf[j] = tB[LB::off(wn * 32 + j * 8 + gid, kk + tig)];
#pragma unroll
            for (int i = 0; i < 8; ++i)
#pragma unroll
                for (int j = 0; j < 4; ++j) dmma_884(acc[i][j][0], acc[i][j][1], af[i], bf[j]);
        }
    }
    cp_async_wait<0>();

    // epilogue: C fragment (row gid, cols 2*tig + {0,1}) of each 8x8 tile
    if (g.ws) {  // split-K slice, plain store
        double* W = g.ws + (int64_t)blockIdx.z * g.M * g.N;
#pragma unroll
        for (int i = 0; i < 8; ++i)
#pragma unroll
            for (int j = 0; j < 4; ++j)
#pragma unroll
                for (int h = 0; h < 2; ++h) {
                    int64_t r = m0 + wm * 64 + i * 8 + gid, c = n0 + wn * 32 + j * 8 + 2 * tig + h;
                    if (r < g.M && c < g.N) W[r + c * g.M] = acc[i][j][h];
                }
        return;
    }
#pragma unroll
    for (int i = 0; i < 8; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j)
#pragma unroll
            for (int h = 0; h < 2; ++h) {
                int64_t r = m0 + wm * 64 + i * 8 + gid, c = n0 + wn * 32 + j * 8 + 2 * tig + h;
                if (r < g.M && c < g.N) {
                    double* p = g.C + r + c * g.ldc;
                    double v = g.alpha * acc[i][j][h];
                    if (g.beta != 0.0) v = fma(g.beta, *p, v);
                    *p = v;
                }
            }
}

// Fixed-order split-K reduction: C = alpha * sum_{z ascending} ws[z] + beta * C.
static __global__ void dgemm_splitk_reduce(int64_t M, int64_t N, int nsplit, const double* ws, double alpha, double beta,
                                    double* C, int64_t ldc, int tri)
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

inline size_t dgemm_smem_bytes(bool TA, bool TB)
{
    int a = (!TA) ? TileLayout<true>::SIZE : TileLayout<false>::SIZE;
    int b = TB ? TileLayout<true>::SIZE : TileLayout<false>::SIZE;
    return (size_t)GEMM_STAGES * (a + b) * sizeof(double);
}

}  // namespace bqrrp
