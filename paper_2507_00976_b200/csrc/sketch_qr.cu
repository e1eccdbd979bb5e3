// sketch_qr.cu — K-SQR: R_sk, the R factor of the Householder QR of the permuted sketch
// (Alg. 2 step wide_qrcp:compute, "Done via standard unpivoted QR factorization, GEQRF").
//
// The sketch lives transposed (MskT, n x d); its trailing window Wsk = MskT(s:n, :)^T is d x w.
// GPU form (same result in exact arithmetic as QR of the whole d x w matrix):
//   1. Wq = Wsk(:, 0:p) (d x p, p = min(d, w)), Householder QR by recursive blocking: 32-column leaf
//      panels factored by one kernel launch (the register cluster leaf for <= 16 x 256 rows: one row per
//      thread, partial norms and dot products pushed to every CTA with st.async + mbarrier; otherwise a
//      shared-memory cluster or cooperative grid leaf; reflector convention H of DESIGN.md Z9/Z20), the
//      leaf also returns its T block (larft); interior nodes apply Q_left^T to the right half with three
//      DMMA GEMMs and merge T (T12 = -T11 (V1^T V2) T22).
//   2. R_sk(:, p:w)^T = Wsk(:, p:w)^T Q_sk with Q_sk = I - V T V^T formed explicitly: ONE DMMA GEMM
//      (optionally deferred to a second stream, or restricted to this rank's row blocks).
//   3. R_sk(:, 0:p)^T (upper trapezoidal, explicit zeros) is written back to MskT(s:s+p, :).
#include <cooperative_groups.h>
#include <cstdlib>

#include "blas.cuh"
#include "dsmem.cuh"
#include "bqrrp_internal.cuh"

namespace cg = cooperative_groups;

namespace bqrrp {

// Per-phase clock64 stamps of the K-SQR register leaf (experiments only: -DBQRRP_LEAF_TIMING builds, read by
// tools/leaf_timing.py; never in the product build).
#ifdef BQRRP_LEAF_TIMING
__device__ long long g_qleaf_ts[2][64][8];
#define QLEAF_TS(j, k)                                                                          \
    do {                                                                                        \
        if (threadIdx.x == 0 && (blockIdx.x == 0 || blockIdx.x == gridDim.x - 1) && (j) < 64)    \
            g_qleaf_ts[blockIdx.x == 0 ? 0 : 1][(j)][(k)] = clock64();                          \
    } while (0)
#else
#define QLEAF_TS(j, k) \
    do {               \
    } while (0)
#endif

constexpr int QR_JBMAX = 32;
constexpr size_t QR_GRID_SMEM = 200 * 1024;  // slab of the cooperative grid leaf (rows per CTA x leaf width)
constexpr int QR_XSTRIDE = 1 + QR_JBMAX;  // s2, p[1..jb)
constexpr int QR_THREADS = 256;

struct QrPanelArgs {
    double* A;
    int64_t ld;
    int64_t m;   // rows of Wq (d)
    int64_t c0;  // first column; active rows [c0, m)
    int jb;
    int R;
    double* tau;
    double* V;  // explicit reflectors, m x p (ld m), pre-zeroed
    double* T;  // T(c0:c0+jb, c0:c0+jb) written at T + c0 + c0*ldt
    int64_t ldt;
    double* xbuf;  // [2][G][QR_XSTRIDE] then [G][jb*jb] Gram partials
    double* rowj;  // [2][QR_JBMAX]: alpha, a_c of the pivot row
};

__global__ void __launch_bounds__(QR_THREADS, 1) qr_panel_kernel(QrPanelArgs a)
{
    cg::grid_group grid = cg::this_grid();
    extern __shared__ double sp[];  // sp[c * R + r]
    __shared__ double red[QR_THREADS / 32][QR_JBMAX + 1];
    __shared__ double wv[QR_JBMAX];
    __shared__ double s_tau, s_beta, s_denom;
    __shared__ double s_taus[QR_JBMAX];
    const int G = gridDim.x, cta = blockIdx.x, tid = threadIdx.x, R = a.R, jb = a.jb;
    const int lane = tid & 31, warp = tid >> 5;
    const int64_t rbeg = a.c0 + (int64_t)cta * R;
    const int64_t rows_here = (rbeg < a.m) ? ((a.m - rbeg < R) ? a.m - rbeg : R) : 0;

    slab_load_async(sp, R, a.A + rbeg + a.c0 * a.ld, a.ld, (int)rows_here, R, jb);

    for (int j = 0; j < jb; ++j) {
        const int par = j & 1;
        const int64_t jr = a.c0 + j;
        // partials over my rows r > jr: q[0] = sum x^2, q[c] = sum x * A(r, c) for c > j
        double q[QR_JBMAX + 1];
#pragma unroll
        for (int c = 0; c <= QR_JBMAX; ++c) q[c] = 0.0;
        for (int r = tid; r < rows_here; r += QR_THREADS) {
            if (rbeg + r <= jr) continue;
            double x = sp[j * R + r];
            q[0] = fma(x, x, q[0]);
#pragma unroll
            for (int c = 1; c < QR_JBMAX; ++c)
                if (j + c < jb) q[c] = fma(x, sp[(j + c) * R + r], q[c]);
        }
#pragma unroll
        for (int c = 0; c < QR_JBMAX; ++c) {
            if (c == 0 || j + c < jb) {
                double v = q[c];
                for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
                if (lane == 0) red[warp][c] = v;
            }
        }
        __syncthreads();
        if (tid < jb - j) {  // tid = c index (0 -> s2)
            double v = 0.0;
            for (int w = 0; w < QR_THREADS / 32; ++w) v += red[w][tid];
            a.xbuf[((int64_t)par * G + cta) * QR_XSTRIDE + tid] = v;
        }
        if (jr >= rbeg && jr < rbeg + rows_here && tid < jb - j)  // alpha = A(jr, j), a_c = A(jr, j + c)
            a.rowj[par * QR_JBMAX + tid] = sp[(j + tid) * R + (jr - rbeg)];
        __threadfence();
        grid.sync();
        // every CTA forms the same reflector
        if (tid < jb - j) {
            double v = 0.0;
            for (int g = 0; g < G; ++g) v += __ldcg(a.xbuf + ((int64_t)par * G + g) * QR_XSTRIDE + tid);
            red[0][tid] = v;  // red[0][0] = sum x^2 below, red[0][c] = P_c
            wv[tid] = __ldcg(a.rowj + par * QR_JBMAX + tid);  // wv[0] = alpha, wv[c] = a_c
        }
        __syncthreads();
        if (tid == 0) {
            double alpha = wv[0];
            double nrm = sqrt(fma(alpha, alpha, red[0][0]));
            if (nrm == 0.0) {
                s_tau = 0.0; s_beta = 0.0; s_denom = 1.0;
            } else {
                double beta = (alpha >= 0.0) ? -nrm : nrm;  // convention H
                s_beta = beta;
                s_tau = (beta - alpha) / beta;
                s_denom = alpha - beta;
            }
            s_taus[j] = s_tau;
            if (cta == 0) a.tau[jr] = s_tau;
        }
        __syncthreads();
        const double tau = s_tau, denom = s_denom;
        if (tid > 0 && tid < jb - j) wv[tid] = wv[tid] + red[0][tid] / denom;  // w_c = v^T A(:, c)
        __syncthreads();
        if (tau != 0.0) {
            for (int r = tid; r < rows_here; r += QR_THREADS) {
                int64_t ar = rbeg + r;
                if (ar < jr) continue;
                if (ar == jr) {
                    sp[j * R + r] = s_beta;
                    for (int c = 1; c < jb - j; ++c) sp[(j + c) * R + r] -= tau * wv[c];
                } else {
                    double v = sp[j * R + r] / denom;
                    sp[j * R + r] = v;
                    for (int c = 1; c < jb - j; ++c) sp[(j + c) * R + r] = fma(-tau * wv[c], v, sp[(j + c) * R + r]);
                }
            }
        }
        __syncthreads();
    }

    // explicit V and Gram partials V^T V over my rows
    double* gram = a.xbuf + 2 * (int64_t)G * QR_XSTRIDE;
    for (int idx = tid; idx < R * jb; idx += QR_THREADS) {
        int r = idx % R, c = idx / R;
        if (r >= rows_here) continue;
        int64_t ar = rbeg + r, cr = a.c0 + c;
        double v = (ar == cr) ? 1.0 : (ar > cr ? sp[idx] : 0.0);
        a.V[ar + cr * a.m] = v;
        a.A[ar + cr * a.ld] = sp[idx];
    }
    for (int pq = tid; pq < jb * jb; pq += QR_THREADS) {
        int p = pq % jb, qq = pq / jb;
        double s = 0.0;
        if (p < qq) {
            for (int r = 0; r < rows_here; ++r) {
                int64_t ar = rbeg + r;
                double vp = (ar == a.c0 + p) ? 1.0 : (ar > a.c0 + p ? sp[p * R + r] : 0.0);
                double vq = (ar == a.c0 + qq) ? 1.0 : (ar > a.c0 + qq ? sp[qq * R + r] : 0.0);
                s = fma(vp, vq, s);
            }
        }
        gram[(int64_t)cta * jb * jb + pq] = s;
    }
    __threadfence();
    grid.sync();
    if (cta != 0) return;
    // CTA 0: T = larft(V, tau) from G = V^T V: T_jj = tau_j, T(0:j, j) = -tau_j T(0:j,0:j) G(0:j, j)
    __shared__ double Gm[QR_JBMAX][QR_JBMAX + 1], Ts[QR_JBMAX][QR_JBMAX + 1];
    for (int pq = tid; pq < jb * jb; pq += QR_THREADS) {
        double s = 0.0;
        for (int g = 0; g < G; ++g) s += __ldcg(gram + (int64_t)g * jb * jb + pq);
        Gm[pq % jb][pq / jb] = s;
        Ts[pq % jb][pq / jb] = 0.0;
    }
    __syncthreads();
    for (int j = 0; j < jb; ++j) {
        double tj = s_taus[j];
        if (tid < j) {
            double s = 0.0;
            for (int l = tid; l < j; ++l) s = fma(Ts[tid][l], Gm[l][j], s);
            Ts[tid][j] = -tj * s;
        }
        if (tid == 0) Ts[j][j] = tj;
        __syncthreads();
    }
    for (int pq = tid; pq < jb * jb; pq += QR_THREADS) {
        int p = pq % jb, qq = pq / jb;
        a.T[(a.c0 + p) + (a.c0 + qq) * a.ldt] = Ts[p][qq];
    }
}

// ---------------------------------------------------------------------------------------------
// Cluster variant (the common case, d <= ~3000): the panel rows are split over the CTAs of ONE thread-
// block cluster (<= 8 CTAs) and each column step exchanges only through distributed shared memory with
// one cluster barrier: every CTA reduces its partials (sum x^2 and x^T A(:, c) for the 31 columns to the
// right) with a 31-shuffle butterfly transpose-reduction, publishes them in its own shared memory, and
// after barrier.cluster every CTA sums the CL partial vectors (fixed order) through DSMEM.
constexpr int QC_THREADS = 256;
constexpr int QC_CLMAX = 8;

struct QrClusterArgs {
    double* A;
    int64_t ld;
    int64_t m;
    int64_t c0;
    int jb;
    int R;
    double* tau;
    double* V;
    double* T;
    int64_t ldt;
};

// q[l] summed over the warp ends in lane l (indices 0..31): 16+8+4+2+1 shuffles.
__device__ __forceinline__ double warp_transpose_reduce32(double (&q)[32], int lane)
{
#pragma unroll
    for (int off = 16; off >= 1; off >>= 1) {
        const bool up = (lane & off) != 0;
#pragma unroll
        for (int i = 0; i < off; ++i) {
            double send = up ? q[i] : q[i + off];
            double recv = __shfl_xor_sync(0xffffffffu, send, off);
            q[i] = (up ? q[i + off] : q[i]) + recv;
        }
    }
    return q[0];
}

__global__ void __launch_bounds__(QC_THREADS, 1) qr_panel_cluster_kernel(QrClusterArgs a)
{
    cg::cluster_group cluster = cg::this_cluster();
    const int CL = (int)cluster.num_blocks(), me = (int)cluster.block_rank();
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, R = a.R, jb = a.jb;
    extern __shared__ double dyn[];
    double* sp = dyn;                  // sp[c * R + r]
    double* part = dyn + R * jb;       // [2][32] this CTA's partials
    double* rowjs = part + 64;         // [2][32] alpha, a_c (owner CTA of row jr)
    double* gram = rowjs + 64;         // [32 * 32] Gram partial
    __shared__ double red[QC_THREADS / 32][33];
    __shared__ double coef[32], s_taus[32];
    __shared__ double s_beta, s_denom, s_tau;
    const int64_t rbeg = a.c0 + (int64_t)me * R;
    const int64_t rows_here = (rbeg < a.m) ? ((a.m - rbeg < R) ? a.m - rbeg : R) : 0;

    slab_load_async(sp, R, a.A + rbeg + a.c0 * a.ld, a.ld, (int)rows_here, R, jb);

    // Per column: 2 block barriers + 1 cluster barrier.  Each thread updates and then reads only its own
    // rows, so the update of step j and the partials of step j+1 need no barrier between them.
    for (int j = 0; j < jb; ++j) {
        const int par = j & 1;
        const int64_t jr = a.c0 + j;
        const int owner = (int)((jr - a.c0) / R);
        double q[32];
#pragma unroll
        for (int c = 0; c < 32; ++c) q[c] = 0.0;
        for (int r = tid; r < rows_here; r += QC_THREADS) {
            if (rbeg + r <= jr) continue;
            double x = sp[j * R + r];
            q[0] = fma(x, x, q[0]);
#pragma unroll
            for (int c = 1; c < 32; ++c)
                if (j + c < jb) q[c] = fma(x, sp[(j + c) * R + r], q[c]);
        }
        red[warp][lane] = warp_transpose_reduce32(q, lane);
        __syncthreads();
        if (tid < 32) {
            double v = 0.0;
#pragma unroll
            for (int w = 0; w < QC_THREADS / 32; ++w) v += red[w][tid];
            part[par * 32 + tid] = v;
        } else if (tid < 64 && me == owner && tid - 32 < jb - j) {
            rowjs[par * 32 + (tid - 32)] = sp[(j + tid - 32) * R + (jr - rbeg)];
        }
        cluster.sync();
        if (warp == 0) {
            double pv[QC_CLMAX];
#pragma unroll
            for (int rk = 0; rk < QC_CLMAX; ++rk)  // all DSMEM loads in flight before the (ordered) sum
                pv[rk] = (rk < CL) ? *cluster.map_shared_rank(part + par * 32 + lane, rk) : 0.0;
            const double ww = (lane < jb - j) ? *cluster.map_shared_rank(rowjs + par * 32 + lane, owner) : 0.0;
            double tot = 0.0;
#pragma unroll
            for (int rk = 0; rk < QC_CLMAX; ++rk) tot += pv[rk];
            const double alpha = __shfl_sync(0xffffffffu, ww, 0);
            const double s2 = __shfl_sync(0xffffffffu, tot, 0);
            const double nrm = sqrt(fma(alpha, alpha, s2));
            double beta = 0.0, tau = 0.0, denom = 1.0;
            if (nrm != 0.0) {
                beta = (alpha >= 0.0) ? -nrm : nrm;  // convention H
                tau = (beta - alpha) / beta;
                denom = alpha - beta;
            }
            coef[lane] = (lane > 0 && lane < jb - j) ? tau * (ww + tot / denom) : 0.0;  // tau w_c, w_c = v^T A(:, c)
            if (lane == 0) {
                s_beta = beta;
                s_tau = tau;
                s_denom = denom;
                s_taus[j] = tau;
                if (me == 0) a.tau[jr] = tau;
            }
        }
        __syncthreads();
        const double tau = s_tau, denom = s_denom;
        if (tau != 0.0) {
            const int ncol = jb - j;
            for (int r = tid; r < rows_here; r += QC_THREADS) {
                int64_t ar = rbeg + r;
                if (ar < jr) continue;
                double v;  // A(r, c) -= coef_c * v: v = 1 on the pivot row (v_0 = 1), x_r / denom below
                if (ar == jr) {
                    sp[j * R + r] = s_beta;
                    v = 1.0;
                } else {
                    v = sp[j * R + r] / denom;
                    sp[j * R + r] = v;
                }
                for (int c0 = 1; c0 < ncol; c0 += 8) {  // 8 independent loads in flight, then 8 FMAs
                    double av[8], cf[8];
#pragma unroll
                    for (int u = 0; u < 8; ++u)
                        if (c0 + u < ncol) { av[u] = sp[(j + c0 + u) * R + r]; cf[u] = coef[c0 + u]; }
#pragma unroll
                    for (int u = 0; u < 8; ++u)
                        if (c0 + u < ncol) sp[(j + c0 + u) * R + r] = fma(-cf[u], v, av[u]);
                }
            }
        }
    }
    __syncthreads();
    // explicit V, write-back, Gram partial of V^T V over my rows
    for (int c = 0; c < jb; ++c)
        for (int r = tid; r < rows_here; r += QC_THREADS) {
            int64_t ar = rbeg + r, cr = a.c0 + c;
            double x = sp[c * R + r];
            a.V[ar + cr * a.m] = (ar == cr) ? 1.0 : (ar > cr ? x : 0.0);
            a.A[ar + cr * a.ld] = x;
        }
    for (int pq = tid; pq < jb * jb; pq += QC_THREADS) {
        int p = pq % jb, qq = pq / jb;
        double s = 0.0;
        if (p < qq) {
            for (int r = 0; r < rows_here; ++r) {
                int64_t ar = rbeg + r;
                double vp = (ar == a.c0 + p) ? 1.0 : (ar > a.c0 + p ? sp[p * R + r] : 0.0);
                double vq = (ar == a.c0 + qq) ? 1.0 : (ar > a.c0 + qq ? sp[qq * R + r] : 0.0);
                s = fma(vp, vq, s);
            }
        }
        gram[pq] = s;
    }
    cluster.sync();
    if (me == 0) {
        // T = larft(V, tau): T_jj = tau_j, T(0:j, j) = -tau_j T(0:j, 0:j) G(0:j, j)
        __shared__ double Gm[32][33], Ts[32][33];
        for (int pq = tid; pq < jb * jb; pq += QC_THREADS) {
            double sum = 0.0;
            for (int rk = 0; rk < CL; ++rk) sum += *cluster.map_shared_rank(gram + pq, rk);
            Gm[pq % jb][pq / jb] = sum;
            Ts[pq % jb][pq / jb] = 0.0;
        }
        __syncthreads();
        for (int j = 0; j < jb; ++j) {
            double tj = s_taus[j];
            if (tid < j) {
                double sum = 0.0;
                for (int l = tid; l < j; ++l) sum = fma(Ts[tid][l], Gm[l][j], sum);
                Ts[tid][j] = -tj * sum;
            }
            if (tid == 0) Ts[j][j] = tj;
            __syncthreads();
        }
        for (int pq = tid; pq < jb * jb; pq += QC_THREADS) {
            int p = pq % jb, qq = pq / jb;
            a.T[(a.c0 + p) + (a.c0 + qq) * a.ldt] = Ts[p][qq];
        }
    }
    cluster.sync();  // keep every CTA's shared memory alive until CTA 0 has read it
}

// ---------------------------------------------------------------------------------------------
// Register-resident cluster leaf (rows <= 16 x 256): one panel row per thread in registers, push-style DSMEM
// exchange (see qr_leaf_fast_kernel below).
constexpr int QL_THREADS = 256, QL_WARPS = QL_THREADS / 32, QL_CLMAX = 16;
constexpr int QT_LD = 34;  // row stride of the per-warp product tile (doubles): 16-byte aligned, conflict-free reads
constexpr size_t QL_DYN_SMEM = sizeof(double) * QL_WARPS * 32 * QT_LD;

struct QrLeafArgs {
    double* A;
    int64_t ld;
    int64_t m;
    int64_t c0;
    int jb;
    double* tau;
    double* V;
    double* T;
    int64_t ldt;
};

// Register-resident cluster leaf, one panel row per thread.  The register window ROTATES:
// at the start of step j av[m] holds column (j + m) mod 32 of the thread's row — columns < j already final
// (reflector entries below the diagonal, R entries on and above it) — so every register index is
// compile-time in a rolled loop: column j is av[0], the step's new value of column j re-enters at av[31],
// and after 32 steps av[m] = column m again.  (Select trees over a fixed window, or a fully unrolled loop,
// measured slower: the latter overflows the 32 KB instruction cache.)  A ragged leaf (jb < 32) runs the
// padding columns as zero columns (tau = 0, no effect) and writes back only jb.
// Per column: each thread forms q[m] = x_r av[m] (x_r = column j below the diagonal), the 31-shuffle
// transpose-reduction leaves the warp sum for window slot m in lane m, the 8 warp sums are combined in shared
// memory (one block barrier) and warp 0 pushes the CTA's 32 sums — and, on CTA 0 (which owns the leaf's pivot
// rows), the pivot row's window — into every CTA's slot with st.async (mbarrier tx-count, double-buffered by
// parity).  After the wait every warp sums the CL CTA slots (fixed order); lane 0 gives alpha and ||x||^2 ->
// beta, tau, denom (convention H, Z9/Z20); lane m < 32 - j is column j + m (the update coefficient tau w_c for
// m >= 1), lane m >= 32 - j is the earlier column c = m + j - 32 (V(:, c)^T v_j, the larft column).
__global__ void __launch_bounds__(QL_THREADS, 1) qr_leaf_fast_kernel(QrLeafArgs a)
{
    constexpr int JB = 32;
    QLEAF_TS(63, 0);
    cg::cluster_group cluster = cg::this_cluster();
    const int CL = (int)cluster.num_blocks(), me = (int)cluster.block_rank();
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, jb = a.jb;
    extern __shared__ __align__(16) double qtile[];  // [QL_WARPS][32][QT_LD] per-warp product tiles
    __shared__ double wsum[2][QL_WARPS][32];
    __shared__ __align__(16) double slot[2][QL_CLMAX][32];
    __shared__ __align__(16) double prow[2][32];
    __shared__ __align__(16) double rowstage[2][32];
    __shared__ __align__(16) double cw[QL_WARPS][32];
    __shared__ double TcS[32][33];  // TcS[j][l] = V(:, l)^T v_j (CTA 0)
    __shared__ double taus[32];
    __shared__ __align__(8) unsigned long long mbar[2];
    if (tid == 0) {
        mbar_init(smem_u32(&mbar[0]), 1);
        mbar_init(smem_u32(&mbar[1]), 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    const int64_t r = a.c0 + (int64_t)me * QL_THREADS + tid;  // this thread's row
    const bool has = r < a.m;
    double av[JB];
#pragma unroll
    for (int c = 0; c < JB; ++c) av[c] = (has && c < jb) ? a.A[r + (a.c0 + c) * a.ld] : 0.0;
    cluster.sync();  // every peer's mbarriers are initialised before the first push
    QLEAF_TS(63, 1);

#pragma unroll 1
    for (int j = 0; j < JB; ++j) {
        const int par = j & 1;
        const int64_t jr = a.c0 + j;
        QLEAF_TS(j, 0);
        const double x = (has && r > jr) ? av[0] : 0.0;
        // warp sums of q[m] = x av[m] (q[0] = x^2): each lane writes its 32 products as a row of the warp's
        // shared-memory tile, lane m sums column m (4 accumulators) — ~85 instructions instead of the 217 of a
        // shuffle transpose-reduction
        {
            double* tile = qtile + warp * (32 * QT_LD);
#pragma unroll
            for (int m = 0; m < 32; m += 2)
                *reinterpret_cast<double2*>(&tile[lane * QT_LD + m]) = make_double2(x * av[m], x * av[m + 1]);
            __syncwarp();
            double s4[4] = {0.0, 0.0, 0.0, 0.0};
#pragma unroll
            for (int rr = 0; rr < 32; ++rr) s4[rr & 3] += tile[rr * QT_LD + lane];
            wsum[par][warp][lane] = (s4[0] + s4[1]) + (s4[2] + s4[3]);
            __syncwarp();  // the tile is rewritten by the next column
        }
        if (me == 0 && tid == j) {  // the pivot row jr (thread j of CTA 0): its window, for warp 0's push
#pragma unroll
            for (int m = 0; m < JB; m += 2)
                *reinterpret_cast<double2*>(&rowstage[par][m]) = make_double2(av[m], av[m + 1]);
        }
        QLEAF_TS(j, 1);
        __syncthreads();
        QLEAF_TS(j, 2);
        const unsigned mb = smem_u32(&mbar[par]);
        if (warp == 0) {
            double t = 0.0;
#pragma unroll
            for (int w = 0; w < QL_WARPS; ++w) t += wsum[par][w][lane];
            // 16-byte pushes, two ranks per instruction: lane l sends the pair (2p, 2p + 1), p = l & 15, to rank
            // 2 it + (l >> 4) — half the st.async instructions of one 8-byte value per lane and rank
            const int pi = lane & 15, half = lane >> 4;
            const double t0 = __shfl_sync(0xffffffffu, t, 2 * pi), t1 = __shfl_sync(0xffffffffu, t, 2 * pi + 1);
            const unsigned my = smem_u32(&slot[par][me][2 * pi]);
            for (int rk = half; rk < CL; rk += 2)
                asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.v2.f64 [%0], {%1, %2}, [%3];" ::"r"(
                                 mapa_u32(my, rk)),
                             "d"(t0), "d"(t1), "r"(mapa_u32(mb, rk))
                             : "memory");
            if (me == 0) {
                const double pv = rowstage[par][lane];
                const double p0 = __shfl_sync(0xffffffffu, pv, 2 * pi), p1 = __shfl_sync(0xffffffffu, pv, 2 * pi + 1);
                const unsigned pr = smem_u32(&prow[par][2 * pi]);
                for (int rk = half; rk < CL; rk += 2)
                    asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.v2.f64 [%0], {%1, %2}, [%3];" ::"r"(
                                     mapa_u32(pr, rk)),
                                 "d"(p0), "d"(p1), "r"(mapa_u32(mb, rk))
                                 : "memory");
            }
        }
        QLEAF_TS(j, 3);
        if (tid == 0) mbar_arrive_expect_tx(mb, (unsigned)((CL * 32 + 32) * sizeof(double)));
        mbar_wait_parity(mb, (unsigned)((j >> 1) & 1));
        QLEAF_TS(j, 4);
        double tot = 0.0;
        for (int rk = 0; rk < CL; ++rk) tot += slot[par][rk][lane];
        const double ww = prow[par][lane];
        const double alpha = __shfl_sync(0xffffffffu, ww, 0);
        const double s2 = __shfl_sync(0xffffffffu, tot, 0);
        const double nrm = sqrt(fma(alpha, alpha, s2));
        double beta = 0.0, tau = 0.0, denom = 1.0;
        if (nrm != 0.0) {
            beta = (alpha >= 0.0) ? -nrm : nrm;  // convention H
            tau = (beta - alpha) / beta;
            denom = alpha - beta;
        }
        const double rden = 1.0 / denom;      // one division per column; products below (<= 1 ulp from dividing)
        const double vdot = ww + tot * rden;  // slot m: column j + m (m < 32 - j) or c = m + j - 32 (m >= 32 - j)
        QLEAF_TS(j, 5);
        cw[warp][lane] = (lane >= 1 && lane < JB - j) ? tau * vdot : 0.0;
        if (me == 0 && warp == 0) {
            if (lane >= JB - j) TcS[j][lane + j - JB] = vdot;
            if (lane == 0) {
                taus[j] = tau;
                if (j < jb) a.tau[jr] = tau;
            }
        }
        __syncwarp();
        // column j's new value, the update of the later columns, and the rotation, in one pass
        double v = 0.0, newj = av[0];
        if (has && r >= jr) {
            if (r == jr) {
                newj = beta;
                v = 1.0;
            } else {
                v = av[0] * rden;
                newj = v;
            }
        }
#pragma unroll
        for (int m = 0; m + 1 < JB; m += 2) {
            const double2 cf = *reinterpret_cast<const double2*>(&cw[warp][m]);
            if (m > 0) av[m - 1] = fma(-cf.x, v, av[m]);
            av[m] = fma(-cf.y, v, av[m + 1]);
        }
        av[JB - 1] = newj;
        QLEAF_TS(j, 6);
        __syncwarp();  // cw is rewritten by the next column
    }
    QLEAF_TS(63, 2);
    // write back: R / reflectors in A, explicit V (av[m] = column m again)
    if (has) {
#pragma unroll
        for (int c = 0; c < JB; ++c) {
            if (c < jb) {
                const int64_t cr = a.c0 + c;
                a.A[r + cr * a.ld] = av[c];
                a.V[r + cr * a.m] = (r == cr) ? 1.0 : (r > cr ? av[c] : 0.0);
            }
        }
    }
    // every push into this CTA has landed (the last wait); arrive now so that no CTA waits for CTA 0's larft
    cluster_arrive();
    QLEAF_TS(63, 3);
    // T (larft): T_jj = tau_j, T(0:j, j) = -tau_j T(0:j, 0:j) (V(:, 0:j)^T v_j).  Lane i keeps row i of T in
    // registers (T(i, l) = 0 for l < i), both loops unrolled so every index is compile-time: column j costs j
    // register FMAs per lane (the same ascending order as the scalar recurrence: the zero terms are exact)
    // instead of a serial shared-memory dot product per lane (26k -> 8.4k cycles per leaf, tools/leaf_timing.py).
    if (me == 0 && warp == 0) {
        double trow[JB];
#pragma unroll
        for (int l = 0; l < JB; ++l) trow[l] = 0.0;
#pragma unroll
        for (int j = 0; j < JB; ++j) {
            if (j < jb) {
                double t = 0.0;
#pragma unroll
                for (int l = 0; l < j; ++l) t = fma(trow[l], TcS[j][l], t);
                trow[j] = lane < j ? -taus[j] * t : (lane == j ? taus[j] : 0.0);
            }
        }
        if (lane < jb) {
#pragma unroll
            for (int j = 0; j < JB; ++j)
                if (j < jb) a.T[(a.c0 + lane) + (a.c0 + j) * a.ldt] = trow[j];
        }
    }
    QLEAF_TS(63, 4);
    cluster_wait();  // no CTA exits while its own pushes to peers may be in flight
}

static bool qr_leaf_reg(Ctx& cx, double* A, int64_t ld, int64_t m, int64_t c0, int jb, double* tau, double* V,
                        double* T, int64_t ldt)
{
    const int64_t rows = m - c0;
    // at least 2 CTAs: the DSMEM pushes (mapa + st.async) need a real cluster (compute-sanitizer memcheck flags
    // them in a 1-CTA cluster); a CTA without rows pushes exact zeros, which leave the fixed-order sums unchanged
    const int CL = (int)imax(2, cdiv(rows, QL_THREADS));
    if (CL > QL_CLMAX || jb > 32) return false;
    static AttrOnce attr_cl, attr_smem;
    ensure_attr(attr_cl, qr_leaf_fast_kernel, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    ensure_attr(attr_smem, qr_leaf_fast_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)QL_DYN_SMEM);
    QrLeafArgs args{A, ld, m, c0, jb, tau, V, T, ldt};
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(CL);
    cfg.blockDim = dim3(QL_THREADS);
    cfg.dynamicSmemBytes = QL_DYN_SMEM;
    cfg.stream = cx.stream;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = CL;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    BQ_CUDA(cudaLaunchKernelEx(&cfg, qr_leaf_fast_kernel, args));
    ++g_launches;
    return true;
}

static bool qr_panel_cluster(Ctx& cx, double* A, int64_t ld, int64_t m, int64_t c0, int jb, double* tau, double* V,
                             double* T, int64_t ldt)
{
    int64_t rows = m - c0;
    int CL = (int)imin(QC_CLMAX, imax(1, cdiv(rows, 256)));
    int R = (int)cdiv(rows, CL);
    size_t smem = ((size_t)R * jb + 64 + 64 + 32 * 32) * sizeof(double);
    if (smem > 200 * 1024) return false;
    static AttrOnce attr;
    ensure_attr(attr, qr_panel_cluster_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    QrClusterArgs args{A, ld, m, c0, jb, R, tau, V, T, ldt};
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(CL);
    cfg.blockDim = dim3(QC_THREADS);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = cx.stream;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = CL;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    BQ_CUDA(cudaLaunchKernelEx(&cfg, qr_panel_cluster_kernel, args));
    ++g_launches;
    return true;
}

static void qr_panel(Ctx& cx, double* A, int64_t ld, int64_t m, int64_t c0, int jb, double* tau, double* V, double* T,
                     int64_t ldt, double* xbuf, double* rowj)
{
    if (qr_leaf_reg(cx, A, ld, m, c0, jb, tau, V, T, ldt)) return;
    if (qr_panel_cluster(cx, A, ld, m, c0, jb, tau, V, T, ldt)) return;
    int64_t rows = m - c0;
    int G = (int)imin(cx.num_sms, imax(1, cdiv(rows, 64)));
    int R = (int)cdiv(rows, G);
    size_t smem = (size_t)R * jb * sizeof(double);
    if (smem > QR_GRID_SMEM)
        throw std::runtime_error("qr_panel: panel taller than qr_max_rows (" + std::to_string(rows) + " rows)");
    static AttrOnce attr;
    ensure_attr(attr, qr_panel_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)QR_GRID_SMEM);
    QrPanelArgs a{A, ld, m, c0, jb, R, tau, V, T, ldt, xbuf, rowj};
    void* args[] = {&a};
    BQ_CUDA(cudaLaunchCooperativeKernel((void*)qr_panel_kernel, dim3(G), dim3(QR_THREADS), args, smem, cx.stream));
    ++g_launches;
}

// Recursive QR of columns [c0, c1) of Wq (rows [c0, m)); V (m x p explicit), Tf (p x p).
// Recursive Householder QR of columns [c0, c1) of A (rows [c0, m), leading dimension lda); V (m x p
// explicit, ld m, pre-zeroed), Tf (p x p, ld p).
// Leaf width: 32 columns unless the panel is so tall that the cooperative grid leaf's slab (cdiv(rows,
// num_sms) x leaf doubles per CTA) would not fit shared memory; then narrower, down to one column
// (num_sms x 25600 rows; taller inputs are rejected up front, qr_max_rows).
static int qr_leaf_width(int64_t rows, int num_sms)
{
    const int64_t Rg = cdiv(rows, num_sms);
    for (int leaf = QR_JBMAX; leaf > 1; leaf /= 2)
        if ((size_t)Rg * leaf * 8 <= QR_GRID_SMEM) return leaf;
    return 1;
}

int64_t qr_max_rows(int num_sms) { return (int64_t)num_sms * (int64_t)(QR_GRID_SMEM / 8); }

static void geqrf_rec(Ctx& cx, double* A, int64_t lda, int64_t m, int64_t c0, int64_t c1, double* tau, double* V,
                      double* Tf, int64_t p, double* W1, double* W2, double* xbuf, double* rowj, int leaf)
{
    int64_t nc = c1 - c0;
    if (nc <= leaf) {
        qr_panel(cx, A, lda, m, c0, (int)nc, tau, V, Tf, p, xbuf, rowj);
        return;
    }
    int64_t mid = c0 + cdiv(nc / 2, leaf) * leaf;
    geqrf_rec(cx, A, lda, m, c0, mid, tau, V, Tf, p, W1, W2, xbuf, rowj, leaf);
    int64_t k1 = mid - c0, ncr = c1 - mid, h = m - c0;
    const double* V1 = V + c0 + c0 * m;    // h x k1
    const double* T11 = Tf + c0 + c0 * p;  // k1 x k1
    double* A2 = A + c0 + mid * lda;       // h x ncr
    // A2 <- (I - V1 T11 V1^T)^T A2 = A2 - V1 T11^T (V1^T A2)
    gemm(cx, true, false, k1, ncr, h, 1.0, V1, m, A2, lda, 0.0, W1, k1);
    gemm(cx, true, false, k1, ncr, k1, 1.0, T11, p, W1, k1, 0.0, W2, k1);
    gemm(cx, false, false, h, ncr, k1, -1.0, V1, m, W2, k1, 1.0, A2, lda);
    geqrf_rec(cx, A, lda, m, mid, c1, tau, V, Tf, p, W1, W2, xbuf, rowj, leaf);
    // T12 = -T11 (V1^T V2) T22, V2 = V(c0:m, mid:c1) (zeros above row mid)
    const double* V2 = V + c0 + mid * m;
    gemm(cx, true, false, k1, ncr, h, 1.0, V1, m, V2, m, 0.0, W1, k1);
    gemm(cx, false, false, k1, ncr, k1, 1.0, T11, p, W1, k1, 0.0, W2, k1);
    gemm(cx, false, false, k1, ncr, ncr, -1.0, W2, k1, Tf + mid + mid * p, p, 0.0, Tf + c0 + mid * p, p);
}

void householder_panel(Ctx& cx, double* A, int64_t lda, int64_t rows, int64_t cols, double* tau, double* V, double* T)
{
    if (rows <= 0 || cols <= 0) return;
    size_t mark = cx.ws_used;
    double* W1 = cx.alloc((size_t)cols * cols);
    double* W2 = cx.alloc((size_t)cols * cols);
    int G = cx.num_sms;
    double* xbuf = cx.alloc(2 * (size_t)G * QR_XSTRIDE + (size_t)G * QR_JBMAX * QR_JBMAX);
    double* rowj = cx.alloc(2 * QR_JBMAX);
    BQ_CUDA(cudaMemsetAsync(V, 0, sizeof(double) * rows * cols, cx.stream));
    BQ_CUDA(cudaMemsetAsync(T, 0, sizeof(double) * cols * cols, cx.stream));
    geqrf_rec(cx, A, lda, rows, 0, cols, tau, V, T, cols, W1, W2, xbuf, rowj, qr_leaf_width(rows, cx.num_sms));
    cx.ws_used = mark;
}

__global__ void store_rsk_kernel(int64_t p, int64_t d, const double* Wq, double* MskT, int64_t ldm)
{
    // MskT(q, row) = R_sk(row, q) = Wq(row, q) for row <= q, 0 otherwise (q < p, row < d)
    int64_t total = p * d;
    for (int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; idx < total; idx += (int64_t)gridDim.x * blockDim.x) {
        int64_t q = idx % p, row = idx / p;
        MskT[q + row * ldm] = (row <= q) ? Wq[row + q * d] : 0.0;
    }
}

// R_sk of the d x w sketch window MskT(0:w, 0:d)^T (MskT points at row s, ld ldm); in place.
void sketch_qr(Ctx& cx, double* MskT, int64_t ldm, int64_t w, int64_t d, const RowBlocks& rows,
               const RskDefer* defer)
{
    int64_t p = imin(d, w);
    if (p <= 0) return;
    size_t mark = cx.ws_used;
    double* Wq = cx.alloc((size_t)d * p);
    double* V = cx.alloc((size_t)d * p);
    double* Tf = cx.alloc((size_t)p * p);
    double* tau = cx.alloc((size_t)p);
    double* W1 = cx.alloc((size_t)p * p);
    double* W2 = cx.alloc((size_t)p * p);
    int G = cx.num_sms;
    double* xbuf = cx.alloc(2 * (size_t)G * QR_XSTRIDE + (size_t)G * QR_JBMAX * QR_JBMAX);
    double* rowj = cx.alloc(2 * QR_JBMAX);
    // Wq = Wsk(:, 0:p) = MskT(0:p, 0:d)^T
    transpose_copy(cx, p, d, MskT, ldm, Wq, d);
    BQ_CUDA(cudaMemsetAsync(V, 0, sizeof(double) * d * p, cx.stream));
    BQ_CUDA(cudaMemsetAsync(Tf, 0, sizeof(double) * p * p, cx.stream));
    geqrf_rec(cx, Wq, d, d, 0, p, tau, V, Tf, p, W1, W2, xbuf, rowj, qr_leaf_width(d, cx.num_sms));
    int64_t rest = w - p;
    if (rest > 0) {
        // p == d here.  Q_sk = H_1...H_p = I - V T V^T formed explicitly (d x d), then
        // R_sk(:, p:w)^T = Wsk(:, p:w)^T Q_sk in one GEMM (2 rest d^2 flops instead of 6 rest d p).
        double* Xt = MskT + p;  // rest x d
        const bool deferred = defer && defer->side && rows.n < 0;
        double* Q = deferred ? defer->Q : cx.alloc((size_t)d * d);
        double* Wt = cx.alloc((size_t)p * d);
        double* Y = deferred ? defer->Y : cx.alloc((size_t)rest * d);
        gemm(cx, false, true, p, d, p, 1.0, Tf, p, V, d, 0.0, Wt, p);  // Wt = T V^T
        BQ_CUDA(cudaMemsetAsync(Q, 0, sizeof(double) * d * d, cx.stream));
        zero_triangle(cx, 'L', d, d, Q, d, /*unit_diag=*/true);
        gemm(cx, false, false, d, d, p, -1.0, V, d, Wt, p, 1.0, Q, d);  // Q = I - V Wt
        if (deferred) {
            // on the second stream: after what is queued there (the previous bulk update), overlapping the
            // critical chain's permutation and latency-bound panel
            cudaEvent_t e;
            BQ_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
            BQ_CUDA(cudaEventRecord(e, cx.stream));
            BQ_CUDA(cudaStreamWaitEvent(defer->side->stream, e, 0));
            BQ_CUDA(cudaEventDestroy(e));
            Ctx sc = side_ctx(cx, *defer->side, 0);  // allocates nothing
            gemm(sc, false, false, rest, d, d, 1.0, Xt, ldm, Q, d, 0.0, Y, rest);
            copy_matrix(sc, rest, d, Y, rest, Xt, ldm);
        } else if (rows.n < 0) {
            gemm(cx, false, false, rest, d, d, 1.0, Xt, ldm, Q, d, 0.0, Y, rest, false, 0, /*no_split=*/true);
            copy_matrix(cx, rest, d, Y, rest, Xt, ldm);
        } else {
            for (int64_t j = 0; j < rows.n; ++j) {
                const int64_t o = rows.off[j], l = imin(rows.len[j], rest - o);
                if (o < 0 || l <= 0) continue;
                gemm(cx, false, false, l, d, d, 1.0, Xt + o, ldm, Q, d, 0.0, Y, l, false, 0, /*no_split=*/true);
                copy_matrix(cx, l, d, Y, l, Xt + o, ldm);
            }
        }
    }
    store_rsk_kernel<<<(unsigned)imin(cdiv(p * d, 256), 4 * cx.num_sms), 256, 0, cx.stream>>>(p, d, Wq, MskT, ldm);
    BQ_LAUNCH_CHECK();
    cx.ws_used = mark;
}

// ---- the K-SQR pipeline (left-looking, overlapping K-LU; bqrrp_internal.cuh SketchQrPipe)

// Wq(i, c0 + c) = MskT(perm[c0 + c], i) for i < d, c < jb (Wq: d x p, ld d): the sketch columns of pivots c0 ..
// c0 + jb - 1, read from the not yet permuted transposed sketch (row q of the permuted window = row perm[q]).
// A 32 x 32 tile per CTA through shared memory: scattered 8-byte reads along the pivot axis, coalesced writes.
__global__ void gather_sketch_block_kernel(int64_t d, int jb, const double* __restrict__ MskT, int64_t ldm,
                                           const int* __restrict__ perm, int64_t c0, double* __restrict__ Wq)
{
    __shared__ double t[32][33];
    __shared__ int src[32];
    const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;  // 32 x 8
    if (threadIdx.x < 32) src[threadIdx.x] = threadIdx.x < jb ? perm[c0 + threadIdx.x] : 0;
    __syncthreads();
    for (int64_t i0 = (int64_t)blockIdx.x * 32; i0 < d; i0 += (int64_t)gridDim.x * 32) {
        for (int c = ty; c < 32; c += 8) {  // lane tx: column i0 + tx of the sketch row src[c]
            const int64_t i = i0 + tx;
            t[c][tx] = (c < jb && i < d) ? MskT[src[c] + i * ldm] : 0.0;
        }
        __syncthreads();
        for (int c = ty; c < jb; c += 8) {  // lane tx: row i0 + tx of Wq column c0 + c
            const int64_t i = i0 + tx;
            if (i < d) Wq[i + (c0 + c) * d] = t[c][tx];
        }
        __syncthreads();
    }
}

void sketch_qr_pipe_begin(SketchQrPipe& P, Ctx& cx, Ctx& q, std::vector<cudaEvent_t>& events, double* MskT,
                          int64_t ldm, int64_t w, int64_t d, Ctx* q2)
{
    P.cx = &cx;
    P.q = &q;
    P.q2 = q2;
    P.ev_t = nullptr;
    P.events = &events;
    P.nev = 0;
    P.MskT = MskT;
    P.ldm = ldm;
    P.w = w;
    P.d = d;
    P.p = imin(d, w);
    P.gathered = P.queued = 0;
    P.mark = cx.ws_used;
    if (P.p <= 0) return;
    P.Wq = cx.alloc((size_t)d * P.p);
    P.V = cx.alloc((size_t)d * P.p);
    P.Tf = cx.alloc((size_t)P.p * P.p);
    P.tau = cx.alloc((size_t)P.p);
    P.W1 = cx.alloc((size_t)d * QR_JBMAX);
    P.W2 = cx.alloc((size_t)d * QR_JBMAX);
    P.xbuf = cx.alloc(2 * (size_t)cx.num_sms * QR_XSTRIDE + (size_t)cx.num_sms * QR_JBMAX * QR_JBMAX);
    P.rowj = cx.alloc(2 * QR_JBMAX);
    // split-K slices of q's skinny long-K GEMMs (V^T B: c x 32 over K = d), when they fit the temporaries' budget
    for (Ctx* c : {&q, q2}) {
        if (!c) continue;
        if (d >= 512) {
            c->splitk_elems = (size_t)16 * QR_JBMAX * d;
            c->splitk = cx.alloc(c->splitk_elems);
        } else {
            c->splitk = nullptr;
            c->splitk_elems = 0;
        }
    }
    if (q2) {
        P.W3 = cx.alloc((size_t)d * QR_JBMAX);
        P.W4 = cx.alloc((size_t)d * QR_JBMAX);
    }
    BQ_CUDA(cudaMemsetAsync(P.V, 0, sizeof(double) * d * P.p, cx.stream));
    BQ_CUDA(cudaMemsetAsync(P.Tf, 0, sizeof(double) * P.p * P.p, cx.stream));
}

static cudaEvent_t pipe_event(SketchQrPipe& P)
{
    if (P.nev == P.events->size()) {
        cudaEvent_t e;
        BQ_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
        P.events->push_back(e);
    }
    return (*P.events)[P.nev++];
}

// Block [c, c + jb) of the sketch QR on q: B = Wq(:, c:c+jb) <- Q_c^T B (Q_c = I - V_c T_c V_c^T, the c reflectors
// so far), the leaf on B(c:d, :), then T(0:c, c:c+jb) = -T_c (V_c^T V_b) T_bb (the recursive form's T12 merge).
static void pipe_block(SketchQrPipe& P, int64_t c, int jb)
{
    Ctx& q = *P.q;
    const int64_t d = P.d, p = P.p;
    double* B = P.Wq + c * d;
    if (c > 0) {
        gemm(q, true, false, c, jb, d, 1.0, P.V, d, B, d, 0.0, P.W1, c);          // W1 = V_c^T B
        if (P.ev_t) BQ_CUDA(cudaStreamWaitEvent(q.stream, P.ev_t, 0));             // T_c complete (q2)
        gemm(q, true, false, c, jb, c, 1.0, P.Tf, p, P.W1, c, 0.0, P.W2, c);      // W2 = T_c^T W1
        gemm(q, false, false, d, jb, c, -1.0, P.V, d, P.W2, c, 1.0, B, d);        // B -= V_c W2
    }
    qr_panel(q, P.Wq, d, d, c, jb, P.tau, P.V, P.Tf, p, P.xbuf, P.rowj);
    if (c > 0) {
        // T merge; on q2 it overlaps the next block's W1 = V^T B (which needs V, not T)
        Ctx* m = &q;
        double *M1 = P.W1, *M2 = P.W2;
        if (P.q2) {
            cudaEvent_t e = pipe_event(P);
            BQ_CUDA(cudaEventRecord(e, q.stream));
            BQ_CUDA(cudaStreamWaitEvent(P.q2->stream, e, 0));
            m = P.q2;
            M1 = P.W3;
            M2 = P.W4;
        }
        gemm(*m, true, false, c, jb, d, 1.0, P.V, d, P.V + c * d, d, 0.0, M1, c);  // V_c^T V_b
        gemm(*m, false, false, c, jb, c, 1.0, P.Tf, p, M1, c, 0.0, M2, c);          // T_c (V_c^T V_b)
        gemm(*m, false, false, c, jb, jb, -1.0, M2, c, P.Tf + c + c * p, p, 0.0, P.Tf + c * p, p);
        if (P.q2) {
            P.ev_t = pipe_event(P);
            BQ_CUDA(cudaEventRecord(P.ev_t, P.q2->stream));
        }
    }
}

void sketch_qr_pipe_columns(SketchQrPipe& P, const int* perm, int64_t c1)
{
    c1 = imin(c1, P.p);
    if (c1 > P.gathered) {
        const int64_t c0 = P.gathered;
        for (int64_t g = c0; g < c1; g += 32) {
            const int jb = (int)imin(32, c1 - g);
            gather_sketch_block_kernel<<<(unsigned)imin(cdiv(P.d, 32), 2 * P.cx->num_sms), 256, 0, P.cx->stream>>>(
                P.d, jb, P.MskT, P.ldm, perm, g, P.Wq);
            BQ_LAUNCH_CHECK();
        }
        P.gathered = c1;
    }
    while (P.queued < P.gathered && (P.gathered - P.queued >= QR_JBMAX || P.gathered == P.p)) {
        const int jb = (int)imin(QR_JBMAX, P.gathered - P.queued);
        cudaEvent_t e = pipe_event(P);
        BQ_CUDA(cudaEventRecord(e, P.cx->stream));
        BQ_CUDA(cudaStreamWaitEvent(P.q->stream, e, 0));
        pipe_block(P, P.queued, jb);
        P.queued += jb;
    }
}

void sketch_qr_pipe_finish(SketchQrPipe& P, const RskDefer* defer)
{
    Ctx& cx = *P.cx;
    const int64_t d = P.d, p = P.p, w = P.w, ldm = P.ldm;
    if (p <= 0) {
        cx.ws_used = P.mark;
        return;
    }
    if (P.queued < p) throw std::runtime_error("sketch_qr_pipe: K-LU did not finish the pivots");
    for (Ctx* c : {P.q, P.q2}) {
        if (!c) continue;
        cudaEvent_t e = pipe_event(P);
        BQ_CUDA(cudaEventRecord(e, c->stream));
        BQ_CUDA(cudaStreamWaitEvent(cx.stream, e, 0));
        c->splitk = nullptr;
        c->splitk_elems = 0;
    }
    double* MskT = P.MskT;
    double* Wq = P.Wq;
    int64_t rest = w - p;
    if (rest > 0) {
        // as sketch_qr: Q_sk = I - V T V^T (d x d) explicit, then R_sk(:, p:w)^T = Wsk(:, p:w)^T Q_sk in one GEMM
        double* Xt = MskT + p;
        const bool deferred = defer && defer->side;
        double* Q = deferred ? defer->Q : cx.alloc((size_t)d * d);
        double* Wt = cx.alloc((size_t)p * d);
        double* Y = deferred ? defer->Y : cx.alloc((size_t)rest * d);
        gemm(cx, false, true, p, d, p, 1.0, P.Tf, p, P.V, d, 0.0, Wt, p);
        BQ_CUDA(cudaMemsetAsync(Q, 0, sizeof(double) * d * d, cx.stream));
        zero_triangle(cx, 'L', d, d, Q, d, /*unit_diag=*/true);
        gemm(cx, false, false, d, d, p, -1.0, P.V, d, Wt, p, 1.0, Q, d);
        if (deferred) {
            cudaEvent_t e2 = pipe_event(P);
            BQ_CUDA(cudaEventRecord(e2, cx.stream));
            BQ_CUDA(cudaStreamWaitEvent(defer->side->stream, e2, 0));
            Ctx sc = side_ctx(cx, *defer->side, 0);
            gemm(sc, false, false, rest, d, d, 1.0, Xt, ldm, Q, d, 0.0, Y, rest);
            copy_matrix(sc, rest, d, Y, rest, Xt, ldm);
        } else {
            gemm(cx, false, false, rest, d, d, 1.0, Xt, ldm, Q, d, 0.0, Y, rest, false, 0, /*no_split=*/true);
            copy_matrix(cx, rest, d, Y, rest, Xt, ldm);
        }
    }
    store_rsk_kernel<<<(unsigned)imin(cdiv(p * d, 256), 4 * cx.num_sms), 256, 0, cx.stream>>>(p, d, Wq, MskT, ldm);
    BQ_LAUNCH_CHECK();
    cx.ws_used = P.mark;
}

}  // namespace bqrrp

#ifdef BQRRP_LEAF_TIMING
extern "C" int bqrrp_debug_qleaf_timing(long long* out)
{
    return cudaMemcpyFromSymbol(out, bqrrp::g_qleaf_ts, sizeof(long long) * 2 * 64 * 8) == cudaSuccess ? 0 : -1;
}
#endif
