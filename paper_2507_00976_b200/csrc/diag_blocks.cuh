// diag_blocks.cuh — the 64 x 64 diagonal-block factorizations (register-resident, one CTA of 256 threads)
// of the blocked POTRF and sign-LU (blas.cu), as device functions so a fused kernel can reuse them (a
// persistent one-kernel k x k POTRF / LU built on them measured no faster than the blocked launch sequence
// at k = 2048: 1.80 vs 1.73 ms, 3.82 vs 3.77 ms; the serial diagonal blocks dominate both).
#pragma once
#include "blas.cuh"

namespace bqrrp {

// One CTA factors a <= 64 x 64 diagonal block with the block in REGISTERS: thread (i = tid % 64,
// g = tid / 64) owns row i, columns c = g + 4q (q < 16).  Step j (right-looking, column left unscaled):
// the owners of column j publish it to shared memory (double-buffered), ONE barrier, then every thread
// updates A(i, c) -= A(i, j) A(c, j) / A(j, j) for its c > j, c <= i.  Columns are scaled by
// 1/sqrt(A(j, j)) at the end.  (A shared-memory version with one (i, c) pair per loop trip ran
// ~1 us per column; this one is a handful of FMAs + 17 shared reads per column.)
// Called by all 256 threads of one CTA.
__device__ __forceinline__ void potrf_diag_block(int n, double* G, int64_t ldg, int j0, int* info, double (*colj)[FACT_NB],
                                 double* piv)
{
    const int tid = threadIdx.x, i = tid & 63, g = tid >> 6;
    constexpr int Q = FACT_NB / 4;
    double a[Q];
#pragma unroll
    for (int q = 0; q < Q; ++q) {
        const int c = g + 4 * q;
        a[q] = (i < n && c < n && c <= i) ? G[i + (int64_t)c * ldg] : 0.0;
    }
    if (*(volatile int*)info != 0) return;  // an earlier block already broke down (uniform)
    int bad = -1;
    // j = 4 jq + jr with jq unrolled, so the owned column a[jq] is a compile-time register index
#pragma unroll
    for (int jq = 0; jq < Q; ++jq) {
        for (int jr = 0; jr < 4; ++jr) {
            const int j = 4 * jq + jr;
            if (j >= n || bad >= 0) break;
            const int par = j & 1;
            if (g == jr) colj[par][i] = a[jq];
            __syncthreads();
            const double d = colj[par][j];
            if (!(d > 0.0)) {  // uniform: every thread sees the same pivot
                bad = j;
                break;
            }
            if (tid == 0) piv[j] = d;
            const double lij = colj[par][i] * (1.0 / d);
            if (i > j) {
#pragma unroll
                for (int q = jq; q < Q; ++q) {
                    const int c = g + 4 * q;
                    if (c > j && c <= i) a[q] = fma(-lij, colj[par][c], a[q]);
                }
            }
        }
    }
    if (bad >= 0) {
        if (tid == 0) atomicCAS(info, 0, j0 + bad + 1);
        return;
    }
    __syncthreads();
    if (i < n) {
#pragma unroll
        for (int q = 0; q < Q; ++q) {
            const int c = g + 4 * q;
            if (c < n) {
                double v = 0.0;
                if (i >= c) {
                    const double sc = sqrt(piv[c]);
                    v = (i == c) ? sc : a[q] / sc;
                }
                G[i + (int64_t)c * ldg] = v;
            }
        }
    }
    __syncthreads();  // the shared buffers are reused by the caller
}


// Sign-choosing no-pivot LU of a <= 64 x 64 block, registers as in potrf_diag (thread (i, g) owns row i,
// columns g + 4q), one barrier per column: at step j the owners publish column j and row j, every thread
// reads a = A(j, j) (final), S_j = -sgn(a), pivot p = a - S_j, and updates A(i, c) -= A(i, j) A(j, c) / p
// for i, c > j.  The multipliers L(i, j) = A(i, j) / p_j are formed at the end.
__device__ __forceinline__ void getrf_sign_diag_block(int n, double* Qm, int64_t ldq, double* S, double (*colj)[FACT_NB],
                                      double (*rowj)[FACT_NB], double* piv)
{
    const int tid = threadIdx.x, i = tid & 63, g = tid >> 6;
    constexpr int Q = FACT_NB / 4;
    double a[Q];
#pragma unroll
    for (int q = 0; q < Q; ++q) {
        const int c = g + 4 * q;
        a[q] = (i < n && c < n) ? Qm[i + (int64_t)c * ldq] : 0.0;
    }
#pragma unroll
    for (int jq = 0; jq < Q; ++jq) {
        for (int jr = 0; jr < 4; ++jr) {
            const int j = 4 * jq + jr;
            if (j >= n) break;
            const int par = j & 1;
            if (g == jr) colj[par][i] = a[jq];
            if (i == j) {
#pragma unroll
                for (int q = 0; q < Q; ++q) rowj[par][g + 4 * q] = a[q];
            }
            __syncthreads();
            const double av = rowj[par][j];
            const double sj = (av >= 0.0) ? -1.0 : 1.0;  // S_jj = -sgn(a), sgn(a) = a >= 0 ? +1 : -1 (Z20)
            const double p = av - sj;
            if (tid == 0) {
                S[j] = sj;
                piv[j] = p;
            }
            if (i > j) {
                const double lij = colj[par][i] * (1.0 / p);
#pragma unroll
                for (int q = jq; q < Q; ++q) {
                    const int c = g + 4 * q;
                    if (c > j) a[q] = fma(-lij, rowj[par][c], a[q]);
                }
            }
        }
    }
    __syncthreads();
    if (i < n) {
#pragma unroll
        for (int q = 0; q < Q; ++q) {
            const int c = g + 4 * q;
            if (c < n) {
                double v = a[q];
                if (i == c) v = piv[c];
                else if (i > c) v = v / piv[c];
                Qm[i + (int64_t)c * ldq] = v;
            }
        }
    }
    __syncthreads();  // the shared buffers are reused by the caller
}


}  // namespace bqrrp
