// blas.cuh — dense building blocks on the DMMA GEMM engine (host launchers).
#pragma once
#include "common.cuh"

namespace bqrrp {

// C = alpha op(A) op(B) + beta C (column-major).  tri: only the lower triangle of C is needed.
// ctas_per_sm > 0: persistent launch of at most ctas_per_sm CTAs per SM looping over the tiles (no
// split-K).  Not used by the driver (measured slower for the bulk update).
// no_split: never split K (each element's K order then does not depend on how M / N are tiled or
// chunked — the sketch uses it so the host entry's chunked sketch is bitwise the device entry's).
// Extra GEMM modes (all off by default):
//   a_lower: op(A) is lower triangular (the TRMM W2 = T^T W of the compact-WY update: T upper, k^2 t flops
//            instead of 2 k^2 t); the zeros above the diagonal are skipped, the K order is unchanged.
//   fixed_tiles: always 64 x 64 tiles and no split-K, so every element's result is independent of M, N and of
//            the other tiles (two such GEMMs over the same operand rows / columns agree bitwise).
//   hs_state / hs_readers: the tile handshake of GemmArgs (implies fixed_tiles).
//   split_m / split_n: the split-K decision is taken as for an Md x Nd product (0 = the real M / N).
struct GemmExtra {
    int64_t split_m = 0, split_n = 0;
    bool a_lower = false;
    bool fixed_tiles = false;
    int* hs_state = nullptr;
    int* hs_readers = nullptr;
};
constexpr int GEMM_FIXED_TILE = 64;  // tile edge of fixed_tiles / handshake GEMMs
void gemm(Ctx& cx, bool ta, bool tb, int64_t M, int64_t N, int64_t K, double alpha, const double* A, int64_t lda,
          const double* B, int64_t ldb, double beta, double* C, int64_t ldc, bool tri = false, int ctas_per_sm = 0,
          bool no_split = false, const GemmExtra* extra = nullptr);

// X op(T) = B, right side, op(T) upper triangular (n x n), in place on B (rows x n).
//   t_lower = false: T stored upper, op(T) = T;  t_lower = true: T stored lower, op(T) = T^T.
//   well_conditioned: op(T) is known to be well conditioned (Cholesky factors of CholQR Gram matrices,
//   the reconstruction's U and unit-lower L): base cases multiply by inverted 64 x 64 diagonal blocks
//   (DMMA) instead of substituting; workspace: ceil(n/64) * 4096 doubles.
void trsm_right_upper(Ctx& cx, int64_t rows, int64_t n, const double* T, int64_t ldt, bool t_lower, bool unit,
                      double* B, int64_t ldb, bool well_conditioned = false);

// L X = B, left side, L unit lower (n x n), in place on B (n x cols).
void trsm_left_lower_unit(Ctx& cx, int64_t n, int64_t cols, const double* L, int64_t ldl, double* B, int64_t ldb);

// Lower Cholesky G = L L^T in place (n x n, lower part read); strict upper part zeroed on return.
// A non-positive pivot sets flags[F_POTRF_INFO] = first failing column + 1 (and stops that block).
void potrf_lower(Ctx& cx, int64_t n, double* G, int64_t ldg);

// Householder reconstruction LU (BD2015 Alg. 5 reading): in place on the top n x n of
// Q (ld), no pivoting, with S_jj = -sgn(current Q_jj) chosen on the fly; pivot = Q_jj - S_jj.
// On return: strict lower = L (unit), upper = U; S[j] = S_jj (+-1).
void getrf_nopiv_sign(Ctx& cx, int64_t n, double* Q, int64_t ldq, double* S);

constexpr int FACT_NB = 64;  // diagonal block of the blocked / persistent k x k factorizations

// small element-wise kernels
void copy_matrix(Ctx& cx, int64_t rows, int64_t cols, const double* src, int64_t lds, double* dst, int64_t ldd);
void transpose_copy(Ctx& cx, int64_t rows, int64_t cols, const double* src, int64_t lds, double* dst, int64_t ldd);
void set_zero(Ctx& cx, int64_t rows, int64_t cols, double* A, int64_t lda);
// uplo: 'L' zero the strict upper part, 'U' zero the strict lower part
void zero_triangle(Ctx& cx, char keep, int64_t n, int64_t cols, double* A, int64_t lda, bool unit_diag = false);

}  // namespace bqrrp
