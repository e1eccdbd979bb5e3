// bqrrp_internal.cuh — internal interfaces between the BQRRP kernels and the driver.
#pragma once
#include "common.cuh"

namespace bqrrp {

// Touched set of the local permutation J_qr (positions relative to s).
struct Touched {
    int* tq = nullptr;    // positions that change
    int* tsrc = nullptr;  // tsrc[t] = J_qr(tq[t]) - 1
    int* nt = nullptr;    // device count
    int64_t maxnt = 0;    // host bound 2*nlu
};

// a1: St(l, i) = gauss(seed, 0, i, l) (m x d, ld m) — the sketching operator S^T.
void sketch_operator_T(Ctx& cx, int64_t m, int64_t d, uint64_t seed, double* St, int64_t ldst);
// a1: MskT = A^T S^T (n x d, ld ldm).
void sketch_apply(Ctx& cx, int64_t m, int64_t n, const double* A, int64_t lda, int64_t d, uint64_t seed, double* MskT,
                  int64_t ldm, double* St /* m x d scratch */);

// a2: partial-pivot LU of the w x d matrix L (in place), ipiv[j] = 0-based pivot row, j < min(w,d);
// perm (w) = the row permutation of piv_transform (J_qr - 1).
void getrf_pivots(Ctx& cx, double* L, int64_t ld, int64_t w, int64_t d, int* ipiv, int* perm);
// Householder QR (GEQRF semantics, convention H) of A (rows x cols, lda) in place: R on/above the
// diagonal, reflectors below; V (rows x cols, ld rows) explicit, T (cols x cols) the compact-WY factor.
void householder_panel(Ctx& cx, double* A, int64_t lda, int64_t rows, int64_t cols, double* tau, double* V, double* T);
// a2: R_sk of the sketch window (transposed storage), in place.
// rows: optional restriction of the R_sk(:, d:w) rows computed (multi-GPU: only the rows of this rank's
// positions; the others are left stale and refreshed by the caller's all-gather): n_rows blocks, block j =
// rows [row_off[j], row_off[j] + row_len[j]) counted from window row p = min(d, w) (host arrays).
struct RowBlocks {
    const int64_t* off = nullptr;
    const int64_t* len = nullptr;
    int64_t n = -1;  // < 0: all rows
};
// defer: run the R_sk(:, d:w) GEMM (the bulk of the sketch QR's flops, 2 (w - d) d^2) on a second stream,
// ordered after the work already queued there; Q (d x d) and Y ((w - d) x d) are caller-owned buffers that
// stay alive until that stream has run it.  The caller orders the next reader of those rows after it.
struct RskDefer {
    Ctx* side = nullptr;
    double* Q = nullptr;
    double* Y = nullptr;
};
void sketch_qr(Ctx& cx, double* MskT, int64_t ldm, int64_t w, int64_t d, const RowBlocks& rows = RowBlocks(),
               const RskDefer* defer = nullptr);

// a3: touched set and gathers
void touched_from_perm(Ctx& cx, int64_t w, int64_t nlu, const int* perm, Touched& T);
void perm_from_ipiv(Ctx& cx, int64_t w, int64_t nlu, const int64_t* ipiv1, int* perm);
void permute_columns(Ctx& cx, int64_t rows, double* X, int64_t ldx, const Touched& T, double* scratch);
void permute_rows(Ctx& cx, int64_t cols, double* X, int64_t ldx, const Touched& T, double* scratch);
void permute_vector(Ctx& cx, int64_t* J, const Touched& T, int64_t* tmp);

// a4: preconditioned CholQR(passes) + Householder reconstruction (passes >= 1) — or, passes == 0, the
// Householder panel of the paper's BQRRP_HQR variant — of the panel A(s:m, s:s+k) written in
// GEQP3 format in place (R11 on/above, V below, tau(s:s+k)); V (h x k, ld h, explicit: unit diagonal,
// zeros above) and the compact-WY T (k x k, ld k) are returned in caller-owned buffers.
// Panels re-factored by Householder QR after a CholQR breakdown (bqrrp_panel_fallbacks()).
extern thread_local long long g_panel_fallbacks;
// hqr_fallback: after the Cholesky passes, read the POTRF breakdown flag (one host sync) and on a breakdown
// factor this panel with Householder QR instead (returns 1; 0 otherwise; the flag is cleared).
int panel_factor(Ctx& cx, int64_t m, double* A, int64_t lda, int64_t s, int64_t k, const double* Rsk11, double* tau,
                 int passes, double* V, double* T, bool hqr_fallback = false, Ctx* side = nullptr);
// Phases of the CholQR panel (panel.cu), on a block of panel rows unless k x k:
//   M_pre = P R_sk11^{-1} -> Q (ld ldq), G = M_pre^T M_pre (lower; zero if rows == 0)
void cholqr_precondition_gram(Ctx& cx, int64_t rows, int64_t k, const double* P, int64_t ldp, const double* Rsk11,
                              double* Q, int64_t ldq, double* G);
//   Q <- Q C^{-T} (C: lower Cholesky factor of the previous Gram), G = Q^T Q (lower)
void cholqr_pass_gram(Ctx& cx, int64_t rows, int64_t k, double* Q, int64_t ldq, const double* C, double* G);
//   Wr = Q_top C^{-T} (k x k) -> L \ U of the sign-choosing LU, S (k)
void recon_top_lu(Ctx& cx, int64_t k, const double* Qtop, int64_t ldq, const double* C, double* Wr, double* S);
//   rows of Y2 = Q (U C^T)^{-1} in place
void recon_rows(Ctx& cx, int64_t rows, int64_t k, double* Q, int64_t ldq, const double* Wr, const double* C);
//   T = -U S L^{-T}, tau = diag(T), R = C_passes^T ... C_1^T R_sk11 (R11 = S R)
void recon_finish(Ctx& cx, int64_t k, const double* Wr, const double* S, const double* const* Cf, int passes,
                  const double* Rsk11, double* T, double* tau, double* R, double* scratch = nullptr);
//   GEQP3 write of the panel (S R on/above, V below) and Q (L \ U on top, Y2 below) -> explicit V in place
void write_panel(Ctx& cx, int64_t h, int64_t k, double* Q, int64_t ldq, const double* R, const double* S, double* Ap,
                 int64_t lda);
void force_breakdown_hook(Ctx& cx);
// a5: C = A(s:m, s+k:n) <- C - V T^T (V^T C).  With cx_bulk, rows k:h of the last GEMM run on
// cx_bulk->stream after ev_top (recorded on cx.stream), and ev_bulk marks their completion.
void wy_update(Ctx& cx, Ctx* cx_bulk, int64_t m, int64_t n, double* A, int64_t lda, int64_t s, int64_t k,
               const double* V, const double* T, double* W, double* W2, cudaEvent_t ev_top, cudaEvent_t ev_bulk);

}  // namespace bqrrp
