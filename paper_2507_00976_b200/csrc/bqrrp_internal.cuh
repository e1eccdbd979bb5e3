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
// a2: R_sk of the sketch window (transposed storage), in place.
void sketch_qr(Ctx& cx, double* MskT, int64_t ldm, int64_t w, int64_t d);

// a3: touched set and gathers
void touched_from_perm(Ctx& cx, int64_t w, int64_t nlu, const int* perm, Touched& T);
void perm_from_ipiv(Ctx& cx, int64_t w, int64_t nlu, const int64_t* ipiv1, int* perm);
void permute_columns(Ctx& cx, int64_t rows, double* X, int64_t ldx, const Touched& T, double* scratch);
void permute_rows(Ctx& cx, int64_t cols, double* X, int64_t ldx, const Touched& T, double* scratch);
void permute_vector(Ctx& cx, int64_t* J, const Touched& T, int64_t* tmp);

// a4 + a5: preconditioned CholQR2 + Householder reconstruction of the panel A(s:m, s:s+k), the
// compact-WY update of A(s:m, s+k:n) and the in-place GEQP3-format write of V, R11, tau.
// Rsk11: k x k upper (ld k).  Returns nothing; failures are flagged in cx.flags.
struct PanelOut {
    double* T;   // k x k (ld k) compact-WY T (upper)
    double* V;   // h x k explicit reflectors (ld h)
};
void panel_and_update(Ctx& cx, int64_t m, int64_t n, double* A, int64_t lda, int64_t s, int64_t k, const double* Rsk11,
                      double* tau, int cholqr_passes, PanelOut& out);

}  // namespace bqrrp
