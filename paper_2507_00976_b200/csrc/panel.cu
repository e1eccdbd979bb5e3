// panel.cu — a4 + a5: the CholQR panel with Householder reconstruction and the compact-WY trailing
// update (Alg. 3 "Cholesky QR + dependencies", in-place recipe P:1032-1053; apply_trans_q
// P:781-808).
//
//   M_pre  = P(:, 0:k) R_sk11^{-1}                               (Alg. 3 step cholqr:precond)
//   for pass in 1..passes:  G = Q^T Q, G = C C^T, Q <- Q C^{-T}   (cholqr; passes = 2 is CholQR2,
//                                                                  DESIGN.md §7.3, SURVEY App. B1;
//                                                                  a breakdown falls back to HQR)
//   Q - [S; 0] = L U (no pivoting, S_jj = -sgn(Q'_jj) on the fly)   (cholqr:orhr_col, BD2015 Alg. 5/6;
//   V = L, T = -U S Y1^{-T}, tau = diag(T)                           P:697-701)
//   R11 = diag(S) C_last^T ... C_1^T R_sk11                        (cholqr:undo_precond, reading Z7)
//   C <- C - V T^T (V^T C) on C = A(s:m, s+k:n)                    (apply_trans_q, compact WY)
#include <cstdlib>

#include "blas.cuh"
#include "bqrrp_internal.cuh"

namespace bqrrp {

// T(i,j) = -U(i,j) S_j for i <= j, 0 below (the right-hand side of T Y1^T = -U S).
__global__ void build_t_rhs_kernel(int64_t k, const double* Q, int64_t ldq, const double* S, double* T)
{
    int64_t total = k * k;
    for (int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; idx < total; idx += (int64_t)gridDim.x * blockDim.x) {
        int64_t i = idx % k, j = idx / k;
        T[idx] = (i <= j) ? -Q[i + j * ldq] * S[j] : 0.0;
    }
}

__global__ void diag_to_tau_kernel(int64_t k, const double* T, double* tau)
{
    int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (j < k) tau[j] = T[j + j * k];
}

// GEQP3-format write of the panel: A(s+i, s+j) = S_i R(i, j) for i <= j (< k); = V(i, j) for i > j.
// Q (the reconstruction's L, unit diagonal implicit, and Y2 below) is converted in place to the
// explicit V (ones on the diagonal, zeros above) used by the WY GEMMs.
__global__ void write_panel_kernel(int64_t h, int64_t k, double* Q, int64_t ldq, const double* R, const double* S,
                                   double* Ap, int64_t lda)
{
    int64_t total = h * k;
    for (int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; idx < total; idx += (int64_t)gridDim.x * blockDim.x) {
        int64_t i = idx % h, j = idx / h;
        double* q = Q + i + j * ldq;
        if (i > j) {
            Ap[i + j * lda] = *q;
        } else {
            Ap[i + j * lda] = S[i] * R[i + j * k];
            *q = (i == j) ? 1.0 : 0.0;
        }
    }
}

// ---- phases of the CholQR panel, shared by the one-GPU panel below and the row-sharded multi-GPU panel
// (steps.cu): every phase works on a block of panel ROWS except the k x k ones.

void cholqr_precondition_gram(Ctx& cx, int64_t rows, int64_t k, const double* P, int64_t ldp, const double* Rsk11,
                              double* Q, int64_t ldq, double* G)
{
    if (rows > 0) {
        if (P != Q) copy_matrix(cx, rows, k, P, ldp, Q, ldq);
        trsm_right_upper(cx, rows, k, Rsk11, k, false, false, Q, ldq);  // M_pre = P R_sk11^{-1}
        gemm(cx, true, false, k, k, rows, 1.0, Q, ldq, Q, ldq, 0.0, G, k, /*tri=*/true);
    } else {
        BQ_CUDA(cudaMemsetAsync(G, 0, sizeof(double) * k * k, cx.stream));
    }
}

void cholqr_pass_gram(Ctx& cx, int64_t rows, int64_t k, double* Q, int64_t ldq, const double* C, double* G)
{
    if (rows > 0) {
        trsm_right_upper(cx, rows, k, C, k, /*t_lower=*/true, false, Q, ldq, true);  // Q <- Q C^{-T}
        gemm(cx, true, false, k, k, rows, 1.0, Q, ldq, Q, ldq, 0.0, G, k, /*tri=*/true);
    } else {
        BQ_CUDA(cudaMemsetAsync(G, 0, sizeof(double) * k * k, cx.stream));
    }
}

void recon_top_lu(Ctx& cx, int64_t k, const double* Qtop, int64_t ldq, const double* C, double* Wr, double* S)
{
    copy_matrix(cx, k, k, Qtop, ldq, Wr, k);
    trsm_right_upper(cx, k, k, C, k, /*t_lower=*/true, false, Wr, k, true);  // top rows of Q_last = Q C^{-T}
    getrf_nopiv_sign(cx, k, Wr, k, S);                                       // Q_last,1 - S = L U
}

void recon_rows(Ctx& cx, int64_t rows, int64_t k, double* Q, int64_t ldq, const double* Wr, const double* C)
{
    if (rows <= 0) return;
    const size_t mark = cx.ws_used;
    double* U = cx.alloc((size_t)k * k);
    double* Mb = cx.alloc((size_t)k * k);
    copy_matrix(cx, k, k, Wr, k, U, k);
    zero_triangle(cx, 'U', k, k, U, k);                                    // U
    gemm(cx, false, true, k, k, k, 1.0, U, k, C, k, 0.0, Mb, k);            // U C^T (upper)
    trsm_right_upper(cx, rows, k, Mb, k, false, false, Q, ldq, true);      // Y2 = Q_prev,2 (U C^T)^{-1}
    cx.ws_used = mark;
}

void recon_finish(Ctx& cx, int64_t k, const double* Wr, const double* S, const double* const* Cf, int passes,
                  const double* Rsk11, double* T, double* tau, double* R, double* scratch)
{
    build_t_rhs_kernel<<<(unsigned)imin(cdiv(k * k, 256), 4 * cx.num_sms), 256, 0, cx.stream>>>(k, Wr, k, S, T);
    BQ_LAUNCH_CHECK();
    trsm_right_upper(cx, k, k, Wr, k, /*t_lower=*/true, /*unit=*/true, T, k, true);  // T Y1^T = -U S
    zero_triangle(cx, 'U', k, k, T, k);
    diag_to_tau_kernel<<<(unsigned)cdiv(k, 128), 128, 0, cx.stream>>>(k, T, tau);
    BQ_LAUNCH_CHECK();
    // R = C_last^T ... C_1^T R_sk11 (the caller applies S: R11 = S R)
    const size_t mark = cx.ws_used;
    double* Wa = scratch ? scratch : cx.alloc((size_t)k * k);
    double* Wb = scratch ? scratch + (size_t)k * k : cx.alloc((size_t)k * k);
    copy_matrix(cx, k, k, Rsk11, k, Wa, k);
    for (int p = 0; p < passes; ++p) {
        gemm(cx, true, false, k, k, k, 1.0, Cf[p], k, Wa, k, 0.0, Wb, k);
        double* t = Wa; Wa = Wb; Wb = t;
    }
    copy_matrix(cx, k, k, Wa, k, R, k);
    cx.ws_used = mark;
}

void write_panel(Ctx& cx, int64_t h, int64_t k, double* Q, int64_t ldq, const double* R, const double* S, double* Ap,
                 int64_t lda)
{
    unsigned eb = (unsigned)imin(cdiv(h * k, 256), 8 * cx.num_sms);
    write_panel_kernel<<<eb, 256, 0, cx.stream>>>(h, k, Q, ldq, R, S, Ap, lda);
    BQ_LAUNCH_CHECK();
}

void force_breakdown_hook(Ctx& cx)
{
    // test hook (bqrrp_options.debug_flags & BQRRP_DEBUG_FORCE_BREAKDOWN): report a POTRF breakdown on every
    // panel, so the fallback / error path is exercised deterministically (a real breakdown depends on rounding)
    if (cx.force_breakdown) BQ_CUDA(cudaMemsetAsync(cx.flags + F_POTRF_INFO, 1, 1, cx.stream));
}

int panel_factor(Ctx& cx, int64_t h, double* Ap, int64_t lda, int64_t k, const double* Rsk11, double* tau,
                 int passes, double* V, double* T, bool hqr_fallback, Ctx* side)
{
    if (passes == 0) {  // BQRRP_HQR: Householder QR of the panel itself
        householder_panel(cx, Ap, lda, h, k, tau, V, T);
        return 0;
    }
    size_t mark = cx.ws_used;
    double* Q = V;  // h x k (ld h): M_pre -> Q_chol -> reconstruction L -> explicit V
    double* Cf[4];
    for (int p = 0; p < passes; ++p) Cf[p] = cx.alloc((size_t)k * k);
    double* S = cx.alloc((size_t)k);
    double* Wr = cx.alloc((size_t)k * k);
    double* R = cx.alloc((size_t)k * k);

    // Cholesky QR passes; the last pass's TRSM is applied only to the top k rows (recon_top_lu) and folded into
    // the reconstruction's TRSM (Y2 = Q_prev,2 C^{-T} U^{-1} = Q_prev,2 (U C^T)^{-1}, recon_rows)
    cholqr_precondition_gram(cx, h, k, Ap, lda, Rsk11, Q, h, Cf[0]);
    potrf_lower(cx, k, Cf[0], k);
    for (int p = 1; p < passes; ++p) {
        cholqr_pass_gram(cx, h, k, Q, h, Cf[p - 1], Cf[p]);
        potrf_lower(cx, k, Cf[p], k);
    }
    force_breakdown_hook(cx);
    if (hqr_fallback) {  // CholQR breakdown (POTRF non-positive pivot): this panel by Householder QR instead
        int info = 0;
        BQ_CUDA(cudaMemcpyAsync(&info, cx.flags + F_POTRF_INFO, sizeof(int), cudaMemcpyDeviceToHost, cx.stream));
        BQ_CUDA(cudaStreamSynchronize(cx.stream));
        if (info) {
            BQ_CUDA(cudaMemsetAsync(cx.flags + F_POTRF_INFO, 0, sizeof(int), cx.stream));
            cx.ws_used = mark;
            householder_panel(cx, Ap, lda, h, k, tau, V, T);
            return 1;
        }
    }
    const double* Cl = Cf[passes - 1];
    recon_top_lu(cx, k, Q, h, Cl, Wr, S);
    if (side && h > 2 * k) {
        // the k x k finish (T-solve, tau, R products) depends only on Wr and S: run it on the side stream
        // (idle during the panel) while the main stream does the tall Y2 TRSM; its scratch (the two k x k
        // products and the inverse-diagonal blocks of its k x k TRSM) is an arena carved here
        Ctx sc = side_ctx(cx, *side, (size_t)2 * k * k + (size_t)(cdiv(k, 64) + 1) * 64 * 64 + 64);
        double* scr = sc.alloc((size_t)2 * k * k);
        cudaEvent_t ef, ej;
        BQ_CUDA(cudaEventCreateWithFlags(&ef, cudaEventDisableTiming));
        BQ_CUDA(cudaEventCreateWithFlags(&ej, cudaEventDisableTiming));
        BQ_CUDA(cudaEventRecord(ef, cx.stream));
        BQ_CUDA(cudaStreamWaitEvent(side->stream, ef, 0));
        recon_finish(sc, k, Wr, S, Cf, passes, Rsk11, T, tau, R, scr);
        BQ_CUDA(cudaEventRecord(ej, side->stream));
        recon_rows(cx, h - k, k, Q + k, h, Wr, Cl);
        copy_matrix(cx, k, k, Wr, k, Q, h);  // L \ U on top
        BQ_CUDA(cudaStreamWaitEvent(cx.stream, ej, 0));
        BQ_CUDA(cudaEventDestroy(ef));
        BQ_CUDA(cudaEventDestroy(ej));
    } else {
        if (h > k) recon_rows(cx, h - k, k, Q + k, h, Wr, Cl);
        copy_matrix(cx, k, k, Wr, k, Q, h);  // L \ U on top
        recon_finish(cx, k, Wr, S, Cf, passes, Rsk11, T, tau, R, nullptr);
    }
    write_panel(cx, h, k, Q, h, R, S, Ap, lda);
    cx.ws_used = mark;
    return 0;
}

// a5, one stream: C (h x t) <- C - V T^T (V^T C): W = V^T C, W2 = T^T W (TRMM: T upper), C -= V W2.
void wy_update(Ctx& cx, int64_t h, int64_t k, int64_t t, const double* V, int64_t ldv, const double* T, double* C,
               int64_t ldc, double* W, double* W2)
{
    if (t <= 0) return;
    wy_top(cx, h, k, t, V, ldv, T, C, ldc, W, W2, /*rows=*/h);
}

// a5 critical part: W = V^T C (K = h), W2 = T^T W, and C(0:rows) -= V(0:rows) W2 (rows = k: R12 only, the
// bulk rows k:h follow on the bulk stream, wy_bulk; rows = h: the whole update).
void wy_top(Ctx& cx, int64_t h, int64_t k, int64_t t, const double* V, int64_t ldv, const double* T, double* C,
            int64_t ldc, double* W, double* W2, int64_t rows, int64_t split_n)
{
    if (t <= 0) return;
    GemmExtra hint, trmm;
    hint.split_n = trmm.split_n = split_n;
    trmm.a_lower = true;
    gemm(cx, true, false, k, t, h, 1.0, V, ldv, C, ldc, 0.0, W, k, false, 0, false, &hint);        // W  = V^T C
    gemm(cx, true, false, k, t, k, 1.0, T, k, W, k, 0.0, W2, k, false, 0, false, &trmm);           // W2 = T^T W
    gemm(cx, false, false, rows, t, k, -1.0, V, ldv, W2, k, 1.0, C, ldc, false, 0, false, &hint);  // C -= V W2
}

// a5 bulk rows k:h on the bulk context: C(k:h) -= V(k:h) W2, in fixed 64 x 64 tiles (bitwise the values the
// lookahead's panel gather computes for its columns) with the tile handshake when hs_state is given.
// One CTA per tile: the high-priority GEMMs of the critical chain take SMs as the bulk's CTAs retire (a
// persistent bulk with 2-4 CTAs/SM starved them: C3 +0.5-0.8 s, profiles/bulk_persistent_r01.json).
void wy_bulk(Ctx& cb, int64_t h, int64_t k, int64_t t, const double* V, int64_t ldv, const double* W2, double* C,
             int64_t ldc, int* hs_state, int* hs_readers)
{
    if (t <= 0 || h <= k) return;
    GemmExtra x;
    x.fixed_tiles = true;
    x.hs_state = hs_state;
    x.hs_readers = hs_readers;
    gemm(cb, false, false, h - k, t, k, -1.0, V + k, ldv, W2, k, 1.0, C + k, ldc, false, 0, true, &x);
}

}  // namespace bqrrp
