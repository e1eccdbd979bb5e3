// bqrrp_internal.cuh — internal interfaces between the BQRRP kernels and the driver.
#pragma once
#include <functional>
#include <string>
#include <vector>

#include "../../include/bqrrp.h"
#include "common.cuh"

namespace bqrrp {

// ---- driver plumbing shared by the one-GPU (bqrrp.cu) and the multi-GPU (dist.cu) entries
struct Layout {
    size_t persistent, temp, splitk, total;
};
// workspace of bqrrp_factor: persistent buffers, temporaries, split-K slices (the slice capacity is part of
// the split-K decision, so the multi-GPU driver carves the same splitk size as the one-GPU run)
Layout layout(int64_t m, int64_t n, int64_t b, int64_t d);
void setup_ctx(Ctx& cx, void* stream);
void carve(Ctx& cx, void* ws, size_t bytes, const Layout& L);
int* pinned_flags();
extern thread_local std::string g_last_error;

struct NcclError : std::runtime_error {
    explicit NcclError(const std::string& s) : std::runtime_error(s) {}
};

// Exceptions -> C-ABI status codes (+ the thread-local message).
template <typename F>
int guarded(F&& f)
{
    try {
        return f();
    } catch (const CudaError& e) {
        g_last_error = e.what();
        return BQRRP_ECUDA;
    } catch (const NcclError& e) {
        g_last_error = e.what();
        return BQRRP_ENCCL;
    } catch (const std::bad_alloc& e) {
        g_last_error = e.what();
        return BQRRP_ENOMEM;
    } catch (const std::exception& e) {
        g_last_error = e.what();
        return std::string(e.what()).find("workspace") != std::string::npos ? BQRRP_ENOMEM : BQRRP_ECUDA;
    }
}

// small step kernels of the driver (bqrrp.cu): J = 1..n; flags[F_NONFINITE] if X has a non-finite entry;
// flags[F_K] = tri_rank (readings Z10 / Z11) and the zero-column flag armed; the zero-column test
// clears it; R_sk11 (k x k upper, ld k) out of the transposed sketch window
void init_j(Ctx& cx, int64_t n, int64_t* J);
void nonfinite_check(Ctx& cx, int64_t rows, int64_t cols, const double* X, int64_t ldx);
void tri_rank_flags(Ctx& cx, const double* MskT_s, int64_t ldm, int64_t kmax, bool first, double rank_tol, double* ref);
void zero_col_flag(Ctx& cx, int64_t h, const double* col);
void extract_rsk11(Ctx& cx, int64_t k, const double* MskT_s, int64_t ldm, double* R);

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
// on_leaf (optional) is called on the host after each leaf is queued with c1 = the number of leading pivots that
// are final from then on in stream order (perm[0:c1) and ipiv[0:c1)): the K-SQR pipeline starts on them.
using LeafDone = std::function<void(int64_t c1)>;
void getrf_pivots(Ctx& cx, double* L, int64_t ld, int64_t w, int64_t d, int* ipiv, int* perm,
                  const LeafDone* on_leaf = nullptr);
// The same pivots by a right-looking blocked LU with a one-block lookahead: the wide trailing update of each leaf
// on the second stream lu2 (allocates nothing), only the next block's on cx (lu.cu).  false = not applicable (w
// beyond the register leaf): nothing queued.  evpool: caller-owned events, reused.
bool getrf_pivots_la(Ctx& cx, Ctx& lu2, std::vector<cudaEvent_t>& evpool, double* L, int64_t ld, int64_t w, int64_t d,
                     int* ipiv, int* perm, const LeafDone* on_leaf = nullptr);
// Largest sketch-transpose height (w = n - s rows) K-LU's grid leaf holds; largest panel height the
// Householder panel (HQR variant and CholQR-breakdown fallback) holds.  Checked before any launch.
int64_t lu_max_rows(int num_sms);
int64_t qr_max_rows(int num_sms);
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
// The same R_sk, pipelined with K-LU (one-GPU lookahead driver): R_sk(:, 0:p) is the QR of the
// sketch columns J(0:p) in pivot order, and K-LU fixes them in order, leaf by leaf.  So the Householder QR runs
// LEFT-looking on its own stream q: as soon as a 32-column block of pivots is final, its sketch columns are
// gathered (on the critical stream, from the not yet permuted MskT rows perm[c]) into Wq, and q applies the
// previous blocks' reflectors to it (three GEMMs), factors it with the K-SQR leaf, and extends T (three GEMMs),
// while K-LU factors the next columns.  finish() joins q and does the rest of sketch_qr (Q_sk, the R_sk(:, d:w)
// GEMM, the in-place store).  Buffers come from cx's bump allocator at begin (released by finish, LIFO with
// the LU's own scratch); q allocates nothing.  events: caller-owned pool, reused across calls.
struct SketchQrPipe {
    Ctx* cx = nullptr;
    Ctx* q = nullptr;
    Ctx* q2 = nullptr;  // optional: the T-merge GEMMs of each block on a second stream (overlapping the next block)
    double* MskT = nullptr;
    int64_t ldm = 0, w = 0, d = 0, p = 0;
    double *Wq = nullptr, *V = nullptr, *Tf = nullptr, *tau = nullptr, *W1 = nullptr, *W2 = nullptr;
    double *xbuf = nullptr, *rowj = nullptr;
    double *W3 = nullptr, *W4 = nullptr;  // q2's scratch
    cudaEvent_t ev_t = nullptr;           // q2 finished the previous block's T merge
    int64_t gathered = 0, queued = 0;
    std::vector<cudaEvent_t>* events = nullptr;
    size_t nev = 0;
    size_t mark = 0;
};
void sketch_qr_pipe_begin(SketchQrPipe& P, Ctx& cx, Ctx& q, std::vector<cudaEvent_t>& events, double* MskT,
                          int64_t ldm, int64_t w, int64_t d, Ctx* q2 = nullptr);
void sketch_qr_pipe_columns(SketchQrPipe& P, const int* perm, int64_t c1);
void sketch_qr_pipe_finish(SketchQrPipe& P, const RskDefer* defer);

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
// The panel Ap (h x k, lda: A(s:m, s:s+k) in place, or the lookahead's gathered copy), tau = tau + s.
int panel_factor(Ctx& cx, int64_t h, double* Ap, int64_t lda, int64_t k, const double* Rsk11, double* tau,
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
// a5: C (h x t, ldc) <- C - V T^T (V^T C) (panel.cu): one stream (wy_update), or split for the lookahead into the
// critical part (wy_top with rows = k: W, W2 = T^T W, R12) and the bulk rows k:h (wy_bulk, on the bulk stream,
// fixed tiles, optional tile handshake).  V explicit h x k (ld ldv), T k x k upper, W / W2 k x t (ld k).
void wy_update(Ctx& cx, int64_t h, int64_t k, int64_t t, const double* V, int64_t ldv, const double* T, double* C,
               int64_t ldc, double* W, double* W2);
// split_n: the split-K decisions of the per-column GEMMs taken for a t = split_n wide update (multi-GPU: the
// whole trailing width, so each rank's columns get the one-GPU bits; 0 = t)
void wy_top(Ctx& cx, int64_t h, int64_t k, int64_t t, const double* V, int64_t ldv, const double* T, double* C,
            int64_t ldc, double* W, double* W2, int64_t rows, int64_t split_n = 0);
void wy_bulk(Ctx& cb, int64_t h, int64_t k, int64_t t, const double* V, int64_t ldv, const double* W2, double* C,
             int64_t ldc, int* hs_state, int* hs_readers);

// a3 for the pivot-aware lookahead (perm.cu).  The next panel's columns (positions q < nq of the
// next window, source perm[q]) of the trailing block C (rows x w, ldc) while the bulk GEMM (fixed 64 x 64 tiles,
// tiles_n tile columns) may be updating C:
//   la_gather_pre: P(:, q) = C(:, perm[q]) for every 64-row tile the bulk has not started (copied under the
//                  tile's reader count); post[R + q * tiles_m] = 1 for the others;
//   la_gather_post: P(R rows, q) = C(R rows, perm[q]) for the marked tiles once the bulk has written them.
// gather_cols_idx: dst(:, q) = X(:, idx[q]) for q < nq.
void la_gather_pre(Ctx& cx, int64_t rows, const double* C, int64_t ldc, const int* perm, int64_t nq, int64_t tiles_n,
                   int* hs_state, int* hs_readers, double* P, int64_t ldp, int* post);
void la_gather_post(Ctx& cx, int64_t rows, const double* C, int64_t ldc, const int* perm, int64_t nq, int64_t tiles_n,
                    const int* hs_state, double* P, int64_t ldp, const int* post);
void gather_cols_idx(Ctx& cx, int64_t rows, const double* X, int64_t ldx, const int* idx, int64_t nq, double* dst,
                     int64_t ldd);

}  // namespace bqrrp
