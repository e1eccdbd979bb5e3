/*
 * bqrrp.h — C ABI of the B200 (sm_100a) BQRRP library, libbqrrp.so.
 *
 * BQRRP = Blocked QR with Randomization and Pivoting (Melnichenko, Murray, Killian, Demmel,
 * Mahoney, Luszczek, Gates; arXiv 2507.00976).  Citations "P:n" are lines of the paper's LaTeX
 * source; readings "Zn" are listed in DESIGN.md §3.
 *
 * Conventions for every entry point
 *   - Matrices are column-major fp64 with a leading dimension; "device" pointers are CUDA device
 *     memory of the current device, "host" pointers are ordinary (preferably pinned) host memory.
 *   - `stream` is a cudaStream_t passed as void* (NULL = legacy default stream).  Work is enqueued on
 *     it (bqrrp_factor* fans out internally to a high-priority critical stream and a low-priority bulk
 *     stream, both joined back to `stream`); device outputs are valid after the stream is synchronised.  bqrrp_factor* additionally
 *     synchronises the stream once per block iteration to read the block rank k (P:490 step
 *     bqrrp:rank_est decides the loop), so *rank is known on return.
 *   - Return value: 0 = success; -i = the i-th argument is illegal (LAPACK info convention; checked
 *     before any launch, nothing is touched); BQRRP_ENUMERIC = non-finite sketch or a Cholesky-QR
 *     breakdown; BQRRP_ENOMEM / BQRRP_ECUDA on allocation / CUDA failure (A, tau, J contents are then
 *     unspecified).  bqrrp_last_error() returns a thread-local message for the last failure.
 *   - The library owns no memory after a call returns and keeps no global state except
 *     per-thread error strings; calls on different streams are independent.
 */
#ifndef BQRRP_H
#define BQRRP_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define BQRRP_OK 0
#define BQRRP_ENUMERIC 1
#define BQRRP_ENOMEM (-100)
#define BQRRP_ECUDA (-101)
#define BQRRP_ENCCL (-102)

typedef struct bqrrp_options {
    /* tri_rank threshold relative to |R_sk^(0)(0,0)| (readings Z10/Z11).
     * <= 0 selects the default 10 * u * sqrt(max(m, n)). */
    double rank_tol;
    /* Panel variant / Cholesky-QR passes (Alg. 3 step cholqr:cholqr): 2 = CholQR2 + Householder
     * reconstruction (default), 1 = the paper's single CholQR pass, 0 = Householder QR of
     * the panel (the paper's BQRRP_HQR variant).  Negative = default. */
    int cholqr_passes;
    /* 0 (default): a panel whose Cholesky QR breaks down (POTRF meets a non-positive pivot, e.g. a rank_tol
     * far below the default) is re-factored by Householder QR (the BQRRP_HQR panel; SURVEY
     * §8(f) N2) instead of failing; costs one host sync per panel.  1: no fallback, breakdown returns
     * BQRRP_ENUMERIC. */
    int no_hqr_fallback;
    /* optional host float[9] out: per-phase milliseconds in the order of SPEC's profile keys
     * {qrcp_wide, tri_rank, col_perm, qr_tall, apply_trans_q, sample_update, other, total} (a sequential
     * partition of the critical stream's timeline) followed by apply_trans_q_bulk, the duration of the
     * bulk trailing-update GEMM that runs concurrently on the low-priority stream;
     * NULL = no timing (timing adds one event pair per phase). */
    float* phase_ms;
    /* 0 (default): the bulk rows of the trailing update run on a low-priority stream, overlapping the sketch
     * update and the next pivot selection.  1: everything on one stream, serialised (the
     * per-phase times then partition the whole step; used to measure each phase alone). */
    int no_lookahead;
} bqrrp_options;

/* Bytes of device workspace bqrrp_factor needs for an m x n matrix with block b and sketch d. */
int bqrrp_workspace_query(int64_t m, int64_t n, int64_t b, int64_t d, size_t* bytes);

/*
 * BQRRP factorization, Alg. 1 with the in-place recipe of §3:
 *   A(:, J) = Q R,  Q = H_1 ... H_l,  H_j = I - tau_j v_j v_j^T  (GEQP3 output format).
 *   m, n      matrix size (>= 0)
 *   A         device, m x n, lda >= max(1, m); overwritten: R (upper trapezoid, rows >= l zero) on and
 *             above the diagonal, v_j (unit head implicit) below; A(l:m, l:n) = 0 (reading Z16)
 *   b         block size (>= 1; b >= min(m,n) means a single iteration)
 *   d         sketch rows, b <= d <= m  (d = ceil(gamma b); d > m is a config violation)
 *   seed      64-bit seed of the counter-based Gaussian sketch
 *   tau       device, min(m,n) doubles; tau(l:) = 0
 *   J         device, n int64, one-based gather permutation
 *   rank      host int64 out: l
 *   workspace device buffer of >= bqrrp_workspace_query bytes, or NULL (allocated stream-ordered
 *             with cudaMallocAsync and freed before return)
 */
int bqrrp_factor(int64_t m, int64_t n, double* A, int64_t lda, int64_t b, int64_t d, uint64_t seed, double* tau,
                 int64_t* J, int64_t* rank, void* workspace, size_t ws_bytes, void* stream);

/* Same as bqrrp_factor with options (NULL = defaults). */
int bqrrp_factor_ex(int64_t m, int64_t n, double* A, int64_t lda, int64_t b, int64_t d, uint64_t seed, double* tau,
                    int64_t* J, int64_t* rank, void* workspace, size_t ws_bytes, void* stream,
                    const bqrrp_options* opts);

/* End-to-end variant on HOST buffers (A_host m x n col-major, ideally pinned; tau_host, J_host): A is
 * uploaded in column chunks on a copy stream while the sketch of the chunks already on the device is
 * computed, and each block column is copied back as soon as its iteration has finalised it, so both PCIe
 * directions overlap the factorization; tau and J at the end.  Synchronous; A_host is read and then
 * overwritten in place.  Device memory comes from the library's pool (see bqrrp_trim_memory). */
int bqrrp_factor_host(int64_t m, int64_t n, double* A_host, int64_t lda, int64_t b, int64_t d, uint64_t seed,
                      double* tau_host, int64_t* J_host, int64_t* rank, void* stream, const bqrrp_options* opts);

/* ---- debug / unit-test entry points (same conventions; all device pointers) ---- */

/* S (d x m, ld d; NULL to skip) and MskT = (S A)^T (n x d, ld n). */
int bqrrp_debug_sketch(int64_t m, int64_t n, const double* A, int64_t lda, int64_t d, uint64_t seed, double* S_out,
                       double* MskT_out, void* stream);

/* C = alpha op(A) op(B) + beta C with the DMMA engine; ta/tb: 0 = N, 1 = T. */
int bqrrp_debug_gemm(int ta, int tb, int64_t M, int64_t N, int64_t K, double alpha, const double* A, int64_t lda,
                     const double* B, int64_t ldb, double beta, double* C, int64_t ldc, void* stream);

/* X op(T) = B in place (B rows x n, ldb), op(T) upper triangular n x n: t_lower = 0 -> op(T) = T (upper
 * part read), 1 -> op(T) = T^T (lower part read); unit = 1: unit diagonal assumed.  inverse = 0:
 * blocked substitution (backward stable); 1: 64 x 64 diagonal blocks inverted and applied by DMMA (used by
 * the panel on its well-conditioned triangles).  The panel's TRSM building block. */
int bqrrp_debug_trsm(int64_t rows, int64_t n, const double* T, int64_t ldt, int t_lower, int unit, int inverse,
                     double* B, int64_t ldb, void* stream);

/* Partial-pivot LU of the w x d matrix L (in place): ipiv (device int64, min(w,d)) one-based LAPACK swap
 * list. */
int bqrrp_debug_lu_pivots(int64_t w, int64_t d, double* L, int64_t ld, int64_t* ipiv, void* stream);

/* R_sk^T of the sketch window W^T (w x d, ld): in place, as stored by the driver (upper trapezoid of
 * R_sk transposed, explicit zeros). */
int bqrrp_debug_sketch_qr(int64_t w, int64_t d, double* WT, int64_t ld, void* stream);

/* Columns [0, w) of X (rows x w) gathered by J_qr = piv_transform(ipiv);
 * ipiv device int64 one-based, length nlu.  Jqr_out (device int64, w; may be NULL) = J_qr. */
int bqrrp_debug_permute(int64_t rows, int64_t w, double* X, int64_t ldx, int64_t nlu, const int64_t* ipiv,
                        int64_t* Jqr_out, void* stream);

/* Panel: CholQR(passes) + Householder reconstruction (passes 1..4) or Householder QR (passes 0) of P (h x k, ld) preconditioned by Rsk11 (k x k
 * upper, ld k), written in GEQP3 format in place (R11 on/above, V below) with tau (k), plus the
 * compact-WY update of the trailing C (h x t, ld) that follows P in memory (t may be 0). */
int bqrrp_debug_panel(int64_t h, int64_t k, int64_t t, double* P, int64_t ld, const double* Rsk11, double* tau,
                      int cholqr_passes, void* stream);

/* ---- multi-GPU step entry points (driven by paper_2507_00976_b200/dist.py) ----
 * A is distributed 1-D block-cyclically over column positions (block width dist_nb = b); the transposed
 * sketch MskT (n x d) and J are replicated; the caller moves data between ranks (torch.distributed:
 * NCCL all-reduce / broadcast on a multi-GPU node).  All pointers device, all calls stream-ordered. */

/* a2 on the replicated sketch window MskT(s:n, :): LU pivots, J_qr touched set (tq[t] <- tsrc[t],
 * positions relative to s, *nt entries in unspecified order, capacity 2 min(n-s, d)), sketch rows and J(s:n) permuted
 * (J may be NULL), R_sk in place, k = tri_rank (ref = |R_sk(0,0)| stored when first).
 * Synchronises the stream; *k_out host. */
int bqrrp_step_pivots(int64_t n, int64_t d, int64_t s, int64_t kmax, double* MskT, int64_t ldm, int64_t* J,
                      double rank_tol, double* ref, int first, int* tq, int* tsrc, int* nt, int64_t* k_out,
                      void* stream);
/* dst(:, t) = X(:, idx[t]) (rows x n_idx), slots with idx[t] < 0 untouched. */
int bqrrp_step_gather_columns(int64_t rows, const double* X, int64_t ldx, const int* idx, int64_t nidx, double* dst,
                              int64_t ldd, void* stream);
/* X(:, idx[t]) = src(:, t), slots with idx[t] < 0 skipped. */
int bqrrp_step_scatter_columns(int64_t rows, double* X, int64_t ldx, const int* idx, int64_t nidx, const double* src,
                               int64_t lds, void* stream);
/* *is_zero_host = 1 iff col(0:h) is all zeros (the P:1008 early exit).  Synchronises. */
int bqrrp_step_zero_column_check(int64_t h, const double* col, int* is_zero_host, void* stream);
/* a4 on the owner of the panel: P (h x k, ldp) in place in GEQP3 format, tau (k), explicit V (h x k, ld h)
 * and T (k x k); R_sk11 read from the sketch window MskT_s (= MskT + s).  BQRRP_ENUMERIC on breakdown. */
int bqrrp_step_panel(int64_t h, int64_t k, double* P, int64_t ldp, const double* MskT_s, int64_t ldm, double* tau,
                     double* V, double* T, int cholqr_passes, void* stream);
/* a5 on one rank's trailing columns: C (h x t, ldc) <- C - V T^T (V^T C). */
int bqrrp_step_wy_update(int64_t h, int64_t k, int64_t t, const double* V, const double* T, double* C, int64_t ldc,
                         void* stream);
/* Row-distributed sketch: as bqrrp_step_pivots, but the rows of R_sk(:, d:w) (the d x d
 * QR's GEMM part) are computed only for the row blocks listed (host arrays; offsets counted from
 * window row min(d, w), i.e. position s + d): this rank's positions.  The other rows of MskT are left stale and
 * must be refreshed (all-gather) before the next pivot selection reads them. */
int bqrrp_step_pivots_rows(int64_t n, int64_t d, int64_t s, int64_t kmax, double* MskT, int64_t ldm, int64_t* J,
                           double rank_tol, double* ref, int first, int* tq, int* tsrc, int* nt, int64_t* k_out,
                           const int64_t* row_off, const int64_t* row_len, int64_t n_rows, void* stream);
/* a6 on this rank's positions only: X = R_sk11 R11^{-1}; for block j: MskT_s(b + pos_off[j] .. + len[j], 0:b)
 * -= R12(:, col_off[j] ..)^T X^T with R12 this rank's k x t_loc top rows (host arrays). */
int bqrrp_step_sample_update_rows(int64_t b, const double* R11, int64_t ldr, const double* R12, int64_t ld12,
                                  double* MskT_s, int64_t ldm, const int64_t* pos_off, const int64_t* col_off,
                                  const int64_t* len, int64_t nblk, void* stream);
/* a4 row-sharded (SURVEY §8(e) phase 2 item 3): each rank holds a block of the panel's rows
 * (column-major, rows x k); the k x k pieces are computed redundantly from all-reduced Gram matrices.
 * Preconditioning + first Gram (Alg. 3 cholqr:precond): Q = P R_sk11^{-1} (R_sk11 = R_sk(0:k,0:k) read
 * from MskT_s), G = Q^T Q (lower, k x k, ld k; zero when rows == 0).  P may equal Q (ldp == ldq). */
int bqrrp_step_cholqr_pre(int64_t rows, int64_t k, const double* P, int64_t ldp, const double* MskT_s, int64_t ldm,
                          double* Q, int64_t ldq, double* G, void* stream);
/* Lower Cholesky of the (all-reduced) Gram G in place, upper part zeroed.  Synchronises; BQRRP_ENUMERIC on a
 * non-positive pivot (the caller then factors the panel with the Householder variant). */
int bqrrp_step_potrf(int64_t k, double* G, int64_t ldg, void* stream);
/* Second CholQR pass on a row block: Q <- Q C^{-T}, G = Q^T Q (lower; zero when rows == 0). */
int bqrrp_step_cholqr_pass(int64_t rows, int64_t k, double* Q, int64_t ldq, const double* C, double* G, void* stream);
/* Householder reconstruction (Alg. 3 cholqr:orhr_col) on the block holding the panel's top k rows:
 * Wr = Q_top C^{-T} (k x k, ld k) factored in place as L \ U with S_jj = -sgn (S: k values). */
int bqrrp_step_recon_top(int64_t k, const double* Qtop, int64_t ldq, const double* C, double* Wr, double* S,
                         void* stream);
/* Y2 rows: Q <- Q (U C^T)^{-1} for a block of rows below the top k (U from Wr). */
int bqrrp_step_recon_rows(int64_t rows, int64_t k, double* Q, int64_t ldq, const double* Wr, const double* C,
                          void* stream);
/* k x k results: T = -U S L^{-T} (compact WY), tau = diag(T), R = C2^T C1^T R_sk11 (C2 may be NULL for one
 * pass; R11 = S R). */
int bqrrp_step_recon_finish(int64_t k, const double* Wr, const double* S, const double* C1, const double* C2,
                            const double* MskT_s, int64_t ldm, double* T, double* tau, double* R, void* stream);
/* top != 0: the first k rows of the block become the explicit unit-lower V rows of L (from Wr). */
int bqrrp_step_v_rows(int64_t rows, int64_t k, double* Q, int64_t ldq, const double* Wr, int top, void* stream);
/* GEQP3 write of the panel A (h x k, lda): S R on and above the diagonal, V (explicit, h x k, ldv) below. */
int bqrrp_step_write_panel(int64_t h, int64_t k, double* V, int64_t ldv, const double* R, const double* S, double* A,
                           int64_t lda, void* stream);
/* a5 split for the lookahead (DESIGN.md §7.5 / §8.1): bqrrp_step_wy_top computes W2 = T^T (V^T C) into the
 * caller's W2 (k x t, ldw >= k; it must stay alive until the bulk call has run) and applies C -= V W2 to rows
 * 0:k (R12) only; bqrrp_step_wy_bulk applies rows k:h, typically on a second stream ordered after the top call.
 * Together they equal bqrrp_step_wy_update. */
int bqrrp_step_wy_top(int64_t h, int64_t k, int64_t t, const double* V, const double* T, double* C, int64_t ldc,
                      double* W2, int64_t ldw, void* stream);
int bqrrp_step_wy_bulk(int64_t h, int64_t k, int64_t t, const double* V, const double* W2, int64_t ldw, double* C,
                       int64_t ldc, void* stream);
/* a6 on the replicated sketch: X = R_sk11 R11^{-1} (R_sk11 from MskT_s), MskT_s(b:b+t, 0:b) -= R12^T X^T with
 * R11 (b x b, ldr) and R12 (b x t, ld12) gathered in position order. */
int bqrrp_step_sample_update(int64_t b, int64_t t, const double* R11, int64_t ldr, const double* R12, int64_t ld12,
                             double* MskT_s, int64_t ldm, void* stream);
/* X(0:rows, 0:cols) = 0. */
int bqrrp_step_zero(int64_t rows, int64_t cols, double* X, int64_t ldx, void* stream);

/* Number of CUDA kernels this library has launched in the calling process (all threads). */
unsigned long long bqrrp_launch_count(void);
/* Panels re-factored by Householder QR after a CholQR breakdown in the last bqrrp_factor* call on this
 * thread (plus bqrrp_step_panel calls since). */
long long bqrrp_panel_fallbacks(void);

/* Device memory the library allocates itself (the workspace when none is passed, bqrrp_factor_host's device
 * copies, debug scratch) comes from a library-owned stream-ordered pool that keeps freed blocks mapped for
 * the next call.  This returns them to the driver (synchronises the current device).  0 or BQRRP_ECUDA. */
int bqrrp_trim_memory(void);

const char* bqrrp_strerror(int status);
const char* bqrrp_last_error(void);
/* Library version string. */
const char* bqrrp_version(void);

#ifdef __cplusplus
}
#endif
#endif /* BQRRP_H */
