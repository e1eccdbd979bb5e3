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
    /* bqrrp_factor_dist only: width of the 1-D block-cyclic column blocks;
     * <= 0 selects b.  Must divide b or be a multiple of it (so each panel lives on one rank). */
    int64_t dist_nb;
    /* Test hooks, 0 in production.  BQRRP_DEBUG_FORCE_BREAKDOWN: every panel reports a POTRF breakdown, so the
     * Householder fallback (or, with no_hqr_fallback, BQRRP_ENUMERIC) is exercised deterministically. */
    int debug_flags;
    /* bqrrp_factor_dist only.  BQRRP_DIST_SHARD_PANEL: the panel's rows are split over min(G, h/k) ranks (the
     * k x k factors replicated from all-reduced Gram matrices; SURVEY §8(e) phase 2 item 3) instead of being
     * factored by the panel's owner.  Off (default), the result is bitwise the one-GPU bqrrp_factor's. */
    int dist_flags;
    /* One-GPU lookahead schedule of panel i+1: 0 (default) = after the bulk trailing GEMM of
     * iteration i, in place (Alg. 1 order; the next pivot selection overlaps the bulk); 1 = factored from a
     * gathered copy of its columns WHILE the bulk runs (measured slower on B200: the panel and the bulk contend
     * for SMs and the next panel's columns are updated twice).  The result is bitwise the same. */
    int panel_lookahead;
    /* One-GPU lookahead: SMs of the bulk trailing GEMM.  0 (default) = auto: an iteration whose
     * bulk GEMM is estimated shorter than the latency-bound chain it overlaps (the sample update and the next pivot
     * selection) runs it on a green-context partition leaving 32 SMs to that chain, the others on the whole device;
     * > 0 = every bulk GEMM on a partition of about that many SMs (rounded to the driver's granularity, 8 on
     * sm_100); -1 = always the whole device (the round-1 schedule).  No partition support in the driver = whole
     * device.  The result is bitwise the same for every value (fixed tiles, no split-K). */
    int bulk_sms;
    /* One-GPU lookahead: 0 (default) = K-SQR pipelined with K-LU (left-looking Householder QR of
     * each 32-column block of sketch columns as soon as K-LU has fixed its pivots, on a third stream); 1 = the
     * recursive K-SQR after K-LU (the round-1 order).  R_sk agrees to rounding (different operation order). */
    int no_sqr_pipeline;
    /* One-GPU lookahead with the K-SQR pipeline: 1 = K-LU as a right-looking blocked LU with a one-block lookahead
     * when the sketch transpose fits the register leaf (w <= 16384; each leaf waits only for its own block's update,
     * the wide trailing update runs on a fourth stream); 0 (default) = the recursive K-LU.  Measured no faster
     * (C2 369 vs 361 ms: the rank-16/32 trailing updates re-stream the whole w x d block from HBM at every leaf,
     * DESIGN.md §7.2).  Same pivot decisions (GETF2's); the factors differ by rounding. */
    int lu_lookahead;
    /* K-LU register leaf (w <= 16384): the largest cluster preferred before going to more rows per thread; 0 = the
     * default 16 (fewest rows per thread); 8 / 4 = smaller clusters (an 8-CTA cluster of full-SM CTAs still fits
     * the SM groups the bulk GEMM's partition leaves free; measured neutral at C2, 8192^2, 16384^2).
     * Pivots and factors are identical. */
    int lu_leaf_cluster;
    /* With the K-SQR pipeline: 0 (default) = for d <= 1024, each block's T merge (T(0:c, b) = -T_c (V_c^T V_b) T_bb,
     * three GEMMs) on a fifth stream, overlapping the next block's V^T B product (larger d: on the pipeline's own
     * stream, measured better at C3); 1 = always on the pipeline's own stream.  Identical results (same GEMMs, same
     * order per element). */
    int no_sqr_merge_stream;
    /* K-LU cooperative grid leaf (sketch transposes taller than the cluster leaves hold, w > ~25k): at most this many
     * CTAs.  0 (default) = per iteration in the lookahead: 32 when the bulk GEMM is estimated longer than the pivot
     * selection it overlaps (fewer CTAs hold more rows each, with narrower leaves, and the other SMs stay with the
     * bulk: C3 -0.9 %), else one per SM.  Same pivots, bitwise the same factorization. */
    int lu_grid_ctas;
} bqrrp_options;
#define BQRRP_DEBUG_FORCE_BREAKDOWN 1
#define BQRRP_DIST_SHARD_PANEL 1

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

/* The a3 column move on an explicit touched set (the kernels bqrrp_factor runs, exposed to time them alone):
 * X(:, tq[t]) <- X_old(:, tsrc[t]) for t < nt (device int32 0-based positions; {tq} = {tsrc} as sets, every
 * source read before any destination is written, through scratch from the library pool).  Asynchronous; the
 * host value nt is copied to the device on `stream` (pinned source not required: nt is staged). */
int bqrrp_debug_permute_touched(int64_t rows, double* X, int64_t ldx, int64_t nt, const int* tq, const int* tsrc,
                                void* stream);

/* The panel's k x k building blocks (Alg. 3), device, column-major:
 * bqrrp_debug_potrf: lower Cholesky factor of the SPD n x n G in place (upper triangle zeroed); BQRRP_ENUMERIC
 * on a non-positive pivot (the CholQR breakdown the HQR fallback catches).
 * bqrrp_debug_recon_lu: the Householder reconstruction's sign-choosing LU (BD2015): Wr (k x k, ld k) =
 * L \ U of Qtop C^{-T} - diag(S) with S_j = -sgn of the running pivot (Z20), C lower k x k (ld k). */
int bqrrp_debug_potrf(int64_t n, double* G, int64_t ldg, void* stream);
int bqrrp_debug_recon_lu(int64_t k, const double* Qtop, int64_t ldq, const double* C, double* Wr, double* S,
                         void* stream);

/* Panel: CholQR(passes) + Householder reconstruction (passes 1..4) or Householder QR (passes 0) of P (h x k, ld) preconditioned by Rsk11 (k x k
 * upper, ld k), written in GEQP3 format in place (R11 on/above, V below) with tau (k), plus the
 * compact-WY update of the trailing C (h x t, ld) that follows P in memory (t may be 0). */
int bqrrp_debug_panel(int64_t h, int64_t k, int64_t t, double* P, int64_t ld, const double* Rsk11, double* tau,
                      int cholqr_passes, void* stream);

/* ---- K-NORM: HBM-bound norm kernels of the pivot-quality / verification path ----
 * Reductions run in a fixed order (bitwise reproducible, independent of the launch grid); sums of squares
 * are formed in fp64, and a column whose sum over- or underflows is recomputed scaled by its largest
 * magnitude.  Asynchronous on `stream`. */

/* norms[j] = ||A(:, j)||_2 for j < n (A device m x n, lda >= max(1, m); norms device, n doubles).  Used for
 * the invariant ||R(0:j+1, j)||_2 = ||A(:, J(j))||_2 of a GEQP3 output (Q orthogonal). */
int bqrrp_column_norms(int64_t m, int64_t n, const double* A, int64_t lda, double* norms, void* stream);

/* out[i] = ||R(i:mn, i:n)||_F for i < mn = min(m, n), R the upper trapezoid of the device m x n matrix (entries
 * below the diagonal are ignored, so a GEQP3 output with its reflectors can be passed as is) — the paper's first
 * pivot-quality metric (the residual norm of the rank-i approximation Q(:, :i) R(:i, :)).
 * workspace: device scratch of >= bqrrp_trailing_norms_workspace bytes, or NULL (library pool; -7 if too small). */
int bqrrp_trailing_norms(int64_t m, int64_t n, const double* R, int64_t ldr, double* out, void* workspace,
                         size_t ws_bytes, void* stream);
int bqrrp_trailing_norms_workspace(int64_t m, int64_t n, size_t* bytes);

/* ---- multi-GPU -----------------------------------------------------------
 * One process per GPU.  A is distributed 1-D block-cyclically over column POSITIONS: position p (0-based) lives on
 * rank (p / nb) mod G, nb = opts->dist_nb (default b; nb must be a multiple of b, so each panel lives on one rank),
 * as local column (p / (nb G)) nb + p mod nb of that rank's A_local.  Pivoted columns move to the rank owning the
 * position they are assigned.  The collectives (P:1099-1165 distributed analogue): an
 * all-gather of the sketch rows (a1, and after every sample update), the column all-to-all-v of the touched set
 * (a3), a broadcast of the panel's V, T, tau (a4) and of R11 (a6), plus one 3-double all-reduce of flags per
 * iteration.  They run on NCCL (bqrrp_comm_init) or on a caller transport (bqrrp_comm_init_transport). */

/* Writes the 128-byte ncclUniqueId of a new NCCL clique into id_out (rank 0; the caller broadcasts it, e.g. with
 * torch.distributed).  NCCL is the process's libnccl.so.2 (dlopen'ed; normally the one torch loaded).
 * BQRRP_ENCCL if NCCL is unavailable. */
int bqrrp_nccl_unique_id(void* id_out);
/* Joins the clique as `rank` of `nranks` on the current CUDA device (collective: every rank calls it).  *comm_out
 * is an opaque handle owned by the caller until bqrrp_comm_destroy.  BQRRP_ENCCL on NCCL failure. */
int bqrrp_comm_init(const void* nccl_unique_id, int rank, int nranks, void** comm_out);
/* Caller-supplied transport (e.g. torch.distributed over gloo in tests).  Every callback gets device buffers and
 * the stream (already synchronised by the library) and must have moved the bytes when it returns 0:
 *   allreduce_sum_f64: buf <- sum over ranks (count doubles);  allgather: recv = nranks blocks of `bytes`, rank
 *   order;  broadcast: `bytes` from root;  alltoallv: per peer byte counts / displacements (nranks entries each,
 *   the own entry is 0).  Every callback is collective: all ranks call it in the same order, also with zero counts. */
typedef struct bqrrp_transport {
    void* ctx;
    int rank, nranks;
    int (*allreduce_sum_f64)(void* ctx, double* buf, size_t count, void* stream);
    int (*allgather)(void* ctx, const void* send, void* recv, size_t bytes, void* stream);
    int (*broadcast)(void* ctx, void* buf, size_t bytes, int root, void* stream);
    int (*alltoallv)(void* ctx, const void* send, const size_t* send_bytes, const size_t* send_displs, void* recv,
                     const size_t* recv_bytes, const size_t* recv_displs, void* stream);
} bqrrp_transport;
int bqrrp_comm_init_transport(const bqrrp_transport* transport, void** comm_out);
/* Releases a handle of bqrrp_comm_init / _init_transport (NULL is a no-op). */
int bqrrp_comm_destroy(void* comm);

/* Number of columns rank `rank` holds of an n-column matrix in the layout above (host only). */
int bqrrp_dist_local_columns(int64_t n, int64_t nb, int nranks, int rank, int64_t* n_local);
/* Device workspace bytes of bqrrp_factor_dist for the largest rank share (host only). */
int bqrrp_workspace_query_dist(int64_t m, int64_t n, int64_t b, int64_t d, int nranks, int64_t dist_nb, size_t* bytes);
/* The a3 exchange plan of one rank (host only; exposed for tests): the nt touched positions move p[t] -> q[t]
 * (0-based).  Slots are taken in ascending q.  send_idx: this rank's local source columns sent to other ranks,
 * grouped by destination rank (send_counts[r] each); recv_idx: local destination columns received, grouped by
 * source rank (recv_counts[r]); local_src -> local_dst: moves within this rank (*n_local_moves).  Output arrays
 * have room for nt entries (counts: nranks). */
int bqrrp_dist_exchange_plan(int64_t n, int64_t nb, int nranks, int rank, int64_t nt, const int64_t* q,
                             const int64_t* p, int32_t* send_idx, int64_t* send_counts, int32_t* recv_idx,
                             int64_t* recv_counts, int32_t* local_src, int32_t* local_dst, int64_t* n_local_moves);

/*
 * Distributed BQRRP (collective: every rank of `comm` calls it with the same m, n, b, d, seed, opts).
 *   A_local   device, m x n_local (bqrrp_dist_local_columns), lda_local >= max(1, m): this rank's columns in the
 *             layout above; overwritten with the same GEQP3 content as bqrrp_factor's A in those columns
 *   tau, J    device, replicated on every rank (min(m, n) doubles; n int64, one-based gather)
 *   rank      host out: l, identical on every rank
 *   workspace device (>= bqrrp_workspace_query_dist bytes) or NULL (library pool)
 * Returns as bqrrp_factor_ex (+ BQRRP_ENCCL; -11 comm NULL, -15 dist_nb not a multiple of b).  Synchronises the
 * stream a few times per iteration (the block rank k, the touched set for the exchange plan, the flags).  With
 * dist_flags = 0 the output is bitwise bqrrp_factor_ex's on the whole matrix (tests/test_dist.py).
 */
int bqrrp_factor_dist(int64_t m, int64_t n, double* A_local, int64_t lda_local, int64_t b, int64_t d, uint64_t seed,
                      double* tau, int64_t* J, int64_t* rank, void* comm, void* workspace, size_t ws_bytes,
                      void* stream, const bqrrp_options* opts);

/* Number of CUDA kernels this library has launched in the calling process (all threads). */
unsigned long long bqrrp_launch_count(void);
/* Panels re-factored by Householder QR after a CholQR breakdown in the last bqrrp_factor* call on this
 * thread (the multi-GPU entry counts the panels factored on this rank). */
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
