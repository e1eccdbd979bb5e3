/*
 * bqrrp_oracle.c — plain, slow, obviously-correct CPU oracle of BQRRP
 * (Melnichenko et al., arXiv 2507.00976, "Blocked QR with Randomization and Pivoting").
 *
 * TEST INFRASTRUCTURE ONLY.  Nothing on the product path may include, link or call this
 * file: only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference
 * legs use it.  It shares no code, header, table or constant generator with the CUDA path
 * (paper_2507_00976_b200/csrc); the two are separate implementations of the readings written
 * down in DESIGN.md.
 *
 * Conventions
 *   - "P:n" cites line n of the paper's LaTeX source; the section / algorithm step
 *     label is named beside it.  Readings where the paper is silent are DESIGN.md §3 "Z*" ids.
 *   - All matrices column-major, fp64.  Compiled with -ffp-contract=off (no FMA contraction)
 *     so every expression below rounds exactly as written.
 *   - Sums run in ascending index order.  OpenMP is used only over independent output columns,
 *     so results do not depend on the thread count.
 *   - The Householder / LU kernels are the unblocked textbook ones (reflector at a time,
 *     DGETF2-style), deliberately: no blocking, fusion or reordering.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

#define IDX(i, j, ld) ((size_t)(i) + (size_t)(j) * (size_t)(ld))

/* ========================================================================================
 * 1. Counter-based Gaussian generator (DESIGN.md §2 "RNG spec").
 *    The paper's software draws S from Random123 counter-based generators (§1.4
 *    "Our software"); S has iid N(0,1) entries (P:476 step bqrrp:sample; §3.2,
 *    variance-one reading Z3).  Entry (i,j) of S is a pure function of (seed, stream, i, j).
 * ======================================================================================== */

/* Philox4x32-10 (Salmon, Moraes, Dror, Shaw, SC'11) — the Random123 generator. */
void oracle_philox4x32_10(const uint32_t ctr_in[4], const uint32_t key_in[2], uint32_t out[4])
{
    uint32_t c0 = ctr_in[0], c1 = ctr_in[1], c2 = ctr_in[2], c3 = ctr_in[3];
    uint32_t k0 = key_in[0], k1 = key_in[1];
    for (int round = 0; round < 10; ++round) {
        if (round > 0) {
            k0 += 0x9E3779B9u;
            k1 += 0xBB67AE85u;
        }
        uint64_t p0 = (uint64_t)0xD2511F53u * (uint64_t)c0;
        uint64_t p1 = (uint64_t)0xCD9E8D57u * (uint64_t)c2;
        uint32_t hi0 = (uint32_t)(p0 >> 32), lo0 = (uint32_t)p0;
        uint32_t hi1 = (uint32_t)(p1 >> 32), lo1 = (uint32_t)p1;
        uint32_t n0 = hi1 ^ c1 ^ k0;
        uint32_t n1 = lo1;
        uint32_t n2 = hi0 ^ c3 ^ k1;
        uint32_t n3 = lo0;
        c0 = n0; c1 = n1; c2 = n2; c3 = n3;
    }
    out[0] = c0; out[1] = c1; out[2] = c2; out[3] = c3;
}

/* Natural log for x in (0, 1] (normal numbers), from + - * / only:
 *   x = 2^e * f, f in [sqrt(2)/2, sqrt(2));  log f = 2 atanh(s), s = (f-1)/(f+1)
 *   log f = 2s + 2s * (s^2 * P(s^2)),  P = sum_{k=1..12} s^(2(k-1)) / (2k+1)   (Horner)
 *   log x = e*ln2_hi + (e*ln2_lo + log f)                                        */
double oracle_log(double x)
{
    static const double inv_odd[12] = {
        0x1.5555555555555p-2, 0x1.999999999999ap-3, 0x1.2492492492492p-3, 0x1.c71c71c71c71cp-4,
        0x1.745d1745d1746p-4, 0x1.3b13b13b13b14p-4, 0x1.1111111111111p-4, 0x1.e1e1e1e1e1e1ep-5,
        0x1.af286bca1af28p-5, 0x1.8618618618618p-5, 0x1.642c8590b2164p-5, 0x1.47ae147ae147bp-5};
    const double ln2_hi = 0x1.62e42fee00000p-1, ln2_lo = 0x1.a39ef35793c76p-33;
    const double sqrt2 = 0x1.6a09e667f3bcdp+0;
    uint64_t bits;
    memcpy(&bits, &x, 8);
    int e = (int)((bits >> 52) & 0x7ff) - 1023;
    uint64_t fb = (bits & 0x000fffffffffffffull) | 0x3ff0000000000000ull; /* f in [1,2) */
    double f;
    memcpy(&f, &fb, 8);
    if (f > sqrt2) {
        f = f * 0.5; /* exact */
        e = e + 1;
    }
    double s = (f - 1.0) / (f + 1.0);
    double s2 = s * s;
    double p = inv_odd[11];
    for (int k = 10; k >= 0; --k) p = p * s2 + inv_odd[k];
    double logf_ = 2.0 * s + (2.0 * s) * (s2 * p);
    double ed = (double)e;
    return ed * ln2_hi + (ed * ln2_lo + logf_);
}

/* sin(x), cos(x) for x in [0, pi/4] by Taylor polynomials (Horner in x^2). */
static double taylor_sin(double x)
{
    static const double c[9] = {-0x1.5555555555555p-3, 0x1.1111111111111p-7, -0x1.a01a01a01a01ap-13,
                                0x1.71de3a556c734p-19, -0x1.ae64567f544e4p-26, 0x1.6124613a86d09p-33,
                                -0x1.ae7f3e733b81fp-41, 0x1.952c77030ad4ap-49, -0x1.2f49b46814157p-57};
    double x2 = x * x;
    double p = c[8];
    for (int k = 7; k >= 0; --k) p = p * x2 + c[k];
    return x + x * (x2 * p);
}
static double taylor_cos(double x)
{
    static const double c[9] = {-0x1.0000000000000p-1, 0x1.5555555555555p-5, -0x1.6c16c16c16c17p-10,
                                0x1.a01a01a01a01ap-16, -0x1.27e4fb7789f5cp-22, 0x1.1eed8eff8d898p-29,
                                -0x1.93974a8c07c9dp-37, 0x1.ae7f3e733b81fp-45, -0x1.6827863b97d97p-53};
    double x2 = x * x;
    double p = c[8];
    for (int k = 7; k >= 0; --k) p = p * x2 + c[k];
    return 1.0 + x2 * p;
}

/* cos(2*pi*u) for u in [0,1): exact quadrant reduction t = 4u = q + r (q = 0..3, r in [0,1)),
 * then cos(pi/2 (q+r)) from sin/cos(pi/2 * r) with r folded to [0, 1/2].                  */
double oracle_cos2pi(double u)
{
    const double half_pi = 0x1.921fb54442d18p+0;
    double t = 4.0 * u;
    int q = (int)t; /* 0..3 */
    double r = t - (double)q;
    double cr, sr; /* cos(pi/2 r), sin(pi/2 r) */
    if (r <= 0.5) {
        double x = half_pi * r;
        cr = taylor_cos(x);
        sr = taylor_sin(x);
    } else {
        double x = half_pi * (1.0 - r);
        cr = taylor_sin(x);
        sr = taylor_cos(x);
    }
    switch (q & 3) {
    case 0: return cr;
    case 1: return -sr;
    case 2: return -cr;
    default: return sr;
    }
}

/* One standard normal: Box-Muller on one Philox block.
 *   key = (lo32 seed, hi32 seed), ctr = (i, lo32 j, hi32 j, stream)
 *   u1 = ((x0:x1 >> 12) + 0.5) * 2^-52  in (0,1);   u2 = (x2:x3 >> 11) * 2^-53  in [0,1)
 *   z  = sqrt(-2 log u1) * cos(2 pi u2)                                                   */
double oracle_gauss(uint64_t seed, uint32_t stream, uint64_t i, uint64_t j)
{
    uint32_t key[2] = {(uint32_t)seed, (uint32_t)(seed >> 32)};
    uint32_t ctr[4] = {(uint32_t)i, (uint32_t)j, (uint32_t)(j >> 32), stream};
    uint32_t x[4];
    oracle_philox4x32_10(ctr, key, x);
    uint64_t a = ((uint64_t)x[0] << 32) | x[1];
    uint64_t c = ((uint64_t)x[2] << 32) | x[3];
    double u1 = ((double)(a >> 12) + 0.5) * 0x1p-52;
    double u2 = (double)(c >> 11) * 0x1p-53;
    return sqrt(-2.0 * oracle_log(u1)) * oracle_cos2pi(u2);
}

/* S (d x m, col-major, ld = d): S(i,j) = gauss(seed, 0, i, j).  P:476 (bqrrp:sample); Z2: d x m. */
void oracle_sketch_operator(int64_t d, int64_t m, uint64_t seed, double *S)
{
#pragma omp parallel for schedule(static)
    for (int64_t j = 0; j < m; ++j)
        for (int64_t i = 0; i < d; ++i) S[IDX(i, j, d)] = oracle_gauss(seed, 0, (uint64_t)i, (uint64_t)j);
}

/* Sketch, stored transposed: MskT (n x d, ld = n) = (S A)^T, i.e.
 *   MskT(j,i) = sum_{l=0..m-1 ascending} A(l,j) * S(i,l)
 * P:478 (bqrrp:sketching "M_sk = S M"), P:969-975 (§3.2).                                   */
void oracle_sketch(int64_t m, int64_t n, const double *A, int64_t lda, int64_t d, uint64_t seed,
                   double *MskT /* n x d, ld n */)
{
    /* St = S^T (m x d) so that row i of S is contiguous; same products, same order. */
    double *St = (double *)malloc(sizeof(double) * (size_t)(d > 0 ? d : 1) * (size_t)(m > 0 ? m : 1));
#pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < d; ++i)
        for (int64_t l = 0; l < m; ++l) St[IDX(l, i, m)] = oracle_gauss(seed, 0, (uint64_t)i, (uint64_t)l);
#pragma omp parallel for schedule(static)
    for (int64_t j = 0; j < n; ++j)
        for (int64_t i = 0; i < d; ++i) {
            double acc = 0.0;
            for (int64_t l = 0; l < m; ++l) acc += A[IDX(l, j, lda)] * St[IDX(l, i, m)];
            MskT[IDX(j, i, n)] = acc;
        }
    free(St);
}

/* ========================================================================================
 * 2. Pivot selection: Alg. 2 "Practical wide QRCP", LU-based.
 * ======================================================================================== */

/* DGETF2-style LU with partial pivoting of L (p x q, ld), in place.  ipiv[j] (1-based,
 * j < min(p,q)): row j was interchanged with row ipiv[j]-1 ("row i of the input
 * matrix was interchanged with row J_lu(i)").  Pivot = first index of max |L(r,j)|, r >= j
 * (Z19, IDAMAX).  Zero pivot column: no swap, no scaling (Z18).  margin[j] (optional) =
 * (|top1| - |top2|) / |top1| over the candidates of column j (parity aid). */
void oracle_getf2(int64_t p, int64_t q, double *L, int64_t ld, int64_t *ipiv, double *margin)
{
    int64_t kmin = p < q ? p : q;
    for (int64_t j = 0; j < kmin; ++j) {
        int64_t piv = j;
        double top1 = fabs(L[IDX(j, j, ld)]), top2 = -1.0;
        for (int64_t r = j + 1; r < p; ++r) {
            double v = fabs(L[IDX(r, j, ld)]);
            if (v > top1) {
                top2 = top1;
                top1 = v;
                piv = r;
            } else if (v > top2) {
                top2 = v;
            }
        }
        if (margin) margin[j] = (top1 > 0.0) ? (top2 < 0.0 ? 1.0 : (top1 - top2) / top1) : 0.0;
        ipiv[j] = piv + 1;
        if (L[IDX(piv, j, ld)] == 0.0) continue; /* Z18 */
        if (piv != j)
            for (int64_t c = 0; c < q; ++c) {
                double t = L[IDX(j, c, ld)];
                L[IDX(j, c, ld)] = L[IDX(piv, c, ld)];
                L[IDX(piv, c, ld)] = t;
            }
        double pv = L[IDX(j, j, ld)];
        for (int64_t r = j + 1; r < p; ++r) L[IDX(r, j, ld)] = L[IDX(r, j, ld)] / pv;
#pragma omp parallel for schedule(static) if ((p - j) * (q - j) > 65536)
        for (int64_t c = j + 1; c < q; ++c) {
            double ujc = L[IDX(j, c, ld)];
            for (int64_t r = j + 1; r < p; ++r) L[IDX(r, c, ld)] = L[IDX(r, c, ld)] - L[IDX(r, j, ld)] * ujc;
        }
    }
}

/* piv_transform ("Permutation formats"): J_qr = (1..w); for j < len(J_lu):
 * swap J_qr(j) with J_qr(J_lu(j) - 1)   (Z5: iterate over the min(w,d) LU pivots).        */
void oracle_piv_transform(int64_t w, int64_t nlu, const int64_t *Jlu, int64_t *Jqr)
{
    for (int64_t q = 0; q < w; ++q) Jqr[q] = q + 1;
    for (int64_t j = 0; j < nlu; ++j) {
        int64_t t = Jqr[j];
        Jqr[j] = Jqr[Jlu[j] - 1];
        Jqr[Jlu[j] - 1] = t;
    }
}

/* Gather semantics of col_perm (Alg. 5 P:1117-1135 with Z6's J(i)-1):
 * new column q = old column Jqr(q) - 1, for q < w, over `rows` rows.                         */
void oracle_col_gather(int64_t rows, int64_t w, double *M, int64_t ld, const int64_t *Jqr)
{
    double *cpy = (double *)malloc(sizeof(double) * (size_t)(rows > 0 ? rows : 1) * (size_t)(w > 0 ? w : 1));
    for (int64_t q = 0; q < w; ++q) memcpy(cpy + (size_t)q * rows, M + (size_t)q * ld, sizeof(double) * rows);
    for (int64_t q = 0; q < w; ++q)
        memcpy(M + (size_t)q * ld, cpy + (size_t)(Jqr[q] - 1) * rows, sizeof(double) * rows);
    free(cpy);
}

/* Same gather on the ROWS of a column-major matrix (the transposed sketch's rows are the
 * sketch's columns, P:568 step wide_qrcp:permute).                                           */
void oracle_row_gather(int64_t w, int64_t cols, double *M, int64_t ld, const int64_t *Jqr)
{
    double *cpy = (double *)malloc(sizeof(double) * (size_t)(w > 0 ? w : 1));
    for (int64_t c = 0; c < cols; ++c) {
        for (int64_t q = 0; q < w; ++q) cpy[q] = M[IDX(q, c, ld)];
        for (int64_t q = 0; q < w; ++q) M[IDX(q, c, ld)] = cpy[Jqr[q] - 1];
    }
    free(cpy);
}

/* Gather of an integer vector (step bqrrp:update_j). */
void oracle_vec_gather(int64_t w, int64_t *J, const int64_t *Jqr)
{
    int64_t *cpy = (int64_t *)malloc(sizeof(int64_t) * (size_t)(w > 0 ? w : 1));
    memcpy(cpy, J, sizeof(int64_t) * w);
    for (int64_t q = 0; q < w; ++q) J[q] = cpy[Jqr[q] - 1];
    free(cpy);
}

/* ========================================================================================
 * 3. Householder reflectors, convention H (Z9/Z20): the output format is GEQP3's
 *    (P:253-277): H = I - tau v v^T, v(0) = 1 implicit, beta on the diagonal of R.
 *      alpha = x0, ||x|| = sqrt(ascending sum of squares)
 *      ||x|| == 0: tau = 0, beta = 0, v = e1
 *      else beta = -sgn(alpha) ||x|| (sgn(a) = a >= 0 ? +1 : -1), v_q = x_q/(alpha-beta),
 *           tau = (beta - alpha)/beta         (no "zero tail => tau = 0" shortcut)
 * ======================================================================================== */

/* x (length len, stride 1) is overwritten: x[0] = beta, x[1:] = v[1:]. Returns tau. */
double oracle_house_vec(int64_t len, double *x)
{
    double ss = 0.0;
    for (int64_t q = 0; q < len; ++q) ss += x[q] * x[q];
    double nrm = sqrt(ss);
    if (nrm == 0.0) return 0.0; /* x is all zeros: beta = 0, v = e1 */
    double alpha = x[0];
    double beta = (alpha >= 0.0) ? -nrm : nrm;
    double denom = alpha - beta;
    for (int64_t q = 1; q < len; ++q) x[q] = x[q] / denom;
    x[0] = beta;
    return (beta - alpha) / beta;
}

/* y <- (I - tau v v^T) y, v(0) = 1 implicit, v(1:) = vtail.  w = y0 + sum_{q>=1} v_q y_q. */
static void apply_reflector(int64_t len, const double *vtail_minus1 /* v[q] at q>=1 */, double tau, double *y)
{
    if (tau == 0.0) return;
    double w = y[0];
    for (int64_t q = 1; q < len; ++q) w += vtail_minus1[q] * y[q];
    double tw = tau * w;
    y[0] = y[0] - tw;
    for (int64_t q = 1; q < len; ++q) y[q] = y[q] - tw * vtail_minus1[q];
}

/* Unblocked Householder QR (GEQRF semantics, convention H) of the leading `kref` columns of
 * M (p x q, ld): reflector j is formed from column j rows j..p-1, applied to columns j+1..kref-1
 * one reflector at a time; then all kref reflectors H_1 ... H_kref (H_1 first) are applied to
 * the trailing columns kref..q-1 (P:498-511 steps bqrrp:qr_tall, bqrrp:apply_q_*; P:781-801
 * "apply_trans_q": C <- Q^T C).  Each trailing column is independent (OpenMP over columns). */
void oracle_house_qr(int64_t p, int64_t q, double *M, int64_t ld, int64_t kref, double *tau)
{
    for (int64_t j = 0; j < kref; ++j) {
        tau[j] = oracle_house_vec(p - j, M + IDX(j, j, ld));
#pragma omp parallel for schedule(static) if ((p - j) * (kref - j) > 65536)
        for (int64_t c = j + 1; c < kref; ++c) apply_reflector(p - j, M + IDX(j, j, ld), tau[j], M + IDX(j, c, ld));
    }
#pragma omp parallel for schedule(dynamic, 4)
    for (int64_t c = kref; c < q; ++c)
        for (int64_t j = 0; j < kref; ++j) apply_reflector(p - j, M + IDX(j, j, ld), tau[j], M + IDX(j, c, ld));
}

/* ========================================================================================
 * 4. tri_rank (P:490-491 step bqrrp:rank_est; §2.2): the paper defers the threshold
 *    to [MBM2024].  Reading Z10/Z11: k = largest k' <= kmax with |Rsk(j,j)| > tol for all
 *    j < k', tol = rank_tol * ref, ref = |R_sk^(0)(0,0)| (global, from iteration 0).
 * ======================================================================================== */
int64_t oracle_tri_rank(int64_t kmax, const double *diag, int64_t dstride, double tol)
{
    int64_t k = 0;
    while (k < kmax && fabs(diag[k * dstride]) > tol) ++k;
    return k;
}

/* ========================================================================================
 * 5. Sketch update (P:517 step bqrrp:update_sample; §3.7), transposed layout:
 *      X = R_sk11 R11^{-1}   (right upper-triangular solve, column by column)
 *      MskT(q, 0:b) -= (X R11^{-1}... ) i.e. MskT(q,i) -= sum_{l<b} X(i,l) * R12(l, q)
 *      MskT(q, b:d) unchanged (= R_sk22^T, already in place).
 *    Rsk11 (b x b, ld_rs), R11 (b x b, ld_r), R12 (b x t, ld_r), MskT rows (t x d, ld_m).
 * ======================================================================================== */
void oracle_sample_update(int64_t b, int64_t t, const double *Rsk11, int64_t ld_rs, const double *R11,
                          int64_t ld_r, const double *R12, double *MskT_tail, int64_t ld_m)
{
    double *X = (double *)calloc((size_t)(b > 0 ? b * b : 1), sizeof(double));
    /* X(:,j) = (Rsk11(:,j) - sum_{l<j} X(:,l) R11(l,j)) / R11(j,j) */
    for (int64_t j = 0; j < b; ++j)
        for (int64_t i = 0; i < b; ++i) {
            double acc = Rsk11[IDX(i, j, ld_rs)];
            for (int64_t l = 0; l < j; ++l) acc = acc - X[IDX(i, l, b)] * R11[IDX(l, j, ld_r)];
            X[IDX(i, j, b)] = acc / R11[IDX(j, j, ld_r)];
        }
    for (int64_t j = 0; j < b; ++j) /* explicitly upper triangular (§3.7 "we explicitly zero out") */
        for (int64_t i = j + 1; i < b; ++i) X[IDX(i, j, b)] = 0.0;
#pragma omp parallel for schedule(static)
    for (int64_t q = 0; q < t; ++q)
        for (int64_t i = 0; i < b; ++i) {
            double acc = 0.0;
            for (int64_t l = 0; l < b; ++l) acc += X[IDX(i, l, b)] * R12[IDX(l, q, ld_r)];
            MskT_tail[IDX(q, i, ld_m)] = MskT_tail[IDX(q, i, ld_m)] - acc;
        }
    free(X);
}

/* ========================================================================================
 * 6. The driver: Alg. 1 step by step with the in-place recipe of §3
 *    (P:925-1080).  Returns 0 on success, -i for an illegal i-th argument.
 *    A (m x n, lda) is overwritten in GEQP3 format; tau (min(m,n)); J (n, 1-based
 *    gather); *rank = ell.  Optional diagnostics:
 *      MskT_out (n x d, ld n): the sketch state on return (used by the closed-form pin);
 *      min_margin: smallest LU pivot margin seen (parity aid);
 *      ks: per-iteration block ranks (length >= ceil(min(m,n)/b));
 *      max_iters >= 0 stops after that many iterations WITHOUT the final zeroing (state
 *      inspection; *rank = -1 then).
 * ======================================================================================== */
int oracle_bqrrp(int64_t m, int64_t n, double *A, int64_t lda, int64_t b, int64_t d, uint64_t seed, double rank_tol,
                 double *tau, int64_t *J, int64_t *rank, double *MskT_out, double *min_margin, int64_t *ks,
                 int64_t max_iters, int nthreads)
{
    /* O0 validation (LAPACK-style -i for the i-th argument) */
    if (m < 0) return -1;
    if (n < 0) return -2;
    if (!A && m * n > 0) return -3;
    if (lda < (m > 1 ? m : 1)) return -4;
    if (b < 1) return -5;
    if (d < b || (m > 0 && d > m)) return -6;
    if (!(rank_tol >= 0.0)) return -8;
#ifdef _OPENMP
    if (nthreads > 0) omp_set_num_threads(nthreads);
#else
    (void)nthreads;
#endif
    int64_t mn = m < n ? m : n;
    if (min_margin) *min_margin = 1.0;
    for (int64_t j = 0; j < mn; ++j) tau[j] = 0.0;
    for (int64_t j = 0; j < n; ++j) J[j] = j + 1; /* O2, P:477 step bqrrp:alloc "J = 1:(n+1)" */
    if (m == 0 || n == 0) {
        *rank = 0;
        return 0;
    }

    /* O1: sketch once ("uses randomness only once") */
    double *MskT = (double *)malloc(sizeof(double) * (size_t)n * (size_t)d);
    oracle_sketch(m, n, A, lda, d, seed, MskT);

    double *L = (double *)malloc(sizeof(double) * (size_t)n * (size_t)d);
    double *W = (double *)malloc(sizeof(double) * (size_t)n * (size_t)d);
    double *tau_sk = (double *)malloc(sizeof(double) * (size_t)d);
    int64_t *ipiv = (int64_t *)malloc(sizeof(int64_t) * (size_t)d);
    int64_t *Jqr = (int64_t *)malloc(sizeof(int64_t) * (size_t)n);
    double *margin = (double *)malloc(sizeof(double) * (size_t)d);
    double ref = 0.0, tol = 0.0;
    int64_t ell = -1;

    for (int64_t i = 0;; ++i) {
        int64_t s = i * b;
        if (s >= mn) { /* Z1/Z17: loop while s < min(m,n) */
            ell = mn;
            break;
        }
        if (max_iters >= 0 && i >= max_iters) break;
        int64_t c = (s + b < n) ? s + b : n; /* P:481-485 (bqrrp:block_partitions) */
        int64_t r = (s + b < m) ? s + b : m;
        int64_t w = n - s, h = m - s;
        int64_t kmax = b < w ? b : w;
        kmax = kmax < h ? kmax : h;

        /* (a) L = copy of the sketch transpose MskT(s:n, 0:d) (Alg. 2 step qrcp:transpose), GETF2 */
        for (int64_t col = 0; col < d; ++col) memcpy(L + (size_t)col * w, MskT + IDX(s, col, n), sizeof(double) * w);
        int64_t nlu = w < d ? w : d;
        oracle_getf2(w, d, L, w, ipiv, margin);
        if (min_margin)
            for (int64_t j = 0; j < nlu; ++j)
                if (margin[j] < *min_margin) *min_margin = margin[j];
        /* (b) J_qr = piv_transform(J_lu) (Alg. 2 step qrcp:piv_transform) */
        oracle_piv_transform(w, nlu, ipiv, Jqr);
        /* (c) permute the sketch's columns = rows of MskT(s:n,:) (Alg. 2 step wide_qrcp:permute) */
        oracle_row_gather(w, d, MskT + s, n, Jqr);
        /* (d) R_sk = R of Householder QR of Wsk = MskT(s:n,:)^T (d x w) (Alg. 2 step
         *     wide_qrcp:compute, GEQRF); store R_sk^T back into MskT(s:n,:) (§3.4) */
        for (int64_t q = 0; q < w; ++q)
            for (int64_t row = 0; row < d; ++row) W[IDX(row, q, d)] = MskT[IDX(s + q, row, n)];
        int64_t ksk = d < w ? d : w;
        oracle_house_qr(d, w, W, d, ksk, tau_sk);
        for (int64_t q = 0; q < w; ++q)
            for (int64_t row = 0; row < d; ++row) MskT[IDX(s + q, row, n)] = (row <= q) ? W[IDX(row, q, d)] : 0.0;
        /* (e) k = tri_rank(R_sk) (step bqrrp:rank_est) */
        if (i == 0) {
            ref = fabs(W[0]);
            tol = rank_tol * ref;
        }
        int64_t k = (ref == 0.0) ? 0 : oracle_tri_rank(kmax, W, d + 1, tol);
        if (ks) ks[i] = k;
        /* (f) permute all m rows of A(:, s:n) and J(s:n) (steps bqrrp:permute_r, permute_m,
         *     update_j merged; Z13/Z14: always the full permutation) */
        oracle_col_gather(m, w, A + IDX(0, s, lda), lda, Jqr);
        oracle_vec_gather(w, J + s, Jqr);
        /* (g) early exit: k == 0 or the pivoted column A(s:m, s) is all zeros (Z12) */
        int all_zero = 1;
        for (int64_t row = s; row < m; ++row)
            if (A[IDX(row, s, lda)] != 0.0) {
                all_zero = 0;
                break;
            }
        if (k == 0 || all_zero) {
            ell = s;
            break;
        }
        /* (h) Householder QR of the k-column panel A(s:m, s:s+k) and Q^T applied to the
         *     trailing A(s:m, s+k:n) (steps bqrrp:qr_tall, apply_q_1/2, update_R11, update_r12;
         *     Z15: panel columns k..bw are projected with the trailing columns) */
        oracle_house_qr(h, w, A + IDX(s, s, lda), lda, k, tau + s);
        /* (i) termination (step bqrrp:termination; Z16) */
        if (k < kmax || c == n || r == m) {
            ell = s + k;
            break;
        }
        /* (j) sketch update (step bqrrp:update_sample) */
        /*     R_sk11 = R_sk(0:b, 0:b), upper triangular, read from the QR output W (d x w) */
        double *Rsk11 = (double *)calloc((size_t)(b * b), sizeof(double));
        for (int64_t col = 0; col < b; ++col)
            for (int64_t row = 0; row <= col; ++row) Rsk11[IDX(row, col, b)] = W[IDX(row, col, d)];
        oracle_sample_update(b, n - c, Rsk11, b, A + IDX(s, s, lda), lda, A + IDX(s, c, lda), MskT + IDX(c, 0, n), n);
        free(Rsk11);
    }

    if (ell >= 0) {
        /* O4: tau(ell:) = 0, A(ell:m, ell:n) = 0 (Z16) */
        for (int64_t j = ell; j < mn; ++j) tau[j] = 0.0;
        for (int64_t col = ell; col < n; ++col)
            for (int64_t row = ell; row < m; ++row) A[IDX(row, col, lda)] = 0.0;
        *rank = ell;
    } else {
        *rank = -1;
    }
    if (MskT_out) memcpy(MskT_out, MskT, sizeof(double) * (size_t)n * (size_t)d);
    free(MskT); free(L); free(W); free(tau_sk); free(ipiv); free(Jqr); free(margin);
    return 0;
}
