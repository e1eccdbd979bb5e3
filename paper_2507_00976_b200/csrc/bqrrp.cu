// bqrrp.cu — the BQRRP driver (Alg. 1, in-place recipe §3) and the C ABI.
//
// One process-wide host loop per call.  Per block iteration i (s = i b, c = min(n, s+b),
// r = min(m, s+b), w = n-s, h = m-s, kmax = min(b, w, h), P:481-485 / DESIGN.md §4):
//   a2  L = MskT(s:n, :) (copy), K-LU pivots, touched set of J_qr, sketch rows permuted, K-SQR -> R_sk
//   a2  tri_rank -> k (device)                                     (step bqrrp:rank_est)
//   a3  A(:, s:n), J(s:n) gathered by J_qr (touched set only)      (steps permute_r/permute_m/update_j)
//       zero-column test of A(s:m, s)
//   --- one host read of {k, zero flag, non-finite flag, potrf info}: the loop's only sync ---
//   a4  CholQR2 + reconstruction -> V, T, tau, R11                 (step bqrrp:qr_tall, Alg. 3)
//   a5  compact-WY update of A(s:m, s+k:n) -> R12 and the next trailing matrix (apply_q_1/2)
//   a7  termination (step bqrrp:termination)
//   a6  sketch update MskT(c:n, 0:b) -= R12^T (R_sk11 R11^{-1})^T  (step bqrrp:update_sample)
#include <cstring>
#include <mutex>
#include <vector>
#include <string>

#include "../../include/bqrrp.h"
#include "blas.cuh"
#include "bqrrp_internal.cuh"


namespace bqrrp {

static thread_local std::string g_last_error;

cudaMemPool_t lib_pool()
{
    static std::mutex mu;
    static cudaMemPool_t pools[64] = {};
    int dev = 0;
    BQ_CUDA(cudaGetDevice(&dev));
    std::lock_guard<std::mutex> lk(mu);
    if (!pools[dev]) {
        cudaMemPoolProps props = {};
        props.allocType = cudaMemAllocationTypePinned;
        props.location.type = cudaMemLocationTypeDevice;
        props.location.id = dev;
        BQ_CUDA(cudaMemPoolCreate(&pools[dev], &props));
        uint64_t thr = UINT64_MAX;
        BQ_CUDA(cudaMemPoolSetAttribute(pools[dev], cudaMemPoolAttrReleaseThreshold, &thr));
    }
    return pools[dev];
}
thread_local long long g_panel_fallbacks = 0;
unsigned long long g_launches = 0;

// ----------------------------------------------------------------------------------- small kernels
__global__ void init_j_kernel(int64_t n, int64_t* J)
{
    for (int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j < n; j += (int64_t)gridDim.x * blockDim.x)
        J[j] = j + 1;
}

__global__ void nonfinite_kernel(int64_t rows, int64_t cols, const double* X, int64_t ldx, int* flags)
{
    int64_t total = rows * cols;
    bool bad = false;
    for (int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; idx < total; idx += (int64_t)gridDim.x * blockDim.x) {
        double v = X[idx % rows + (idx / rows) * ldx];
        if (!isfinite(v)) bad = true;
    }
    if (bad) flags[F_NONFINITE] = 1;
}

// k = tri_rank(R_sk) (reading Z10/Z11): ref = |R_sk^(0)(0,0)| set at i = 0; diag(R_sk)(j) =
// MskT(s+j, j).  Also arms the zero-column flag (cleared by zero_col_kernel).
__global__ void tri_rank_kernel(const double* MskT_s, int64_t ldm, int64_t kmax, int first, double rank_tol, double* ref,
                                int* flags)
{
    __shared__ int first_fail;
    if (threadIdx.x == 0) first_fail = (int)kmax;
    __syncthreads();
    const double r = first ? fabs(MskT_s[0]) : *ref;
    if (r > 0.0) {
        const double tol = rank_tol * r;
        for (int64_t j = threadIdx.x; j < kmax; j += blockDim.x)
            if (!(fabs(MskT_s[j + j * ldm]) > tol)) atomicMin(&first_fail, (int)j);
    } else if (threadIdx.x == 0) {
        first_fail = 0;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        if (first) *ref = r;
        flags[F_K] = first_fail;  // largest prefix with |R_sk(j,j)| > tol
        flags[F_ZERO_COL] = 1;
    }
}

__global__ void zero_col_kernel(int64_t h, const double* col, int* flags)
{
    bool nz = false;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < h; i += (int64_t)gridDim.x * blockDim.x)
        if (col[i] != 0.0) nz = true;
    if (__syncthreads_or(nz) && threadIdx.x == 0) flags[F_ZERO_COL] = 0;
}

// Rsk11(i, j) = R_sk(i, j) = MskT(s+j, i) for i <= j < k, 0 below (k x k, ld k).
__global__ void extract_rsk11_kernel(int64_t k, const double* MskT_s, int64_t ldm, double* R)
{
    int64_t total = k * k;
    for (int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; idx < total; idx += (int64_t)gridDim.x * blockDim.x) {
        int64_t i = idx % k, j = idx / k;
        R[idx] = (i <= j) ? MskT_s[j + i * ldm] : 0.0;
    }
}

__global__ void ipiv_to_i64_kernel(int64_t n, const int* in0, int64_t* out1)
{
    int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (j < n) out1[j] = (int64_t)in0[j] + 1;
}

// ----------------------------------------------------------------------------------- workspace
struct Layout {
    size_t persistent, temp, splitk, total;
};

static Layout layout(int64_t m, int64_t n, int64_t b, int64_t d)
{
    auto r = [](size_t doubles) { return ((doubles * 8 + 255) & ~size_t(255)); };
    size_t mn = (size_t)imin(m, n);
    size_t bb = (size_t)imin(b, (int64_t)mn);
    size_t P = 0;
    P += r((size_t)n * d) * 2;             // MskT, L
    P += r((size_t)2 * d * m > (size_t)m * d ? (size_t)2 * d * m : (size_t)m * d);  // column scratch / S^T
    P += r((size_t)2 * d * d);             // row scratch
    P += r((size_t)2 * d) * 3;             // vec tmp (int64), tq, tsrc
    P += r((size_t)d) + r(8) + r((size_t)n);  // ipiv, nt, perm
    P += r(bb * bb) * 3;                   // Rsk11, X, T
    P += r((size_t)d * d) + r((size_t)n * d);  // deferred R_sk GEMM: Q_sk and its output rows
    P += r((size_t)m * bb) + r(bb * (size_t)n) * 2;  // V, W, W2
    P += r(8) * 2;                         // ref, flags
    // temporaries: sketch QR vs panel (never live together)
    size_t p = (size_t)d;
    size_t sq = r(p * p) * 7 + r(p) + r(2 * 160 * 33 + 160 * 32 * 32) + r(64) + r((size_t)n * p);
    size_t lu = r(2 * 160 * 34) + r(64);
    size_t pn = r(bb * bb) * 8 + r(bb) + r((size_t)cdiv((int64_t)bb, 64) * 4096 + 4096);  // + TRSM Dinv
    size_t T = sq > pn ? sq : pn;
    T = T > lu ? T : lu;
    // split-K partials: 16 slices of the largest square product, plus 4 slices of a b x n GEMM1 output so
    // the wave-efficiency split of few-wave W = V^T C calls is not capped by the buffer (C4: 25.9 TFLOP/s
    // at split 1 for 512 x 3584 x 258048, where 5 slices fill the last wave)
    size_t sk = r((size_t)16 * (p > bb ? p * p : bb * bb) + (size_t)4 * 1024 * 1024 + (size_t)4 * bb * (size_t)n);
    Layout L{P, T, sk, P + T + sk + (1u << 20)};
    return L;
}

static int validate(int64_t m, int64_t n, const void* A, int64_t lda, int64_t b, int64_t d, const void* tau,
                    const void* J, const void* rank)
{
    if (m < 0) return -1;
    if (n < 0) return -2;
    if (!A && m > 0 && n > 0) return -3;
    if (lda < (m > 1 ? m : 1)) return -4;
    if (b < 1) return -5;
    if (d < b || (m > 0 && d > m)) return -6;
    if (!tau && m > 0 && n > 0) return -8;
    if (!J && n > 0) return -9;
    if (!rank) return -10;
    return 0;
}

// ----------------------------------------------------------------------------------- the driver
// Host staging for bqrrp_factor_host: A arrives from pinned host memory in column chunks on its own copy
// stream and each chunk's sketch rows are computed as soon as it lands (the sketch is column-separable:
// MskT(cols, :) = A(:, cols)^T S^T), and every block column goes back to the host on a second copy stream
// as soon as it is final (after its iteration's panel: later iterations only touch columns >= c), so both
// PCIe directions overlap the factorization instead of bracketing it.
struct HostIO {
    const double* A_in = nullptr;  // host, ld ld_host
    double* A_out = nullptr;       // host, ld ld_host
    int64_t ld_host = 0;
    cudaStream_t h2d = nullptr, d2h = nullptr;
    int64_t done = 0;  // columns [0, done) already queued to the host
    std::vector<cudaEvent_t> evs;
    cudaEvent_t event()
    {
        cudaEvent_t e;
        BQ_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
        evs.push_back(e);
        return e;
    }
    // queue columns [done, upto) device -> host after the work queued so far on `after`
    void flush(cudaStream_t after, int64_t m, const double* A, int64_t lda, int64_t upto)
    {
        if (upto <= done) return;
        cudaEvent_t e = event();
        BQ_CUDA(cudaEventRecord(e, after));
        BQ_CUDA(cudaStreamWaitEvent(d2h, e, 0));
        BQ_CUDA(cudaMemcpy2DAsync(A_out + done * ld_host, ld_host * sizeof(double), A + done * lda, lda * sizeof(double),
                                  m * sizeof(double), upto - done, cudaMemcpyDeviceToHost, d2h));
        done = upto;
    }
    ~HostIO()
    {
        for (auto e : evs) cudaEventDestroy(e);
    }
};

static int64_t factor_impl(Ctx& cx, Ctx* cxb, cudaEvent_t ev_top, cudaEvent_t ev_bulk, int64_t m, int64_t n, double* A,
                           int64_t lda, int64_t b, int64_t d, uint64_t seed, double* tau, int64_t* J, double rank_tol,
                           int passes, bool hqr_fallback, int* host_flags, HostIO* hio = nullptr)
{
    const int64_t mn = imin(m, n);
    double* MskT = cx.alloc((size_t)n * d);
    double* Lb = cx.alloc((size_t)n * d);
    double* colscr = cx.alloc(imax(2 * d * m, m * d));
    double* rowscr = cx.alloc((size_t)2 * d * d);
    int64_t* vtmp = cx.alloc_as<int64_t>((size_t)2 * d);
    Touched T;
    T.tq = cx.alloc_as<int>((size_t)2 * d);
    T.tsrc = cx.alloc_as<int>((size_t)2 * d);
    T.nt = cx.alloc_as<int>(2);
    int* ipiv = cx.alloc_as<int>((size_t)d);
    int* perm = cx.alloc_as<int>((size_t)n);
    int64_t bb = imin(b, mn);
    double* Rsk11 = cx.alloc((size_t)bb * bb);
    double* X = cx.alloc((size_t)bb * bb);
    double* ref = cx.alloc(1);
    // panel outputs and WY scratch stay alive across the overlap of the bulk GEMM with the next a2
    double* Vp = cx.alloc((size_t)m * bb);
    double* Tp = cx.alloc((size_t)bb * bb);
    double* W = cx.alloc((size_t)bb * n);
    double* W2 = cx.alloc((size_t)bb * n);
    bool bulk_pending = false;
    RskDefer rsk;  // the R_sk(:, d:) GEMM of every pivot selection on the side stream (lookahead only)
    if (cxb) {
        rsk.side = cxb;
        rsk.Q = cx.alloc((size_t)d * d);
        rsk.Y = cx.alloc((size_t)n * d);
    }
    cudaEvent_t ev_x0 = nullptr, ev_x1 = nullptr;  // side-stream X of the sample update
    BQ_CUDA(cudaEventCreateWithFlags(&ev_x0, cudaEventDisableTiming));
    BQ_CUDA(cudaEventCreateWithFlags(&ev_x1, cudaEventDisableTiming));
    struct EvGuard {
        cudaEvent_t a, b;
        ~EvGuard() { cudaEventDestroy(a); cudaEventDestroy(b); }
    } ev_guard{ev_x0, ev_x1};

    cx.mark(PH_OTHER);
    init_j_kernel<<<(unsigned)imin(cdiv(n, 256), 1024), 256, 0, cx.stream>>>(n, J);
    BQ_LAUNCH_CHECK();
    BQ_CUDA(cudaMemsetAsync(tau, 0, sizeof(double) * mn, cx.stream));
    BQ_CUDA(cudaMemsetAsync(cx.flags, 0, sizeof(int) * F_NFLAGS, cx.stream));
    // a1: sketch (S^T lives in the column scratch until the loop starts)
    if (hio) {
        sketch_operator_T(cx, m, d, seed, colscr, m);
        const int64_t chunk = imax(b, cdiv(n, 16));
        for (int64_t c0 = 0; c0 < n; c0 += chunk) {
            const int64_t nc = imin(chunk, n - c0);
            BQ_CUDA(cudaMemcpy2DAsync(A + c0 * lda, lda * sizeof(double), hio->A_in + c0 * hio->ld_host,
                                      hio->ld_host * sizeof(double), m * sizeof(double), nc, cudaMemcpyHostToDevice,
                                      hio->h2d));
            cudaEvent_t e = hio->event();
            BQ_CUDA(cudaEventRecord(e, hio->h2d));
            BQ_CUDA(cudaStreamWaitEvent(cx.stream, e, 0));
            gemm(cx, true, false, nc, d, m, 1.0, A + c0 * lda, lda, colscr, m, 0.0, MskT + c0, n, false, 0,
                 /*no_split=*/true);  // MskT rows (no split-K: bitwise the device entry's one-GEMM sketch)
        }
    } else {
        sketch_apply(cx, m, n, A, lda, d, seed, MskT, n, colscr);
    }
    nonfinite_kernel<<<(unsigned)imin(cdiv(n * d, 256), 4 * cx.num_sms), 256, 0, cx.stream>>>(n, d, MskT, n, cx.flags);
    BQ_LAUNCH_CHECK();

    int64_t ell = mn;
    for (int64_t i = 0;; ++i) {
        const int64_t s = i * b;
        if (s >= mn) { ell = mn; break; }
        const int64_t c = imin(n, s + b), r = imin(m, s + b), w = n - s, h = m - s;
        const int64_t kmax = imin(imin(b, w), h);
        // ---- a2: pivots from LU of the sketch transpose, then R_sk
        cx.mark(PH_QRCP_WIDE);
        copy_matrix(cx, w, d, MskT + s, n, Lb, n);
        getrf_pivots(cx, Lb, n, w, d, ipiv, perm);
        const int64_t nlu = imin(w, d);
        touched_from_perm(cx, w, nlu, perm, T);
        permute_rows(cx, d, MskT + s, n, T, rowscr);
        sketch_qr(cx, MskT + s, n, w, d, RowBlocks(), cxb ? &rsk : nullptr);
        cx.mark(PH_TRI_RANK);
        tri_rank_kernel<<<1, 1024, 0, cx.stream>>>(MskT + s, n, kmax, i == 0, rank_tol, ref, cx.flags);
        BQ_LAUNCH_CHECK();
        // ---- a3: column permutation of A (all m rows) and J (after the previous bulk update landed)
        cx.mark(PH_COL_PERM);
        if (bulk_pending) {
            BQ_CUDA(cudaStreamWaitEvent(cx.stream, ev_bulk, 0));
            bulk_pending = false;
        }
        permute_columns(cx, m, A + s * lda, lda, T, colscr);
        permute_vector(cx, J + s, T, vtmp);
        zero_col_kernel<<<(unsigned)imin(cdiv(h, 256), 64), 256, 0, cx.stream>>>(h, A + s + s * lda, cx.flags);
        BQ_LAUNCH_CHECK();
        BQ_CUDA(cudaMemcpyAsync(host_flags, cx.flags, sizeof(int) * F_NFLAGS, cudaMemcpyDeviceToHost, cx.stream));
        BQ_CUDA(cudaStreamSynchronize(cx.stream));
        if (host_flags[F_NONFINITE] || host_flags[F_POTRF_INFO]) return -1;
        const int64_t k = host_flags[F_K];
        if (k == 0 || host_flags[F_ZERO_COL]) { ell = s; break; }
        // ---- a4 + a5: panel and trailing update
        cx.mark(PH_QR_TALL);
        extract_rsk11_kernel<<<(unsigned)imin(cdiv(k * k, 256), 4 * cx.num_sms), 256, 0, cx.stream>>>(k, MskT + s, n,
                                                                                                        Rsk11);
        BQ_LAUNCH_CHECK();
        g_panel_fallbacks += panel_factor(cx, m, A, lda, s, k, Rsk11, tau, passes, Vp, Tp, hqr_fallback, cxb);
        // ---- a5 (the bulk rows overlap the sketch update and the next a2) and a7
        cx.mark(PH_APPLY_QT);
        const bool terminal = (k < kmax || c == n || r == m);
        if (hio && !terminal) hio->flush(cx.stream, m, A, lda, c);  // block column [s, c) is final
        // a6's X = R_sk11 R11^{-1} (b x b) needs only the panel: on the idle side stream during GEMM1
        // (ahead of the bulk rows there, which wait for GEMM1 anyway); no split-K slices on that stream
        const bool x_side = !terminal && cxb;
        if (x_side) {
            BQ_CUDA(cudaEventRecord(ev_x0, cx.stream));
            BQ_CUDA(cudaStreamWaitEvent(cxb->stream, ev_x0, 0));
            Ctx sc = *cxb;
            sc.timer = nullptr;
            copy_matrix(sc, b, b, Rsk11, k, X, b);
            trsm_right_upper(sc, b, b, A + s + s * lda, lda, false, false, X, b);  // X = R_sk11 R11^{-1}
            zero_triangle(sc, 'U', b, b, X, b);
            BQ_CUDA(cudaEventRecord(ev_x1, cxb->stream));
        }
        wy_update(cx, terminal ? nullptr : cxb, m, n, A, lda, s, k, Vp, Tp, W, W2, ev_top, ev_bulk);
        if (!terminal && cxb && h > k && n - s - k > 0) bulk_pending = true;
        if (terminal) { ell = s + k; break; }
        // ---- a6: sketch update (k == b here)
        cx.mark(PH_SAMPLE_UPDATE);
        if (x_side) {
            BQ_CUDA(cudaStreamWaitEvent(cx.stream, ev_x1, 0));
        } else {
            copy_matrix(cx, b, b, Rsk11, k, X, b);
            trsm_right_upper(cx, b, b, A + s + s * lda, lda, false, false, X, b);  // X = R_sk11 R11^{-1}
            zero_triangle(cx, 'U', b, b, X, b);
        }
        gemm(cx, true, true, n - c, b, b, -1.0, A + s + c * lda, lda, X, b, 1.0, MskT + c, n);
    }
    // O4: tau(ell:) = 0, A(ell:m, ell:n) = 0 (reading Z16)
    cx.mark(PH_OTHER);
    if (bulk_pending) BQ_CUDA(cudaStreamWaitEvent(cx.stream, ev_bulk, 0));
    if (ell < mn) BQ_CUDA(cudaMemsetAsync(tau + ell, 0, sizeof(double) * (mn - ell), cx.stream));
    set_zero(cx, m - ell, n - ell, A + ell + ell * lda, lda);
    if (hio) hio->flush(cx.stream, m, A, lda, n);
    cx.mark(PH_OTHER);
    BQ_CUDA(cudaMemcpyAsync(host_flags, cx.flags, sizeof(int) * F_NFLAGS, cudaMemcpyDeviceToHost, cx.stream));
    BQ_CUDA(cudaStreamSynchronize(cx.stream));
    if (host_flags[F_NONFINITE] || host_flags[F_POTRF_INFO]) return -1;
    return ell;
}

static int* pinned_flags()
{
    static thread_local int* p = nullptr;
    if (!p) BQ_CUDA(cudaMallocHost(&p, sizeof(int) * F_NFLAGS));
    return p;
}

static void setup_ctx(Ctx& cx, void* stream)
{
    cx.stream = (cudaStream_t)stream;
    int dev = 0;
    BQ_CUDA(cudaGetDevice(&dev));
    BQ_CUDA(cudaDeviceGetAttribute(&cx.num_sms, cudaDevAttrMultiProcessorCount, dev));
}

// Carve splitk + flags from the tail of the workspace.
static void carve(Ctx& cx, void* ws, size_t bytes, const Layout& L)
{
    cx.ws = (char*)ws;
    cx.ws_bytes = bytes;
    cx.ws_used = 0;
    cx.splitk = cx.alloc(L.splitk / 8);
    cx.splitk_elems = L.splitk / 8;
    cx.flags = cx.alloc_as<int>(F_NFLAGS);
}

}  // namespace bqrrp

using namespace bqrrp;

template <typename F>
static int guarded(F&& f)
{
    try {
        return f();
    } catch (const CudaError& e) {
        g_last_error = e.what();
        return BQRRP_ECUDA;
    } catch (const std::bad_alloc& e) {
        g_last_error = e.what();
        return BQRRP_ENOMEM;
    } catch (const std::exception& e) {
        g_last_error = e.what();
        return std::strstr(e.what(), "workspace") ? BQRRP_ENOMEM : BQRRP_ECUDA;
    }
}

extern "C" {

int bqrrp_workspace_query(int64_t m, int64_t n, int64_t b, int64_t d, size_t* bytes)
{
    if (m < 0) return -1;
    if (n < 0) return -2;
    if (b < 1) return -3;
    if (d < b || (m > 0 && d > m)) return -4;
    if (!bytes) return -5;
    *bytes = layout(m, n, b, d).total;
    return 0;
}

static int factor_ex_impl(int64_t m, int64_t n, double* A, int64_t lda, int64_t b, int64_t d, uint64_t seed,
                          double* tau, int64_t* J, int64_t* rank, void* workspace, size_t ws_bytes, void* stream,
                          const bqrrp_options* opts, HostIO* hio);

int bqrrp_factor_ex(int64_t m, int64_t n, double* A, int64_t lda, int64_t b, int64_t d, uint64_t seed, double* tau,
                    int64_t* J, int64_t* rank, void* workspace, size_t ws_bytes, void* stream, const bqrrp_options* opts)
{
    return factor_ex_impl(m, n, A, lda, b, d, seed, tau, J, rank, workspace, ws_bytes, stream, opts, nullptr);
}

static int factor_ex_impl(int64_t m, int64_t n, double* A, int64_t lda, int64_t b, int64_t d, uint64_t seed,
                          double* tau, int64_t* J, int64_t* rank, void* workspace, size_t ws_bytes, void* stream,
                          const bqrrp_options* opts, HostIO* hio)
{
    int v = validate(m, n, A, lda, b, d, tau, J, rank);
    if (v != 0) return v;
    double rank_tol = (opts && opts->rank_tol > 0) ? opts->rank_tol : 10.0 * 0x1p-53 * sqrt((double)(m > n ? m : n));
    int passes = (opts && opts->cholqr_passes >= 0 && opts->cholqr_passes <= 4) ? opts->cholqr_passes : 2;
    g_panel_fallbacks = 0;
    return guarded([&]() -> int {
        Ctx cx;
        setup_ctx(cx, stream);
        if (m == 0 || n == 0) {
            *rank = 0;
            if (n > 0) {
                init_j_kernel<<<(unsigned)imin(cdiv(n, 256), 1024), 256, 0, cx.stream>>>(n, J);
                BQ_LAUNCH_CHECK();
            }
            return 0;
        }
        Layout L = layout(m, n, b, d);
        void* ws = workspace;
        bool own = false;
        if (!ws) {
            BQ_CUDA(lib_malloc_async(&ws, L.total, cx.stream));
            ws_bytes = L.total;
            own = true;
        } else if (ws_bytes < L.total) {
            g_last_error = "workspace smaller than bqrrp_workspace_query";
            return -11;
        }
        carve(cx, ws, ws_bytes, L);
        // critical chain on a high-priority stream, the bulk trailing GEMM on a low-priority one;
        // both joined to the caller's stream at entry and exit
        int prio_lo = 0, prio_hi = 0;
        BQ_CUDA(cudaDeviceGetStreamPriorityRange(&prio_lo, &prio_hi));
        cudaStream_t user = cx.stream, s_hi = nullptr, s_lo = nullptr;
        cudaEvent_t ev_in = nullptr, ev_top = nullptr, ev_bulk = nullptr, ev_hi_done = nullptr;
        BQ_CUDA(cudaStreamCreateWithPriority(&s_hi, cudaStreamNonBlocking, prio_hi));
        BQ_CUDA(cudaStreamCreateWithPriority(&s_lo, cudaStreamNonBlocking, prio_lo));
        BQ_CUDA(cudaEventCreateWithFlags(&ev_in, cudaEventDisableTiming));
        BQ_CUDA(cudaEventCreateWithFlags(&ev_top, cudaEventDisableTiming));
        BQ_CUDA(cudaEventCreateWithFlags(&ev_bulk, cudaEventDisableTiming));
        BQ_CUDA(cudaEventCreateWithFlags(&ev_hi_done, cudaEventDisableTiming));
        BQ_CUDA(cudaEventRecord(ev_in, user));
        BQ_CUDA(cudaStreamWaitEvent(s_hi, ev_in, 0));
        BQ_CUDA(cudaStreamWaitEvent(s_lo, ev_in, 0));
        cx.stream = s_hi;
        Ctx cxb = cx;
        cxb.stream = s_lo;
        cxb.splitk = nullptr;  // the split-K scratch belongs to the critical stream
        cxb.splitk_elems = 0;
        Timer tm;
        if (opts && opts->phase_ms) {
            tm.on = true;
            tm.st = s_hi;
            cx.timer = &tm;
            cxb.timer = &tm;
        }
        int64_t ell = -1;
        int status = 0;
        auto cleanup = [&]() {
            cudaEventRecord(ev_hi_done, s_hi);
            cudaStreamWaitEvent(user, ev_hi_done, 0);
            cudaEventRecord(ev_bulk, s_lo);
            cudaStreamWaitEvent(user, ev_bulk, 0);
            cudaStreamDestroy(s_hi);
            cudaStreamDestroy(s_lo);
            cudaEventDestroy(ev_in);
            cudaEventDestroy(ev_top);
            cudaEventDestroy(ev_bulk);
            cudaEventDestroy(ev_hi_done);
            cx.stream = user;
        };
        try {
            ell = factor_impl(cx, (opts && opts->no_lookahead) ? nullptr : &cxb, ev_top, ev_bulk, m, n, A, lda, b, d,
                              seed, tau, J, rank_tol, passes, !(opts && opts->no_hqr_fallback), pinned_flags(), hio);
        } catch (...) {
            cleanup();
            if (own) cudaFreeAsync(ws, user);
            throw;
        }
        cleanup();
        if (opts && opts->phase_ms) tm.finish(opts->phase_ms);
        if (own) BQ_CUDA(cudaFreeAsync(ws, user));
        if (ell < 0) {
            g_last_error = "non-finite sketch or Cholesky-QR breakdown";
            status = BQRRP_ENUMERIC;
            *rank = 0;
        } else {
            *rank = ell;
        }
        return status;
    });
}

int bqrrp_factor(int64_t m, int64_t n, double* A, int64_t lda, int64_t b, int64_t d, uint64_t seed, double* tau,
                 int64_t* J, int64_t* rank, void* workspace, size_t ws_bytes, void* stream)
{
    return bqrrp_factor_ex(m, n, A, lda, b, d, seed, tau, J, rank, workspace, ws_bytes, stream, nullptr);
}

int bqrrp_factor_host(int64_t m, int64_t n, double* A_host, int64_t lda, int64_t b, int64_t d, uint64_t seed,
                      double* tau_host, int64_t* J_host, int64_t* rank, void* stream, const bqrrp_options* opts)
{
    int v = validate(m, n, A_host, lda, b, d, tau_host, J_host, rank);
    if (v != 0) return v;
    return guarded([&]() -> int {
        cudaStream_t st = (cudaStream_t)stream;
        int64_t mn = imin(m, n);
        double *dA = nullptr, *dtau = nullptr;
        int64_t* dJ = nullptr;
        size_t wsb = 0;
        bqrrp_workspace_query(m, n, b, d, &wsb);
        void* ws = nullptr;
        BQ_CUDA(lib_malloc_async(&dA, sizeof(double) * (size_t)imax(1, m * n), st));
        BQ_CUDA(lib_malloc_async(&dtau, sizeof(double) * (size_t)imax(1, mn), st));
        BQ_CUDA(lib_malloc_async(&dJ, sizeof(int64_t) * (size_t)imax(1, n), st));
        BQ_CUDA(lib_malloc_async(&ws, wsb, st));
        int status = 0;
        if (m > 0 && n > 0) {
            // the copies run on their own streams, overlapped with the factorization (HostIO above)
            HostIO hio;
            hio.A_in = A_host;
            hio.A_out = A_host;
            hio.ld_host = lda;
            BQ_CUDA(cudaStreamCreateWithFlags(&hio.h2d, cudaStreamNonBlocking));
            BQ_CUDA(cudaStreamCreateWithFlags(&hio.d2h, cudaStreamNonBlocking));
            cudaEvent_t e0 = hio.event();
            BQ_CUDA(cudaEventRecord(e0, st));  // after the allocations
            BQ_CUDA(cudaStreamWaitEvent(hio.h2d, e0, 0));
            BQ_CUDA(cudaStreamWaitEvent(hio.d2h, e0, 0));
            status = factor_ex_impl(m, n, dA, imax(1, m), b, d, seed, dtau, dJ, rank, ws, wsb, stream, opts, &hio);
            cudaEvent_t e1 = hio.event();
            BQ_CUDA(cudaEventRecord(e1, hio.d2h));
            BQ_CUDA(cudaStreamWaitEvent(st, e1, 0));
            BQ_CUDA(cudaEventRecord(e1, hio.h2d));
            BQ_CUDA(cudaStreamWaitEvent(st, e1, 0));
            if (status == 0) {
                BQ_CUDA(cudaMemcpyAsync(tau_host, dtau, sizeof(double) * mn, cudaMemcpyDeviceToHost, st));
                BQ_CUDA(cudaMemcpyAsync(J_host, dJ, sizeof(int64_t) * n, cudaMemcpyDeviceToHost, st));
            }
            BQ_CUDA(cudaStreamSynchronize(st));
            cudaStreamDestroy(hio.h2d);
            cudaStreamDestroy(hio.d2h);
        } else {
            status = factor_ex_impl(m, n, dA, imax(1, m), b, d, seed, dtau, dJ, rank, ws, wsb, stream, opts, nullptr);
            if (status == 0 && n > 0)
                BQ_CUDA(cudaMemcpyAsync(J_host, dJ, sizeof(int64_t) * n, cudaMemcpyDeviceToHost, st));
        }
        cudaFreeAsync(dA, st);
        cudaFreeAsync(dtau, st);
        cudaFreeAsync(dJ, st);
        cudaFreeAsync(ws, st);
        BQ_CUDA(cudaStreamSynchronize(st));
        return status;
    });
}

// ------------------------------------------------------------------------------------ debug entries
int bqrrp_debug_sketch(int64_t m, int64_t n, const double* A, int64_t lda, int64_t d, uint64_t seed, double* S_out,
                       double* MskT_out, void* stream)
{
    if (m < 1) return -1;
    if (n < 0) return -2;
    if (!A) return -3;
    if (lda < m) return -4;
    if (d < 1) return -5;
    if (!MskT_out) return -8;
    return guarded([&]() -> int {
        Ctx cx;
        setup_ctx(cx, stream);
        double* St = nullptr;
        BQ_CUDA(lib_malloc_async(&St, sizeof(double) * m * d, cx.stream));
        Layout L{0, 0, (size_t)16 * 1024 * 1024, 0};
        void* ws = nullptr;
        BQ_CUDA(lib_malloc_async(&ws, L.splitk + 4096, cx.stream));
        carve(cx, ws, L.splitk + 4096, L);
        sketch_apply(cx, m, n, A, lda, d, seed, MskT_out, n, St);
        if (S_out) transpose_copy(cx, m, d, St, m, S_out, d);
        cudaFreeAsync(St, cx.stream);
        cudaFreeAsync(ws, cx.stream);
        BQ_CUDA(cudaStreamSynchronize(cx.stream));
        return 0;
    });
}

int bqrrp_debug_gemm(int ta, int tb, int64_t M, int64_t N, int64_t K, double alpha, const double* A, int64_t lda,
                     const double* B, int64_t ldb, double beta, double* C, int64_t ldc, void* stream)
{
    if (M < 0) return -3;
    if (N < 0) return -4;
    if (K < 0) return -5;
    return guarded([&]() -> int {
        Ctx cx;
        setup_ctx(cx, stream);
        size_t sk = (size_t)32 * (size_t)imax(1, M * N);
        void* ws = nullptr;
        BQ_CUDA(lib_malloc_async(&ws, sk * 8 + 4096, cx.stream));
        Layout L{0, 0, sk * 8, 0};
        carve(cx, ws, sk * 8 + 4096, L);
        gemm(cx, ta != 0, tb != 0, M, N, K, alpha, A, lda, B, ldb, beta, C, ldc);
        cudaFreeAsync(ws, cx.stream);
        BQ_CUDA(cudaStreamSynchronize(cx.stream));
        return 0;
    });
}

int bqrrp_debug_trsm(int64_t rows, int64_t n, const double* T, int64_t ldt, int t_lower, int unit, int inverse,
                     double* B, int64_t ldb, void* stream)
{
    if (rows < 0) return -1;
    if (n < 0) return -2;
    return guarded([&]() -> int {
        Ctx cx;
        setup_ctx(cx, stream);
        size_t sk = (size_t)16 * 64 * 64 + (4u << 20) / 8;
        size_t bytes = (sk + (size_t)cdiv(imax(n, 1), 64) * 4096 + 8192) * 8;
        void* ws = nullptr;
        BQ_CUDA(lib_malloc_async(&ws, bytes, cx.stream));
        Layout L{0, 0, sk * 8, 0};
        carve(cx, ws, bytes, L);
        trsm_right_upper(cx, rows, n, T, ldt, t_lower != 0, unit != 0, B, ldb, inverse != 0);
        cudaFreeAsync(ws, cx.stream);
        BQ_CUDA(cudaStreamSynchronize(cx.stream));
        return 0;
    });
}

static size_t debug_ws_bytes(int64_t rows, int64_t d)
{
    // scratch (rows x d panels, d x d factors) + the split-K slices carved first (16 d^2 + 4 MiB)
    return (size_t)(64ull << 20) + (size_t)rows * (size_t)d * 8 * 6 + (size_t)d * d * 8 * (8 + 16);
}

int bqrrp_debug_lu_pivots(int64_t w, int64_t d, double* L, int64_t ld, int64_t* ipiv, void* stream)
{
    if (w < 0) return -1;
    if (d < 0) return -2;
    return guarded([&]() -> int {
        Ctx cx;
        setup_ctx(cx, stream);
        size_t wsb = debug_ws_bytes(w, d);
        void* ws = nullptr;
        BQ_CUDA(lib_malloc_async(&ws, wsb, cx.stream));
        Layout Ly{0, 0, (size_t)16 * imax(1, d * d) * 8 + (4u << 20), 0};
        carve(cx, ws, wsb, Ly);
        int* ip = cx.alloc_as<int>((size_t)imax(1, d));
        int* pm = cx.alloc_as<int>((size_t)imax(1, w));
        getrf_pivots(cx, L, ld, w, d, ip, pm);
        int64_t nlu = imin(w, d);
        if (nlu > 0) {
            ipiv_to_i64_kernel<<<(unsigned)cdiv(nlu, 128), 128, 0, cx.stream>>>(nlu, ip, ipiv);
            BQ_LAUNCH_CHECK();
        }
        cudaFreeAsync(ws, cx.stream);
        BQ_CUDA(cudaStreamSynchronize(cx.stream));
        return 0;
    });
}

int bqrrp_debug_sketch_qr(int64_t w, int64_t d, double* WT, int64_t ld, void* stream)
{
    if (w < 0) return -1;
    if (d < 1) return -2;
    return guarded([&]() -> int {
        Ctx cx;
        setup_ctx(cx, stream);
        size_t wsb = debug_ws_bytes(w, d);
        void* ws = nullptr;
        BQ_CUDA(lib_malloc_async(&ws, wsb, cx.stream));
        Layout Ly{0, 0, (size_t)16 * d * d * 8 + (4u << 20), 0};
        carve(cx, ws, wsb, Ly);
        sketch_qr(cx, WT, ld, w, d);
        cudaFreeAsync(ws, cx.stream);
        BQ_CUDA(cudaStreamSynchronize(cx.stream));
        return 0;
    });
}

__global__ void jqr_from_touched_kernel(int64_t w, const int* tq, const int* tsrc, const int* nt, int64_t* Jqr)
{
    for (int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; q < w; q += (int64_t)gridDim.x * blockDim.x)
        Jqr[q] = q + 1;
    __syncthreads();
}
__global__ void jqr_apply_touched_kernel(const int* tq, const int* tsrc, const int* nt, int64_t* Jqr)
{
    int n = *nt;
    for (int t = blockIdx.x * blockDim.x + threadIdx.x; t < n; t += gridDim.x * blockDim.x) Jqr[tq[t]] = tsrc[t] + 1;
}

int bqrrp_debug_permute(int64_t rows, int64_t w, double* X, int64_t ldx, int64_t nlu, const int64_t* ipiv,
                        int64_t* Jqr_out, void* stream)
{
    if (rows < 0) return -1;
    if (w < 0) return -2;
    if (nlu < 0 || nlu > w) return -5;
    return guarded([&]() -> int {
        Ctx cx;
        setup_ctx(cx, stream);
        size_t wsb = (size_t)(8u << 20) + (size_t)2 * imax(1, nlu) * imax(1, rows) * 8 + (size_t)w * 4;
        void* ws = nullptr;
        BQ_CUDA(lib_malloc_async(&ws, wsb, cx.stream));
        Layout Ly{0, 0, 4096, 0};
        carve(cx, ws, wsb, Ly);
        Touched T;
        T.tq = cx.alloc_as<int>((size_t)2 * imax(1, nlu));
        T.tsrc = cx.alloc_as<int>((size_t)2 * imax(1, nlu));
        T.nt = cx.alloc_as<int>(2);
        int* pm = cx.alloc_as<int>((size_t)imax(1, w));
        double* scr = cx.alloc((size_t)2 * imax(1, nlu) * imax(1, rows));
        perm_from_ipiv(cx, w, nlu, ipiv, pm);
        touched_from_perm(cx, w, nlu, pm, T);
        permute_columns(cx, rows, X, ldx, T, scr);
        if (Jqr_out && w > 0) {
            jqr_from_touched_kernel<<<(unsigned)imin(cdiv(w, 256), 1024), 256, 0, cx.stream>>>(w, T.tq, T.tsrc, T.nt,
                                                                                               Jqr_out);
            BQ_LAUNCH_CHECK();
            jqr_apply_touched_kernel<<<16, 256, 0, cx.stream>>>(T.tq, T.tsrc, T.nt, Jqr_out);
            BQ_LAUNCH_CHECK();
        }
        cudaFreeAsync(ws, cx.stream);
        BQ_CUDA(cudaStreamSynchronize(cx.stream));
        return 0;
    });
}

int bqrrp_debug_panel(int64_t h, int64_t k, int64_t t, double* P, int64_t ld, const double* Rsk11, double* tau,
                      int cholqr_passes, void* stream)
{
    if (h < 1) return -1;
    if (k < 1 || k > h) return -2;
    if (t < 0) return -3;
    if (cholqr_passes < 0 || cholqr_passes > 4) return -8;
    return guarded([&]() -> int {
        Ctx cx;
        setup_ctx(cx, stream);
        size_t wsb = (size_t)(64u << 20) + ((size_t)h * k + (size_t)9 * k * k + (size_t)2 * k * (t + 1)) * 8 +
                     (size_t)16 * k * k * 8;
        void* ws = nullptr;
        BQ_CUDA(lib_malloc_async(&ws, wsb, cx.stream));
        Layout Ly{0, 0, (size_t)16 * k * k * 8 + (4u << 20), 0};
        carve(cx, ws, wsb, Ly);
        BQ_CUDA(cudaMemsetAsync(cx.flags, 0, sizeof(int) * F_NFLAGS, cx.stream));
        double* V = cx.alloc((size_t)h * k);
        double* Tb = cx.alloc((size_t)k * k);
        double* W = cx.alloc((size_t)k * (t + 1));
        double* W2 = cx.alloc((size_t)k * (t + 1));
        panel_factor(cx, h, P, ld, 0, k, Rsk11, tau, cholqr_passes, V, Tb);
        wy_update(cx, nullptr, h, k + t, P, ld, 0, k, V, Tb, W, W2, nullptr, nullptr);
        int* hf = pinned_flags();
        BQ_CUDA(cudaMemcpyAsync(hf, cx.flags, sizeof(int) * F_NFLAGS, cudaMemcpyDeviceToHost, cx.stream));
        cudaFreeAsync(ws, cx.stream);
        BQ_CUDA(cudaStreamSynchronize(cx.stream));
        return hf[F_POTRF_INFO] ? BQRRP_ENUMERIC : 0;
    });
}

const char* bqrrp_strerror(int status)
{
    switch (status) {
    case BQRRP_OK: return "success";
    case BQRRP_ENUMERIC: return "numerical failure (non-finite sketch or Cholesky-QR breakdown)";
    case BQRRP_ENOMEM: return "out of device memory / workspace too small";
    case BQRRP_ECUDA: return "CUDA error";
    case BQRRP_ENCCL: return "NCCL error";
    default: return status < 0 ? "illegal argument" : "unknown status";
    }
}

const char* bqrrp_last_error(void) { return g_last_error.c_str(); }

unsigned long long bqrrp_launch_count(void) { return g_launches; }

long long bqrrp_panel_fallbacks(void) { return g_panel_fallbacks; }

int bqrrp_trim_memory(void)
{
    return guarded([&]() -> int {
        BQ_CUDA(cudaDeviceSynchronize());
        BQ_CUDA(cudaMemPoolTrimTo(lib_pool(), 0));
        return 0;
    });
}

const char* bqrrp_version(void) { return "bqrrp-b200 0.1 (sm_100a, DMMA f64)"; }

}  // extern "C"
