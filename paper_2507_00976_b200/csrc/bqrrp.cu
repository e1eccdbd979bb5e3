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
#include <cuda.h>
#include <cstring>
#include <mutex>
#include <vector>
#include <string>

#include "../../include/bqrrp.h"
#include "blas.cuh"
#include "bqrrp_internal.cuh"


namespace bqrrp {

thread_local std::string g_last_error;

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
cudaStream_t green_stream(int sms, int* got)
{
    // driver entry points through the runtime (no link-time libcuda dependency)
    using GetRes = CUresult (*)(CUdevice, CUdevResource*, CUdevResourceType);
    using Split = CUresult (*)(CUdevResource*, unsigned*, const CUdevResource*, CUdevResource*, unsigned, unsigned);
    using Desc = CUresult (*)(CUdevResourceDesc*, CUdevResource*, unsigned);
    using Green = CUresult (*)(CUgreenCtx*, CUdevResourceDesc, CUdevice, unsigned);
    using GStream = CUresult (*)(CUstream*, CUgreenCtx, unsigned, int);
    struct Entry {
        int dev, req, got;
        cudaStream_t st;
    };
    static std::mutex mu;
    static std::vector<Entry> cache;
    int dev = 0;
    BQ_CUDA(cudaGetDevice(&dev));
    std::lock_guard<std::mutex> lk(mu);
    for (const Entry& e : cache)
        if (e.dev == dev && e.req == sms) {
            *got = e.got;
            return e.st;
        }
    auto entry = [](const char* name) -> void* {
        void* p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint(name, &p, cudaEnableDefault, &q) != cudaSuccess || q != cudaDriverEntryPointSuccess)
            return nullptr;
        return p;
    };
    auto getres = (GetRes)entry("cuDeviceGetDevResource");
    auto split = (Split)entry("cuDevSmResourceSplitByCount");
    auto desc = (Desc)entry("cuDevResourceGenerateDesc");
    auto green = (Green)entry("cuGreenCtxCreate");
    auto gstream = (GStream)entry("cuGreenCtxStreamCreate");
    Entry e{dev, sms, 0, nullptr};
    int prio_lo = 0, prio_hi = 0;
    BQ_CUDA(cudaDeviceGetStreamPriorityRange(&prio_lo, &prio_hi));
    // Cluster-aware split (CU_DEV_SM_RESOURCE_SPLIT_MAX_POTENTIAL_CLUSTER_SIZE) into groups of 16 SMs: the partition
    // is every group but the last few, plus the remainder, so the SMs left free are whole groups where the chain's
    // 8-CTA leaf clusters can be placed while the bulk runs (a plain split by count leaves SMs scattered over the
    // GPCs, and no cluster of full-SM CTAs fits there: tools/green_probe.cu).  9 groups + 4 on a 148-SM B200.
    CUdevResource all, grp[64], rest;
    unsigned ng = 0;
    CUdevResourceDesc dsc;
    CUgreenCtx g;
    CUstream s;
    const unsigned flags = CU_DEV_SM_RESOURCE_SPLIT_MAX_POTENTIAL_CLUSTER_SIZE;
    if (getres && split && desc && green && gstream && getres(dev, &all, CU_DEV_RESOURCE_TYPE_SM) == CUDA_SUCCESS &&
        split(nullptr, &ng, &all, nullptr, flags, 16) == CUDA_SUCCESS && ng >= 2 && ng <= 64) {
        const int nfree = (int)(((int)all.sm.smCount - sms + 15) / 16);  // whole groups left to the chain
        if (split(grp, &ng, &all, &rest, flags, 16) == CUDA_SUCCESS && nfree >= 1 && nfree < (int)ng) {
            CUdevResource sel[65];
            unsigned ns = 0, cnt = 0;
            for (unsigned i = 0; i + nfree < ng; ++i) {
                sel[ns++] = grp[i];
                cnt += grp[i].sm.smCount;
            }
            if (rest.sm.smCount) {
                sel[ns++] = rest;
                cnt += rest.sm.smCount;
            }
            if (desc(&dsc, sel, ns) == CUDA_SUCCESS && green(&g, dsc, dev, CU_GREEN_CTX_DEFAULT_STREAM) == CUDA_SUCCESS &&
                gstream(&s, g, CU_STREAM_NON_BLOCKING, prio_lo) == CUDA_SUCCESS) {
                e.st = (cudaStream_t)s;
                e.got = (int)cnt;
            }
        }
    }
    cudaGetLastError();  // a failed probe leaves no sticky runtime error
    cache.push_back(e);
    *got = e.got;
    return e.st;
}

thread_local long long g_panel_fallbacks = 0;
std::atomic<unsigned long long> g_launches{0};

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

void init_j(Ctx& cx, int64_t n, int64_t* J)
{
    if (n <= 0) return;
    init_j_kernel<<<(unsigned)imin(cdiv(n, 256), 1024), 256, 0, cx.stream>>>(n, J);
    BQ_LAUNCH_CHECK();
}
void nonfinite_check(Ctx& cx, int64_t rows, int64_t cols, const double* X, int64_t ldx)
{
    if (rows <= 0 || cols <= 0) return;
    nonfinite_kernel<<<(unsigned)imin(cdiv(rows * cols, 256), 4 * cx.num_sms), 256, 0, cx.stream>>>(rows, cols, X, ldx,
                                                                                                      cx.flags);
    BQ_LAUNCH_CHECK();
}
void tri_rank_flags(Ctx& cx, const double* MskT_s, int64_t ldm, int64_t kmax, bool first, double rank_tol, double* ref)
{
    tri_rank_kernel<<<1, 1024, 0, cx.stream>>>(MskT_s, ldm, kmax, first ? 1 : 0, rank_tol, ref, cx.flags);
    BQ_LAUNCH_CHECK();
}
void zero_col_flag(Ctx& cx, int64_t h, const double* col)
{
    zero_col_kernel<<<(unsigned)imin(cdiv(h, 256), 64), 256, 0, cx.stream>>>(h, col, cx.flags);
    BQ_LAUNCH_CHECK();
}
void extract_rsk11(Ctx& cx, int64_t k, const double* MskT_s, int64_t ldm, double* R)
{
    extract_rsk11_kernel<<<(unsigned)imin(cdiv(k * k, 256), 4 * cx.num_sms), 256, 0, cx.stream>>>(k, MskT_s, ldm, R);
    BQ_LAUNCH_CHECK();
}

// ----------------------------------------------------------------------------------- workspace
Layout layout(int64_t m, int64_t n, int64_t b, int64_t d)
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
    // lookahead: second V, the gathered next panel, W2's gathered columns, the bulk GEMM's
    // tile handshake (state + readers per 64 x 64 tile) and the gather's post flags
    const size_t tiles = (size_t)cdiv(m, 64) * (size_t)cdiv(n, 64);
    P += r((size_t)m * bb) * 2 + r(bb * bb) + r((tiles + 1) / 2) * 2 + r(((size_t)cdiv(m, 64) * bb + 1) / 2);
    P += r(8) * 2;                         // ref, flags
    // temporaries: sketch QR vs panel (never live together)
    size_t p = (size_t)d;
    size_t sq = r(p * p) * 7 + r(p) + r(2 * 160 * 33 + 160 * 32 * 32) + r(64) + r((size_t)n * p);
    size_t lu = r(2 * 160 * 34) + r(64);
    sq += lu;  // the pipelined sketch QR's buffers stay live under K-LU's own scratch (SketchQrPipe)
    // panel: 8 k x k factors / products, S, the main stream's TRSM Dinv, and the side-stream arena of
    // recon_finish (its two k x k products come out of the 8; its own TRSM Dinv)
    const size_t dinv = (size_t)cdiv((int64_t)bb, 64) * 4096 + 4096;
    size_t pn = r(bb * bb) * 8 + r(bb) + r(dinv) + r(dinv + 64);
    size_t T = sq > pn ? sq : pn;
    T = T > lu ? T : lu;
    // split-K partials: 16 slices of the largest square product, plus 4 slices of a b x n GEMM1 output so
    // the wave-efficiency split of few-wave W = V^T C calls is not capped by the buffer (C4: 25.9 TFLOP/s
    // at split 1 for 512 x 3584 x 258048, where 5 slices fill the last wave).  That split is only taken
    // below 32 x num_sms 64 x 64 tiles (blas.cu), so the GEMM1 slices are capped at that output size.
    const size_t gemm1_cap = (size_t)32 * 160 * 64 * 64;
    const size_t g1 = bb * (size_t)n < gemm1_cap ? bb * (size_t)n : gemm1_cap;
    size_t sk = r((size_t)16 * (p > bb ? p * p : bb * bb) + (size_t)4 * 1024 * 1024 + (size_t)4 * g1);
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

// Streams of one factorization.  crit (high priority): the critical chain; bulk (low priority):
// the bulk rows of every trailing update; aux (high priority): small fork-join pieces of the critical chain
// (the panel's k x k finish, the sample update's X, the pivot selection's R_sk(:, d:) GEMM).  nullptr bulk =
// one stream, serialised (no_lookahead).
struct Sched {
    Ctx* bulk = nullptr;
    Ctx* aux = nullptr;
    cudaEvent_t ev_top = nullptr, ev_bulk = nullptr;
    int panel_la = 0;  // bqrrp_options.panel_lookahead: 1 = panel i+1 overlapped with bulk i, else after it
    Ctx* qr = nullptr;  // the pipelined sketch QR's stream (SketchQrPipe), or nullptr: sketch_qr after K-LU
    Ctx* lu2 = nullptr;  // the lookahead LU's trailing-update stream (getrf_pivots_la), or nullptr: recursive K-LU
    Ctx* qr2 = nullptr;  // the pipelined sketch QR's T-merge stream, or nullptr: T merged on qr
    Ctx* bulk_part[4] = {};    // the bulk context on SM partitions (green contexts) of part_sms[] SMs, or nullptr
    int part_sms[4] = {};
    int nparts = 0;
    bool part_always = false;  // bqrrp_options.bulk_sms > 0: every bulk on bulk_part[0]
    // The bulk context of one iteration.  The bulk GEMM (2 (h-k) k t flops) overlaps the latency-bound chain (the
    // sample update and the next pivot selection: about 7 us per sketch column under the bulk's contention plus its
    // GEMMs, ~3 w d^2 + 4/3 d^3 flops at ~20 TFLOP/s, plus ~5 us per column for the cooperative-grid LU leaf beyond
    // 16384 rows).  When the bulk is the shorter of the two it runs on the smallest partition that finishes it
    // within ~1.15x the chain (the chain itself speeds up with the SMs it gets back), leaving the other SMs to the
    // chain's cluster kernels (measured: C2 qrcp_wide 196 -> 178 ms with the bulk on 100 SMs,
    // profiles/bulk_partition_r02.json); otherwise on the whole device.
    static double bulk_est_us(int64_t h, int64_t k, int64_t t)
    {
        return 2.0 * (double)(h - k) * (double)k * (double)t / 34e12 * 1e6;
    }
    static double chain_est_us(int64_t d, int64_t w_next)
    {
        const double dd = (double)d, ww = (double)w_next;
#ifndef BQRRP_CHAIN_US_PER_COL  // tuned with the K-SQR pipeline: 5 / 7 / 9 / 12 us, profiles/r02/chain_constant_ab_r02.txt
#define BQRRP_CHAIN_US_PER_COL 7.0
#endif
        return dd * (w_next > 16384 ? 14.0 : BQRRP_CHAIN_US_PER_COL) + (3.0 * ww * dd * dd + 4.0 / 3.0 * dd * dd * dd) / 20e6;
    }
    // K-LU's cooperative grid leaf (w > ~25k rows) for the next pivot selection: capped at 32 CTAs (narrower leaves,
    // the other SMs stay with the bulk GEMM) when the bulk is the long pole — the leaf's every launch otherwise
    // drains the whole device of bulk CTAs (C3 13.41 -> 13.30 s; 16 / 24 / 48 / 64 CTAs measured 13.41 / 13.33 /
    // 13.31 / 13.32 s, profiles/r02/lu_grid_cap_ab_r02.txt) — else one CTA per SM (the leaf on the critical path).
    int lu_grid_for(int64_t h, int64_t k, int64_t t, int64_t d, int64_t w_next) const
    {
        if (lu_grid_user > 0) return lu_grid_user;
        return bulk_est_us(h, k, t) > chain_est_us(d, w_next) ? 32 : 0;
    }
    int lu_grid_user = 0;  // bqrrp_options.lu_grid_ctas (> 0: always that cap)
    Ctx& bulk_for(int64_t h, int64_t k, int64_t t, int64_t d, int64_t w_next, int num_sms) const
    {
        if (nparts == 0) return *bulk;
        if (part_always) return *bulk_part[0];
        const double bulk_us = bulk_est_us(h, k, t);
        const double chain_us = chain_est_us(d, w_next);
        Ctx* best = bulk;
        for (int i = 0; i < nparts; ++i)  // part_sms[] descending: the smallest partition that keeps up
            if (bulk_us * num_sms / part_sms[i] <= 1.15 * chain_us) best = bulk_part[i];
        return *best;
    }
};


// Buffers and steps of one factorization; the two schedules below compose the steps.
struct Run {
    Ctx& cx;
    const Sched& sc;
    int64_t m, n, b, d;
    double* A;
    int64_t lda;
    uint64_t seed;
    double* tau;
    int64_t* J;
    double rank_tol;
    int passes;
    bool hqr_fallback;
    int* hf;
    HostIO* hio;
    int64_t mn, bb;
    double *MskT, *Lb, *colscr, *rowscr, *Rsk11, *X, *ref, *Vp[2], *Tp, *W, *W2;
    double *Pn = nullptr, *W2g = nullptr;  // lookahead: the next panel (gathered), W2's gathered columns
    int *hs_state = nullptr, *hs_readers = nullptr, *post = nullptr;
    int64_t* vtmp;
    Touched T;
    int *ipiv, *perm;
    RskDefer rsk;
    std::vector<cudaEvent_t> evs;
    std::vector<cudaEvent_t> qevs;   // SketchQrPipe's event pool
    std::vector<cudaEvent_t> luevs;  // getrf_pivots_la's event pool

    Run(Ctx& cx_, const Sched& sc_, int64_t m_, int64_t n_, double* A_, int64_t lda_, int64_t b_, int64_t d_,
        uint64_t seed_, double* tau_, int64_t* J_, double rank_tol_, int passes_, bool hqr_, int* hf_, HostIO* hio_)
        : cx(cx_), sc(sc_), m(m_), n(n_), b(b_), d(d_), A(A_), lda(lda_), seed(seed_), tau(tau_), J(J_),
          rank_tol(rank_tol_), passes(passes_), hqr_fallback(hqr_), hf(hf_), hio(hio_)
    {
        mn = imin(m, n);
        bb = imin(b, mn);
        MskT = cx.alloc((size_t)n * d);
        Lb = cx.alloc((size_t)n * d);
        colscr = cx.alloc(imax(2 * d * m, m * d));
        rowscr = cx.alloc((size_t)2 * d * d);
        vtmp = cx.alloc_as<int64_t>((size_t)2 * d);
        T.tq = cx.alloc_as<int>((size_t)2 * d);
        T.tsrc = cx.alloc_as<int>((size_t)2 * d);
        T.nt = cx.alloc_as<int>(2);
        ipiv = cx.alloc_as<int>((size_t)d);
        perm = cx.alloc_as<int>((size_t)n);
        Rsk11 = cx.alloc((size_t)bb * bb);
        X = cx.alloc((size_t)bb * bb);
        ref = cx.alloc(1);
        Vp[0] = cx.alloc((size_t)m * bb);
        Vp[1] = sc.bulk ? cx.alloc((size_t)m * bb) : Vp[0];  // panel i+1 is built while bulk i reads V_i
        Tp = cx.alloc((size_t)bb * bb);
        W = cx.alloc((size_t)bb * n);
        W2 = cx.alloc((size_t)bb * n);
        if (sc.bulk) {
            rsk.side = sc.aux;
            rsk.Q = cx.alloc((size_t)d * d);
            rsk.Y = cx.alloc((size_t)n * d);
            Pn = cx.alloc((size_t)m * bb);
            W2g = cx.alloc((size_t)bb * bb);
            const size_t tiles = (size_t)cdiv(m, GEMM_FIXED_TILE) * (size_t)cdiv(n, GEMM_FIXED_TILE);
            hs_state = cx.alloc_as<int>(tiles);
            hs_readers = cx.alloc_as<int>(tiles);
            post = cx.alloc_as<int>((size_t)cdiv(m, GEMM_FIXED_TILE) * bb);
            BQ_CUDA(cudaMemsetAsync(hs_readers, 0, tiles * sizeof(int), cx.stream));
        }
    }
    ~Run()
    {
        for (auto e : evs) cudaEventDestroy(e);
        for (auto e : qevs) cudaEventDestroy(e);
        for (auto e : luevs) cudaEventDestroy(e);
    }
    cudaEvent_t event()
    {
        cudaEvent_t e;
        BQ_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
        evs.push_back(e);
        return e;
    }
    // `to` waits for the work queued so far on `from`
    void join(cudaStream_t to, cudaStream_t from)
    {
        cudaEvent_t e = event();
        BQ_CUDA(cudaEventRecord(e, from));
        BQ_CUDA(cudaStreamWaitEvent(to, e, 0));
    }

    // O2 + a1: J = 1..n, tau = 0, flags, the sketch (host entry: per uploaded column chunk)
    void prologue()
    {
        cx.mark(PH_OTHER);
        init_j_kernel<<<(unsigned)imin(cdiv(n, 256), 1024), 256, 0, cx.stream>>>(n, J);
        BQ_LAUNCH_CHECK();
        BQ_CUDA(cudaMemsetAsync(tau, 0, sizeof(double) * mn, cx.stream));
        BQ_CUDA(cudaMemsetAsync(cx.flags, 0, sizeof(int) * F_NFLAGS, cx.stream));
        if (hio) {  // S^T lives in the column scratch until the loop starts
            sketch_operator_T(cx, m, d, seed, colscr, m);
            // 64 chunks: the first sketch GEMM waits for 1/64 of A instead of 1/16 (C3: ~10 instead of ~40 ms of PCIe)
            const int64_t chunk = imax(b, cdiv(n, 64));
            for (int64_t c0 = 0; c0 < n; c0 += chunk) {
                const int64_t nc = imin(chunk, n - c0);
                BQ_CUDA(cudaMemcpy2DAsync(A + c0 * lda, lda * sizeof(double), hio->A_in + c0 * hio->ld_host,
                                          hio->ld_host * sizeof(double), m * sizeof(double), nc,
                                          cudaMemcpyHostToDevice, hio->h2d));
                cudaEvent_t e = hio->event();
                BQ_CUDA(cudaEventRecord(e, hio->h2d));
                BQ_CUDA(cudaStreamWaitEvent(cx.stream, e, 0));
                gemm(cx, true, false, nc, d, m, 1.0, A + c0 * lda, lda, colscr, m, 0.0, MskT + c0, n, false, 0,
                     /*no_split=*/true);  // MskT rows (no split-K: bitwise the device entry's one-GEMM sketch)
            }
        } else {
            sketch_apply(cx, m, n, A, lda, d, seed, MskT, n, colscr);
        }
        nonfinite_kernel<<<(unsigned)imin(cdiv(n * d, 256), 4 * cx.num_sms), 256, 0, cx.stream>>>(n, d, MskT, n,
                                                                                                    cx.flags);
        BQ_LAUNCH_CHECK();
    }

    // a2 on the window at s (Alg. 2): LU pivots of the sketch transpose, the touched set of J_qr,
    // sketch rows permuted, R_sk (its (w-d) x d GEMM part deferred to aux in the lookahead), tri_rank -> flags
    void pivots(int64_t i, int64_t s)
    {
        const int64_t w = n - s, kmax = imin(imin(b, w), m - s);
        cx.mark(PH_QRCP_WIDE);
        copy_matrix(cx, w, d, MskT + s, n, Lb, n);
        if (sc.qr) {  // K-SQR pipelined with K-LU (left-looking, its own stream)
            SketchQrPipe P;
            sketch_qr_pipe_begin(P, cx, *sc.qr, qevs, MskT + s, n, w, d, sc.qr2);
            const LeafDone on_leaf = [&](int64_t c1) { sketch_qr_pipe_columns(P, perm, c1); };
            if (!(sc.lu2 && getrf_pivots_la(cx, *sc.lu2, luevs, Lb, n, w, d, ipiv, perm, &on_leaf)))
                getrf_pivots(cx, Lb, n, w, d, ipiv, perm, &on_leaf);
            touched_from_perm(cx, w, imin(w, d), perm, T);
            permute_rows(cx, d, MskT + s, n, T, rowscr);
            sketch_qr_pipe_finish(P, &rsk);
        } else {
            getrf_pivots(cx, Lb, n, w, d, ipiv, perm);
            touched_from_perm(cx, w, imin(w, d), perm, T);
            permute_rows(cx, d, MskT + s, n, T, rowscr);
            sketch_qr(cx, MskT + s, n, w, d, RowBlocks(), sc.bulk ? &rsk : nullptr);
        }
        cx.mark(PH_TRI_RANK);
        tri_rank_kernel<<<1, 1024, 0, cx.stream>>>(MskT + s, n, kmax, i == 0, rank_tol, ref, cx.flags);
        BQ_LAUNCH_CHECK();
    }

    // a3: columns of A(0:m, s:n) and J(s:n) gathered by J_qr (touched set only)
    void permute(int64_t s)
    {
        cx.mark(PH_COL_PERM);
        permute_columns(cx, m, A + s * lda, lda, T, colscr);
        permute_vector(cx, J + s, T, vtmp);
    }

    // the zero-column test (reading Z12) of a column of h rows, then the loop's one host read of
    // {k, zero flag, non-finite flag, POTRF breakdown}.  Returns false on a numerical failure.
    bool check(int64_t h, const double* col)
    {
        zero_col_kernel<<<(unsigned)imin(cdiv(h, 256), 64), 256, 0, cx.stream>>>(h, col, cx.flags);
        BQ_LAUNCH_CHECK();
        BQ_CUDA(cudaMemcpyAsync(hf, cx.flags, sizeof(int) * F_NFLAGS, cudaMemcpyDeviceToHost, cx.stream));
        BQ_CUDA(cudaStreamSynchronize(cx.stream));
        return !(hf[F_NONFINITE] || hf[F_POTRF_INFO]);
    }

    // a4 (Alg. 3) on the panel Ap (h x k, ld), tau(s:s+k); V, T into Vp[slot], Tp
    void panel(int64_t s, int64_t h, int64_t k, double* Ap, int64_t ld, int slot)
    {
        cx.mark(PH_QR_TALL);
        extract_rsk11_kernel<<<(unsigned)imin(cdiv(k * k, 256), 4 * cx.num_sms), 256, 0, cx.stream>>>(k, MskT + s, n,
                                                                                                        Rsk11);
        BQ_LAUNCH_CHECK();
        g_panel_fallbacks += panel_factor(cx, h, Ap, ld, k, Rsk11, tau + s, passes, Vp[slot], Tp, hqr_fallback,
                                          sc.aux);
    }

    // a6's X = R_sk11 R11^{-1} (b x b; R11 = A(s:s+b, s:s+b), upper), on aux when there is one
    cudaEvent_t sample_x(int64_t s)
    {
        if (!sc.aux) {
            copy_matrix(cx, b, b, Rsk11, b, X, b);
            trsm_right_upper(cx, b, b, A + s + s * lda, lda, false, false, X, b);
            zero_triangle(cx, 'U', b, b, X, b);
            return nullptr;
        }
        join(sc.aux->stream, cx.stream);
        Ctx ac = side_ctx(cx, *sc.aux, 0);  // allocates nothing (substitution TRSM)
        copy_matrix(ac, b, b, Rsk11, b, X, b);
        trsm_right_upper(ac, b, b, A + s + s * lda, lda, false, false, X, b);
        zero_triangle(ac, 'U', b, b, X, b);
        cudaEvent_t e = event();
        BQ_CUDA(cudaEventRecord(e, sc.aux->stream));
        return e;
    }

    // a6: MskT(c:n, 0:b) -= R12^T X^T
    void sample_update(int64_t s, int64_t c, cudaEvent_t ex)
    {
        cx.mark(PH_SAMPLE_UPDATE);
        if (ex) BQ_CUDA(cudaStreamWaitEvent(cx.stream, ex, 0));
        gemm(cx, true, true, n - c, b, b, -1.0, A + s + c * lda, lda, X, b, 1.0, MskT + c, n);
    }
};

// One stream, Alg. 1 in order (no_lookahead).
static int64_t loop_serial(Run& R)
{
    Ctx& cx = R.cx;
    const int64_t m = R.m, n = R.n, b = R.b;
    for (int64_t i = 0;; ++i) {
        const int64_t s = i * b;
        if (s >= R.mn) return R.mn;
        const int64_t c = imin(n, s + b), r = imin(m, s + b), w = n - s, h = m - s;
        const int64_t kmax = imin(imin(b, w), h);
        R.pivots(i, s);
        R.permute(s);
        if (!R.check(h, R.A + s + s * R.lda)) return -1;
        const int64_t k = R.hf[F_K];
        if (k == 0 || R.hf[F_ZERO_COL]) return s;
        R.panel(s, h, k, R.A + s + s * R.lda, R.lda, 0);
        cx.mark(PH_APPLY_QT);
        const bool terminal = (k < kmax || c == n || r == m);
        if (R.hio && !terminal) R.hio->flush(cx.stream, m, R.A, R.lda, c);
        wy_update(cx, h, k, n - s - k, R.Vp[0], h, R.Tp, R.A + s + (s + k) * R.lda, R.lda, R.W, R.W2);
        if (terminal) return s + k;
        R.sample_x(s);
        R.sample_update(s, c, nullptr);
    }
}

// The pivot-aware lookahead.  Iteration i, with panel i factored:
//   crit: GEMM1 W = V^T C, W2 = T^T W, R12 rows -> [bulk stream: C(k:h) -= V(k:h) W2, tile handshake]
//   crit: a6 (X from aux), a2 of i+1 (R_sk GEMM on aux), then the next panel's columns gathered from the
//         trailing block while the bulk runs (la_gather_pre / _post around the same update of just those
//         columns, bitwise the bulk's), the host read of k, panel i+1 on the gathered copy
//   crit: wait for the bulk, a3 of i+1 on A and J, the factored panel copied into place.
// So panel i+1 (and the latency-bound pivot selection) overlaps the bulk GEMM of iteration i; only GEMM1, the
// permutation and the copy are serial.
static int64_t loop_lookahead(Run& R)
{
    Ctx& cx = R.cx;
    const Sched& sc = R.sc;
    const int64_t m = R.m, n = R.n, b = R.b;
    double* A = R.A;
    const int64_t lda = R.lda;
    // iteration 0: pivots, permutation, panel in place
    R.pivots(0, 0);
    R.permute(0);
    if (!R.check(m, A)) return -1;
    int64_t k = R.hf[F_K];
    if (k == 0 || R.hf[F_ZERO_COL]) return 0;
    R.panel(0, m, k, A, lda, 0);
    for (int64_t i = 0;; ++i) {
        const int64_t s = i * b, slot = i & 1;
        const int64_t c = imin(n, s + b), r = imin(m, s + b), w = n - s, h = m - s;
        const int64_t kmax = imin(imin(b, w), h);
        const bool terminal = (k < kmax || c == n || r == m);
        if (R.hio && !terminal) R.hio->flush(cx.stream, m, A, lda, c);  // block column [s, c) is final
        double* V = R.Vp[slot];
        double* C = A + s + (s + k) * lda;
        const int64_t t = n - s - k;
        cx.mark(PH_APPLY_QT);
        if (terminal) {
            wy_update(cx, h, k, t, V, h, R.Tp, C, lda, R.W, R.W2);
            return s + k;
        }
        // ---- a5: critical part, then the bulk rows on the bulk stream (k == b here)
        cudaEvent_t ex = R.sample_x(s);
        const int64_t tiles_m = cdiv(h - k, GEMM_FIXED_TILE), tiles_n = cdiv(t, GEMM_FIXED_TILE);
        BQ_CUDA(cudaMemsetAsync(R.hs_state, 0, sizeof(int) * tiles_m * tiles_n, cx.stream));
        wy_top(cx, h, k, t, V, h, R.Tp, C, lda, R.W, R.W2, /*rows=*/k);
        BQ_CUDA(cudaEventRecord(sc.ev_top, cx.stream));
        Ctx& bk = sc.panel_la == 1 ? *sc.bulk : sc.bulk_for(h, k, t, R.d, n - c, cx.num_sms);
        BQ_CUDA(cudaStreamWaitEvent(bk.stream, sc.ev_top, 0));
        if (bk.timer) bk.timer->begin_interval(bk.stream, PH_APPLY_QT_BULK);
        wy_bulk(bk, h, k, t, V, h, R.W2, C, lda, R.hs_state, R.hs_readers);
        if (bk.timer) bk.timer->end_interval(bk.stream);
        BQ_CUDA(cudaEventRecord(sc.ev_bulk, bk.stream));
        // ---- a6, then a2 of the next iteration (overlapping the bulk)
        R.sample_update(s, c, ex);
        const int64_t s1 = c, h1 = m - s1, w1 = n - s1;
        const int64_t kmax1 = imin(imin(b, w1), h1);
        cx.lu_grid_max = sc.lu_grid_for(h, k, t, R.d, w1);
        R.pivots(i + 1, s1);
        double* Cb = A + s1 + s1 * lda;  // = C + k rows: the bulk's rows, columns from the next window's start
        if (sc.panel_la != 1) {
            // (default: measured faster than the overlapped form at C2 and C3, profiles/schedule_ab_r02.json)
            // ---- panel i+1 after the bulk, in place (Alg. 1 order): a3, the zero test, a4
            BQ_CUDA(cudaStreamWaitEvent(cx.stream, sc.ev_bulk, 0));
            R.permute(s1);
            if (!R.check(h1, Cb)) return -1;
            const int64_t k1 = R.hf[F_K];
            if (k1 == 0 || R.hf[F_ZERO_COL]) return s1;
            R.panel(s1, h1, k1, Cb, lda, (int)(slot ^ 1));
            k = k1;
            continue;
        }
        // ---- the next panel's columns: P(:, q) = C(k:h, perm[q]) - V(k:h) W2(:, perm[q]), q < kmax1
        cx.mark(PH_QR_TALL);
        la_gather_pre(cx, h1, Cb, lda, R.perm, kmax1, tiles_n, R.hs_state, R.hs_readers, R.Pn, h1, R.post);
        gather_cols_idx(cx, k, R.W2, k, R.perm, kmax1, R.W2g, k);
        GemmExtra fixed;
        fixed.fixed_tiles = true;  // the bulk's tiling: bitwise the bulk's values for these columns
        gemm(cx, false, false, h1, kmax1, k, -1.0, V + k, h, R.W2g, k, 1.0, R.Pn, h1, false, 0, true, &fixed);
        la_gather_post(cx, h1, Cb, lda, R.perm, kmax1, tiles_n, R.hs_state, R.Pn, h1, R.post);
        if (!R.check(h1, R.Pn)) return -1;
        const int64_t k1 = R.hf[F_K];
        if (k1 == 0 || R.hf[F_ZERO_COL]) {  // early exit after the permutation (oracle O3 f, g)
            BQ_CUDA(cudaStreamWaitEvent(cx.stream, sc.ev_bulk, 0));
            R.permute(s1);
            return s1;
        }
        R.panel(s1, h1, k1, R.Pn, h1, (int)(slot ^ 1));
        // ---- a3 of i+1 once the bulk has landed, and the factored panel into place
        BQ_CUDA(cudaStreamWaitEvent(cx.stream, sc.ev_bulk, 0));
        R.permute(s1);
        copy_matrix(cx, h1, k1, R.Pn, h1, Cb, lda);
        k = k1;
    }
}

static int64_t factor_impl(Ctx& cx, const Sched& sc, int64_t m, int64_t n, double* A, int64_t lda, int64_t b,
                           int64_t d, uint64_t seed, double* tau, int64_t* J, double rank_tol, int passes,
                           bool hqr_fallback, int* host_flags, HostIO* hio = nullptr)
{
    Run R(cx, sc, m, n, A, lda, b, d, seed, tau, J, rank_tol, passes, hqr_fallback, host_flags, hio);
    R.prologue();
    int64_t ell = sc.bulk ? loop_lookahead(R) : loop_serial(R);
    if (ell < 0) return -1;
    // O4: tau(ell:) = 0, A(ell:m, ell:n) = 0 (reading Z16)
    cx.mark(PH_OTHER);
    if (sc.bulk) BQ_CUDA(cudaStreamWaitEvent(cx.stream, sc.ev_bulk, 0));
    if (sc.aux) R.join(cx.stream, sc.aux->stream);
    const int64_t mn = R.mn;
    if (ell < mn) BQ_CUDA(cudaMemsetAsync(tau + ell, 0, sizeof(double) * (mn - ell), cx.stream));
    set_zero(cx, m - ell, n - ell, A + ell + ell * lda, lda);
    if (hio) hio->flush(cx.stream, m, A, lda, n);
    cx.mark(PH_OTHER);
    BQ_CUDA(cudaMemcpyAsync(host_flags, cx.flags, sizeof(int) * F_NFLAGS, cudaMemcpyDeviceToHost, cx.stream));
    BQ_CUDA(cudaStreamSynchronize(cx.stream));
    if (host_flags[F_NONFINITE] || host_flags[F_POTRF_INFO]) return -1;
    return ell;
}

int* pinned_flags()
{
    static thread_local int* p = nullptr;
    if (!p) BQ_CUDA(cudaMallocHost(&p, sizeof(int) * F_NFLAGS));
    return p;
}

void setup_ctx(Ctx& cx, void* stream)
{
    cx.stream = (cudaStream_t)stream;
    int dev = 0;
    BQ_CUDA(cudaGetDevice(&dev));
    BQ_CUDA(cudaDeviceGetAttribute(&cx.num_sms, cudaDevAttrMultiProcessorCount, dev));
}

// Carve splitk + flags from the tail of the workspace.
void carve(Ctx& cx, void* ws, size_t bytes, const Layout& L)
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
        cx.force_breakdown = opts && (opts->debug_flags & BQRRP_DEBUG_FORCE_BREAKDOWN);
        if (opts && (opts->lu_leaf_cluster == 4 || opts->lu_leaf_cluster == 8 || opts->lu_leaf_cluster == 16))
            cx.lu_gpref = opts->lu_leaf_cluster;
        if (opts && opts->lu_grid_ctas > 0) cx.lu_grid_max = opts->lu_grid_ctas;  // (lookahead: per iteration)
        if (m == 0 || n == 0) {
            *rank = 0;
            if (n > 0) {
                init_j_kernel<<<(unsigned)imin(cdiv(n, 256), 1024), 256, 0, cx.stream>>>(n, J);
                BQ_LAUNCH_CHECK();
            }
            return 0;
        }
        // shape limits of the leaf kernels, before any launch
        if (n > lu_max_rows(cx.num_sms)) {
            g_last_error = "n = " + std::to_string(n) + " exceeds the K-LU grid leaf's capacity (" +
                           std::to_string(lu_max_rows(cx.num_sms)) + " sketch rows)";
            return -2;
        }
        if (m > qr_max_rows(cx.num_sms) && (passes == 0 || !(opts && opts->no_hqr_fallback))) {
            g_last_error = "m = " + std::to_string(m) + " exceeds the Householder panel's capacity (" +
                           std::to_string(qr_max_rows(cx.num_sms)) + " rows; needed by cholqr_passes = 0 and by the "
                           "CholQR-breakdown fallback: set no_hqr_fallback)";
            return -1;
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
        // critical chain and its helper (aux) on high-priority streams, the bulk trailing GEMM on a
        // low-priority one (Sched); all joined to the caller's stream at entry and exit
        int prio_lo = 0, prio_hi = 0;
        BQ_CUDA(cudaDeviceGetStreamPriorityRange(&prio_lo, &prio_hi));
        cudaStream_t user = cx.stream, s_hi = nullptr, s_lo = nullptr, s_aux = nullptr, s_qr = nullptr, s_lu = nullptr,
                     s_qr2 = nullptr;
        cudaEvent_t ev_in = nullptr, ev_top = nullptr, ev_bulk = nullptr, ev_done = nullptr;
        BQ_CUDA(cudaStreamCreateWithPriority(&s_hi, cudaStreamNonBlocking, prio_hi));
        BQ_CUDA(cudaStreamCreateWithPriority(&s_lo, cudaStreamNonBlocking, prio_lo));
        BQ_CUDA(cudaStreamCreateWithPriority(&s_aux, cudaStreamNonBlocking, prio_hi));
        BQ_CUDA(cudaStreamCreateWithPriority(&s_qr, cudaStreamNonBlocking, prio_hi));
        BQ_CUDA(cudaStreamCreateWithPriority(&s_lu, cudaStreamNonBlocking, prio_hi));
        BQ_CUDA(cudaStreamCreateWithPriority(&s_qr2, cudaStreamNonBlocking, prio_hi));
        BQ_CUDA(cudaEventCreateWithFlags(&ev_in, cudaEventDisableTiming));
        BQ_CUDA(cudaEventCreateWithFlags(&ev_top, cudaEventDisableTiming));
        BQ_CUDA(cudaEventCreateWithFlags(&ev_bulk, cudaEventDisableTiming));
        BQ_CUDA(cudaEventCreateWithFlags(&ev_done, cudaEventDisableTiming));
        BQ_CUDA(cudaEventRecord(ev_in, user));
        for (cudaStream_t st : {s_hi, s_lo, s_aux, s_qr, s_lu, s_qr2}) BQ_CUDA(cudaStreamWaitEvent(st, ev_in, 0));
        cx.stream = s_hi;
        Ctx cxb = cx, cxa = cx, cxq = cx, cxl = cx, cxq2 = cx;
        cxb.stream = s_lo;
        cxa.stream = s_aux;
        cxq.stream = s_qr;
        cxl.stream = s_lu;
        cxq2.stream = s_qr2;
        for (Ctx* c : {&cxb, &cxa, &cxq, &cxl, &cxq2}) {  // the split-K scratch belongs to the critical stream
            c->splitk = nullptr;
            c->splitk_elems = 0;
        }
        cxa.timer = nullptr;
        cxq.timer = nullptr;
        cxq.ws = nullptr;  // the pipelined sketch QR's stream allocates nothing (its buffers come from cx)
        cxq.ws_bytes = cxq.ws_used = 0;
        cxl.timer = nullptr;
        cxl.ws = nullptr;  // nor does the lookahead LU's update stream
        cxl.ws_bytes = cxl.ws_used = 0;
        cxq2.timer = nullptr;
        cxq2.ws = nullptr;  // nor the sketch QR's T-merge stream
        cxq2.ws_bytes = cxq2.ws_used = 0;
        Ctx cxp[3] = {cxb, cxb, cxb};
        cudaStream_t s_parts[3] = {};
        int part_sms[3] = {}, nparts = 0;
        const int bulk_sms = opts ? opts->bulk_sms : 0;
        if (bulk_sms >= 0 && !(opts && opts->no_lookahead)) {
            // auto (0): partitions of 132 / 116 / 100 SMs (on 148), chosen per iteration (Sched::bulk_for)
            const int req[3] = {cx.num_sms - 16, cx.num_sms - 32, cx.num_sms - 48};
            for (int i = 0; i < (bulk_sms > 0 ? 1 : 3); ++i) {
                int got = 0;
                cudaStream_t st = green_stream(bulk_sms > 0 ? bulk_sms : req[i], &got);
                if (!st || got <= 0 || got >= cx.num_sms) continue;
                BQ_CUDA(cudaStreamWaitEvent(st, ev_in, 0));
                s_parts[nparts] = st;
                part_sms[nparts] = got;
                cxp[nparts].stream = st;
                ++nparts;
            }
        }
        Timer tm;
        if (opts && opts->phase_ms) {
            tm.on = true;
            tm.st = s_hi;
            cx.timer = &tm;
            cxb.timer = &tm;
            for (Ctx& c : cxp) c.timer = &tm;
        }
        Sched sc;
        if (!(opts && opts->no_lookahead)) {
            sc.bulk = &cxb;
            sc.aux = &cxa;
            sc.ev_top = ev_top;
            sc.ev_bulk = ev_bulk;
            sc.panel_la = opts ? opts->panel_lookahead : 0;
            sc.lu_grid_user = opts ? opts->lu_grid_ctas : 0;
            if (!(opts && opts->no_sqr_pipeline)) {
                sc.qr = &cxq;
                // the T-merge stream pays where the sketch-QR chain is on the critical path (d <= 1024: C2 -0.6 %,
                // 4096^2..8192^2 -2 %); at d = 2048 (C3) the pivot selection hides behind the bulk GEMM and the
                // extra stream only adds contention (+0.1-0.3 %, profiles/r02/sqr_merge_stream_ab_r02.txt)
                if (!(opts && opts->no_sqr_merge_stream) && d <= 1024) sc.qr2 = &cxq2;
                if (opts && opts->lu_lookahead) sc.lu2 = &cxl;
            }
            for (int i = 0; i < nparts; ++i) {
                sc.bulk_part[i] = &cxp[i];
                sc.part_sms[i] = part_sms[i];
            }
            sc.nparts = nparts;
            sc.part_always = bulk_sms > 0;
        }
        int64_t ell = -1;
        int status = 0;
        auto cleanup = [&]() {
            for (cudaStream_t st : {s_hi, s_lo, s_aux, s_qr, s_lu, s_qr2, s_parts[0], s_parts[1], s_parts[2]}) {
                if (!st) continue;
                cudaEventRecord(ev_done, st);
                cudaStreamWaitEvent(user, ev_done, 0);
            }
            for (cudaStream_t st : {s_hi, s_lo, s_aux, s_qr, s_lu, s_qr2}) cudaStreamDestroy(st);
            for (cudaEvent_t e : {ev_in, ev_top, ev_bulk, ev_done}) cudaEventDestroy(e);
            cx.stream = user;
        };
        try {
            ell = factor_impl(cx, sc, m, n, A, lda, b, d, seed, tau, J, rank_tol, passes,
                              !(opts && opts->no_hqr_fallback), pinned_flags(), hio);
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

int bqrrp_debug_permute_touched(int64_t rows, double* X, int64_t ldx, int64_t nt, const int* tq, const int* tsrc,
                                void* stream)
{
    if (rows < 0) return -1;
    if (!X && rows > 0 && nt > 0) return -2;
    if (ldx < (rows > 1 ? rows : 1)) return -3;
    if (nt < 0) return -4;
    if ((!tq || !tsrc) && nt > 0) return -5;
    return guarded([&]() -> int {
        Ctx cx;
        setup_ctx(cx, stream);
        if (nt == 0 || rows == 0) return 0;
        size_t wsb = (size_t)4096 + (size_t)nt * (size_t)rows * 8 + 256;
        void* ws = nullptr;
        BQ_CUDA(lib_malloc_async(&ws, wsb, cx.stream));
        Layout Ly{0, 0, 0, 0};
        carve(cx, ws, wsb, Ly);
        Touched T;
        T.tq = const_cast<int*>(tq);
        T.tsrc = const_cast<int*>(tsrc);
        T.nt = cx.flags + F_NT;
        T.maxnt = nt;
        const int ntv = (int)nt;
        BQ_CUDA(cudaMemcpyAsync(T.nt, &ntv, sizeof(int), cudaMemcpyHostToDevice, cx.stream));
        double* scr = cx.alloc((size_t)nt * rows);
        permute_columns(cx, rows, X, ldx, T, scr);
        BQ_CUDA(cudaFreeAsync(ws, cx.stream));
        return 0;
    });
}

int bqrrp_debug_potrf(int64_t n, double* G, int64_t ldg, void* stream)
{
    if (n < 0) return -1;
    if (!G && n > 0) return -2;
    if (ldg < (n > 1 ? n : 1)) return -3;
    return guarded([&]() -> int {
        Ctx cx;
        setup_ctx(cx, stream);
        if (n == 0) return 0;
        const size_t sk = (size_t)16 * n * n + (4u << 20) / 8;
        const size_t bytes = (sk + (size_t)cdiv(n, 64) * 4096 + 8192) * 8;
        void* ws = nullptr;
        BQ_CUDA(lib_malloc_async(&ws, bytes, cx.stream));
        Layout Ly{0, 0, sk * 8, 0};
        carve(cx, ws, bytes, Ly);
        BQ_CUDA(cudaMemsetAsync(cx.flags, 0, sizeof(int) * F_NFLAGS, cx.stream));
        potrf_lower(cx, n, G, ldg);
        int* hf = pinned_flags();
        BQ_CUDA(cudaMemcpyAsync(hf, cx.flags, sizeof(int) * F_NFLAGS, cudaMemcpyDeviceToHost, cx.stream));
        BQ_CUDA(cudaFreeAsync(ws, cx.stream));
        BQ_CUDA(cudaStreamSynchronize(cx.stream));
        return hf[F_POTRF_INFO] ? BQRRP_ENUMERIC : 0;
    });
}

int bqrrp_debug_recon_lu(int64_t k, const double* Qtop, int64_t ldq, const double* C, double* Wr, double* S,
                         void* stream)
{
    if (k < 1) return -1;
    if (!Qtop) return -2;
    if (ldq < k) return -3;
    if (!C) return -4;
    if (!Wr) return -5;
    if (!S) return -6;
    return guarded([&]() -> int {
        Ctx cx;
        setup_ctx(cx, stream);
        const size_t sk = (size_t)16 * k * k + (4u << 20) / 8;
        const size_t bytes = (sk + (size_t)cdiv(k, 64) * 4096 * 2 + 8192) * 8;
        void* ws = nullptr;
        BQ_CUDA(lib_malloc_async(&ws, bytes, cx.stream));
        Layout Ly{0, 0, sk * 8, 0};
        carve(cx, ws, bytes, Ly);
        recon_top_lu(cx, k, Qtop, ldq, C, Wr, S);
        BQ_CUDA(cudaFreeAsync(ws, cx.stream));
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
        panel_factor(cx, h, P, ld, k, Rsk11, tau, cholqr_passes, V, Tb);
        wy_update(cx, h, k, t, V, h, Tb, P + k * ld, ld, W, W2);
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

unsigned long long bqrrp_launch_count(void) { return g_launches.load(); }

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
