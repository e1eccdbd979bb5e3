// steps.cu — step-level C-ABI entry points used by the multi-GPU driver (paper_2507_00976_b200/dist.py,
// SURVEY §8(e)): A is distributed 1-D block-cyclically over column positions; the sketch is replicated;
// each function below is one step of Alg. 1 on one rank's data.  Collectives (the sketch all-gather X1,
// the panel broadcast X2, the column exchange X3) are issued by the caller through torch.distributed
// (NCCL on a multi-GPU node); every arithmetic step runs in this library's kernels.
#include <cstring>
#include <string>

#include "../../include/bqrrp.h"
#include "blas.cuh"
#include "bqrrp_internal.cuh"

namespace bqrrp {

// dst(:, t) = X(:, idx[t]) for idx[t] >= 0 (else the slot is left untouched); rows x n_idx.
__global__ void gather_idx_kernel(int64_t rows, const double* __restrict__ X, int64_t ldx, const int* __restrict__ idx,
                                  int64_t nidx, double* __restrict__ dst, int64_t ldd)
{
    int64_t t = blockIdx.y;
    if (t >= nidx) return;
    int j = idx[t];
    if (j < 0) return;
    const double* s = X + (int64_t)j * ldx;
    double* d = dst + t * ldd;
    for (int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; r < rows; r += (int64_t)gridDim.x * blockDim.x)
        d[r] = s[r];
}

__global__ void scatter_idx_kernel(int64_t rows, double* __restrict__ X, int64_t ldx, const int* __restrict__ idx,
                                   int64_t nidx, const double* __restrict__ src, int64_t lds)
{
    int64_t t = blockIdx.y;
    if (t >= nidx) return;
    int j = idx[t];
    if (j < 0) return;
    double* d = X + (int64_t)j * ldx;
    const double* s = src + t * lds;
    for (int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; r < rows; r += (int64_t)gridDim.x * blockDim.x)
        d[r] = s[r];
}

__global__ void tri_rank_step_kernel(const double* MskT_s, int64_t ldm, int64_t kmax, int first, double rank_tol,
                                     double* ref, int* kout)
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
        *kout = first_fail;
    }
}

__global__ void extract_rsk_kernel(int64_t k, const double* MskT_s, int64_t ldm, double* R)
{
    int64_t total = k * k;
    for (int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; idx < total; idx += (int64_t)gridDim.x * blockDim.x) {
        int64_t i = idx % k, j = idx / k;
        R[idx] = (i <= j) ? MskT_s[j + i * ldm] : 0.0;
    }
}

__global__ void zero_check_kernel(int64_t h, const double* col, int* out)
{
    bool nz = false;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < h; i += (int64_t)gridDim.x * blockDim.x)
        if (col[i] != 0.0) nz = true;
    if (__syncthreads_or(nz) && threadIdx.x == 0) *out = 0;
}

static thread_local std::string g_step_error;

template <typename F>
static int step_guard(F&& f)
{
    try {
        return f();
    } catch (const std::exception& e) {
        g_step_error = e.what();
        return BQRRP_ECUDA;
    }
}

struct StepWs {
    Ctx cx;
    void* ws = nullptr;
    StepWs(void* stream, size_t bytes, size_t splitk_bytes)
    {
        cx.stream = (cudaStream_t)stream;
        int dev = 0;
        BQ_CUDA(cudaGetDevice(&dev));
        BQ_CUDA(cudaDeviceGetAttribute(&cx.num_sms, cudaDevAttrMultiProcessorCount, dev));
        size_t total = bytes + splitk_bytes + 4096;
        BQ_CUDA(lib_malloc_async(&ws, total, cx.stream));
        cx.ws = (char*)ws;
        cx.ws_bytes = total;
        cx.ws_used = 0;
        cx.splitk = cx.alloc(splitk_bytes / 8);
        cx.splitk_elems = splitk_bytes / 8;
        cx.flags = cx.alloc_as<int>(F_NFLAGS);
        BQ_CUDA(cudaMemsetAsync(cx.flags, 0, sizeof(int) * F_NFLAGS, cx.stream));
    }
    ~StepWs()
    {
        if (ws) cudaFreeAsync(ws, cx.stream);
    }
};

}  // namespace bqrrp

using namespace bqrrp;

extern "C" {

static int step_pivots_impl(int64_t n, int64_t d, int64_t s, int64_t kmax, double* MskT, int64_t ldm, int64_t* J,
                            double rank_tol, double* ref, int first, int* tq, int* tsrc, int* nt, int64_t* k_out,
                            const RowBlocks& rows, void* stream);

int bqrrp_step_pivots(int64_t n, int64_t d, int64_t s, int64_t kmax, double* MskT, int64_t ldm, int64_t* J,
                      double rank_tol, double* ref, int first, int* tq, int* tsrc, int* nt, int64_t* k_out,
                      void* stream)
{
    return step_pivots_impl(n, d, s, kmax, MskT, ldm, J, rank_tol, ref, first, tq, tsrc, nt, k_out, RowBlocks(),
                            stream);
}

int bqrrp_step_pivots_rows(int64_t n, int64_t d, int64_t s, int64_t kmax, double* MskT, int64_t ldm, int64_t* J,
                           double rank_tol, double* ref, int first, int* tq, int* tsrc, int* nt, int64_t* k_out,
                           const int64_t* row_off, const int64_t* row_len, int64_t n_rows, void* stream)
{
    if (n_rows < 0 || (n_rows > 0 && (!row_off || !row_len))) return -17;
    RowBlocks rb;
    rb.off = row_off;
    rb.len = row_len;
    rb.n = n_rows;
    return step_pivots_impl(n, d, s, kmax, MskT, ldm, J, rank_tol, ref, first, tq, tsrc, nt, k_out, rb, stream);
}

static int step_pivots_impl(int64_t n, int64_t d, int64_t s, int64_t kmax, double* MskT, int64_t ldm, int64_t* J,
                            double rank_tol, double* ref, int first, int* tq, int* tsrc, int* nt, int64_t* k_out,
                            const RowBlocks& rows, void* stream)
{
    if (n < 1) return -1;
    if (d < 1) return -2;
    if (s < 0 || s >= n) return -3;
    if (!MskT || ldm < n) return -6;
    return step_guard([&]() -> int {
        const int64_t w = n - s, nlu = imin(w, d);
        size_t bytes = ((size_t)w * d + (size_t)d * d * 8 + (size_t)2 * d * d + (size_t)w * d + 4 * (size_t)n + 8 * d +
                        (size_t)2 * 160 * 33 + 160 * 32 * 32 + 4096) * 8;
        StepWs sw(stream, bytes, (size_t)16 * d * d * 8 + (4u << 20));
        Ctx& cx = sw.cx;
        double* Lb = cx.alloc((size_t)w * d);
        int* ipiv = cx.alloc_as<int>((size_t)d);
        int* perm = cx.alloc_as<int>((size_t)w);
        double* rowscr = cx.alloc((size_t)2 * d * d);
        int64_t* vtmp = cx.alloc_as<int64_t>((size_t)2 * d);
        int* kdev = cx.alloc_as<int>(2);
        Touched T;
        T.tq = tq;
        T.tsrc = tsrc;
        T.nt = nt;
        copy_matrix(cx, w, d, MskT + s, ldm, Lb, w);
        getrf_pivots(cx, Lb, w, w, d, ipiv, perm);
        touched_from_perm(cx, w, nlu, perm, T);
        permute_rows(cx, d, MskT + s, ldm, T, rowscr);
        if (J) permute_vector(cx, J + s, T, vtmp);
        sketch_qr(cx, MskT + s, ldm, w, d, rows);
        tri_rank_step_kernel<<<1, 1024, 0, cx.stream>>>(MskT + s, ldm, kmax, first, rank_tol, ref, kdev);
        BQ_LAUNCH_CHECK();
        int kh = 0;
        BQ_CUDA(cudaMemcpyAsync(&kh, kdev, sizeof(int), cudaMemcpyDeviceToHost, cx.stream));
        BQ_CUDA(cudaStreamSynchronize(cx.stream));
        *k_out = kh;
        return 0;
    });
}

int bqrrp_step_gather_columns(int64_t rows, const double* X, int64_t ldx, const int* idx, int64_t nidx, double* dst,
                              int64_t ldd, void* stream)
{
    if (rows < 0) return -1;
    if (nidx < 0) return -5;
    if (rows == 0 || nidx == 0) return 0;
    return step_guard([&]() -> int {
        dim3 grid((unsigned)imin(cdiv(rows, 256 * 8), 64), (unsigned)nidx);
        gather_idx_kernel<<<grid, 256, 0, (cudaStream_t)stream>>>(rows, X, ldx, idx, nidx, dst, ldd);
        BQ_LAUNCH_CHECK();
        return 0;
    });
}

int bqrrp_step_scatter_columns(int64_t rows, double* X, int64_t ldx, const int* idx, int64_t nidx, const double* src,
                               int64_t lds, void* stream)
{
    if (rows < 0) return -1;
    if (nidx < 0) return -5;
    if (rows == 0 || nidx == 0) return 0;
    return step_guard([&]() -> int {
        dim3 grid((unsigned)imin(cdiv(rows, 256 * 8), 64), (unsigned)nidx);
        scatter_idx_kernel<<<grid, 256, 0, (cudaStream_t)stream>>>(rows, X, ldx, idx, nidx, src, lds);
        BQ_LAUNCH_CHECK();
        return 0;
    });
}

int bqrrp_step_zero_column_check(int64_t h, const double* col, int* is_zero_host, void* stream)
{
    return step_guard([&]() -> int {
        StepWs sw(stream, 4096, 0);
        int* f = sw.cx.alloc_as<int>(2);
        int one = 1;
        BQ_CUDA(cudaMemcpyAsync(f, &one, sizeof(int), cudaMemcpyHostToDevice, sw.cx.stream));
        if (h > 0) {
            zero_check_kernel<<<(unsigned)imin(cdiv(h, 256), 64), 256, 0, sw.cx.stream>>>(h, col, f);
            BQ_LAUNCH_CHECK();
        }
        BQ_CUDA(cudaMemcpyAsync(is_zero_host, f, sizeof(int), cudaMemcpyDeviceToHost, sw.cx.stream));
        BQ_CUDA(cudaStreamSynchronize(sw.cx.stream));
        return 0;
    });
}

int bqrrp_step_panel(int64_t h, int64_t k, double* P, int64_t ldp, const double* MskT_s, int64_t ldm, double* tau,
                     double* V, double* T, int cholqr_passes, void* stream)
{
    if (h < 1) return -1;
    if (k < 1 || k > h) return -2;
    if (cholqr_passes < 0 || cholqr_passes > 4) return -10;
    return step_guard([&]() -> int {
        size_t bytes = ((size_t)k * k * 12 + (size_t)k + 2 * 160 * 33 + 160 * 32 * 32 + 4096 + 64 * (size_t)k + 8192) * 8;
        StepWs sw(stream, bytes, (size_t)16 * k * k * 8 + (4u << 20));
        Ctx& cx = sw.cx;
        double* Rsk11 = cx.alloc((size_t)k * k);
        extract_rsk_kernel<<<(unsigned)imin(cdiv(k * k, 256), 4 * cx.num_sms), 256, 0, cx.stream>>>(k, MskT_s, ldm,
                                                                                                    Rsk11);
        BQ_LAUNCH_CHECK();
        g_panel_fallbacks += panel_factor(cx, h, P, ldp, 0, k, Rsk11, tau, cholqr_passes, V, T, /*hqr_fallback=*/true);
        int info = 0;
        BQ_CUDA(cudaMemcpyAsync(&info, cx.flags + F_POTRF_INFO, sizeof(int), cudaMemcpyDeviceToHost, cx.stream));
        BQ_CUDA(cudaStreamSynchronize(cx.stream));
        return info ? BQRRP_ENUMERIC : 0;
    });
}

// ---- row-sharded CholQR panel (SURVEY §8(e) phase 2 item 3): the phases of panel_factor on
// one rank's block of panel rows, the k x k pieces replicated; the caller all-reduces the Gram matrices.
int bqrrp_step_cholqr_pre(int64_t rows, int64_t k, const double* P, int64_t ldp, const double* MskT_s, int64_t ldm,
                          double* Q, int64_t ldq, double* G, void* stream)
{
    if (rows < 0) return -1;
    if (k < 1) return -2;
    if (rows > 0 && (ldp < rows || ldq < rows)) return -4;
    return step_guard([&]() -> int {
        StepWs sw(stream, ((size_t)k * k + 8192) * 8, (size_t)16 * k * k * 8 + (4u << 20));
        Ctx& cx = sw.cx;
        double* Rsk11 = cx.alloc((size_t)k * k);
        extract_rsk_kernel<<<(unsigned)imin(cdiv(k * k, 256), 4 * cx.num_sms), 256, 0, cx.stream>>>(k, MskT_s, ldm,
                                                                                                    Rsk11);
        BQ_LAUNCH_CHECK();
        cholqr_precondition_gram(cx, rows, k, P, ldp, Rsk11, Q, ldq, G);
        return 0;
    });
}

int bqrrp_step_potrf(int64_t k, double* G, int64_t ldg, void* stream)
{
    if (k < 1) return -1;
    if (ldg < k) return -3;
    return step_guard([&]() -> int {
        StepWs sw(stream, 8192 * 8, (size_t)16 * k * k * 8 + (4u << 20));
        Ctx& cx = sw.cx;
        potrf_lower(cx, k, G, ldg);
        force_breakdown_hook(cx);
        int info = 0;
        BQ_CUDA(cudaMemcpyAsync(&info, cx.flags + F_POTRF_INFO, sizeof(int), cudaMemcpyDeviceToHost, cx.stream));
        BQ_CUDA(cudaStreamSynchronize(cx.stream));
        return info ? BQRRP_ENUMERIC : 0;
    });
}

int bqrrp_step_cholqr_pass(int64_t rows, int64_t k, double* Q, int64_t ldq, const double* C, double* G, void* stream)
{
    if (rows < 0) return -1;
    if (k < 1) return -2;
    return step_guard([&]() -> int {
        StepWs sw(stream, ((size_t)k * 64 + 8192) * 8, (size_t)16 * k * k * 8 + (4u << 20));
        cholqr_pass_gram(sw.cx, rows, k, Q, ldq, C, G);
        return 0;
    });
}

int bqrrp_step_recon_top(int64_t k, const double* Qtop, int64_t ldq, const double* C, double* Wr, double* S,
                         void* stream)
{
    if (k < 1) return -1;
    return step_guard([&]() -> int {
        StepWs sw(stream, ((size_t)k * 64 + 8192) * 8, (size_t)16 * k * k * 8 + (4u << 20));
        recon_top_lu(sw.cx, k, Qtop, ldq, C, Wr, S);
        return 0;
    });
}

int bqrrp_step_recon_rows(int64_t rows, int64_t k, double* Q, int64_t ldq, const double* Wr, const double* C,
                          void* stream)
{
    if (rows < 0) return -1;
    if (k < 1) return -2;
    if (rows == 0) return 0;
    return step_guard([&]() -> int {
        StepWs sw(stream, ((size_t)2 * k * k + (size_t)k * 64 + 8192) * 8, (size_t)16 * k * k * 8 + (4u << 20));
        recon_rows(sw.cx, rows, k, Q, ldq, Wr, C);
        return 0;
    });
}

// explicit V rows of a row block: top block (row0 == 0) gets the unit-lower L of Wr in its first k rows
__global__ void v_rows_kernel(int64_t rows, int64_t k, double* Q, int64_t ldq, const double* Wr, int top)
{
    int64_t total = rows * k;
    for (int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; idx < total; idx += (int64_t)gridDim.x * blockDim.x) {
        int64_t i = idx % rows, j = idx / rows;
        if (top && i < k) Q[i + j * ldq] = (i > j) ? Wr[i + j * k] : (i == j ? 1.0 : 0.0);
    }
}

int bqrrp_step_recon_finish(int64_t k, const double* Wr, const double* S, const double* C1, const double* C2,
                            const double* MskT_s, int64_t ldm, double* T, double* tau, double* R, void* stream)
{
    if (k < 1) return -1;
    return step_guard([&]() -> int {
        StepWs sw(stream, ((size_t)4 * k * k + (size_t)k * 64 + 8192) * 8, (size_t)16 * k * k * 8 + (4u << 20));
        Ctx& cx = sw.cx;
        double* Rsk11 = cx.alloc((size_t)k * k);
        extract_rsk_kernel<<<(unsigned)imin(cdiv(k * k, 256), 4 * cx.num_sms), 256, 0, cx.stream>>>(k, MskT_s, ldm,
                                                                                                    Rsk11);
        BQ_LAUNCH_CHECK();
        const double* Cf[2] = {C1, C2};
        recon_finish(cx, k, Wr, S, Cf, C2 ? 2 : 1, Rsk11, T, tau, R, nullptr);
        return 0;
    });
}

int bqrrp_step_v_rows(int64_t rows, int64_t k, double* Q, int64_t ldq, const double* Wr, int top, void* stream)
{
    if (rows < 0) return -1;
    if (rows == 0 || !top) return 0;
    return step_guard([&]() -> int {
        cudaStream_t st = (cudaStream_t)stream;
        int dev = 0, nsm = 1;
        BQ_CUDA(cudaGetDevice(&dev));
        BQ_CUDA(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev));
        v_rows_kernel<<<(unsigned)imin(cdiv(rows * k, 256), 8 * nsm), 256, 0, st>>>(rows, k, Q, ldq, Wr, 1);
        BQ_LAUNCH_CHECK();
        return 0;
    });
}

int bqrrp_step_write_panel(int64_t h, int64_t k, double* V, int64_t ldv, const double* R, const double* S, double* A,
                           int64_t lda, void* stream)
{
    if (h < 1) return -1;
    if (k < 1 || k > h) return -2;
    return step_guard([&]() -> int {
        StepWs sw(stream, 8192 * 8, 4096);
        write_panel(sw.cx, h, k, V, ldv, R, S, A, lda);
        return 0;
    });
}

int bqrrp_step_wy_update(int64_t h, int64_t k, int64_t t, const double* V, const double* T, double* C, int64_t ldc,
                         void* stream)
{
    if (h < 1) return -1;
    if (k < 1) return -2;
    if (t < 0) return -3;
    if (t == 0) return 0;
    return step_guard([&]() -> int {
        StepWs sw(stream, ((size_t)2 * k * t + 4096) * 8, (size_t)16 * k * k * 8 + (4u << 20));
        Ctx& cx = sw.cx;
        double* W = cx.alloc((size_t)k * t);
        double* W2 = cx.alloc((size_t)k * t);
        // the same GEMM sequence as wy_update (one stream): W = V^T C, W2 = T^T W, C -= V W2
        gemm(cx, true, false, k, t, h, 1.0, V, h, C, ldc, 0.0, W, k);
        gemm(cx, true, false, k, t, k, 1.0, T, k, W, k, 0.0, W2, k);
        gemm(cx, false, false, h, t, k, -1.0, V, h, W2, k, 1.0, C, ldc);
        return 0;
    });
}

int bqrrp_step_wy_top(int64_t h, int64_t k, int64_t t, const double* V, const double* T, double* C, int64_t ldc,
                      double* W2, int64_t ldw, void* stream)
{
    if (h < 1) return -1;
    if (k < 1) return -2;
    if (t < 0) return -3;
    if (!W2 || ldw < k) return -9;
    if (t == 0) return 0;
    return step_guard([&]() -> int {
        StepWs sw(stream, ((size_t)k * t + 4096) * 8, (size_t)16 * k * k * 8 + (4u << 20));
        Ctx& cx = sw.cx;
        double* W = cx.alloc((size_t)k * t);
        gemm(cx, true, false, k, t, h, 1.0, V, h, C, ldc, 0.0, W, k);      // W  = V^T C
        gemm(cx, true, false, k, t, k, 1.0, T, k, W, k, 0.0, W2, ldw);     // W2 = T^T W
        gemm(cx, false, false, imin(k, h), t, k, -1.0, V, h, W2, ldw, 1.0, C, ldc);  // rows 0:k (R12)
        return 0;
    });
}

int bqrrp_step_wy_bulk(int64_t h, int64_t k, int64_t t, const double* V, const double* W2, int64_t ldw, double* C,
                       int64_t ldc, void* stream)
{
    if (h < 1) return -1;
    if (k < 1) return -2;
    if (t < 0) return -3;
    if (!W2 || ldw < k) return -6;
    if (t == 0 || h <= k) return 0;
    return step_guard([&]() -> int {
        StepWs sw(stream, 4096 * 8, (size_t)16 * 8 + (4u << 20));
        Ctx& cx = sw.cx;
        cx.splitk = nullptr;  // one CTA per tile, no split-K scratch shared with the critical stream
        cx.splitk_elems = 0;
        gemm(cx, false, false, h - k, t, k, -1.0, V + k, h, W2, ldw, 1.0, C + k, ldc);  // rows k:h
        return 0;
    });
}

int bqrrp_step_sample_update(int64_t b, int64_t t, const double* R11, int64_t ldr, const double* R12, int64_t ld12,
                             double* MskT_s, int64_t ldm, void* stream)
{
    if (b < 1) return -1;
    if (t < 0) return -2;
    return step_guard([&]() -> int {
        StepWs sw(stream, ((size_t)2 * b * b + 4096) * 8, (size_t)16 * b * b * 8 + (4u << 20));
        Ctx& cx = sw.cx;
        double* X = cx.alloc((size_t)b * b);
        extract_rsk_kernel<<<(unsigned)imin(cdiv(b * b, 256), 4 * cx.num_sms), 256, 0, cx.stream>>>(b, MskT_s, ldm, X);
        BQ_LAUNCH_CHECK();
        trsm_right_upper(cx, b, b, R11, ldr, false, false, X, b);  // X = R_sk11 R11^{-1}
        zero_triangle(cx, 'U', b, b, X, b);
        if (t > 0) gemm(cx, true, true, t, b, b, -1.0, R12, ld12, X, b, 1.0, MskT_s + b, ldm);
        return 0;
    });
}

int bqrrp_step_sample_update_rows(int64_t b, const double* R11, int64_t ldr, const double* R12, int64_t ld12,
                                  double* MskT_s, int64_t ldm, const int64_t* pos_off, const int64_t* col_off,
                                  const int64_t* len, int64_t nblk, void* stream)
{
    if (b < 1) return -1;
    if (nblk < 0 || (nblk > 0 && (!pos_off || !col_off || !len))) return -12;
    return step_guard([&]() -> int {
        StepWs sw(stream, ((size_t)2 * b * b + 4096) * 8, (size_t)16 * b * b * 8 + (4u << 20));
        Ctx& cx = sw.cx;
        double* X = cx.alloc((size_t)b * b);
        extract_rsk_kernel<<<(unsigned)imin(cdiv(b * b, 256), 4 * cx.num_sms), 256, 0, cx.stream>>>(b, MskT_s, ldm, X);
        BQ_LAUNCH_CHECK();
        trsm_right_upper(cx, b, b, R11, ldr, false, false, X, b);  // X = R_sk11 R11^{-1}
        zero_triangle(cx, 'U', b, b, X, b);
        for (int64_t j = 0; j < nblk; ++j)  // this rank's positions: MskT(c + pos_off, 0:b) -= R12(:, col_off)^T X^T
            if (len[j] > 0)
                gemm(cx, true, true, len[j], b, b, -1.0, R12 + col_off[j] * ld12, ld12, X, b, 1.0,
                     MskT_s + b + pos_off[j], ldm);
        return 0;
    });
}

int bqrrp_step_zero(int64_t rows, int64_t cols, double* X, int64_t ldx, void* stream)
{
    if (rows <= 0 || cols <= 0) return 0;
    return step_guard([&]() -> int {
        StepWs sw(stream, 4096, 0);
        set_zero(sw.cx, rows, cols, X, ldx);
        return 0;
    });
}

}  // extern "C"
