// norm.cu — K-NORM: the HBM-bound norm kernels of the pivot-quality / verification path.
//
// * Column 2-norms ||A(:, j)||_2 — the sampled invariant ||R(0:j+1, j)|| = ||A(:, J(j))|| (Q orthogonal,
//   GEQP3 output P:253-277) and the column-norm view of pivot quality.
// * Trailing Frobenius norms ||R(i:, i:)||_F for every i < min(m, n) — the paper's first pivot-quality metric
//   ("the Frobenius norms of the trailing submatrix of the output R-factor, R(i:, i:)", the
//   residual of the rank-i approximation Q(:, :i) R(:i, :)); |R(i, i)| (the second metric) is
//   read off the diagonal.
//
// Both are one pass over the data (bound by HBM): 16-byte loads where the columns are
// 16-byte aligned, deterministic fixed-order reductions (the result does not depend on the grid size).
// Sums of squares are formed in fp64; a column whose sum over- or underflows is recomputed scaled by its
// largest magnitude (LAPACK dnrm2's concern, rare: only for |a| outside ~[1e-146, 1e143]).
#include "../../include/bqrrp.h"
#include "bqrrp_internal.cuh"

namespace bqrrp {

constexpr int NORM_THREADS = 256;

// Fixed-order block sum of one double per thread (all NORM_THREADS threads call it); result in every thread.
__device__ __forceinline__ double block_sum(double v, double* red)
{
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    __syncthreads();  // red may still be read by a previous call
    if (lane == 0) red[warp] = v;
    __syncthreads();
    double s = 0.0;
#pragma unroll
    for (int w = 0; w < NORM_THREADS / 32; ++w) s += red[w];
    return s;
}
__device__ __forceinline__ double block_max(double v, double* red)
{
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    __syncthreads();
    if (lane == 0) red[warp] = v;
    __syncthreads();
    double s = 0.0;
#pragma unroll
    for (int w = 0; w < NORM_THREADS / 32; ++w) s = fmax(s, red[w]);
    return s;
}

// One CTA per column (grid-stride over columns).  Per thread: 4 independent double2 loads in flight per step.
__global__ void __launch_bounds__(NORM_THREADS) col_norms_kernel(int64_t m, int64_t n, const double* __restrict__ A,
                                                                 int64_t lda, double* __restrict__ out)
{
    __shared__ double red[NORM_THREADS / 32];
    const bool vec = ((((uintptr_t)A) & 15) == 0) && ((lda & 1) == 0);
    for (int64_t j = blockIdx.x; j < n; j += gridDim.x) {
        const double* a = A + j * lda;
        double s0 = 0.0, s1 = 0.0, mx = 0.0;
        if (vec) {
            const double2* a2 = reinterpret_cast<const double2*>(a);
            const int64_t pairs = m >> 1;
            int64_t p = threadIdx.x;
            for (; p + 3 * NORM_THREADS < pairs; p += 4 * NORM_THREADS) {
                double2 v[4];
#pragma unroll
                for (int u = 0; u < 4; ++u) v[u] = __ldcs(a2 + p + u * NORM_THREADS);
#pragma unroll
                for (int u = 0; u < 4; ++u) {
                    s0 = fma(v[u].x, v[u].x, s0);
                    s1 = fma(v[u].y, v[u].y, s1);
                    mx = fmax(mx, fmax(fabs(v[u].x), fabs(v[u].y)));
                }
            }
            for (; p < pairs; p += NORM_THREADS) {
                const double2 v = __ldcs(a2 + p);
                s0 = fma(v.x, v.x, s0);
                s1 = fma(v.y, v.y, s1);
                mx = fmax(mx, fmax(fabs(v.x), fabs(v.y)));
            }
            if ((m & 1) && threadIdx.x == 0) {
                const double v = a[m - 1];
                s0 = fma(v, v, s0);
                mx = fmax(mx, fabs(v));
            }
        } else {
            for (int64_t r = threadIdx.x; r < m; r += NORM_THREADS) {
                const double v = a[r];
                s0 = fma(v, v, s0);
                mx = fmax(mx, fabs(v));
            }
        }
        double s = block_sum(s0 + s1, red);
        const double amax = block_max(mx, red);
        // over/underflow of the plain sum of squares: rescale by the column's largest magnitude
        if (amax > 0.0 && (!(s <= 1e300) || s < 1e-290)) {
            const double inv = 1.0 / amax;
            double t = 0.0;
            for (int64_t r = threadIdx.x; r < m; r += NORM_THREADS) {
                const double v = a[r] * inv;
                t = fma(v, v, t);
            }
            s = block_sum(t, red);
            if (threadIdx.x == 0) out[j] = amax * sqrt(s);
        } else if (threadIdx.x == 0) {
            out[j] = (amax > 0.0) ? sqrt(s) : 0.0;
        }
    }
}

// Trailing norms, pass 1: partial row sums of squares of the upper trapezoid over column chunks.
//   part[c * mn + r] = sum_{j in chunk c, j >= r} R(r, j)^2,  for the chunks c >= r / TN_CHUNK.
// CTA (row block bx of NORM_THREADS rows, chunk by); a warp reads 32 consecutive rows of one column (256 B).
constexpr int TN_CHUNK = 1024;
__global__ void __launch_bounds__(NORM_THREADS) trailing_rows_kernel(int64_t mn, int64_t n, const double* __restrict__ R,
                                                                     int64_t ldr, double* __restrict__ part)
{
    const int64_t r0 = (int64_t)blockIdx.x * NORM_THREADS;
    const int64_t c0 = (int64_t)blockIdx.y * TN_CHUNK;
    if (c0 + TN_CHUNK <= r0) return;  // chunk entirely left of the block's diagonal: not read by pass 2
    const int64_t r = r0 + threadIdx.x;
    const int64_t jb = c0 > r0 ? c0 : r0, je = (c0 + TN_CHUNK < n) ? c0 + TN_CHUNK : n;
    double s[4] = {0.0, 0.0, 0.0, 0.0};
    if (r < mn) {
        const double* row = R + r;
        int64_t j = jb;
        for (; j + 8 <= je; j += 8) {
            double v[8];
#pragma unroll
            for (int u = 0; u < 8; ++u) v[u] = __ldcs(row + (j + u) * ldr);
#pragma unroll
            for (int u = 0; u < 8; ++u) {
                const double x = (j + u >= r) ? v[u] : 0.0;
                s[u & 3] = fma(x, x, s[u & 3]);
            }
        }
        for (; j < je; ++j) {
            const double v = row[j * ldr];
            const double x = (j >= r) ? v : 0.0;
            s[0] = fma(x, x, s[0]);
        }
        part[blockIdx.y * mn + r] = (s[0] + s[1]) + (s[2] + s[3]);
    }
}

// Pass 2: rowsq[r] = sum over the chunks c >= r / TN_CHUNK of part (fixed order), into out.
__global__ void trailing_rowsum_kernel(int64_t mn, int64_t nch, const double* __restrict__ part, double* __restrict__ out)
{
    for (int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; r < mn; r += (int64_t)gridDim.x * blockDim.x) {
        double s = 0.0;
        for (int64_t c = r / TN_CHUNK; c < nch; ++c) s += part[c * mn + r];
        out[r] = s;
    }
}

// Pass 3 (one CTA of 1024 threads): out[i] = sqrt(sum_{r >= i} rowsq[r]) — thread t owns a contiguous segment,
// segment totals combined by a fixed-order suffix scan in shared memory.
__global__ void __launch_bounds__(1024) trailing_scan_kernel(int64_t mn, double* out)
{
    __shared__ double tot[1024];
    const int t = threadIdx.x;
    const int64_t seg = (mn + 1023) / 1024;
    const int64_t rb = t * seg, re = (rb + seg < mn) ? rb + seg : mn;
    double s = 0.0;
    for (int64_t r = rb; r < re; ++r) s += out[r];
    tot[t] = s;
    __syncthreads();
    // inclusive suffix scan (Hillis-Steele, fixed pairing)
    for (int o = 1; o < 1024; o <<= 1) {
        const double add = (t + o < 1024) ? tot[t + o] : 0.0;
        __syncthreads();
        tot[t] += add;
        __syncthreads();
    }
    double acc = (t + 1 < 1024) ? tot[t + 1] : 0.0;  // everything after this segment
    for (int64_t r = re - 1; r >= rb; --r) {
        acc += out[r];
        out[r] = sqrt(acc);
    }
}

void column_norms(Ctx& cx, int64_t m, int64_t n, const double* A, int64_t lda, double* out)
{
    if (n <= 0) return;
    if (m <= 0) {
        BQ_CUDA(cudaMemsetAsync(out, 0, sizeof(double) * n, cx.stream));
        return;
    }
    const unsigned grid = (unsigned)imin(n, (int64_t)cx.num_sms * 8);
    col_norms_kernel<<<grid, NORM_THREADS, 0, cx.stream>>>(m, n, A, lda, out);
    BQ_LAUNCH_CHECK();
}

size_t trailing_norms_scratch(int64_t m, int64_t n)
{
    const int64_t mn = imin(m, n);
    return (size_t)cdiv(imax(n, 1), TN_CHUNK) * (size_t)imax(mn, 1);
}

void trailing_norms(Ctx& cx, int64_t m, int64_t n, const double* R, int64_t ldr, double* out, double* part)
{
    const int64_t mn = imin(m, n);
    if (mn <= 0) return;
    const int64_t nch = cdiv(n, TN_CHUNK);
    dim3 g1((unsigned)cdiv(mn, NORM_THREADS), (unsigned)nch);
    trailing_rows_kernel<<<g1, NORM_THREADS, 0, cx.stream>>>(mn, n, R, ldr, part);
    BQ_LAUNCH_CHECK();
    trailing_rowsum_kernel<<<(unsigned)imin(cdiv(mn, 256), 4 * cx.num_sms), 256, 0, cx.stream>>>(mn, nch, part, out);
    BQ_LAUNCH_CHECK();
    trailing_scan_kernel<<<1, 1024, 0, cx.stream>>>(mn, out);
    BQ_LAUNCH_CHECK();
}

}  // namespace bqrrp

using namespace bqrrp;

extern "C" {

int bqrrp_column_norms(int64_t m, int64_t n, const double* A, int64_t lda, double* norms, void* stream)
{
    if (m < 0) return -1;
    if (n < 0) return -2;
    if (!A && m > 0 && n > 0) return -3;
    if (lda < (m > 1 ? m : 1)) return -4;
    if (!norms && n > 0) return -5;
    return guarded([&]() -> int {
        Ctx cx;
        setup_ctx(cx, stream);
        column_norms(cx, m, n, A, lda, norms);
        return 0;
    });
}

int bqrrp_trailing_norms(int64_t m, int64_t n, const double* R, int64_t ldr, double* out, void* workspace,
                         size_t ws_bytes, void* stream)
{
    if (m < 0) return -1;
    if (n < 0) return -2;
    if (!R && m > 0 && n > 0) return -3;
    if (ldr < (m > 1 ? m : 1)) return -4;
    if (!out && m > 0 && n > 0) return -5;
    const size_t need = trailing_norms_scratch(m, n) * sizeof(double);
    if (workspace && ws_bytes < need) return -7;
    return guarded([&]() -> int {
        Ctx cx;
        setup_ctx(cx, stream);
        if (imin(m, n) <= 0) return 0;
        void* ws = workspace;
        if (!ws) BQ_CUDA(lib_malloc_async(&ws, need, cx.stream));
        trailing_norms(cx, m, n, R, ldr, out, (double*)ws);
        if (!workspace) BQ_CUDA(cudaFreeAsync(ws, cx.stream));
        return 0;
    });
}

int bqrrp_trailing_norms_workspace(int64_t m, int64_t n, size_t* bytes)
{
    if (m < 0) return -1;
    if (n < 0) return -2;
    if (!bytes) return -3;
    *bytes = trailing_norms_scratch(m, n) * sizeof(double);
    return 0;
}

}  // extern "C"
