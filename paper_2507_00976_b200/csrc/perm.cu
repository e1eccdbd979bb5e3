// perm.cu — K-PERM: pivot-format conversion and the touched-set column permutation.
//
// piv_transform ("Permutation formats"): J_qr = (1..w); for j < len(J_lu):
// swap(J_qr(j), J_qr(J_lu(j) - 1)).  K-LU maintains perm = J_qr - 1 as it pivots.  J_qr is a product
// of at most nlu = min(w, d) transpositions, so it moves at most 2*nlu positions.  The kernels here
// read the touched set (tq[t] = position, tsrc[t] = J_qr(tq[t]) - 1) off perm and apply the gather semantics of
// col_perm (Alg. 5): new(:, q) = old(:, J_qr(q) - 1), moving only T, to the
// columns of A (all m rows, steps bqrrp:permute_r + permute_m merged), to the rows of
// the transposed sketch (Alg. 2 step wide_qrcp:permute) and to J (step bqrrp:update_j).
// Copies are exact: results are bit-identical to the oracle's gather.
#include "bqrrp_internal.cuh"

namespace bqrrp {

// Touched set straight off the permutation vector: positions q with perm[q] != q (at most 2 nlu of
// them).  Emission order is arbitrary (atomic counter); the gather/scatter result does not depend on it.
__global__ void touched_from_perm_kernel(int64_t w, const int* __restrict__ perm, int* tq, int* tsrc, int* nt)
{
    for (int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; q < w; q += (int64_t)gridDim.x * blockDim.x) {
        int p = perm[q];
        if (p != (int)q) {
            int t = atomicAdd(nt, 1);
            tq[t] = (int)q;
            tsrc[t] = p;
        }
    }
}

// Sequential piv_transform of a one-based swap list into perm (debug entry only).
__global__ void perm_from_ipiv_kernel(int64_t w, int64_t nlu, const int64_t* __restrict__ ipiv1, int* perm)
{
    if (blockIdx.x != 0 || threadIdx.x != 0) return;
    for (int64_t q = 0; q < w; ++q) perm[q] = (int)q;
    for (int64_t j = 0; j < nlu; ++j) {
        int64_t p = ipiv1[j] - 1;
        int t = perm[j];
        perm[j] = perm[p];
        perm[p] = t;
    }
}

// One column segment d[0:rows] = s[0:rows], by the CTA slice (chunk, nchunks): 16-byte copies when both
// columns are 16-byte aligned (even leading dimensions, the usual case), 8-byte otherwise.  Coalesced: the
// thread-fastest index is the row.
__device__ __forceinline__ void copy_col(double* __restrict__ d, const double* __restrict__ s, int64_t rows, int64_t chunk,
                                         int64_t nchunks)
{
    if (((((uintptr_t)d) | ((uintptr_t)s)) & 15) == 0) {
        const int64_t pairs = rows >> 1;
        const double2* s2 = reinterpret_cast<const double2*>(s);
        double2* d2 = reinterpret_cast<double2*>(d);
        for (int64_t p = chunk * blockDim.x + threadIdx.x; p < pairs; p += nchunks * blockDim.x) d2[p] = __ldg(s2 + p);
        if ((rows & 1) && chunk == 0 && threadIdx.x == 0) d[rows - 1] = s[rows - 1];
    } else {
        for (int64_t r = chunk * blockDim.x + threadIdx.x; r < rows; r += nchunks * blockDim.x) d[r] = s[r];
    }
}

// scratch(:, t) = X(:, src[t]) for all `rows` rows; 2-D grid (row chunk, t).
__global__ void gather_cols_kernel(int64_t rows, const double* __restrict__ X, int64_t ldx, const int* __restrict__ src,
                                   const int* __restrict__ nt, double* __restrict__ scratch, int64_t lds)
{
    int t = blockIdx.y;
    if (t >= *nt) return;
    copy_col(scratch + (int64_t)t * lds, X + (int64_t)src[t] * ldx, rows, blockIdx.x, gridDim.x);
}

__global__ void scatter_cols_kernel(int64_t rows, double* __restrict__ X, int64_t ldx, const int* __restrict__ dst,
                                    const int* __restrict__ nt, const double* __restrict__ scratch, int64_t lds)
{
    int t = blockIdx.y;
    if (t >= *nt) return;
    copy_col(X + (int64_t)dst[t] * ldx, scratch + (int64_t)t * lds, rows, blockIdx.x, gridDim.x);
}

// dst(:, q) = X(:, idx[q]), q < nq (grid (row chunk, q)).
__global__ void gather_idx_kernel(int64_t rows, const double* __restrict__ X, int64_t ldx, const int* __restrict__ idx,
                                  double* __restrict__ dst, int64_t ldd)
{
    const int q = blockIdx.y;
    copy_col(dst + (int64_t)q * ldd, X + (int64_t)idx[q] * ldx, rows, blockIdx.x, gridDim.x);
}

// ---- pivot-aware lookahead gathers.  Warp per (64-row tile R, panel column q); the bulk
// GEMM's tile holding those rows of column perm[q] is T = R * tiles_n + perm[q] / 64.
constexpr int LA_TILE = 64;

__device__ __forceinline__ int la_ld_acquire(const int* p)
{
    int v;
    asm volatile("ld.acquire.gpu.global.b32 %0, [%1];\n" : "=r"(v) : "l"(p) : "memory");
    return v;
}

// C is read through L2 (ld.global.cg: never a stale L1 line) and is not __restrict__: the bulk GEMM writes it
// concurrently (other tiles).
__global__ void la_gather_pre_kernel(int64_t rows, const double* C, int64_t ldc, const int* __restrict__ perm,
                                     int64_t nq, int64_t tiles_n, int* hs_state, int* hs_readers, double* __restrict__ P,
                                     int64_t ldp, int* post)
{
    const int lane = threadIdx.x & 31;
    const int64_t q = (int64_t)blockIdx.y * (blockDim.x >> 5) + (threadIdx.x >> 5);
    const int64_t R = blockIdx.x;
    if (q >= nq) return;
    const int src = perm[q];
    const int64_t T = R * tiles_n + src / LA_TILE;
    int pre = 0;
    if (lane == 0) {
        // Dekker with the bulk CTA of T: (readers++, fence.sc, read state) vs its (state = 1, fence.sc, read
        // readers): either we see "started" or it sees our reader and holds its stores until we are done
        atomicAdd(hs_readers + T, 1);
        asm volatile("fence.sc.gpu;\n" ::: "memory");
        pre = (la_ld_acquire(hs_state + T) == 0);
        if (!pre) atomicSub(hs_readers + T, 1);
    }
    pre = __shfl_sync(0xffffffffu, pre, 0);
    if (lane == 0) post[R + q * gridDim.x] = pre ? 0 : 1;
    if (!pre) return;
    const int64_t r0 = R * LA_TILE;
    const double* s = C + (int64_t)src * ldc;
    double* d = P + q * ldp;
    for (int64_t r = r0 + lane; r < r0 + LA_TILE && r < rows; r += 32) d[r] = __ldcg(s + r);
    __syncwarp();
    if (lane == 0) {
        __threadfence();  // the warp's loads are complete (their values are stored) before the release
        atomicSub(hs_readers + T, 1);
    }
}

__global__ void la_gather_post_kernel(int64_t rows, const double* C, int64_t ldc, const int* __restrict__ perm,
                                      int64_t nq, int64_t tiles_n, const int* hs_state, double* __restrict__ P, int64_t ldp,
                                      const int* post)
{
    const int lane = threadIdx.x & 31;
    const int64_t q = (int64_t)blockIdx.y * (blockDim.x >> 5) + (threadIdx.x >> 5);
    const int64_t R = blockIdx.x;
    if (q >= nq || !post[R + q * gridDim.x]) return;
    const int src = perm[q];
    const int64_t T = R * tiles_n + src / LA_TILE;
    if (lane == 0)
        while (la_ld_acquire(hs_state + T) != 2) __nanosleep(128);
    __syncwarp();
    const int64_t r0 = R * LA_TILE;
    const double* s = C + (int64_t)src * ldc;
    double* d = P + q * ldp;
    for (int64_t r = r0 + lane; r < r0 + LA_TILE && r < rows; r += 32) d[r] = __ldcg(s + r);
}

// Rows of a column-major matrix (cols columns): scratch[t + c*maxnt] = X[src[t] + c*ldx].
__global__ void gather_rows_kernel(int64_t cols, const double* __restrict__ X, int64_t ldx, const int* __restrict__ src,
                                   const int* __restrict__ nt, double* __restrict__ scratch, int64_t maxnt)
{
    int n = *nt;
    int64_t total = (int64_t)n * cols;
    for (int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; idx < total; idx += (int64_t)gridDim.x * blockDim.x) {
        int64_t t = idx % n, c = idx / n;
        scratch[t + c * maxnt] = X[src[t] + c * ldx];
    }
}

__global__ void scatter_rows_kernel(int64_t cols, double* __restrict__ X, int64_t ldx, const int* __restrict__ dst,
                                    const int* __restrict__ nt, const double* __restrict__ scratch, int64_t maxnt)
{
    int n = *nt;
    int64_t total = (int64_t)n * cols;
    for (int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; idx < total; idx += (int64_t)gridDim.x * blockDim.x) {
        int64_t t = idx % n, c = idx / n;
        X[dst[t] + c * ldx] = scratch[t + c * maxnt];
    }
}

// J(tq[t]) = Jold(tsrc[t]) — one CTA (nt <= 2 nlu).
__global__ void permute_vec_kernel(int64_t* J, const int* __restrict__ tq, const int* __restrict__ tsrc,
                                   const int* __restrict__ nt, int64_t* tmp)
{
    int n = *nt;
    for (int t = threadIdx.x; t < n; t += blockDim.x) tmp[t] = J[tsrc[t]];
    __syncthreads();
    for (int t = threadIdx.x; t < n; t += blockDim.x) J[tq[t]] = tmp[t];
}

void touched_from_perm(Ctx& cx, int64_t w, int64_t nlu, const int* perm, Touched& T)
{
    T.maxnt = 2 * nlu;
    BQ_CUDA(cudaMemsetAsync(T.nt, 0, sizeof(int), cx.stream));
    if (nlu <= 0 || w <= 0) return;
    touched_from_perm_kernel<<<(unsigned)imin(cdiv(w, 256), 4 * cx.num_sms), 256, 0, cx.stream>>>(w, perm, T.tq,
                                                                                                   T.tsrc, T.nt);
    BQ_LAUNCH_CHECK();
}

void perm_from_ipiv(Ctx& cx, int64_t w, int64_t nlu, const int64_t* ipiv1, int* perm)
{
    perm_from_ipiv_kernel<<<1, 32, 0, cx.stream>>>(w, nlu, ipiv1, perm);
    BQ_LAUNCH_CHECK();
}

void permute_columns(Ctx& cx, int64_t rows, double* X, int64_t ldx, const Touched& T, double* scratch)
{
    if (T.maxnt <= 0 || rows <= 0) return;
    unsigned chunks = (unsigned)imin(cdiv(rows, 256 * 8), 64);
    dim3 grid(chunks, (unsigned)T.maxnt);
    gather_cols_kernel<<<grid, 256, 0, cx.stream>>>(rows, X, ldx, T.tsrc, T.nt, scratch, rows);
    BQ_LAUNCH_CHECK();
    scatter_cols_kernel<<<grid, 256, 0, cx.stream>>>(rows, X, ldx, T.tq, T.nt, scratch, rows);
    BQ_LAUNCH_CHECK();
}

void permute_rows(Ctx& cx, int64_t cols, double* X, int64_t ldx, const Touched& T, double* scratch)
{
    if (T.maxnt <= 0 || cols <= 0) return;
    unsigned blocks = (unsigned)imin(cdiv(T.maxnt * cols, 256), 8 * cx.num_sms);
    gather_rows_kernel<<<blocks, 256, 0, cx.stream>>>(cols, X, ldx, T.tsrc, T.nt, scratch, T.maxnt);
    BQ_LAUNCH_CHECK();
    scatter_rows_kernel<<<blocks, 256, 0, cx.stream>>>(cols, X, ldx, T.tq, T.nt, scratch, T.maxnt);
    BQ_LAUNCH_CHECK();
}

void permute_vector(Ctx& cx, int64_t* J, const Touched& T, int64_t* tmp)
{
    if (T.maxnt <= 0) return;
    permute_vec_kernel<<<1, 1024, 0, cx.stream>>>(J, T.tq, T.tsrc, T.nt, tmp);
    BQ_LAUNCH_CHECK();
}

void gather_cols_idx(Ctx& cx, int64_t rows, const double* X, int64_t ldx, const int* idx, int64_t nq, double* dst,
                     int64_t ldd)
{
    if (rows <= 0 || nq <= 0) return;
    dim3 grid((unsigned)imin(cdiv(rows, 256 * 8), 64), (unsigned)nq);
    gather_idx_kernel<<<grid, 256, 0, cx.stream>>>(rows, X, ldx, idx, dst, ldd);
    BQ_LAUNCH_CHECK();
}

void la_gather_pre(Ctx& cx, int64_t rows, const double* C, int64_t ldc, const int* perm, int64_t nq, int64_t tiles_n,
                   int* hs_state, int* hs_readers, double* P, int64_t ldp, int* post)
{
    if (rows <= 0 || nq <= 0) return;
    dim3 grid((unsigned)cdiv(rows, LA_TILE), (unsigned)cdiv(nq, 8));
    la_gather_pre_kernel<<<grid, 256, 0, cx.stream>>>(rows, C, ldc, perm, nq, tiles_n, hs_state, hs_readers, P, ldp,
                                                      post);
    BQ_LAUNCH_CHECK();
}

void la_gather_post(Ctx& cx, int64_t rows, const double* C, int64_t ldc, const int* perm, int64_t nq, int64_t tiles_n,
                    const int* hs_state, double* P, int64_t ldp, const int* post)
{
    if (rows <= 0 || nq <= 0) return;
    dim3 grid((unsigned)cdiv(rows, LA_TILE), (unsigned)cdiv(nq, 8));
    la_gather_post_kernel<<<grid, 256, 0, cx.stream>>>(rows, C, ldc, perm, nq, tiles_n, hs_state, P, ldp, post);
    BQ_LAUNCH_CHECK();
}

}  // namespace bqrrp
