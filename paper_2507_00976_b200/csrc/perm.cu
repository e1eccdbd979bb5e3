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

// scratch(:, t) = X(:, src[t]) for all `rows` rows; column-contiguous copies, 2-D grid (t, row chunk).
__global__ void gather_cols_kernel(int64_t rows, const double* __restrict__ X, int64_t ldx, const int* __restrict__ src,
                                   const int* __restrict__ nt, double* __restrict__ scratch, int64_t lds)
{
    int t = blockIdx.y;
    if (t >= *nt) return;
    const double* s = X + (int64_t)src[t] * ldx;
    double* d = scratch + (int64_t)t * lds;
    for (int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; r < rows; r += (int64_t)gridDim.x * blockDim.x)
        d[r] = s[r];
}

__global__ void scatter_cols_kernel(int64_t rows, double* __restrict__ X, int64_t ldx, const int* __restrict__ dst,
                                    const int* __restrict__ nt, const double* __restrict__ scratch, int64_t lds)
{
    int t = blockIdx.y;
    if (t >= *nt) return;
    double* d = X + (int64_t)dst[t] * ldx;
    const double* s = scratch + (int64_t)t * lds;
    for (int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; r < rows; r += (int64_t)gridDim.x * blockDim.x)
        d[r] = s[r];
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

}  // namespace bqrrp
