// perm.cu — K-PERM: pivot-format conversion and the touched-set column permutation.
//
// piv_transform ("Permutation formats"): J_qr = (1..w); for j < len(J_lu):
// swap(J_qr(j), J_qr(J_lu(j) - 1)).  J_qr is a product of at most nlu = min(w, d) transpositions,
// so it moves at most 2*nlu positions: T = {0..nlu-1} U {ipiv(j)}.  The kernels here compute the
// touched set (tq[t] = position, tsrc[t] = J_qr(tq[t]) - 1) and apply the gather semantics of
// col_perm (Alg. 5): new(:, q) = old(:, J_qr(q) - 1), moving only T, to the
// columns of A (all m rows, steps bqrrp:permute_r + permute_m merged), to the rows of
// the transposed sketch (Alg. 2 step wide_qrcp:permute) and to J (step bqrrp:update_j).
// Copies are exact: results are bit-identical to the oracle's gather.
#include "bqrrp_internal.cuh"

namespace bqrrp {

constexpr int PT_HASH = 8192;  // open-addressing table for positions >= nlu (<= nlu <= 4096 entries)

// One CTA.  ipiv: 0-based absolute rows (length nlu).  Output: tq, tsrc (length nt <= 2 nlu), nt.
__global__ void piv_to_touched_kernel(int nlu, const int* __restrict__ ipiv, int* tq, int* tsrc, int* nt_out)
{
    extern __shared__ int sh[];
    int* direct = sh;               // direct[q] = current source of position q < nlu
    int* hkey = sh + nlu;           // hash: position (>= nlu) or -1
    int* hval = hkey + PT_HASH;     // its current source
    int* hord = hval + PT_HASH;     // insertion order of hash slots
    __shared__ int nins, cnt;
    for (int i = threadIdx.x; i < nlu; i += blockDim.x) direct[i] = i;
    for (int i = threadIdx.x; i < PT_HASH; i += blockDim.x) hkey[i] = -1;
    if (threadIdx.x == 0) { nins = 0; cnt = 0; }
    __syncthreads();
    if (threadIdx.x == 0) {
        for (int j = 0; j < nlu; ++j) {
            int p = ipiv[j];
            if (p == j) continue;
            int vj = direct[j];
            if (p < nlu) {
                direct[j] = direct[p];
                direct[p] = vj;
            } else {
                unsigned h = ((unsigned)p * 2654435761u) & (PT_HASH - 1);
                while (hkey[h] != -1 && hkey[h] != p) h = (h + 1) & (PT_HASH - 1);
                if (hkey[h] == -1) { hkey[h] = p; hval[h] = p; hord[nins++] = (int)h; }
                direct[j] = hval[h];
                hval[h] = vj;
            }
        }
    }
    __syncthreads();
    // emit moved positions (identity entries dropped)
    for (int q = threadIdx.x; q < nlu; q += blockDim.x)
        if (direct[q] != q) {
            int t = atomicAdd(&cnt, 1);
            tq[t] = q;
            tsrc[t] = direct[q];
        }
    for (int e = threadIdx.x; e < nins; e += blockDim.x) {
        int h = hord[e];
        if (hval[h] != hkey[h]) {
            int t = atomicAdd(&cnt, 1);
            tq[t] = hkey[h];
            tsrc[t] = hval[h];
        }
    }
    __syncthreads();
    if (threadIdx.x == 0) *nt_out = cnt;
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

void touched_set(Ctx& cx, int64_t nlu, const int* ipiv, Touched& T)
{
    T.maxnt = 2 * nlu;
    if (nlu <= 0) {
        BQ_CUDA(cudaMemsetAsync(T.nt, 0, sizeof(int), cx.stream));
        return;
    }
    if (nlu > PT_HASH / 2) throw std::runtime_error("piv_to_touched: sketch size above 4096");
    size_t smem = sizeof(int) * ((size_t)nlu + 3 * PT_HASH);
    static bool attr = false;
    if (!attr) {
        BQ_CUDA(cudaFuncSetAttribute(piv_to_touched_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 160 * 1024));
        attr = true;
    }
    piv_to_touched_kernel<<<1, 256, smem, cx.stream>>>((int)nlu, ipiv, T.tq, T.tsrc, T.nt);
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
