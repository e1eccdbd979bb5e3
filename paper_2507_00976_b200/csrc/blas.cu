// blas.cu — GEMM launcher (split-K heuristic), recursive TRSM, blocked POTRF and the
// sign-choosing no-pivot LU of the Householder reconstruction.  Every O(n^3) piece is cast onto the
// DMMA GEMM engine (dgemm.cuh); the diagonal blocks (<= 64) are factored by one CTA in shared memory.
#include "blas.cuh"
#include "dgemm.cuh"

namespace bqrrp {

// ------------------------------------------------------------------------------------------- GEMM
template <bool TA, bool TB>
static void launch_gemm(Ctx& cx, const GemmArgs& g, dim3 grid)
{
    static bool attr_set = false;
    size_t sm = dgemm_smem_bytes(TA, TB);
    if (!attr_set) {
        BQ_CUDA(cudaFuncSetAttribute(dgemm_kernel<TA, TB>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
        attr_set = true;
    }
    dgemm_kernel<TA, TB><<<grid, GEMM_THREADS, sm, cx.stream>>>(g);
    BQ_LAUNCH_CHECK();
}

void gemm(Ctx& cx, bool ta, bool tb, int64_t M, int64_t N, int64_t K, double alpha, const double* A, int64_t lda,
          const double* B, int64_t ldb, double beta, double* C, int64_t ldc, bool tri)
{
    if (M <= 0 || N <= 0) return;
    int64_t tm = cdiv(M, GEMM_BM), tn = cdiv(N, GEMM_BN);
    int64_t tiles = tri ? (tm * (tm + 1)) / 2 : tm * tn;
    int nsplit = 1;
    int64_t kchunk = K > 0 ? K : 1;
    if (K >= 1024 && tiles < cx.num_sms && cx.splitk) {
        int64_t want = cdiv(2 * cx.num_sms, tiles);
        want = imin(want, 32);
        want = imin(want, K / 256);
        int64_t cap = (int64_t)(cx.splitk_elems / (size_t)(M * N));
        want = imin(want, cap);
        if (want >= 2) {
            kchunk = cdiv(cdiv(K, want), GEMM_BK) * GEMM_BK;
            nsplit = (int)cdiv(K, kchunk);
        }
    }
    GemmArgs g{M, N, K, alpha, beta, A, lda, B, ldb, C, ldc, nsplit > 1 ? cx.splitk : nullptr, kchunk, tri ? 1 : 0};
    dim3 grid((unsigned)tm, (unsigned)tn, (unsigned)nsplit);
    if (!ta && !tb) launch_gemm<false, false>(cx, g, grid);
    else if (ta && !tb) launch_gemm<true, false>(cx, g, grid);
    else if (!ta && tb) launch_gemm<false, true>(cx, g, grid);
    else launch_gemm<true, true>(cx, g, grid);
    if (nsplit > 1) {
        int64_t total = M * N;
        int blocks = (int)imin(cdiv(total, 256), 4 * cx.num_sms);
        dgemm_splitk_reduce<<<blocks, 256, 0, cx.stream>>>(M, N, nsplit, cx.splitk, alpha, beta, C, ldc, tri ? 1 : 0);
        BQ_LAUNCH_CHECK();
    }
}

// ------------------------------------------------------------------------------------------- TRSM
constexpr int TRSM_NB = 64;

// Right side: one thread per row r solves x op(T) = b (left-looking, ascending l).
__global__ void __launch_bounds__(128) trsm_ru_base(int64_t rows, int n, const double* __restrict__ T, int64_t ldt,
                                                     int t_lower, int unit, double* __restrict__ B, int64_t ldb)
{
    __shared__ double U[TRSM_NB][TRSM_NB + 1];  // U[l][j] = op(T)(l, j)
    for (int idx = threadIdx.x; idx < n * n; idx += blockDim.x) {
        int l = idx % n, j = idx / n;
        U[l][j] = (l <= j) ? (t_lower ? T[j + (int64_t)l * ldt] : T[l + (int64_t)j * ldt]) : 0.0;
    }
    __syncthreads();
    int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (r >= rows) return;
    double x[TRSM_NB];
#pragma unroll
    for (int j = 0; j < TRSM_NB; ++j) x[j] = (j < n) ? B[r + (int64_t)j * ldb] : 0.0;
#pragma unroll
    for (int j = 0; j < TRSM_NB; ++j) {
        if (j < n) {
            double v = x[j];
#pragma unroll
            for (int l = 0; l < j; ++l) v = fma(-x[l], U[l][j], v);
            x[j] = unit ? v : v / U[j][j];
        }
    }
#pragma unroll
    for (int j = 0; j < TRSM_NB; ++j)
        if (j < n) B[r + (int64_t)j * ldb] = x[j];
}

void trsm_right_upper(Ctx& cx, int64_t rows, int64_t n, const double* T, int64_t ldt, bool t_lower, bool unit,
                      double* B, int64_t ldb)
{
    if (rows <= 0 || n <= 0) return;
    if (n <= TRSM_NB) {
        trsm_ru_base<<<(unsigned)cdiv(rows, 128), 128, 0, cx.stream>>>(rows, (int)n, T, ldt, t_lower, unit, B, ldb);
        BQ_LAUNCH_CHECK();
        return;
    }
    int64_t n1 = cdiv(n / 2, TRSM_NB) * TRSM_NB;
    int64_t n2 = n - n1;
    trsm_right_upper(cx, rows, n1, T, ldt, t_lower, unit, B, ldb);
    if (!t_lower)  // op(T)(0:n1, n1:n) = T(0:n1, n1:n)
        gemm(cx, false, false, rows, n2, n1, -1.0, B, ldb, T + n1 * ldt, ldt, 1.0, B + n1 * ldb, ldb);
    else  // op(T)(0:n1, n1:n) = T(n1:n, 0:n1)^T
        gemm(cx, false, true, rows, n2, n1, -1.0, B, ldb, T + n1, ldt, 1.0, B + n1 * ldb, ldb);
    trsm_right_upper(cx, rows, n2, T + n1 + n1 * ldt, ldt, t_lower, unit, B + n1 * ldb, ldb);
}

// Left side, unit lower: one thread per column c solves L x = b.
__global__ void __launch_bounds__(128) trsm_llu_base(int n, int64_t cols, const double* __restrict__ L, int64_t ldl,
                                                      double* __restrict__ B, int64_t ldb)
{
    __shared__ double Ls[TRSM_NB][TRSM_NB + 1];
    for (int idx = threadIdx.x; idx < n * n; idx += blockDim.x) {
        int i = idx % n, l = idx / n;
        Ls[i][l] = (l < i) ? L[i + (int64_t)l * ldl] : 0.0;
    }
    __syncthreads();
    int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (c >= cols) return;
    double x[TRSM_NB];
#pragma unroll
    for (int i = 0; i < TRSM_NB; ++i) x[i] = (i < n) ? B[i + c * ldb] : 0.0;
#pragma unroll
    for (int i = 0; i < TRSM_NB; ++i) {
        if (i < n) {
            double v = x[i];
#pragma unroll
            for (int l = 0; l < i; ++l) v = fma(-Ls[i][l], x[l], v);
            x[i] = v;
        }
    }
#pragma unroll
    for (int i = 0; i < TRSM_NB; ++i)
        if (i < n) B[i + c * ldb] = x[i];
}

void trsm_left_lower_unit(Ctx& cx, int64_t n, int64_t cols, const double* L, int64_t ldl, double* B, int64_t ldb)
{
    if (n <= 0 || cols <= 0) return;
    if (n <= TRSM_NB) {
        trsm_llu_base<<<(unsigned)cdiv(cols, 128), 128, 0, cx.stream>>>((int)n, cols, L, ldl, B, ldb);
        BQ_LAUNCH_CHECK();
        return;
    }
    int64_t n1 = cdiv(n / 2, TRSM_NB) * TRSM_NB;
    int64_t n2 = n - n1;
    trsm_left_lower_unit(cx, n1, cols, L, ldl, B, ldb);
    gemm(cx, false, false, n2, cols, n1, -1.0, L + n1, ldl, B, ldb, 1.0, B + n1, ldb);
    trsm_left_lower_unit(cx, n2, cols, L + n1 + n1 * ldl, ldl, B + n1, ldb);
}

// ------------------------------------------------------------------------------------------- POTRF
constexpr int FACT_NB = 64;

__global__ void __launch_bounds__(256) potrf_diag(int n, double* G, int64_t ldg, int j0, int* info)
{
    __shared__ double A[FACT_NB][FACT_NB + 1];
    __shared__ int failed;
    for (int idx = threadIdx.x; idx < n * n; idx += blockDim.x) {
        int i = idx % n, j = idx / n;
        A[i][j] = (i >= j) ? G[i + (int64_t)j * ldg] : 0.0;
    }
    if (threadIdx.x == 0) failed = (*info != 0);
    __syncthreads();
    for (int j = 0; j < n && !failed; ++j) {
        if (threadIdx.x == 0) {
            double a = A[j][j];
            if (!(a > 0.0)) {
                failed = 1;
                atomicCAS(info, 0, j0 + j + 1);
            } else {
                A[j][j] = sqrt(a);
            }
        }
        __syncthreads();
        if (failed) break;
        double djj = A[j][j];
        for (int i = j + 1 + threadIdx.x; i < n; i += blockDim.x) A[i][j] = A[i][j] / djj;
        __syncthreads();
        int m = n - j - 1;
        for (int idx = threadIdx.x; idx < m * m; idx += blockDim.x) {
            int i = j + 1 + idx % m, c = j + 1 + idx / m;
            if (c <= i) A[i][c] = fma(-A[i][j], A[c][j], A[i][c]);
        }
        __syncthreads();
    }
    for (int idx = threadIdx.x; idx < n * n; idx += blockDim.x) {
        int i = idx % n, j = idx / n;
        G[i + (int64_t)j * ldg] = (i >= j) ? A[i][j] : 0.0;
    }
}

void potrf_lower(Ctx& cx, int64_t n, double* G, int64_t ldg)
{
    for (int64_t j0 = 0; j0 < n; j0 += FACT_NB) {
        int64_t jb = imin(FACT_NB, n - j0);
        double* Gjj = G + j0 + j0 * ldg;
        potrf_diag<<<1, 256, 0, cx.stream>>>((int)jb, Gjj, ldg, (int)j0, cx.flags + F_POTRF_INFO);
        BQ_LAUNCH_CHECK();
        int64_t rest = n - j0 - jb;
        if (rest > 0) {
            double* G21 = Gjj + jb;
            trsm_right_upper(cx, rest, jb, Gjj, ldg, /*t_lower=*/true, /*unit=*/false, G21, ldg);
            gemm(cx, false, true, rest, rest, jb, -1.0, G21, ldg, G21, ldg, 1.0, G21 + jb * ldg, ldg, /*tri=*/true);
        }
    }
    zero_triangle(cx, 'L', n, n, G, ldg);
}

// ------------------------------------------------------------------------------------------- sign LU
__global__ void __launch_bounds__(256) getrf_sign_diag(int n, double* Q, int64_t ldq, double* S)
{
    __shared__ double A[FACT_NB][FACT_NB + 1];
    for (int idx = threadIdx.x; idx < n * n; idx += blockDim.x) {
        int i = idx % n, j = idx / n;
        A[i][j] = Q[i + (int64_t)j * ldq];
    }
    __syncthreads();
    for (int j = 0; j < n; ++j) {
        if (threadIdx.x == 0) {
            double a = A[j][j];
            double s = (a >= 0.0) ? -1.0 : 1.0;  // S_jj = -sgn(a), sgn(a) = a >= 0 ? +1 : -1 (Z20)
            S[j] = s;
            A[j][j] = a - s;
        }
        __syncthreads();
        double piv = A[j][j];
        for (int i = j + 1 + threadIdx.x; i < n; i += blockDim.x) A[i][j] = A[i][j] / piv;
        __syncthreads();
        int m = n - j - 1;
        for (int idx = threadIdx.x; idx < m * m; idx += blockDim.x) {
            int i = j + 1 + idx % m, c = j + 1 + idx / m;
            A[i][c] = fma(-A[i][j], A[j][c], A[i][c]);
        }
        __syncthreads();
    }
    for (int idx = threadIdx.x; idx < n * n; idx += blockDim.x) {
        int i = idx % n, j = idx / n;
        Q[i + (int64_t)j * ldq] = A[i][j];
    }
}

void getrf_nopiv_sign(Ctx& cx, int64_t n, double* Q, int64_t ldq, double* S)
{
    for (int64_t j0 = 0; j0 < n; j0 += FACT_NB) {
        int64_t jb = imin(FACT_NB, n - j0);
        double* Qjj = Q + j0 + j0 * ldq;
        getrf_sign_diag<<<1, 256, 0, cx.stream>>>((int)jb, Qjj, ldq, S + j0);
        BQ_LAUNCH_CHECK();
        int64_t rest = n - j0 - jb;
        if (rest > 0) {
            // U12 = L11^{-1} A12 ; L21 = A21 U11^{-1} ; A22 -= L21 U12
            trsm_left_lower_unit(cx, jb, rest, Qjj, ldq, Qjj + jb * ldq, ldq);
            trsm_right_upper(cx, rest, jb, Qjj, ldq, false, false, Qjj + jb, ldq);
            gemm(cx, false, false, rest, rest, jb, -1.0, Qjj + jb, ldq, Qjj + jb * ldq, ldq, 1.0, Qjj + jb + jb * ldq,
                 ldq);
        }
    }
}

// ------------------------------------------------------------------------------------------- misc
__global__ void copy_kernel(int64_t rows, int64_t cols, const double* __restrict__ s, int64_t lds, double* __restrict__ d,
                            int64_t ldd)
{
    int64_t total = rows * cols;
    for (int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; idx < total; idx += (int64_t)gridDim.x * blockDim.x) {
        int64_t r = idx % rows, c = idx / rows;
        d[r + c * ldd] = s[r + c * lds];
    }
}

void copy_matrix(Ctx& cx, int64_t rows, int64_t cols, const double* src, int64_t lds, double* dst, int64_t ldd)
{
    if (rows <= 0 || cols <= 0) return;
    BQ_CUDA(cudaMemcpy2DAsync(dst, ldd * sizeof(double), src, lds * sizeof(double), rows * sizeof(double), cols,
                              cudaMemcpyDeviceToDevice, cx.stream));
}

__global__ void transpose_kernel(int64_t rows, int64_t cols, const double* __restrict__ s, int64_t lds,
                                 double* __restrict__ d, int64_t ldd)
{
    __shared__ double t[32][33];
    int64_t r0 = (int64_t)blockIdx.x * 32, c0 = (int64_t)blockIdx.y * 32;
    for (int k = threadIdx.y; k < 32; k += blockDim.y) {
        int64_t r = r0 + threadIdx.x, c = c0 + k;
        if (r < rows && c < cols) t[k][threadIdx.x] = s[r + c * lds];
    }
    __syncthreads();
    for (int k = threadIdx.y; k < 32; k += blockDim.y) {
        int64_t c = c0 + threadIdx.x, r = r0 + k;  // dst(c, r) = src(r, c)
        if (r < rows && c < cols) d[c + r * ldd] = t[threadIdx.x][k];
    }
}

void transpose_copy(Ctx& cx, int64_t rows, int64_t cols, const double* src, int64_t lds, double* dst, int64_t ldd)
{
    if (rows <= 0 || cols <= 0) return;
    dim3 grid((unsigned)cdiv(rows, 32), (unsigned)cdiv(cols, 32));
    transpose_kernel<<<grid, dim3(32, 8), 0, cx.stream>>>(rows, cols, src, lds, dst, ldd);
    BQ_LAUNCH_CHECK();
}

__global__ void zero_kernel(int64_t rows, int64_t cols, double* A, int64_t lda)
{
    int64_t total = rows * cols;
    for (int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; idx < total; idx += (int64_t)gridDim.x * blockDim.x)
        A[idx % rows + (idx / rows) * lda] = 0.0;
}

void set_zero(Ctx& cx, int64_t rows, int64_t cols, double* A, int64_t lda)
{
    if (rows <= 0 || cols <= 0) return;
    if (lda == rows) {
        BQ_CUDA(cudaMemsetAsync(A, 0, rows * cols * sizeof(double), cx.stream));
        return;
    }
    zero_kernel<<<(unsigned)imin(cdiv(rows * cols, 256), 8 * cx.num_sms), 256, 0, cx.stream>>>(rows, cols, A, lda);
    BQ_LAUNCH_CHECK();
}

__global__ void zero_tri_kernel(int keep_lower, int64_t n, int64_t cols, double* A, int64_t lda, int unit)
{
    int64_t total = n * cols;
    for (int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; idx < total; idx += (int64_t)gridDim.x * blockDim.x) {
        int64_t i = idx % n, j = idx / n;
        if (keep_lower ? (i < j) : (i > j)) A[i + j * lda] = 0.0;
        else if (unit && i == j) A[i + j * lda] = 1.0;
    }
}

void zero_triangle(Ctx& cx, char keep, int64_t n, int64_t cols, double* A, int64_t lda, bool unit_diag)
{
    if (n <= 0 || cols <= 0) return;
    zero_tri_kernel<<<(unsigned)imin(cdiv(n * cols, 256), 8 * cx.num_sms), 256, 0, cx.stream>>>(
        keep == 'L', n, cols, A, lda, unit_diag ? 1 : 0);
    BQ_LAUNCH_CHECK();
}

}  // namespace bqrrp
