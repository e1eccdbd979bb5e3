// sketch.cu — a1: the Gaussian sketch, applied once (P:476-479 steps bqrrp:sample / bqrrp:sketching;
// P:525 "uses randomness only once"; §3.2).  S is d x m (reading Z2), iid N(0,1)
// (variance one, Z3), drawn from the counter-based generator of rng.cuh; the sketch is stored
// transposed, MskT = (S A)^T = A^T S^T (n x d), so that the LU pivot search (a2) and the sketch update
// (a6) touch contiguous columns.
#include "blas.cuh"
#include "bqrrp_internal.cuh"
#include "rng.cuh"

namespace bqrrp {

__global__ void sketch_operator_T_kernel(int64_t m, int64_t d, uint64_t seed, double* St, int64_t ldst)
{
    int64_t total = m * d;
    for (int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; idx < total; idx += (int64_t)gridDim.x * blockDim.x) {
        int64_t l = idx % m, i = idx / m;
        St[l + i * ldst] = rng_gauss(seed, 0u, (uint64_t)i, (uint64_t)l);
    }
}

void sketch_operator_T(Ctx& cx, int64_t m, int64_t d, uint64_t seed, double* St, int64_t ldst)
{
    if (m <= 0 || d <= 0) return;
    unsigned blocks = (unsigned)imin(cdiv(m * d, 256), 16 * cx.num_sms);
    sketch_operator_T_kernel<<<blocks, 256, 0, cx.stream>>>(m, d, seed, St, ldst);
    BQ_LAUNCH_CHECK();
}

void sketch_apply(Ctx& cx, int64_t m, int64_t n, const double* A, int64_t lda, int64_t d, uint64_t seed, double* MskT,
                  int64_t ldm, double* St)
{
    sketch_operator_T(cx, m, d, seed, St, m);
    // MskT (n x d) = A^T (n x m) * St (m x d)
    gemm(cx, true, false, n, d, m, 1.0, A, lda, St, m, 0.0, MskT, ldm, false, 0, /*no_split=*/true);
}

}  // namespace bqrrp
