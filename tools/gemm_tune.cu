// gemm_tune.cu — time the DMMA GEMM engine's tile configurations against cuBLAS on the shapes the
// BQRRP iteration uses (C3 trailing update, C3 GEMM1, square), check max |mine - cuBLAS|.
// Build: nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -lineinfo tools/gemm_tune.cu -lcublas
#include <cublas_v2.h>
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "../paper_2507_00976_b200/csrc/dgemm.cuh"

using namespace bqrrp;
// v2 candidates: BM, BN, BK, WARPS_M, WARPS_N, STAGES, MIN_BLOCKS
using V64k16 = Gemm2Cfg<64, 64, 16, 2, 2, 3, 4>;
using V64k16s4 = Gemm2Cfg<64, 64, 16, 2, 2, 4, 3>;
using V64k32 = Gemm2Cfg<64, 64, 32, 2, 2, 3, 2>;
using V128x64 = Gemm2Cfg<128, 64, 16, 4, 2, 3, 2>;
using V128x128 = Gemm2Cfg<128, 128, 16, 2, 4, 3, 1>;
using V128x128w16 = Gemm2Cfg<128, 128, 16, 4, 4, 3, 1>;
using V64x32 = Gemm2Cfg<64, 32, 16, 2, 2, 3, 4>;

__global__ void fill(double* p, size_t n, unsigned seed)
{
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
        unsigned h = (unsigned)(i * 2654435761u) ^ seed;
        h ^= h >> 13; h *= 0x5bd1e995; h ^= h >> 15;
        p[i] = (double)(h & 0xffff) / 65536.0 - 0.5;
    }
}
__global__ void maxdiff(const double* a, const double* b, size_t n, double* out)
{
    double m = 0;
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x)
        m = fmax(m, fabs(a[i] - b[i]));
    atomicMax((unsigned long long*)out, __double_as_longlong(m));
}

template <class Cfg, bool TA, bool TB>
float run(int64_t M, int64_t N, int64_t K, const double* A, int64_t lda, const double* B, int64_t ldb, double* C,
          int reps, double alpha = 1.0, double beta = 0.0)
{
    GemmArgs g{M, N, K, alpha, beta, A, lda, B, ldb, C, M, nullptr, K, 0};
    size_t sm = dgemm_smem_bytes<Cfg, TA, TB>();
    cudaFuncSetAttribute(dgemm_kernel<Cfg, TA, TB>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    dim3 grid(((M + Cfg::BM - 1) / Cfg::BM) * ((N + Cfg::BN - 1) / Cfg::BN), 1, 1);
    dgemm_kernel<Cfg, TA, TB><<<grid, Cfg::THREADS, sm>>>(g);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0); cudaEventCreate(&e1);
    float best = 1e30f;
    for (int r = 0; r < reps; ++r) {
        cudaEventRecord(e0);
        dgemm_kernel<Cfg, TA, TB><<<grid, Cfg::THREADS, sm>>>(g);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        if (ms < best) best = ms;
    }
    return best;
}

template <class Cfg, bool TA, bool TB>
float run2(int64_t M, int64_t N, int64_t K, const double* A, int64_t lda, const double* B, int64_t ldb, double* C,
           int reps, double alpha = 1.0, double beta = 0.0)
{
    GemmArgs g{M, N, K, alpha, beta, A, lda, B, ldb, C, M, nullptr, K, 0};
    size_t sm = dgemm2_smem_bytes<Cfg, TA, TB>();
    cudaFuncSetAttribute(dgemm2_kernel<Cfg, TA, TB>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    dim3 grid(((M + Cfg::BM - 1) / Cfg::BM) * ((N + Cfg::BN - 1) / Cfg::BN), 1, 1);
    int vec = dgemm2_vec_ok(g);
    dgemm2_kernel<Cfg, TA, TB><<<grid, Cfg::THREADS, sm>>>(g, vec);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0); cudaEventCreate(&e1);
    float best = 1e30f;
    for (int r = 0; r < reps; ++r) {
        cudaEventRecord(e0);
        dgemm2_kernel<Cfg, TA, TB><<<grid, Cfg::THREADS, sm>>>(g, vec);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        if (ms < best) best = ms;
    }
    cudaError_t err = cudaGetLastError();
    if (err != cudaSuccess) { fprintf(stderr, "cuda error %s\n", cudaGetErrorString(err)); exit(1); }
    return best;
}

int main()
{
    struct Shape { int64_t M, N, K; bool ta, tb; const char* name; double alpha = 1.0, beta = 0.0; };
    std::vector<Shape> shapes = {
        {8192, 8192, 8192, false, false, "sq8192_NN"},
        {16384, 16384, 2048, false, false, "trail_GEMM2_NN_K2048"},
        {16384, 15360, 1024, false, false, "c2_GEMM2_NN_K1024"},
        {16384, 15360, 1024, false, false, "c2_GEMM2_NN_K1024_beta1", -1.0, 1.0},
        {65536, 4096, 2048, false, false, "c3_GEMM2_slab_beta1", -1.0, 1.0},
        {2048, 16384, 16384, true, false, "trail_GEMM1_TN"},
        {8192, 8192, 8192, true, false, "sq8192_TN"},
        {8192, 8192, 8192, false, true, "sq8192_NT"},
    };
    size_t maxel = 0;
    for (auto& s : shapes) {
        maxel = std::max(maxel, (size_t)s.M * s.K);
        maxel = std::max(maxel, (size_t)s.K * s.N);
        maxel = std::max(maxel, (size_t)s.M * s.N);
    }
    double *A, *B, *C, *Cr, *err;
    cudaMalloc(&A, maxel * 8); cudaMalloc(&B, maxel * 8); cudaMalloc(&C, maxel * 8); cudaMalloc(&Cr, maxel * 8);
    cudaMalloc(&err, 8);
    fill<<<1024, 256>>>(A, maxel, 1); fill<<<1024, 256>>>(B, maxel, 2);
    cublasHandle_t h;
    cublasCreate(&h);
    printf("{\n");
    for (auto& s : shapes) {
        int64_t lda = s.ta ? s.K : s.M, ldb = s.tb ? s.N : s.K;
        double one = s.alpha, zero = s.beta;
        cublasOperation_t oa = s.ta ? CUBLAS_OP_T : CUBLAS_OP_N, ob = s.tb ? CUBLAS_OP_T : CUBLAS_OP_N;
        cublasDgemm(h, oa, ob, s.M, s.N, s.K, &one, A, lda, B, ldb, &zero, Cr, s.M);
        cudaEvent_t e0, e1;
        cudaEventCreate(&e0); cudaEventCreate(&e1);
        float cb = 1e30f;
        for (int r = 0; r < 5; ++r) {
            cudaEventRecord(e0);
            cublasDgemm(h, oa, ob, s.M, s.N, s.K, &one, A, lda, B, ldb, &zero, Cr, s.M);
            cudaEventRecord(e1);
            cudaEventSynchronize(e1);
            float ms; cudaEventElapsedTime(&ms, e0, e1);
            if (ms < cb) cb = ms;
        }
        double fl = 2.0 * s.M * s.N * s.K;
        printf("  \"%s\": {\"cublas\": %.2f", s.name, fl / (cb * 1e-3) / 1e12);
        auto report = [&](const char* nm, float ms) {
            cudaMemset(err, 0, 8);
            maxdiff<<<512, 256>>>(C, Cr, (size_t)s.M * s.N, err);
            double e; cudaMemcpy(&e, err, 8, cudaMemcpyDeviceToHost);
            printf(", \"%s\": %.2f, \"%s_err\": %.1e", nm, fl / (ms * 1e-3) / 1e12, nm, e);
        };
#define RUNV(CFG, NM)                                                                                       \
    cudaMemset(C, 0, (size_t)s.M * s.N * 8);                                                                        \
    if (!s.ta && !s.tb) report(NM, run<CFG, false, false>(s.M, s.N, s.K, A, lda, B, ldb, C, 5, s.alpha, s.beta)); \
    else if (s.ta && !s.tb) report(NM, run<CFG, true, false>(s.M, s.N, s.K, A, lda, B, ldb, C, 5, s.alpha, s.beta)); \
    else report(NM, run<CFG, false, true>(s.M, s.N, s.K, A, lda, B, ldb, C, 5, s.alpha, s.beta));
#define RUNV2(CFG, NM)                                                                                       \
    cudaMemset(C, 0, (size_t)s.M * s.N * 8);                                                                        \
    if (!s.ta && !s.tb) report(NM, run2<CFG, false, false>(s.M, s.N, s.K, A, lda, B, ldb, C, 5, s.alpha, s.beta)); \
    else if (s.ta && !s.tb) report(NM, run2<CFG, true, false>(s.M, s.N, s.K, A, lda, B, ldb, C, 5, s.alpha, s.beta)); \
    else report(NM, run2<CFG, false, true>(s.M, s.N, s.K, A, lda, B, ldb, C, 5, s.alpha, s.beta));
        RUNV(CfgMid, "v1_64x64");
        RUNV2(V64k16, "v2_64x64k16");
        RUNV2(V64k16s4, "v2_64x64k16s4");
        RUNV2(V64k32, "v2_64x64k32");
        RUNV2(V128x64, "v2_128x64");
        RUNV2(V128x128, "v2_128x128");
        RUNV2(V128x128w16, "v2_128x128w16");
        RUNV2(V64x32, "v2_64x32");
        printf("},\n");
        fflush(stdout);
    }
    printf("  \"done\": 1\n}\n");
    return 0;
}
