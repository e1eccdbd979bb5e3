// fp64_bench.cu — measure the B200 FP64 roofline denominators:
//   * DMMA.8x8x4 issue-bound throughput (mma.sync.m8n8k4.f64, register-resident operands)
//   * DFMA throughput (plain FP64 FMA pipe)
//   * cuBLAS DGEMM 8192^3: best-of-10 burst and a 4 s back-to-back sustained loop (library reference)
//   * this repo's DMMA GEMM engine on the same shapes, with a max-relative-error check vs cuBLAS.
// Prints one JSON object.  Build: nvcc -O3 -gencode arch=compute_100a,code=sm_100a -lcublas
#include <cublas_v2.h>
#include <cuda_runtime.h>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "../paper_2507_00976_b200/csrc/dgemm.cuh"

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { fprintf(stderr, "%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e)); exit(1); } } while (0)

__global__ void dmma_peak(double* out, int iters)
{
    double a = threadIdx.x * 1e-3, b = blockIdx.x * 1e-3;
    double c[8][2];
#pragma unroll
    for (int i = 0; i < 8; ++i) c[i][0] = c[i][1] = 0.0;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int i = 0; i < 8; ++i) bqrrp::dmma_884(c[i][0], c[i][1], a, b);
    }
    double s = 0;
#pragma unroll
    for (int i = 0; i < 8; ++i) s += c[i][0] + c[i][1];
    if (s == 12345.678) out[0] = s;
}

__global__ void dfma_peak(double* out, int iters)
{
    double x[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) x[i] = threadIdx.x + i;
    double y = 1.0000001, z = 1e-9;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int i = 0; i < 8; ++i) x[i] = fma(x[i], y, z);
    }
    double s = 0;
#pragma unroll
    for (int i = 0; i < 8; ++i) s += x[i];
    if (s == 12345.678) out[0] = s;
}

__global__ void fill(double* p, size_t n, unsigned seed)
{
    size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x;
    for (; i < n; i += (size_t)gridDim.x * blockDim.x) {
        unsigned h = (unsigned)(i * 2654435761u) ^ seed;
        h ^= h >> 13; h *= 0x5bd1e995; h ^= h >> 15;
        p[i] = (double)(h & 0xffff) / 65536.0 - 0.5;
    }
}

__global__ void maxrel(const double* a, const double* b, size_t n, double* out)
{
    __shared__ double s[256];
    double m = 0;
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x)
        m = fmax(m, fabs(a[i] - b[i]));
    s[threadIdx.x] = m;
    __syncthreads();
    for (int o = 128; o > 0; o >>= 1) { if (threadIdx.x < o) s[threadIdx.x] = fmax(s[threadIdx.x], s[threadIdx.x + o]); __syncthreads(); }
    if (threadIdx.x == 0) {
        unsigned long long* p = (unsigned long long*)out;
        atomicMax(p, __double_as_longlong(s[0]));
    }
}

template <bool TA, bool TB>
void my_gemm(int64_t M, int64_t N, int64_t K, const double* A, int64_t lda, const double* B, int64_t ldb, double* C,
             int64_t ldc, cudaStream_t st)
{
    bqrrp::GemmArgs g{M, N, K, 1.0, 0.0, A, lda, B, ldb, C, ldc, nullptr, K, 0};
    size_t sm = bqrrp::dgemm_smem_bytes<bqrrp::CfgWide, TA, TB>();
    static bool init = false;
    if (!init) { CK(cudaFuncSetAttribute(bqrrp::dgemm_kernel<bqrrp::CfgWide, TA, TB>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm)); init = true; }
    dim3 grid(((M + 127) / 128) * ((N + 63) / 64), 1, 1);
    bqrrp::dgemm_kernel<bqrrp::CfgWide, TA, TB><<<grid, bqrrp::CfgWide::THREADS, sm, st>>>(g);
}

int main(int argc, char** argv)
{
    int nsm = 0;
    CK(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0));
    double* dummy;
    CK(cudaMalloc(&dummy, 8));
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0); cudaEventCreate(&e1);
    float ms;
    printf("{\n  \"sms\": %d,\n", nsm);

    // DMMA peak: 8 independent chains per warp, 4 warps/SMSP
    {
        int iters = 20000, blocks = nsm * 4, threads = 512;
        dmma_peak<<<blocks, threads>>>(dummy, 100);
        CK(cudaDeviceSynchronize());
        double best = 0;
        for (int r = 0; r < 5; ++r) {
            cudaEventRecord(e0);
            dmma_peak<<<blocks, threads>>>(dummy, iters);
            cudaEventRecord(e1);
            CK(cudaEventSynchronize(e1));
            cudaEventElapsedTime(&ms, e0, e1);
            double flops = 2.0 * 256 * 8 * (double)iters * blocks * (threads / 32);
            best = fmax(best, flops / (ms * 1e-3) / 1e12);
        }
        printf("  \"dmma_tflops\": %.3f,\n", best);
    }
    {
        int iters = 20000, blocks = nsm * 4, threads = 512;
        dfma_peak<<<blocks, threads>>>(dummy, 100);
        CK(cudaDeviceSynchronize());
        double best = 0;
        for (int r = 0; r < 5; ++r) {
            cudaEventRecord(e0);
            dfma_peak<<<blocks, threads>>>(dummy, iters);
            cudaEventRecord(e1);
            CK(cudaEventSynchronize(e1));
            cudaEventElapsedTime(&ms, e0, e1);
            double flops = 2.0 * 8 * (double)iters * blocks * threads;
            best = fmax(best, flops / (ms * 1e-3) / 1e12);
        }
        printf("  \"dfma_tflops\": %.3f,\n", best);
    }

    const int64_t N = argc > 1 ? atoll(argv[1]) : 8192;
    size_t nn = (size_t)N * N;
    double *A, *B, *C, *C2, *err;
    CK(cudaMalloc(&A, nn * 8)); CK(cudaMalloc(&B, nn * 8)); CK(cudaMalloc(&C, nn * 8)); CK(cudaMalloc(&C2, nn * 8));
    CK(cudaMalloc(&err, 8));
    fill<<<1024, 256>>>(A, nn, 1); fill<<<1024, 256>>>(B, nn, 2);
    cublasHandle_t h;
    cublasCreate(&h);
    double one = 1, zero = 0;
    double flops = 2.0 * N * N * N;
    auto cub = [&](cublasOperation_t ta, cublasOperation_t tb) {
        cublasDgemm(h, ta, tb, N, N, N, &one, A, N, B, N, &zero, C, N);
    };
    cub(CUBLAS_OP_N, CUBLAS_OP_N);
    CK(cudaDeviceSynchronize());
    double best = 0;
    for (int r = 0; r < 10; ++r) {
        cudaEventRecord(e0); cub(CUBLAS_OP_N, CUBLAS_OP_N); cudaEventRecord(e1);
        CK(cudaEventSynchronize(e1)); cudaEventElapsedTime(&ms, e0, e1);
        best = fmax(best, flops / (ms * 1e-3) / 1e12);
    }
    printf("  \"cublas_dgemm_%lld_tflops_burst\": %.3f,\n", (long long)N, best);
    {
        auto t0 = std::chrono::steady_clock::now();
        int cnt = 0;
        cudaEventRecord(e0);
        while (std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count() < 4.0) {
            cub(CUBLAS_OP_N, CUBLAS_OP_N); ++cnt;
            if (cnt % 8 == 0) cudaDeviceSynchronize();
        }
        cudaEventRecord(e1); CK(cudaEventSynchronize(e1)); cudaEventElapsedTime(&ms, e0, e1);
        printf("  \"cublas_dgemm_%lld_tflops_sustained\": %.3f,\n", (long long)N, cnt * flops / (ms * 1e-3) / 1e12);
    }

    auto run_mine = [&](int variant) {
        switch (variant) {
        case 0: my_gemm<false, false>(N, N, N, A, N, B, N, C2, N, 0); break;
        case 1: my_gemm<true, false>(N, N, N, A, N, B, N, C2, N, 0); break;
        case 2: my_gemm<false, true>(N, N, N, A, N, B, N, C2, N, 0); break;
        default: my_gemm<true, true>(N, N, N, A, N, B, N, C2, N, 0); break;
        }
    };
    const char* names[4] = {"NN", "TN", "NT", "TT"};
    cublasOperation_t ops[2] = {CUBLAS_OP_N, CUBLAS_OP_T};
    for (int v = 0; v < 4; ++v) {
        run_mine(v);
        CK(cudaDeviceSynchronize());
        best = 0;
        for (int r = 0; r < 10; ++r) {
            cudaEventRecord(e0); run_mine(v); cudaEventRecord(e1);
            CK(cudaEventSynchronize(e1)); cudaEventElapsedTime(&ms, e0, e1);
            best = fmax(best, flops / (ms * 1e-3) / 1e12);
        }
        cub(ops[v & 1], ops[v >> 1]);
        CK(cudaMemset(err, 0, 8));
        maxrel<<<512, 256>>>(C, C2, nn, err);
        double herr;
        CK(cudaMemcpy(&herr, err, 8, cudaMemcpyDeviceToHost));
        printf("  \"mine_%s_tflops\": %.3f, \"mine_%s_maxabs_err_vs_cublas\": %.3e,\n", names[v], best, names[v], herr);
    }
    {
        auto t0 = std::chrono::steady_clock::now();
        int cnt = 0;
        cudaEventRecord(e0);
        while (std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count() < 4.0) {
            run_mine(0); ++cnt;
            if (cnt % 8 == 0) cudaDeviceSynchronize();
        }
        cudaEventRecord(e1); CK(cudaEventSynchronize(e1)); cudaEventElapsedTime(&ms, e0, e1);
        printf("  \"mine_NN_tflops_sustained\": %.3f,\n", cnt * flops / (ms * 1e-3) / 1e12);
    }
    printf("  \"n\": %lld\n}\n", (long long)N);
    return 0;
}
