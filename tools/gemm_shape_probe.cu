// gemm_shape_probe.cu — one launch of the library's DMMA GEMM on a given shape through the same tile
// choice as blas.cu's large-GEMM path (v2 64x64, BK 16, 3 stages, rasterised), e.g. the C3 bulk trailing GEMM at
// iteration 0: M = N = 63488, K = 2048, alpha = -1, beta = 1 (NN) — for an `ncu --set full` capture
// of dram bytes per launch (bench.py roofline.traffic).
// Build: nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -lineinfo tools/gemm_shape_probe.cu
#include <cstdio>
#include <cstdlib>

#include "../paper_2507_00976_b200/csrc/dgemm.cuh"

using namespace bqrrp;

__global__ void fill(double* p, size_t n, unsigned seed)
{
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
        unsigned h = (unsigned)(i * 2654435761u) ^ seed;
        h ^= h >> 13; h *= 0x5bd1e995; h ^= h >> 15;
        p[i] = (double)(h & 0xffff) / 65536.0 - 0.5;
    }
}

int main(int argc, char** argv)
{
    const int64_t M = argc > 1 ? atoll(argv[1]) : 63488, N = argc > 2 ? atoll(argv[2]) : 63488,
                  K = argc > 3 ? atoll(argv[3]) : 2048;
    double *A, *B, *C;
    cudaMalloc(&A, (size_t)M * K * 8);
    cudaMalloc(&B, (size_t)K * N * 8);
    cudaMalloc(&C, (size_t)M * N * 8);
    fill<<<2048, 256>>>(A, (size_t)M * K, 1);
    fill<<<2048, 256>>>(B, (size_t)K * N, 2);
    fill<<<2048, 256>>>(C, (size_t)M * N, 3);
    GemmArgs g{M, N, K, -1.0, 1.0, A, M, B, K, C, M, nullptr, K, 0};
    using Cfg = Cfg2Mid;  // the library's large-GEMM configuration (blas.cu)
    constexpr size_t sm = dgemm2_smem_bytes<Cfg, false, false>();
    cudaFuncSetAttribute(dgemm2_kernel<Cfg, false, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    const int vec = dgemm2_vec_ok(g);
    dim3 grid((unsigned)(((M + 63) / 64) * ((N + 63) / 64)));
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    dgemm2_kernel<Cfg, false, false><<<grid, Cfg::THREADS, sm>>>(g, vec);  // warm
    cudaEventRecord(e0);
    dgemm2_kernel<Cfg, false, false><<<grid, Cfg::THREADS, sm>>>(g, vec);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    double fl = 2.0 * M * N * K, bytes = 8.0 * ((double)M * K + (double)K * N + 2.0 * M * N);
    printf("{\"M\": %lld, \"N\": %lld, \"K\": %lld, \"ms\": %.3f, \"tflops\": %.2f, \"algorithmic_bytes\": %.4e, "
           "\"err\": \"%s\"}\n",
           (long long)M, (long long)N, (long long)K, ms, fl / (ms * 1e-3) / 1e12, bytes,
           cudaGetErrorString(cudaGetLastError()));
    return 0;
}
