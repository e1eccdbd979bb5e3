// gemm_probe.cu — one cuBLAS DGEMM and one repo DGEMM (csrc/dgemm.cuh) on the same 8192^3 NN problem,
// for side-by-side ncu --set full captures.  Build: nvcc -O3 -gencode arch=compute_100a,code=sm_100a
// -lineinfo tools/gemm_probe.cu -lcublas
#include <cublas_v2.h>
#include <cstdio>
#include <cstdlib>

#include "../paper_2507_00976_b200/csrc/dgemm.cuh"

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
    const int64_t N = argc > 1 ? atoll(argv[1]) : 8192;
    size_t nn = (size_t)N * N;
    double *A, *B, *C;
    cudaMalloc(&A, nn * 8); cudaMalloc(&B, nn * 8); cudaMalloc(&C, nn * 8);
    fill<<<1024, 256>>>(A, nn, 1); fill<<<1024, 256>>>(B, nn, 2);
    cublasHandle_t h;
    cublasCreate(&h);
    double one = 1, zero = 0;
    cublasDgemm(h, CUBLAS_OP_N, CUBLAS_OP_N, N, N, N, &one, A, N, B, N, &zero, C, N);
    bqrrp::GemmArgs g{N, N, N, 1.0, 0.0, A, N, B, N, C, N, nullptr, N, 0};
    size_t sm = bqrrp::dgemm_smem_bytes<bqrrp::CfgWide, false, false>();
    cudaFuncSetAttribute(bqrrp::dgemm_kernel<bqrrp::CfgWide, false, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    dim3 grid((N + 127) / 128, (N + 63) / 64, 1);
    bqrrp::dgemm_kernel<bqrrp::CfgWide, false, false><<<grid, bqrrp::CfgWide::THREADS, sm>>>(g);
    cudaDeviceSynchronize();
    printf("done %s\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}
