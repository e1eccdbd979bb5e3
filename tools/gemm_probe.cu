// gemm_probe.cu — one repo DGEMM launch (config chosen by argv[2]) on an 8192^3 NN problem, for
// ncu --set full captures.  Build: nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -lineinfo
// tools/gemm_probe.cu
#include <cstdio>
#include <cstdlib>
#include <cstring>

#include "../paper_2507_00976_b200/csrc/dgemm.cuh"

using namespace bqrrp;
using CfgSmall4 = GemmCfg<64, 32, 2, 2, 4>;

__global__ void fill(double* p, size_t n, unsigned seed)
{
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
        unsigned h = (unsigned)(i * 2654435761u) ^ seed;
        h ^= h >> 13; h *= 0x5bd1e995; h ^= h >> 15;
        p[i] = (double)(h & 0xffff) / 65536.0 - 0.5;
    }
}

template <class Cfg>
void run(int64_t N, const double* A, const double* B, double* C)
{
    GemmArgs g{N, N, N, 1.0, 0.0, A, N, B, N, C, N, nullptr, N, 0};
    size_t sm = dgemm_smem_bytes<Cfg, false, false>();
    cudaFuncSetAttribute(dgemm_kernel<Cfg, false, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    dim3 grid(((N + Cfg::BM - 1) / Cfg::BM) * ((N + Cfg::BN - 1) / Cfg::BN), 1, 1);
    dgemm_kernel<Cfg, false, false><<<grid, Cfg::THREADS, sm>>>(g);
}

int main(int argc, char** argv)
{
    const int64_t N = argc > 1 ? atoll(argv[1]) : 8192;
    const char* cfg = argc > 2 ? argv[2] : "small4";
    size_t nn = (size_t)N * N;
    double *A, *B, *C;
    cudaMalloc(&A, nn * 8); cudaMalloc(&B, nn * 8); cudaMalloc(&C, nn * 8);
    fill<<<1024, 256>>>(A, nn, 1); fill<<<1024, 256>>>(B, nn, 2);
    if (!strcmp(cfg, "small4")) run<CfgSmall4>(N, A, B, C);
    else if (!strcmp(cfg, "small")) run<CfgSmall>(N, A, B, C);
    else if (!strcmp(cfg, "mid")) run<CfgMid>(N, A, B, C);
    else run<CfgWide>(N, A, B, C);
    cudaDeviceSynchronize();
    printf("done %s %s\n", cfg, cudaGetErrorString(cudaGetLastError()));
    return 0;
}
