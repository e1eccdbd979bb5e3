// sync_bench.cu — cost of one grid-wide barrier (cooperative groups vs a hand-rolled counter barrier) and
// of one cluster barrier, for the latency-bound panel kernels (K-LU, K-SQR).  Prints JSON (us / barrier).
// Build: nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a tools/sync_bench.cu
#include <cooperative_groups.h>
#include <cstdio>

namespace cg = cooperative_groups;

__global__ void cg_loop(int iters, double* sink)
{
    cg::grid_group g = cg::this_grid();
    double acc = 0;
    for (int i = 0; i < iters; ++i) {
        acc += i;
        g.sync();
    }
    if (acc == -1) sink[0] = acc;
}

__device__ __forceinline__ unsigned ld_acquire(const unsigned* p)
{
    unsigned v;
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}

// monotonically increasing arrival counter: barrier i completes when count >= G * (i + 1)
__global__ void counter_loop(int iters, unsigned* counter, double* sink)
{
    const unsigned G = gridDim.x;
    double acc = 0;
    for (int i = 0; i < iters; ++i) {
        acc += i;
        __syncthreads();
        if (threadIdx.x == 0) {
            asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(counter) : "memory");
            const unsigned target = G * (unsigned)(i + 1);
            while (ld_acquire(counter) < target) {
            }
        }
        __syncthreads();
    }
    if (acc == -1) sink[0] = acc;
}

__global__ void cluster_loop(int iters, double* sink)
{
    cg::cluster_group cl = cg::this_cluster();
    double acc = 0;
    for (int i = 0; i < iters; ++i) {
        acc += i;
        cl.sync();
    }
    if (acc == -1) sink[0] = acc;
}

int main()
{
    double* sink;
    unsigned* counter;
    cudaMalloc(&sink, 8);
    cudaMalloc(&counter, 4);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    const int iters = 2000;
    printf("{\n");
    int Gs[] = {4, 8, 16, 32, 64, 148};
    for (int G : Gs) {
        int it = iters;
        void* args[] = {&it, &sink};
        cudaLaunchCooperativeKernel((void*)cg_loop, dim3(G), dim3(256), args, 0, 0);
        cudaEventRecord(e0);
        cudaLaunchCooperativeKernel((void*)cg_loop, dim3(G), dim3(256), args, 0, 0);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        printf("  \"cg_grid_sync_G%d_us\": %.3f,\n", G, 1e3 * ms / iters);
        cudaMemset(counter, 0, 4);
        void* args2[] = {&it, &counter, &sink};
        cudaLaunchCooperativeKernel((void*)counter_loop, dim3(G), dim3(256), args2, 0, 0);
        cudaMemset(counter, 0, 4);
        cudaEventRecord(e0);
        cudaLaunchCooperativeKernel((void*)counter_loop, dim3(G), dim3(256), args2, 0, 0);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        cudaEventElapsedTime(&ms, e0, e1);
        printf("  \"counter_barrier_G%d_us\": %.3f,\n", G, 1e3 * ms / iters);
    }
    cudaFuncSetAttribute(cluster_loop, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    int CLs[] = {2, 4, 8, 16};
    for (int CL : CLs) {
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3(CL);
        cfg.blockDim = dim3(256);
        cudaLaunchAttribute at[1];
        at[0].id = cudaLaunchAttributeClusterDimension;
        at[0].val.clusterDim.x = CL;
        at[0].val.clusterDim.y = 1;
        at[0].val.clusterDim.z = 1;
        cfg.attrs = at;
        cfg.numAttrs = 1;
        cudaLaunchKernelEx(&cfg, cluster_loop, iters, sink);
        cudaEventRecord(e0);
        cudaError_t err = cudaLaunchKernelEx(&cfg, cluster_loop, iters, sink);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        printf("  \"cluster_sync_CL%d_us\": %.3f, \"cluster_CL%d_err\": \"%s\",\n", CL, 1e3 * ms / iters, CL,
               cudaGetErrorString(err));
    }
    printf("  \"iters\": %d\n}\n", iters);
    return 0;
}
