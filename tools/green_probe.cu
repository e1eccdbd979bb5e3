// Green-context probe (B200): can a stream bound to an SM partition (driver green context) take runtime-API
// launches on memory of the primary context, and does it confine the kernel to its SMs?  Also: latency of a
// small high-priority 16-CTA cluster kernel launched while a long low-priority kernel fills (a) the whole device,
// (b) a green partition of N SMs.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/green_probe tools/green_probe.cu && /tmp/green_probe 120
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdlib>
#include <set>

#define CK(x)                                                                              \
    do {                                                                                   \
        cudaError_t e_ = (x);                                                              \
        if (e_ != cudaSuccess) {                                                           \
            printf("%s:%d %s: %s\n", __FILE__, __LINE__, #x, cudaGetErrorString(e_));      \
            exit(1);                                                                       \
        }                                                                                  \
    } while (0)
#define CKD(x)                                                     \
    do {                                                           \
        CUresult r_ = (x);                                         \
        if (r_ != CUDA_SUCCESS) {                                  \
            printf("%s:%d %s: CUresult %d\n", __FILE__, __LINE__, #x, (int)r_); \
            exit(1);                                               \
        }                                                          \
    } while (0)

template <class F>
static F drv(const char* name)
{
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    CK(cudaGetDriverEntryPoint(name, &p, cudaEnableDefault, &q));
    if (!p) {
        printf("no %s\n", name);
        exit(1);
    }
    return (F)p;
}

__global__ void smid_kernel(int* out)
{
    unsigned s;
    asm volatile("mov.u32 %0, %%smid;" : "=r"(s));
    if (threadIdx.x == 0) out[blockIdx.x] = (int)s;
}

__global__ void busy_kernel(double* x, long iters)
{
    double a = x[threadIdx.x], b = 1.0000001;
    for (long i = 0; i < iters; ++i) a = fma(a, b, 1e-9);
    if (a == 12345.0) x[threadIdx.x] = a;
}

__global__ void __cluster_dims__(16, 1, 1) small_cluster_kernel(double* x)
{
    if (threadIdx.x == 0) x[blockIdx.x] += 1.0;
}

__global__ void busy_big_kernel(double* x, long iters)
{
    extern __shared__ double sm[];
    double a = x[threadIdx.x], b = 1.0000001;
    for (long i = 0; i < iters; ++i) a = fma(a, b, 1e-9);
    sm[threadIdx.x] = a;
    if (a == 12345.0) x[threadIdx.x] = sm[threadIdx.x ^ 1];
}

__global__ void cluster16_big_kernel(double* x)
{
    extern __shared__ double sm[];
    sm[threadIdx.x] = 1.0;
    if (threadIdx.x == 0) x[64 + blockIdx.x] += sm[0];
}

int main(int argc, char** argv)
{
    const int nsm = argc > 1 ? atoi(argv[1]) : 120;
    CK(cudaSetDevice(0));
    CK(cudaFree(0));
    auto pGetRes = drv<CUresult (*)(CUdevice, CUdevResource*, CUdevResourceType)>("cuDeviceGetDevResource");
    auto pSplit = drv<CUresult (*)(CUdevResource*, unsigned*, const CUdevResource*, CUdevResource*, unsigned, unsigned)>(
        "cuDevSmResourceSplitByCount");
    auto pDesc = drv<CUresult (*)(CUdevResourceDesc*, CUdevResource*, unsigned)>("cuDevResourceGenerateDesc");
    auto pGreen = drv<CUresult (*)(CUgreenCtx*, CUdevResourceDesc, CUdevice, unsigned)>("cuGreenCtxCreate");
    auto pGStream = drv<CUresult (*)(CUstream*, CUgreenCtx, unsigned, int)>("cuGreenCtxStreamCreate");
    CUdevResource all, part, rest;
    CKD(pGetRes(0, &all, CU_DEV_RESOURCE_TYPE_SM));
    unsigned ng = 1;
    CKD(pSplit(&part, &ng, &all, &rest, 0, (unsigned)nsm));
    printf("device SMs %u, partition %u SMs, remaining %u\n", all.sm.smCount, part.sm.smCount, rest.sm.smCount);
    CUdevResourceDesc desc;
    CKD(pDesc(&desc, &part, 1));
    CUgreenCtx g;
    CKD(pGreen(&g, desc, 0, CU_GREEN_CTX_DEFAULT_STREAM));
    int lo, hi;
    CK(cudaDeviceGetStreamPriorityRange(&lo, &hi));
    CUstream gs;
    CKD(pGStream(&gs, g, CU_STREAM_NON_BLOCKING, lo));
    cudaStream_t gstream = (cudaStream_t)gs;
    int* d_sm;
    CK(cudaMalloc(&d_sm, 4096 * sizeof(int)));
    smid_kernel<<<4096, 128, 0, gstream>>>(d_sm);
    CK(cudaGetLastError());
    CK(cudaStreamSynchronize(gstream));
    int h_sm[4096];
    CK(cudaMemcpy(h_sm, d_sm, sizeof h_sm, cudaMemcpyDeviceToHost));
    std::set<int> s(h_sm, h_sm + 4096);
    printf("runtime launch on the green stream: %zu distinct SMs used (partition %u)\n", s.size(), part.sm.smCount);
    smid_kernel<<<4096, 128>>>(d_sm);
    CK(cudaDeviceSynchronize());
    CK(cudaMemcpy(h_sm, d_sm, sizeof h_sm, cudaMemcpyDeviceToHost));
    std::set<int> s2(h_sm, h_sm + 4096);
    printf("runtime launch on the default stream: %zu distinct SMs used\n", s2.size());

    // latency of a small high-priority cluster kernel while a long low-priority kernel occupies the device / part
    double* x;
    CK(cudaMalloc(&x, 1 << 20));
    CK(cudaMemset(x, 0, 1 << 20));
    cudaStream_t full_lo, hi_s;
    CK(cudaStreamCreateWithPriority(&full_lo, cudaStreamNonBlocking, lo));
    CK(cudaStreamCreateWithPriority(&hi_s, cudaStreamNonBlocking, hi));
    cudaEvent_t e0, e1;
    CK(cudaEventCreate(&e0));
    CK(cudaEventCreate(&e1));
    for (int mode = 0; mode < 3; ++mode) {
        cudaStream_t bs = mode == 1 ? full_lo : gstream;
        if (mode > 0) busy_kernel<<<148 * 8, 256, 0, bs>>>(x, 4000000);  // ~ tens of ms, 8 CTAs per SM
        for (int w = 0; w < 3; ++w) small_cluster_kernel<<<16, 128, 0, hi_s>>>(x);  // warm
        CK(cudaStreamSynchronize(hi_s));
        float best = 1e30f, sum = 0.f;
        for (int r = 0; r < 20; ++r) {
            CK(cudaEventRecord(e0, hi_s));
            small_cluster_kernel<<<16, 128, 0, hi_s>>>(x);
            CK(cudaEventRecord(e1, hi_s));
            CK(cudaEventSynchronize(e1));
            float ms;
            CK(cudaEventElapsedTime(&ms, e0, e1));
            best = ms < best ? ms : best;
            sum += ms;
        }
        printf("%s: 16-CTA cluster kernel latency best %.1f us, mean %.1f us\n",
               mode == 0 ? "idle device" : (mode == 1 ? "busy kernel on the whole device" : "busy kernel on the green partition"),
               best * 1e3f, sum / 20 * 1e3f);
        CK(cudaDeviceSynchronize());
    }
    // full-SM footprint: the busy kernel takes 200 KB of shared memory per CTA (one per SM) on the partition; a
    // 16-CTA cluster with the same footprint (one CTA per SM) then needs 16 whole free SMs in one GPC
    {
        const int big = 200 * 1024;
        CK(cudaFuncSetAttribute(busy_big_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, big));
        CK(cudaFuncSetAttribute(cluster16_big_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, big));
        CK(cudaFuncSetAttribute(cluster16_big_kernel, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
        for (int csize : {16, 8, 4}) {
            cudaLaunchConfig_t cfg = {};
            cfg.gridDim = dim3(csize);
            cfg.blockDim = dim3(128);
            cfg.dynamicSmemBytes = big;
            cfg.stream = hi_s;
            cudaLaunchAttribute at[1];
            at[0].id = cudaLaunchAttributeClusterDimension;
            at[0].val.clusterDim.x = csize;
            at[0].val.clusterDim.y = 1;
            at[0].val.clusterDim.z = 1;
            cfg.attrs = at;
            cfg.numAttrs = 1;
            int ncl = 0;
            CK(cudaOccupancyMaxActiveClusters(&ncl, cluster16_big_kernel, &cfg));
            for (int mode = 0; mode < 2; ++mode) {
                cudaStream_t bs = mode == 0 ? full_lo : gstream;
                // busy: one CTA per SM of its stream's SMs, ~30 ms
                busy_big_kernel<<<mode == 0 ? 148 : part.sm.smCount, 128, big, bs>>>(x, 3000000);
                CK(cudaGetLastError());
                float best = 1e30f, sum = 0.f;
                for (int r = 0; r < 10; ++r) {
                    CK(cudaEventRecord(e0, hi_s));
                    CK(cudaLaunchKernelEx(&cfg, cluster16_big_kernel, x));
                    CK(cudaEventRecord(e1, hi_s));
                    CK(cudaEventSynchronize(e1));
                    float ms;
                    CK(cudaEventElapsedTime(&ms, e0, e1));
                    best = ms < best ? ms : best;
                    sum += ms;
                }
                printf("cluster %d x 200KB (max active clusters on an idle device %d) while a full-SM busy kernel fills %s: "
                       "first-10 latency best %.1f us mean %.1f us\n", csize, ncl,
                       mode == 0 ? "the whole device" : "the green partition", best * 1e3f, sum / 10 * 1e3f);
                CK(cudaDeviceSynchronize());
            }
        }
    }
    // GPC-aware split: groups of 16 SMs that can host a maximal cluster (CU_DEV_SM_RESOURCE_SPLIT_MAX_POTENTIAL_
    // CLUSTER_SIZE); the bulk context gets all groups but the last (+ the remainder), the last group stays free
    {
        unsigned ngq = 0;
        CKD(pSplit(nullptr, &ngq, &all, nullptr, CU_DEV_SM_RESOURCE_SPLIT_MAX_POTENTIAL_CLUSTER_SIZE, 16));
        CUdevResource grp[64], rem2;
        unsigned ng2 = ngq;
        CKD(pSplit(grp, &ng2, &all, &rem2, CU_DEV_SM_RESOURCE_SPLIT_MAX_POTENTIAL_CLUSTER_SIZE, 16));
        printf("max-cluster split into groups of 16: %u groups (", ng2);
        for (unsigned i = 0; i < ng2; ++i) printf("%u ", grp[i].sm.smCount);
        printf("), remainder %u SMs\n", rem2.sm.smCount);
        CUdevResource sel[65];
        unsigned ns = 0;
        for (unsigned i = 0; i + 1 < ng2; ++i) sel[ns++] = grp[i];
        if (rem2.sm.smCount) sel[ns++] = rem2;
        CUdevResourceDesc d2;
        CKD(pDesc(&d2, sel, ns));
        CUgreenCtx g2;
        CKD(pGreen(&g2, d2, 0, CU_GREEN_CTX_DEFAULT_STREAM));
        CUstream gs2;
        CKD(pGStream(&gs2, g2, CU_STREAM_NON_BLOCKING, lo));
        unsigned nbulk = 0;
        for (unsigned i = 0; i < ns; ++i) nbulk += sel[i].sm.smCount;
        const int big = 200 * 1024;
        for (int csize : {16, 8}) {
            cudaLaunchConfig_t cfg = {};
            cfg.gridDim = dim3(csize);
            cfg.blockDim = dim3(128);
            cfg.dynamicSmemBytes = big;
            cfg.stream = hi_s;
            cudaLaunchAttribute at[1];
            at[0].id = cudaLaunchAttributeClusterDimension;
            at[0].val.clusterDim.x = csize;
            at[0].val.clusterDim.y = 1;
            at[0].val.clusterDim.z = 1;
            cfg.attrs = at;
            cfg.numAttrs = 1;
            busy_big_kernel<<<nbulk, 128, big, (cudaStream_t)gs2>>>(x, 3000000);
            CK(cudaGetLastError());
            float best = 1e30f, sum = 0.f;
            for (int r = 0; r < 10; ++r) {
                CK(cudaEventRecord(e0, hi_s));
                CK(cudaLaunchKernelEx(&cfg, cluster16_big_kernel, x));
                CK(cudaEventRecord(e1, hi_s));
                CK(cudaEventSynchronize(e1));
                float ms;
                CK(cudaEventElapsedTime(&ms, e0, e1));
                best = ms < best ? ms : best;
                sum += ms;
            }
            printf("cluster %d x 200KB while a full-SM busy kernel fills the %u-SM GPC-aware partition: latency best %.1f us "
                   "mean %.1f us\n", csize, nbulk, best * 1e3f, sum / 10 * 1e3f);
            CK(cudaDeviceSynchronize());
        }
    }
    printf("ok\n");
    return 0;
}
