// Microbenchmark of the per-column cluster exchange used by the register leaves (K-LU, K-SQR): G CTAs of one
// cluster, 256 threads each, ROUNDS rounds; per round every CTA sends a record of REC doubles to every CTA and
// waits until it has all G records.  Variants:
//   0: st.async + mbarrier complete_tx (the leaves' current form), warp 0 pushes (lane l: value l, loop over ranks)
//   1: barrier.cluster arrive/wait, then warp 0 pulls the G records with ld.shared::cluster
//   2: st.async with the push spread over lanes (lane l -> rank l % G) + mbarrier
// Prints cycles per round (clock64 of CTA 0 thread 0).
#include <cooperative_groups.h>
#include <cstdio>
#include <cstdlib>
namespace cg = cooperative_groups;

__device__ __forceinline__ unsigned smem_u32(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }
__device__ __forceinline__ unsigned mapa_u32(unsigned addr, int rank)
{
    unsigned r;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(addr), "r"(rank));
    return r;
}
__device__ __forceinline__ void st_async_f64(unsigned remote_addr, double v, unsigned remote_mbar)
{
    asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.b64 [%0], %1, [%2];" ::"r"(remote_addr),
                 "l"(__double_as_longlong(v)), "r"(remote_mbar)
                 : "memory");
}
__device__ __forceinline__ void mbar_init(unsigned mbar, unsigned count)
{
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(mbar), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(unsigned mbar, unsigned bytes)
{
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(mbar), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait_parity(unsigned mbar, unsigned parity)
{
    asm volatile("{\n.reg .pred p;\nWAIT_%=:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n@!p bra WAIT_%=;\n}\n" ::"r"(mbar),
                 "r"(parity)
                 : "memory");
}

constexpr int REC = 34, GMAX = 16;

__global__ void __launch_bounds__(256, 1) bench(int variant, int rounds, long long* out, double* sink)
{
    cg::cluster_group cluster = cg::this_cluster();
    const int G = cluster.num_blocks(), me = cluster.block_rank(), tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    __shared__ __align__(16) double slot[2][GMAX][REC];
    __shared__ __align__(16) double mine[2][REC];
    __shared__ __align__(8) unsigned long long mbar[2];
    if (tid == 0) {
        mbar_init(smem_u32(&mbar[0]), 1);
        mbar_init(smem_u32(&mbar[1]), 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    cluster.sync();
    double acc = 0.0;
    long long t0 = clock64();
    for (int j = 0; j < rounds; ++j) {
        const int par = j & 1;
        const double val = acc + j + me;
        if (variant == 0 || variant == 2) {
            const unsigned mb = smem_u32(&mbar[par]);
            if (warp == 0) {
                const unsigned dst = smem_u32(&slot[par][me][0]);
                if (variant == 0) {
                    for (int rk = 0; rk < G; ++rk) {
                        const unsigned rm = mapa_u32(mb, rk), rd = mapa_u32(dst, rk);
                        if (lane < 2) st_async_f64(rd + 8 * lane, val, rm);
                        st_async_f64(rd + 8 * (2 + lane), val + lane, rm);
                    }
                } else {
                    // lane l handles ranks l % G, values in chunks
                    for (int idx = lane; idx < G * REC; idx += 32) {
                        const int rk = idx / REC, e = idx % REC;
                        st_async_f64(mapa_u32(dst, rk) + 8 * e, val + e, mapa_u32(mb, rk));
                    }
                }
            }
            if (tid == 0) mbar_arrive_expect_tx(mb, (unsigned)(G * REC * sizeof(double)));
            mbar_wait_parity(mb, (unsigned)((j >> 1) & 1));
            if (lane < G) acc += slot[par][lane][0] * 1e-30;
        } else {
            if (tid < REC) mine[par][tid] = val + tid;
            cluster.sync();
            if (warp == 0) {
                double v[GMAX];
#pragma unroll
                for (int rk = 0; rk < GMAX; ++rk) v[rk] = (rk < G) ? *cluster.map_shared_rank(&mine[par][lane], rk) : 0.0;
#pragma unroll
                for (int rk = 0; rk < GMAX; ++rk) acc += v[rk] * 1e-30;
            }
        }
        __syncthreads();
    }
    long long t1 = clock64();
    cluster.sync();
    if (me == 0 && tid == 0) *out = (t1 - t0) / rounds;
    if (acc == 12345.0) *sink = acc;
}

int main(int argc, char** argv)
{
    long long* d_out;
    double* d_sink;
    cudaMalloc(&d_out, 8);
    cudaMalloc(&d_sink, 8);
    cudaFuncSetAttribute(bench, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    for (int G : {2, 4, 8, 16}) {
        for (int variant = 0; variant < 3; ++variant) {
            cudaLaunchConfig_t cfg = {};
            cfg.gridDim = dim3(G);
            cfg.blockDim = dim3(256);
            cudaLaunchAttribute at[1];
            at[0].id = cudaLaunchAttributeClusterDimension;
            at[0].val.clusterDim.x = G;
            at[0].val.clusterDim.y = 1;
            at[0].val.clusterDim.z = 1;
            cfg.attrs = at;
            cfg.numAttrs = 1;
            cudaLaunchKernelEx(&cfg, bench, variant, 2000, d_out, d_sink);
            cudaError_t e = cudaDeviceSynchronize();
            long long cyc = 0;
            cudaMemcpy(&cyc, d_out, 8, cudaMemcpyDeviceToHost);
            printf("G=%2d variant=%d cycles/round=%lld %s\n", G, variant, cyc, e ? cudaGetErrorString(e) : "");
        }
    }
    return 0;
}
