// dsmem.cuh — distributed-shared-memory push with mbarrier transaction counting (sm_90+ cluster
// primitives), used by the register K-SQR leaf (sketch_qr.cu) and the cluster K-LU leaf (lu.cu).
#pragma once
#include <cstdint>

namespace bqrrp {

// DSMEM push with transaction counting: st.async writes 8 bytes into a peer CTA's shared memory and
// decrements that CTA's mbarrier tx-count by 8 when the write has landed; the receiver arms its mbarrier
// with the bytes it expects per phase and waits on the phase parity (no cluster-wide barrier, no fence).
__device__ __forceinline__ unsigned smem_u32(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }
__device__ __forceinline__ unsigned mapa_u32(unsigned addr, int rank)
{
    unsigned r;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(addr), "r"(rank));
    return r;
}
__device__ __forceinline__ void st_async_f64(unsigned remote_addr, double v, unsigned remote_mbar)
{
    asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.b64 [%0], %1, [%2];"
                 ::"r"(remote_addr), "l"(__double_as_longlong(v)), "r"(remote_mbar) : "memory");
}
__device__ __forceinline__ void mbar_init(unsigned mbar, unsigned count)
{
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(mbar), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(unsigned mbar, unsigned bytes)
{
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(mbar), "r"(bytes) : "memory");
}
// acquire at CLUSTER scope: the peers' writes (st.async payloads) and everything they did before their pushes
// (e.g. their DSMEM reads of this CTA's staging buffers) happen-before what this CTA does after the wait
__device__ __forceinline__ void mbar_wait_parity(unsigned mbar, unsigned parity)
{
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "WAIT_%=:\n"
        "mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 p, [%0], %1;\n"
        "@!p bra WAIT_%=;\n"
        "}\n" ::"r"(mbar), "r"(parity) : "memory");
}

// Split cluster barrier: arrive (release) now, wait (acquire) later — a CTA that has nothing left to share can
// signal "done with my peers' memory" early and keep working (or exit) without waiting for the slowest CTA.
__device__ __forceinline__ void cluster_arrive() { asm volatile("barrier.cluster.arrive.release.aligned;" ::: "memory"); }
__device__ __forceinline__ void cluster_wait() { asm volatile("barrier.cluster.wait.acquire.aligned;" ::: "memory"); }

}  // namespace bqrrp
