// lu.cu — K-LU: partial-pivot LU of the tall w x d sketch transpose, for its pivots
// (Alg. 2 "Practical wide QRCP": GETRF on the transposed sketch).
//
// Recursive right-looking LU.  Leaves are jb-column panels factored by one kernel launch whose CTAs split
// the panel rows; per column every CTA offers its local first-max candidate (|value|, row, full panel row),
// all CTAs pick the same winner (largest |value|, lowest row index on ties: IDAMAX, reading Z19), swap and
// apply the rank-1 update to their own rows.  Three leaf kernels by active row count:
// <= 4096 rows a register-resident cluster leaf, <= one 16-CTA cluster's shared memory a shared-memory
// cluster leaf (both exchange by st.async + mbarrier pushes), larger a cooperative grid leaf (one grid
// barrier per column, exchange through L2).  An exactly-zero pivot
// column is skipped (no swap, no scaling; Z18).  Each interchange is applied at once to the whole row
// of the LU matrix (all d columns, as LAPACK's laswp on both sides would) and to the permutation
// vector perm (perm = J_qr - 1 of piv_transform), so no separate laswp pass exists and the
// touched set of the permutation is read straight off perm.
#include <cooperative_groups.h>
#include <cstdlib>

#include "blas.cuh"
#include "dsmem.cuh"
#include "bqrrp_internal.cuh"

namespace cg = cooperative_groups;

namespace bqrrp {

struct LuPanelArgs {
    double* L;
    int64_t ld;
    int64_t w;   // rows of the LU matrix
    int64_t d;   // columns of the LU matrix
    int64_t c0;  // first panel column (= first active row)
    int jb;      // panel width
    int R;       // rows per CTA
    int* ipiv;   // out: ipiv[c0 + j] = pivot row (0-based, absolute)
    int* perm;   // running row permutation (w)
    double* xbuf;  // exchange: [2][G][LU_XSTRIDE]
    double* rowj;  // exchange: [2][LU_JBMAX]
};

constexpr int LU_JBMAX = 32;
constexpr int LU_XSTRIDE = 2 + LU_JBMAX;
constexpr int LU_THREADS = 256;

__device__ __forceinline__ bool better(double v, int64_t i, double bv, int64_t bi)
{
    return v > bv || (v == bv && i < bi);
}

// After a panel: apply its jb interchanges (row c0+j <-> spiv[j], in order) to the columns outside the
// panel and to perm as ONE gather of the <= 2 jb rows they touch (independent loads, one latency round)
// instead of jb dependent swaps inside the column loop.  Called by every CTA of the panel kernel with
// its thread range [gtid, ., gstride) over the outside columns.
__device__ void apply_panel_interchanges(const LuPanelArgs& a, const int64_t* spiv, int64_t* trow, int64_t* tsrc,
                                         int* s_nt, int64_t gtid, int64_t gstride)
{
    const int jb = a.jb;
    if (threadIdx.x == 0) {
        int nt = 0;
        for (int j = 0; j < jb; ++j) {
            const int64_t jr = a.c0 + j, p = spiv[j];
            if (p == jr) continue;
            int ia = -1, ib = -1;
            for (int t = 0; t < nt; ++t) {
                if (trow[t] == jr) ia = t;
                if (trow[t] == p) ib = t;
            }
            if (ia < 0) { trow[nt] = jr; tsrc[nt] = jr; ia = nt++; }
            if (ib < 0) { trow[nt] = p; tsrc[nt] = p; ib = nt++; }
            int64_t t = tsrc[ia];
            tsrc[ia] = tsrc[ib];
            tsrc[ib] = t;
        }
        *s_nt = nt;
    }
    __syncthreads();
    const int nt = *s_nt;
    if (nt == 0) return;
    const int64_t n_out = a.d - jb;
    for (int64_t e = gtid; e < n_out; e += gstride) {
        const int64_t c = (e < a.c0) ? e : e + jb;
        double* pc = a.L + c * a.ld;
        // a gather is only safe if every source is read before any destination is written: the rows
        // are the same set, so read all of them (16 loads in flight per chunk) before writing
        double v[2 * LU_JBMAX];
        for (int t0 = 0; t0 < nt; t0 += 16) {
#pragma unroll
            for (int t = 0; t < 16; ++t)
                if (t0 + t < nt) v[t0 + t] = pc[tsrc[t0 + t]];
        }
        for (int t0 = 0; t0 < nt; t0 += 16) {
#pragma unroll
            for (int t = 0; t < 16; ++t)
                if (t0 + t < nt) pc[trow[t0 + t]] = v[t0 + t];
        }
    }
    if (gtid == 0) {
        int pv[2 * LU_JBMAX];
        for (int t = 0; t < nt; ++t) pv[t] = a.perm[tsrc[t]];
        for (int t = 0; t < nt; ++t) a.perm[trow[t]] = pv[t];
    }
}

__global__ void __launch_bounds__(LU_THREADS, 1) lu_panel_kernel(LuPanelArgs a)
{
    cg::grid_group grid = cg::this_grid();
    extern __shared__ double sp[];  // sp[c * R + r]
    __shared__ double red_v[LU_THREADS / 32];
    __shared__ int64_t red_i[LU_THREADS / 32];
    __shared__ double pivrow[LU_JBMAX], oldrow[LU_JBMAX];
    __shared__ int64_t s_piv;
    __shared__ int64_t spiv[LU_JBMAX], trow[2 * LU_JBMAX], tsrc[2 * LU_JBMAX];
    __shared__ int s_nt;

    const int G = gridDim.x, cta = blockIdx.x, tid = threadIdx.x, R = a.R, jb = a.jb;
    const int lane = tid & 31, warp = tid >> 5;
    const int64_t rbeg = a.c0 + (int64_t)cta * R;  // absolute first row of this CTA
    const int64_t rows_here = (rbeg < a.w) ? ((a.w - rbeg < R) ? a.w - rbeg : R) : 0;
    const int64_t gtid = (int64_t)cta * LU_THREADS + tid, gstride = (int64_t)G * LU_THREADS;

    slab_load_async(sp, R, a.L + rbeg + a.c0 * a.ld, a.ld, (int)rows_here, R, jb);

    for (int j = 0; j < jb; ++j) {
        const int par = j & 1;
        const int64_t jr = a.c0 + j;  // absolute row of the pivot position
        // local first-max of |L(r, j)| over active rows r >= jr
        double bv = -1.0;
        int64_t bi = INT64_MAX;
        for (int r = tid; r < rows_here; r += LU_THREADS) {
            int64_t ar = rbeg + r;
            if (ar < jr) continue;
            double v = fabs(sp[j * R + r]);
            if (v > bv) { bv = v; bi = ar; }  // ascending rows per thread: first index kept on ties
        }
        for (int o = 16; o > 0; o >>= 1) {
            double ov = __shfl_down_sync(0xffffffffu, bv, o);
            int64_t oi = __shfl_down_sync(0xffffffffu, bi, o);
            if (better(ov, oi, bv, bi)) { bv = ov; bi = oi; }
        }
        if (lane == 0) { red_v[warp] = bv; red_i[warp] = bi; }
        __syncthreads();
        if (tid == 0) {
            for (int wv = 1; wv < LU_THREADS / 32; ++wv)
                if (better(red_v[wv], red_i[wv], bv, bi)) { bv = red_v[wv]; bi = red_i[wv]; }
            double* slot = a.xbuf + ((int64_t)par * G + cta) * LU_XSTRIDE;
            slot[0] = bv;
            slot[1] = __longlong_as_double((long long)bi);
            s_piv = bi;
        }
        __syncthreads();
        if (tid < jb) {
            double* slot = a.xbuf + ((int64_t)par * G + cta) * LU_XSTRIDE;
            slot[2 + tid] = (s_piv != INT64_MAX) ? sp[tid * R + (s_piv - rbeg)] : 0.0;
            if (jr >= rbeg && jr < rbeg + rows_here) a.rowj[par * LU_JBMAX + tid] = sp[tid * R + (jr - rbeg)];
        }
        grid.sync();
        // every CTA picks the same winner: warp 0 alone reads the G candidates (lane-strided), reduces them
        // with shuffles (first-max, IDAMAX order) and fetches the winner's row and row jr — one block barrier
        // instead of three
        if (warp == 0) {
            double v = -1.0;
            int64_t i = INT64_MAX;
            int wq = 0;
            for (int q = lane; q < G; q += 32) {
                const double* slot = a.xbuf + ((int64_t)par * G + q) * LU_XSTRIDE;
                double cv = __ldcg(slot);
                int64_t ci = (int64_t)__double_as_longlong(__ldcg(slot + 1));
                if (better(cv, ci, v, i)) { v = cv; i = ci; wq = q; }
            }
            for (int o = 16; o > 0; o >>= 1) {
                double ov = __shfl_down_sync(0xffffffffu, v, o);
                int64_t oi = __shfl_down_sync(0xffffffffu, i, o);
                int ow = __shfl_down_sync(0xffffffffu, wq, o);
                if (better(ov, oi, v, i)) { v = ov; i = oi; wq = ow; }
            }
            i = __shfl_sync(0xffffffffu, i, 0);
            wq = __shfl_sync(0xffffffffu, wq, 0);
            if (lane < jb) {
                pivrow[lane] = __ldcg(a.xbuf + ((int64_t)par * G + wq) * LU_XSTRIDE + 2 + lane);
                oldrow[lane] = __ldcg(a.rowj + par * LU_JBMAX + lane);
            }
            if (lane == 0) {
                s_piv = i;
                if (cta == 0) a.ipiv[jr] = (int)i;
            }
        }
        __syncthreads();
        const int64_t piv = s_piv;
        const double u = pivrow[j];
        if (tid == 0) spiv[j] = (u != 0.0) ? piv : jr;
        if (u != 0.0) {
            if (piv != jr) {
                if (piv >= rbeg && piv < rbeg + rows_here && tid < jb) sp[tid * R + (piv - rbeg)] = oldrow[tid];
                if (jr >= rbeg && jr < rbeg + rows_here && tid < jb) sp[tid * R + (jr - rbeg)] = pivrow[tid];
            }
            __syncthreads();
            for (int r = tid; r < rows_here; r += LU_THREADS) {
                if (rbeg + r <= jr) continue;
                double l = sp[j * R + r] / u;
                sp[j * R + r] = l;
                for (int c = j + 1; c < jb; ++c) sp[c * R + r] = fma(-l, pivrow[c], sp[c * R + r]);
            }
        }
        __syncthreads();
    }
    for (int c = 0; c < jb; ++c)
        for (int r = tid; r < rows_here; r += LU_THREADS) a.L[rbeg + r + (a.c0 + c) * a.ld] = sp[c * R + r];
    __syncthreads();
    apply_panel_interchanges(a, spiv, trow, tsrc, &s_nt, gtid, gstride);
}

// ---------------------------------------------------------------------------------------------
// Cluster variant (panels that fit the shared memory of one <= 16-CTA cluster): the same algorithm with
// the exchange in distributed shared memory and one barrier.cluster per column instead of a grid
// barrier through L2.  Records are double-buffered by column parity (see the QR panel for the argument).
constexpr int LUC_CLMAX = 16;
constexpr int LUC_SLOT = 2 + LU_JBMAX;  // val, idx, candidate row

__global__ void __launch_bounds__(LU_THREADS, 1) lu_panel_cluster_kernel(LuPanelArgs a)
{
    cg::cluster_group cluster = cg::this_cluster();
    const int CL = (int)cluster.num_blocks(), me = (int)cluster.block_rank();
    extern __shared__ double dyn[];
    const int R = a.R, jb = a.jb, tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    double* sp = dyn;                       // sp[c * R + r]
    // exchange: slot[par][src] = (|value|, row, candidate row[32]) pushed by every CTA of the cluster;
    // rowj[par] = row jr pushed by its owner — all into THIS CTA's memory (st.async + mbarrier tx-count)
    double* slot = dyn + (size_t)R * jb;             // [2][CL][LUC_SLOT]
    double* rowjs = slot + 2 * (size_t)CL * LUC_SLOT;  // [2][LU_JBMAX]
    __shared__ __align__(8) unsigned long long mbar[2];
    __shared__ double red_v[LU_THREADS / 32];
    __shared__ int64_t red_i[LU_THREADS / 32];
    __shared__ double pivrow[LU_JBMAX], oldrow[LU_JBMAX];
    __shared__ int64_t s_piv;
    __shared__ int s_win;
    __shared__ int64_t spiv[LU_JBMAX], trow[2 * LU_JBMAX], tsrc[2 * LU_JBMAX];
    __shared__ int s_nt;
    const int64_t rbeg = a.c0 + (int64_t)me * R;
    const int64_t rows_here = (rbeg < a.w) ? ((a.w - rbeg < R) ? a.w - rbeg : R) : 0;
    const int64_t gtid = (int64_t)me * LU_THREADS + tid, gstride = (int64_t)CL * LU_THREADS;

    if (tid == 0) {
        mbar_init(smem_u32(&mbar[0]), 1);
        mbar_init(smem_u32(&mbar[1]), 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    slab_load_async(sp, R, a.L + rbeg + a.c0 * a.ld, a.ld, (int)rows_here, R, jb);
    cluster.sync();  // every peer's mbarriers are initialised before the first push

    // Per column: 2 block barriers and one mbarrier wait: every CTA pushes its candidate record into every
    // CTA's slot and the owner of row jr pushes that row (st.async), so after the wait each CTA picks the
    // winner from its OWN shared memory (no cluster barrier, no fence, no remote reads).  Slots are
    // double-buffered by parity: a CTA pushes column j+2 only after its column-(j+1) wait, i.e. after every
    // peer pushed column j+1, which each peer does only after reading its column-j slots.  Every thread owns
    // whole rows (r = tid + k 256); the interchange is folded into the row update.
    for (int j = 0; j < jb; ++j) {
        const int par = j & 1;
        const int64_t jr = a.c0 + j;
        const int owner = (int)((jr - a.c0) / R);
        double bv = -1.0;
        int64_t bi = INT64_MAX;
        for (int r = tid; r < rows_here; r += LU_THREADS) {
            int64_t ar = rbeg + r;
            if (ar < jr) continue;
            double v = fabs(sp[j * R + r]);
            if (v > bv) { bv = v; bi = ar; }  // ascending rows per thread: first index kept on ties
        }
        for (int o = 16; o > 0; o >>= 1) {
            double ov = __shfl_down_sync(0xffffffffu, bv, o);
            int64_t oi = __shfl_down_sync(0xffffffffu, bi, o);
            if (better(ov, oi, bv, bi)) { bv = ov; bi = oi; }
        }
        if (lane == 0) { red_v[warp] = bv; red_i[warp] = bi; }
        __syncthreads();  // (1)
        const unsigned mb = smem_u32(&mbar[par]);
        if (warp == 0) {  // this CTA's candidate: value, row and its full panel row, pushed to every CTA
            double v = (lane < LU_THREADS / 32) ? red_v[lane] : -1.0;
            int64_t i = (lane < LU_THREADS / 32) ? red_i[lane] : INT64_MAX;
            for (int o = 16; o > 0; o >>= 1) {
                double ov = __shfl_down_sync(0xffffffffu, v, o);
                int64_t oi = __shfl_down_sync(0xffffffffu, i, o);
                if (better(ov, oi, v, i)) { v = ov; i = oi; }
            }
            v = __shfl_sync(0xffffffffu, v, 0);
            i = __shfl_sync(0xffffffffu, i, 0);
            const unsigned dst = smem_u32(slot + ((size_t)par * CL + me) * LUC_SLOT);
            const double rowv = (lane < jb && i != INT64_MAX) ? sp[lane * R + (i - rbeg)] : 0.0;
            for (int rk = 0; rk < CL; ++rk) {
                const unsigned rm = mapa_u32(mb, rk), rd = mapa_u32(dst, rk);
                if (lane == 0) {
                    st_async_f64(rd, v, rm);
                    st_async_f64(rd + 8, __longlong_as_double((long long)i), rm);
                }
                if (lane < jb) st_async_f64(rd + 8 * (2 + lane), rowv, rm);
            }
        } else if (warp == 1 && me == owner && lane < jb) {  // the current row j, pushed to every CTA
            const double rv = sp[lane * R + (jr - rbeg)];
            const unsigned dst = smem_u32(rowjs + par * LU_JBMAX + lane);
            for (int rk = 0; rk < CL; ++rk) st_async_f64(mapa_u32(dst, rk), rv, mapa_u32(mb, rk));
        }
        if (tid == 0) mbar_arrive_expect_tx(mb, (unsigned)((CL * (2 + jb) + jb) * sizeof(double)));
        mbar_wait_parity(mb, (unsigned)((j >> 1) & 1));
        if (warp == 0) {  // every CTA picks the same winner, from its own copy of the records
            double v = -1.0;
            int64_t i = INT64_MAX;
            int wq = 0;
            if (lane < CL) {
                const double* pr = slot + ((size_t)par * CL + lane) * LUC_SLOT;
                v = pr[0];
                i = (int64_t)__double_as_longlong(pr[1]);
                wq = lane;
            }
            for (int o = 16; o > 0; o >>= 1) {
                double ov = __shfl_down_sync(0xffffffffu, v, o);
                int64_t oi = __shfl_down_sync(0xffffffffu, i, o);
                int ow = __shfl_down_sync(0xffffffffu, wq, o);
                if (better(ov, oi, v, i)) { v = ov; i = oi; wq = ow; }
            }
            i = __shfl_sync(0xffffffffu, i, 0);
            wq = __shfl_sync(0xffffffffu, wq, 0);
            if (lane < jb) {
                pivrow[lane] = slot[((size_t)par * CL + wq) * LUC_SLOT + 2 + lane];
                oldrow[lane] = rowjs[par * LU_JBMAX + lane];
            }
            if (lane == 0) {
                s_piv = i;
                if (me == 0) a.ipiv[jr] = (int)i;
            }
        }
        __syncthreads();  // (2)
        const int64_t piv = s_piv;
        const double u = pivrow[j];
        if (tid == 0) spiv[j] = (u != 0.0) ? piv : jr;
        if (u != 0.0) {
            for (int r = tid; r < rows_here; r += LU_THREADS) {
                const int64_t ar = rbeg + r;
                if (ar < jr) continue;
                if (ar == jr) {
                    if (piv != jr)
                        for (int c = 0; c < jb; ++c) sp[c * R + r] = pivrow[c];
                    continue;
                }
                const bool swapped = (ar == piv);
                if (swapped)
                    for (int c = 0; c < j; ++c) sp[c * R + r] = oldrow[c];
                const double l = (swapped ? oldrow[j] : sp[j * R + r]) / u;
                sp[j * R + r] = l;
                for (int c0 = j + 1; c0 < jb; c0 += 8) {  // 8 independent loads in flight, then 8 FMAs
                    double av[8], pv[8];
#pragma unroll
                    for (int uu = 0; uu < 8; ++uu)
                        if (c0 + uu < jb) {
                            av[uu] = swapped ? oldrow[c0 + uu] : sp[(c0 + uu) * R + r];
                            pv[uu] = pivrow[c0 + uu];
                        }
#pragma unroll
                    for (int uu = 0; uu < 8; ++uu)
                        if (c0 + uu < jb) sp[(c0 + uu) * R + r] = fma(-l, pv[uu], av[uu]);
                }
            }
        }
    }
    __syncthreads();
    for (int c = 0; c < jb; ++c)
        for (int r = tid; r < rows_here; r += LU_THREADS) a.L[rbeg + r + (a.c0 + c) * a.ld] = sp[c * R + r];
    cluster.sync();  // peers may still read this CTA's last records
    apply_panel_interchanges(a, spiv, trow, tsrc, &s_nt, gtid, gstride);
}

constexpr size_t LUC_SMEM_MAX = 196 * 1024;

// ---------------------------------------------------------------------------------------------
// Register-resident cluster leaf (rows <= 16 CTAs x 256 threads x RPT, RPT <= 2): each thread owns RPT rows
// of the 32-column panel in registers (no shared-memory slab traffic).  Per column: local first-max ->
// warp shuffles -> ONE block barrier -> every thread derives the CTA candidate; the warp owning it pushes
// (|value|, row, its panel row) into every CTA's slot with st.async (mbarrier tx-count), CTA 0's warp 0
// pushes row jr (rows c0 .. c0+31 are its lanes); after the mbarrier wait, warp 0 picks the winner (IDAMAX
// order, Z19) from LOCAL shared memory, one more block barrier, every thread swaps / scales / updates its
// own rows.  Slots are double-buffered by column parity (a CTA pushes column j+2 only after its column-
// (j+1) wait, i.e. after every peer pushed column j+1, which each does after its column-j reads).  (A grid
// form exchanging through global records with release/acquire tags was ~1.8x slower than the
// shared-memory grid kernel and was removed.)
__device__ __forceinline__ double select32(const double (&v)[32], int j)
{
    double l1[16], l2[8], l3[4], l4[2];
#pragma unroll
    for (int i = 0; i < 16; ++i) l1[i] = (j & 1) ? v[2 * i + 1] : v[2 * i];
#pragma unroll
    for (int i = 0; i < 8; ++i) l2[i] = (j & 2) ? l1[2 * i + 1] : l1[2 * i];
#pragma unroll
    for (int i = 0; i < 4; ++i) l3[i] = (j & 4) ? l2[2 * i + 1] : l2[2 * i];
#pragma unroll
    for (int i = 0; i < 2; ++i) l4[i] = (j & 8) ? l3[2 * i + 1] : l3[2 * i];
    return (j & 16) ? l4[1] : l4[0];
}

constexpr int LR_REC = 2 + LU_JBMAX;  // |value|, row, panel row
constexpr int LR_CLMAX = 16;

template <int RPT>
__global__ void __launch_bounds__(LU_THREADS, 1) lu_leaf_reg_kernel(LuPanelArgs a)
{
    cg::cluster_group cluster = cg::this_cluster();
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, jb = a.jb;
    const int G = (int)cluster.num_blocks(), me = (int)cluster.block_rank();
    constexpr int RC = LU_THREADS * RPT;  // rows per CTA
    const int64_t rbeg = a.c0 + (int64_t)me * RC;
    __shared__ double red_v[LU_THREADS / 32];
    __shared__ int64_t red_i[LU_THREADS / 32];
    __shared__ double pivrow[LU_JBMAX], oldrow[LU_JBMAX];
    __shared__ int64_t s_piv;
    __shared__ int64_t spiv[LU_JBMAX], trow[2 * LU_JBMAX], tsrc[2 * LU_JBMAX];
    __shared__ int s_nt;
    __shared__ double slot[2][LR_CLMAX][LR_REC];  // records pushed by every CTA of the cluster
    __shared__ double rowjs[2][LU_JBMAX];         // row jr, pushed by CTA 0
    __shared__ __align__(8) unsigned long long mbar[2];
    if (tid == 0) {
        mbar_init(smem_u32(&mbar[0]), 1);
        mbar_init(smem_u32(&mbar[1]), 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }

    double av[RPT][32];
    int64_t rr[RPT];
#pragma unroll
    for (int i = 0; i < RPT; ++i) {
        rr[i] = rbeg + tid + (int64_t)i * LU_THREADS;
        const bool ok = rr[i] < a.w;
#pragma unroll
        for (int c = 0; c < 32; ++c) av[i][c] = (ok && c < jb) ? a.L[rr[i] + (a.c0 + c) * a.ld] : 0.0;
    }
    cluster.sync();  // every peer's mbarriers are initialised before the first push

#pragma unroll 1
    for (int j = 0; j < jb; ++j) {
        const int par = j & 1;
        const int64_t jr = a.c0 + j;
        const unsigned mb = smem_u32(&mbar[par]);
        // local first-max of |L(r, j)| over my active rows (ascending rows: first index kept on ties)
        double bv = -1.0;
        int64_t bi = INT64_MAX;
        double xj[RPT];
#pragma unroll
        for (int i = 0; i < RPT; ++i) {
            xj[i] = select32(av[i], j);
            if (rr[i] < a.w && rr[i] >= jr) {
                const double v = fabs(xj[i]);
                if (v > bv) { bv = v; bi = rr[i]; }
            }
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            const double ov = __shfl_down_sync(0xffffffffu, bv, o);
            const int64_t oi = __shfl_down_sync(0xffffffffu, bi, o);
            if (better(ov, oi, bv, bi)) { bv = ov; bi = oi; }
        }
        if (lane == 0) { red_v[warp] = bv; red_i[warp] = bi; }
        __syncthreads();  // (1)
        double cv = red_v[0];
        int64_t ci = red_i[0];
#pragma unroll
        for (int wv = 1; wv < LU_THREADS / 32; ++wv)
            if (better(red_v[wv], red_i[wv], cv, ci)) { cv = red_v[wv]; ci = red_i[wv]; }
        // push this CTA's candidate: the warp owning row ci gathers it by shuffles (lane c takes entry c)
        const int owner_t = (ci == INT64_MAX) ? 0 : (int)((ci - rbeg) % LU_THREADS);
        const int owner_i = (ci == INT64_MAX) ? 0 : (int)((ci - rbeg) / LU_THREADS);
        if (warp == (owner_t >> 5)) {
            double mine = 0.0;
#pragma unroll
            for (int c = 0; c < 32; ++c) {
                double src = 0.0;
#pragma unroll
                for (int i = 0; i < RPT; ++i) src = (i == owner_i) ? av[i][c] : src;
                const double t = __shfl_sync(0xffffffffu, src, owner_t & 31);
                mine = (lane == c) ? t : mine;
            }
            if (ci == INT64_MAX) mine = 0.0;
            const unsigned dst = smem_u32(&slot[par][me][0]);
            for (int rk = 0; rk < G; ++rk) {
                const unsigned rm = mapa_u32(mb, rk), rd = mapa_u32(dst, rk);
                if (lane == 0) {
                    st_async_f64(rd, (ci == INT64_MAX) ? -1.0 : cv, rm);
                    st_async_f64(rd + 8, __longlong_as_double((long long)ci), rm);
                }
                st_async_f64(rd + 8 * (2 + lane), mine, rm);
            }
        }
        if (me == 0 && warp == 0) {  // row jr = row c0 + j = lane j's first row
            double rj = 0.0;
#pragma unroll
            for (int c = 0; c < 32; ++c) {
                const double t = __shfl_sync(0xffffffffu, av[0][c], j);
                rj = (lane == c) ? t : rj;
            }
            const unsigned dst = smem_u32(&rowjs[par][lane]);
            for (int rk = 0; rk < G; ++rk) st_async_f64(mapa_u32(dst, rk), rj, mapa_u32(mb, rk));
        }
        if (tid == 0) mbar_arrive_expect_tx(mb, (unsigned)((G * LR_REC + LU_JBMAX) * sizeof(double)));
        mbar_wait_parity(mb, (unsigned)((j >> 1) & 1));
        if (warp == 0) {  // every CTA picks the same winner from its own copy of the records
            double v = -1.0;
            int64_t idx = INT64_MAX;
            int wq = 0;
            if (lane < G) {
                v = slot[par][lane][0];
                idx = (int64_t)__double_as_longlong(slot[par][lane][1]);
                wq = lane;
            }
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) {
                const double ov = __shfl_down_sync(0xffffffffu, v, o);
                const int64_t oi = __shfl_down_sync(0xffffffffu, idx, o);
                const int ow = __shfl_down_sync(0xffffffffu, wq, o);
                if (better(ov, oi, v, idx)) { v = ov; idx = oi; wq = ow; }
            }
            idx = __shfl_sync(0xffffffffu, idx, 0);
            wq = __shfl_sync(0xffffffffu, wq, 0);
            if (lane < jb) {
                pivrow[lane] = slot[par][wq][2 + lane];
                oldrow[lane] = rowjs[par][lane];
            }
            if (lane == 0) {
                s_piv = idx;
                if (me == 0) a.ipiv[jr] = (int)idx;
            }
        }
        __syncthreads();  // (2)
        const int64_t piv = s_piv;
        const double u = pivrow[j];
        if (tid == 0) spiv[j] = (u != 0.0) ? piv : jr;
        if (u != 0.0) {  // (an exactly zero pivot column: no swap, no scaling, Z18)
#pragma unroll
            for (int i = 0; i < RPT; ++i) {
                const int64_t r = rr[i];
                if (r >= a.w || r < jr) continue;
                if (r == jr) {
                    if (piv != jr) {
#pragma unroll
                        for (int c = 0; c < 32; ++c)
                            if (c < jb) av[i][c] = pivrow[c];
                    }
                    continue;
                }
                const bool swapped = (r == piv);
                const double l = (swapped ? oldrow[j] : xj[i]) / u;
#pragma unroll
                for (int c = 0; c < 32; ++c) {
                    const double base = swapped ? oldrow[c < jb ? c : 0] : av[i][c];
                    av[i][c] = (c < j) ? base : ((c == j) ? l : fma(-l, pivrow[c < jb ? c : 0], base));
                }
            }
        }
    }
#pragma unroll
    for (int i = 0; i < RPT; ++i)
        if (rr[i] < a.w) {
#pragma unroll
            for (int c = 0; c < 32; ++c)
                if (c < jb) a.L[rr[i] + (a.c0 + c) * a.ld] = av[i][c];
        }
    cluster.sync();  // no CTA exits while peers may still push into it
    const int64_t gtid = (int64_t)me * LU_THREADS + tid, gstride = (int64_t)G * LU_THREADS;
    apply_panel_interchanges(a, spiv, trow, tsrc, &s_nt, gtid, gstride);
}

static bool lu_reg_fits(int64_t rows)
{
    // one row per thread: with two rows per thread it measured slower than the shared-memory cluster kernel
    // (8192 rows: 8.5 vs 6.5 us per column), at <= 4096 rows slightly faster (5.7-5.9 vs 5.9-6.1)
    return rows <= (int64_t)LR_CLMAX * LU_THREADS;
}

static bool lu_panel_reg(Ctx& cx, double* L, int64_t ld, int64_t w, int64_t d, int64_t c0, int jb, int* ipiv, int* perm)
{
    const int64_t rows = w - c0;
    if (!lu_reg_fits(rows) || jb > 32) return false;
    const int rpt = rows <= (int64_t)LR_CLMAX * LU_THREADS ? 1 : 2;
    const int G = (int)cdiv(rows, (int64_t)LU_THREADS * rpt);
    LuPanelArgs a{L, ld, w, d, c0, jb, LU_THREADS * rpt, ipiv, perm, nullptr, nullptr};
    static AttrOnce attr1, attr2;
    ensure_attr(attr1, lu_leaf_reg_kernel<1>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    ensure_attr(attr2, lu_leaf_reg_kernel<2>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(G);
    cfg.blockDim = dim3(LU_THREADS);
    cfg.stream = cx.stream;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = G;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    if (rpt == 1) BQ_CUDA(cudaLaunchKernelEx(&cfg, lu_leaf_reg_kernel<1>, a));
    else BQ_CUDA(cudaLaunchKernelEx(&cfg, lu_leaf_reg_kernel<2>, a));
    ++g_launches;
    return true;
}

static bool lu_cluster_fits(int64_t rows, int jb, int* CLout, int* Rout)
{
    int CL = (int)imin(LUC_CLMAX, imax(1, cdiv(rows, 512)));
    int R = (int)cdiv(rows, CL);
    auto bytes = [&](int cl, int r) { return (size_t)r * jb * 8 + ((size_t)2 * cl * LUC_SLOT + 2 * LU_JBMAX) * 8; };
    while (bytes(CL, R) > LUC_SMEM_MAX && CL < LUC_CLMAX) {
        ++CL;
        R = (int)cdiv(rows, CL);
    }
    if (bytes(CL, R) > LUC_SMEM_MAX) return false;
    *CLout = CL;
    *Rout = R;
    return true;
}

static bool lu_panel_cluster(Ctx& cx, double* L, int64_t ld, int64_t w, int64_t d, int64_t c0, int jb, int* ipiv,
                             int* perm)
{
    int CL, R;
    if (!lu_cluster_fits(w - c0, jb, &CL, &R)) return false;
    static AttrOnce attr_smem, attr_cl;
    ensure_attr(attr_smem, lu_panel_cluster_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)LUC_SMEM_MAX);
    ensure_attr(attr_cl, lu_panel_cluster_kernel, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    LuPanelArgs a{L, ld, w, d, c0, jb, R, ipiv, perm, nullptr, nullptr};
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(CL);
    cfg.blockDim = dim3(LU_THREADS);
    cfg.dynamicSmemBytes = (size_t)R * jb * 8 + ((size_t)2 * CL * LUC_SLOT + 2 * LU_JBMAX) * 8;
    cfg.stream = cx.stream;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = CL;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    BQ_CUDA(cudaLaunchKernelEx(&cfg, lu_panel_cluster_kernel, a));
    ++g_launches;
    return true;
}

struct LuExchange {  // global exchange buffers of the cooperative grid leaf
    double* xbuf;
    double* rowj;
};

static void lu_panel(Ctx& cx, double* L, int64_t ld, int64_t w, int64_t d, int64_t c0, int jb, int* ipiv, int* perm,
                     LuExchange& ex)
{
    if (lu_panel_reg(cx, L, ld, w, d, c0, jb, ipiv, perm)) return;
    double* xbuf = ex.xbuf;
    double* rowj = ex.rowj;
    if (lu_panel_cluster(cx, L, ld, w, d, c0, jb, ipiv, perm)) return;
    int64_t rows = w - c0;
    // few enough CTAs that the barrier stays cheap, enough that the slab fits shared memory
    const int gmax = cx.num_sms;
    int G = (int)imin(gmax, imax(1, cdiv(rows, 256)));
    int R = (int)cdiv(rows, G);
    if ((size_t)R * jb * sizeof(double) > 200 * 1024) {
        G = (int)imin(gmax, cdiv(rows * jb * (int64_t)sizeof(double), 200 * 1024));
        R = (int)cdiv(rows, G);
    }
    size_t smem = (size_t)R * jb * sizeof(double);
    if (smem > 200 * 1024)
        throw std::runtime_error("lu_panel: sketch transpose taller than lu_max_rows (" + std::to_string(rows) + " rows)");
    static AttrOnce attr;
    ensure_attr(attr, lu_panel_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    LuPanelArgs a{L, ld, w, d, c0, jb, R, ipiv, perm, xbuf, rowj};
    void* args[] = {&a};
    BQ_CUDA(cudaLaunchCooperativeKernel((void*)lu_panel_kernel, dim3(G), dim3(LU_THREADS), args, smem, cx.stream));
    ++g_launches;
}

static int lu_leaf_width(int64_t rows, int num_sms)
{
    if (lu_reg_fits(rows)) return 32;  // the register cluster leaf (<= 16 x 512 rows)
    // a leaf that one cluster can hold (32, else 16 columns), else the widest the grid kernel can hold
    int CL, R;
    if (lu_cluster_fits(rows, 32, &CL, &R)) return 32;
    if (lu_cluster_fits(rows, 16, &CL, &R)) return 16;
    // the cooperative grid leaf keeps a slab of cdiv(rows, num_sms) rows x leaf columns per CTA in shared
    // memory: narrower leaves for taller sketches (down to one column: 148 x 25600 rows; taller inputs are
    // rejected up front, lu_max_rows)
    const int64_t Rg = cdiv(rows, num_sms);
    for (int leaf = 32; leaf > 1; leaf /= 2)
        if (Rg * leaf * 8 <= 200 * 1024) return leaf;
    return 1;
}

int64_t lu_max_rows(int num_sms) { return (int64_t)num_sms * (200 * 1024 / 8); }

static void getrf_rec(Ctx& cx, double* L, int64_t ld, int64_t w, int64_t d, int64_t c0, int64_t c1, int* ipiv,
                      int* perm, LuExchange& ex, int leaf)
{
    int64_t nc = c1 - c0;
    if (nc <= leaf) {
        lu_panel(cx, L, ld, w, d, c0, (int)nc, ipiv, perm, ex);
        return;
    }
    int64_t mid = c0 + cdiv(nc / 2, leaf) * leaf;
    getrf_rec(cx, L, ld, w, d, c0, mid, ipiv, perm, ex, leaf);
    // (the left half's interchanges were applied to whole rows inside its panels)
    // U12 = L11^{-1} A12 ; A22 -= L21 U12
    int64_t ncr = c1 - mid;
    double* L11 = L + c0 + c0 * ld;
    double* A12 = L + c0 + mid * ld;
    trsm_left_lower_unit(cx, mid - c0, ncr, L11, ld, A12, ld);
    gemm(cx, false, false, w - mid, ncr, mid - c0, -1.0, L + mid + c0 * ld, ld, A12, ld, 1.0, L + mid + mid * ld, ld);
    getrf_rec(cx, L, ld, w, d, mid, c1, ipiv, perm, ex, leaf);
}

__global__ void iota_kernel(int64_t n, int* p)
{
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        p[i] = (int)i;
}

void getrf_pivots(Ctx& cx, double* L, int64_t ld, int64_t w, int64_t d, int* ipiv, int* perm)
{
    int64_t nlu = imin(w, d);
    iota_kernel<<<(unsigned)imin(cdiv(w, 256), 1024), 256, 0, cx.stream>>>(w, perm);
    BQ_LAUNCH_CHECK();
    if (nlu <= 0) return;
    size_t mark = cx.ws_used;
    LuExchange ex;
    ex.xbuf = cx.alloc(2 * (size_t)cx.num_sms * LU_XSTRIDE);
    ex.rowj = cx.alloc(2 * LU_JBMAX);
    int leaf = lu_leaf_width(w, cx.num_sms);
    getrf_rec(cx, L, ld, w, nlu, 0, nlu, ipiv, perm, ex, leaf);
    cx.ws_used = mark;
}

}  // namespace bqrrp
