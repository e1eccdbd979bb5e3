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

// Per-phase clock64 stamps of the register leaf (experiments only: compiled in with -DBQRRP_LEAF_TIMING into a
// separate library, never in the product build; tools/leaf_timing.py reads them).
#ifdef BQRRP_LEAF_TIMING
__device__ long long g_leaf_ts[2][64][8];
#define LEAF_TS(j, k)                                                                            \
    do {                                                                                         \
        if (threadIdx.x == 0 && (blockIdx.x == 0 || blockIdx.x == gridDim.x - 1) && (j) < 64)     \
            g_leaf_ts[blockIdx.x == 0 ? 0 : 1][(j)][(k)] = clock64();                            \
    } while (0)
#else
#define LEAF_TS(j, k) \
    do {              \
    } while (0)
#endif

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
    // register leaf only: the columns [mc0, mc1) its row moves are applied to (mc1 < 0: all d), and an optional
    // record of the moves (mvout[0] = count, mvout[1 + t] = source row, mvout[1 + 2 LU_JBMAX + t] = destination)
    // for the lookahead LU's deferred row interchanges (getrf_pivots_la)
    int64_t mc0 = 0, mc1 = -1;
    int* mvout = nullptr;
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
// Register-resident cluster leaf: G <= 16 CTAs of one cluster, each thread owns RPT rows of
// the JB-column leaf panel in registers.
//  * Rows are never interchanged: every row carries its logical position pos (initially its own index); the
//    step-j interchange of rows jr = c0 + j and piv only swaps their labels (nobody needs row jr's values).
//  * The register window ROTATES: at step j a row's registers hold its columns j .. JB-1 in av[0 ..], so every
//    register index is compile-time in a rolled loop (no select trees; a fully unrolled loop overflows the
//    32 KB instruction cache).  The columns that leave the window are final and go straight to global memory
//    at the row's PHYSICAL index: an active row's multiplier L(r, j) at step j, the pivot row's U part when it
//    wins; at the end the moved rows (pos != own index, <= 2 JB of them) are moved to their logical positions
//    in all d columns at once.
// Per column:
//   1. thread candidate over its active rows (pos >= jr): key = bits of |x| (monotone for x >= 0), ties to the
//      smaller logical position — exactly IDAMAX's first-index rule in the swapped order (Z19);
//   2. warp argmax with three redux.sync (max of the high key word, max of the low word among those, min
//      position among those);
//   3. each warp's winner stores its row into shared memory, one block barrier;
//   4. warp 0 reduces the 8 warp records the same way and pushes the CTA record (|x| bits, pos, row) into
//      every CTA's slot with st.async (mbarrier tx-count), slots double-buffered by column parity;
//   5. after the mbarrier wait every warp picks the cluster winner from its own shared memory, relabels, and
//      — lookahead — forms column j+1 of its rows and starts its exchange (the winner stores its row with the
//      step-j update applied) BEFORE the full rank-1 update / rotation of step j, which then overlaps it.
// Division by the pivot as DGETF2 and the oracle; an exactly zero pivot column changes nothing (Z18).
constexpr int LF_NT = 256, LF_NW = LF_NT / 32, LF_GMAX = 16;

__device__ __forceinline__ void argmax3(unsigned hi, unsigned lo, unsigned p, unsigned& mh, unsigned& ml, unsigned& mp)
{
    mh = __reduce_max_sync(0xffffffffu, hi);
    ml = __reduce_max_sync(0xffffffffu, hi == mh ? lo : 0u);
    mp = __reduce_min_sync(0xffffffffu, (hi == mh && lo == ml) ? p : 0xffffffffu);
}

// Rows src -> dst of the listed moves (nmv <= 2 LU_JBMAX) in all d columns and in perm.  A warp owns whole columns
// (four at a time), lane t the moves t and t + 32: every source of a column is loaded (8 loads in flight per lane)
// before the warp barrier, every destination stored after it.  (Round-2 form: the earlier thread-per-column loop
// kept 8 loads in flight per THREAD and spent ~47k cycles per leaf at d = 1024; tools/leaf_timing.py.)
__device__ void apply_moves_all(double* L, int64_t ld, int64_t cb, int64_t ce, int* perm, int nmv, const int* mv_src,
                                const int* mv_dst, int64_t gwarp, int64_t nwarps, int lane)
{
    if (nmv == 0) return;
    const bool h0 = lane < nmv, h1 = lane + 32 < nmv;
    const int s0 = h0 ? mv_src[lane] : 0, d0 = h0 ? mv_dst[lane] : 0;
    const int s1 = h1 ? mv_src[lane + 32] : 0, d1 = h1 ? mv_dst[lane + 32] : 0;
    constexpr int CB = 4;
    for (int64_t c0 = cb + gwarp * CB; c0 < ce; c0 += nwarps * CB) {
        double v0[CB], v1[CB];
#pragma unroll
        for (int q = 0; q < CB; ++q) {
            const double* pc = L + (c0 + q) * ld;
            const bool ok = c0 + q < ce;
            v0[q] = (ok && h0) ? pc[s0] : 0.0;
            v1[q] = (ok && h1) ? pc[s1] : 0.0;
        }
        __syncwarp();
#pragma unroll
        for (int q = 0; q < CB; ++q) {
            double* pc = L + (c0 + q) * ld;
            if (c0 + q < ce) {
                if (h0) pc[d0] = v0[q];
                if (h1) pc[d1] = v1[q];
            }
        }
    }
    if (perm && gwarp == 0) {
        const int p0 = h0 ? perm[s0] : 0, p1 = h1 ? perm[s1] : 0;
        __syncwarp();
        if (h0) perm[d0] = p0;
        if (h1) perm[d1] = p1;
    }
}

// The recorded row moves of one register leaf (LuPanelArgs::mvout) applied to columns [cb, ce) (warp per column).
__global__ void lu_laswp_kernel(double* L, int64_t ld, int64_t cb, int64_t ce, const int* __restrict__ mv)
{
    const int nmv = mv[0];
    const int lane = threadIdx.x & 31;
    apply_moves_all(L, ld, cb, ce, nullptr, nmv, mv + 1, mv + 1 + 2 * LU_JBMAX,
                    (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5), (int64_t)gridDim.x * (blockDim.x >> 5),
                    lane);
}

template <int JB, int RPT>
__global__ void __launch_bounds__(LF_NT, 1) lu_leaf_fast_kernel(LuPanelArgs a)
{
    LEAF_TS(63, 0);
    cg::cluster_group cluster = cg::this_cluster();
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, jb = a.jb;
    const int G = (int)cluster.num_blocks(), me = (int)cluster.block_rank();
    constexpr int RC = LF_NT * RPT;  // rows per CTA
    const int64_t rbeg = a.c0 + (int64_t)me * RC;
    __shared__ __align__(16) double wrow[2][LF_NW][JB];
    __shared__ unsigned long long wkey[2][LF_NW];
    __shared__ unsigned wpos[2][LF_NW];
    __shared__ __align__(16) double rec[2][LF_GMAX][2 + JB];  // pushed CTA records: |x| bits, pos, row
    __shared__ __align__(8) unsigned long long mbar[2];
    __shared__ int mv_src[2 * LU_JBMAX], mv_dst[2 * LU_JBMAX], lmv_src[2 * LU_JBMAX], lmv_dst[2 * LU_JBMAX];
    __shared__ int mv_cnt, lmv_cnt;
    if (tid == 0) {
        mbar_init(smem_u32(&mbar[0]), 1);
        mbar_init(smem_u32(&mbar[1]), 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        lmv_cnt = 0;
    }
    for (int idx = tid; idx < 2 * LF_GMAX * (2 + JB); idx += LF_NT) (&rec[0][0][0])[idx] = 0.0;  // stale slots finite
    double av[RPT][JB];
    int pos[RPT];
    int64_t rr[RPT];
#pragma unroll
    for (int i = 0; i < RPT; ++i) {
        rr[i] = rbeg + tid + (int64_t)i * LF_NT;
        const bool ok = rr[i] < a.w;
        pos[i] = ok ? (int)rr[i] : -1;  // -1: padding row, never active
#pragma unroll
        for (int c = 0; c < JB; ++c) av[i][c] = (ok && c < jb) ? a.L[rr[i] + (a.c0 + c) * a.ld] : 0.0;
    }
    cluster.sync();  // every peer's mbarriers are initialised before the first push
    LEAF_TS(63, 1);

    // Column j's candidate / record exchange (steps 1-4).  xc[i] = column j of my row i; the warp winner stores
    // its row with the pending step-(j-1) update (multiplier lw[i], pivot row pr, relative to column j-1) applied
    // and rotated: w[c] = av[c+1] - l pr[c] (columns j + c).
    auto push_column = [&](int j, const double (&xc)[RPT], const double (&lw)[RPT], const double (&pr)[JB]) {
        const int par = j & 1;
        const int jr = (int)a.c0 + j;
        unsigned hi = 0u, lo = 0u, bp = 0xffffffffu;
        int bi = 0;
#pragma unroll
        for (int i = 0; i < RPT; ++i) {
            if (pos[i] >= jr) {
                const unsigned long long k = (unsigned long long)__double_as_longlong(fabs(xc[i]));
                const unsigned h = (unsigned)(k >> 32), l = (unsigned)k;
                if (h > hi || (h == hi && (l > lo || (l == lo && (unsigned)pos[i] < bp)))) {
                    hi = h;
                    lo = l;
                    bp = (unsigned)pos[i];
                    bi = i;
                }
            }
        }
        unsigned mh, ml, mp;
        argmax3(hi, lo, bp, mh, ml, mp);
        if (lane == 0) {
            wkey[par][warp] = ((unsigned long long)mh << 32) | ml;
            wpos[par][warp] = mp;
        }
        if (bp == mp && mp != 0xffffffffu) {
#pragma unroll
            for (int i = 0; i < RPT; ++i)
                if (bi == i) {
                    const double li = lw[i];
                    if (j == 0) {
#pragma unroll
                        for (int c = 0; c < JB; c += 2)
                            *reinterpret_cast<double2*>(&wrow[par][warp][c]) = make_double2(av[i][c], av[i][c + 1]);
                    } else {
#pragma unroll
                        for (int c = 0; c < JB; c += 2)
                            *reinterpret_cast<double2*>(&wrow[par][warp][c]) = make_double2(
                                fma(-li, pr[c], av[i][c + 1]), c + 2 < JB ? fma(-li, pr[c + 1], av[i][c + 2]) : 0.0);
                    }
                }
        }
        __syncthreads();
        LEAF_TS(j - 1, 4);
        const unsigned mb = smem_u32(&mbar[par]);
        if (warp == 0) {
            const unsigned long long k = (lane < LF_NW) ? wkey[par][lane] : 0ull;
            const unsigned p = (lane < LF_NW) ? wpos[par][lane] : 0xffffffffu;
            unsigned ch, cl, cp;
            argmax3((unsigned)(k >> 32), (unsigned)k, p, ch, cl, cp);
            const unsigned who = __ballot_sync(0xffffffffu, lane < LF_NW && p == cp && (unsigned)(k >> 32) == ch &&
                                                                (unsigned)k == cl);
            const int wq = who ? __ffs(who) - 1 : 0;
            // the CTA record (|x| bits, pos, row: columns j + c at c) into every CTA's slot, 16-byte st.async, the
            // G x NCH chunks spread over the warp's lanes (one instruction moves 512 bytes)
            const int NCH = 1 + (JB - j + 1) / 2;  // header + the live columns j .. JB-1 (stale beyond: never used)
            const float rnch = 1.0f / (float)NCH;  // idx / NCH by a float reciprocal (exact for idx < 2^12)
            const unsigned dst = smem_u32(&rec[par][me][0]);
            for (int idx = lane; idx < G * NCH; idx += 32) {
                const int rk = (int)(((float)idx + 0.5f) * rnch), e = idx - rk * NCH;
                double v0, v1;
                if (e == 0) {
                    v0 = __longlong_as_double((long long)(((unsigned long long)ch << 32) | cl));
                    v1 = __longlong_as_double((long long)cp);
                } else {
                    const double2 t = *reinterpret_cast<const double2*>(&wrow[par][wq][2 * e - 2]);
                    v0 = t.x;
                    v1 = t.y;
                }
                asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.v2.f64 [%0], {%1, %2}, [%3];" ::"r"(
                                 mapa_u32(dst + 16 * e, rk)),
                             "d"(v0), "d"(v1), "r"(mapa_u32(mb, rk))
                             : "memory");
            }
        }
        LEAF_TS(j - 1, 5);
        if (tid == 0) mbar_arrive_expect_tx(mb, (unsigned)(G * (1 + (JB - j + 1) / 2) * 2 * sizeof(double)));
    };

    double xc[RPT], lm[RPT], pr[JB], u_pull = 0.0;
#pragma unroll
    for (int i = 0; i < RPT; ++i) {
        xc[i] = av[i][0];
        lm[i] = 0.0;
    }
#pragma unroll
    for (int c = 0; c < JB; ++c) pr[c] = 0.0;
    push_column(0, xc, lm, pr);

#pragma unroll 1
    for (int j = 0; j < jb; ++j) {
        const int par = j & 1;
        const int jr = (int)a.c0 + j;
        LEAF_TS(j, 0);
        mbar_wait_parity(smem_u32(&mbar[par]), (unsigned)((j >> 1) & 1));
        LEAF_TS(j, 1);
        // 5. the cluster winner (every warp, from the pushed records in its own shared memory)
        const unsigned long long k = (lane < G) ? (unsigned long long)__double_as_longlong(rec[par][lane][0]) : 0ull;
        const unsigned p = (lane < G) ? (unsigned)__double_as_longlong(rec[par][lane][1]) : 0xffffffffu;
        unsigned gh, gl, gp;
        argmax3((unsigned)(k >> 32), (unsigned)k, p, gh, gl, gp);
        const unsigned who = __ballot_sync(0xffffffffu, lane < G && p == gp && (unsigned)(k >> 32) == gh &&
                                                            (unsigned)k == gl);
        const int q = __ffs(who) - 1;
        const int ps = (int)gp;
        if (tid == 0 && me == 0) a.ipiv[jr] = ps;
        LEAF_TS(j, 2);
        const double* prow = &rec[par][q][2];  // pivot row, columns j + c at c
        u_pull = prow[0];
#pragma unroll
        for (int c = 0; c + 1 < JB; ++c) pr[c] = prow[c + 1];
        pr[JB - 1] = 0.0;
        const double u = u_pull;
        int was[RPT];  // 0: inactive, 1: pivot row of step j, 2: active (updated)
        double lq[RPT];
#pragma unroll
        for (int i = 0; i < RPT; ++i) {
            const int pn = (pos[i] == jr) ? ps : ((pos[i] == ps) ? jr : pos[i]);
            was[i] = (pn == jr) ? 1 : ((pn > jr) ? 2 : 0);
            pos[i] = pn;
            lq[i] = (was[i] == 2 && u != 0.0) ? xc[i] / u : xc[i];  // L(r, j) (unscaled on an exactly zero column)
            lm[i] = (was[i] == 2 && u != 0.0) ? lq[i] : 0.0;         // the update's multiplier (0: rotate only)
        }
        LEAF_TS(j, 3);
        // lookahead: column j + 1 of my rows, its exchange started now
        if (j + 1 < jb) {
#pragma unroll
            for (int i = 0; i < RPT; ++i) xc[i] = fma(-lm[i], pr[0], av[i][1]);
            push_column(j + 1, xc, lm, pr);
        }
        LEAF_TS(j, 6);
        // the columns that leave the window (overlapping the exchange): L(r, j) of active rows, the pivot row's U
#pragma unroll
        for (int i = 0; i < RPT; ++i) {
            if (was[i] == 2) {
                a.L[rr[i] + (int64_t)jr * a.ld] = lq[i];
            } else if (was[i] == 1) {
#pragma unroll
                for (int c = 0; c < JB; ++c)
                    if (c < jb - j) a.L[rr[i] + (a.c0 + j + c) * a.ld] = av[i][c];
            }
        }
        // the step-j update with the rotation (overlaps the exchange of column j + 1)
#pragma unroll
        for (int i = 0; i < RPT; ++i) {
#pragma unroll
            for (int c = 0; c + 1 < JB; ++c) av[i][c] = fma(-lm[i], pr[c], av[i][c + 1]);
            av[i][JB - 1] = 0.0;
        }
        LEAF_TS(j, 7);
    }
    LEAF_TS(63, 2);
    // the moved rows: each CTA lists its own (shared memory), every CTA gathers all lists in rank order after one
    // cluster barrier (remote reads), then the cluster moves them in all d columns
#pragma unroll
    for (int i = 0; i < RPT; ++i) {
        if (pos[i] >= 0 && pos[i] != (int)rr[i]) {
            const int t = atomicAdd(&lmv_cnt, 1);
            lmv_src[t] = (int)rr[i];
            lmv_dst[t] = pos[i];
        }
    }
    __threadfence();  // the panel's global writes before the other CTAs move rows
    cluster.sync();   // every CTA's list complete
    if (warp == 0) {  // lane rk reads rank rk's count, a warp scan places the lists in rank order, lane rk copies its own
        const int n = lane < G ? *cluster.map_shared_rank(&lmv_cnt, lane) : 0;
        int off = n;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int y = __shfl_up_sync(0xffffffffu, off, o);
            if (lane >= o) off += y;
        }
        if (lane == 31) mv_cnt = off;
        off -= n;
        if (n > 0) {
            const int* rs = cluster.map_shared_rank(lmv_src, lane);
            const int* rd = cluster.map_shared_rank(lmv_dst, lane);
            for (int t = 0; t < n; ++t) {
                mv_src[off + t] = rs[t];
                mv_dst[off + t] = rd[t];
            }
        }
    }
    __syncthreads();
    cluster_arrive();  // done reading the peers' lists: they may exit once every CTA has arrived here
    LEAF_TS(63, 4);
    if (a.mvout && me == 0) {
        for (int t = tid; t < mv_cnt; t += LF_NT) {
            a.mvout[1 + t] = mv_src[t];
            a.mvout[1 + 2 * LU_JBMAX + t] = mv_dst[t];
        }
        if (tid == 0) a.mvout[0] = mv_cnt;
    }
    apply_moves_all(a.L, a.ld, a.mc0, a.mc1 < 0 ? a.d : a.mc1, a.perm, mv_cnt, mv_src, mv_dst,
                    (int64_t)me * LF_NW + warp, (int64_t)G * LF_NW, lane);
    LEAF_TS(63, 3);
    cluster_wait();
}

// Register leaf capacity: JB = 32 with one or two rows per thread (<= 4096 / 8192 rows), JB = 16 with four
// (<= 16384 rows).
static bool lu_reg_fits(int64_t rows, int jb)
{
    return rows <= (int64_t)LF_GMAX * LF_NT * (jb <= 16 ? 4 : 2);
}

template <int JB, int RPT>
static void launch_lu_leaf_fast(Ctx& cx, const LuPanelArgs& a, int G)
{
    static AttrOnce attr;
    ensure_attr(attr, lu_leaf_fast_kernel<JB, RPT>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(G);
    cfg.blockDim = dim3(LF_NT);
    cfg.stream = cx.stream;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = G;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    BQ_CUDA(cudaLaunchKernelEx(&cfg, lu_leaf_fast_kernel<JB, RPT>, a));
    ++g_launches;
}

static bool lu_panel_reg(Ctx& cx, double* L, int64_t ld, int64_t w, int64_t d, int64_t c0, int jb, int* ipiv, int* perm,
                         int64_t mc0 = 0, int64_t mc1 = -1, int* mvout = nullptr)
{
    const int64_t rows = w - c0;
    if (jb > 32 || !lu_reg_fits(rows, jb)) return false;
    // rows per thread: the smallest that keeps the cluster at <= cx.lu_gpref CTAs (16 by default; 8 lets a cluster of
    // full-SM CTAs find room in the SM groups the bulk GEMM leaves free, DESIGN.md §7.5 — measured neutral), else 16
    const int rmax = jb <= 16 ? 4 : 2;
    int rpt = 0;
    for (int gcap : {cx.lu_gpref, LF_GMAX}) {
        for (int r = 1; r <= rmax && !rpt; r *= 2)
            if (rows <= (int64_t)gcap * LF_NT * r) rpt = r;
        if (rpt) break;
    }
    if (!rpt) return false;
    // at least 2 CTAs: the DSMEM pushes need a real cluster (compute-sanitizer memcheck rejects st.async in a 1-CTA
    // cluster); a CTA without rows offers no candidate
    const int G = (int)imax(2, cdiv(rows, (int64_t)LF_NT * rpt));
    LuPanelArgs a{L, ld, w, d, c0, jb, LF_NT * rpt, ipiv, perm, nullptr, nullptr};
    a.mc0 = mc0;
    a.mc1 = mc1;
    a.mvout = mvout;
    if (jb > 16) {
        if (rpt == 1) launch_lu_leaf_fast<32, 1>(cx, a, G);
        else launch_lu_leaf_fast<32, 2>(cx, a, G);
    } else {
        if (rpt == 1) launch_lu_leaf_fast<16, 1>(cx, a, G);
        else if (rpt == 2) launch_lu_leaf_fast<16, 2>(cx, a, G);
        else launch_lu_leaf_fast<16, 4>(cx, a, G);
    }
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
    const int gmax = cx.lu_grid_max > 0 ? (int)imin(cx.lu_grid_max, cx.num_sms) : cx.num_sms;
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
    if (lu_reg_fits(rows, 32)) return 32;  // the register cluster leaf, 32 columns (<= 16 x 512 rows)
    if (lu_reg_fits(rows, 16)) return 16;  // the register cluster leaf, 16 columns (<= 16 x 1024 rows)
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
                      int* perm, LuExchange& ex, int leaf, const LeafDone* on_leaf)
{
    int64_t nc = c1 - c0;
    if (nc <= leaf) {
        lu_panel(cx, L, ld, w, d, c0, (int)nc, ipiv, perm, ex);
        if (on_leaf) (*on_leaf)(c1);  // perm[0:c1) is final now (later leaves only move rows >= c1)
        return;
    }
    int64_t mid = c0 + cdiv(nc / 2, leaf) * leaf;
    getrf_rec(cx, L, ld, w, d, c0, mid, ipiv, perm, ex, leaf, on_leaf);
    // (the left half's interchanges were applied to whole rows inside its panels)
    // U12 = L11^{-1} A12 ; A22 -= L21 U12
    int64_t ncr = c1 - mid;
    double* L11 = L + c0 + c0 * ld;
    double* A12 = L + c0 + mid * ld;
    trsm_left_lower_unit(cx, mid - c0, ncr, L11, ld, A12, ld);
    gemm(cx, false, false, w - mid, ncr, mid - c0, -1.0, L + mid + c0 * ld, ld, A12, ld, 1.0, L + mid + mid * ld, ld);
    getrf_rec(cx, L, ld, w, d, mid, c1, ipiv, perm, ex, leaf, on_leaf);
}

__global__ void iota_kernel(int64_t n, int* p)
{
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        p[i] = (int)i;
}

void getrf_pivots(Ctx& cx, double* L, int64_t ld, int64_t w, int64_t d, int* ipiv, int* perm, const LeafDone* on_leaf)
{
    int64_t nlu = imin(w, d);
    iota_kernel<<<(unsigned)imin(cdiv(w, 256), 1024), 256, 0, cx.stream>>>(w, perm);
    BQ_LAUNCH_CHECK();
    if (nlu <= 0) return;
    size_t mark = cx.ws_used;
    LuExchange ex;
    ex.xbuf = cx.alloc(2 * (size_t)cx.num_sms * LU_XSTRIDE);
    ex.rowj = cx.alloc(2 * LU_JBMAX);
    int leaf = lu_leaf_width(w, cx.lu_grid_max > 0 ? (int)imin(cx.lu_grid_max, cx.num_sms) : cx.num_sms);
    getrf_rec(cx, L, ld, w, nlu, 0, nlu, ipiv, perm, ex, leaf, on_leaf);
    cx.ws_used = mark;
}

// Right-looking blocked LU with a one-block lookahead, for sketch transposes the register leaf
// holds (w <= 16384).  Only the pivots are used downstream, so factors left of the current block are never
// permuted again.  Step c (leaf block B = [c, c + jb)):
//   crit: leaf(B) — its row moves applied to B only, recorded (mvout);
//   lu2:  the rest R = [c + jb + jb1, nlu): moves of B, U = L_BB^{-1} A(B, R), A(c+jb:w, R) -= L(c+jb:w, B) U;
//   crit: the next block N = [c + jb, c + jb + jb1) likewise (after lu2 finished step c - jb, which covered N),
//         then leaf(N) — so each leaf waits only for one narrow update while lu2 does the wide one.
// Returns false (nothing queued) when the leaf would not be the register leaf.
bool getrf_pivots_la(Ctx& cx, Ctx& lu2, std::vector<cudaEvent_t>& evpool, double* L, int64_t ld, int64_t w, int64_t d,
                     int* ipiv, int* perm, const LeafDone* on_leaf)
{
    const int64_t nlu = imin(w, d);
    const int leaf = lu_leaf_width(w, cx.num_sms);
    if (nlu <= 0 || !lu_reg_fits(w, leaf)) return false;
    iota_kernel<<<(unsigned)imin(cdiv(w, 256), 1024), 256, 0, cx.stream>>>(w, perm);
    BQ_LAUNCH_CHECK();
    const size_t mark = cx.ws_used;
    const int64_t nsteps = cdiv(nlu, leaf);
    const int MVS = 1 + 4 * LU_JBMAX;
    int* mv = cx.alloc_as<int>((size_t)nsteps * MVS);
    size_t nev = 0;
    auto ev = [&]() {
        if (nev == evpool.size()) {
            cudaEvent_t e;
            BQ_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
            evpool.push_back(e);
        }
        return evpool[nev++];
    };
    auto laswp = [&](Ctx& c, int64_t cb, int64_t ce, const int* m) {
        if (ce <= cb) return;
        const int64_t warps = cdiv(ce - cb, 4);
        lu_laswp_kernel<<<(unsigned)imin(cdiv(warps, 8), 4 * (int64_t)c.num_sms), 256, 0, c.stream>>>(L, ld, cb, ce, m);
        BQ_LAUNCH_CHECK();
    };
    // update of columns [cb, ce) by step (c, jb): interchanges, U rows, trailing rows
    auto update = [&](Ctx& c2, int64_t c, int jb, const int* m, int64_t cb, int64_t ce) {
        if (ce <= cb) return;
        laswp(c2, cb, ce, m);
        trsm_left_lower_unit(c2, jb, ce - cb, L + c + c * ld, ld, L + c + cb * ld, ld);
        gemm(c2, false, false, w - c - jb, ce - cb, jb, -1.0, L + (c + jb) + c * ld, ld, L + c + cb * ld, ld, 1.0,
             L + (c + jb) + cb * ld, ld, false, 0, /*no_split=*/true);
    };
    cudaEvent_t ev_lu2_prev = nullptr;  // lu2 finished the previous step's rest update
    for (int64_t step = 0; step < nsteps; ++step) {
        const int64_t c = step * leaf;
        const int jb = (int)imin(leaf, nlu - c);
        int* m = mv + step * MVS;
        if (!lu_panel_reg(cx, L, ld, w, nlu, c, jb, ipiv, perm, c, c + jb, m))
            throw std::runtime_error("getrf_pivots_la: register leaf does not fit");
        if (on_leaf) (*on_leaf)(c + jb);
        const int64_t n0 = c + jb, n1 = imin(nlu, n0 + leaf);  // the next block [n0, n1), the rest [n1, nlu)
        if (n0 >= nlu) break;
        cudaEvent_t e_leaf = ev();
        BQ_CUDA(cudaEventRecord(e_leaf, cx.stream));
        BQ_CUDA(cudaStreamWaitEvent(lu2.stream, e_leaf, 0));
        update(lu2, c, jb, m, n1, nlu);
        if (ev_lu2_prev) BQ_CUDA(cudaStreamWaitEvent(cx.stream, ev_lu2_prev, 0));  // [n0, n1) had step c - leaf's update
        update(cx, c, jb, m, n0, n1);
        ev_lu2_prev = ev();
        BQ_CUDA(cudaEventRecord(ev_lu2_prev, lu2.stream));
    }
    if (ev_lu2_prev) BQ_CUDA(cudaStreamWaitEvent(cx.stream, ev_lu2_prev, 0));
    cx.ws_used = mark;
    return true;
}

}  // namespace bqrrp

#ifdef BQRRP_LEAF_TIMING
extern "C" int bqrrp_debug_leaf_timing(long long* out)
{
    return cudaMemcpyFromSymbol(out, bqrrp::g_leaf_ts, sizeof(long long) * 2 * 64 * 8) == cudaSuccess ? 0 : -1;
}
#endif
