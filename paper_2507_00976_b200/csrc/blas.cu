// blas.cu — GEMM launcher (split-K heuristic), recursive TRSM, blocked POTRF and the
// sign-choosing no-pivot LU of the Householder reconstruction.  Every O(n^3) piece is cast onto the
// DMMA GEMM engine (dgemm.cuh); the diagonal blocks (<= 64) are factored by one CTA in shared memory.
#include <cstdlib>
#include <mutex>

#include "blas.cuh"
#include "dgemm.cuh"
#include "diag_blocks.cuh"

namespace bqrrp {

// Optional GEMM trace (profiling aid): BQRRP_GEMM_TRACE=<file> records every engine call with its shape
// and CUDA-event duration; written at process exit as CSV.
namespace {
struct GemmTraceRec {
    int64_t M, N, K;
    int ta, tb, tri, nsplit;
    cudaEvent_t e0, e1;
};
struct GemmTrace {
    const char* path = std::getenv("BQRRP_GEMM_TRACE");
    std::vector<GemmTraceRec> recs;
    std::mutex mu;
    ~GemmTrace()
    {
        if (!path || recs.empty()) return;
        FILE* f = std::fopen(path, "w");
        if (!f) return;
        std::fprintf(f, "M,N,K,ta,tb,tri,nsplit,ms\n");
        for (auto& r : recs) {
            float ms = 0.f;
            cudaEventSynchronize(r.e1);
            cudaEventElapsedTime(&ms, r.e0, r.e1);
            std::fprintf(f, "%lld,%lld,%lld,%d,%d,%d,%d,%.6f\n", (long long)r.M, (long long)r.N, (long long)r.K, r.ta, r.tb,
                         r.tri, r.nsplit, ms);
        }
        std::fclose(f);
    }
};
GemmTrace g_trace;
}  // namespace

// ------------------------------------------------------------------------------------------- GEMM
template <class Cfg, bool TA, bool TB>
static void launch_gemm_t(Ctx& cx, const GemmArgs& g, dim3 grid)
{
    static AttrOnce attr;
    constexpr size_t sm = dgemm2_smem_bytes<Cfg, TA, TB>();
    ensure_attr(attr, dgemm2_kernel<Cfg, TA, TB>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    dgemm2_kernel<Cfg, TA, TB><<<grid, Cfg::THREADS, sm, cx.stream>>>(g, dgemm2_vec_ok(g));
    BQ_LAUNCH_CHECK();
}

template <class Cfg>
static void launch_gemm(Ctx& cx, bool ta, bool tb, const GemmArgs& g, int nsplit, int ctas_per_sm)
{
    int64_t tiles = cdiv(g.M, Cfg::BM) * cdiv(g.N, Cfg::BN);
    if (ctas_per_sm > 0) tiles = imin(tiles, (int64_t)ctas_per_sm * cx.num_sms);  // persistent
    dim3 grid((unsigned)tiles, 1, (unsigned)nsplit);
    if (!ta && !tb) launch_gemm_t<Cfg, false, false>(cx, g, grid);
    else if (ta && !tb) launch_gemm_t<Cfg, true, false>(cx, g, grid);
    else if (!ta && tb) launch_gemm_t<Cfg, false, true>(cx, g, grid);
    else launch_gemm_t<Cfg, true, true>(cx, g, grid);
}

// Tile choice: the big tile when it still gives >= 2 waves, then 64x64, then 64x32 (more CTAs for the
// small and skinny GEMMs of the recursions).  Split-K (fixed slices, fixed-order sum) when even the
// chosen tiling leaves the SMs idle and K is long.
void gemm(Ctx& cx, bool ta, bool tb, int64_t M, int64_t N, int64_t K, double alpha, const double* A, int64_t lda,
          const double* B, int64_t ldb, double beta, double* C, int64_t ldc, bool tri, int ctas_per_sm,
          bool no_split, const GemmExtra* extra)
{
    if (M <= 0 || N <= 0) return;
    const bool fixed = extra && (extra->fixed_tiles || extra->hs_state);
    if (fixed) {
        static_assert(Cfg2Mid::BM == GEMM_FIXED_TILE && Cfg2Mid::BN == GEMM_FIXED_TILE, "fixed tile");
        GemmArgs g{M, N, K, alpha, beta, A, lda, B, ldb, C, ldc, nullptr, K > 0 ? K : 1, tri ? 1 : 0,
                   extra->a_lower ? 1 : 0, extra->hs_state, extra->hs_readers};
        launch_gemm<Cfg2Mid>(cx, ta, tb, g, 1, 0);
        return;
    }
    // The split-K decision (the only choice that changes result bits: the tiling never changes an element's K
    // order) is taken on the decision shape Md x Nd: the real one, or the hint of a caller computing one
    // block of a larger product (the multi-GPU driver's per-rank columns), so that every
    // element gets the same K slices as in the whole product.
    const int64_t Md = (extra && extra->split_m > 0) ? extra->split_m : M;
    const int64_t Nd = (extra && extra->split_n > 0) ? extra->split_n : N;
    auto ntiles = [&](int bm, int bn) {
        int64_t tm = cdiv(Md, bm), tn = cdiv(Nd, bn);
        return tri ? (tm * tn + tm) / 2 : tm * tn;
    };
    // v2 64x64 / BK 16 / 3 stages / grouped rasterisation is the best tile on every large shape and operand
    // order (35.3-36.0 TFLOP/s, profiles/gemm_tune_r01d_v2.json); 64x32 gives more CTAs to small GEMMs.
    int cfg;  // 1 mid (64x64), 2 small (64x32)
    int bm, bn;
    if (Nd > 32 && ntiles(Cfg2Mid::BM, Cfg2Mid::BN) >= cx.num_sms) { cfg = 1; bm = Cfg2Mid::BM; bn = Cfg2Mid::BN; }
    else { cfg = 2; bm = Cfg2Small::BM; bn = Cfg2Small::BN; }
    int64_t tiles = ntiles(bm, bn);
    const size_t MNd = (size_t)(Md * Nd);
    int nsplit = 1;
    int64_t kchunk = K > 0 ? K : 1;
    if (K >= 8192 && ntiles(Cfg2Mid::BM, Cfg2Mid::BN) < cx.num_sms && cx.splitk && ctas_per_sm == 0 &&
        !no_split) {
        // few output tiles over a long K (the panel Grams of tall, narrow panels: C4's 262144 x 512, C2's
        // 16384 x 1024): 64x64 tiles split into K-chunks of >= 2048 rows, ~2 waves of 4 resident CTAs per
        // SM.  The 64x32 two-wave split below left these HBM-bound (every tile pair re-streams its K range:
        // 25.8 GB for one 262144 x 512 Gram); consecutive CTAs here share a K-chunk, read from L2.
        cfg = 1;
        bm = Cfg2Mid::BM;
        bn = Cfg2Mid::BN;
        tiles = ntiles(bm, bn);
        int64_t sp = cdiv(8 * (int64_t)cx.num_sms, tiles);
        sp = imin(sp, imin(K / 2048, (int64_t)64));
        sp = imin(sp, (int64_t)(cx.splitk_elems / MNd));
        if (sp >= 2) {
            kchunk = cdiv(cdiv(K, sp), Cfg2Mid::BK) * Cfg2Mid::BK;
            nsplit = (int)cdiv(K, kchunk);
        }
    } else if (K >= 256 && tiles < 2 * cx.num_sms && cx.splitk && ctas_per_sm == 0 && !no_split) {
        int64_t want = cdiv(2 * cx.num_sms, tiles);
        want = imin(want, 32);
        want = imin(want, K / 128);
        int64_t cap = (int64_t)(cx.splitk_elems / MNd);
        want = imin(want, cap);
        if (want >= 2) {
            kchunk = cdiv(cdiv(K, want), Cfg2Mid::BK) * Cfg2Mid::BK;
            nsplit = (int)cdiv(K, kchunk);
        }
    } else if (K >= 4096 && tiles < 8 * 4 * cx.num_sms && cx.splitk && ctas_per_sm == 0 && cfg == 1 && !no_split) {
        // a few waves of long-K tiles (the panel's Gram SYRKs, late-iteration GEMM1): pick the split whose
        // last wave is fullest (4 resident 64x64 CTAs per SM), if it beats no split by > 4 %
        const int64_t slots = 4 * (int64_t)cx.num_sms;
        auto eff = [&](int64_t sp) {
            const int64_t w = tiles * sp;
            return (double)w / (double)(cdiv(w, slots) * slots);
        };
        const int64_t cap = imin(16, imin(K / 1024, (int64_t)(cx.splitk_elems / MNd)));
        int64_t best = 1;
        double beff = eff(1);
        for (int64_t sp = 2; sp <= cap; ++sp)
            if (eff(sp) > beff + 0.04 + 0.002 * (double)sp) { best = sp; beff = eff(sp); }
        if (best >= 2) {
            kchunk = cdiv(cdiv(K, best), Cfg2Mid::BK) * Cfg2Mid::BK;
            nsplit = (int)cdiv(K, kchunk);
        }
    }
    GemmArgs g{M, N, K, alpha, beta, A, lda, B, ldb, C, ldc, nsplit > 1 ? cx.splitk : nullptr, kchunk, tri ? 1 : 0,
               (extra && extra->a_lower) ? 1 : 0, nullptr, nullptr};
    GemmTraceRec rec{};
    if (g_trace.path) {
        rec = GemmTraceRec{M, N, K, ta, tb, tri, nsplit, nullptr, nullptr};
        cudaEventCreate(&rec.e0);
        cudaEventCreate(&rec.e1);
        cudaEventRecord(rec.e0, cx.stream);
    }
    if (cfg == 1) launch_gemm<Cfg2Mid>(cx, ta, tb, g, nsplit, ctas_per_sm);
    else launch_gemm<Cfg2Small>(cx, ta, tb, g, nsplit, ctas_per_sm);
    if (nsplit > 1) {
        int64_t total = M * N;
        int blocks = (int)imin(cdiv(total, 256), 4 * cx.num_sms);
        dgemm_splitk_reduce<<<blocks, 256, 0, cx.stream>>>(M, N, nsplit, cx.splitk, alpha, beta, C, ldc, tri ? 1 : 0);
        BQ_LAUNCH_CHECK();
    }
    if (g_trace.path) {
        cudaEventRecord(rec.e1, cx.stream);
        std::lock_guard<std::mutex> lk(g_trace.mu);
        g_trace.recs.push_back(rec);
    }
}

// ------------------------------------------------------------------------------------------- TRSM
constexpr int TRSM_NB = 64;

// Base triangular solve on a 64-wide triangular dimension, tiled over the independent dimension.
// Element (t, r) of the right-hand side (t: triangular index, r: independent index) lives at
// B[t * st + r * sr].  coef(l, t) (l < t) is the coupling of unknown l into equation t and diag(t) the
// pivot:  x_t = (b_t - sum_{l<t} coef(l, t) x_l) / diag(t).
//   right side, X op(T) = B:  st = ldb, sr = 1,   coef(l, t) = op(T)(l, t), diag = op(T)(t, t)
//   left side,  L X = B:      st = 1,   sr = ldb, coef(l, t) = L(t, l),     diag = 1 (unit)
// One THREAD per independent index r: its 64 unknowns live in registers and are eliminated column by
// column (x_t = b_t / diag(t), then b_tt -= coef(t, tt) x_t for tt > t: 63 independent FMAs per step),
// the coefficients are broadcast reads from shared memory — no barrier inside the solve.  Rows are
// read / written straight from global memory when r is the contiguous axis (right side), else through a
// shared transpose.  Coefficients outside n x n are zero and 1/diag = 1 there, so ragged n needs no
// branches.
constexpr int TB_R = 128, TB_THREADS = TB_R;

// NB = the triangular size rounded up to 16 / 32 / 64: a thread's solve costs NB (NB - 1) / 2 FMAs in a chain of
// NB steps, so a 16-wide solve (the LU recursion's bottom nodes at 16-column leaves) does 120 instead of 2016.
template <int NB>
__global__ void __launch_bounds__(TB_THREADS) trsm_base_kernel(int n, int64_t nr, const double* __restrict__ T,
                                                                int64_t ldt, int mode, int unit, double* __restrict__ B,
                                                                int64_t st, int64_t sr)
{
    // mode 0: right, T stored upper (op(T) = T); mode 1: right, T stored lower (op(T) = T^T);
    // mode 2: left, T stored lower (unit)
    extern __shared__ double dsm[];
    double(*C)[NB + 1] = reinterpret_cast<double(*)[NB + 1]>(dsm);                // C[l][t] = coef(l, t)
    double* rdiag = dsm + NB * (NB + 1);                                            // 1 / diag(t)
    double(*Bs)[TB_R + 1] = reinterpret_cast<double(*)[TB_R + 1]>(rdiag + NB);    // Bs[t][r] (sr != 1)
    const int tid = threadIdx.x;
    for (int idx = tid; idx < NB * NB; idx += TB_THREADS) {
        const int l = idx % NB, t = idx / NB;
        double v = 0.0;
        if (l < t && t < n) {
            if (mode == 0) v = T[l + (int64_t)t * ldt];
            else v = T[t + (int64_t)l * ldt];  // mode 1: op(T)(l, t) = T(t, l); mode 2: L(t, l)
        }
        C[l][t] = v;
    }
    if (tid < NB) rdiag[tid] = (unit || tid >= n) ? 1.0 : 1.0 / T[tid + (int64_t)tid * ldt];
    const int64_t r0 = (int64_t)blockIdx.x * TB_R;
    const int nloc = (int)((nr - r0 < TB_R) ? nr - r0 : TB_R);
    double x[NB];
    if (sr != 1) {  // left side: stage the n x TB_R tile through shared memory (coalesced along t)
        for (int idx = tid; idx < NB * TB_R; idx += TB_THREADS) {
            const int t = idx % NB, r = idx / NB;
            Bs[t][r] = (t < n && r < nloc) ? B[t + (r0 + r) * sr] : 0.0;
        }
    }
    __syncthreads();
    const bool mine = tid < nloc;
    if (sr == 1) {
#pragma unroll
        for (int t = 0; t < NB; ++t) x[t] = (mine && t < n) ? B[t * st + (r0 + tid)] : 0.0;
    } else {
#pragma unroll
        for (int t = 0; t < NB; ++t) x[t] = Bs[t][tid];
    }
#pragma unroll
    for (int t = 0; t < NB; ++t) {
        x[t] *= rdiag[t];
#pragma unroll
        for (int tt = t + 1; tt < NB; ++tt) x[tt] = fma(-x[t], C[t][tt], x[tt]);
    }
    if (sr == 1) {
        if (mine) {
#pragma unroll
            for (int t = 0; t < NB; ++t)
                if (t < n) B[t * st + (r0 + tid)] = x[t];
        }
    } else {
#pragma unroll
        for (int t = 0; t < NB; ++t) Bs[t][tid] = x[t];
        __syncthreads();
        for (int idx = tid; idx < NB * TB_R; idx += TB_THREADS) {
            const int t = idx % NB, r = idx / NB;
            if (t < n && r < nloc) B[t + (r0 + r) * sr] = Bs[t][r];
        }
    }
}

template <int NB>
static void trsm_base_launch(Ctx& cx, int n, int64_t nr, const double* T, int64_t ldt, int mode, int unit, double* B,
                             int64_t st, int64_t sr)
{
    const size_t smem = sizeof(double) * (NB * (NB + 1) + NB + (sr != 1 ? NB * (TB_R + 1) : 0));
    static AttrOnce attr;
    ensure_attr(attr, trsm_base_kernel<NB>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                (int)(sizeof(double) * (NB * (NB + 1) + NB + NB * (TB_R + 1))));
    trsm_base_kernel<NB><<<(unsigned)cdiv(nr, TB_R), TB_THREADS, smem, cx.stream>>>(n, nr, T, ldt, mode, unit, B, st, sr);
    BQ_LAUNCH_CHECK();
}

// The 32- and 64-wide solves split every right-hand side over a quad of threads: thread q of the quad owns the
// unknowns t = 4 i + q (interleaved, so every step keeps all four busy), the owner of x_t scales it and a
// shuffle broadcasts it to the quad, which updates its own later unknowns — a chain of NB steps of ~NB/8 FMAs
// each instead of one thread's NB (NB - 1) / 2 (measured: the single-thread 64-wide solve took ~22 us).
constexpr int TQ_THREADS = 128, TQ_R = TQ_THREADS / 4;

template <int NB>
__global__ void __launch_bounds__(TQ_THREADS) trsm_quad_kernel(int n, int64_t nr, const double* __restrict__ T,
                                                                int64_t ldt, int mode, int unit, double* __restrict__ B,
                                                                int64_t st, int64_t sr)
{
    constexpr int NI = NB / 4;
    __shared__ double C[NB][NB + 1];  // C[l][t] = coef(l, t)
    __shared__ double rdiag[NB];
    const int tid = threadIdx.x, lane = tid & 31, q = tid & 3;
    for (int idx = tid; idx < NB * NB; idx += TQ_THREADS) {
        const int l = idx % NB, t = idx / NB;
        double v = 0.0;
        if (l < t && t < n) {
            if (mode == 0) v = T[l + (int64_t)t * ldt];
            else v = T[t + (int64_t)l * ldt];  // mode 1: op(T)(l, t) = T(t, l); mode 2: L(t, l)
        }
        C[l][t] = v;
    }
    if (tid < NB) rdiag[tid] = (unit || tid >= n) ? 1.0 : 1.0 / T[tid + (int64_t)tid * ldt];
    const int64_t r = (int64_t)blockIdx.x * TQ_R + (tid >> 2);
    const bool mine = r < nr;
    double x[NI];
#pragma unroll
    for (int i = 0; i < NI; ++i) {
        const int t = 4 * i + q;
        x[i] = (mine && t < n) ? B[t * st + r * sr] : 0.0;
    }
    __syncthreads();
    const int base = lane & ~3;
#pragma unroll
    for (int t = 0; t < NB; ++t) {
        const int qo = t & 3, io = t >> 2;
        if (q == qo) x[io] *= rdiag[t];
        const double xt = __shfl_sync(0xffffffffu, x[io], base | qo);
        if (q > qo) x[io] = fma(-xt, C[t][4 * io + q], x[io]);
#pragma unroll
        for (int i = io + 1; i < NI; ++i) x[i] = fma(-xt, C[t][4 * i + q], x[i]);
    }
    if (mine) {
#pragma unroll
        for (int i = 0; i < NI; ++i) {
            const int t = 4 * i + q;
            if (t < n) B[t * st + r * sr] = x[i];
        }
    }
}

static void trsm_base(Ctx& cx, int n, int64_t nr, const double* T, int64_t ldt, int mode, int unit, double* B,
                      int64_t st, int64_t sr)
{
    if (n <= 16) {
        trsm_base_launch<16>(cx, n, nr, T, ldt, mode, unit, B, st, sr);
        return;
    }
    const unsigned grid = (unsigned)cdiv(nr, TQ_R);
    if (n <= 32) trsm_quad_kernel<32><<<grid, TQ_THREADS, 0, cx.stream>>>(n, nr, T, ldt, mode, unit, B, st, sr);
    else trsm_quad_kernel<64><<<grid, TQ_THREADS, 0, cx.stream>>>(n, nr, T, ldt, mode, unit, B, st, sr);
    BQ_LAUNCH_CHECK();
}

// ---- inverse-based base case (well-conditioned triangles only: CholQR / reconstruction factors)
// The 64-wide diagonal blocks of op(T) are inverted once per TRSM call (one CTA per block, all blocks in
// parallel); each base case is then X = B * inv(D), a 64-row x 64 x 64 DMMA product per CTA, in place,
// with no per-unknown barrier.  Error ~ kappa(D) u per element (vs backward-stable substitution), hence
// only used where op(T) is known to be well conditioned.

// Dinv (64 x 64 per block, ld 64, zero-padded) = inv(op(T)(b0:b0+64, b0:b0+64)), op(T) upper.
// Thread group (4 lanes) per column j of the inverse: back substitution x_i = (e_ij - sum U_il x_l) / U_ii,
// i = j .. 0, the sum split over the 4 lanes and combined by shuffles.
__global__ void __launch_bounds__(256) tri_inv_diag_kernel(int n, const double* __restrict__ T, int64_t ldt, int mode,
                                                           int unit, double* __restrict__ Dinv)
{
    extern __shared__ double ism[];
    double(*U)[TRSM_NB + 1] = reinterpret_cast<double(*)[TRSM_NB + 1]>(ism);
    double(*X)[TRSM_NB + 1] = reinterpret_cast<double(*)[TRSM_NB + 1]>(ism + TRSM_NB * (TRSM_NB + 1));
    const int tid = threadIdx.x;
    const int b0 = blockIdx.x * TRSM_NB, bn = (n - b0 < TRSM_NB) ? n - b0 : TRSM_NB;
    const double* Tb = T + b0 + (int64_t)b0 * ldt;
    for (int idx = tid; idx < TRSM_NB * TRSM_NB; idx += 256) {
        int l = idx % TRSM_NB, t = idx / TRSM_NB;
        double v = 0.0;
        if (l < bn && t < bn && l <= t) {
            v = (mode == 0) ? Tb[l + (int64_t)t * ldt] : Tb[t + (int64_t)l * ldt];
            if (unit && l == t) v = 1.0;
        }
        U[l][t] = v;
        X[l][t] = 0.0;
    }
    __syncthreads();
    const int j = tid >> 2, q = tid & 3;
    const bool col = j < bn;
    for (int i = TRSM_NB - 1; i >= 0; --i) {
        double part = 0.0;
        if (col && i <= j)
            for (int l = i + 1 + q; l <= j; l += 4) part = fma(U[i][l], X[l][j], part);
        part += __shfl_xor_sync(0xffffffffu, part, 1);
        part += __shfl_xor_sync(0xffffffffu, part, 2);
        if (col && q == 0 && i <= j) X[i][j] = ((i == j ? 1.0 : 0.0) - part) / U[i][i];
        __syncwarp();
    }
    __syncthreads();
    double* D = Dinv + (int64_t)blockIdx.x * TRSM_NB * TRSM_NB;
    for (int idx = tid; idx < TRSM_NB * TRSM_NB; idx += 256) D[idx] = X[idx % TRSM_NB][idx / TRSM_NB];
}

constexpr size_t TINV_SMEM = sizeof(double) * 2 * TRSM_NB * (TRSM_NB + 1);
constexpr int TI_LD = TRSM_NB + 4;  // 4 mod 16 doubles: conflict-free DMMA fragment loads
constexpr size_t TI_SMEM = sizeof(double) * 2 * TRSM_NB * TI_LD;

// B(r0:r0+64, 0:n) <- B(r0:r0+64, 0:n) * Dinv (n <= 64), in place; 4 warps, each 32 x 32 (4 x 4 DMMA tiles).
__global__ void __launch_bounds__(128) trsm_inv_apply_kernel(int n, int64_t nr, const double* __restrict__ Dinv,
                                                             double* B, int64_t ldb)
{
    extern __shared__ __align__(16) double tsm[];
    double* sB = tsm;                   // [k][r]
    double* sD = tsm + TRSM_NB * TI_LD;  // [t][k]
    const int tid = threadIdx.x;
    const int64_t r0 = (int64_t)blockIdx.x * TRSM_NB;
    for (int idx = tid; idx < TRSM_NB * TRSM_NB; idx += 128) {
        int r = idx % TRSM_NB, k = idx / TRSM_NB;
        bool ok = (k < n) && (r0 + r < nr);
        cp_async8z(&sB[k * TI_LD + r], ok ? B + (r0 + r) + (int64_t)k * ldb : B, ok);
        cp_async8z(&sD[k * TI_LD + r], Dinv + idx, true);  // Dinv[r + k*64] = D(r, k): sD[t = k][k' = r]
    }
    cp_async_wait_all();
    __syncthreads();
    const int lane = tid & 31, warp = tid >> 5, wm = warp & 1, wn = warp >> 1, gid = lane >> 2, tig = lane & 3;
    double acc[4][4][2];
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int jj = 0; jj < 4; ++jj) acc[i][jj][0] = acc[i][jj][1] = 0.0;
    const int kn = (n + 3) & ~3;
    for (int kk = 0; kk < kn; kk += 4) {
        double af[4], bf[4];
#pragma unroll
        for (int i = 0; i < 4; ++i) af[i] = sB[(kk + tig) * TI_LD + wm * 32 + i * 8 + gid];
#pragma unroll
        for (int jj = 0; jj < 4; ++jj) bf[jj] = sD[(wn * 32 + jj * 8 + gid) * TI_LD + kk + tig];
#pragma unroll
        for (int i = 0; i < 4; ++i)
#pragma unroll
            for (int jj = 0; jj < 4; ++jj) dmma_884(acc[i][jj][0], acc[i][jj][1], af[i], bf[jj]);
    }
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int jj = 0; jj < 4; ++jj)
#pragma unroll
            for (int h = 0; h < 2; ++h) {
                int64_t r = r0 + wm * 32 + i * 8 + gid;
                int c = wn * 32 + jj * 8 + 2 * tig + h;
                if (r < nr && c < n) B[r + (int64_t)c * ldb] = acc[i][jj][h];
            }
}

constexpr int64_t TRSM_INV_MIN_ROWS = 4096;

static void trsm_ru_rec(Ctx& cx, int64_t rows, int64_t n, const double* T, int64_t ldt, bool t_lower, bool unit,
                        double* B, int64_t ldb, const double* Dinv)
{
    if (n <= TRSM_NB) {
        if (Dinv) {
            trsm_inv_apply_kernel<<<(unsigned)cdiv(rows, TRSM_NB), 128, TI_SMEM, cx.stream>>>((int)n, rows, Dinv, B,
                                                                                               ldb);
            BQ_LAUNCH_CHECK();
        } else {
            trsm_base(cx, (int)n, rows, T, ldt, t_lower ? 1 : 0, unit ? 1 : 0, B, ldb, 1);
        }
        return;
    }
    int64_t n1 = cdiv(n / 2, TRSM_NB) * TRSM_NB;
    int64_t n2 = n - n1;
    trsm_ru_rec(cx, rows, n1, T, ldt, t_lower, unit, B, ldb, Dinv);
    if (!t_lower)  // op(T)(0:n1, n1:n) = T(0:n1, n1:n)
        gemm(cx, false, false, rows, n2, n1, -1.0, B, ldb, T + n1 * ldt, ldt, 1.0, B + n1 * ldb, ldb);
    else  // op(T)(0:n1, n1:n) = T(n1:n, 0:n1)^T
        gemm(cx, false, true, rows, n2, n1, -1.0, B, ldb, T + n1, ldt, 1.0, B + n1 * ldb, ldb);
    trsm_ru_rec(cx, rows, n2, T + n1 + n1 * ldt, ldt, t_lower, unit, B + n1 * ldb, ldb,
                Dinv ? Dinv + (n1 / TRSM_NB) * TRSM_NB * TRSM_NB : nullptr);
}

void trsm_right_upper(Ctx& cx, int64_t rows, int64_t n, const double* T, int64_t ldt, bool t_lower, bool unit,
                      double* B, int64_t ldb, bool well_conditioned)
{
    if (rows <= 0 || n <= 0) return;
    // the inversion launch pays off only when the apply kernels are wide (tall B: the CholQR passes and Y2)
    if (!well_conditioned || rows < TRSM_INV_MIN_ROWS) {
        trsm_ru_rec(cx, rows, n, T, ldt, t_lower, unit, B, ldb, nullptr);
        return;
    }
    static AttrOnce attr_apply, attr_inv;
    ensure_attr(attr_apply, trsm_inv_apply_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)TI_SMEM);
    ensure_attr(attr_inv, tri_inv_diag_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)TINV_SMEM);
    const size_t mark = cx.ws_used;
    const int64_t nblk = cdiv(n, TRSM_NB);
    double* Dinv = cx.alloc((size_t)nblk * TRSM_NB * TRSM_NB);
    tri_inv_diag_kernel<<<(unsigned)nblk, 256, TINV_SMEM, cx.stream>>>((int)n, T, ldt, t_lower ? 1 : 0, unit ? 1 : 0, Dinv);
    BQ_LAUNCH_CHECK();
    trsm_ru_rec(cx, rows, n, T, ldt, t_lower, unit, B, ldb, Dinv);
    cx.ws_used = mark;
}

void trsm_left_lower_unit(Ctx& cx, int64_t n, int64_t cols, const double* L, int64_t ldl, double* B, int64_t ldb)
{
    if (n <= 0 || cols <= 0) return;
    if (n <= TRSM_NB) {
        trsm_base(cx, (int)n, cols, L, ldl, 2, 1, B, 1, ldb);
        return;
    }
    int64_t n1 = cdiv(n / 2, TRSM_NB) * TRSM_NB;
    int64_t n2 = n - n1;
    trsm_left_lower_unit(cx, n1, cols, L, ldl, B, ldb);
    gemm(cx, false, false, n2, cols, n1, -1.0, L + n1, ldl, B, ldb, 1.0, B + n1, ldb);
    trsm_left_lower_unit(cx, n2, cols, L + n1 + n1 * ldl, ldl, B + n1, ldb);
}

// ------------------------------------------------------------------------------------------- POTRF

__global__ void __launch_bounds__(256) potrf_diag(int n, double* G, int64_t ldg, int j0, int* info)
{
    __shared__ double colj[2][FACT_NB];
    __shared__ double piv[FACT_NB];
    potrf_diag_block(n, G, ldg, j0, info, colj, piv);
}

void potrf_lower(Ctx& cx, int64_t n, double* G, int64_t ldg)
{
    for (int64_t j0 = 0; j0 < n; j0 += FACT_NB) {
        int64_t jb = imin(FACT_NB, n - j0);
        double* Gjj = G + j0 + j0 * ldg;
        potrf_diag<<<1, 256, 0, cx.stream>>>((int)jb, Gjj, ldg, (int)j0, cx.flags + F_POTRF_INFO);
        BQ_LAUNCH_CHECK();
        int64_t rest = n - j0 - jb;
        if (rest > 0) {
            double* G21 = Gjj + jb;
            trsm_right_upper(cx, rest, jb, Gjj, ldg, /*t_lower=*/true, /*unit=*/false, G21, ldg, true);
            gemm(cx, false, true, rest, rest, jb, -1.0, G21, ldg, G21, ldg, 1.0, G21 + jb * ldg, ldg, /*tri=*/true);
        }
    }
    zero_triangle(cx, 'L', n, n, G, ldg);
}

// ------------------------------------------------------------------------------------------- sign LU
__global__ void __launch_bounds__(256) getrf_sign_diag(int n, double* Qm, int64_t ldq, double* S)
{
    __shared__ double colj[2][FACT_NB], rowj[2][FACT_NB];
    __shared__ double piv[FACT_NB];
    getrf_sign_diag_block(n, Qm, ldq, S, colj, rowj, piv);
}

void getrf_nopiv_sign(Ctx& cx, int64_t n, double* Q, int64_t ldq, double* S)
{
    for (int64_t j0 = 0; j0 < n; j0 += FACT_NB) {
        int64_t jb = imin(FACT_NB, n - j0);
        double* Qjj = Q + j0 + j0 * ldq;
        getrf_sign_diag<<<1, 256, 0, cx.stream>>>((int)jb, Qjj, ldq, S + j0);
        BQ_LAUNCH_CHECK();
        int64_t rest = n - j0 - jb;
        if (rest > 0) {
            // U12 = L11^{-1} A12 ; L21 = A21 U11^{-1} ; A22 -= L21 U12
            trsm_left_lower_unit(cx, jb, rest, Qjj, ldq, Qjj + jb * ldq, ldq);
            trsm_right_upper(cx, rest, jb, Qjj, ldq, false, false, Qjj + jb, ldq, true);
            gemm(cx, false, false, rest, rest, jb, -1.0, Qjj + jb, ldq, Qjj + jb * ldq, ldq, 1.0, Qjj + jb + jb * ldq,
                 ldq);
        }
    }
}

// ------------------------------------------------------------------------------------------- misc
__global__ void copy_kernel(int64_t rows, int64_t cols, const double* __restrict__ s, int64_t lds, double* __restrict__ d,
                            int64_t ldd)
{
    int64_t total = rows * cols;
    for (int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; idx < total; idx += (int64_t)gridDim.x * blockDim.x) {
        int64_t r = idx % rows, c = idx / rows;
        d[r + c * ldd] = s[r + c * lds];
    }
}

void copy_matrix(Ctx& cx, int64_t rows, int64_t cols, const double* src, int64_t lds, double* dst, int64_t ldd)
{
    if (rows <= 0 || cols <= 0) return;
    BQ_CUDA(cudaMemcpy2DAsync(dst, ldd * sizeof(double), src, lds * sizeof(double), rows * sizeof(double), cols,
                              cudaMemcpyDeviceToDevice, cx.stream));
}

__global__ void transpose_kernel(int64_t rows, int64_t cols, const double* __restrict__ s, int64_t lds,
                                 double* __restrict__ d, int64_t ldd)
{
    __shared__ double t[32][33];
    int64_t r0 = (int64_t)blockIdx.x * 32, c0 = (int64_t)blockIdx.y * 32;
    for (int k = threadIdx.y; k < 32; k += blockDim.y) {
        int64_t r = r0 + threadIdx.x, c = c0 + k;
        if (r < rows && c < cols) t[k][threadIdx.x] = s[r + c * lds];
    }
    __syncthreads();
    for (int k = threadIdx.y; k < 32; k += blockDim.y) {
        int64_t c = c0 + threadIdx.x, r = r0 + k;  // dst(c, r) = src(r, c)
        if (r < rows && c < cols) d[c + r * ldd] = t[threadIdx.x][k];
    }
}

void transpose_copy(Ctx& cx, int64_t rows, int64_t cols, const double* src, int64_t lds, double* dst, int64_t ldd)
{
    if (rows <= 0 || cols <= 0) return;
    dim3 grid((unsigned)cdiv(rows, 32), (unsigned)cdiv(cols, 32));
    transpose_kernel<<<grid, dim3(32, 8), 0, cx.stream>>>(rows, cols, src, lds, dst, ldd);
    BQ_LAUNCH_CHECK();
}

__global__ void zero_kernel(int64_t rows, int64_t cols, double* A, int64_t lda)
{
    int64_t total = rows * cols;
    for (int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; idx < total; idx += (int64_t)gridDim.x * blockDim.x)
        A[idx % rows + (idx / rows) * lda] = 0.0;
}

void set_zero(Ctx& cx, int64_t rows, int64_t cols, double* A, int64_t lda)
{
    if (rows <= 0 || cols <= 0) return;
    if (lda == rows) {
        BQ_CUDA(cudaMemsetAsync(A, 0, rows * cols * sizeof(double), cx.stream));
        return;
    }
    zero_kernel<<<(unsigned)imin(cdiv(rows * cols, 256), 8 * cx.num_sms), 256, 0, cx.stream>>>(rows, cols, A, lda);
    BQ_LAUNCH_CHECK();
}

__global__ void zero_tri_kernel(int keep_lower, int64_t n, int64_t cols, double* A, int64_t lda, int unit)
{
    int64_t total = n * cols;
    for (int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; idx < total; idx += (int64_t)gridDim.x * blockDim.x) {
        int64_t i = idx % n, j = idx / n;
        if (keep_lower ? (i < j) : (i > j)) A[i + j * lda] = 0.0;
        else if (unit && i == j) A[i + j * lda] = 1.0;
    }
}

void zero_triangle(Ctx& cx, char keep, int64_t n, int64_t cols, double* A, int64_t lda, bool unit_diag)
{
    if (n <= 0 || cols <= 0) return;
    zero_tri_kernel<<<(unsigned)imin(cdiv(n * cols, 256), 8 * cx.num_sms), 256, 0, cx.stream>>>(
        keep == 'L', n, cols, A, lda, unit_diag ? 1 : 0);
    BQ_LAUNCH_CHECK();
}

}  // namespace bqrrp
