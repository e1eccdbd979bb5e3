// dist.cu — bqrrp_factor_dist: BQRRP over G GPUs, one process per GPU.
//
// A is distributed 1-D block-cyclically over column POSITIONS (block width nb = dist_nb, default b; position p
// lives on rank (p / nb) mod G), so every panel lives on one rank and a pivoted column moves to the rank that
// owns the position it is assigned.  The transposed sketch MskT (n x d), J and tau are replicated.  Per
// iteration (Alg. 1):
//   a2  every rank runs the same pivot selection on the replicated sketch (LU, touched set, d x d sketch QR,
//       tri_rank: identical inputs, deterministic kernels -> identical pivots); the R_sk(:, d:w) rows are
//       computed for this rank's own positions only (the sketch rows are refreshed by X1 after a6)
//   a3  X3: the <= 2 min(d, w) touched columns move source -> destination: owners gather them, one
//       all-to-all-v carries the cross-rank ones, local moves stay local
//   a4  the owner of the panel factors it (bitwise the one-GPU panel) and X2 broadcasts V, T, tau; or
//       (dist_flags & BQRRP_DIST_SHARD_PANEL) the panel's ROWS are scattered over min(G, h/k) ranks, each
//       preconditions / Grams / solves its rows, the k x k Cholesky and reconstruction factors are replicated
//       from all-reduced Grams, V's rows are all-gathered
//   a5  every rank updates its own trailing columns: GEMM1 + TRMM + R12 rows on the critical stream, the bulk
//       rows on a low-priority stream that overlaps a6 and the next a2 (as on one GPU)
//   a6  the sample update of this rank's own sketch rows, then X1: one all-gather of every rank's updated rows
// NCCL (or, for tests, a caller-supplied transport) only moves buffers; every arithmetic step is one of this
// library's kernels.  Pin: with the owner panel the result is BITWISE the one-GPU factorization: every
// per-column / per-row GEMM takes its split-K decision on the global shape (GemmExtra::split_m/n), the panel
// and its k x k finish run exactly as on one GPU, and the replicated decisions see identical inputs.
#include <dlfcn.h>
#include <nccl.h>

#include <algorithm>
#include <cstring>
#include <memory>
#include <mutex>
#include <numeric>
#include <string>
#include <vector>

#include "../../include/bqrrp.h"
#include "blas.cuh"
#include "bqrrp_internal.cuh"

namespace bqrrp {

// ------------------------------------------------------------------------------------------ NCCL, dlopen'ed
// The process's libnccl.so.2 (normally the one torch already loaded), else the system / wheel copy: the
// library itself has no link-time NCCL dependency.
struct NcclApi {
    decltype(&ncclGetUniqueId) getUniqueId = nullptr;
    decltype(&ncclCommInitRank) commInitRank = nullptr;
    decltype(&ncclCommDestroy) commDestroy = nullptr;
    decltype(&ncclAllReduce) allReduce = nullptr;
    decltype(&ncclAllGather) allGather = nullptr;
    decltype(&ncclBroadcast) broadcast = nullptr;
    decltype(&ncclSend) send = nullptr;
    decltype(&ncclRecv) recv = nullptr;
    decltype(&ncclGroupStart) groupStart = nullptr;
    decltype(&ncclGroupEnd) groupEnd = nullptr;
    decltype(&ncclGetErrorString) errorString = nullptr;
};

static NcclApi& nccl()
{
    static NcclApi api;
    static bool tried = false;
    static std::string why;
    static std::mutex mu;
    std::lock_guard<std::mutex> lk(mu);
    if (!tried) {
        tried = true;
        void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);
        const char* paths[] = {"libnccl.so.2", "/usr/lib/x86_64-linux-gnu/libnccl.so.2"};
        for (const char* p : paths)
            if (!h) h = dlopen(p, RTLD_NOW | RTLD_GLOBAL);
        if (!h) {
            why = std::string("libnccl.so.2 not loadable: ") + dlerror();
        } else {
#define BQ_SYM(f, s) api.f = reinterpret_cast<decltype(api.f)>(dlsym(h, s))
            BQ_SYM(getUniqueId, "ncclGetUniqueId");
            BQ_SYM(commInitRank, "ncclCommInitRank");
            BQ_SYM(commDestroy, "ncclCommDestroy");
            BQ_SYM(allReduce, "ncclAllReduce");
            BQ_SYM(allGather, "ncclAllGather");
            BQ_SYM(broadcast, "ncclBroadcast");
            BQ_SYM(send, "ncclSend");
            BQ_SYM(recv, "ncclRecv");
            BQ_SYM(groupStart, "ncclGroupStart");
            BQ_SYM(groupEnd, "ncclGroupEnd");
            BQ_SYM(errorString, "ncclGetErrorString");
#undef BQ_SYM
            if (!api.commInitRank || !api.allReduce || !api.send || !api.groupEnd) why = "libnccl.so.2 lacks symbols";
        }
    }
    if (!why.empty()) throw NcclError(why);
    return api;
}

#define BQ_NCCL(x)                                                                                              \
    do {                                                                                                        \
        ncclResult_t r_ = (x);                                                                                  \
        if (r_ != ncclSuccess)                                                                                  \
            throw NcclError(std::string(#x) + ": " + (nccl().errorString ? nccl().errorString(r_) : "?"));      \
    } while (0)

// ------------------------------------------------------------------------------------------ transports
struct Comm {
    int rank = 0, size = 1;
    virtual ~Comm() {}
    virtual void allreduce_sum(double* buf, size_t count, cudaStream_t st) = 0;
    // recv = size blocks of `bytes`, rank order
    virtual void allgather(const void* send, void* recv, size_t bytes, cudaStream_t st) = 0;
    virtual void broadcast(void* buf, size_t bytes, int root, cudaStream_t st) = 0;
    // per-peer byte counts and displacements (size entries each)
    virtual void alltoallv(const char* send, const size_t* scount, const size_t* sdispl, char* recv,
                           const size_t* rcount, const size_t* rdispl, cudaStream_t st) = 0;
};

struct NcclComm : Comm {
    ncclComm_t c = nullptr;
    ~NcclComm() override
    {
        if (c) nccl().commDestroy(c);
    }
    void allreduce_sum(double* buf, size_t count, cudaStream_t st) override
    {
        if (count) BQ_NCCL(nccl().allReduce(buf, buf, count, ncclFloat64, ncclSum, c, st));
    }
    void allgather(const void* send, void* recv, size_t bytes, cudaStream_t st) override
    {
        if (bytes) BQ_NCCL(nccl().allGather(send, recv, bytes, ncclUint8, c, st));
    }
    void broadcast(void* buf, size_t bytes, int root, cudaStream_t st) override
    {
        if (bytes) BQ_NCCL(nccl().broadcast(buf, buf, bytes, ncclUint8, root, c, st));
    }
    void alltoallv(const char* send, const size_t* scount, const size_t* sdispl, char* recv, const size_t* rcount,
                   const size_t* rdispl, cudaStream_t st) override
    {
        BQ_NCCL(nccl().groupStart());
        for (int p = 0; p < size; ++p) {
            if (p == rank) continue;
            if (scount[p]) BQ_NCCL(nccl().send(send + sdispl[p], scount[p], ncclUint8, p, c, st));
            if (rcount[p]) BQ_NCCL(nccl().recv(recv + rdispl[p], rcount[p], ncclUint8, p, c, st));
        }
        BQ_NCCL(nccl().groupEnd());
    }
};

// Caller-supplied transport (tests: torch.distributed over gloo).  The stream is synchronised before each
// call; the callee moves the bytes synchronously.
struct CallbackComm : Comm {
    bqrrp_transport t;
    void check(int rc, const char* what)
    {
        if (rc != 0) throw NcclError(std::string("transport ") + what + " failed (" + std::to_string(rc) + ")");
    }
    void allreduce_sum(double* buf, size_t count, cudaStream_t st) override
    {
        BQ_CUDA(cudaStreamSynchronize(st));
        if (count) check(t.allreduce_sum_f64(t.ctx, buf, count, st), "allreduce");
    }
    void allgather(const void* send, void* recv, size_t bytes, cudaStream_t st) override
    {
        BQ_CUDA(cudaStreamSynchronize(st));
        if (bytes) check(t.allgather(t.ctx, send, recv, bytes, st), "allgather");
    }
    void broadcast(void* buf, size_t bytes, int root, cudaStream_t st) override
    {
        BQ_CUDA(cudaStreamSynchronize(st));
        if (bytes) check(t.broadcast(t.ctx, buf, bytes, root, st), "broadcast");
    }
    void alltoallv(const char* send, const size_t* scount, const size_t* sdispl, char* recv, const size_t* rcount,
                   const size_t* rdispl, cudaStream_t st) override
    {
        BQ_CUDA(cudaStreamSynchronize(st));
        check(t.alltoallv(t.ctx, send, scount, sdispl, recv, rcount, rdispl, st), "alltoallv");
    }
};

// ------------------------------------------------------------------------------------------ block-cyclic map
struct BlockCyclic {
    int64_t n = 0, nb = 1;
    int G = 1;
    int owner(int64_t p) const { return (int)((p / nb) % G); }
    // index of position p among its owner's positions
    int64_t loc(int64_t p) const { return (p / (nb * G)) * nb + p % nb; }
    // number of rank r's positions < p
    int64_t count_below(int r, int64_t p) const
    {
        const int64_t cyc = nb * G, full = p / cyc, rem = p - full * cyc;
        return full * nb + imin(nb, imax(0, rem - (int64_t)r * nb));
    }
    int64_t n_loc(int r) const { return count_below(r, n); }
};

// X3 plan for one rank: the touched slots sorted by destination position; every rank derives the same order.
struct ExchangePlan {
    std::vector<int> send_idx, recv_idx, local_src, local_dst;  // local column indices
    std::vector<int64_t> send_cnt, recv_cnt;                     // columns per peer
};

static void plan_exchange(const BlockCyclic& bc, int me, int64_t nt, const int64_t* q, const int64_t* p, ExchangePlan& P)
{
    std::vector<int64_t> order(nt);
    std::iota(order.begin(), order.end(), 0);
    std::sort(order.begin(), order.end(), [&](int64_t a, int64_t b) { return q[a] < q[b]; });
    P.send_idx.clear();
    P.recv_idx.clear();
    P.local_src.clear();
    P.local_dst.clear();
    P.send_cnt.assign(bc.G, 0);
    P.recv_cnt.assign(bc.G, 0);
    std::vector<std::vector<int>> sends(bc.G), recvs(bc.G);
    for (int64_t t : order) {
        const int so = bc.owner(p[t]), dso = bc.owner(q[t]);
        if (so == me && dso == me) {
            P.local_src.push_back((int)bc.loc(p[t]));
            P.local_dst.push_back((int)bc.loc(q[t]));
        } else if (so == me) {
            sends[dso].push_back((int)bc.loc(p[t]));
        } else if (dso == me) {
            recvs[so].push_back((int)bc.loc(q[t]));
        }
    }
    for (int r = 0; r < bc.G; ++r) {
        P.send_cnt[r] = (int64_t)sends[r].size();
        P.recv_cnt[r] = (int64_t)recvs[r].size();
        P.send_idx.insert(P.send_idx.end(), sends[r].begin(), sends[r].end());
        P.recv_idx.insert(P.recv_idx.end(), recvs[r].begin(), recvs[r].end());
    }
}

// ------------------------------------------------------------------------------------------ kernels
// X(:, idx[t]) = src(:, t), t < nidx
__global__ void scatter_idx_kernel(int64_t rows, double* __restrict__ X, int64_t ldx, const int* __restrict__ idx,
                                   const double* __restrict__ src, int64_t lds)
{
    const int t = blockIdx.y;
    double* d = X + (int64_t)idx[t] * ldx;
    const double* s = src + (int64_t)t * lds;
    for (int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; r < rows; r += (int64_t)gridDim.x * blockDim.x)
        d[r] = s[r];
}

// MskT(p, :) = G(owner(p) block, loc(p), :) for positions p in [p0, n) whose owner != me; the gathered buffer
// holds, per rank, nmax rows (ld nmax) of that rank's positions >= p0 in order, d columns each.
__global__ void unpack_rows_kernel(int64_t n, int64_t p0, int64_t d, int64_t nb, int G, int me, const double* __restrict__ Gb,
                                   int64_t nmax, const int64_t* __restrict__ base, double* __restrict__ MskT, int64_t ldm)
{
    const int64_t rows = n - p0, total = rows * d;
    for (int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; idx < total; idx += (int64_t)gridDim.x * blockDim.x) {
        const int64_t pp = idx % rows, c = idx / rows, p = p0 + pp;
        const int r = (int)((p / nb) % G);
        if (r == me) continue;
        const int64_t li = (p / (nb * G)) * nb + p % nb - base[r];  // index among r's positions >= p0
        MskT[p + c * ldm] = Gb[(int64_t)r * nmax * d + li + c * nmax];
    }
}

// buf(li, :) = MskT(p, :) for this rank's positions p >= p0 (li = index among them)
__global__ void pack_rows_kernel(int64_t n, int64_t p0, int64_t d, int64_t nb, int G, int me, const double* __restrict__ MskT,
                                 int64_t ldm, int64_t base, double* __restrict__ buf, int64_t ldb)
{
    const int64_t rows = n - p0, total = rows * d;
    for (int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; idx < total; idx += (int64_t)gridDim.x * blockDim.x) {
        const int64_t pp = idx % rows, c = idx / rows, p = p0 + pp;
        if ((int)((p / nb) % G) != me) continue;
        buf[(p / (nb * G)) * nb + p % nb - base + c * ldb] = MskT[p + c * ldm];
    }
}

// {zero column, POTRF breakdown, non-finite} as doubles, summed over ranks by one all-reduce
__global__ void flags_to_f64_kernel(const int* flags, double* out)
{
    if (threadIdx.x == 0) {
        out[0] = flags[F_ZERO_COL];
        out[1] = flags[F_POTRF_INFO] ? 1.0 : 0.0;
        out[2] = flags[F_NONFINITE] ? 1.0 : 0.0;
    }
}

// ------------------------------------------------------------------------------------------ the driver
struct DistBufs {
    double *MskT, *Lb, *rowscr, *Rsk11, *X, *R11, *ref, *V, *Tp, *W, *W2, *xbuf, *rbuf, *dfl, *rowsbuf, *rowsgat;
    double *Q, *Gr1, *Gr2, *Wr, *Sv, *Rm;
    int64_t* vtmp;
    int64_t* dbase;
    int *ipiv, *perm, *idxbuf;
    Touched T;
};

struct DistSizes {
    int64_t nmax, xcols, persistent_doubles;
};

// Largest per-rank column count, and the exchange / scratch widths (doubles) shared by the layout and the run.
static DistSizes dist_sizes(int64_t m, int64_t n, int64_t b, int64_t d, int G, int64_t nb)
{
    BlockCyclic bc{n, nb, G};
    DistSizes z{};
    for (int r = 0; r < G; ++r) z.nmax = imax(z.nmax, bc.n_loc(r));
    const int64_t bb = imin(b, imin(m, n));
    // exchange send / receive buffers (<= 2 min(w, d) columns of m rows), the sketch operator S^T (m x d), the
    // row-sharded panel's scattered / gathered row blocks ((h + G) x k), R11 (b x b)
    z.xcols = imax(2 * d, imax(d, cdiv((m + G) * bb, imax(m, 1)) + 1));
    auto r = [](int64_t x) { return (x + 31) / 32 * 32; };
    int64_t P = 0;
    P += r(n * d) * 2 + r(2 * d * d) + r(bb * bb) * 4 + r(8) + r(m * bb) + r(bb * imax(z.nmax, 1)) * 2;
    P += r(m * z.xcols) * 2 + r(8) + r(z.nmax * d + d) + r((int64_t)G * z.nmax * d + d);
    P += r(m * bb) + r(bb * bb) * 4 + r(bb);  // sharded panel: Q, two Grams, Wr, Rm, S
    P += r(2 * d) + r(G) + r(d) * 3 + r(n) + r(8 * d);  // int64 / int arrays (over-sized as doubles)
    z.persistent_doubles = P;
    return z;
}

struct DistRun {
    Ctx& cx;
    Ctx* bulk;  // low-priority stream (lookahead) or nullptr
    Ctx* aux;   // the panel's k x k finish (as on one GPU)
    cudaEvent_t ev_top, ev_bulk;
    Comm& comm;
    BlockCyclic bc;
    int G, me;
    int64_t m, n, b, d, n_loc, mn, bb, nmax, xcols;
    double* A;
    int64_t lda;
    uint64_t seed;
    double* tau;
    double rank_tol;
    int64_t* J;
    int passes;
    bool hqr_fallback, shard_panel;
    int* hf;      // pinned host flags
    int* hbuf;    // pinned host ints: tq, tsrc (2d each), index plan (4 x 2d)
    DistBufs B;
    std::vector<int64_t> off, len;

    void init()
    {
        mn = imin(m, n);
        bb = imin(b, mn);
        n_loc = bc.n_loc(me);
        DistSizes z = dist_sizes(m, n, b, d, G, bc.nb);
        nmax = z.nmax;
        xcols = z.xcols;
        B.MskT = cx.alloc((size_t)n * d);
        B.Lb = cx.alloc((size_t)n * d);
        B.rowscr = cx.alloc((size_t)2 * d * d);
        B.Rsk11 = cx.alloc((size_t)bb * bb);
        B.X = cx.alloc((size_t)bb * bb);
        B.R11 = cx.alloc((size_t)bb * bb);
        B.ref = cx.alloc(1);
        B.V = cx.alloc((size_t)m * bb);
        B.Tp = cx.alloc((size_t)bb * bb);
        B.W = cx.alloc((size_t)bb * imax(n_loc, 1));
        B.W2 = cx.alloc((size_t)bb * imax(n_loc, 1));
        B.xbuf = cx.alloc((size_t)m * xcols);
        B.rbuf = cx.alloc((size_t)m * xcols);
        B.dfl = cx.alloc(4);
        B.rowsbuf = cx.alloc((size_t)nmax * d + d);
        B.rowsgat = cx.alloc((size_t)G * nmax * d + d);
        B.Q = cx.alloc((size_t)m * bb);
        B.Gr1 = cx.alloc((size_t)bb * bb);
        B.Gr2 = cx.alloc((size_t)bb * bb);
        B.Wr = cx.alloc((size_t)bb * bb);
        B.Rm = cx.alloc((size_t)bb * bb);
        B.Sv = cx.alloc((size_t)bb);
        B.vtmp = cx.alloc_as<int64_t>((size_t)2 * d);
        B.dbase = cx.alloc_as<int64_t>((size_t)G);
        B.T.tq = cx.alloc_as<int>((size_t)2 * d);
        B.T.tsrc = cx.alloc_as<int>((size_t)2 * d);
        B.T.nt = cx.flags + F_NT;  // read back with the other flags
        B.ipiv = cx.alloc_as<int>((size_t)d);
        B.perm = cx.alloc_as<int>((size_t)n);
        B.idxbuf = cx.alloc_as<int>((size_t)8 * d);
    }

    void sync() { BQ_CUDA(cudaStreamSynchronize(cx.stream)); }
    void read_flags()
    {
        BQ_CUDA(cudaMemcpyAsync(hf, cx.flags, sizeof(int) * F_NFLAGS, cudaMemcpyDeviceToHost, cx.stream));
        sync();
    }

    // X1: every rank's sketch rows of positions >= p0 (packed in position order, nmax x d per rank, ld nmax)
    // all-gathered, then unpacked by position (a rank's own rows come back bit-identical)
    void allgather_rows(int64_t p0)
    {
        if (p0 >= n) return;
        int64_t nm = 0;
        std::vector<int64_t> base(G);
        for (int r = 0; r < G; ++r) {
            base[r] = bc.count_below(r, p0);
            nm = imax(nm, bc.n_loc(r) - base[r]);
        }
        if (nm == 0) return;
        BQ_CUDA(cudaMemcpyAsync(B.dbase, base.data(), sizeof(int64_t) * G, cudaMemcpyHostToDevice, cx.stream));
        const unsigned blk = (unsigned)imin(cdiv((n - p0) * d, 256), 8 * cx.num_sms);
        pack_rows_kernel<<<blk, 256, 0, cx.stream>>>(n, p0, d, bc.nb, G, me, B.MskT, n, base[me], B.rowsbuf, nm);
        BQ_LAUNCH_CHECK();
        comm.allgather(B.rowsbuf, B.rowsgat, sizeof(double) * nm * d, cx.stream);
        unpack_rows_kernel<<<blk, 256, 0, cx.stream>>>(n, p0, d, bc.nb, G, me, B.rowsgat, nm, B.dbase, B.MskT, n);
        BQ_LAUNCH_CHECK();
        sync();  // `base` is a stack buffer of the async copy
    }

    // a1: the sketch rows of this rank's columns (the one-GPU GEMM per element: no split-K), then X1
    void sketch()
    {
        if (n_loc > 0) {
            // MskT_loc (n_loc x d) straight into the pack buffer (ld nmax), S^T in the exchange buffer
            sketch_apply(cx, m, n_loc, A, lda, d, seed, B.rowsbuf, nmax, B.xbuf);
        }
        std::vector<int64_t> base(G, 0);
        BQ_CUDA(cudaMemcpyAsync(B.dbase, base.data(), sizeof(int64_t) * G, cudaMemcpyHostToDevice, cx.stream));
        comm.allgather(B.rowsbuf, B.rowsgat, sizeof(double) * nmax * d, cx.stream);
        const unsigned blk = (unsigned)imin(cdiv(n * d, 256), 8 * cx.num_sms);
        unpack_rows_kernel<<<blk, 256, 0, cx.stream>>>(n, 0, d, bc.nb, G, -1, B.rowsgat, nmax, B.dbase, B.MskT, n);
        BQ_LAUNCH_CHECK();
        sync();
    }

    // X3 (a3): touched columns from their source positions to their destinations (all m rows), and J
    void exchange(int64_t s, int64_t nt)
    {
        const int* htq = hbuf;
        const int* htsrc = hbuf + 2 * d;
        int* hidx = hbuf + 4 * d;
        std::vector<int64_t> q(nt), p(nt);
        for (int64_t t = 0; t < nt; ++t) {
            q[t] = s + htq[t];
            p[t] = s + htsrc[t];
        }
        ExchangePlan P;
        plan_exchange(bc, me, nt, q.data(), p.data(), P);
        const int64_t ns = (int64_t)P.send_idx.size(), nl = (int64_t)P.local_src.size(),
                      nr = (int64_t)P.recv_idx.size();
        // every source (sends, then local moves) is gathered before any destination is written
        std::copy(P.send_idx.begin(), P.send_idx.end(), hidx);
        std::copy(P.local_src.begin(), P.local_src.end(), hidx + ns);
        std::copy(P.recv_idx.begin(), P.recv_idx.end(), hidx + ns + nl);
        std::copy(P.local_dst.begin(), P.local_dst.end(), hidx + ns + nl + nr);
        const int64_t ni = ns + nl + nr + nl;
        if (ni) BQ_CUDA(cudaMemcpyAsync(B.idxbuf, hidx, sizeof(int) * ni, cudaMemcpyHostToDevice, cx.stream));
        gather_cols_idx(cx, m, A, lda, B.idxbuf, ns + nl, B.xbuf, m);
        std::vector<size_t> sc(G), sd(G), rc(G), rd(G);
        size_t so = 0, ro = 0;
        for (int r = 0; r < G; ++r) {
            sc[r] = (size_t)P.send_cnt[r] * m * sizeof(double);
            rc[r] = (size_t)P.recv_cnt[r] * m * sizeof(double);
            sd[r] = so;
            rd[r] = ro;
            so += sc[r];
            ro += rc[r];
        }
        // collective: every rank takes part even when it has nothing to send or receive (a caller transport's
        // all-to-all blocks until all ranks enter it)
        if (G > 1)
            comm.alltoallv((const char*)B.xbuf, sc.data(), sd.data(), (char*)B.rbuf, rc.data(), rd.data(), cx.stream);
        const unsigned chunks = (unsigned)imin(cdiv(m, 256 * 8), 64);
        if (nr) {
            scatter_idx_kernel<<<dim3(chunks, (unsigned)nr), 256, 0, cx.stream>>>(m, A, lda, B.idxbuf + ns + nl, B.rbuf, m);
            BQ_LAUNCH_CHECK();
        }
        if (nl) {
            scatter_idx_kernel<<<dim3(chunks, (unsigned)nl), 256, 0, cx.stream>>>(m, A, lda, B.idxbuf + ns + nl + nr,
                                                                                 B.xbuf + ns * m, m);
            BQ_LAUNCH_CHECK();
        }
        permute_vector(cx, J + s, B.T, B.vtmp);  // replicated J (the device touched set is identical everywhere)
        sync();                                  // the pinned index plan is reused next iteration
    }

    // a4 on the owner (bitwise the one-GPU panel, including its k x k finish on the aux stream), X2 broadcast
    // of V (explicit, h x k), T and tau(s:s+k)
    void panel_owner(int64_t s, int64_t h, int64_t k, int owner)
    {
        if (owner == me)
            g_panel_fallbacks += panel_factor(cx, h, A + s + bc.loc(s) * lda, lda, k, B.Rsk11, tau + s, passes, B.V,
                                              B.Tp, hqr_fallback, aux);
        comm.broadcast(B.V, sizeof(double) * h * k, owner, cx.stream);
        comm.broadcast(B.Tp, sizeof(double) * k * k, owner, cx.stream);
        comm.broadcast(tau + s, sizeof(double) * k, owner, cx.stream);
    }

    // a4 row-sharded (SURVEY §8(e) phase 2 item 3): the owner scatters the panel's row blocks (block g of hc
    // rows -> rank g < Gp = min(G, h / k)); each rank preconditions, Grams and solves its rows; the k x k POTRFs
    // and the reconstruction finish are replicated from all-reduced Grams; rank 0 (the top k rows) factors the
    // reconstruction LU and broadcasts it; V's rows are all-gathered.  Returns false on a POTRF breakdown
    // (identical on every rank; nothing written): the caller then runs the owner's panel with its fallback.
    bool panel_sharded(int64_t s, int64_t h, int64_t k, int owner)
    {
        const int Gp = (int)imin(G, h / k);
        const int64_t hc = cdiv(h, Gp);
        auto rows_of = [&](int g) { return g < Gp ? imax(0, imin(h, (int64_t)(g + 1) * hc) - (int64_t)g * hc) : 0; };
        const int64_t rows = rows_of(me);
        std::vector<size_t> sc(G, 0), sd(G, 0), rc(G, 0), rd(G, 0);
        if (owner == me) {
            const int64_t j0 = bc.loc(s);
            for (int g = 0; g < Gp; ++g) {
                double* dst = (g == me) ? B.Q : B.xbuf + (size_t)g * hc * k;
                copy_matrix(cx, rows_of(g), k, A + s + (int64_t)g * hc + j0 * lda, lda, dst, hc);
                if (g != me) {
                    sc[g] = sizeof(double) * hc * k;
                    sd[g] = sizeof(double) * g * hc * k;
                }
            }
        } else if (me < Gp) {
            rc[owner] = sizeof(double) * hc * k;
        }
        comm.alltoallv((const char*)B.xbuf, sc.data(), sd.data(), (char*)B.Q, rc.data(), rd.data(), cx.stream);
        const double* Cf[2] = {B.Gr1, B.Gr2};
        cholqr_precondition_gram(cx, rows, k, B.Q, hc, B.Rsk11, B.Q, hc, B.Gr1);
        comm.allreduce_sum(B.Gr1, (size_t)k * k, cx.stream);
        potrf_lower(cx, k, B.Gr1, k);
        if (passes == 2) {
            cholqr_pass_gram(cx, rows, k, B.Q, hc, B.Gr1, B.Gr2);
            comm.allreduce_sum(B.Gr2, (size_t)k * k, cx.stream);
            potrf_lower(cx, k, B.Gr2, k);
        }
        force_breakdown_hook(cx);
        read_flags();
        if (hf[F_POTRF_INFO]) {
            BQ_CUDA(cudaMemsetAsync(cx.flags + F_POTRF_INFO, 0, sizeof(int), cx.stream));
            return false;
        }
        const double* Cl = Cf[passes - 1];
        if (me == 0) recon_top_lu(cx, k, B.Q, hc, Cl, B.Wr, B.Sv);
        comm.broadcast(B.Wr, sizeof(double) * k * k, 0, cx.stream);
        comm.broadcast(B.Sv, sizeof(double) * k, 0, cx.stream);
        if (me == 0) {
            recon_rows(cx, rows - k, k, B.Q + k, hc, B.Wr, Cl);
            copy_matrix(cx, k, k, B.Wr, k, B.Q, hc);  // L \ U on top
        } else if (rows > 0) {
            recon_rows(cx, rows, k, B.Q, hc, B.Wr, Cl);
        }
        recon_finish(cx, k, B.Wr, B.Sv, Cf, passes, B.Rsk11, B.Tp, tau + s, B.Rm, nullptr);
        comm.allgather(B.Q, B.rbuf, sizeof(double) * hc * k, cx.stream);
        for (int g = 0; g < Gp; ++g) copy_matrix(cx, rows_of(g), k, B.rbuf + (size_t)g * hc * k, hc, B.V + (int64_t)g * hc, h);
        // GEQP3 write on the owner; elsewhere only the conversion of V to its explicit form (into scratch)
        if (owner == me) write_panel(cx, h, k, B.V, h, B.Rm, B.Sv, A + s + bc.loc(s) * lda, lda);
        else write_panel(cx, h, k, B.V, h, B.Rm, B.Sv, B.xbuf, h);
        return true;
    }

    // a6: X = R_sk11 R11^{-1} (replicated, on a context without split-K slices as on one GPU), then this
    // rank's rows of MskT(c:n, 0:b) -= R12^T X^T (split decision of the whole (n - c) x b update), then X1
    void sample_update(int64_t s, int64_t c, int owner)
    {
        if (owner == me) copy_matrix(cx, b, b, A + s + bc.loc(s) * lda, lda, B.R11, b);
        comm.broadcast(B.R11, sizeof(double) * b * b, owner, cx.stream);
        Ctx nos = cx;
        nos.splitk = nullptr;
        nos.splitk_elems = 0;
        copy_matrix(nos, b, b, B.Rsk11, b, B.X, b);
        trsm_right_upper(nos, b, b, B.R11, b, false, false, B.X, b);
        zero_triangle(nos, 'U', b, b, B.X, b);
        for (int64_t q0 = (c / bc.nb) * bc.nb; q0 < n; q0 += bc.nb) {
            if (bc.owner(q0) != me) continue;
            const int64_t lo = imax(q0, c), hi = imin(q0 + bc.nb, n);
            if (hi <= lo) continue;
            GemmExtra hint;
            hint.split_m = n - c;
            gemm(cx, true, true, hi - lo, b, b, -1.0, A + s + bc.loc(lo) * lda, lda, B.X, b, 1.0, B.MskT + lo, n, false,
                 0, false, &hint);
        }
        allgather_rows(c);
    }
};

static int64_t dist_loop(DistRun& D, bool lookahead)
{
    Ctx& cx = D.cx;
    const int64_t m = D.m, n = D.n, b = D.b, d = D.d;
    cx.mark(PH_OTHER);
    D.sketch();
    nonfinite_check(cx, n, d, D.B.MskT, n);
    bool bulk_pending = false;
    for (int64_t i = 0;; ++i) {
        const int64_t s = i * b;
        if (s >= D.mn) return D.mn;
        const int64_t c = imin(n, s + b), r = imin(m, s + b), w = n - s, h = m - s;
        const int64_t kmax = imin(imin(b, w), h);
        // ---- a2 (replicated; R_sk(:, d:w) only for this rank's positions when G > 1)
        cx.mark(PH_QRCP_WIDE);
        copy_matrix(cx, w, d, D.B.MskT + s, n, D.B.Lb, n);
        getrf_pivots(cx, D.B.Lb, n, w, d, D.B.ipiv, D.B.perm);
        touched_from_perm(cx, w, imin(w, d), D.B.perm, D.B.T);
        permute_rows(cx, d, D.B.MskT + s, n, D.B.T, D.B.rowscr);
        D.off.clear();
        D.len.clear();
        const int64_t p0 = s + imin(d, w);
        for (int64_t q0 = (s / D.bc.nb) * D.bc.nb; q0 < n; q0 += D.bc.nb) {
            if (D.bc.owner(q0) != D.me) continue;
            const int64_t lo = imax(q0, p0), hi = imin(q0 + D.bc.nb, n);
            if (hi > lo) {
                D.off.push_back(lo - p0);
                D.len.push_back(hi - lo);
            }
        }
        RowBlocks rb;
        rb.off = D.off.data();
        rb.len = D.len.data();
        rb.n = D.G > 1 ? (int64_t)D.off.size() : -1;
        sketch_qr(cx, D.B.MskT + s, n, w, d, rb, nullptr);
        cx.mark(PH_TRI_RANK);
        tri_rank_flags(cx, D.B.MskT + s, n, kmax, i == 0, D.rank_tol, D.B.ref);
        D.read_flags();
        const int64_t k = D.hf[F_K];
        const int64_t nt = D.hf[F_NT];
        if (nt > 0) {
            BQ_CUDA(cudaMemcpyAsync(D.hbuf, D.B.T.tq, sizeof(int) * nt, cudaMemcpyDeviceToHost, cx.stream));
            BQ_CUDA(cudaMemcpyAsync(D.hbuf + 2 * d, D.B.T.tsrc, sizeof(int) * nt, cudaMemcpyDeviceToHost, cx.stream));
        }
        // ---- a3 (after this rank's bulk rows of the previous update landed)
        cx.mark(PH_COL_PERM);
        if (bulk_pending) {
            BQ_CUDA(cudaStreamWaitEvent(cx.stream, D.ev_bulk, 0));
            bulk_pending = false;
        }
        D.sync();
        if (nt > 0) D.exchange(s, nt);
        // ---- a7 early exit: the owner tests A(s:m, s); flags summed over ranks
        const int owner = D.bc.owner(s);
        if (owner == D.me) zero_col_flag(cx, h, D.A + s + D.bc.loc(s) * D.lda);
        else BQ_CUDA(cudaMemsetAsync(cx.flags + F_ZERO_COL, 0, sizeof(int), cx.stream));
        flags_to_f64_kernel<<<1, 32, 0, cx.stream>>>(cx.flags, D.B.dfl);
        BQ_LAUNCH_CHECK();
        D.comm.allreduce_sum(D.B.dfl, 3, cx.stream);
        double hfl[3];
        BQ_CUDA(cudaMemcpyAsync(hfl, D.B.dfl, sizeof(hfl), cudaMemcpyDeviceToHost, cx.stream));
        D.sync();
        if (hfl[1] != 0.0 || hfl[2] != 0.0) return -1;
        if (k == 0 || hfl[0] != 0.0) return s;
        // ---- a4
        cx.mark(PH_QR_TALL);
        extract_rsk11(cx, k, D.B.MskT + s, n, D.B.Rsk11);
        const bool sharded = D.shard_panel && D.G > 1 && (D.passes == 1 || D.passes == 2) && h / k >= 2 &&
                             D.panel_sharded(s, h, k, owner);
        if (!sharded) D.panel_owner(s, h, k, owner);
        // ---- a5 on this rank's own trailing columns (positions >= s + k), split decisions of the whole update
        cx.mark(PH_APPLY_QT);
        const bool terminal = (k < kmax || c == n || r == m);
        const int64_t jt = D.bc.count_below(D.me, s + k), t_loc = D.n_loc - jt, t = n - s - k;
        if (t_loc > 0) {
            double* C = D.A + s + jt * D.lda;
            if (!lookahead || terminal || h <= k) {
                wy_top(cx, h, k, t_loc, D.B.V, h, D.B.Tp, C, D.lda, D.B.W, D.B.W2, h, t);
            } else {
                wy_top(cx, h, k, t_loc, D.B.V, h, D.B.Tp, C, D.lda, D.B.W, D.B.W2, k, t);
                BQ_CUDA(cudaEventRecord(D.ev_top, cx.stream));
                BQ_CUDA(cudaStreamWaitEvent(D.bulk->stream, D.ev_top, 0));
                wy_bulk(*D.bulk, h, k, t_loc, D.B.V, h, D.B.W2, C, D.lda, nullptr, nullptr);
                BQ_CUDA(cudaEventRecord(D.ev_bulk, D.bulk->stream));
                bulk_pending = true;
            }
        }
        if (terminal) {
            if (bulk_pending) BQ_CUDA(cudaStreamWaitEvent(cx.stream, D.ev_bulk, 0));
            return s + k;
        }
        // ---- a6 (overlapping this rank's bulk rows)
        cx.mark(PH_SAMPLE_UPDATE);
        D.sample_update(s, c, owner);
    }
}

// Per-rank workspace (bytes) of bqrrp_factor_dist: the one-GPU split-K slices and temporaries (the split-K
// capacity must equal the one-GPU run's: its decisions depend on it) plus the distributed buffers.
static size_t dist_workspace_bytes(int64_t m, int64_t n, int64_t b, int64_t d, int G, int64_t nb, size_t* splitk)
{
    const Layout L1 = layout(m, n, b, d);
    const DistSizes z = dist_sizes(m, n, b, d, G, nb);
    *splitk = L1.splitk;
    return L1.temp + L1.splitk + (size_t)z.persistent_doubles * 8 + (64u << 20);
}

}  // namespace bqrrp

using namespace bqrrp;

extern "C" {

int bqrrp_nccl_unique_id(void* id_out)
{
    if (!id_out) return -1;
    return guarded([&]() -> int {
        ncclUniqueId id;
        BQ_NCCL(nccl().getUniqueId(&id));
        std::memcpy(id_out, &id, sizeof(id));
        return 0;
    });
}

int bqrrp_comm_init(const void* nccl_unique_id, int rank, int nranks, void** comm_out)
{
    if (!nccl_unique_id) return -1;
    if (nranks < 1) return -3;
    if (rank < 0 || rank >= nranks) return -2;
    if (!comm_out) return -4;
    return guarded([&]() -> int {
        auto c = std::make_unique<NcclComm>();
        ncclUniqueId id;
        std::memcpy(&id, nccl_unique_id, sizeof(id));
        BQ_NCCL(nccl().commInitRank(&c->c, nranks, id, rank));
        c->rank = rank;
        c->size = nranks;
        *comm_out = static_cast<Comm*>(c.release());
        return 0;
    });
}

int bqrrp_comm_init_transport(const bqrrp_transport* t, void** comm_out)
{
    if (!t || !t->allreduce_sum_f64 || !t->allgather || !t->broadcast || !t->alltoallv) return -1;
    if (t->nranks < 1 || t->rank < 0 || t->rank >= t->nranks) return -1;
    if (!comm_out) return -2;
    auto c = new CallbackComm();
    c->t = *t;
    c->rank = t->rank;
    c->size = t->nranks;
    *comm_out = static_cast<Comm*>(c);
    return 0;
}

int bqrrp_comm_destroy(void* comm)
{
    if (!comm) return 0;
    return guarded([&]() -> int {
        delete static_cast<Comm*>(comm);
        return 0;
    });
}

int bqrrp_dist_local_columns(int64_t n, int64_t nb, int nranks, int rank, int64_t* n_local)
{
    if (n < 0) return -1;
    if (nb < 1) return -2;
    if (nranks < 1) return -3;
    if (rank < 0 || rank >= nranks) return -4;
    if (!n_local) return -5;
    BlockCyclic bc{n, nb, nranks};
    *n_local = bc.n_loc(rank);
    return 0;
}

int bqrrp_dist_exchange_plan(int64_t n, int64_t nb, int nranks, int rank, int64_t nt, const int64_t* q,
                             const int64_t* p, int32_t* send_idx, int64_t* send_counts, int32_t* recv_idx,
                             int64_t* recv_counts, int32_t* local_src, int32_t* local_dst, int64_t* n_local_moves)
{
    if (n < 0 || nb < 1 || nranks < 1 || rank < 0 || rank >= nranks || nt < 0) return -1;
    if (nt > 0 && (!q || !p)) return -6;
    BlockCyclic bc{n, nb, nranks};
    ExchangePlan P;
    plan_exchange(bc, rank, nt, q, p, P);
    std::copy(P.send_idx.begin(), P.send_idx.end(), send_idx);
    std::copy(P.recv_idx.begin(), P.recv_idx.end(), recv_idx);
    std::copy(P.local_src.begin(), P.local_src.end(), local_src);
    std::copy(P.local_dst.begin(), P.local_dst.end(), local_dst);
    for (int r = 0; r < nranks; ++r) {
        send_counts[r] = P.send_cnt[r];
        recv_counts[r] = P.recv_cnt[r];
    }
    *n_local_moves = (int64_t)P.local_src.size();
    return 0;
}

int bqrrp_workspace_query_dist(int64_t m, int64_t n, int64_t b, int64_t d, int nranks, int64_t dist_nb, size_t* bytes)
{
    if (m < 0) return -1;
    if (n < 0) return -2;
    if (b < 1) return -3;
    if (d < b || (m > 0 && d > m)) return -4;
    if (nranks < 1) return -5;
    if (!bytes) return -7;
    size_t sk = 0;
    *bytes = dist_workspace_bytes(m, n, b, d, nranks, dist_nb > 0 ? dist_nb : b, &sk);
    return 0;
}

int bqrrp_factor_dist(int64_t m, int64_t n, double* A_local, int64_t lda_local, int64_t b, int64_t d, uint64_t seed,
                      double* tau, int64_t* J, int64_t* rank, void* comm, void* workspace, size_t ws_bytes,
                      void* stream, const bqrrp_options* opts)
{
    if (m < 0) return -1;
    if (n < 0) return -2;
    if (!comm) return -11;
    Comm* cm = static_cast<Comm*>(comm);
    const int64_t nb = (opts && opts->dist_nb > 0) ? opts->dist_nb : b;
    BlockCyclic bc0{n, nb, cm->size};
    const int64_t n_loc = bc0.n_loc(cm->rank);
    if (!A_local && m > 0 && n_loc > 0) return -3;
    if (lda_local < (m > 1 ? m : 1)) return -4;
    if (b < 1) return -5;
    if (d < b || (m > 0 && d > m)) return -6;
    if (!tau && m > 0 && n > 0) return -8;
    if (!J && n > 0) return -9;
    if (!rank) return -10;
    if (nb % b != 0 && b % nb != 0) return -15;  // every panel must live on one rank
    if (nb < b) return -15;
    const double rank_tol = (opts && opts->rank_tol > 0) ? opts->rank_tol : 10.0 * 0x1p-53 * sqrt((double)(m > n ? m : n));
    const int passes = (opts && opts->cholqr_passes >= 0 && opts->cholqr_passes <= 4) ? opts->cholqr_passes : 2;
    g_panel_fallbacks = 0;
    return guarded([&]() -> int {
        Ctx cx;
        setup_ctx(cx, stream);
        cx.force_breakdown = opts && (opts->debug_flags & BQRRP_DEBUG_FORCE_BREAKDOWN);
        if (m == 0 || n == 0) {
            *rank = 0;
            if (n > 0) init_j(cx, n, J);
            return 0;
        }
        if (n > lu_max_rows(cx.num_sms)) return -2;
        size_t sk = 0;
        const size_t need = dist_workspace_bytes(m, n, b, d, cm->size, nb, &sk);
        void* ws = workspace;
        bool own = false;
        if (!ws) {
            BQ_CUDA(lib_malloc_async(&ws, need, cx.stream));
            ws_bytes = need;
            own = true;
        } else if (ws_bytes < need) {
            g_last_error = "workspace smaller than bqrrp_workspace_query_dist";
            return -13;
        }
        Layout L{0, 0, sk, need};
        carve(cx, ws, ws_bytes, L);
        int prio_lo = 0, prio_hi = 0;
        BQ_CUDA(cudaDeviceGetStreamPriorityRange(&prio_lo, &prio_hi));
        cudaStream_t user = cx.stream, s_hi = nullptr, s_lo = nullptr, s_aux = nullptr;
        cudaEvent_t ev_in = nullptr, ev_top = nullptr, ev_bulk = nullptr, ev_done = nullptr;
        BQ_CUDA(cudaStreamCreateWithPriority(&s_hi, cudaStreamNonBlocking, prio_hi));
        BQ_CUDA(cudaStreamCreateWithPriority(&s_lo, cudaStreamNonBlocking, prio_lo));
        BQ_CUDA(cudaStreamCreateWithPriority(&s_aux, cudaStreamNonBlocking, prio_hi));
        for (cudaEvent_t* e : {&ev_in, &ev_top, &ev_bulk, &ev_done})
            BQ_CUDA(cudaEventCreateWithFlags(e, cudaEventDisableTiming));
        BQ_CUDA(cudaEventRecord(ev_in, user));
        for (cudaStream_t st : {s_hi, s_lo, s_aux}) BQ_CUDA(cudaStreamWaitEvent(st, ev_in, 0));
        cx.stream = s_hi;
        Ctx cxb = cx, cxa = cx;
        cxb.stream = s_lo;
        cxa.stream = s_aux;
        for (Ctx* c : {&cxb, &cxa}) {
            c->splitk = nullptr;
            c->splitk_elems = 0;
        }
        Timer tm;
        if (opts && opts->phase_ms) {
            tm.on = true;
            tm.st = s_hi;
            cx.timer = &tm;
        }
        const bool lookahead = !(opts && opts->no_lookahead);
        DistRun D{cx, lookahead ? &cxb : nullptr, lookahead ? &cxa : nullptr, ev_top, ev_bulk, *cm, bc0, cm->size,
                  cm->rank, m, n, b, d, 0, 0, 0, 0, 0, A_local, lda_local, seed, tau, rank_tol, J, passes,
                  !(opts && opts->no_hqr_fallback), opts && (opts->dist_flags & BQRRP_DIST_SHARD_PANEL),
                  pinned_flags(), nullptr, {}, {}, {}};
        int* hb = nullptr;
        BQ_CUDA(cudaMallocHost(&hb, sizeof(int) * 8 * (size_t)d));
        D.hbuf = hb;
        int64_t ell = -1;
        auto cleanup = [&]() {
            for (cudaStream_t st : {s_hi, s_lo, s_aux}) {
                cudaEventRecord(ev_done, st);
                cudaStreamWaitEvent(user, ev_done, 0);
            }
            cudaStreamSynchronize(user);
            for (cudaStream_t st : {s_hi, s_lo, s_aux}) cudaStreamDestroy(st);
            for (cudaEvent_t e : {ev_in, ev_top, ev_bulk, ev_done}) cudaEventDestroy(e);
            cudaFreeHost(hb);
            cx.stream = user;
        };
        try {
            D.init();
            init_j(cx, n, J);
            BQ_CUDA(cudaMemsetAsync(tau, 0, sizeof(double) * D.mn, cx.stream));
            BQ_CUDA(cudaMemsetAsync(cx.flags, 0, sizeof(int) * F_NFLAGS, cx.stream));
            ell = dist_loop(D, lookahead);
            if (ell >= 0) {
                // O4 (reading Z16): tau(ell:) = 0, A(ell:m, ell:n) = 0 on this rank's columns
                cx.mark(PH_OTHER);
                BQ_CUDA(cudaStreamWaitEvent(cx.stream, ev_bulk, 0));
                if (ell < D.mn) BQ_CUDA(cudaMemsetAsync(tau + ell, 0, sizeof(double) * (D.mn - ell), cx.stream));
                const int64_t jl = bc0.count_below(cm->rank, ell);
                set_zero(cx, m - ell, n_loc - jl, A_local + ell + jl * lda_local, lda_local);
                cx.mark(PH_OTHER);
            }
        } catch (...) {
            cleanup();
            if (own) cudaFreeAsync(ws, user);
            throw;
        }
        cleanup();
        if (opts && opts->phase_ms) tm.finish(opts->phase_ms);
        if (own) BQ_CUDA(cudaFreeAsync(ws, user));
        if (ell < 0) {
            g_last_error = "non-finite sketch or Cholesky-QR breakdown";
            *rank = 0;
            return BQRRP_ENUMERIC;
        }
        *rank = ell;
        return 0;
    });
}

}  // extern "C"
