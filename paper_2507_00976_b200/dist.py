"""Multi-GPU BQRRP (phase 1): A is distributed 1-D block-cyclically over column POSITIONS
(block width nb = b, so every panel lives on one rank); the transposed sketch MskT (n x d), J and tau are
replicated.  Per iteration (Alg. 1):

  a2  every rank runs the same pivot selection on the replicated sketch (deterministic kernels, identical
      inputs -> identical pivots, k and R_sk on every rank)                      bqrrp_step_pivots
  a3  X3: the <= 2 min(d, w) touched columns are packed by their owners into one buffer whose slots are
      filled by exactly one rank, summed across ranks (exact: every other rank contributes zeros) and
      unpacked by the new owners                                                 gather / all-reduce / scatter
  a4  the panel owner factors it; X2: V, T, tau (and R11) broadcast               bqrrp_step_panel
  a5  every rank updates its own trailing columns                                  bqrrp_step_wy_update
  a6  X1: R12 (k x t) assembled in position order by an exact all-reduce, then the replicated sketch update
                                                                                   bqrrp_step_sample_update

Every arithmetic step runs in libbqrrp.so's kernels; torch.distributed (NCCL on a multi-GPU node, gloo in
the single-GPU tests where two ranks share one device) only moves buffers.  The result equals the
single-GPU factorization (J and rank identical, R / V / tau to rounding: the local GEMMs see different N
and may choose different tilings, which does not change any element's K order, and split-K is only
taken for small-MN shapes).
"""
from __future__ import annotations

import ctypes

import numpy as np

from . import BqrrpError, _check, _stream_ptr, default_rank_tol, lib

__all__ = ["BlockCyclic", "factor_dist", "local_columns"]


class BlockCyclic:
    """1-D block-cyclic map of n column positions over G ranks with block width nb."""

    def __init__(self, n: int, nb: int, G: int, rank: int):
        self.n, self.nb, self.G, self.rank = n, nb, G, rank
        p = np.arange(n)
        self.owner_of = (p // nb) % G
        self.pos = p[self.owner_of == rank]  # this rank's positions, ascending
        self.loc_of = np.full(n, -1, dtype=np.int64)
        self.loc_of[self.pos] = np.arange(len(self.pos))

    @property
    def n_loc(self) -> int:
        return len(self.pos)

    def first_local_at_or_after(self, p: int) -> int:
        return int(np.searchsorted(self.pos, p))

    def blocks_of_from(self, r: int, p: int):
        """First positions of rank r's nb-blocks that end after position p (p is a multiple of nb in use)."""
        first = (p // self.nb) * self.nb
        return [q0 for q0 in range(first, self.n, self.nb) if (q0 // self.nb) % self.G == r]

    def own_blocks_from(self, p: int):
        return self.blocks_of_from(self.rank, p)


def local_columns(A, nb: int, G: int, rank: int):
    """This rank's block-cyclic columns of a full column-major tensor (for tests and the bench)."""
    import torch

    bc = BlockCyclic(A.shape[1], nb, G, rank)
    idx = torch.as_tensor(bc.pos, device=A.device)
    loc = A.index_select(1, idx)
    return loc.t().contiguous().t(), bc


def _ptr(t):
    return ctypes.c_void_p(t.data_ptr())


def _dense(t):
    """The contiguous tensor behind a column-major view (colmaj(r, c) is a transposed row-major (c, r) block):
    NCCL collectives reject non-contiguous tensors ("Tensors must be contiguous"), and a collective acts on
    the same bytes either way."""
    if t.is_contiguous():
        return t
    tt = t.t()
    if tt.is_contiguous():
        return tt
    raise ValueError("collective buffer is neither row- nor column-major contiguous")


def _declare():
    L = lib()
    if getattr(L, "_dist_declared", False):
        return L
    i64, d, P, i32 = ctypes.c_int64, ctypes.c_double, ctypes.c_void_p, ctypes.c_int
    L.bqrrp_step_pivots.argtypes = [i64, i64, i64, i64, P, i64, P, d, P, i32, P, P, P, ctypes.POINTER(i64), P]
    L.bqrrp_step_gather_columns.argtypes = [i64, P, i64, P, i64, P, i64, P]
    L.bqrrp_step_scatter_columns.argtypes = [i64, P, i64, P, i64, P, i64, P]
    L.bqrrp_step_zero_column_check.argtypes = [i64, P, ctypes.POINTER(i32), P]
    L.bqrrp_step_panel.argtypes = [i64, i64, P, i64, P, i64, P, P, P, i32, P]
    L.bqrrp_step_wy_update.argtypes = [i64, i64, i64, P, P, P, i64, P]
    L.bqrrp_step_pivots_rows.argtypes = [i64, i64, i64, i64, P, i64, P, d, P, i32, P, P, P, ctypes.POINTER(i64), P,
                                         P, i64, P]
    L.bqrrp_step_sample_update_rows.argtypes = [i64, P, i64, P, i64, P, i64, P, P, P, i64, P]
    L.bqrrp_step_cholqr_pre.argtypes = [i64, i64, P, i64, P, i64, P, i64, P, P]
    L.bqrrp_step_potrf.argtypes = [i64, P, i64, P]
    L.bqrrp_step_cholqr_pass.argtypes = [i64, i64, P, i64, P, P, P]
    L.bqrrp_step_recon_top.argtypes = [i64, P, i64, P, P, P, P]
    L.bqrrp_step_recon_rows.argtypes = [i64, i64, P, i64, P, P, P]
    L.bqrrp_step_recon_finish.argtypes = [i64, P, P, P, P, P, i64, P, P, P, P]
    L.bqrrp_step_v_rows.argtypes = [i64, i64, P, i64, P, i32, P]
    L.bqrrp_step_write_panel.argtypes = [i64, i64, P, i64, P, P, P, i64, P]
    L.bqrrp_step_wy_top.argtypes = [i64, i64, i64, P, P, P, i64, P, i64, P]
    L.bqrrp_step_wy_bulk.argtypes = [i64, i64, i64, P, P, i64, P, i64, P]
    L.bqrrp_step_sample_update.argtypes = [i64, i64, P, i64, P, i64, P, i64, P]
    L.bqrrp_step_zero.argtypes = [i64, i64, P, i64, P]
    L.bqrrp_debug_sketch.argtypes = [i64, i64, P, i64, i64, ctypes.c_uint64, P, P, P]
    L._dist_declared = True
    return L


def factor_dist(A_loc, m: int, n: int, b: int, d: int | None = None, seed: int = 0, rank_tol: float | None = None,
                cholqr_passes: int = 2, group=None, lookahead: bool = True, exchange: str = "auto",
                shard_panel: bool = True, shard_sketch: bool = True):
    """Distributed BQRRP.  A_loc: this rank's block-cyclic columns (m x n_loc, column-major float64 CUDA).
    Returns (A_loc, tau, J, rank) with A_loc overwritten in GEQP3 format (R above, V below, in this rank's
    columns), tau (min(m,n)) and J (n, one-based gather) replicated.

    lookahead: the critical chain runs on a high-priority stream and each rank's bulk trailing rows (rows k:h
    of C -= V W2, bqrrp_step_wy_bulk) on a low-priority one, overlapping the R12 exchange, the replicated
    sample update and the next pivot selection; the next column exchange waits for it.
    exchange: "a2a" (point-to-point column moves), "allreduce" (exact-sum of the touched set) or "auto"
    (a2a on NCCL).
    shard_panel: the CholQR panel's row work (preconditioning TRSM, both Gram SYRKs, the pass-1 TRSM and the
    Y2 TRSM) is split over the ranks by rows, the k x k factorizations are replicated (bqrrp_step_cholqr_pre /
    potrf / cholqr_pass / recon_*); a POTRF breakdown falls back to the owner's Householder panel.
    shard_sketch: the R_sk(:, d:) GEMM of the pivot selection and the sample update run on this rank's
    positions only, and one all-gather of the updated sketch rows per iteration (instead of the R12 exchange)
    keeps the replicated pivot selection whole."""
    import torch

    caller = torch.cuda.current_stream(A_loc.device)
    crit = torch.cuda.Stream(device=A_loc.device, priority=-1)
    bulk = torch.cuda.Stream(device=A_loc.device, priority=0) if lookahead else None
    crit.wait_stream(caller)
    if bulk is not None:
        bulk.wait_stream(caller)
    with torch.cuda.stream(crit):
        out = _factor_dist_impl(A_loc, m, n, b, d, seed, rank_tol, cholqr_passes, group, bulk, exchange, shard_panel,
                                shard_sketch)
    caller.wait_stream(crit)
    if bulk is not None:
        caller.wait_stream(bulk)
    return out


def _allgather_sketch_rows(MskT, c, n, d, b, bc, me, G, group, colmaj, dev):
    """Every rank contributes the sketch rows of its own positions >= c (b-row blocks, stacked and padded to
    the largest block count); after one all-gather each rank copies the other ranks' blocks into MskT."""
    import torch
    import torch.distributed as dist

    blocks = [bc.blocks_of_from(r, c) for r in range(G)]
    nmax = max(len(x) for x in blocks)
    if nmax == 0:
        return
    buf = colmaj(nmax * b, d)
    for j, q0 in enumerate(blocks[me]):
        ln = min(b, n - q0)
        buf[j * b:j * b + ln].copy_(MskT[q0:q0 + ln])
    gathered = torch.empty(G * nmax * b * d, dtype=torch.float64, device=dev)
    dist.all_gather_into_tensor(gathered, _dense(buf).reshape(-1), group=group)
    for r in range(G):
        if r == me:
            continue
        blk = gathered[r * nmax * b * d:(r + 1) * nmax * b * d].view(d, nmax * b).t()
        for j, q0 in enumerate(blocks[r]):
            ln = min(b, n - q0)
            MskT[q0:q0 + ln].copy_(blk[j * b:j * b + ln])


def _exchange_a2a(L, A_loc, lda, m, q, p, bc, me, G, group, st, dev, colmaj):
    """X3 (a3): move column position p[t] -> q[t] for every touched slot t (q sorted).  Every source column is
    gathered (sends in (destination rank, slot) order, then this rank's local moves) before any destination is
    written; one all_to_all_single carries the cross-rank columns; receives arrive in (source rank, slot) order."""
    import torch
    import torch.distributed as dist

    src, dst = bc.owner_of[p], bc.owner_of[q]
    s_idx = np.nonzero((src == me) & (dst != me))[0]
    s_idx = s_idx[np.argsort(dst[s_idx], kind="stable")]
    r_idx = np.nonzero((dst == me) & (src != me))[0]
    r_idx = r_idx[np.argsort(src[r_idx], kind="stable")]
    l_idx = np.nonzero((src == me) & (dst == me))[0]
    ns, nr, nl = len(s_idx), len(r_idx), len(l_idx)
    pack = np.concatenate([bc.loc_of[p[s_idx]], bc.loc_of[p[l_idx]]]).astype(np.int32)
    buf = colmaj(m, max(ns + nl, 1))
    if ns + nl > 0:
        _check(L.bqrrp_step_gather_columns(m, _ptr(A_loc), lda, _ptr(torch.as_tensor(pack, device=dev)), ns + nl,
                                           _ptr(buf), m, st), "gather")
    recv = colmaj(m, max(nr, 1))
    send_counts = (np.bincount(dst[s_idx], minlength=G) * m).tolist()
    recv_counts = (np.bincount(src[r_idx], minlength=G) * m).tolist()
    dist.all_to_all_single(recv.t().reshape(-1)[: nr * m], buf.t().reshape(-1)[: ns * m], recv_counts, send_counts,
                           group=group)
    if nr > 0:
        idx = torch.as_tensor(bc.loc_of[q[r_idx]].astype(np.int32), device=dev)
        _check(L.bqrrp_step_scatter_columns(m, _ptr(A_loc), lda, _ptr(idx), nr, _ptr(recv), m, st), "scatter")
    if nl > 0:
        idx = torch.as_tensor(bc.loc_of[q[l_idx]].astype(np.int32), device=dev)
        _check(L.bqrrp_step_scatter_columns(m, _ptr(A_loc), lda, _ptr(idx), nl, _ptr(buf[:, ns:]), m, st), "scatter")


def _panel_sharded(L, A_loc, lda, m, s, h, k, b, n, MskT, bc, me, G, owner, group, st, dev, colmaj, passes, V, T, tk,
                   R11):
    """a4 with the panel's rows split over Gp = min(G, h // k) ranks (rank 0 holds the top k rows).  Returns
    False (nothing written) if a replicated POTRF breaks down: the caller then runs the owner's panel, whose
    Householder fallback handles it.  On success V (h x k explicit), T, tk and, on the owner, the panel columns
    of A_loc (GEQP3 format) and R11 are set."""
    import torch
    import torch.distributed as dist

    f64 = dict(dtype=torch.float64, device=dev)
    P = colmaj(h, k)
    j0 = int(bc.loc_of[s]) if owner == me else 0
    if owner == me:
        P.copy_(A_loc[s:, j0:j0 + k])
    dist.broadcast(_dense(P), src=owner, group=group)
    Gp = min(G, h // k)
    hc = -(-h // Gp)
    r0 = me * hc
    rows = max(0, min(h, r0 + hc) - r0) if me < Gp else 0
    ldq = max(rows, 1)
    Q = colmaj(ldq, k)
    C1 = colmaj(k, k)
    _check(L.bqrrp_step_cholqr_pre(rows, k, _ptr(P[min(r0, h - 1):]), h, _ptr(MskT[s:]), n, _ptr(Q), ldq, _ptr(C1), st),
           "cholqr_pre")
    dist.all_reduce(_dense(C1), group=group)
    if L.bqrrp_step_potrf(k, _ptr(C1), k, st) != 0:
        return False
    C2 = None
    if passes == 2:
        C2 = colmaj(k, k)
        _check(L.bqrrp_step_cholqr_pass(rows, k, _ptr(Q), ldq, _ptr(C1), _ptr(C2), st), "cholqr_pass")
        dist.all_reduce(_dense(C2), group=group)
        if L.bqrrp_step_potrf(k, _ptr(C2), k, st) != 0:
            return False
    Cl = C2 if C2 is not None else C1
    Wr = colmaj(k, k)
    Sv = torch.zeros(k, **f64)
    if me == 0:
        _check(L.bqrrp_step_recon_top(k, _ptr(Q), ldq, _ptr(Cl), _ptr(Wr), _ptr(Sv), st), "recon_top")
    dist.broadcast(_dense(Wr), src=0, group=group)
    dist.broadcast(_dense(Sv), src=0, group=group)
    if me == 0:
        _check(L.bqrrp_step_recon_rows(rows - k, k, _ptr(Q[k:]), ldq, _ptr(Wr), _ptr(Cl), st), "recon_rows")
        _check(L.bqrrp_step_v_rows(rows, k, _ptr(Q), ldq, _ptr(Wr), 1, st), "v_rows")
    elif rows > 0:
        _check(L.bqrrp_step_recon_rows(rows, k, _ptr(Q), ldq, _ptr(Wr), _ptr(Cl), st), "recon_rows")
    Rm = colmaj(k, k)
    _check(L.bqrrp_step_recon_finish(k, _ptr(Wr), _ptr(Sv), _ptr(C1), _ptr(C2) if C2 is not None else None,
                                     _ptr(MskT[s:]), n, _ptr(T), _ptr(tk), _ptr(Rm), st), "recon_finish")
    # V rows: every rank's block (padded to hc rows) all-gathered, then stacked in row order
    Vb = colmaj(hc, k)
    if rows > 0:
        Vb[:rows].copy_(Q[:rows])
    gathered = torch.empty(G * hc * k, **f64)
    dist.all_gather_into_tensor(gathered, Vb.t().reshape(-1), group=group)
    for g_ in range(Gp):
        rg = max(0, min(h, (g_ + 1) * hc) - g_ * hc)
        blk = gathered[g_ * hc * k:(g_ + 1) * hc * k].view(k, hc).t()
        V[g_ * hc:g_ * hc + rg].copy_(blk[:rg])
    if owner == me:
        _check(L.bqrrp_step_write_panel(h, k, _ptr(V), h, _ptr(Rm), _ptr(Sv), _ptr(A_loc[s:, j0:]), lda, st), "write")
        if k == b:
            R11.copy_(torch.triu(A_loc[s:s + b, j0:j0 + b]))
    return True


def _factor_dist_impl(A_loc, m, n, b, d, seed, rank_tol, cholqr_passes, group, bulk, exchange, shard_panel,
                      shard_sketch):
    import torch
    import torch.distributed as dist

    L = _declare()
    G = dist.get_world_size(group)
    me = dist.get_rank(group)
    dev = A_loc.device
    st = _stream_ptr()
    d = b if d is None else d
    mn = min(m, n)
    if rank_tol is None:
        rank_tol = default_rank_tol(m, n)
    bc = BlockCyclic(n, b, G, me)
    assert A_loc.shape == (m, bc.n_loc) and (A_loc.stride(0) == 1 or m <= 1), "A_loc: m x n_loc column-major"
    lda = max(A_loc.stride(1), m)
    f64 = dict(dtype=torch.float64, device=dev)

    def allreduce_sum(t):
        dist.all_reduce(_dense(t), op=dist.ReduceOp.SUM, group=group)

    # X3 as point-to-point moves (all_to_all_single: each moved column crosses the fabric once) on NCCL; the
    # exact-sum all-reduce of the whole touched set (2x the volume, every column to every rank) otherwise
    use_a2a = exchange == "a2a" or (exchange == "auto" and dist.get_backend(group) == "nccl")
    shard_sketch = shard_sketch and G > 1

    def colmaj(rows, cols):
        return torch.zeros((cols, rows), **f64).t()

    # ---- a1: local sketch rows, assembled into the replicated MskT (n x d) by an exact all-reduce
    MskT = colmaj(n, d)
    if bc.n_loc > 0:
        MskT_loc = colmaj(bc.n_loc, d)
        _check(L.bqrrp_debug_sketch(m, bc.n_loc, _ptr(A_loc), lda, d, seed, None, _ptr(MskT_loc), st),
               "bqrrp_debug_sketch")
        MskT[torch.as_tensor(bc.pos, device=dev)] = MskT_loc
    allreduce_sum(MskT)
    J = torch.arange(1, n + 1, dtype=torch.int64, device=dev)
    tau = torch.zeros(max(mn, 1), **f64)
    ref = torch.zeros(1, **f64)
    tq = torch.zeros(2 * d, dtype=torch.int32, device=dev)
    tsrc = torch.zeros(2 * d, dtype=torch.int32, device=dev)
    nt = torch.zeros(1, dtype=torch.int32, device=dev)
    ell = mn
    i = 0
    pending = None  # bulk trailing update of the previous iteration (lookahead)
    while True:
        s = i * b
        if s >= mn:
            ell = mn
            break
        c, r, w, h = min(n, s + b), min(m, s + b), n - s, m - s
        kmax = min(b, w, h)
        # ---- a2 (replicated)
        k = ctypes.c_int64(0)
        if shard_sketch:
            # R_sk(:, d:w) only for this rank's positions (the rest of MskT is refreshed by the row all-gather
            # after the sample update)
            p0 = s + min(d, n - s)
            offs, lens = [], []
            for q0 in bc.own_blocks_from(s):
                lo, hi = max(q0, p0), min(q0 + b, n)
                if hi > lo:
                    offs.append(lo - p0)
                    lens.append(hi - lo)
            offs_a = np.ascontiguousarray(offs, dtype=np.int64)
            lens_a = np.ascontiguousarray(lens, dtype=np.int64)
            _check(L.bqrrp_step_pivots_rows(n, d, s, kmax, _ptr(MskT), n, _ptr(J), float(rank_tol), _ptr(ref),
                                            int(i == 0), _ptr(tq), _ptr(tsrc), _ptr(nt), ctypes.byref(k),
                                            offs_a.ctypes.data_as(ctypes.c_void_p),
                                            lens_a.ctypes.data_as(ctypes.c_void_p), len(offs), st),
                   "bqrrp_step_pivots_rows")
        else:
            _check(L.bqrrp_step_pivots(n, d, s, kmax, _ptr(MskT), n, _ptr(J), float(rank_tol), _ptr(ref),
                                       int(i == 0), _ptr(tq), _ptr(tsrc), _ptr(nt), ctypes.byref(k), st),
                   "bqrrp_step_pivots")
        k = int(k.value)
        ntv = int(nt.item())
        # ---- a3: X3 column exchange through one exactly-summed buffer (after this rank's bulk update landed)
        if pending is not None:
            torch.cuda.current_stream().wait_event(pending)
            pending = None
        if ntv > 0:
            q = tq[:ntv].cpu().numpy().astype(np.int64) + s
            p = tsrc[:ntv].cpu().numpy().astype(np.int64) + s
            # the kernel emits the touched set in atomic (per-rank) order: sort by destination so that slot t of
            # the exchange buffer names the same column on every rank
            o = np.argsort(q, kind="stable")
            q, p = q[o], p[o]
            if use_a2a:
                _exchange_a2a(L, A_loc, lda, m, q, p, bc, me, G, group, st, dev, colmaj)
            else:
                pack = np.where(bc.owner_of[p] == me, bc.loc_of[p], -1).astype(np.int32)
                unpack = np.where(bc.owner_of[q] == me, bc.loc_of[q], -1).astype(np.int32)
                buf = colmaj(m, ntv)
                _check(L.bqrrp_step_gather_columns(m, _ptr(A_loc), lda, _ptr(torch.as_tensor(pack, device=dev)), ntv,
                                                   _ptr(buf), m, st), "gather")
                allreduce_sum(buf)
                _check(L.bqrrp_step_scatter_columns(m, _ptr(A_loc), lda, _ptr(torch.as_tensor(unpack, device=dev)),
                                                    ntv, _ptr(buf), m, st), "scatter")
        # ---- a7 early exit: the owner of position s tests A(s:m, s)
        owner = int(bc.owner_of[s])
        flag = torch.zeros(1, **f64)
        if owner == me:
            z = ctypes.c_int(0)
            _check(L.bqrrp_step_zero_column_check(h, _ptr(A_loc[s:, int(bc.loc_of[s])]), ctypes.byref(z), st), "zc")
            flag.fill_(float(z.value))
        allreduce_sum(flag)
        if k == 0 or flag.item() != 0.0:
            ell = s
            break
        # ---- a4: row-sharded CholQR panel (every rank factors a block of the panel's rows; V all-gathered) or
        #      on the owner with an X2 broadcast of V, T, tau (+ R11)
        V = colmaj(h, k)
        T = colmaj(k, k)
        tk = torch.zeros(k, **f64)
        R11 = colmaj(b, b)
        status = torch.zeros(1, **f64)
        sharded = (shard_panel and G > 1 and cholqr_passes in (1, 2) and h // k >= 2
                   and _panel_sharded(L, A_loc, lda, m, s, h, k, b, n, MskT, bc, me, G, owner, group, st, dev, colmaj,
                                      cholqr_passes, V, T, tk, R11))
        if sharded:
            pass
        elif owner == me:
            j0 = int(bc.loc_of[s])
            st_panel = L.bqrrp_step_panel(h, k, _ptr(A_loc[s:, j0:]), lda, _ptr(MskT[s:]), n, _ptr(tk), _ptr(V),
                                          _ptr(T), int(cholqr_passes), st)
            status.fill_(float(st_panel))
            if k == b:
                R11.copy_(torch.triu(A_loc[s:s + b, j0:j0 + b]))
        if not sharded:
            allreduce_sum(status)
            if status.item() != 0.0:
                raise BqrrpError(int(status.item()), "bqrrp_step_panel (distributed)")
            for t_ in (V, T, tk):
                dist.broadcast(_dense(t_), src=owner, group=group)
        tau[s:s + k] = tk
        # ---- a5 on every rank's own trailing columns (positions >= s + k)
        j_tr = bc.first_local_at_or_after(s + k)
        t_loc = bc.n_loc - j_tr
        if t_loc > 0:
            C = A_loc[s:, j_tr:]
            terminal = k < kmax or c == n or r == m
            if bulk is None or terminal or h <= k:
                _check(L.bqrrp_step_wy_update(h, k, t_loc, _ptr(V), _ptr(T), _ptr(C), lda, st), "wy")
            else:
                W2 = colmaj(k, t_loc)
                _check(L.bqrrp_step_wy_top(h, k, t_loc, _ptr(V), _ptr(T), _ptr(C), lda, _ptr(W2), k, st), "wy_top")
                ev_top = torch.cuda.Event()
                ev_top.record()
                bulk.wait_event(ev_top)
                _check(L.bqrrp_step_wy_bulk(h, k, t_loc, _ptr(V), _ptr(W2), k, _ptr(C), lda,
                                            ctypes.c_void_p(bulk.cuda_stream)), "wy_bulk")
                V.record_stream(bulk)
                W2.record_stream(bulk)
                pending = torch.cuda.Event()
                pending.record(bulk)
        if k < kmax or c == n or r == m:
            ell = s + k
            break
        # ---- a6: R11 and R12 (k x t, position order) assembled on every rank, replicated sketch update
        dist.broadcast(_dense(R11), src=owner, group=group)
        t = n - c
        j_c = bc.first_local_at_or_after(c)
        if shard_sketch:
            # this rank's sketch rows only (its own R12 columns are local), then every rank's rows all-gathered
            # so the next (replicated) pivot selection sees the whole updated sketch
            pos_off, col_off, lens = [], [], []
            for q0 in bc.own_blocks_from(c):
                pos_off.append(q0 - c)
                col_off.append(int(bc.loc_of[q0]) - j_c)
                lens.append(min(b, n - q0))
            arrs = [np.ascontiguousarray(x, dtype=np.int64) for x in (pos_off, col_off, lens)]
            _check(L.bqrrp_step_sample_update_rows(b, _ptr(R11), b, _ptr(A_loc[s:s + k, j_c:] if bc.n_loc > j_c
                                                                          else A_loc), lda, _ptr(MskT[s:]), n,
                                                   *[a_.ctypes.data_as(ctypes.c_void_p) for a_ in arrs], len(lens),
                                                   st), "sample_update_rows")
            _allgather_sketch_rows(MskT, c, n, d, b, bc, me, G, group, colmaj, dev)
            i += 1
            continue
        if use_a2a:
            # X1 as an all-gather of every rank's own R12 columns (padded to the largest share), then one
            # gather into position order: each column crosses the fabric once (the exact-sum all-reduce
            # moves the whole k x t block twice)
            q_own = bc.owner_of[c:n]
            counts = np.bincount(q_own, minlength=G)
            cmax = int(counts.max())
            loc = colmaj(k, cmax)
            if bc.n_loc - j_c > 0:
                loc[:, : bc.n_loc - j_c] = A_loc[s:s + k, j_c:]
            gathered = colmaj(k, G * cmax)
            dist.all_gather_into_tensor(gathered.t().reshape(-1), loc.t().reshape(-1), group=group)
            rank_in = np.zeros(n - c, dtype=np.int64)  # index of position c+u among its owner's positions >= c
            for g_ in range(G):
                sel = q_own == g_
                rank_in[sel] = np.arange(int(sel.sum()))
            idx = torch.as_tensor((q_own * cmax + rank_in).astype(np.int32), device=dev)
            R12 = colmaj(k, t)
            _check(L.bqrrp_step_gather_columns(k, _ptr(gathered), k, _ptr(idx), t, _ptr(R12), k, st), "gather R12")
        else:
            R12 = colmaj(k, t)
            if bc.n_loc - j_c > 0:
                slots = torch.as_tensor(bc.pos[j_c:] - c, device=dev)
                R12[:, slots] = A_loc[s:s + k, j_c:]
            allreduce_sum(R12)
        _check(L.bqrrp_step_sample_update(b, t, _ptr(R11), b, _ptr(R12), k, _ptr(MskT[s:]), n, st), "sample_update")
        i += 1
    if pending is not None:
        torch.cuda.current_stream().wait_event(pending)
    # ---- O4: tau(ell:) = 0, A(ell:m, ell:n) = 0 on the columns this rank owns
    if ell < mn:
        tau[ell:mn] = 0.0
    j_l = bc.first_local_at_or_after(ell)
    if ell < m and bc.n_loc - j_l > 0:
        _check(L.bqrrp_step_zero(m - ell, bc.n_loc - j_l, _ptr(A_loc[ell:, j_l:]), lda, st), "zero")
    torch.cuda.current_stream().synchronize()
    return A_loc, tau[:mn], J, ell
