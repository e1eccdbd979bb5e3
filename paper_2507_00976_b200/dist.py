"""Multi-GPU BQRRP: a thin binding of the C-ABI entry
``bqrrp_factor_dist`` (paper_2507_00976_b200/csrc/dist.cu).

The whole distributed factorization — the block-cyclic loop, its host syncs, the exchange plans and every
collective — runs inside libbqrrp.so.  This module only marshals arguments and sets up the communicator:

* ``comm_nccl(group)``: rank 0 draws an NCCL unique id (``bqrrp_nccl_unique_id``), torch.distributed broadcasts
  the 128 bytes, every rank joins with ``bqrrp_comm_init`` (one process per GPU).
* ``comm_torch(group)``: a ``bqrrp_transport`` whose callbacks run torch.distributed collectives (gloo in the
  tests, where several ranks share one GPU); the library synchronises its stream before each callback.

A is distributed 1-D block-cyclically over column POSITIONS (block width nb = dist_nb, default b): position p
lives on rank (p // nb) % G.  ``local_columns`` cuts a rank's share out of a full matrix.
"""
from __future__ import annotations

import ctypes

import numpy as np

from . import Options, _check, _options, _stream_ptr, default_rank_tol, lib  # noqa: F401

__all__ = ["BlockCyclic", "local_columns", "comm_nccl", "comm_torch", "Comm", "factor_dist", "exchange_plan",
           "SHARD_PANEL"]

SHARD_PANEL = 1  # bqrrp_options.dist_flags: BQRRP_DIST_SHARD_PANEL

_SZ = ctypes.c_size_t
_AR = ctypes.CFUNCTYPE(ctypes.c_int, ctypes.c_void_p, ctypes.c_void_p, _SZ, ctypes.c_void_p)
_AG = ctypes.CFUNCTYPE(ctypes.c_int, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p, _SZ, ctypes.c_void_p)
_BC = ctypes.CFUNCTYPE(ctypes.c_int, ctypes.c_void_p, ctypes.c_void_p, _SZ, ctypes.c_int, ctypes.c_void_p)
_A2A = ctypes.CFUNCTYPE(ctypes.c_int, ctypes.c_void_p, ctypes.c_void_p, ctypes.POINTER(_SZ), ctypes.POINTER(_SZ),
                        ctypes.c_void_p, ctypes.POINTER(_SZ), ctypes.POINTER(_SZ), ctypes.c_void_p)


class _Transport(ctypes.Structure):
    _fields_ = [("ctx", ctypes.c_void_p), ("rank", ctypes.c_int), ("nranks", ctypes.c_int),
                ("allreduce_sum_f64", _AR), ("allgather", _AG), ("broadcast", _BC), ("alltoallv", _A2A)]


def _declare():
    L = lib()
    if getattr(L, "_dist_declared", False):
        return L
    i64, P, i32 = ctypes.c_int64, ctypes.c_void_p, ctypes.c_int
    L.bqrrp_nccl_unique_id.argtypes = [P]
    L.bqrrp_comm_init.argtypes = [P, i32, i32, ctypes.POINTER(P)]
    L.bqrrp_comm_init_transport.argtypes = [ctypes.POINTER(_Transport), ctypes.POINTER(P)]
    L.bqrrp_comm_destroy.argtypes = [P]
    L.bqrrp_dist_local_columns.argtypes = [i64, i64, i32, i32, ctypes.POINTER(i64)]
    L.bqrrp_workspace_query_dist.argtypes = [i64, i64, i64, i64, i32, i64, ctypes.POINTER(_SZ)]
    L.bqrrp_dist_exchange_plan.argtypes = [i64, i64, i32, i32, i64, P, P, P, P, P, P, P, P, ctypes.POINTER(i64)]
    L.bqrrp_factor_dist.argtypes = [i64, i64, P, i64, i64, i64, ctypes.c_uint64, P, P, ctypes.POINTER(i64), P, P, _SZ,
                                    P, ctypes.POINTER(Options)]
    L._dist_declared = True
    return L


class BlockCyclic:
    """1-D block-cyclic map of n column positions over G ranks with block width nb (the library's layout)."""

    def __init__(self, n: int, nb: int, G: int, rank: int):
        self.n, self.nb, self.G, self.rank = n, nb, G, rank
        p = np.arange(n)
        self.owner_of = (p // nb) % G
        self.pos = p[self.owner_of == rank]  # this rank's positions, ascending = its local column order

    @property
    def n_loc(self) -> int:
        return len(self.pos)


def local_columns(A, nb: int, G: int, rank: int):
    """This rank's block-cyclic columns of a full column-major tensor (for tests and the bench)."""
    import torch

    bc = BlockCyclic(A.shape[1], nb, G, rank)
    idx = torch.as_tensor(bc.pos, device=A.device)
    loc = A.index_select(1, idx)
    return loc.t().contiguous().t(), bc


def exchange_plan(n: int, nb: int, G: int, rank: int, q, p):
    """The a3 exchange plan of one rank (bqrrp_dist_exchange_plan; host only, no GPU needed)."""
    L = _declare()
    q = np.ascontiguousarray(q, dtype=np.int64)
    p = np.ascontiguousarray(p, dtype=np.int64)
    nt = len(q)
    out = {k: np.zeros(max(nt, 1), dtype=np.int32) for k in ("send", "recv", "lsrc", "ldst")}
    sc = np.zeros(G, dtype=np.int64)
    rc = np.zeros(G, dtype=np.int64)
    nl = ctypes.c_int64(0)
    P_ = lambda a: a.ctypes.data_as(ctypes.c_void_p)  # noqa: E731
    _check(L.bqrrp_dist_exchange_plan(n, nb, G, rank, nt, P_(q), P_(p), P_(out["send"]), P_(sc), P_(out["recv"]),
                                      P_(rc), P_(out["lsrc"]), P_(out["ldst"]), ctypes.byref(nl)),
           "bqrrp_dist_exchange_plan")
    return dict(send_idx=out["send"][: sc.sum()], send_counts=sc, recv_idx=out["recv"][: rc.sum()], recv_counts=rc,
                local_src=out["lsrc"][: nl.value], local_dst=out["ldst"][: nl.value])


class Comm:
    """An opaque bqrrp communicator (bqrrp_comm_init / bqrrp_comm_init_transport); destroy() releases it."""

    def __init__(self, handle, keep=None, rank=0, size=1):
        self.handle, self._keep, self.rank, self.size = handle, keep, rank, size

    def destroy(self):
        if self.handle:
            _check(_declare().bqrrp_comm_destroy(self.handle), "bqrrp_comm_destroy")
            self.handle = None

    def __del__(self):
        try:
            self.destroy()
        except Exception:
            pass


def comm_nccl(group=None) -> Comm:
    """NCCL clique over the ranks of a torch.distributed group (one process per GPU)."""
    import torch
    import torch.distributed as dist

    L = _declare()
    rank, size = dist.get_rank(group), dist.get_world_size(group)
    uid = torch.zeros(128, dtype=torch.uint8)
    if rank == 0:
        buf = (ctypes.c_uint8 * 128)()
        _check(L.bqrrp_nccl_unique_id(ctypes.cast(buf, ctypes.c_void_p)), "bqrrp_nccl_unique_id")
        uid = torch.tensor(list(bytes(buf)), dtype=torch.uint8)
    holder = [uid]
    dist.broadcast_object_list(holder, src=dist.get_global_rank(group, 0) if group is not None else 0, group=group)
    raw = (ctypes.c_uint8 * 128)(*holder[0].tolist())
    h = ctypes.c_void_p()
    _check(L.bqrrp_comm_init(ctypes.cast(raw, ctypes.c_void_p), rank, size, ctypes.byref(h)), "bqrrp_comm_init")
    return Comm(h, rank=rank, size=size)


class _Raw:
    """A raw device buffer as a torch tensor (no copy) through __cuda_array_interface__."""

    def __init__(self, ptr: int, nbytes: int):
        self.__cuda_array_interface__ = {"shape": (nbytes,), "typestr": "|u1", "data": (ptr, False), "version": 3}


def comm_torch(group=None) -> Comm:
    """bqrrp_transport over torch.distributed collectives (any backend that handles CUDA tensors: gloo in the
    single-GPU tests, where the ranks share one device)."""
    import torch
    import torch.distributed as dist

    L = _declare()
    rank, size = dist.get_rank(group), dist.get_world_size(group)

    def dev(ptr, nbytes):
        return torch.as_tensor(_Raw(ptr, nbytes), device="cuda")

    def guard(f):
        def w(*a):
            try:
                f(*a)
                torch.cuda.synchronize()
                return 0
            except Exception as e:  # reported as the transport's status -> BQRRP_ENCCL
                print(f"bqrrp transport callback failed: {e!r}")
                return 1
        return w

    @guard
    def allreduce(ctx, buf, count, stream):
        t = dev(buf, count * 8).view(torch.float64)
        dist.all_reduce(t, group=group)

    @guard
    def allgather(ctx, send, recv, nbytes, stream):
        dist.all_gather_into_tensor(dev(recv, nbytes * size), dev(send, nbytes).clone(), group=group)

    @guard
    def broadcast(ctx, buf, nbytes, root, stream):
        src = dist.get_global_rank(group, root) if group is not None else root
        dist.broadcast(dev(buf, nbytes), src=src, group=group)

    @guard
    def alltoallv(ctx, send, scount, sdispl, recv, rcount, rdispl, stream):
        sc = [int(scount[r]) for r in range(size)]
        rc = [int(rcount[r]) for r in range(size)]
        parts = [dev(send + int(sdispl[r]), sc[r]) for r in range(size) if sc[r]]
        sbuf = torch.cat(parts) if parts else torch.zeros(0, dtype=torch.uint8, device="cuda")
        rbuf = torch.zeros(sum(rc), dtype=torch.uint8, device="cuda")
        dist.all_to_all_single(rbuf, sbuf, rc, sc, group=group)
        off = 0
        for r in range(size):
            if rc[r]:
                dev(recv + int(rdispl[r]), rc[r]).copy_(rbuf[off:off + rc[r]])
                off += rc[r]

    cbs = (_AR(allreduce), _AG(allgather), _BC(broadcast), _A2A(alltoallv))
    tr = _Transport(None, rank, size, *cbs)
    h = ctypes.c_void_p()
    _check(L.bqrrp_comm_init_transport(ctypes.byref(tr), ctypes.byref(h)), "bqrrp_comm_init_transport")
    return Comm(h, keep=(cbs, tr), rank=rank, size=size)


def factor_dist(A_loc, m: int, n: int, b: int, d: int | None = None, seed: int = 0, rank_tol: float | None = None,
                cholqr_passes: int = 2, comm: Comm | None = None, lookahead: bool = True, shard_panel: bool = False,
                dist_nb: int = 0, stream=None, hqr_fallback: bool = True, phase_times: bool = False):
    """Distributed BQRRP (bqrrp_factor_dist).  A_loc: this rank's block-cyclic columns (m x n_loc, column-major
    float64 CUDA).  Returns (A_loc, tau, J, rank) with A_loc overwritten in GEQP3 format in this rank's columns,
    tau (min(m, n)) and J (n, one-based) replicated.  shard_panel: the row-sharded panel (else the owner's panel:
    bitwise the one-GPU result)."""
    import torch

    from . import PHASES, _require_fortran_f64_cuda

    L = _declare()
    if comm is None:
        raise ValueError("factor_dist needs a communicator: comm_nccl(group) or comm_torch(group)")
    d = b if d is None else d
    lda = _require_fortran_f64_cuda(A_loc) if A_loc.numel() else max(m, 1)
    mn = min(m, n)
    tau = torch.empty(max(mn, 1), dtype=torch.float64, device=A_loc.device)
    J = torch.empty(max(n, 1), dtype=torch.int64, device=A_loc.device)
    rank = ctypes.c_int64(0)
    phases = (ctypes.c_float * len(PHASES))() if phase_times else None
    opts = _options(rank_tol, cholqr_passes, phases, hqr_fallback, lookahead, False, dist_nb)
    opts.dist_flags = SHARD_PANEL if shard_panel else 0
    st = L.bqrrp_factor_dist(m, n, ctypes.c_void_p(A_loc.data_ptr()) if A_loc.numel() else None, lda, b, d, seed,
                             ctypes.c_void_p(tau.data_ptr()), ctypes.c_void_p(J.data_ptr()), ctypes.byref(rank),
                             comm.handle, None, 0, _stream_ptr(stream), ctypes.byref(opts))
    _check(st, "bqrrp_factor_dist")
    out = (A_loc, tau[:mn], J[:n], int(rank.value))
    if phase_times:
        out = out + ({k: float(phases[i]) for i, k in enumerate(PHASES)},)
    return out
