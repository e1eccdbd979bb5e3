"""Multi-GPU BQRRP (bqrrp_factor_dist, csrc/dist.cu).

CPU part (no GPU): the block-cyclic layout and the a3 exchange plan of the C library, checked against a
direct simulation — and, at world size 2 and 3 over gloo on CPU, by actually moving column ids between processes
with the plans each rank computes.  GPU part: two or three ranks sharing the test box's one B200 (a gloo
transport, bqrrp_comm_init_transport) run the distributed factorization through the C ABI; with the owner panel
and the lookahead (the defaults) the result must be BITWISE the single-GPU factorization (SURVEY §8(e)'s
strongest pin), with the row-sharded panel or without the lookahead J / rank identical and R, V, tau per column
to 1e-12.
"""
import datetime
import os
import socket

import numpy as np
import pytest
import torch
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _lib_local_columns(n, nb, G, r):
    import ctypes

    from paper_2507_00976_b200.dist import _declare

    out = ctypes.c_int64(0)
    assert _declare().bqrrp_dist_local_columns(n, nb, G, r, ctypes.byref(out)) == 0
    return out.value


def test_block_cyclic_layout_matches_library():
    from paper_2507_00976_b200.dist import BlockCyclic

    for n, nb, G in [(23, 4, 3), (64, 8, 2), (5, 8, 4), (100, 3, 7), (0, 2, 2)]:
        maps = [BlockCyclic(n, nb, G, r) for r in range(G)]
        allpos = np.sort(np.concatenate([m.pos for m in maps])) if n else np.zeros(0)
        assert np.array_equal(allpos, np.arange(n))  # a partition of the positions
        for r, bc in enumerate(maps):
            assert np.all((bc.pos // nb) % G == r)
            assert bc.n_loc == _lib_local_columns(n, nb, G, r)


def _simulate_exchange(n, nb, G, q, p):
    """Apply every rank's plan to local arrays of column ids; returns the resulting global position -> id map."""
    from paper_2507_00976_b200.dist import BlockCyclic, exchange_plan

    maps = [BlockCyclic(n, nb, G, r) for r in range(G)]
    local = [m.pos.copy() for m in maps]  # column id = original position
    plans = [exchange_plan(n, nb, G, r, q, p) for r in range(G)]
    sends = {}
    for r, P in enumerate(plans):
        off = 0
        for dst in range(G):
            c = int(P["send_counts"][dst])
            sends[(r, dst)] = local[r][P["send_idx"][off:off + c]].copy()
            off += c
        moved = local[r][P["local_src"]].copy()
        local[r] = local[r].copy()
        local[r][P["local_dst"]] = moved
    for r, P in enumerate(plans):
        off = 0
        for src in range(G):
            c = int(P["recv_counts"][src])
            assert c == len(sends[(src, r)])
            local[r][P["recv_idx"][off:off + c]] = sends[(src, r)]
            off += c
    glob = np.zeros(n, dtype=np.int64)
    for r, m in enumerate(maps):
        glob[m.pos] = local[r]
    return glob


@pytest.mark.parametrize("n,nb,G,nlu", [(40, 4, 2, 10), (97, 8, 3, 30), (64, 16, 4, 16), (33, 5, 2, 33)])
def test_exchange_plan_realises_the_gather(n, nb, G, nlu):
    """The touched-set exchange (gather semantics new(q) = old(J_qr(q) - 1)) realised by the per-rank
    plans equals the global gather, for random LU swap lists."""
    import oracle

    rng = np.random.default_rng(n * G + nlu)
    for _ in range(5):
        s = nb * int(rng.integers(0, max(1, (n // nb) - 1)))
        w = n - s
        k = min(nlu, w)
        ipiv = np.array([rng.integers(j, w) + 1 for j in range(k)], dtype=np.int64)
        Jqr = oracle.piv_transform(w, ipiv)
        qs = np.nonzero(Jqr - 1 != np.arange(w))[0]
        q, p = s + qs, s + (Jqr[qs] - 1)
        glob = _simulate_exchange(n, nb, G, q, p)
        expect = np.arange(n)
        expect[s:] = s + (Jqr - 1)
        assert np.array_equal(glob, expect)


def _cpu_exchange_worker(rank, world, port, n, nb, q, p, out):
    import torch.distributed as dist

    from paper_2507_00976_b200.dist import BlockCyclic, exchange_plan

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        bc = BlockCyclic(n, nb, world, rank)
        P = exchange_plan(n, nb, world, rank, q, p)
        local = torch.as_tensor(bc.pos.copy(), dtype=torch.int64)
        send = local[torch.as_tensor(P["send_idx"], dtype=torch.int64)].clone()
        moved = local[torch.as_tensor(P["local_src"], dtype=torch.int64)].clone()
        recv = torch.zeros(int(P["recv_counts"].sum()), dtype=torch.int64)
        dist.all_to_all_single(recv, send, P["recv_counts"].tolist(), P["send_counts"].tolist())
        local[torch.as_tensor(P["local_dst"], dtype=torch.int64)] = moved
        local[torch.as_tensor(P["recv_idx"], dtype=torch.int64)] = recv
        glob = torch.zeros(n, dtype=torch.int64)
        glob[torch.as_tensor(bc.pos)] = local
        dist.all_reduce(glob)
        if rank == 0:
            out["glob"] = glob.numpy().copy()
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_exchange_plan_over_gloo_cpu(world):
    """The N > 1 column exchange on CPU: world-size 2 / 3 gloo processes move column ids with all_to_all_single
    following the library's plans; the result is the global gather."""
    import oracle

    n, nb = 60, 4
    rng = np.random.default_rng(world)
    s = 8
    w = n - s
    ipiv = np.array([rng.integers(j, w) + 1 for j in range(16)], dtype=np.int64)
    Jqr = oracle.piv_transform(w, ipiv)
    qs = np.nonzero(Jqr - 1 != np.arange(w))[0]
    q, p = s + qs, s + (Jqr[qs] - 1)
    out = mp.Manager().dict()
    mp.spawn(_cpu_exchange_worker, args=(world, _free_port(), n, nb, q, p, out), nprocs=world, join=True)
    expect = np.arange(n)
    expect[s:] = s + (Jqr - 1)
    assert np.array_equal(out["glob"], expect)


# ------------------------------------------------------------------------------------------------ GPU
def _worker(rank, world, port, m, n, b, d, seed, gen, out, lookahead, shard, nb):
    import torch.distributed as dist

    import inputs
    import paper_2507_00976_b200 as bq
    from paper_2507_00976_b200.dist import comm_torch, factor_dist, local_columns

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(0)
    # a short collective timeout: a protocol mismatch between ranks fails the test instead of hanging the suite
    dist.init_process_group("gloo", rank=rank, world_size=world, timeout=datetime.timedelta(seconds=240))
    comm = comm_torch()
    try:
        A = inputs.low_rank(m, n, gen, seed=seed) if gen else inputs.gaussian(m, n, seed=seed)
        Ad = torch.tensor(np.ascontiguousarray(A.T), device="cuda").t()
        A_loc, bc = local_columns(Ad, nb or b, world, rank)
        A_loc, tau, J, ell = factor_dist(A_loc, m, n, b, d, seed=seed + 1, comm=comm, lookahead=lookahead,
                                         shard_panel=shard, dist_nb=nb)
        full = torch.zeros((n, m), dtype=torch.float64, device="cuda").t()
        full[:, torch.as_tensor(bc.pos, device="cuda")] = A_loc
        dist.all_reduce(full.t())  # the contiguous storage behind the column-major view
        if rank == 0:
            # the distributed loop runs K-SQR after K-LU (recursive), as the one-GPU entry with sqr_pipeline=False
            Ar, taur, Jr, ellr = bq.factor(Ad.clone().t().contiguous().t(), b, d, seed=seed + 1, sqr_pipeline=False)
            out["res"] = dict(ell=ell, ellr=ellr, F=full.cpu().numpy(), tau=tau.cpu().numpy(), J=J.cpu().numpy(),
                              Fr=Ar.cpu().numpy(), taur=taur.cpu().numpy(), Jr=Jr.cpu().numpy())
    finally:
        comm.destroy()
        dist.barrier()
        dist.destroy_process_group()


def _run(world, m, n, b, d, gen, lookahead=True, shard=False, nb=0):
    out = mp.Manager().dict()
    mp.spawn(_worker, args=(world, _free_port(), m, n, b, d, 5, gen, out, lookahead, shard, nb), nprocs=world,
             join=True)
    return out["res"]


@pytest.mark.gpu
@pytest.mark.timeout(900)
@pytest.mark.parametrize("m,n,b,d,gen", [(1024, 1024, 128, 160, 0), (700, 450, 64, 80, 0), (512, 768, 64, 64, 0),
                                         (512, 512, 64, 80, 150), (2048, 1024, 256, 256, 0)])
@pytest.mark.parametrize("world", [2, 3])
def test_dist_bitwise_equals_single_gpu(gpu, m, n, b, d, gen, world):
    """Owner panel + lookahead (the defaults): A, tau, J and the rank are bitwise the one-GPU bqrrp_factor's with the
    same K-SQR order (no_sqr_pipeline: the distributed loop factors the sketch after K-LU)."""
    r = _run(world, m, n, b, d, gen)
    assert r["ell"] == r["ellr"]
    assert np.array_equal(r["J"], r["Jr"])
    assert np.array_equal(r["tau"], r["taur"])
    assert np.array_equal(r["F"], r["Fr"]), float(np.abs(r["F"] - r["Fr"]).max())


@pytest.mark.gpu
@pytest.mark.timeout(900)
@pytest.mark.parametrize("m,n,b,d,gen", [(1024, 1024, 128, 160, 0), (700, 450, 64, 80, 0), (512, 512, 64, 80, 150)])
@pytest.mark.parametrize("world", [2, 3])
@pytest.mark.parametrize("lookahead,shard,nb", [(True, True, 0), (False, False, 0), (False, True, 0), (True, False, 2)])
def test_dist_matches_single_gpu(gpu, m, n, b, d, gen, world, lookahead, shard, nb):
    """Row-sharded panel (all-reduced Grams: a different summation order), no lookahead, or a block width
    dist_nb = 2b: J and rank identical (J(:l) for rank-deficient inputs), R / V / tau per column to 1e-12."""
    import _parity

    r = _run(world, m, n, b, d, gen, lookahead, shard, nb * b)
    l = r["ellr"]
    assert r["ell"] == l
    if gen:
        assert np.array_equal(r["J"][:l], r["Jr"][:l])
        Rg = _parity.r_cols(r["F"], l)[:, np.argsort(r["J"])]
        Rr = _parity.r_cols(r["Fr"], l)[:, np.argsort(r["Jr"])]
        _parity.assert_colwise(Rg, Rr, what="R (by original column)")
        _parity.assert_colwise(_parity.v_cols(r["F"], l), _parity.v_cols(r["Fr"], l), what="V")
    else:
        assert np.array_equal(r["J"], r["Jr"])
        _parity.compare_factors(r["F"], r["tau"], r["Fr"], r["taur"], l)
    assert np.all(r["F"][l:, l:] == 0) and np.all(r["tau"][l:] == 0)


@pytest.mark.gpu
def test_bench_distributed_mode_two_ranks_one_gpu(gpu):
    """bench.py's N > 1 path (one distributed factorization, strong scaling) end to end with torchrun,
    two ranks sharing cuda:0 over gloo: one JSON line from rank 0 with the contract's keys."""
    import json
    import subprocess
    import sys

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", str(_free_port()), os.path.join(root, "bench.py"),
           "--gpus", "2", "--steps", "1", "--warmup", "1", "--config", "C1", "--backend", "gloo", "--share-gpu"]
    res = subprocess.run(cmd, capture_output=True, text=True, timeout=600, cwd=root)
    assert res.returncode == 0, res.stderr[-3000:]
    lines = [l for l in res.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and d["scaling"] == "strong" and d["value"] > 0
    assert d["config"]["rank_found"] == 1024
    for key in ("roofline", "e2e", "gpu_launches", "clocks", "ms_per_step"):
        assert key in d
