"""Multi-GPU BQRRP driver (paper_2507_00976_b200/dist.py).

CPU part: the block-cyclic position map.  GPU part: two ranks sharing the one B200 of the test box (gloo
process group, whose all-reduce / broadcast accept CUDA tensors) run the distributed factorization and
must reproduce the single-GPU factorization: same J and rank, R / V / tau to rounding (1e-12), zeros past
the rank — the column exchange, the panel broadcast and the replicated sketch update all exercised.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.multiprocessing as mp


def test_block_cyclic_map():
    from paper_2507_00976_b200.dist import BlockCyclic

    n, nb, G = 23, 4, 3
    maps = [BlockCyclic(n, nb, G, r) for r in range(G)]
    allpos = np.sort(np.concatenate([mp_.pos for mp_ in maps]))
    assert np.array_equal(allpos, np.arange(n))  # a partition of the positions
    for r, bc in enumerate(maps):
        assert np.all((bc.pos // nb) % G == r)
        assert np.array_equal(bc.loc_of[bc.pos], np.arange(bc.n_loc))
        for p in range(n + 1):  # local suffix of positions >= p is contiguous
            j = bc.first_local_at_or_after(p)
            assert np.all(bc.pos[j:] >= p) and np.all(bc.pos[:j] < p)
        for p in range(0, n, nb):  # the row blocks the row-distributed sketch computes and all-gathers
            blocks = bc.own_blocks_from(p)
            covered = np.concatenate([np.arange(q0, min(q0 + nb, n)) for q0 in blocks]) if blocks else np.arange(0)
            assert np.array_equal(covered, bc.pos[bc.first_local_at_or_after(p):])
    for p in range(0, n, nb):  # every position >= p is in exactly one rank's blocks
        union = np.sort(np.concatenate([np.arange(q0, min(q0 + nb, n)) for bc in maps for q0 in bc.own_blocks_from(p)]))
        assert np.array_equal(union, np.arange(p, n))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _require_contiguous_collectives(dist):
    """NCCL rejects non-contiguous tensors ("Tensors must be contiguous"); gloo does not.  The tests run on gloo,
    so make every collective the driver issues check it, as NCCL would."""
    def wrap(fn):
        def checked(*args, **kw):
            for a in list(args) + list(kw.values()):
                if hasattr(a, "is_contiguous") and hasattr(a, "is_cuda"):
                    assert a.is_contiguous(), f"{fn.__name__}: non-contiguous tensor {tuple(a.shape)} {a.stride()}"
            return fn(*args, **kw)
        return checked

    for name in ("broadcast", "all_reduce", "all_gather_into_tensor", "all_to_all_single"):
        setattr(dist, name, wrap(getattr(dist, name)))


def _worker(rank, world, port, m, n, b, d, seed, gen, out, exchange="allreduce", lookahead=True, shard=True):
    import torch.distributed as dist

    import inputs
    import paper_2507_00976_b200 as bq
    from paper_2507_00976_b200.dist import factor_dist, local_columns

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    _require_contiguous_collectives(dist)
    try:
        A = inputs.low_rank(m, n, gen, seed=seed) if gen else inputs.gaussian(m, n, seed=seed)
        Ad = torch.tensor(np.ascontiguousarray(A.T), device="cuda").t()
        A_loc, bc = local_columns(Ad, b, world, rank)
        A_loc, tau, J, ell = factor_dist(A_loc, m, n, b, d, seed=seed + 1, exchange=exchange, lookahead=lookahead,
                                         shard_panel=shard, shard_sketch=shard)
        full = torch.zeros((n, m), dtype=torch.float64, device="cuda").t()
        full[:, torch.as_tensor(bc.pos, device="cuda")] = A_loc
        dist.all_reduce(full.t())  # the contiguous storage behind the column-major view
        if rank == 0:
            Ar, taur, Jr, ellr = bq.factor(Ad.clone().t().contiguous().t(), b, d, seed=seed + 1)
            same_j = bool(torch.equal(J, Jr))
            l = ellr
            prefix_j = bool(torch.equal(J[:l], Jr[:l]))
            Rg, Rr = torch.triu(full)[:l], torch.triu(Ar)[:l]
            if not same_j:  # rank-deficient: J(l:) is decided on rounding noise; compare by column index
                Rg, Rr = Rg[:, torch.argsort(J)], Rr[:, torch.argsort(Jr)]
            Vg, Vr = torch.tril(full[:, :l], -1), torch.tril(Ar[:, :l], -1)
            out["res"] = dict(
                ell=ell, ellr=ellr, same_j=same_j, prefix_j=prefix_j, gen=gen,
                dR=float(torch.linalg.norm(Rg - Rr) / torch.linalg.norm(Rr)),
                dV=float(torch.linalg.norm(Vg - Vr) / max(float(torch.linalg.norm(Vr)), 1.0)),
                dtau=float((tau - taur).abs().max()) if len(tau) else 0.0,
                tail_zero=bool((full[l:, l:] == 0).all()),
                bitwise=bool(torch.equal(full, Ar)))
    finally:
        dist.barrier()
        dist.destroy_process_group()


@pytest.mark.gpu
@pytest.mark.parametrize("m,n,b,d,gen", [(1024, 1024, 128, 160, 0), (700, 450, 64, 80, 0), (512, 768, 64, 64, 0),
                                         (512, 512, 64, 80, 150)])
@pytest.mark.parametrize("world", [2, 3])
@pytest.mark.parametrize("exchange,lookahead,shard", [("allreduce", True, False), ("a2a", True, True),
                                                     ("a2a", False, True), ("allreduce", False, False)])
def test_dist_matches_single_gpu(gpu, m, n, b, d, gen, world, exchange, lookahead, shard):
    """The distributed factorization equals the single-GPU one, for both column-exchange forms (X3 as an
    exact-sum all-reduce, or point-to-point all_to_all moves as used on NCCL), with / without the lookahead,
    and with the panel on its owner or row-sharded over the ranks (shard also restricts the R_sk GEMM and the
    sample update to each rank's positions, with the sketch rows all-gathered)."""
    port = _free_port()
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_worker, args=(world, port, m, n, b, d, 5, gen, out, exchange, lookahead, shard), nprocs=world,
             join=True)
    r = out["res"]
    assert r["ell"] == r["ellr"]
    assert r["same_j"] if not gen else r["prefix_j"]
    assert r["dR"] <= 1e-12 and r["dV"] <= 1e-12 and r["dtau"] <= 1e-12, r
    assert r["tail_zero"]


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
