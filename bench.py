#!/usr/bin/env python
"""bench.py — effective FP64 TFLOP/s of BQRRP (GEQRF flop count 2mn^2 - 2n^3/3) on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config C2] [--impl ours|reference]

Default workload: C3 (65536 x 65536, b = d = 2048), the configuration the metric is quoted on.
One step = one full BQRRP factorization (all hot-path rows a1-a7: sketch, LU/QR pivot selection,
touched-set permutation, CholQR2 panel + reconstruction, WY trailing update, sketch update) of the
config's synthetic matrix, inputs resident in HBM.  A is restored from a pristine device copy before
every step OUTSIDE the timed events (the factorization is in place); each step is timed with CUDA events
on the library's stream; the K step times are summed.  Inputs (34 GB at C3) are larger than L2.

N > 1 (torchrun): ONE distributed factorization of the same matrix (dist.py: 1-D block-cyclic columns,
replicated sketch, NCCL exchanges; "scaling": "strong" — the N = 1 line is the same fixed workload, so it
says "strong" too).  value = canonical flops of the one matrix / max-over-ranks time.  --replicas: each
rank factors its own matrix instead ("scaling": "weak", value = flops of all ranks / max-over-ranks time).

--impl reference: the reference arm of this tier is the plain CPU oracle (oracle/), timed on the host
cores, each step a bounded sample of the workload (rank 0 only).
"""
from __future__ import annotations

import argparse
import datetime
import json
import os
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "fp64 BQRRP effective TFLOP/s (GEQRF flops) at 1/2/4/8 B200, % FP64 TC peak"

# BASELINE.json configs.  The metric ("... at 1/2/4/8 B200") is quoted on configs[2] =
# C3 (65536^2, the north-star target, "block-column sharded at 1/2/4/8 B200"); it fits one B200
# (34 GB), so C3 is the default N=1 workload.  C1/C2/C4 are parity/secondary cases (--config).
CONFIGS = {
    "C1": dict(m=1024, n=1024, b=128, d=160, desc="1024x1024 fp64 Gaussian, b=128, d=1.25b=160, seed 0"),
    "C2": dict(m=16384, n=16384, b=1024, d=1024, desc="16384x16384 fp64 Gaussian, b=1024, d=b, seed 0"),
    "C3": dict(m=65536, n=65536, b=2048, d=2048, desc="65536x65536 fp64 Gaussian, b=2048, d=b, seed 0"),
    "C4": dict(m=262144, n=8192, b=512, d=512, desc="262144x8192 tall fp64 Gaussian, b=512, d=b, seed 0"),
}
# CPU-oracle sample per config (a bounded piece of the same workload: same generator, same b and d)
ORACLE_SAMPLE = {"C1": (1024, 1024), "C2": (4096, 4096), "C3": (4096, 4096), "C4": (16384, 1024)}

PEAKS_FILE = os.path.join(ROOT, "profiles", "fp64_peak_r01.json")
NCU_SUMMARY = os.path.join(ROOT, "profiles", "r02", "ncu_summary_r02.json")


def canonical_flops(m: int, n: int) -> float:
    """BASELINE.json's GEQRF count 2 m n^2 - 2 n^3 / 3 (m >= n; mirrored for wide)."""
    if m < n:
        m, n = n, m
    return 2.0 * m * n * n - 2.0 * n ** 3 / 3.0


def trailing_update_flops(m: int, n: int, b: int) -> float:
    """Algorithmic flops of the a5 compact-WY update over a full-rank run: per
    iteration GEMM1 2hkt + the TRMM W2 = T^T W k^2 t (T triangular; the kernel skips the zero half) + GEMM2
    2hkt (h = m-s, k = b, t = n-s-k)."""
    tot = 0.0
    s = 0
    mn = min(m, n)
    while s < mn:
        k = min(b, mn - s)
        h, t = m - s, n - s - k
        if t > 0:
            tot += 4.0 * h * k * t + 1.0 * k * k * t
        s += b
    return tot


def peak_fp64() -> tuple[float, str]:
    try:
        d = json.load(open(PEAKS_FILE))
        return float(d["dmma_tflops"]), "measured DMMA.8x8x4 issue rate, profiles/fp64_peak_r01.json"
    except Exception:
        return 37.2, "spec 148 SM x 128 flop/clk x 1.965 GHz (no measurement file)"


# ------------------------------------------------------------------------------------- clocks
class ClockSampler:
    """nvidia-smi clocks + throttle reasons during the timed region (B200_PROFILING.md clocks line)."""

    REASONS = {0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap", 0x8: "hw_slowdown",
               0x10: "sync_boost", 0x20: "sw_thermal_slowdown", 0x40: "hw_thermal_slowdown",
               0x80: "hw_power_brake_slowdown", 0x100: "display_clock_setting"}

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.first = ""
        self.t0 = self.t1 = None

    def __enter__(self):
        # nvidia-smi is started and its first sample read BEFORE the timed region begins: its NVML initialisation
        # stalls CUDA submissions for tens of ms (measured: a C2 step 377 ms with the sampler starting inside the
        # timed region vs 360 ms without).  Samples are kept by timestamp: only those taken inside the region.
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index),
                 "--query-gpu=timestamp,clocks.sm,clocks.max.sm,clocks_event_reasons.active",
                 "--format=csv,noheader,nounits", "-lms", "200"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.first = self.proc.stdout.readline()  # blocks until NVML is up and the first sample is out
        except Exception:
            self.proc = None
        time.sleep(0.3)  # let the sampler settle into its 200 ms loop
        self.t0 = time.time()
        return self

    def __exit__(self, *a):
        self.t1 = time.time()
        self.out = ""
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.out, _ = self.proc.communicate(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        sm, mx, reasons = [], 0.0, set()
        for line in (self.out or "").splitlines():
            p = [x.strip() for x in line.split(",")]
            if len(p) < 4:
                continue
            try:
                ts = datetime.datetime.strptime(p[0], "%Y/%m/%d %H:%M:%S.%f").timestamp()
                if self.t0 is not None and not (self.t0 - 0.25 <= ts <= self.t1 + 0.25):
                    continue  # outside the timed region
                smv, mxv, bits = float(p[1]), float(p[2]), int(p[3], 16)
            except ValueError:
                continue
            sm.append(smv)
            mx = max(mx, mxv)
            for bit, name in self.REASONS.items():
                if bits & bit and name != "gpu_idle":
                    reasons.add(name)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"], "samples": 0}
        sm.sort()
        return {"sm_mhz": sm[len(sm) // 2], "sm_max_mhz": mx, "reasons": sorted(reasons), "samples": len(sm)}


# ------------------------------------------------------------------------------------- HBM paths
def hbm_peak() -> tuple[float, str]:
    try:
        return float(json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"]), "MEASURED_PEAKS.json hbm_gbs"
    except Exception:
        return 6550.0, "B200_PROFILING.md fallback"


def hbm_paths(bq, A0, A, m: int, n: int, d: int, stream, reps: int = 3) -> dict:
    """GB/s of the HBM-bound kernels on the bench workload's own buffers, outside the timed region (SURVEY §8(d.2),
    north_star "HBM GB/s for the permutation and norm paths"): each kernel timed alone with CUDA events on the
    stream it runs on (best of `reps` after one warm launch); algorithmic bytes = what the operation must move.
      K-NORM columns: ||A0(:, j)||, every column of the pristine input (reads m n 8 B);
      K-NORM trailing: ||R(i:, i:)||_F of the factorization just computed (reads the upper trapezoid once);
      K-PERM: the a3 touched-set move (gather to scratch + scatter back) of 2d columns of A, the C3 iteration-0
              touched-set size, random positions (reads + writes 2 x 2d x m x 8 B)."""
    import torch

    peak, src = hbm_peak()
    mn = min(m, n)
    out = {"peak_gbs": peak, "peak_source": src}

    def timed(fn):
        fn()
        best = None
        for _ in range(reps):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            fn()
            e1.record(stream)
            torch.cuda.synchronize()
            t = e0.elapsed_time(e1)
            best = t if best is None else min(best, t)
        return best

    norms = torch.empty(n, dtype=torch.float64, device=A0.device)
    t = timed(lambda: bq.column_norms(A0, out=norms, stream=stream))
    byts = m * n * 8
    out["k_norm_columns"] = {"ms": t, "bytes": byts, "gbs": byts / t / 1e6, "frac": byts / t / 1e6 / peak,
                             "kernel": "col_norms_kernel"}
    tn = torch.empty(mn, dtype=torch.float64, device=A0.device)
    ws = torch.empty(bq.trailing_norms_workspace(m, n), dtype=torch.uint8, device=A0.device)
    t = timed(lambda: bq.trailing_norms(A, out=tn, workspace=ws, stream=stream))
    byts = (n * mn - mn * (mn - 1) // 2) * 8
    out["k_norm_trailing"] = {"ms": t, "bytes": byts, "gbs": byts / t / 1e6, "frac": byts / t / 1e6 / peak,
                              "kernel": "trailing_rows_kernel + rowsum + scan (3 launches)"}
    nt = min(2 * d, n)
    g = torch.Generator().manual_seed(5)
    tq = torch.randperm(n, generator=g)[:nt].to(torch.int32)
    tsrc = tq[torch.randperm(nt, generator=g)]
    tq, tsrc = tq.to(A.device), tsrc.to(A.device)
    t = timed(lambda: bq.debug_permute_touched(A, tq, tsrc, stream=stream))
    byts = 4 * nt * m * 8
    out["k_perm"] = {"ms": t, "bytes": byts, "gbs": byts / t / 1e6, "frac": byts / t / 1e6 / peak, "columns": nt,
                     "kernel": "gather_cols_kernel + scatter_cols_kernel (16-byte copies)"}
    return out


# ------------------------------------------------------------------------------------- multi-rank
def max_over_ranks(value: float, device=None) -> float:
    """The contract's multi-GPU timing rule: every rank times itself on its device; the job time is the
    max over ranks (all_reduce MAX).  Works on any backend (NCCL on the GPU box, gloo in the CPU tests)."""
    import torch
    import torch.distributed as dist

    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size() == 1:
        return float(value)
    t = torch.tensor([float(value)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def aggregate_value(flops_per_step_per_rank: float, steps: int, world: int, t_ms_max: float) -> float:
    """Whole-job TFLOP/s: the flops of all ranks over the max-over-ranks device time."""
    return flops_per_step_per_rank * steps * world / (t_ms_max * 1e-3) / 1e12


# ------------------------------------------------------------------------------------- oracle timing
def oracle_sample(cfg_name: str, seed: int = 0):
    """Time the CPU oracle as it stands on a bounded sample of the workload; returns (TFLOP/s, seconds, desc)."""
    import inputs
    import oracle

    cfg = CONFIGS[cfg_name]
    sm, sn = ORACLE_SAMPLE[cfg_name]
    b, d = min(cfg["b"], sm, sn), min(cfg["d"], sm)
    A = inputs.gaussian(sm, sn, seed=seed)
    t0 = time.perf_counter()
    out = oracle.bqrrp(A, b, d, seed=seed)
    dt = time.perf_counter() - t0
    desc = (f"oracle_bqrrp (plain C, OpenMP over independent columns) on a {sm}x{sn} Gaussian sample "
            f"of the {cfg_name} workload (same generator, b={b}, d={d}); rank {out.rank}; "
            f"canonical GEQRF flops / wall time")
    return canonical_flops(sm, sn) / dt / 1e12, dt, desc


def oracle_plan():
    """The BASELINE.md CPU plan run once by tools/oracle_baseline.py (C1 at 1 thread and all cores, C2 all cores,
    C3 / C4 extrapolated by the algorithmic-flop ratio), summarised from its committed record."""
    path = os.path.join(ROOT, "profiles", "oracle_baseline_r02.json")
    try:
        d = json.load(open(path))
    except Exception:
        return None
    rows = {}
    for r in d["rows"]:
        key = f"{r['config']}_{r['threads']}t" + ("_extrapolated" if r.get("extrapolated") else "")
        rows[key] = {"seconds": round(r["seconds_best"], 3), "tflops": r["tflops_canonical"]}
    return {"record": "profiles/oracle_baseline_r02.json", "cpu": d.get("cpu"), "cores": d.get("cores"), "runs": rows}


def cpu_model() -> str:
    """The host CPU model (for the cpu_baseline record)."""
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    cores = os.cpu_count()
    times = []
    desc = ""
    for it in range(args.warmup + args.steps):
        v, dt, desc = oracle_sample(args.config)
        if it >= args.warmup:
            times.append((v, dt))
    tot_t = sum(t for _, t in times)
    sm, sn = ORACLE_SAMPLE[args.config]
    value = canonical_flops(sm, sn) * len(times) / tot_t / 1e12
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "TFLOP/s", "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * tot_t / max(len(times), 1),
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": args.config + " " + CONFIGS[args.config]["desc"], "sample": f"{sm}x{sn}"},
        "cpu_baseline": {"value": value, "unit": "TFLOP/s", "cores": cores, "kind": "oracle", "sample": desc,
                         "cpu": cpu_model()},
        "e2e": {"value": value, "unit": "TFLOP/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line))
    return 0


# ------------------------------------------------------------------------------------- our arm
def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="C3", choices=sorted(CONFIGS))
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--seed", type=int, default=0)
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--backend", default="nccl", help="process-group backend for N > 1 (gloo: tests)")
    ap.add_argument("--share-gpu", action="store_true", help="all ranks on cuda:0 (gloo tests on a 1-GPU box)")
    ap.add_argument("--replicas", action="store_true",
                    help="N > 1: independent replicas (weak scaling) instead of one distributed factorization")
    args = ap.parse_args()
    if args.impl == "reference":
        return run_reference(args)

    import torch
    import torch.distributed as dist

    import inputs
    import paper_2507_00976_b200 as bq

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = 0 if args.share_gpu else int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    if world > 1:
        if args.backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group(args.backend)
    dev = torch.device("cuda", local)
    stream = torch.cuda.current_stream()

    cfg = CONFIGS[args.config]
    m, n, b, d = cfg["m"], cfg["n"], cfg["b"], cfg["d"]
    if world > 1 and not args.replicas:
        return run_distributed(args, cfg, world, rank, local, dev)
    A0 = inputs.gaussian_cuda(m, n, seed=args.seed + rank, device=dev)  # column-major view
    A = torch.empty_like(A0.t()).t()
    ws = torch.empty(bq.workspace_query(m, n, b, d), dtype=torch.uint8, device=dev)
    tau = torch.empty(min(m, n), dtype=torch.float64, device=dev)
    J = torch.empty(n, dtype=torch.int64, device=dev)

    def step(phase=False):
        return bq.factor(A, b, d, seed=args.seed, workspace=ws, tau=tau, J=J, phase_times=phase)

    for _ in range(args.warmup):
        A.copy_(A0)
        step()
    torch.cuda.synchronize()

    # ---- timed region: K steps, per-step CUDA events (restore outside the events)
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    phases_acc = {}
    launches0 = bq.launch_count()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    with ClockSampler(local) as clk:
        for i in range(args.steps):
            A.copy_(A0)
            ev[i][0].record(stream)
            out = step(phase=True)
            ev[i][1].record(stream)
            for k_, v_ in out[4].items():
                phases_acc[k_] = phases_acc.get(k_, 0.0) + v_
        torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    launches = bq.launch_count() - launches0
    ranks_found = out[3]
    t_ms = max_over_ranks(sum(s.elapsed_time(e) for s, e in ev), dev)
    flops_step = canonical_flops(m, n)
    value = aggregate_value(flops_step, args.steps, world, t_ms)
    peak, peak_src = peak_fp64()

    # ---- roofline of the dominant kernel: the a5 trailing-update DMMA GEMMs (phase apply_trans_q)
    tr_flops = trailing_update_flops(m, n, b)
    # critical-stream part + the bulk GEMM timed on its own stream (it overlaps the next pivot selection)
    apply_ms = (phases_acc.get("apply_trans_q", 0.0) + phases_acc.get("apply_trans_q_bulk", 0.0)) / args.steps
    achieved = tr_flops / (apply_ms * 1e-3) / 1e12 if apply_ms > 0 else None
    traffic, traffic_note = None, None
    try:
        ns = json.load(open(NCU_SUMMARY))
        traffic = ns.get("dgemm_trailing_dram_bytes_per_launch")
        traffic_note = ("dram read+write bytes of ONE launch (the C3 iteration-0 bulk GEMM, ncu --set full, 32-row "
                        "rasterisation groups); its "
                        "algorithmic bytes: %.4g" % ns.get("algorithmic_bytes_per_launch", float("nan")))
    except Exception:
        pass
    roofline = {"bound": "tensor", "achieved": achieved, "peak": peak, "unit": "TFLOP/s",
                "frac": (achieved / peak) if achieved else None, "traffic": traffic, "traffic_note": traffic_note,
                "kernel": "a5 compact-WY trailing update (dgemm2_kernel: W=V^T C, W=T^T W, C-=V W) per factorization; "
                          "the bulk C-=V W rows are timed with events on their own (low-priority) stream",
                "algorithmic_flops_per_step": tr_flops, "kernel_ms_per_step": apply_ms,
                "peak_source": peak_src, "share_of_step": apply_ms / (t_ms / args.steps)}

    hbm = hbm_paths(bq, A0, A, m, n, d, stream) if rank == 0 else None

    # ---- end to end through the C ABI with host buffers (H2D + factor + D2H inside the timed region)
    e2e = None
    if not args.no_e2e:
        A_host0 = torch.empty((n, m), dtype=torch.float64).pin_memory()
        A_host0.copy_(A0.t())
        A_host0 = A_host0.t()  # m x n column-major (pinned)
        A_host = torch.empty((n, m), dtype=torch.float64).pin_memory().t()
        tau_h = torch.empty(min(m, n), dtype=torch.float64).pin_memory()
        J_h = torch.empty(n, dtype=torch.int64).pin_memory()
        ks = 1 if m * n > (1 << 30) else max(1, min(args.steps, 3))
        tot = 0.0
        for i in range(ks + 1):
            A_host.copy_(A_host0)
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            bq.factor_host(A_host, b, d, seed=args.seed, tau_host=tau_h, J_host=J_h)
            e1.record(stream)
            torch.cuda.synchronize()
            if i > 0:
                tot += e0.elapsed_time(e1)
        te = max_over_ranks(tot / ks, dev)
        e2e = {"value": aggregate_value(flops_step, 1, world, te), "unit": "TFLOP/s",
               "h2d_bytes_per_step": m * n * 8, "d2h_bytes_per_step": m * n * 8 + min(m, n) * 8 + n * 8,
               "ms_per_step": te, "api": "bqrrp_factor_host (pinned host buffers)"}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        v, dt, desc = oracle_sample(args.config)
        cpu = {"value": v, "unit": "TFLOP/s", "cores": os.cpu_count(), "kind": "oracle", "sample": desc,
               "cpu": cpu_model(),
               "seconds": dt, "plan": oracle_plan()}

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": "TFLOP/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": t_ms / args.steps, "higher_is_better": True,
            "scaling": "weak" if args.replicas else "strong",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": f"{args.config} {cfg['desc']}", "m": m, "n": n, "b": b, "d": d,
                       "parallelism": "replicas" if world > 1 else "single",
                       "l2": "inputs larger than L2 (A = %.2f GB)" % (m * n * 8 / 1e9),
                       "timing": "per-step CUDA events around bqrrp_factor; A restored from a pristine copy outside the events",
                       "rank_found": ranks_found},
            "pct_fp64_peak": 100.0 * (value / world) / peak,
            "roofline": roofline, "hbm_paths": hbm, "cpu_baseline": cpu, "e2e": e2e, "gpu_launches": launches,
            "clocks": clk.summary(), "phase_ms_per_step": {k_: v_ / args.steps for k_, v_ in phases_acc.items()},
        }
        print(json.dumps(line))
    if world > 1:
        dist.destroy_process_group()
    return 0


def run_distributed(args, cfg, world, rank, local, dev):
    """N > 1: ONE factorization of the config's matrix, 1-D block-cyclic over the ranks (SURVEY §8(e),
    paper_2507_00976_b200/dist.py; NCCL all-reduce / broadcast for the sketch, panel and column exchanges).
    Strong scaling: value = canonical flops of the one matrix / max-over-ranks time."""
    import torch
    import torch.distributed as dist

    import inputs
    import paper_2507_00976_b200 as bq
    from paper_2507_00976_b200.dist import comm_nccl, comm_torch, factor_dist, local_columns

    m, n, b, d = cfg["m"], cfg["n"], cfg["b"], cfg["d"]
    # the library's own communicator: an NCCL clique (bqrrp_comm_init) on the GPU box, a torch.distributed
    # transport for the gloo tests that share one GPU
    comm = comm_nccl() if args.backend == "nccl" else comm_torch()
    stream = torch.cuda.current_stream()
    A_full = inputs.gaussian_cuda(m, n, seed=args.seed, device=dev)  # identical on every rank
    A_loc0, bc = local_columns(A_full, b, world, rank)
    del A_full
    torch.cuda.empty_cache()
    A_loc = torch.empty_like(A_loc0.t()).t()

    def step():
        return factor_dist(A_loc, m, n, b, d, seed=args.seed, comm=comm)

    for _ in range(args.warmup):
        A_loc.copy_(A_loc0)
        step()
    torch.cuda.synchronize()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    launches0 = bq.launch_count()
    dist.barrier()
    torch.cuda.synchronize()
    with ClockSampler(local) as clk:
        for i in range(args.steps):
            A_loc.copy_(A_loc0)
            ev[i][0].record(stream)
            out = step()
            ev[i][1].record(stream)
        torch.cuda.synchronize()
    dist.barrier()
    launches = bq.launch_count() - launches0
    t_ms = max_over_ranks(sum(s_.elapsed_time(e_) for s_, e_ in ev), dev)
    flops_step = canonical_flops(m, n)
    value = aggregate_value(flops_step, args.steps, 1, t_ms)  # one matrix, all ranks
    peak, peak_src = peak_fp64()
    e2e = None
    if not args.no_e2e:  # each rank: its columns host -> device, distributed factorization, back to host
        Ah0 = torch.empty((A_loc0.shape[1], m), dtype=torch.float64).pin_memory()
        Ah0.copy_(A_loc0.t())
        Ah = torch.empty_like(Ah0).pin_memory()
        tau_h = torch.empty(min(m, n), dtype=torch.float64).pin_memory()
        J_h = torch.empty(n, dtype=torch.int64).pin_memory()
        Ah.copy_(Ah0)
        dist.barrier()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        A_loc.t().copy_(Ah, non_blocking=True)
        _, tau, J, _ = step()
        Ah.copy_(A_loc.t(), non_blocking=True)
        tau_h.copy_(tau, non_blocking=True)
        J_h.copy_(J, non_blocking=True)
        e1.record(stream)
        torch.cuda.synchronize()
        te = max_over_ranks(e0.elapsed_time(e1), dev)
        e2e = {"value": aggregate_value(flops_step, 1, 1, te), "unit": "TFLOP/s",
               "h2d_bytes_per_step": m * A_loc0.shape[1] * 8,
               "d2h_bytes_per_step": m * A_loc0.shape[1] * 8 + min(m, n) * 8 + n * 8, "ms_per_step": te,
               "api": "paper_2507_00976_b200.dist.factor_dist (per-rank pinned host columns)"}
    if rank == 0:
        per_gpu = value / world
        line = {
            "metric": METRIC, "value": value, "unit": "TFLOP/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": t_ms / args.steps, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": f"{args.config} {cfg['desc']}", "m": m, "n": n, "b": b, "d": d,
                       "parallelism": f"block-cyclic columns over {world} GPUs (dist_nb = b), bqrrp_factor_dist "
                                      f"({'NCCL' if args.backend == 'nccl' else args.backend})",
                       "l2": "inputs larger than L2", "rank_found": out[3],
                       "timing": "per-step CUDA events around factor_dist, max over ranks"},
            "pct_fp64_peak": 100.0 * per_gpu / peak,
            "roofline": {"bound": "tensor", "achieved": per_gpu, "peak": peak, "unit": "TFLOP/s",
                         "frac": per_gpu / peak, "traffic": None,
                         "kernel": "whole distributed factorization, per GPU (canonical flops / time / N)",
                         "peak_source": peak_src},
            "cpu_baseline": None, "e2e": e2e, "gpu_launches": launches, "clocks": clk.summary(),
        }
        print(json.dumps(line))
    comm.destroy()
    dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
