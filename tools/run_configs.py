"""Run BASELINE configs C4 (262144 x 8192 tall, b = d = 512) and C5 (32768^2 graded spectrum, numerical
rank 8192, b = 1024, d = 1280) on one B200: time, canonical (C4) / truncated (C5) TFLOP/s, and the
property checks of tests/test_gpu_fullsize.py (residual / orthogonality estimators; for C5 the found
rank, the truncated residual and the Eckart-Young / interlacing inequalities of SURVEY P-QUAL at
sampled indices).  Writes profiles/configs_r01.json.

    python tools/run_configs.py [--only C4|C5] [--tols 1e-13,3e-14,1e-14]
"""
import argparse
import json
import math
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

import torch  # noqa: E402

import bench  # noqa: E402
import inputs  # noqa: E402
import paper_2507_00976_b200 as bq  # noqa: E402
from test_gpu_fullsize import _apply_q  # noqa: E402


def timed_factor(A0, b, d, seed=0, rank_tol=None):
    m, n = A0.shape
    A = torch.empty_like(A0.t()).t()
    ws = torch.empty(bq.workspace_query(m, n, b, d), dtype=torch.uint8, device="cuda")
    best = None
    for r in range(2):
        A.copy_(A0)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        out = bq.factor(A, b, d, seed=seed, workspace=ws, rank_tol=rank_tol, phase_times=True)
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1)
        if r == 1:
            best = (ms, out)
    return best


def residual_est(A0, A, tau, J, rank, nvec=2):
    m, n = A0.shape
    g = torch.Generator(device="cuda")
    g.manual_seed(7)
    X = torch.randn((n, nvec), generator=g, device="cuda", dtype=torch.float64)
    AX = A0[:, J - 1] @ X
    R = torch.triu(A[:rank, :])
    Y = torch.zeros((m, nvec), dtype=torch.float64, device="cuda")
    Y[:rank] = R @ X
    QRX = _apply_q(A, tau[:rank], Y)
    return float(torch.linalg.norm(AX - QRX) / torch.linalg.norm(AX))


def graded_cuda(m, n, k, sigma_last=1e-14, seed=0):
    g = torch.Generator(device="cuda")
    g.manual_seed(seed + 2)
    X, _ = torch.linalg.qr(torch.randn((m, k), generator=g, device="cuda", dtype=torch.float64))
    g.manual_seed(seed + 3)
    Y, _ = torch.linalg.qr(torch.randn((n, k), generator=g, device="cuda", dtype=torch.float64))
    sigma = sigma_last ** (torch.arange(k, device="cuda", dtype=torch.float64) / (k - 1))
    A = (X * sigma) @ Y.t()
    return A.t().contiguous().t(), sigma


def run_c4():
    m, n, b, d = 262144, 8192, 512, 512
    A0 = inputs.gaussian_cuda(m, n, seed=0)
    ms, (A, tau, J, rank, ph) = timed_factor(A0, b, d)
    res = residual_est(A0, A, tau, J, rank)
    tf = bench.canonical_flops(m, n) / (ms * 1e-3) / 1e12
    return {"config": "C4 262144x8192 Gaussian b=d=512", "ms": ms, "tflops": tf,
            "pct_p64": 100 * tf / bench.peak_fp64()[0], "rank": rank, "residual_est": res, "phases_ms": ph}


def run_c5(tols):
    m = n = 32768
    k, b, d = 8192, 1024, 1280
    A0, sigma = graded_cuda(m, n, k)
    nrmA = float(torch.linalg.norm(A0))
    out = []
    for tol in tols:
        ms, (A, tau, J, rank, ph) = timed_factor(A0, b, d, rank_tol=tol)
        res = residual_est(A0, A, tau, J, rank)
        # P-QUAL at sampled i: ||R(i:, i:)||_F >= (sum_{j>=i} sigma_j^2)^(1/2) (Eckart-Young);
        # sum_{j<=i} log|R(j,j)| <= sum_{j<=i} log sigma_j (interlacing of the leading products)
        R = torch.triu(A[:rank, :])
        quals = []
        for i in [0, 1024, 4096, 6000, min(rank - 1, 7500)]:
            if i >= rank:
                continue
            trail = float(torch.linalg.norm(R[i:, i:]))
            opt = float(torch.sqrt(torch.sum(sigma[i:] ** 2)))
            logdiag = float(torch.sum(torch.log(torch.abs(torch.diagonal(R)[: i + 1]))))
            logsig = float(torch.sum(torch.log(sigma[: i + 1])))
            quals.append({"i": i, "trail_R": trail, "trail_opt": opt, "ratio": trail / opt if opt > 0 else None,
                          "eckart_young_ok": trail >= opt * (1 - 1e-12), "sum_log_diag": logdiag,
                          "sum_log_sigma": logsig, "interlacing_ok": logdiag <= logsig + 1e-9})
        fl = 4.0 * m * n * rank - 2.0 * (m + n) * rank ** 2 + 4.0 * rank ** 3 / 3.0  # truncated count (SURVEY d.3)
        out.append({"config": "C5 32768^2 graded sigma_i = 1e-14^(i/8191), rank 8192, b=1024 d=1280",
                    "rank_tol": tol, "rank": rank, "ms": ms, "truncated_tflops": fl / (ms * 1e-3) / 1e12,
                    "truncated_residual_est": res, "norm_A": nrmA, "quality": quals, "phases_ms": ph})
        print(json.dumps(out[-1]), flush=True)
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--only", default="")
    ap.add_argument("--tols", default="2.01e-14", help="C5 rank_tol values; default alpha = 1 (alpha u sqrt(n), the "
                    "value calibrated in tools/c5_calibration.py, DESIGN.md §10)")
    ap.add_argument("--out", default=os.path.join(ROOT, "profiles", "configs_r02.json"))
    args = ap.parse_args()
    res = {}
    if args.only in ("", "C4"):
        res["C4"] = run_c4()
        print(json.dumps(res["C4"]), flush=True)
        torch.cuda.empty_cache()
    if args.only in ("", "C5"):
        res["C5"] = run_c5([float(x) for x in args.tols.split(",")])
    json.dump(res, open(args.out, "w"), indent=1)


if __name__ == "__main__":
    main()
