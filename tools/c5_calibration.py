"""C5 rank_tol calibration on the scaled analogue: a 4096^2 graded-spectrum matrix,
numerical rank 1024, sigma_i = 1e-14^(i/1023) (C5's decay scaled by 8), b = n/32 = 128, d = 1.25 b = 160.

rank_tol is expressed as alpha u sqrt(max(m, n)) (the noise floor of the trailing matrix relative to |R(0,0)| scales
as u sqrt(n), App. B3), so the alpha calibrated here transfers to C5 (32768^2).  For each alpha the ORACLE
(oracle.bqrrp, CPU) and the GPU path report the found rank l and the truncated residual
||A(:, J) - Q(:, :l) R(:l, :)||_F / ||A||_F; the acceptance (App. B3): residual <= 1e-13 and l <= 1024 + b.

    python tools/c5_calibration.py --oracle   (CPU only)  ->  profiles/c5_calibration_oracle_r02.json
    python tools/c5_calibration.py --gpu      (B200)      ->  profiles/c5_calibration_gpu_r02.json
"""
import argparse
import json
import math
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

import inputs  # noqa: E402

N, K, B, D = 4096, 1024, 128, 160
ALPHAS = [100.0, 30.0, 10.0, 3.0, 1.0, 0.3]
U = 2.0 ** -53


def tol_of(alpha, n=N):
    return alpha * U * math.sqrt(n)


def truncated_residual(A0, F, tau, J, l):
    """||A0(:, J) - Q(:, :l) R(:l, :)||_F / ||A0||_F with Q applied reflector by reflector (numpy)."""
    m, n = A0.shape
    Y = np.zeros((m, n))
    Y[:l] = np.triu(F[:l, :])
    for j in range(l - 1, -1, -1):
        v = np.concatenate(([1.0], F[j + 1:, j]))
        Y[j:] -= tau[j] * np.outer(v, v @ Y[j:])
    return float(np.linalg.norm(A0[:, J - 1] - Y) / np.linalg.norm(A0))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--oracle", action="store_true")
    ap.add_argument("--gpu", action="store_true")
    args = ap.parse_args()
    A0, sigma = inputs.graded(N, N, K, sigma_last=1e-14, seed=0)
    rows = []
    if args.oracle:
        import oracle

        for a in ALPHAS:
            t0 = time.perf_counter()
            o = oracle.bqrrp(A0, B, D, seed=0, rank_tol=tol_of(a))
            dt = time.perf_counter() - t0
            res = truncated_residual(A0, o.A, o.tau, o.J, o.rank)
            rows.append({"side": "oracle", "alpha": a, "rank_tol": tol_of(a), "rank": o.rank, "residual": res,
                         "accept": bool(res <= 1e-13 and o.rank <= K + B), "seconds": dt})
            print(json.dumps(rows[-1]), flush=True)
        out = os.path.join(ROOT, "profiles", "c5_calibration_oracle_r02.json")
    else:
        import torch

        import paper_2507_00976_b200 as bq

        for a in ALPHAS:
            dA = torch.tensor(np.ascontiguousarray(A0.T), device="cuda").t()
            F, tau, J, l = bq.factor(dA, B, D, seed=0, rank_tol=tol_of(a))
            res = truncated_residual(A0, F.cpu().numpy(), tau.cpu().numpy(), J.cpu().numpy(), l)
            rows.append({"side": "gpu", "alpha": a, "rank_tol": tol_of(a), "rank": l, "residual": res,
                         "accept": bool(res <= 1e-13 and l <= K + B), "panel_fallbacks": bq.panel_fallbacks()})
            print(json.dumps(rows[-1]), flush=True)
        out = os.path.join(ROOT, "profiles", "c5_calibration_gpu_r02.json")
    ok = [r["alpha"] for r in rows if r["accept"]]
    summary = {"what": "C5 rank_tol calibration on the 4096^2 / rank-1024 analogue (SURVEY App. B3)",
               "matrix": f"inputs.graded({N}, {N}, {K}, 1e-14, seed=0)", "b": B, "d": D,
               "rank_tol": "alpha * u * sqrt(max(m, n))", "rows": rows,
               "largest_accepted_alpha": max(ok) if ok else None,
               "sigma_gt_1e-13": int(np.sum(sigma > 1e-13))}
    json.dump(summary, open(out, "w"), indent=1)
    print(json.dumps({k: v for k, v in summary.items() if k != "rows"}))


if __name__ == "__main__":
    main()
