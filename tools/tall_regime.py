"""the CQRRPT regime (m >> n): the single-shot form of the method against the blocked one
on the C4 matrix (262144 x 8192 Gaussian, seed 0).

With b >= n, Alg. 1 runs ONE iteration: sketch (a1) -> LU-on-sketch pivot selection and R_sk
(a2, the "QRCP of the sketch") -> preconditioned Cholesky QR of A(:, J) (a4: M_pre = A(:, J) R_sk^-1,
CholQR2, Householder reconstruction) with no trailing update — CQRRPT ([MBM2024]) with the
paper's LUQR sketch pivoting and a GEQP3-format output.  This tool times b in {512, 1024, 2048, 4096,
8192 (= n, single shot)} with d = b and reports canonical GEQRF TFLOP/s, the residual estimate and the
phase split.  Writes profiles/tall_regime_r01.json.

    python tools/tall_regime.py [--bs 512,1024,2048,4096,8192]
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tools"))
sys.path.insert(0, os.path.join(ROOT, "tests"))

import torch  # noqa: E402

import bench  # noqa: E402
import inputs  # noqa: E402
from run_configs import residual_est, timed_factor  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--bs", default="512,1024,2048,4096,8192")
    ap.add_argument("--m", type=int, default=262144)
    ap.add_argument("--n", type=int, default=8192)
    ap.add_argument("--out", default=os.path.join(ROOT, "profiles", "tall_regime_r01.json"))
    args = ap.parse_args()
    m, n = args.m, args.n
    A0 = inputs.gaussian_cuda(m, n, seed=0)
    out = []
    for b in [int(x) for x in args.bs.split(",")]:
        d = b
        ms, (A, tau, J, rank, ph) = timed_factor(A0, b, d)
        res = residual_est(A0, A, tau, J, rank)
        tf = bench.canonical_flops(m, n) / (ms * 1e-3) / 1e12
        rec = {"m": m, "n": n, "b": b, "d": d, "single_shot": b >= n, "ms": ms, "tflops": tf,
               "pct_p64": 100 * tf / bench.peak_fp64()[0], "rank": rank, "residual_est": res,
               "phases_ms": ph}
        out.append(rec)
        print(json.dumps(rec), flush=True)
        del A, tau, J
        torch.cuda.empty_cache()
    json.dump({"what": "C4 blocked vs single-shot (CQRRPT regime, SURVEY N4)", "runs": out},
              open(args.out, "w"), indent=1)


if __name__ == "__main__":
    main()
