"""N1: pivot quality of the GPU BQRRP on Kahan matrices against LAPACK GEQP3 — the paper's
§6 experiment (eq. `alg:kahan_generator`, fig `kahan_spectrum`, fig `piv_qual`), scaled to
n <= 4096 so that GEQP3 (scipy -> LAPACK dgeqp3) and the SVD (numpy) stay cheap.

Metrics: ratio_i = ||R_geqp3(i:, i:)||_F / ||R_bqrrp(i:, i:)||_F and |R(i,i)| / sigma_i for
both methods.  Matrix: the classical Kahan generator (reading Z27, the removed MATLAB generator
P:1321-1347), p = 1000, theta = 1.2.  Block sizes scaled from the paper's {64, 4096} at n = 16384.

    python tools/kahan_quality.py [--sizes 1024,4096] [--out profiles/kahan_quality_r01.json]
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import scipy.linalg  # noqa: E402
import torch  # noqa: E402

import inputs  # noqa: E402
import paper_2507_00976_b200 as bq  # noqa: E402


def trailing_norms(R):
    """S_i = ||R(i:, i:)||_F for upper-triangular R (row r contributes ||R(r, r:)||^2 for r >= i)."""
    rn2 = np.sum(np.triu(R) ** 2, axis=1)
    return np.sqrt(np.cumsum(rn2[::-1])[::-1])


def run(n, b, rank_tol):
    M = inputs.kahan(n, theta=1.2, p=1000.0)
    sigma = np.linalg.svd(M, compute_uv=False)
    Rg, _ = scipy.linalg.qr(M, pivoting=True, mode="r")
    dA = torch.tensor(np.ascontiguousarray(M.T), device="cuda").t()
    Ab, tau, J, rank, ph = bq.factor(dA, b, b, seed=0, rank_tol=rank_tol, phase_times=True)
    Rb = np.triu(Ab.cpu().numpy())[:n]
    # the BQRRP side's metric on the GPU (K-NORM, bqrrp_trailing_norms: R's trailing Frobenius norms straight off
    # the GEQP3-format output); the GEQP3 side in numpy — and the two forms cross-checked on the BQRRP R
    tb = bq.trailing_norms(Ab).cpu().numpy()
    tg, tb_np = trailing_norms(Rg), trailing_norms(Rb)
    knorm_vs_numpy = float(np.max(np.abs(tb - tb_np) / np.maximum(tb_np, 1e-300)))
    lim = min(rank, int(0.9 * n))
    ratio = tg[:lim] / tb[:lim]
    dg = np.abs(np.diag(Rg)) / sigma
    db = np.abs(np.diag(Rb)) / sigma
    lower = (n * (n + 1) / 2) ** -0.5  # GEQP3's guaranteed lower bound on |R(i,i)| / sigma_i
    return {"n": n, "b": b, "rank_tol": rank_tol, "rank": rank,
            "ratio_median_i_lt_0.9n": float(np.median(ratio)), "ratio_min": float(ratio.min()),
            "ratio_max": float(ratio.max()),
            "diag_over_sigma_bqrrp_min": float(db[:lim].min()), "diag_over_sigma_bqrrp_max": float(db[:lim].max()),
            "diag_over_sigma_geqp3_min": float(dg[:lim].min()), "diag_over_sigma_geqp3_max": float(dg[:lim].max()),
            "geqp3_lower_bound": lower, "panel_fallbacks": bq.panel_fallbacks(), "factor_ms": ph["total"],
            "knorm_vs_numpy_max_rel": knorm_vs_numpy,
            "ratio_samples": {str(i): float(ratio[i]) for i in np.linspace(0, lim - 1, 12).astype(int)}}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--sizes", default="1024,4096")
    ap.add_argument("--out", default=os.path.join(ROOT, "profiles", "kahan_quality_r02.json"))
    args = ap.parse_args()
    rows = []
    for n in [int(x) for x in args.sizes.split(",")]:
        for b in (max(16, n // 256), n // 4):
            for tol in (None, 1e-300):
                try:
                    rows.append(run(n, b, tol))
                except Exception as e:  # e.g. a Cholesky-QR breakdown with the rank test disabled
                    rows.append({"n": n, "b": b, "rank_tol": tol, "error": str(e)[:200]})
                print(json.dumps(rows[-1]), flush=True)
    json.dump({"what": "Kahan pivot quality, GPU BQRRP vs LAPACK dgeqp3 (paper §6, scaled)", "rows": rows},
              open(args.out, "w"), indent=1)


if __name__ == "__main__":
    main()
