"""Write the oracle fingerprints the bench-shape parity tests compare against (tests/golden/oracle_*.npz).

The oracle (plain C, Alg. 1 step by step) needs minutes to an hour on a few host cores at the shapes the
bench times, so its outputs at those shapes are computed ONCE by this script, which calls only `oracle/`
and `inputs/`, and stored as fingerprints: the pivots and tau in full, per-column summaries of R and V for
every column, and a fixed sample of full columns / rows of R and V.  The GPU tests
(tests/test_gpu_golden.py) regenerate the same seeded inputs and compare element by element on that data.

    python tools/make_oracle_golden.py [case ...]      (cases: lu panel e2e c2 b4096; default all)
"""
from __future__ import annotations

import argparse
import hashlib
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import inputs  # noqa: E402
import oracle  # noqa: E402

GOLDEN = os.path.join(ROOT, "tests", "golden")

# The cases (shapes of the bench's own block iteration, SURVEY §8(c) c.6 rule 5).
CASES = {
    # K-LU on the C3 iteration-0 shape: the sketch transpose of a 65536-column matrix at d = 2048
    "lu": dict(w=65536, d=2048, seed=65536 + 2048),
    # the panel at the C3 height and block: h = 65536, k = 2048
    "panel": dict(h=65536, k=2048, seed=12345),
    # end to end with the bench's block and sketch size, several iterations: 16384 x 8192, b = d = 2048
    "e2e": dict(m=16384, n=8192, b=2048, d=2048, seed=16384 + 3 * 8192, sketch_seed=0),
    # BASELINE C2: 16384^2, b = d = 1024, seed 0
    "c2": dict(m=16384, n=16384, b=1024, d=1024, seed=0, sketch_seed=0),
    # b = d = 4096 (h > 2k at iteration 0): the panel's k x k finish runs on the side stream with the
    # inverse-diagonal TRSM (its scratch must not alias the sketch)
    "b4096": dict(m=10240, n=8192, b=4096, d=4096, seed=10240 + 8192, sketch_seed=3),
}


def input_digest(A: np.ndarray) -> str:
    """sha256 of the column-major bytes: the GPU test checks it regenerated the same matrix."""
    return hashlib.sha256(np.asfortranarray(A).tobytes(order="F")).hexdigest()


def sample_cols(n: int, b: int) -> np.ndarray:
    """Columns at block edges (first / last of the first, second, middle and last blocks) and a few
    seeded interior ones."""
    rng = np.random.default_rng(n + b)
    nb = (n + b - 1) // b
    edges = {0, b - 1, b, 2 * b - 1, (nb // 2) * b, (nb // 2) * b + b // 2, n - b, n - 1}
    extra = set(int(x) for x in rng.integers(0, n, size=4))
    return np.array(sorted(c for c in edges | extra if 0 <= c < n), dtype=np.int64)


def r_summaries(F: np.ndarray, l: int, cols: np.ndarray, rows: np.ndarray, vstride: int = 1):
    """Per-column summaries of R = triu(F)(:l, :) and V = tril(F(:, :l), -1), plus sampled columns/rows."""
    m, n = F.shape
    R = lambda j: F[: min(j + 1, l), j]  # noqa: E731
    rnorm = np.array([np.linalg.norm(R(j)) for j in range(n)])
    rdiag = np.array([F[j, j] if j < l else 0.0 for j in range(min(m, n))])
    vnorm = np.array([np.linalg.norm(F[j + 1:, j]) for j in range(l)])
    rcols = [F[: min(j + 1, l), j].copy() for j in cols]
    vcols = [F[j + 1::vstride, j].copy() if j < l else np.zeros(0) for j in cols]
    rrows = [F[i, i:].copy() if i < l else np.zeros(0) for i in rows]
    return rnorm, rdiag, vnorm, rcols, vcols, rrows


def pack(lst):
    """Ragged list of 1-D arrays -> (concatenated, offsets)."""
    off = np.zeros(len(lst) + 1, dtype=np.int64)
    for i, a in enumerate(lst):
        off[i + 1] = off[i] + len(a)
    return (np.concatenate(lst) if lst else np.zeros(0)), off


def case_lu(p):
    w, d = p["w"], p["d"]
    L = inputs.gaussian(w, d, seed=p["seed"])
    t = time.time()
    _, ipiv, margin = oracle.getf2(L)
    return dict(w=w, d=d, seed=p["seed"], digest=input_digest(L), ipiv=ipiv, margin=margin), time.time() - t


def case_panel(p):
    h, k = p["h"], p["k"]
    P = inputs.gaussian(h, k, seed=p["seed"])
    t = time.time()
    F, tau = oracle.house_qr(P, kref=k)
    cols = sample_cols(k, 256)
    rnorm, rdiag, vnorm, rcols, vcols, rrows = r_summaries(F, k, cols, np.array([0, 1, k // 2, k - 1]), vstride=8)
    rc, rco = pack(rcols)
    vc, vco = pack(vcols)
    rr, rro = pack(rrows)
    return dict(h=h, k=k, seed=p["seed"], digest=input_digest(P), tau=tau, rnorm=rnorm, rdiag=rdiag, vnorm=vnorm,
                cols=cols, rcols=rc, rcols_off=rco, vcols=vc, vcols_off=vco, vstride=8,
                rows=np.array([0, 1, k // 2, k - 1]), rrows=rr, rrows_off=rro), time.time() - t


def case_factor(p):
    m, n, b, d = p["m"], p["n"], p["b"], p["d"]
    A = inputs.gaussian(m, n, seed=p["seed"])
    digest = input_digest(A)
    t = time.time()
    out = oracle.bqrrp(A, b, d, seed=p["sketch_seed"])
    el = time.time() - t
    l = out.rank
    cols = sample_cols(n, b)
    rows = np.array([0, b - 1, b, n // 2, min(m, n) - 1], dtype=np.int64)
    rnorm, rdiag, vnorm, rcols, vcols, rrows = r_summaries(out.A, l, cols, rows)
    rc, rco = pack(rcols)
    vc, vco = pack(vcols)
    rr, rro = pack(rrows)
    return dict(m=m, n=n, b=b, d=d, seed=p["seed"], sketch_seed=p["sketch_seed"], digest=digest, J=out.J,
                tau=out.tau, rank=l, min_margin=out.min_margin, ks=out.ks, rnorm=rnorm, rdiag=rdiag, vnorm=vnorm,
                cols=cols, rcols=rc, rcols_off=rco, vcols=vc, vcols_off=vco, vstride=1, rows=rows, rrows=rr,
                rrows_off=rro), el


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("cases", nargs="*", default=list(CASES))
    a = ap.parse_args()
    oracle.build()
    os.makedirs(GOLDEN, exist_ok=True)
    for name in a.cases:
        p = CASES[name]
        fn = {"lu": case_lu, "panel": case_panel}.get(name, case_factor)
        data, el = fn(p)
        data["oracle_seconds"] = el
        data["generator"] = "tools/make_oracle_golden.py (oracle/ + inputs/ only)"
        path = os.path.join(GOLDEN, f"oracle_{name}.npz")
        np.savez_compressed(path, **data)
        print(f"{name}: {el:.1f} s -> {path} ({os.path.getsize(path) / 1e6:.2f} MB)", flush=True)


if __name__ == "__main__":
    main()
