"""The CPU-baseline plan of BASELINE.md / SURVEY §8(d.5): the plain C oracle (oracle/, test infrastructure — run
here only as the reported baseline, never on the product path) timed on the host cores:

  C1 (1024^2, b = 128, d = 160): 1 thread and all cores, best of 3;
  C2 (16384^2, b = d = 1024): all cores, one run (--c2; ~17 min on 8 cores, ~8 on 16);
  C3, C4: not run — extrapolated from C2 by the algorithmic-flop ratio (C3 = 4.51e14 / 8.29e12 x
  the C2 time, C4 = 4.15e13 / 8.29e12 x), labelled as extrapolated.

Wall clock around oracle.bqrrp only (input generation excluded); canonical GEQRF TFLOP/s as for the GPU.

    python tools/oracle_baseline.py [--c2] [--out profiles/oracle_baseline_r02.json]
"""
import argparse
import json
import os
import platform
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import bench  # noqa: E402
import inputs  # noqa: E402
import oracle  # noqa: E402

ALG_FLOPS = {"C2": 8.29e12, "C3": 4.51e14, "C4": 4.15e13}  # SURVEY §8(d.3), CholQR2 algorithmic


def run(cfg, nthreads, reps):
    c = bench.CONFIGS[cfg]
    m, n, b, d = c["m"], c["n"], c["b"], c["d"]
    A = inputs.gaussian(m, n, seed=0)
    best = None
    for _ in range(reps):
        t0 = time.perf_counter()
        out = oracle.bqrrp(A, b, d, seed=0, nthreads=nthreads)
        dt = time.perf_counter() - t0
        best = dt if best is None else min(best, dt)
    return {"config": cfg, "m": m, "n": n, "b": b, "d": d, "threads": nthreads, "runs": reps, "seconds_best": best,
            "tflops_canonical": bench.canonical_flops(m, n) / best / 1e12, "rank": out.rank}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--c2", action="store_true")
    ap.add_argument("--out", default=os.path.join(ROOT, "profiles", "oracle_baseline_r02.json"))
    args = ap.parse_args()
    cores = os.cpu_count()
    rows = [run("C1", 1, 3), run("C1", cores, 3)]
    for r in rows:
        print(json.dumps(r), flush=True)
    if args.c2:
        r = run("C2", cores, 1)
        rows.append(r)
        print(json.dumps(r), flush=True)
        for cfg in ("C3", "C4"):
            c = bench.CONFIGS[cfg]
            t = r["seconds_best"] * ALG_FLOPS[cfg] / ALG_FLOPS["C2"]
            rows.append({"config": cfg, "m": c["m"], "n": c["n"], "b": c["b"], "d": c["d"], "threads": cores,
                         "seconds_best": t, "tflops_canonical": bench.canonical_flops(c["m"], c["n"]) / t / 1e12,
                         "extrapolated": f"from the C2 run by the algorithmic-flop ratio {ALG_FLOPS[cfg]:.3g} / "
                                         f"{ALG_FLOPS['C2']:.3g} (SURVEY §8(d.3)); not run"})
            print(json.dumps(rows[-1]), flush=True)
    res = {"what": "plain C oracle (oracle/bqrrp_oracle.c, OpenMP over independent columns), BASELINE.md CPU plan",
           "cpu": bench.cpu_model(), "cores": cores, "host": platform.node(), "rows": rows}
    with open(args.out, "w") as f:
        json.dump(res, f, indent=1)


if __name__ == "__main__":
    main()
