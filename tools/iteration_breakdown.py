"""Per-iteration kernel composition of one factorization from an ncu launch list (gpu__time_duration.sum).

Iterations are delimited by `write_panel_kernel` (one launch per BQRRP iteration, the end of the panel). For
each iteration: serialised kernel time, split into the big trailing-update GEMMs (> 1 ms per launch), the
other GEMMs, and the latency-bound kernels (LU / QR leaves, diagonal blocks, base TRSMs, permutation), by
stream.  ncu serialises launches, so these are per-kernel costs, not the overlapped wall time.

usage: python tools/iteration_breakdown.py launches.csv [--every N] [--json out.json]
"""
import argparse
import csv
import json
from collections import defaultdict


def load(path):
    rows = list(csv.reader(l for l in open(path) if not l.startswith("==")))
    h = rows[0]
    ki, vi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
    si, gi = h.index("Stream"), h.index("Grid Size")
    scale = {"nsecond": 1e-3, "usecond": 1.0, "msecond": 1e3, "second": 1e6}
    out = []
    for r in rows[1:]:
        if len(r) <= vi:
            continue
        name = r[ki].split("(")[0].split("<")[0].replace("void ", "").replace("bqrrp::", "").strip()
        out.append((name, r[si], r[gi], float(r[vi].replace(",", "")) * scale.get(r[ui], 1e-3)))
    return out


def breakdown(launches):
    ends = [i for i, l in enumerate(launches) if l[0] == "write_panel_kernel"]
    its = []
    start = 0
    for it, e in enumerate(ends):
        seq = launches[start:e + 1]
        start = e + 1
        cls = defaultdict(float)
        cnt = defaultdict(int)
        for name, stream, grid, us in seq:
            if name == "dgemm2_kernel":
                c = "gemm_big" if us > 1000 else "gemm_small"
            elif name.startswith("lu_"):
                c = "lu_leaves"
            elif name.startswith("qr_"):
                c = "qr_leaves"
            elif name in ("potrf_diag", "getrf_sign_diag", "tri_inv_diag_kernel"):
                c = "kxk_diag_blocks"
            elif name.startswith("trsm"):
                c = "trsm_base_apply"
            elif "cols" in name or "rows" in name:
                c = "permutation"
            else:
                c = "other"
            cls[c] += us
            cnt[c] += 1
        its.append({"iteration": it, "launches": len(seq), "serialised_ms": round(sum(cls.values()) / 1e3, 3),
                    "ms": {k: round(v / 1e3, 3) for k, v in sorted(cls.items(), key=lambda x: -x[1])},
                    "count": dict(cnt)})
    return its


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("csv")
    ap.add_argument("--every", type=int, default=4)
    ap.add_argument("--json", default=None)
    a = ap.parse_args()
    its = breakdown(load(a.csv))
    keys = ["gemm_big", "gemm_small", "lu_leaves", "qr_leaves", "kxk_diag_blocks", "trsm_base_apply", "permutation",
            "other"]
    print(f"{'it':>3} {'launches':>8} {'total ms':>9} " + " ".join(f"{k:>15}" for k in keys))
    for r in its:
        if r["iteration"] % a.every and r["iteration"] != len(its) - 1:
            continue
        print(f"{r['iteration']:3d} {r['launches']:8d} {r['serialised_ms']:9.2f} " +
              " ".join(f"{r['ms'].get(k, 0.0):15.2f}" for k in keys))
    tot = defaultdict(float)
    for r in its:
        for k, v in r["ms"].items():
            tot[k] += v
    print("sum " + " ".join(f"{k}={v:.1f}ms" for k, v in sorted(tot.items(), key=lambda x: -x[1])))
    if a.json:
        json.dump({"iterations": its, "totals_ms": dict(tot)}, open(a.json, "w"), indent=1)


if __name__ == "__main__":
    main()
