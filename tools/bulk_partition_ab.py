"""A/B of the bulk trailing GEMM's SM partition (bqrrp_options.bulk_sms): whole device (-1),
auto (0) and fixed green-context partitions, event-timed whole factorizations (best of `reps` after a warm-up),
with the factor checked bitwise against the whole-device run.
usage: python tools/bulk_partition_ab.py C2|<m> [b] [--reps R] [--sms -1,0,132,116] [--json out.json] [--no-pipe] [--lula] [--panel-la 1] [--lucl 8|16] [--no-merge-stream] [--lu-grid N] [--lib path.so]"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import bench  # noqa: E402
import inputs  # noqa: E402
import paper_2507_00976_b200 as bq  # noqa: E402


def arg(name, default):
    return sys.argv[sys.argv.index(name) + 1] if name in sys.argv else default


if "--lib" in sys.argv:  # an experimental build of the library (e.g. other compile-time constants)
    bq._LIB_PATH = arg("--lib", "")
name = sys.argv[1]
if name.isdigit():
    m = n = int(name)
    b = d = int(sys.argv[2])
else:
    cfg = bench.CONFIGS[name]
    m, n, b, d = cfg["m"], cfg["n"], cfg["b"], cfg["d"]
reps = int(arg("--reps", "3"))
sms = [int(x) for x in arg("--sms", "-1,0,132,116,100").split(",")]
A0 = inputs.gaussian_cuda(m, n, seed=0)
A = torch.empty_like(A0.t()).t()
ws = torch.empty(bq.workspace_query(m, n, b, d), dtype=torch.uint8, device="cuda")
canon = 2.0 * m * n * n - 2.0 * n ** 3 / 3 if m >= n else 2.0 * n * m * m - 2.0 * m ** 3 / 3
ref = None
rows = []
for s in sms:
    best, phases = 1e30, None
    for r in range(reps + 1):
        A.copy_(A0)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        out = bq.factor(A, b, d, seed=0, workspace=ws, bulk_sms=s, phase_times=(r == reps or "--phases" in sys.argv),
                        sqr_pipeline="--no-pipe" not in sys.argv, lu_lookahead="--lula" in sys.argv,
                        panel_lookahead=int(arg("--panel-la", "0")), lu_leaf_cluster=int(arg("--lucl", "0")),
                        sqr_merge_stream="--no-merge-stream" not in sys.argv, lu_grid_ctas=int(arg("--lu-grid", "0")))
        e1.record()
        torch.cuda.synchronize()
        if r > 0 and r < reps:
            best = min(best, e0.elapsed_time(e1))
        if r == reps:
            phases = {k: round(v, 2) for k, v in out[4].items()}
            if reps == 1:
                best = min(best, e0.elapsed_time(e1))
    if ref is None:
        ref = (A.clone(), out[1].clone(), out[2].clone())
        same = True
    else:
        same = bool(torch.equal(ref[0], A) and torch.equal(ref[1], out[1]) and torch.equal(ref[2], out[2]))
    row = {"bulk_sms": s, "ms": best, "tflops": canon / best / 1e9, "bitwise_same_as_first": same, "phases": phases}
    rows.append(row)
    print(json.dumps(row), flush=True)
if "--json" in sys.argv:
    json.dump({"m": m, "n": n, "b": b, "d": d, "rows": rows}, open(arg("--json", ""), "w"), indent=1)
