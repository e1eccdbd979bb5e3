"""A/B of the one-GPU schedules on one config: panel_lookahead 0 (panel i+1 after the bulk, default) or 1
(overlapped with the bulk from a gathered copy), and the serial schedule; each warm, then `reps` factorizations timed with CUDA events (best and
mean), phases of the last.  Usage: python tools/schedule_ab.py C3 [reps]"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import bench  # noqa: E402
import inputs  # noqa: E402
import paper_2507_00976_b200 as bq  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "C2"
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 2
cfg = bench.CONFIGS[name]
m, n, b, d = cfg["m"], cfg["n"], cfg["b"], cfg["d"]
A0 = inputs.gaussian_cuda(m, n, seed=0)
A = torch.empty_like(A0.t()).t()
ws = torch.empty(bq.workspace_query(m, n, b, d), dtype=torch.uint8, device="cuda")
modes = [("panel_after_bulk", dict(panel_lookahead=0)), ("panel_overlapped", dict(panel_lookahead=1)),
         ("serial", dict(lookahead=False))]
res = {}
for label, kw in modes:
    times = []
    for i in range(reps + 1):
        A.copy_(A0)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        out = bq.factor(A, b, d, seed=0, workspace=ws, phase_times=(i == reps), **kw)
        e1.record()
        torch.cuda.synchronize()
        if i:
            times.append(e0.elapsed_time(e1))
    fl = bench.canonical_flops(m, n)
    res[label] = {"ms_best": min(times), "ms_mean": sum(times) / len(times), "tflops_best": fl / min(times) / 1e9,
                  "phases_ms": {k: round(v, 1) for k, v in out[4].items()}}
    print(name, label, json.dumps(res[label]), flush=True)
print(json.dumps({"config": name, "results": res}))
