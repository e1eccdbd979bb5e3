"""One latency-bound leaf kernel at C3 sizes, warm and event-timed (for ncu --set full captures too):
  lu  w x 32 partial-pivot LU leaf (grid kernel for w > ~24k, cluster kernel below)   [K-LU, a2]
  qr  2048 x 32 Householder leaf of the sketch QR (cluster kernel)                     [K-SQR, a2]
Usage: python tools/leaf_probe.py lu 63488 | qr 2048   (prints us per column)"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_2507_00976_b200 as bq  # noqa: E402

kind = sys.argv[1] if len(sys.argv) > 1 else "lu"
rows = int(sys.argv[2]) if len(sys.argv) > 2 else 63488
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 5
g = torch.Generator(device="cuda").manual_seed(0)
X0 = torch.randn(32, rows, dtype=torch.float64, device="cuda", generator=g).t()  # rows x 32, column-major
if kind == "qr":  # WT = MskT window, w x d = 32 x rows column-major: the d x 32 sketch block is one leaf
    X0 = torch.randn(rows, 32, dtype=torch.float64, device="cuda", generator=g).t()
best = 1e30
for r in range(reps + 1):
    X = X0.clone().t().contiguous().t()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    if kind == "lu":
        bq.debug_lu_pivots(X)
    else:
        bq.debug_sketch_qr(X)
    e1.record()
    torch.cuda.synchronize()
    if r:
        best = min(best, e0.elapsed_time(e1))
print(f"{kind} rows={rows}: {best * 1e3:.1f} us per leaf call = {best * 1e3 / 32:.2f} us per column (incl. launch)")
