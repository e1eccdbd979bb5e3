"""One warm K-LU pivot selection and one K-SQR (R_sk) at C3 iteration-0 size (w = 63488, d = 2048),
for per-kernel launch lists: ncu --metrics gpu__time_duration.sum ... python tools/qrcp_probe.py [w] [d]"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_2507_00976_b200 as bq  # noqa: E402

w = int(sys.argv[1]) if len(sys.argv) > 1 else 63488
d = int(sys.argv[2]) if len(sys.argv) > 2 else 2048
g = torch.Generator(device="cuda").manual_seed(0)
L0 = torch.randn(d, w, dtype=torch.float64, device="cuda", generator=g).t()
for _ in range(2):
    L = L0.clone().t().contiguous().t()
    bq.debug_lu_pivots(L)
    W = L0.clone().t().contiguous().t()
    bq.debug_sketch_qr(W)
    torch.cuda.synchronize()
print("done")
