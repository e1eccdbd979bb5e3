"""Time the a4 panel alone (bqrrp_debug_panel: preconditioned CholQR2 + reconstruction, no trailing block)
on a C3-sized panel: h x k Gaussian, R_sk11 = R of a Gaussian sketch of it.
Usage: python tools/panel_probe.py [h] [k] [reps]   (run under ncu for the per-kernel launch list)"""
import sys

import torch

import os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2507_00976_b200 as bq  # noqa: E402

h = int(sys.argv[1]) if len(sys.argv) > 1 else 65536
k = int(sys.argv[2]) if len(sys.argv) > 2 else 2048
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 3
g = torch.Generator(device="cuda").manual_seed(0)
P0 = torch.randn(k, h, dtype=torch.float64, device="cuda", generator=g).t()  # column-major h x k
S = torch.randn(k, h, dtype=torch.float64, device="cuda", generator=g)
Rsk = torch.linalg.qr(S @ P0, mode="r")[1]
P = torch.empty_like(P0)
times = []
for r in range(reps + 1):
    P.copy_(P0)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    bq.debug_panel(P, k, Rsk)
    e1.record()
    torch.cuda.synchronize()
    if r:
        times.append(e0.elapsed_time(e1))
flops = 5.0 * h * k * k
print(f"panel h={h} k={k}: best {min(times):.2f} ms  ({flops / min(times) / 1e9:.1f} TFLOP/s of ~5hk^2)  all {times}")
