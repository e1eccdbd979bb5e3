"""Warm, event-timed latency of the step-level pieces at C3 sizes (b = d = 2048), through the debug C-ABI
entries: K-LU pivots (w x d), K-SQR (R_sk of the d x w sketch window), the a4 panel (h x k) and the k x k
chain pieces (POTRF via the panel is inside debug_panel; TRSM k x k substitution / inverse).
Usage: python tools/latency_probe.py [reps]"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_2507_00976_b200 as bq  # noqa: E402

reps = int(sys.argv[1]) if len(sys.argv) > 1 else 3
g = torch.Generator(device="cuda").manual_seed(0)


def cm(r, c):
    return torch.randn(c, r, dtype=torch.float64, device="cuda", generator=g).t()


def timeit(fn, setup):
    best = 1e30
    for _ in range(reps + 1):
        args = setup()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn(*args)
        e1.record()
        torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1))
    return best


out = {}
d = 2048
for w in (63488, 32768, 16384, 4096):
    L0 = cm(w, d)
    out[f"lu_pivots_w{w}_d{d}"] = timeit(lambda L: bq.debug_lu_pivots(L), lambda: (L0.clone().t().contiguous().t(),))
    W0 = cm(w, d)
    out[f"sketch_qr_w{w}_d{d}"] = timeit(lambda W: bq.debug_sketch_qr(W), lambda: (W0.clone().t().contiguous().t(),))
    print(json.dumps({k: round(v, 3) for k, v in out.items()}), flush=True)
for h in (65536, 32768, 4096):
    k = 2048
    P0 = cm(h, k)
    S = torch.randn(k, h, dtype=torch.float64, device="cuda", generator=g)
    R = torch.linalg.qr(S @ P0, mode="r")[1]
    out[f"panel_h{h}_k{k}"] = timeit(lambda P: bq.debug_panel(P, k, R), lambda: (P0.clone().t().contiguous().t(),))
T = torch.triu(cm(2048, 2048)) + 50 * torch.eye(2048, dtype=torch.float64, device="cuda")
T = T.t().contiguous().t()
B0 = cm(2048, 2048)
for inv in (False, True):
    out[f"trsm_2048x2048_inv{int(inv)}"] = timeit(lambda B: bq.debug_trsm(T, B, inverse=inv),
                                                  lambda: (B0.clone().t().contiguous().t(),))
print(json.dumps({k: round(v, 3) for k, v in out.items()}, indent=1))
