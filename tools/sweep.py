"""N3: B200 block-size sweep and per-phase breakdown — the analogue of the paper's
fig `qr_performance_gpu` (m in {2048 ... 32768}, b in {32 ... 2048}, gamma = 1) and
fig `gpu_runtime_breakdown`.  Canonical GEQRF TFLOP/s, best of `reps` after one warm-up.

    python tools/sweep.py [--sizes 2048,4096,...] [--blocks 32,64,...] [--out profiles/sweep_r01.json]
"""
import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import bench  # noqa: E402
import inputs  # noqa: E402
import paper_2507_00976_b200 as bq  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--sizes", default="2048,4096,8192,16384,32768")
    ap.add_argument("--blocks", default="32,64,128,256,512,1024,2048")
    ap.add_argument("--reps", type=int, default=2)
    ap.add_argument("--max-iters", type=int, default=256, help="skip (m, b) with more block iterations")
    ap.add_argument("--out", default=os.path.join(ROOT, "profiles", "sweep_r02.json"))
    ap.add_argument("--variants", default="cqr", help="comma list of cqr (CholQR2 panel), hqr (cholqr_passes = 0, the "
                    "paper's BQRRP_HQR), and the suffix -serial (one stream: the phases then partition the whole step, "
                    "the fig gpu_runtime_breakdown analogue, P:1226-1258)")
    args = ap.parse_args()
    sizes = [int(x) for x in args.sizes.split(",")]
    blocks = [int(x) for x in args.blocks.split(",")]
    rows = []
    for m in sizes:
        A0 = inputs.gaussian_cuda(m, m, seed=0)
        A = torch.empty_like(A0.t()).t()
        for b in blocks:
            if b > m or m // b > args.max_iters:
                continue
            ws = torch.empty(bq.workspace_query(m, m, b, b), dtype=torch.uint8, device="cuda")
            for var in args.variants.split(","):
                passes = 0 if var.startswith("hqr") else 2
                lookahead = not var.endswith("-serial")
                best = None
                for r in range(args.reps + 1):
                    A.copy_(A0)
                    torch.cuda.synchronize()
                    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                    e0.record()
                    out = bq.factor(A, b, b, seed=0, workspace=ws, phase_times=True, cholqr_passes=passes,
                                    lookahead=lookahead)
                    e1.record()
                    torch.cuda.synchronize()
                    ms = e0.elapsed_time(e1)
                    if r > 0 and (best is None or ms < best[0]):
                        best = (ms, out[4], out[3])
                ms, ph, rank = best
                tf = bench.canonical_flops(m, m) / (ms * 1e-3) / 1e12
                rows.append({"m": m, "b": b, "d": b, "variant": var, "ms": ms, "tflops": tf, "rank": rank,
                             "pct_p64": 100 * tf / bench.peak_fp64()[0], "phases_ms": ph})
                print(json.dumps(rows[-1]), flush=True)
            del ws
        del A0, A
        torch.cuda.empty_cache()
    json.dump({"what": "canonical GEQRF TFLOP/s of bqrrp_factor on one B200, square Gaussian, d = b, best of "
                       f"{args.reps} after a warm-up; phases = critical-stream partition + bulk GEMM",
               "when": time.strftime("%Y-%m-%d %H:%M:%S"), "rows": rows}, open(args.out, "w"), indent=1)


if __name__ == "__main__":
    main()
