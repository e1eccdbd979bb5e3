"""Kernel timeline of one warm factorization (CUPTI through torch.profiler; no nsys in this image).

Reports, over the timed factorization: wall time, time with at least one of our kernels running (device busy),
the idle gaps (no kernel on any stream: host launch latency, the per-iteration host read of k), per-stream busy
time, and the per-kernel-name totals with real (in-stream, warm) durations -- unlike an ncu launch list, which
serialises launches and flushes caches.

usage: python tools/timeline.py C2 [--no-lookahead] [--json out.json] [--gaps N]
"""
import json
import os
import sys
from collections import defaultdict

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402
from torch.profiler import ProfilerActivity, profile  # noqa: E402

import bench  # noqa: E402
import inputs  # noqa: E402
import paper_2507_00976_b200 as bq  # noqa: E402


def main():
    name = sys.argv[1] if len(sys.argv) > 1 else "C2"
    lookahead = "--no-lookahead" not in sys.argv
    out_json = sys.argv[sys.argv.index("--json") + 1] if "--json" in sys.argv else None
    ngaps = int(sys.argv[sys.argv.index("--gaps") + 1]) if "--gaps" in sys.argv else 15
    if name.isdigit():
        m = n = int(name)
        b = d = int(sys.argv[2])
    else:
        cfg = bench.CONFIGS[name]
        m, n, b, d = cfg["m"], cfg["n"], cfg["b"], cfg["d"]
    A0 = inputs.gaussian_cuda(m, n, seed=0)
    A = torch.empty_like(A0.t()).t()
    ws = torch.empty(bq.workspace_query(m, n, b, d), dtype=torch.uint8, device="cuda")
    A.copy_(A0)
    bq.factor(A, b, d, seed=0, workspace=ws, lookahead=lookahead)  # warm-up
    A.copy_(A0)
    torch.cuda.synchronize()
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        bq.factor(A, b, d, seed=0, workspace=ws, lookahead=lookahead)
        e1.record()
        torch.cuda.synchronize()
    wall_ms = e0.elapsed_time(e1)
    ks = []
    for ev in prof.events():
        if ev.device_type != torch.autograd.DeviceType.CUDA:
            continue
        nm = ev.name
        if nm.startswith("Memcpy") or nm.startswith("Memset") or "elementwise" in nm or "copy_" in nm:
            kind = "mem"
        else:
            kind = "kernel"
        t0 = ev.time_range.start
        t1 = ev.time_range.end
        ks.append((t0, t1, nm, getattr(ev, "device_resource_id", 0), kind))
    ks.sort()
    if not ks:
        print("no kernels captured")
        return
    t_begin, t_end = ks[0][0], max(k[1] for k in ks)
    # union of busy intervals, gaps
    busy = 0.0
    gaps = []
    cur0, cur1 = ks[0][0], ks[0][1]
    for t0, t1, nm, sid, kind in ks[1:]:
        if t0 > cur1:
            busy += cur1 - cur0
            gaps.append((t0 - cur1, cur1 - t_begin, nm))
            cur0, cur1 = t0, t1
        else:
            cur1 = max(cur1, t1)
    busy += cur1 - cur0
    per_stream = defaultdict(float)
    per_name = defaultdict(lambda: [0, 0.0])
    for t0, t1, nm, sid, kind in ks:
        per_stream[sid] += t1 - t0
        short = nm.split("(")[0][:70]
        per_name[short][0] += 1
        per_name[short][1] += t1 - t0
    span_ms = (t_end - t_begin) / 1e3
    gap_ms = sum(g[0] for g in gaps) / 1e3
    print(f"{name} m={m} n={n} b={b} d={d} lookahead={lookahead}: wall {wall_ms:.2f} ms (events), kernel span "
          f"{span_ms:.2f} ms, device busy {busy / 1e3:.2f} ms, idle gaps {gap_ms:.2f} ms in {len(gaps)} gaps, "
          f"{len(ks)} launches")
    hist = defaultdict(lambda: [0, 0.0])
    for g, _, _ in gaps:
        key = "<2us" if g < 2 else "2-5us" if g < 5 else "5-10us" if g < 10 else "10-50us" if g < 50 else ">=50us"
        hist[key][0] += 1
        hist[key][1] += g / 1e3
    print("gap histogram (count, ms):", {k: (v[0], round(v[1], 2)) for k, v in hist.items()})
    print("largest gaps (us, at ms, next kernel):")
    for g, at, nm in sorted(gaps, reverse=True)[:ngaps]:
        print(f"  {g:9.1f}  {at / 1e3:9.2f}  {nm[:80]}")
    print("per stream busy (ms):", {k: round(v / 1e3, 2) for k, v in per_stream.items()})
    print("per kernel (launches, ms, avg us):")
    for nm, (c, t) in sorted(per_name.items(), key=lambda x: -x[1][1])[:30]:
        print(f"  {nm:72s} {c:6d} {t / 1e3:9.2f} {t / c:9.2f}")
    for sid in sorted(per_stream, key=per_stream.get, reverse=True):
        if per_stream[sid] < 0.1 * max(per_stream.values()):
            continue
        pc = defaultdict(lambda: [0, 0.0])
        for t0, t1, nm, s_, kind in ks:
            if s_ == sid:
                short = nm.split("(")[0][:70]
                pc[short][0] += 1
                pc[short][1] += t1 - t0
        print(f"stream {sid} ({per_stream[sid] / 1e3:.1f} ms busy) per kernel (launches, ms, avg us):")
        for nm, (c, t) in sorted(pc.items(), key=lambda x: -x[1][1])[:12]:
            print(f"  {nm:72s} {c:6d} {t / 1e3:9.2f} {t / c:9.2f}")
    if "--iter" in sys.argv:  # one iteration (between consecutive panel starts) stream by stream
        it = int(sys.argv[sys.argv.index("--iter") + 1])
        starts = [k[0] for k in ks if k[2].startswith("bqrrp::extract_rsk11_kernel")]
        if it + 1 < len(starts):
            w0, w1 = starts[it], starts[it + 1]
            print(f"iteration {it}: {(w1 - w0) / 1e3:.2f} ms from panel start to the next panel start")
            for sid in sorted(per_stream, key=per_stream.get, reverse=True):
                sel = [k for k in ks if k[3] == sid and w0 <= k[0] < w1]
                if not sel:
                    continue
                busy_w = sum(k[1] - k[0] for k in sel)
                print(f" stream {sid}: {len(sel)} kernels, busy {busy_w / 1e3:.2f} ms, first {(sel[0][0] - w0) / 1e3:.2f}"
                      f" last end {(max(k[1] for k in sel) - w0) / 1e3:.2f} ms")
                prev_end = None
                for k in sel:
                    gap = (k[0] - prev_end) if prev_end is not None else 0.0
                    if k[1] - k[0] >= 40 or gap >= 40:
                        print(f"    @{(k[0] - w0) / 1e3:8.3f} ms  gap {gap:7.1f} us  dur {k[1] - k[0]:8.1f} us  {k[2][:60]}")
                    prev_end = k[1] if prev_end is None else max(prev_end, k[1])
    if out_json:
        json.dump({"config": name, "m": m, "n": n, "b": b, "d": d, "lookahead": lookahead, "wall_ms": wall_ms,
                   "span_ms": span_ms, "busy_ms": busy / 1e3, "gap_ms": gap_ms, "n_gaps": len(gaps),
                   "launches": len(ks), "gap_hist": {k: v for k, v in hist.items()},
                   "per_stream_ms": {str(k): v / 1e3 for k, v in per_stream.items()},
                   "per_kernel": {k: {"launches": v[0], "ms": v[1] / 1e3} for k, v in per_name.items()}},
                  open(out_json, "w"), indent=1)


if __name__ == "__main__":
    main()
