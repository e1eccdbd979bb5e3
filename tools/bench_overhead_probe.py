"""Where do bench.py's per-step milliseconds beyond the library's own phase total come from?  C2 steps timed as
bench.py does (per-step CUDA events around bq.factor on the caller's stream, A restored outside the events), with and
without the nvidia-smi clock sampler and with and without per-phase timing.
usage: python tools/bench_overhead_probe.py [C2] [steps]"""
import contextlib
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import bench  # noqa: E402
import inputs  # noqa: E402
import paper_2507_00976_b200 as bq  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "C2"
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 5
cfg = bench.CONFIGS[name]
m, n, b, d = cfg["m"], cfg["n"], cfg["b"], cfg["d"]
A0 = inputs.gaussian_cuda(m, n, seed=0)
A = torch.empty_like(A0.t()).t()
ws = torch.empty(bq.workspace_query(m, n, b, d), dtype=torch.uint8, device="cuda")
tau = torch.empty(min(m, n), dtype=torch.float64, device="cuda")
J = torch.empty(n, dtype=torch.int64, device="cuda")
stream = torch.cuda.current_stream()
for sampler in (True, False):
    for phase in (True, False):
        for _ in range(3):
            A.copy_(A0)
            bq.factor(A, b, d, seed=0, workspace=ws, tau=tau, J=J)
        torch.cuda.synchronize()
        ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(steps)]
        tot = 0.0
        cm = bench.ClockSampler(0) if sampler else contextlib.nullcontext()
        with cm:
            for i in range(steps):
                A.copy_(A0)
                ev[i][0].record(stream)
                out = bq.factor(A, b, d, seed=0, workspace=ws, tau=tau, J=J, phase_times=phase)
                ev[i][1].record(stream)
                if phase:
                    tot += out[4]["total"]
            torch.cuda.synchronize()
        per = [s.elapsed_time(e) for s, e in ev]
        print(f"sampler={sampler} phase={phase}: ms/step {sum(per) / steps:.2f} (per step {[round(x, 1) for x in per]})"
              + (f", library phase total {tot / steps:.2f}" if phase else ""), flush=True)
