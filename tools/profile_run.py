"""One warm factorization of a config for profilers (ncu launch lists / --set full captures).
Usage: python tools/profile_run.py C2 [--warm 1]"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import bench  # noqa: E402
import inputs  # noqa: E402
import paper_2507_00976_b200 as bq  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "C2"
warm = int(sys.argv[sys.argv.index("--warm") + 1]) if "--warm" in sys.argv else 1
passes = int(sys.argv[sys.argv.index("--passes") + 1]) if "--passes" in sys.argv else 2
lookahead = "--no-lookahead" not in sys.argv
# ncu cannot profile kernels on green-context streams ("Failed to prepare kernel for profiling"): the bulk GEMM's
# SM partition is off by default here (bqrrp_options.bulk_sms = -1); --bulk-sms 0 selects the library default
bulk_sms = int(sys.argv[sys.argv.index("--bulk-sms") + 1]) if "--bulk-sms" in sys.argv else -1
cfg = bench.CONFIGS[name]
m, n, b, d = cfg["m"], cfg["n"], cfg["b"], cfg["d"]
A0 = inputs.gaussian_cuda(m, n, seed=0)
A = torch.empty_like(A0.t()).t()
ws = torch.empty(bq.workspace_query(m, n, b, d), dtype=torch.uint8, device="cuda")
for i in range(warm + 1):
    A.copy_(A0)
    torch.cuda.synchronize()
    if i == warm:
        torch.cuda.nvtx.range_push("timed")
    out = bq.factor(A, b, d, seed=0, workspace=ws, phase_times=True, cholqr_passes=passes,
                    lookahead=lookahead, bulk_sms=bulk_sms)
    torch.cuda.synchronize()
print(name, "passes", passes, "lookahead", lookahead, "rank", out[3], "phases(ms)", {k: round(v, 2) for k, v in out[4].items()})
