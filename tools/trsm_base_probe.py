"""Launch sequence for timing the 64-column base TRSM (trsm_base_kernel) back to back and interleaved with a
GEMM launch (different code between two solves).  The debug entries synchronise, so the per-kernel
durations come from an ncu launch list of this script, e.g.
  ncu --metrics gpu__time_duration.sum --cache-control none --csv python tools/trsm_base_probe.py
Usage: python tools/trsm_base_probe.py [rows ...]"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_2507_00976_b200 as bq  # noqa: E402

REPS = 20


def colmaj(x):
    return x.t().contiguous().t()


def run(body):
    for _ in range(REPS):
        body()
    torch.cuda.synchronize()


def main():
    rows_list = [int(a) for a in sys.argv[1:]] or [128, 2048, 8192]
    gen = torch.Generator(device="cuda").manual_seed(0)
    # T = I + 0.01 triu(N): B <- B T^{-1} stays O(1) over thousands of in-place repetitions
    T = colmaj(0.01 * torch.triu(torch.randn(64, 64, dtype=torch.float64, device="cuda", generator=gen)) +
               torch.eye(64, dtype=torch.float64, device="cuda"))
    TL = colmaj(T.t())  # the same op(T) stored lower (mode 1: strided coefficient loads)
    G = colmaj(torch.randn(64, 64, dtype=torch.float64, device="cuda", generator=gen))
    Cg = colmaj(torch.empty(64, 64, dtype=torch.float64, device="cuda"))
    run(lambda: bq.debug_gemm(False, False, 1.0, G, G, 0.0, Cg))
    for rows in rows_list:
        B = colmaj(torch.randn(rows, 64, dtype=torch.float64, device="cuda", generator=gen))
        run(lambda: bq.debug_trsm(T, B))
        run(lambda: (bq.debug_trsm(T, B), bq.debug_gemm(False, False, 1.0, G, G, 0.0, Cg)))
        run(lambda: bq.debug_trsm(TL, B, t_lower=True))
    print("done")


if __name__ == "__main__":
    main()
