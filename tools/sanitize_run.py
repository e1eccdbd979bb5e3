"""One factorization through the C ABI for compute-sanitizer (memcheck / racecheck / synccheck / initcheck).

    compute-sanitizer --tool racecheck python tools/sanitize_run.py C1
    compute-sanitizer --tool memcheck  python tools/sanitize_run.py 8192 1024

Shapes: C1 (1024^2, b = 128, d = 160: register LU / QR cluster leaves, the k x k chain) or `m b`
(m x m, d = b).  The bulk GEMM's green-context partition is off (bulk_sms = -1: the sanitizer, like ncu, cannot
instrument launches on green-context streams; the kernel is the same dgemm2 as on the main path); `--lula` turns on
the lookahead K-LU (its laswp kernel and recorded moves).  Prints rank and the residual-free fingerprint (sum |R diag|) so a sanitizer-perturbed run
is visibly the same factorization.
"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import inputs  # noqa: E402
import paper_2507_00976_b200 as bq  # noqa: E402


def main():
    import torch

    if sys.argv[1] == "C1":
        m, b, d = 1024, 128, 160
    else:
        m, b = int(sys.argv[1]), int(sys.argv[2])
        d = b
    A = inputs.gaussian(m, m, seed=0)
    dA = torch.from_numpy(np.asfortranarray(A).T).cuda().t()
    Ag, tau, J, rk = bq.factor(dA, b, d, seed=0, bulk_sms=-1, lu_lookahead="--lula" in sys.argv)
    torch.cuda.synchronize()
    print(f"m={m} b={b} d={d} rank={rk} sum|diag R|={float(Ag.diagonal().abs().sum()):.12e} "
          f"launches={bq.launch_count()}")


if __name__ == "__main__":
    main()
