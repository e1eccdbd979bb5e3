"""The HBM-bound kernels alone at the C3 shape, for ncu captures (dram bytes vs algorithmic bytes):
K-PERM (gather_cols / scatter_cols on 2d = 4096 random columns of a 65536 x 65536 matrix) and K-NORM
(col_norms on all columns, trailing_rows on the upper trapezoid).  Same calls bench.py times (hbm_paths).
    python tools/hbm_probe.py [m]"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import bench  # noqa: E402
import inputs  # noqa: E402
import paper_2507_00976_b200 as bq  # noqa: E402

m = int(sys.argv[1]) if len(sys.argv) > 1 else 65536
A = inputs.gaussian_cuda(m, m, seed=0)
B = torch.empty_like(A.t()).t()
B.copy_(A)
print(bench.hbm_paths(bq, A, B, m, m, 2048, torch.cuda.current_stream(), reps=2))
