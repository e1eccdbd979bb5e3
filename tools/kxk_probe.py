"""Warm event-timed k x k pieces of the panel (k = b = 2048 at C3) through the step C ABI: POTRF of an SPD
Gram matrix, the reconstruction top (k x k TRSM + sign-choosing LU), a k x k TRSM, and a k^3 GEMM for scale.
Usage: python tools/kxk_probe.py [k]"""
import ctypes
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_2507_00976_b200 as bq  # noqa: E402


k = int(sys.argv[1]) if len(sys.argv) > 1 else 2048
L = bq.lib()
g = torch.Generator(device="cuda").manual_seed(0)
X = torch.randn(4 * k, k, dtype=torch.float64, device="cuda", generator=g)
G0 = (X.t() @ X).contiguous()  # SPD, symmetric (column-major == row-major)
Q0 = torch.linalg.qr(torch.randn(4 * k, k, dtype=torch.float64, device="cuda", generator=g))[0]
Q0 = Q0.t().contiguous().t()
C = torch.linalg.cholesky(torch.eye(k, dtype=torch.float64, device="cuda") * 1.0).t().contiguous().t()
st = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
P = ctypes.c_void_p


def ptr(t):
    return P(t.data_ptr())


def timeit(fn, reps=5):
    best = 1e30
    for _ in range(reps + 1):
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        e1.record()
        torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1))
    return best


out = {}
Gw = G0.clone()
out["potrf_ms"] = timeit(lambda: (Gw.copy_(G0), L.bqrrp_debug_potrf(k, ptr(Gw), k, st)))
Wr = torch.empty(k, k, dtype=torch.float64, device="cuda")
S = torch.empty(k, dtype=torch.float64, device="cuda")
out["recon_top_ms"] = timeit(lambda: L.bqrrp_debug_recon_lu(k, ptr(Q0), 4 * k, ptr(C), ptr(Wr), ptr(S), st))
T = torch.triu(torch.randn(k, k, dtype=torch.float64, device="cuda", generator=g)) + 50 * torch.eye(
    k, dtype=torch.float64, device="cuda")
T = T.t().contiguous().t()
B0 = torch.randn(k, k, dtype=torch.float64, device="cuda", generator=g).t().contiguous().t()
Bw = B0.clone()
out["trsm_kxk_ms"] = timeit(lambda: (Bw.copy_(B0), bq.debug_trsm(T, Bw)))
out["trsm_kxk_inv_ms"] = timeit(lambda: (Bw.copy_(B0), bq.debug_trsm(T, Bw, inverse=True)))
Cg = torch.empty(k, k, dtype=torch.float64, device="cuda").t()
out["gemm_k3_ms"] = timeit(lambda: bq.debug_gemm(False, False, 1.0, B0, B0, 0.0, Cg))
print({kk: round(v, 3) for kk, v in out.items()})
