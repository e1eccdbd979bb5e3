"""paper_2507_00976_b200 — B200-native BQRRP (arXiv 2507.00976) behind a C ABI.

This module is argument marshalling only: every step of the factorization runs in the CUDA kernels
of ``libbqrrp.so`` (sm_100a), reached through ``include/bqrrp.h`` with ctypes.  PyTorch provides
device memory and streams.  There is no CPU fallback: if the library or a CUDA device is missing,
the calls raise.
"""
from __future__ import annotations

import ctypes
import math
import os

__all__ = ["lib", "factor", "factor_host", "workspace_query", "trim_memory", "BqrrpError", "default_rank_tol", "PHASES",
           "column_norms", "trailing_norms"]

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "libbqrrp.so")
_lib = None

PHASES = ("qrcp_wide", "tri_rank", "col_perm", "qr_tall", "apply_trans_q", "sample_update", "other", "total",
          "apply_trans_q_bulk")


class BqrrpError(RuntimeError):
    def __init__(self, status: int, where: str):
        msg = f"{where}: status {status}"
        if _lib is not None:
            msg += f" ({_lib.bqrrp_strerror(status).decode()}; {_lib.bqrrp_last_error().decode()})"
        super().__init__(msg)
        self.status = status


class Options(ctypes.Structure):
    _fields_ = [("rank_tol", ctypes.c_double), ("cholqr_passes", ctypes.c_int), ("no_hqr_fallback", ctypes.c_int),
                ("phase_ms", ctypes.POINTER(ctypes.c_float)), ("no_lookahead", ctypes.c_int),
                ("dist_nb", ctypes.c_int64), ("debug_flags", ctypes.c_int), ("dist_flags", ctypes.c_int),
                ("panel_lookahead", ctypes.c_int), ("bulk_sms", ctypes.c_int),
                ("no_sqr_pipeline", ctypes.c_int), ("lu_lookahead", ctypes.c_int),
                ("lu_leaf_cluster", ctypes.c_int), ("no_sqr_merge_stream", ctypes.c_int),
                ("lu_grid_ctas", ctypes.c_int)]


def lib() -> ctypes.CDLL:
    """Load the in-tree libbqrrp.so (built by __graft_entry__.build / paper_2507_00976_b200/build.py)."""
    global _lib
    if _lib is None:
        if not os.path.exists(_LIB_PATH):
            raise ImportError(f"{_LIB_PATH} missing: run `python paper_2507_00976_b200/build.py` (nvcc, sm_100a)")
        L = ctypes.CDLL(_LIB_PATH)
        i64, u64, d, P, i32 = ctypes.c_int64, ctypes.c_uint64, ctypes.c_double, ctypes.c_void_p, ctypes.c_int
        L.bqrrp_workspace_query.argtypes = [i64, i64, i64, i64, ctypes.POINTER(ctypes.c_size_t)]
        L.bqrrp_factor_ex.argtypes = [i64, i64, P, i64, i64, i64, u64, P, P, ctypes.POINTER(i64), P, ctypes.c_size_t,
                                      P, ctypes.POINTER(Options)]
        L.bqrrp_factor_host.argtypes = [i64, i64, P, i64, i64, i64, u64, P, P, ctypes.POINTER(i64), P,
                                        ctypes.POINTER(Options)]
        L.bqrrp_debug_sketch.argtypes = [i64, i64, P, i64, i64, u64, P, P, P]
        L.bqrrp_debug_gemm.argtypes = [i32, i32, i64, i64, i64, d, P, i64, P, i64, d, P, i64, P]
        L.bqrrp_debug_lu_pivots.argtypes = [i64, i64, P, i64, P, P]
        L.bqrrp_debug_sketch_qr.argtypes = [i64, i64, P, i64, P]
        L.bqrrp_debug_permute.argtypes = [i64, i64, P, i64, i64, P, P, P]
        L.bqrrp_debug_panel.argtypes = [i64, i64, i64, P, i64, P, P, i32, P]
        L.bqrrp_debug_potrf.argtypes = [i64, P, i64, P]
        L.bqrrp_debug_recon_lu.argtypes = [i64, P, i64, P, P, P, P]
        L.bqrrp_debug_permute_touched.argtypes = [i64, P, i64, i64, P, P, P]
        L.bqrrp_column_norms.argtypes = [i64, i64, P, i64, P, P]
        L.bqrrp_trailing_norms.argtypes = [i64, i64, P, i64, P, P, ctypes.c_size_t, P]
        L.bqrrp_trailing_norms_workspace.argtypes = [i64, i64, ctypes.POINTER(ctypes.c_size_t)]
        L.bqrrp_strerror.restype = ctypes.c_char_p
        L.bqrrp_strerror.argtypes = [i32]
        L.bqrrp_last_error.restype = ctypes.c_char_p
        L.bqrrp_version.restype = ctypes.c_char_p
        L.bqrrp_launch_count.restype = ctypes.c_ulonglong
        L.bqrrp_panel_fallbacks.restype = ctypes.c_longlong
        _lib = L
    return _lib


def launch_count() -> int:
    """Kernels launched by libbqrrp.so in this process so far."""
    return int(lib().bqrrp_launch_count())


def trim_memory() -> None:
    """Return the device memory cached by the library's own pool to the driver (bqrrp_trim_memory)."""
    _check(lib().bqrrp_trim_memory(), "bqrrp_trim_memory")


def panel_fallbacks() -> int:
    """Panels of the last factor call (this thread) re-factored by Householder QR after a CholQR breakdown."""
    return int(lib().bqrrp_panel_fallbacks())


def default_rank_tol(m: int, n: int) -> float:
    """Reading Z10: 10 u sqrt(max(m, n)) relative to |R_sk^(0)(0,0)|."""
    return 10.0 * 2.0 ** -53 * math.sqrt(max(m, n, 1))


def _check(status: int, where: str):
    if status != 0:
        raise BqrrpError(status, where)


def _stream_ptr(stream=None):
    import torch

    s = stream if stream is not None else torch.cuda.current_stream()
    return ctypes.c_void_p(s.cuda_stream)


def _require_fortran_f64_cuda(A):
    import torch

    if not isinstance(A, torch.Tensor) or A.dtype != torch.float64 or not A.is_cuda or A.dim() != 2:
        raise TypeError("A must be a 2-D float64 CUDA tensor")
    if A.stride(0) != 1 and A.shape[0] > 1:
        raise ValueError("A must be column-major (Fortran order): use A.t().contiguous().t()")
    return max(A.stride(1), max(A.shape[0], 1))


def workspace_query(m: int, n: int, b: int, d: int) -> int:
    out = ctypes.c_size_t(0)
    _check(lib().bqrrp_workspace_query(m, n, b, d, ctypes.byref(out)), "bqrrp_workspace_query")
    return int(out.value)


def _options(rank_tol, cholqr_passes, phases, hqr_fallback=True, lookahead=True, debug_force_breakdown=False,
             dist_nb=0, panel_lookahead=0, bulk_sms=0, sqr_pipeline=True, lu_lookahead=False, lu_leaf_cluster=0,
             sqr_merge_stream=True, lu_grid_ctas=0):
    o = Options()
    o.lu_grid_ctas = int(lu_grid_ctas)
    o.no_sqr_merge_stream = 0 if sqr_merge_stream else 1
    o.lu_leaf_cluster = int(lu_leaf_cluster)
    o.lu_lookahead = 1 if lu_lookahead else 0
    o.no_sqr_pipeline = 0 if sqr_pipeline else 1
    o.bulk_sms = int(bulk_sms)
    o.panel_lookahead = int(panel_lookahead)
    o.dist_nb = int(dist_nb)
    o.debug_flags = 1 if debug_force_breakdown else 0
    o.no_lookahead = 0 if lookahead else 1
    o.rank_tol = float(rank_tol) if rank_tol else 0.0
    o.cholqr_passes = int(cholqr_passes)
    o.no_hqr_fallback = 0 if hqr_fallback else 1
    o.phase_ms = ctypes.cast(phases, ctypes.POINTER(ctypes.c_float)) if phases is not None else None
    return o


def factor(A, b: int, d: int | None = None, seed: int = 0, rank_tol: float | None = None, cholqr_passes: int = 2,
           workspace=None, tau=None, J=None, stream=None, phase_times: bool = False, hqr_fallback: bool = True,
           lookahead: bool = True, debug_force_breakdown: bool = False, panel_lookahead: int = 0,
           bulk_sms: int = 0, sqr_pipeline: bool = True, lu_lookahead: bool = False,
           lu_leaf_cluster: int = 0, sqr_merge_stream: bool = True, lu_grid_ctas: int = 0):
    """BQRRP of A in place (Alg. 1); returns (A, tau, J, rank[, phase_ms dict]).

    A: float64 CUDA tensor in column-major layout (m x n); overwritten in GEQP3 format.
    d: sketch rows (default b, gamma = 1 as in the paper's experiments).
    hqr_fallback: a panel whose Cholesky QR breaks down is re-factored by Householder QR (else
    BqrrpError status 1); panel_fallbacks() counts them.
    lookahead: False runs every step on one stream (phase times then measure each step alone).
    debug_force_breakdown: test hook (bqrrp_options.debug_flags): every panel reports a CholQR breakdown.
    panel_lookahead: 0 = panel i+1 after the bulk GEMM of iteration i (default), 1 = overlapped with it from a
    gathered copy (bitwise the same result).
    bulk_sms: SMs of the bulk trailing GEMM (bqrrp_options.bulk_sms): 0 = auto (a green-context partition leaving
    32 SMs to the latency-bound chain when the bulk is the shorter of the two), > 0 = always a partition of that
    size, -1 = always the whole device.  Bitwise the same result for every value.
    """
    import torch

    lda = _require_fortran_f64_cuda(A)
    m, n = A.shape
    d = b if d is None else d
    mn = min(m, n)
    if tau is None:
        tau = torch.empty(max(mn, 1), dtype=torch.float64, device=A.device)
    if J is None:
        J = torch.empty(max(n, 1), dtype=torch.int64, device=A.device)
    ws_ptr, ws_bytes = None, 0
    if workspace is not None:
        ws_ptr, ws_bytes = ctypes.c_void_p(workspace.data_ptr()), workspace.numel() * workspace.element_size()
    rank = ctypes.c_int64(0)
    phases = (ctypes.c_float * len(PHASES))() if phase_times else None
    opts = _options(rank_tol, cholqr_passes, phases, hqr_fallback, lookahead, debug_force_breakdown,
                    panel_lookahead=panel_lookahead, bulk_sms=bulk_sms, sqr_pipeline=sqr_pipeline,
                    lu_lookahead=lu_lookahead, lu_leaf_cluster=lu_leaf_cluster,
                    sqr_merge_stream=sqr_merge_stream, lu_grid_ctas=lu_grid_ctas)
    st = lib().bqrrp_factor_ex(m, n, ctypes.c_void_p(A.data_ptr()), lda, b, d, seed, ctypes.c_void_p(tau.data_ptr()),
                               ctypes.c_void_p(J.data_ptr()), ctypes.byref(rank), ws_ptr, ws_bytes,
                               _stream_ptr(stream), ctypes.byref(opts))
    _check(st, "bqrrp_factor")
    out = (A, tau[:mn], J[:n], int(rank.value))
    if phase_times:
        out = out + ({k: float(phases[i]) for i, k in enumerate(PHASES)},)
    return out


def factor_host(A_host, b: int, d: int | None = None, seed: int = 0, rank_tol: float | None = None,
                cholqr_passes: int = 2, tau_host=None, J_host=None, stream=None):
    """End-to-end: host (ideally pinned) column-major float64 tensor in, host outputs back (C-ABI
    bqrrp_factor_host: H2D copy, factorization, D2H copies inside)."""
    import torch

    if A_host.dtype != torch.float64 or A_host.is_cuda or A_host.dim() != 2:
        raise TypeError("A_host must be a 2-D float64 host tensor")
    m, n = A_host.shape
    if A_host.stride(0) != 1 and m > 1:
        raise ValueError("A_host must be column-major")
    lda = max(A_host.stride(1), max(m, 1))
    d = b if d is None else d
    mn = min(m, n)
    if tau_host is None:
        tau_host = torch.empty(max(mn, 1), dtype=torch.float64, pin_memory=True)
    if J_host is None:
        J_host = torch.empty(max(n, 1), dtype=torch.int64, pin_memory=True)
    rank = ctypes.c_int64(0)
    opts = _options(rank_tol, cholqr_passes, None)
    st = lib().bqrrp_factor_host(m, n, ctypes.c_void_p(A_host.data_ptr()), lda, b, d, seed,
                                 ctypes.c_void_p(tau_host.data_ptr()), ctypes.c_void_p(J_host.data_ptr()),
                                 ctypes.byref(rank), _stream_ptr(stream), ctypes.byref(opts))
    _check(st, "bqrrp_factor_host")
    return A_host, tau_host[:mn], J_host[:n], int(rank.value)


# ------------------------------------------------------------------ K-NORM (bqrrp_column_norms / _trailing_norms)
def column_norms(A, out=None, stream=None):
    """||A(:, j)||_2 for every column of the column-major float64 CUDA tensor A (bqrrp_column_norms)."""
    import torch

    lda = _require_fortran_f64_cuda(A)
    m, n = A.shape
    if out is None:
        out = torch.empty(max(n, 1), dtype=torch.float64, device=A.device)
    _check(lib().bqrrp_column_norms(m, n, ctypes.c_void_p(A.data_ptr()), lda, ctypes.c_void_p(out.data_ptr()),
                                    _stream_ptr(stream)), "bqrrp_column_norms")
    return out[:n]


def trailing_norms_workspace(m: int, n: int) -> int:
    out = ctypes.c_size_t(0)
    _check(lib().bqrrp_trailing_norms_workspace(m, n, ctypes.byref(out)), "bqrrp_trailing_norms_workspace")
    return int(out.value)


def trailing_norms(R, out=None, workspace=None, stream=None):
    """||R(i:, i:)||_F for i < min(m, n) of the upper trapezoid of R (bqrrp_trailing_norms)."""
    import torch

    ldr = _require_fortran_f64_cuda(R)
    m, n = R.shape
    mn = min(m, n)
    if out is None:
        out = torch.empty(max(mn, 1), dtype=torch.float64, device=R.device)
    ws_ptr, ws_bytes = None, 0
    if workspace is not None:
        ws_ptr, ws_bytes = ctypes.c_void_p(workspace.data_ptr()), workspace.numel() * workspace.element_size()
    _check(lib().bqrrp_trailing_norms(m, n, ctypes.c_void_p(R.data_ptr()), ldr, ctypes.c_void_p(out.data_ptr()),
                                      ws_ptr, ws_bytes, _stream_ptr(stream)), "bqrrp_trailing_norms")
    return out[:mn]


# ------------------------------------------------------------------ debug entry points (tests)
def debug_sketch(A, d: int, seed: int, want_S: bool = True):
    import torch

    lda = _require_fortran_f64_cuda(A)
    m, n = A.shape
    MskT = torch.empty((d, n), dtype=torch.float64, device=A.device).t()
    S = torch.empty((m, d), dtype=torch.float64, device=A.device).t() if want_S else None
    _check(lib().bqrrp_debug_sketch(m, n, ctypes.c_void_p(A.data_ptr()), lda, d, seed,
                                    ctypes.c_void_p(S.data_ptr()) if S is not None else None,
                                    ctypes.c_void_p(MskT.data_ptr()), _stream_ptr()), "bqrrp_debug_sketch")
    return S, MskT


def debug_gemm(ta: bool, tb: bool, alpha, A, B, beta, C):
    M, N = C.shape
    K = A.shape[0] if ta else A.shape[1]
    _check(lib().bqrrp_debug_gemm(int(ta), int(tb), M, N, K, float(alpha), ctypes.c_void_p(A.data_ptr()),
                                  _require_fortran_f64_cuda(A), ctypes.c_void_p(B.data_ptr()),
                                  _require_fortran_f64_cuda(B), float(beta), ctypes.c_void_p(C.data_ptr()),
                                  _require_fortran_f64_cuda(C), _stream_ptr()), "bqrrp_debug_gemm")
    return C


def debug_trsm(T, B, t_lower: bool = False, unit: bool = False, inverse: bool = False):
    """B <- B op(T)^{-1} in place (bqrrp_debug_trsm)."""
    rows, n = B.shape
    L = lib()
    L.bqrrp_debug_trsm.argtypes = [ctypes.c_int64, ctypes.c_int64, ctypes.c_void_p, ctypes.c_int64, ctypes.c_int,
                                   ctypes.c_int, ctypes.c_int, ctypes.c_void_p, ctypes.c_int64, ctypes.c_void_p]
    _check(L.bqrrp_debug_trsm(rows, n, ctypes.c_void_p(T.data_ptr()), _require_fortran_f64_cuda(T), int(t_lower),
                              int(unit), int(inverse), ctypes.c_void_p(B.data_ptr()), _require_fortran_f64_cuda(B),
                              _stream_ptr()), "bqrrp_debug_trsm")
    return B


def debug_lu_pivots(L):
    import torch

    ld = _require_fortran_f64_cuda(L)
    w, d = L.shape
    ipiv = torch.zeros(max(min(w, d), 1), dtype=torch.int64, device=L.device)
    _check(lib().bqrrp_debug_lu_pivots(w, d, ctypes.c_void_p(L.data_ptr()), ld, ctypes.c_void_p(ipiv.data_ptr()),
                                       _stream_ptr()), "bqrrp_debug_lu_pivots")
    return L, ipiv[: min(w, d)]


def debug_sketch_qr(WT):
    ld = _require_fortran_f64_cuda(WT)
    w, d = WT.shape
    _check(lib().bqrrp_debug_sketch_qr(w, d, ctypes.c_void_p(WT.data_ptr()), ld, _stream_ptr()),
           "bqrrp_debug_sketch_qr")
    return WT


def debug_permute(X, ipiv):
    import torch

    ld = _require_fortran_f64_cuda(X)
    rows, w = X.shape
    Jqr = torch.zeros(max(w, 1), dtype=torch.int64, device=X.device)
    _check(lib().bqrrp_debug_permute(rows, w, ctypes.c_void_p(X.data_ptr()), ld, ipiv.numel(),
                                     ctypes.c_void_p(ipiv.data_ptr()), ctypes.c_void_p(Jqr.data_ptr()),
                                     _stream_ptr()), "bqrrp_debug_permute")
    return X, Jqr[:w]


def debug_permute_touched(X, tq, tsrc, stream=None):
    """X(:, tq[t]) = X_old(:, tsrc[t]) (int32 CUDA tensors; bqrrp_debug_permute_touched)."""
    ld = _require_fortran_f64_cuda(X)
    rows = X.shape[0]
    _check(lib().bqrrp_debug_permute_touched(rows, ctypes.c_void_p(X.data_ptr()), ld, tq.numel(),
                                             ctypes.c_void_p(tq.data_ptr()), ctypes.c_void_p(tsrc.data_ptr()),
                                             _stream_ptr(stream)), "bqrrp_debug_permute_touched")
    return X


def debug_panel(P, k: int, Rsk11, cholqr_passes: int = 2):
    """P: h x (k + t) column-major; first k columns are the panel, the rest the trailing block."""
    import torch

    ld = _require_fortran_f64_cuda(P)
    h, cols = P.shape
    tau = torch.zeros(k, dtype=torch.float64, device=P.device)
    R = Rsk11.t().contiguous().t()
    _check(lib().bqrrp_debug_panel(h, k, cols - k, ctypes.c_void_p(P.data_ptr()), ld, ctypes.c_void_p(R.data_ptr()),
                                   ctypes.c_void_p(tau.data_ptr()), cholqr_passes, _stream_ptr()), "bqrrp_debug_panel")
    return P, tau
