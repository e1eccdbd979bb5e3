"""CPU oracle of BQRRP (arXiv 2507.00976) — TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline`` /
``--impl reference`` legs may import this package.  The product path
(``paper_2507_00976_b200``) never imports it, and this package never imports the product.

The arithmetic lives in ``bqrrp_oracle.c`` (plain C, fp64, ``-ffp-contract=off``); this module
only marshals numpy arrays through ctypes.  Every function cites the paper passage it follows in
the C source.  Parity status of each function is listed in DESIGN.md §6 (all pinned; the
``rank_tol`` default is a reading, Z10).
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "bqrrp_oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")

U = np.finfo(np.float64).eps / 2  # unit roundoff 2^-53


def build(force: bool = False) -> str:
    """Compile the oracle (gcc, -ffp-contract=off so expressions round as written)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        subprocess.check_call(
            ["gcc", "-O2", "-fPIC", "-shared", "-fopenmp", "-ffp-contract=off", "-o", _LIB, _SRC]
        )
    return _LIB


_lib = None


def lib() -> ctypes.CDLL:
    global _lib
    if _lib is None:
        _lib = ctypes.CDLL(build())
        d, i64, u64, u32 = ctypes.c_double, ctypes.c_int64, ctypes.c_uint64, ctypes.c_uint32
        P = ctypes.c_void_p
        _lib.oracle_philox4x32_10.argtypes = [P, P, P]
        _lib.oracle_log.argtypes = [d]
        _lib.oracle_log.restype = d
        _lib.oracle_cos2pi.argtypes = [d]
        _lib.oracle_cos2pi.restype = d
        _lib.oracle_gauss.argtypes = [u64, u32, u64, u64]
        _lib.oracle_gauss.restype = d
        _lib.oracle_sketch_operator.argtypes = [i64, i64, u64, P]
        _lib.oracle_sketch.argtypes = [i64, i64, P, i64, i64, u64, P]
        _lib.oracle_getf2.argtypes = [i64, i64, P, i64, P, P]
        _lib.oracle_piv_transform.argtypes = [i64, i64, P, P]
        _lib.oracle_col_gather.argtypes = [i64, i64, P, i64, P]
        _lib.oracle_row_gather.argtypes = [i64, i64, P, i64, P]
        _lib.oracle_vec_gather.argtypes = [i64, P, P]
        _lib.oracle_house_vec.argtypes = [i64, P]
        _lib.oracle_house_vec.restype = d
        _lib.oracle_house_qr.argtypes = [i64, i64, P, i64, i64, P]
        _lib.oracle_tri_rank.argtypes = [i64, P, i64, d]
        _lib.oracle_tri_rank.restype = i64
        _lib.oracle_sample_update.argtypes = [i64, i64, P, i64, P, i64, P, P, i64]
        _lib.oracle_bqrrp.argtypes = [i64, i64, P, i64, i64, i64, u64, d, P, P, P, P, P, P, i64, ctypes.c_int]
        _lib.oracle_bqrrp.restype = ctypes.c_int
    return _lib


def _ptr(a: np.ndarray):
    return a.ctypes.data_as(ctypes.c_void_p)


def _fortran(a, dtype=np.float64) -> np.ndarray:
    return np.array(a, dtype=dtype, order="F", copy=True)


def default_rank_tol(m: int, n: int) -> float:
    """Z10: rank_tol = 10 u sqrt(max(m, n)), relative to |R_sk^(0)(0,0)|."""
    return 10.0 * U * float(np.sqrt(max(m, n, 1)))


# ---------------------------------------------------------------- RNG
def philox4x32_10(ctr, key) -> np.ndarray:
    c = np.array(ctr, dtype=np.uint32)
    k = np.array(key, dtype=np.uint32)
    out = np.zeros(4, dtype=np.uint32)
    lib().oracle_philox4x32_10(_ptr(c), _ptr(k), _ptr(out))
    return out


def log(x: float) -> float:
    return lib().oracle_log(float(x))


def cos2pi(u: float) -> float:
    return lib().oracle_cos2pi(float(u))


def gauss(seed: int, stream: int, i: int, j: int) -> float:
    return lib().oracle_gauss(seed, stream, i, j)


def sketch_operator(d: int, m: int, seed: int) -> np.ndarray:
    S = np.zeros((d, m), order="F")
    lib().oracle_sketch_operator(d, m, seed, _ptr(S))
    return S


def sketch(A: np.ndarray, d: int, seed: int) -> np.ndarray:
    """MskT = (S A)^T, n x d."""
    A = _fortran(A)
    m, n = A.shape
    MskT = np.zeros((n, d), order="F")
    lib().oracle_sketch(m, n, _ptr(A), max(m, 1), d, seed, _ptr(MskT))
    return MskT


# ---------------------------------------------------------------- pivot selection
def getf2(L: np.ndarray):
    """LU with partial pivoting (DGETF2).  Returns (LU in place, ipiv 1-based, margins)."""
    L = _fortran(L)
    p, q = L.shape
    kmin = min(p, q)
    ipiv = np.zeros(max(kmin, 1), dtype=np.int64)
    margin = np.zeros(max(kmin, 1))
    lib().oracle_getf2(p, q, _ptr(L), max(p, 1), _ptr(ipiv), _ptr(margin))
    return L, ipiv[:kmin], margin[:kmin]


def piv_transform(w: int, Jlu) -> np.ndarray:
    Jlu = np.array(Jlu, dtype=np.int64)
    Jqr = np.zeros(max(w, 1), dtype=np.int64)
    lib().oracle_piv_transform(w, len(Jlu), _ptr(Jlu), _ptr(Jqr))
    return Jqr[:w]


def col_gather(M: np.ndarray, Jqr) -> np.ndarray:
    M = _fortran(M)
    rows, w = M.shape
    J = np.array(Jqr, dtype=np.int64)
    lib().oracle_col_gather(rows, w, _ptr(M), max(rows, 1), _ptr(J))
    return M


def vec_gather(J, Jqr) -> np.ndarray:
    J = np.array(J, dtype=np.int64)
    Jq = np.array(Jqr, dtype=np.int64)
    lib().oracle_vec_gather(len(J), _ptr(J), _ptr(Jq))
    return J


def house_vec(x):
    """Convention H reflector.  Returns (beta, v (v[0]=1), tau)."""
    x = np.array(x, dtype=np.float64)
    tau = lib().oracle_house_vec(len(x), _ptr(x))
    v = x.copy()
    beta = v[0]
    v[0] = 1.0
    return beta, v, tau


def house_qr(M: np.ndarray, kref: int | None = None):
    """Unblocked Householder QR (convention H) of the leading kref columns, applied to the rest."""
    M = _fortran(M)
    p, q = M.shape
    if kref is None:
        kref = min(p, q)
    tau = np.zeros(max(kref, 1))
    lib().oracle_house_qr(p, q, _ptr(M), max(p, 1), kref, _ptr(tau))
    return M, tau[:kref]


def tri_rank(diag, kmax: int, tol: float) -> int:
    dg = np.array(diag, dtype=np.float64)
    return int(lib().oracle_tri_rank(kmax, _ptr(dg), 1, tol))


def sample_update(Rsk11, R11, R12, MskT_tail) -> np.ndarray:
    Rsk11, R11, R12, T = _fortran(Rsk11), _fortran(R11), _fortran(R12), _fortran(MskT_tail)
    b = Rsk11.shape[0]
    t = R12.shape[1]
    lib().oracle_sample_update(b, t, _ptr(Rsk11), b, _ptr(R11), b, _ptr(R12), _ptr(T), max(t, 1))
    return T


# ---------------------------------------------------------------- driver
class OracleResult:
    def __init__(self, A, tau, J, rank, MskT, min_margin, ks):
        self.A, self.tau, self.J, self.rank = A, tau, J, rank
        self.MskT, self.min_margin, self.ks = MskT, min_margin, ks


def bqrrp(A: np.ndarray, b: int, d: int, seed: int = 0, rank_tol: float | None = None,
          max_iters: int = -1, nthreads: int = 0, want_sketch: bool = False) -> OracleResult:
    """Alg. 1 with the §3 in-place recipe.  A is copied, not modified."""
    A = _fortran(A)
    m, n = A.shape
    if rank_tol is None:
        rank_tol = default_rank_tol(m, n)
    mn = min(m, n)
    tau = np.zeros(max(mn, 1))
    J = np.zeros(max(n, 1), dtype=np.int64)
    rank = np.zeros(1, dtype=np.int64)
    MskT = np.zeros((n, d), order="F") if want_sketch else None
    mm = np.ones(1)
    nit = (mn + b - 1) // b if b > 0 else 0
    ks = np.full(max(nit, 1), -1, dtype=np.int64)
    st = lib().oracle_bqrrp(m, n, _ptr(A), max(m, 1), b, d, seed, float(rank_tol), _ptr(tau), _ptr(J),
                            _ptr(rank), _ptr(MskT) if MskT is not None else None, _ptr(mm), _ptr(ks),
                            max_iters, nthreads)
    if st != 0:
        raise ValueError(f"oracle_bqrrp: illegal argument {-st}")
    return OracleResult(A, tau[:mn], J[:n], int(rank[0]), MskT, float(mm[0]), ks[:nit])


# ---------------------------------------------------------------- checkers (numpy)
def explicit_q(A_f: np.ndarray, tau: np.ndarray, ncols: int) -> np.ndarray:
    """Q(:, :ncols) = H_1 ... H_l I(:, :ncols) from GEQP3-format reflectors.
    Uses LAPACK dorgqr (an implementation independent of the oracle) when ncols == l."""
    m = A_f.shape[0]
    l = len(tau)
    if ncols == l and 0 < l <= m:
        import scipy.linalg.lapack as la

        q, _, info = la.dorgqr(np.asfortranarray(A_f[:, :l]), np.asarray(tau, dtype=np.float64))
        assert info == 0
        return q
    return _explicit_q_loop(A_f, tau, ncols)


def _explicit_q_loop(A_f: np.ndarray, tau: np.ndarray, ncols: int) -> np.ndarray:
    m = A_f.shape[0]
    Q = np.eye(m, ncols)
    l = len(tau)
    for j in range(l - 1, -1, -1):
        if tau[j] == 0.0:
            continue
        v = np.zeros(m)
        v[j] = 1.0
        v[j + 1:] = A_f[j + 1:, j]
        Q -= tau[j] * np.outer(v, v @ Q)
    return Q


def upper_r(A_f: np.ndarray, rank: int) -> np.ndarray:
    R = np.triu(A_f)[:rank, :]
    return R


def residual(A0: np.ndarray, out: OracleResult) -> float:
    """||A0(:, J) - Q(:, :l) R(:l, :)||_F / ||A0||_F."""
    nrm = np.linalg.norm(A0)
    if nrm == 0:
        return 0.0
    l = out.rank
    Q = explicit_q(out.A, out.tau[:l], l)
    R = upper_r(out.A, l)
    return float(np.linalg.norm(A0[:, out.J - 1] - Q @ R) / nrm)


def orthogonality(out: OracleResult) -> float:
    l = out.rank
    Q = explicit_q(out.A, out.tau[:l], l)
    return float(np.linalg.norm(Q.T @ Q - np.eye(l)))


def geqrf_flops(m: int, n: int) -> float:
    """LAWN 41 GEQRF count ('canonical FLOP rate'): 2mn^2 - 2n^3/3 + mn + n^2 + 14n/3 (m >= n)."""
    if m < n:
        m, n = n, m  # LAWN41 mirrors for m < n via the transposed count; BASELINE uses square
    return 2.0 * m * n * n - 2.0 * n ** 3 / 3.0 + m * n + n * n + 14.0 * n / 3.0


def geqrf_flops_leading(m: int, n: int) -> float:
    """BASELINE.json's canonical count 2mn^2 - 2n^3/3."""
    return 2.0 * m * n * n - 2.0 * n ** 3 / 3.0


def _fro(x: np.ndarray) -> float:
    """sqrt(sum x^2), written as s sqrt(sum (x/s)^2) with s = max|x| so that no square over- or underflows."""
    x = np.abs(np.ravel(np.asarray(x, dtype=np.float64)))
    s = float(x.max()) if x.size else 0.0
    if s == 0.0:
        return 0.0
    y = x / s
    return s * float(np.sqrt(np.dot(y, y)))


def column_norms(A: np.ndarray) -> np.ndarray:
    """||A(:, j)||_2 for every column (the definition, one scaled sum of squares per column)."""
    A = np.asarray(A, dtype=np.float64)
    return np.array([_fro(A[:, j]) for j in range(A.shape[1])], dtype=np.float64)


def trailing_norms(R: np.ndarray) -> np.ndarray:
    """||R(i:, i:)||_F for i < min(m, n) of the upper trapezoid of R — the first pivot-quality metric of P:1269-1272
    ("the Frobenius norms of the trailing submatrix of the output R-factor, R(i:, i:)"), each entry taken by its
    definition: the Frobenius norm of the trailing block of triu(R) (O(min(m,n) m n): small cases; `indices` of
    trailing_norms_at for samples)."""
    return trailing_norms_at(R, range(min(R.shape)))


def trailing_norms_at(R: np.ndarray, indices) -> np.ndarray:
    """||triu(R)(i:, i:)||_F for the given i (one Frobenius norm per requested i)."""
    R = np.asarray(R, dtype=np.float64)
    mn = min(R.shape)
    out = []
    for i in indices:
        blk = np.triu(R[i:mn, i:])  # rows i..mn-1 of the upper trapezoid (triu of the block keeps j >= row)
        out.append(_fro(blk))
    return np.array(out, dtype=np.float64)
