"""Seeded synthetic inputs shared by the oracle and the CUDA path (DESIGN.md §5 "input recipe").

This module holds NO arithmetic of the method: it only draws test matrices of the shapes and
value distributions of the paper's workloads (iid N(0,1) entries, "each matrix entry is
independently sampled from the standard normal distribution"; rank-deficient and graded-spectrum
variants for the rank / pivot-quality checks).  Host generation uses numpy's PCG64; the
device generator (large bench sizes) is a counter-based splitmix64 hash + Box-Muller in torch ops
(`counter_gaussian`: a pure function of (seed, i, j), independent of torch's RNG) — both plumbing,
neither is the sketch RNG of the method (Philox, implemented separately on each side).
"""
from __future__ import annotations

import numpy as np


def gaussian(m: int, n: int, seed: int = 0) -> np.ndarray:
    """m x n, iid N(0,1), Fortran order."""
    rng = np.random.default_rng(seed)
    return np.asfortranarray(rng.standard_normal((m, n)))


def integer_valued(m: int, n: int, seed: int = 0, lo: int = -4, hi: int = 4) -> np.ndarray:
    """Small integers (exact products and sums: bit-exact GEMM checks)."""
    rng = np.random.default_rng(seed)
    return np.asfortranarray(rng.integers(lo, hi + 1, size=(m, n)).astype(np.float64))


def low_rank(m: int, n: int, k: int, seed: int = 0) -> np.ndarray:
    """A = G1 G2^T with Gaussian G1 (m x k), G2 (n x k): exact rank k (SURVEY P-DRV)."""
    rng = np.random.default_rng(seed)
    G1 = rng.standard_normal((m, k))
    G2 = rng.standard_normal((n, k))
    return np.asfortranarray(G1 @ G2.T)


def orthonormal(m: int, k: int, seed: int) -> np.ndarray:
    rng = np.random.default_rng(seed)
    Q, _ = np.linalg.qr(rng.standard_normal((m, k)))
    return Q


def graded(m: int, n: int, rank: int, sigma_last: float = 1e-14, seed: int = 0):
    """A = X diag(sigma) Y^T, sigma_i = sigma_last^(i/(rank-1)) (geometric decay, BASELINE C5 / Z30).
    Returns (A, sigma)."""
    X = orthonormal(m, rank, seed)
    Y = orthonormal(n, rank, seed + 7919)
    i = np.arange(rank)
    sigma = sigma_last ** (i / max(rank - 1, 1))
    return np.asfortranarray((X * sigma) @ Y.T), sigma


def separated_columns(m: int, n: int, ratio: float = 1e4, seed: int = 0):
    """A = Q_A diag(c) Pi with c_j = ratio^-j and a random column shuffle Pi (SURVEY P-GEQP3).
    Returns (A, expected 1-based GEQP3 order)."""
    rng = np.random.default_rng(seed)
    QA, _ = np.linalg.qr(rng.standard_normal((m, n)))
    c = ratio ** (-np.arange(n, dtype=np.float64))
    perm = rng.permutation(n)  # column j of A is scaled column perm[j]
    A = QA[:, perm] * c[perm]
    order = np.argsort(perm, kind="stable") + 1  # A's columns sorted by descending c
    return np.asfortranarray(A), order


def kahan(n: int, theta: float = 1.2, p: float = 1000.0) -> np.ndarray:
    """Classical Kahan matrix (reading Z27): K = diag(1, s, ..., s^(n-1)) (I - c U_strict),
    s = sin(theta), c = cos(theta), plus the perturbation eps*p*diag(n, ..., 1)... kept as the
    removed generator of P:1321-1347 prints it: a tiny diagonal perturbation to break ties."""
    s, c = np.sin(theta), np.cos(theta)
    K = np.triu(-c * np.ones((n, n)), 1) + np.eye(n)
    K = np.diag(s ** np.arange(n)) @ K
    K += np.finfo(np.float64).eps * p * np.diag(np.arange(n, 0, -1, dtype=np.float64))
    return np.asfortranarray(K)


# ---- counter-based N(0,1) for the large (device) inputs: entry (i, j) is a pure function of (seed, i, j), so the
# bench matrices do not depend on the torch version's RNG.  A splitmix64 finaliser of the linear index (a generic
# 64-bit hash, not the method's Philox sketch generator) gives two 53-bit uniforms, Box-Muller the normal.
_GOLDEN = -7046029254386353131  # 0x9E3779B97F4A7C15 as int64
_M1 = -4658895280553007687  # 0xBF58476D1CE4E5B9
_M2 = -7723592293110705685  # 0x94D049BB133111EB


def _splitmix64_torch(x):
    """splitmix64 finaliser on int64 tensors (wrapping multiplies; logical shifts by masking)."""
    x = x ^ ((x >> 30) & ((1 << 34) - 1))
    x = x * _M1
    x = x ^ ((x >> 27) & ((1 << 37) - 1))
    x = x * _M2
    return x ^ ((x >> 31) & ((1 << 33) - 1))


def counter_gaussian(m: int, n: int, seed: int = 0, device: str = "cuda", chunk: int = 1 << 26):
    """m x n column-major (Fortran-strided view) iid N(0,1): entry (i, j) from the 64-bit hash of the linear index
    i + j m and the seed.  Identical on any device and torch version up to the last ulp of log/cos."""
    import torch

    out = torch.empty((n, m), dtype=torch.float64, device=device)
    flat = out.view(-1)  # column-major: flat[i + j m]
    key = (int(seed) * 0x632BE59BD9B4E019) & ((1 << 63) - 1)
    two53 = 2.0 ** -53
    for lo in range(0, m * n, chunk):
        hi = min(m * n, lo + chunk)
        idx = torch.arange(lo, hi, dtype=torch.int64, device=device)
        base = idx * 2 * _GOLDEN + key
        h1 = _splitmix64_torch(base)
        h2 = _splitmix64_torch(base + _GOLDEN)
        u1 = (((h1 >> 11) & ((1 << 53) - 1)).to(torch.float64) + 0.5) * two53  # (0, 1)
        u2 = ((h2 >> 11) & ((1 << 53) - 1)).to(torch.float64) * two53  # [0, 1)
        flat[lo:hi] = torch.sqrt(-2.0 * torch.log(u1)) * torch.cos((2.0 * torch.pi) * u2)
        del idx, base, h1, h2, u1, u2
    return out.t()


def gaussian_cuda(m: int, n: int, seed: int = 0, device: str = "cuda"):
    """Device-side N(0,1) matrix (m x n, Fortran-strided view): the counter-based generator above."""
    return counter_gaussian(m, n, seed=seed, device=device)
