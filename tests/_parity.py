"""Per-column parity checks shared by the GPU parity tests (reading Z25 made per column).

GEQP3 output F (m x n): R = triu(F)(:l, :), reflector j = [0 .. 0, 1, F(j+1:m, j)] (unit head implicit).
Every check is per column, so a few wrong late columns cannot hide inside a Frobenius norm of the whole
matrix:
  * J identical (the caller decides when that is required);
  * R: ||R_g(:, j) - R_o(:, j)|| <= tol * ||R_o(:, j)||                for every column j;
  * V: ||v_g,j - v_o,j|| <= tol * ||v_o,j||  (||v|| >= 1: the unit head)  for every reflector j < l;
  * tau: |tau_g,j - tau_o,j| <= tol                                       (tau in [1, 2], convention H).
"""
from __future__ import annotations

import numpy as np

TOL = 1e-12


def r_cols(F: np.ndarray, l: int) -> np.ndarray:
    """R = triu(F)(:l, :) (explicit zeros below the diagonal)."""
    return np.triu(F)[:l, :]


def v_cols(F: np.ndarray, l: int) -> np.ndarray:
    """Explicit reflectors V (m x l): unit diagonal, zeros above, F below."""
    m = F.shape[0]
    V = np.tril(F[:, :l], -1)
    idx = np.arange(min(m, l))
    V[idx, idx] = 1.0
    return V


def colwise_rel(X_g: np.ndarray, X_o: np.ndarray) -> np.ndarray:
    """Per-column ||X_g(:, j) - X_o(:, j)|| / ||X_o(:, j)|| (0 where both columns are zero)."""
    d = np.linalg.norm(X_g - X_o, axis=0)
    r = np.linalg.norm(X_o, axis=0)
    with np.errstate(invalid="ignore", divide="ignore"):
        out = np.where(r > 0, d / np.where(r > 0, r, 1.0), np.where(d > 0, np.inf, 0.0))
    return out


def assert_colwise(X_g, X_o, tol=TOL, what="R"):
    rel = colwise_rel(X_g, X_o)
    if rel.size:
        j = int(np.argmax(rel))
        assert rel[j] <= tol, f"{what}: column {j} relative error {rel[j]:.3e} > {tol:.0e}"


def compare_factors(F_g, tau_g, F_o, tau_o, l, tol=TOL):
    """R and V per column, tau per entry (J already known identical)."""
    assert_colwise(r_cols(F_g, l), r_cols(F_o, l), tol, "R")
    assert_colwise(v_cols(F_g, l), v_cols(F_o, l), tol, "V")
    if l:
        dt = np.abs(np.asarray(tau_g[:l]) - np.asarray(tau_o[:l]))
        j = int(np.argmax(dt))
        assert dt[j] <= tol, f"tau[{j}] differs by {dt[j]:.3e}"
