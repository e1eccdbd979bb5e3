"""Pins of the oracle's K-NORM definitions (oracle.column_norms / trailing_norms), against what the mathematics
fixes rather than a retyped formula:

  * the paper's own interpretation of the first pivot-quality metric: ||R(i:, i:)||_F is the
    residual ||A - Q(:, :i) R(:i, :)||_F of the rank-i approximation — checked with LAPACK's QR (numpy) and the
    explicit product, a different computation;
  * closed forms: the identity (sqrt(n - i)), a diagonal (suffix sums of squares), orthonormal columns scaled by c;
  * invariants: ||R(0:, 0:)||_F = ||A||_F, entries below the diagonal ignored, the wide case.
"""
import numpy as np
import pytest

import oracle


def test_trailing_identity_closed_form():
    n = 17
    got = oracle.trailing_norms(np.eye(n))
    assert np.allclose(got, np.sqrt(n - np.arange(n)), rtol=0, atol=1e-15)


def test_trailing_diagonal_suffix_sums():
    d = np.array([3.0, -4.0, 12.0, 0.0, 5.0])
    got = oracle.trailing_norms(np.diag(d))
    want = np.sqrt(np.array([194.0, 185.0, 169.0, 25.0, 25.0]))  # 9+16+144+0+25, ...
    assert np.allclose(got, want, rtol=4e-16, atol=0)


@pytest.mark.parametrize("m,n", [(30, 20), (20, 20), (12, 25)])
def test_trailing_is_rank_i_residual(m, n):
    """||R(i:, i:)||_F = ||A - Q(:, :i) R(:i, :)||_F for A = Q R (LAPACK QR via numpy)."""
    rng = np.random.default_rng(m * 100 + n)
    A = rng.standard_normal((m, n))
    Q, R = np.linalg.qr(A, mode="complete")
    mn = min(m, n)
    got = oracle.trailing_norms(R)
    want = np.array([np.linalg.norm(A - Q[:, :i] @ R[:i, :]) for i in range(mn)])
    assert np.allclose(got, want, rtol=1e-13, atol=0)
    assert abs(got[0] - np.linalg.norm(A)) <= 1e-13 * np.linalg.norm(A)


def test_trailing_ignores_strict_lower_part():
    rng = np.random.default_rng(5)
    R = np.triu(rng.standard_normal((15, 11)))
    G = R + np.tril(rng.standard_normal((15, 11)), -1) * 1e3
    assert np.array_equal(oracle.trailing_norms(R), oracle.trailing_norms(G))


def test_trailing_at_matches_full():
    rng = np.random.default_rng(6)
    R = rng.standard_normal((9, 14))
    full = oracle.trailing_norms(R)
    idx = [0, 3, 8]
    assert np.array_equal(oracle.trailing_norms_at(R, idx), full[idx])


def test_column_norms_closed_forms():
    assert np.array_equal(oracle.column_norms(np.array([[3.0, 0.0], [4.0, -2.0]])), np.array([5.0, 2.0]))
    rng = np.random.default_rng(1)
    Q, _ = np.linalg.qr(rng.standard_normal((40, 6)))
    c = np.array([1.0, 1e-200, 1e200, 3.5, 0.0, 1e-300])
    got = oracle.column_norms(Q * c)
    assert np.allclose(got[[0, 1, 2, 3, 5]], c[[0, 1, 2, 3, 5]], rtol=1e-14, atol=0)
    assert got[4] == 0.0
