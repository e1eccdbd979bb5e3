"""Pins for the oracle's building blocks: LU pivoting, pivot formats, gathers, Householder
convention H, tri_rank, sample update, flop counts.

What pins them (never the oracle's own formula re-typed):
  * SPEC worked examples (tests/golden/spec_examples.json, each with its S:/P: citation);
  * LAPACK via scipy/numpy (dgetrf pivots, dgeqrf reflectors + tau share convention H on
    inputs with nonzero tails);
  * Alg. 4's sequential swap/find/update permutation — a different algorithm with the
    same result as the gather — exhaustively for n <= 6;
  * replay identities (P.T = L.U), |L| <= 1, Q^T A = R, orthogonality.
"""
import itertools
import json
import os

import numpy as np
import pytest
import scipy.linalg

import inputs
import oracle

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "spec_examples.json")))


# ------------------------------------------------------------------ LU (Alg. 2)
def test_getf2_spec_examples():
    for ex in GOLD["getf2"]:
        LU, ipiv, _ = oracle.getf2(np.array(ex["A"], dtype=float))
        assert list(ipiv) == ex["ipiv"], ex["cite"]
        if "U" in ex:
            assert np.array_equal(np.triu(LU), np.array(ex["U"], dtype=float)), ex["cite"]
        if "L10" in ex:
            assert LU[1, 0] == ex["L10"]


@pytest.mark.parametrize("shape", [(64, 16), (200, 40), (33, 33), (20, 50)])
def test_getf2_pivots_match_lapack_dgetrf(shape):
    A = inputs.gaussian(*shape, seed=sum(shape))
    LU, ipiv, _ = oracle.getf2(A)
    lu_ref, piv_ref = scipy.linalg.lu_factor(A)
    assert np.array_equal(ipiv, piv_ref[: len(ipiv)] + 1)
    assert np.allclose(LU, lu_ref, rtol=0, atol=1e-12 * np.abs(lu_ref).max())


def test_getf2_replay_and_bounded_multipliers():
    A = inputs.gaussian(120, 30, seed=8)
    LU, ipiv, margin = oracle.getf2(A)
    p, q = A.shape
    PA = A.copy()
    for j, pv in enumerate(ipiv):  # replay the swap list on A (P:587-589 semantics)
        PA[[j, pv - 1]] = PA[[pv - 1, j]]
    L = np.tril(LU, -1)[:, :q] + np.eye(p, q)
    U = np.triu(LU)[:q]
    assert np.linalg.norm(PA - L @ U) <= 1e-13 * np.linalg.norm(A)
    assert np.abs(np.tril(LU, -1)).max() <= 1.0
    assert np.all((margin >= 0) & (margin <= 1))


def test_getf2_first_index_tie_break_and_zero_column():
    # all candidates tie in |.|: IDAMAX picks the first (Z19)
    A = np.array([[1.0, 2.0], [-1.0, 5.0], [1.0, 7.0]])
    _, ipiv, margin = oracle.getf2(A)
    assert ipiv[0] == 1 and margin[0] == 0.0
    A = np.array([[0.0, 1.0], [-2.0, 5.0], [2.0, 7.0]])
    _, ipiv, _ = oracle.getf2(A)
    assert ipiv[0] == 2
    # exact zero pivot column: no swap, continue (Z18)
    A = np.array([[0.0, 1.0], [0.0, 3.0], [0.0, 2.0]])
    LU, ipiv, _ = oracle.getf2(A)
    assert ipiv[0] == 1 and ipiv[1] == 2
    assert np.array_equal(LU[:, 0], [0.0, 0.0, 0.0])
    # integer matrices: LAPACK's IDAMAX agrees exactly
    for seed in range(20):
        A = inputs.integer_valued(7, 4, seed=seed, lo=-2, hi=2)
        if np.linalg.matrix_rank(A) < 4:
            continue
        _, ipiv, _ = oracle.getf2(A)
        _, piv_ref = scipy.linalg.lu_factor(A)
        assert np.array_equal(ipiv, piv_ref[:4] + 1), seed


# ------------------------------------------------------------------ pivot formats / gathers
def test_piv_transform_spec_examples():
    for ex in GOLD["piv_transform"]:
        assert list(oracle.piv_transform(ex["w"], ex["Jlu"])) == ex["Jqr"], ex["cite"]


def test_piv_transform_gather_reproduces_swap_replay_exhaustive():
    """piv_transform + gather == replaying the LU swap list on the rows, all swap lists n <= 5."""
    for n in range(1, 6):
        for nlu in range(0, n + 1):
            for Jlu in itertools.product(*[range(j + 1, n + 1) for j in range(nlu)]):
                Jqr = oracle.piv_transform(n, Jlu)
                rows = np.arange(n)
                for j, pv in enumerate(Jlu):
                    rows[[j, pv - 1]] = rows[[pv - 1, j]]
                assert np.array_equal(Jqr - 1, rows)
                assert sorted(Jqr) == list(range(1, n + 1))


def _alg4_sequential(M, J):
    """Alg. 4 as printed: swap, find, update J — a different algorithm from the gather."""
    M = M.copy()
    J = list(J)
    for i in range(len(J)):
        j = J[i] - 1
        M[:, [i, j]] = M[:, [j, i]]
        # "find the index of an element with value i+1": searched in the unprocessed tail
        # J(i+1:) (reading Z31; positions <= i are final and may hold i+1 themselves)
        if i + 1 < len(J) and (i + 1) in J[i + 1:]:
            idx = J.index(i + 1, i + 1)
            J[idx] = j + 1
    return M


def test_gather_equals_sequential_alg4_exhaustive():
    for n in range(1, 7):
        M = np.arange(3 * n, dtype=float).reshape(3, n, order="F")
        for perm in itertools.permutations(range(1, n + 1)):
            g = oracle.col_gather(M, perm)
            assert np.array_equal(g, _alg4_sequential(M, perm))
            assert np.array_equal(g, M[:, np.array(perm) - 1])


def test_gather_spec_examples_and_round_trip():
    ex = GOLD["gather"][0]
    M = np.array([[0.0, 1.0, 2.0]])
    assert list(oracle.col_gather(M, ex["J"])[0]) == [0.0 + int(c[1]) for c in ex["out"]]
    ex = GOLD["gather"][1]
    assert list(oracle.vec_gather(ex["J_tail"], ex["J_local"])) == ex["out"]
    rng = np.random.default_rng(0)
    M = rng.standard_normal((5, 9))
    J = rng.permutation(9) + 1
    Jinv = np.argsort(J - 1) + 1
    assert np.array_equal(oracle.col_gather(oracle.col_gather(M, J), Jinv), M)


# ------------------------------------------------------------------ Householder (convention H)
def test_house_vec_spec_examples():
    for ex in GOLD["house_vec"]:
        beta, v, tau = oracle.house_vec(ex["x"])
        assert beta == ex["beta"] and tau == ex["tau"], ex["cite"]
        assert np.allclose(v, ex["v"], rtol=0, atol=1e-16), ex["cite"]
        x = np.array(ex["x"])
        H = np.eye(len(x)) - tau * np.outer(v, v)
        e1 = np.zeros(len(x))
        e1[0] = beta
        assert np.allclose(H @ x, e1, atol=1e-15)


@pytest.mark.parametrize("shape", [(64, 16), (50, 50), (30, 45), (200, 7)])
def test_house_qr_matches_lapack_dgeqrf(shape):
    """numpy's raw QR is LAPACK dgeqrf: same reflectors/tau (beta = -sgn(alpha)||x||) when tails are nonzero."""
    A = inputs.gaussian(*shape, seed=shape[0] * 7 + shape[1])
    F, tau = oracle.house_qr(A)
    h, tau_ref = np.linalg.qr(A, mode="raw")
    ref = h.T
    m, n = shape
    k = min(m - 1, n)  # reflectors with a nonzero tail: LAPACK dlarfg == convention H
    assert np.allclose(tau[:k], tau_ref[:k], rtol=0, atol=1e-14)
    assert np.linalg.norm(F[:, :k] - ref[:, :k]) <= 1e-13 * np.linalg.norm(ref)
    if m <= n:
        # length-1 reflector (Z9): LAPACK returns tau = 0, beta = x0; convention H tau = 2, beta = -x0
        assert tau_ref[m - 1] == 0.0 and tau[m - 1] == 2.0
        assert np.allclose(F[m - 1, m - 1:], -ref[m - 1, m - 1:], rtol=1e-12, atol=1e-12)
        assert np.linalg.norm(F[:m - 1, k:] - ref[:m - 1, k:]) <= 1e-13 * np.linalg.norm(ref)
    else:
        assert np.linalg.norm(F - ref) <= 1e-13 * np.linalg.norm(ref)


def test_house_qr_identity_convention_h():
    """Z9: QR of I gives R = -I and tau = 2 on every column (every tail is zero)."""
    F, tau = oracle.house_qr(np.eye(4))
    assert np.array_equal(np.diag(F), -np.ones(4))
    assert np.array_equal(tau, 2 * np.ones(4))


def test_house_qr_qt_a_is_r_and_orthogonal():
    A = inputs.gaussian(80, 20, seed=1)
    F, tau = oracle.house_qr(A)
    Q = oracle.explicit_q(F, tau, 80)
    assert np.linalg.norm(Q.T @ Q - np.eye(80)) < 1e-13
    QtA = Q.T @ A
    assert np.linalg.norm(QtA - np.triu(F)[:80]) <= 1e-13 * np.linalg.norm(A)
    assert np.all((tau >= 1) & (tau <= 2))


# ------------------------------------------------------------------ tri_rank, sample update
def test_tri_rank_spec_examples():
    for ex in GOLD["tri_rank"]:
        tol = oracle.default_rank_tol(3, 3) * abs(ex["diag"][0])
        k = oracle.tri_rank(ex["diag"], ex["kmax"], tol) if ex["diag"][0] != 0 else 0
        assert k == ex["k"], ex["cite"]


def test_sample_update_scalar_example():
    ex = GOLD["sample_update"][0]
    out = oracle.sample_update([[ex["Rsk11"]]], [[ex["R11"]]], [[ex["R12"]]], [[ex["Rsk12"]]])
    assert out[0, 0] == ex["out"]


def test_sample_update_dense_bracket_expression():
    """Alg. 1 step 24: top block = R_sk12 - R_sk11 R11^{-1} R12 to <= 8u, against the exact
    value of the bracket expression (50-digit mpmath, no shared rounding with any fp64 routine): normwise
    and componentwise relative to the expression's natural scale |R_sk12| + |R_sk11| |R11^{-1} R12|."""
    import mpmath

    mpmath.mp.dps = 50
    rng = np.random.default_rng(4)
    M = lambda a: mpmath.matrix(np.asarray(a).tolist())  # noqa: E731
    for _ in range(20):
        b, t = 4, 16
        Rsk11 = np.triu(rng.standard_normal((b, b))) + 3 * np.eye(b)
        R11 = np.triu(rng.standard_normal((b, b))) + 3 * np.eye(b)
        R12 = rng.standard_normal((b, t))
        Rsk12 = rng.standard_normal((b, t))
        out = oracle.sample_update(Rsk11, R11, R12, Rsk12.T.copy()).T
        exact = M(Rsk12) - M(Rsk11) * (mpmath.inverse(M(R11)) * M(R12))
        err = np.array((M(out) - exact).tolist(), dtype=float)
        ref = np.array(exact.tolist(), dtype=float)
        assert np.linalg.norm(err) <= 8 * oracle.U * np.linalg.norm(ref)
        scale = np.abs(Rsk12) + np.abs(Rsk11) @ np.abs(scipy.linalg.solve_triangular(R11, R12, lower=False))
        assert np.all(np.abs(err) <= 8 * oracle.U * scale)


def test_flop_counts():
    for ex in GOLD["geqrf_flops"]:
        assert abs(oracle.geqrf_flops(ex["m"], ex["n"]) - ex["flops"]) <= 1e-12 * ex["flops"], ex["cite"]
    for ex in GOLD["ormqr_flops"]:
        n, m, k = ex["n"], ex["m"], ex["k"]
        assert 4 * n * m * k - 2 * n * k * k + 3 * n * k == ex["flops"]
