"""Pins for the oracle driver (Alg. 1, with the §3 in-place recipe).

What pins it:
  * invariants the paper fixes: GEQP3 output format, ||A P - Q R|| / ||A|| <= 1e-13,
    ||Q^T Q - I|| <= 1e-13 (north_star, literal at these sizes, Z24), R upper-trapezoidal;
  * the Duersch-Gu sketch update's closed form (P:517 derivation): after iteration 0 the
    updated sketch equals Q_sk^T (S Q)(:, b:) A22, built here with numpy from S, the explicit Q
    and LAPACK's QR of the permuted sketch;
  * special cases that reduce to library routines: the single-panel collapse (b >= n) gives
    J = LAPACK-LU pivots of the sketch transpose and R = LAPACK QR of A(:, J);
  * exact rank recovery on A = G1 G2^T; the zero matrix; brute-force GEQP3 order on columns with
    well-separated norms; the P:603 gamma-prefix invariance; bitwise determinism and
    thread-count independence.
"""
import numpy as np
import pytest
import scipy.linalg

import inputs
import oracle


def _check_format(out, m, n):
    l = out.rank
    assert 0 <= l <= min(m, n)
    assert sorted(out.J) == list(range(1, n + 1))
    assert np.all(out.tau[l:] == 0)
    assert np.all(out.A[l:, l:] == 0)
    t = out.tau[:l]
    assert np.all((t >= 1 - 1e-12) & (t <= 2 + 1e-12))


@pytest.mark.parametrize("shape,b", [((256, 256), 8), ((256, 256), 32), ((256, 64), 16), ((64, 256), 16),
                                     ((100, 100), 32), ((128, 128), 64), ((96, 80), 96), ((300, 120), 50)])
def test_residual_and_orthogonality(shape, b):
    m, n = shape
    A = inputs.gaussian(m, n, seed=m + n + b)
    d = min(m, -(-5 * b // 4))
    d = max(d, b) if b <= m else m
    if b > m:
        b = m
    out = oracle.bqrrp(A, b, d, seed=1)
    _check_format(out, m, n)
    assert out.rank == min(m, n)
    assert oracle.residual(A, out) <= 1e-13
    assert oracle.orthogonality(out) <= 1e-13


def test_c1_config():
    """BASELINE C1: 1024^2 Gaussian, b=128, d=1.25b=160, seed 0 (SURVEY d.1)."""
    A = inputs.gaussian(1024, 1024, seed=0)
    out = oracle.bqrrp(A, 128, 160, seed=0)
    _check_format(out, 1024, 1024)
    assert out.rank == 1024
    assert oracle.residual(A, out) <= 1e-13
    assert oracle.orthogonality(out) <= 1e-13
    assert out.min_margin > 1e-10  # pivots well separated: GPU parity on J is expected (SURVEY c.6)


def test_zero_matrix():
    """M = 0 -> l = 0, J = identity, tau = 0."""
    out = oracle.bqrrp(np.zeros((8, 8)), 4, 4, seed=0)
    assert out.rank == 0
    assert list(out.J) == list(range(1, 9))
    assert np.all(out.tau == 0) and np.all(out.A == 0)


def test_empty():
    out = oracle.bqrrp(np.zeros((4, 0)), 2, 2, seed=0)
    assert out.rank == 0


@pytest.mark.parametrize("m,n", [(64, 16), (40, 40), (50, 30)])
def test_single_panel_collapse(m, n):
    """b >= n: J = pivots of LAPACK LU on the sketch transpose; R, tau = LAPACK QR of A(:, J)."""
    A = inputs.gaussian(m, n, seed=m * n)
    b = n
    d = n
    out = oracle.bqrrp(A, b, d, seed=3)
    # the sketch itself is pinned against S @ A in test_oracle_rng; LU pivots via LAPACK dgetrf
    S = oracle.sketch_operator(d, m, seed=3)
    _, piv = scipy.linalg.lu_factor((S @ A).T)
    Jqr = np.arange(n)
    for j, p in enumerate(piv[: min(n, d)]):
        Jqr[[j, p]] = Jqr[[p, j]]
    assert np.array_equal(out.J - 1, Jqr)
    h, tau_ref = np.linalg.qr(A[:, out.J - 1], mode="raw")
    ref = h.T
    k = min(m - 1, n)
    assert np.linalg.norm(np.triu(out.A)[:, :k] - np.triu(ref)[:, :k]) <= 1e-13 * np.linalg.norm(A)
    assert np.linalg.norm(np.tril(out.A, -1) - np.tril(ref, -1)) <= 1e-12 * np.linalg.norm(np.tril(ref, -1))
    assert np.allclose(out.tau[:k], tau_ref[:k], atol=1e-13)


@pytest.mark.parametrize("k_true", [16, 32, 55])
def test_exact_rank_recovery(k_true):
    """A = G1 G2^T (rank k) -> l = k (SURVEY P-DRV; B3 tolerance window)."""
    m = n = 128
    b = 32
    A = inputs.low_rank(m, n, k_true, seed=k_true)
    out = oracle.bqrrp(A, b, 40, seed=0)
    assert out.rank == k_true
    _check_format(out, m, n)
    assert oracle.residual(A, out) <= 1e-13


def test_rank_deficient_ell_window():
    """SPEC acceptance: rank-r inputs terminate with l in [r, r+b] (here l == r)."""
    for r in (0, 16, 48):
        A = inputs.low_rank(128, 128, r, seed=5) if r > 0 else np.zeros((128, 128))
        out = oracle.bqrrp(A, 32, 32, seed=2)
        assert r <= out.rank <= r + 32


def test_geqp3_agreement_well_separated():
    """P-GEQP3: columns with norms 1, 1e-4, 1e-8, 1e-12 (shuffled): the pivot order is the sort
    order of the norms, which brute-force GEQP3 gives; b in {1, n}. >= 99 of 100 seeds."""
    ok = 0
    for seed in range(100):
        A, order = inputs.separated_columns(16, 4, ratio=1e4, seed=seed)
        good = True
        for b in (1, 4):
            out = oracle.bqrrp(A, b, b, seed=seed + 1000)
            good &= np.array_equal(out.J, order)
        ok += good
    assert ok >= 99


def test_geqp3_brute_force_reference_order():
    """The brute-force GEQP3 (argmax of recomputed trailing norms, lowest index on ties) used above."""
    A, order = inputs.separated_columns(16, 4, ratio=1e4, seed=0)
    R = A.copy()
    J = list(range(4))
    for i in range(4):
        nrm = np.linalg.norm(R[i:, i:], axis=0)
        p = i + int(np.argmax(nrm))
        R[:, [i, p]] = R[:, [p, i]]
        J[i], J[p] = J[p], J[i]
        Q, _ = np.linalg.qr(R[i:, i:i + 1], mode="complete")
        R[i:, i:] = Q.T @ R[i:, i:]
    assert np.array_equal(np.array(J) + 1, order)


def test_gamma_prefix_invariance():
    """the first b components of J_qr are the same for gamma = 1 and gamma > 1 (i = 0)."""
    A = inputs.gaussian(200, 160, seed=9)
    b = 32
    o1 = oracle.bqrrp(A, b, b, seed=4, max_iters=1)
    o2 = oracle.bqrrp(A, b, 40, seed=4, max_iters=1)
    assert np.array_equal(o1.J[:b], o2.J[:b])


def test_sketch_update_closed_form():
    """with S Q = [S1 S2], the updated sketch equals Q_sk^T S2 A22 (exact identity)."""
    m, n, b, d = 120, 96, 24, 30
    A = inputs.gaussian(m, n, seed=12)
    out = oracle.bqrrp(A, b, d, seed=6, max_iters=1, want_sketch=True)
    assert out.rank == -1  # state after one iteration, not finalised
    S = oracle.sketch_operator(d, m, seed=6)
    J0 = out.J - 1
    Wsk = S @ A[:, J0]  # the permuted sketch (the oracle permutes the same way, pinned separately)
    h, tau_sk = np.linalg.qr(Wsk, mode="raw")  # LAPACK: Q_sk with convention-H signs
    Qsk = oracle.explicit_q(h.T, tau_sk, d)[:d, :d]
    # Z9: the last sketch reflector has length 1 (d <= w); LAPACK takes tau = 0 there, convention H
    # takes tau = 2, i.e. H_d = diag(1, ..., 1, -1): flip the last column of LAPACK's Q_sk.
    Qsk[:, d - 1] *= -1.0
    Q = oracle.explicit_q(out.A, out.tau[:b], m)
    S2 = (S @ Q)[:, b:]
    A22 = out.A[b:, b:]
    ref = Qsk.T @ S2 @ A22  # d x (n - b)
    got = out.MskT[b:, :].T
    assert np.linalg.norm(got - ref) <= 1e-12 * np.linalg.norm(ref)


def test_determinism_and_thread_independence():
    A = inputs.gaussian(300, 260, seed=21)
    o1 = oracle.bqrrp(A, 32, 40, seed=8, nthreads=1)
    o2 = oracle.bqrrp(A, 32, 40, seed=8, nthreads=4)
    o3 = oracle.bqrrp(A, 32, 40, seed=8, nthreads=4)
    for o in (o2, o3):
        assert np.array_equal(o1.A, o.A) and np.array_equal(o1.tau, o.tau) and np.array_equal(o1.J, o.J)


def test_block_size_independence():
    A = inputs.gaussian(128, 128, seed=31)
    for b in (8, 16, 32, 64, 128):
        out = oracle.bqrrp(A, b, b, seed=0)
        assert out.rank == 128
        assert oracle.residual(A, out) <= 1e-13
        assert oracle.orthogonality(out) <= 1e-13


def test_illegal_arguments():
    A = np.zeros((4, 4))
    with pytest.raises(ValueError):
        oracle.bqrrp(A, 0, 1)  # b < 1
    with pytest.raises(ValueError):
        oracle.bqrrp(A, 2, 1)  # d < b
    with pytest.raises(ValueError):
        oracle.bqrrp(A, 2, 5)  # d > m (S:448 config violation)
