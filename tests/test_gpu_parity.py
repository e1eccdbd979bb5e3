"""GPU parity: the CUDA path (through the C ABI) against the CPU oracle on identical seeded inputs.

Tolerances: RNG, gathers and integer-valued GEMMs bit-exact; J and rank identical
when the oracle's smallest LU pivot margin exceeds 1e-10 (SURVEY c.6 rule 2); R, V relative 1e-12
normwise and max|dtau| <= 1e-12 (reading Z25); residual <= 1e-13, orthogonality per Z24.
"""
import numpy as np
import pytest

import _parity
import inputs
import oracle

pytestmark = pytest.mark.gpu


def _bq():
    import paper_2507_00976_b200 as bq

    bq.lib()
    return bq


def _dev(a):
    """Column-major float64 CUDA tensor (shape of a, strides (1, m))."""
    import torch

    return torch.tensor(np.ascontiguousarray(np.asarray(a, dtype=np.float64).T), device="cuda").t()


def _host(t):
    return t.detach().cpu().numpy()


# ----------------------------------------------------------------------------- GEMM engine
@pytest.mark.parametrize("ta", [False, True])
@pytest.mark.parametrize("tb", [False, True])
@pytest.mark.parametrize("M,N,K", [(1, 1, 1), (300, 200, 77), (129, 257, 513), (64, 64, 8192), (1000, 33, 2048)])
def test_gemm_integer_bitexact(gpu, ta, tb, M, N, K):
    bq = _bq()
    rng = np.random.default_rng(M * 7 + N * 3 + K)
    A = rng.integers(-8, 9, size=(K, M) if ta else (M, K)).astype(np.float64)
    B = rng.integers(-8, 9, size=(N, K) if tb else (K, N)).astype(np.float64)
    C = rng.integers(-8, 9, size=(M, N)).astype(np.float64)
    ref = 2.0 * ((A.T if ta else A) @ (B.T if tb else B)) - 3.0 * C
    dC = _dev(C)
    bq.debug_gemm(ta, tb, 2.0, _dev(A), _dev(B), -3.0, dC)
    assert np.array_equal(_host(dC), ref)


# ----------------------------------------------------------------------------- TRSM building block
@pytest.mark.parametrize("rows,n", [(1000, 200), (64, 64), (4097, 130), (5, 7), (300, 1)])
@pytest.mark.parametrize("t_lower,unit", [(False, False), (True, False), (True, True)])
@pytest.mark.parametrize("inverse", [False, True])
def test_trsm_matches_triangular_solve(gpu, rows, n, t_lower, unit, inverse):
    """X op(T) = B for a well-conditioned triangle (kappa ~ 10: the Cholesky factor of a perturbed identity
    Gram matrix, the panel's case), ragged in both dimensions; substitution and the inverted-diagonal-block
    path against scipy's solve_triangular (fp64)."""
    import scipy.linalg as sla

    bq = _bq()
    rng = np.random.default_rng(rows * 31 + n)
    G = np.eye(n) + 0.2 * rng.standard_normal((n, n)) / np.sqrt(n)
    U = np.linalg.qr(G)[1]
    U = U * np.sign(np.diag(U))[:, None]
    if unit:
        U = U / np.diag(U)[:, None]
    T = U.T.copy() if t_lower else U.copy()
    T_in = T + (np.triu(rng.standard_normal((n, n)), 1) if t_lower else np.tril(rng.standard_normal((n, n)), -1))
    if unit:  # the diagonal must not be read
        T_in[np.diag_indices(n)] = 7.0
    B = rng.standard_normal((rows, n))
    ref = sla.solve_triangular(U, B.T, trans="T", lower=False).T  # X U = B  <=>  U^T X^T = B^T
    dB = _dev(B)
    bq.debug_trsm(_dev(T_in), dB, t_lower=t_lower, unit=unit, inverse=inverse)
    X = _host(dB)
    assert np.linalg.norm(X - ref) <= 1e-13 * np.linalg.norm(ref)


# ----------------------------------------------------------------------------- a1 sketch
def test_sketch_operator_bitexact(gpu):
    bq = _bq()
    m, n, d = 1024, 64, 160
    A = inputs.gaussian(m, n, seed=1)
    S, MskT = bq.debug_sketch(_dev(A), d, seed=0)
    So = oracle.sketch_operator(d, m, seed=0)
    assert np.array_equal(_host(S), So)  # bit-exact host == device RNG
    ref = oracle.sketch(A, d, seed=0)
    assert np.linalg.norm(_host(MskT) - ref) <= 1e-14 * np.linalg.norm(ref)


def test_sketch_operator_bitexact_large_seed(gpu):
    bq = _bq()
    m, n, d = 3000, 8, 40
    A = np.eye(m)[:, :n]
    seed = 0xDEADBEEFCAFEF00D
    S, MskT = bq.debug_sketch(_dev(A), d, seed=seed)
    assert np.array_equal(_host(S), oracle.sketch_operator(d, m, seed=seed))
    assert np.array_equal(_host(MskT).T, oracle.sketch_operator(d, m, seed=seed)[:, :n])  # S I exact


def test_sketch_integer_inputs_exact(gpu):
    """Integer-valued A: each product a*S is exact and the sums of <= 2^53-bounded... compare to the
    exactly rounded sum (math.fsum) within the accumulation-order bound."""
    bq = _bq()
    A = inputs.integer_valued(512, 16, seed=3)
    _, MskT = bq.debug_sketch(_dev(A), 32, seed=5)
    ref = oracle.sketch(A, 32, seed=5)
    assert np.abs(_host(MskT) - ref).max() <= 512 * 2.0 ** -52 * np.abs(ref).max()


# ----------------------------------------------------------------------------- a2 LU pivots
@pytest.mark.parametrize("w,d", [(300, 64), (1000, 160), (5000, 300), (200, 200), (150, 400), (4097, 33),
                                 (8000, 200), (8193, 40), (12000, 50), (16384, 100), (20000, 96),
                                 (40000, 64), (70001, 100)])
def test_lu_pivots_match_oracle(gpu, w, d):
    """Every leaf regime of K-LU: the register cluster leaf (32 columns with one / two rows per thread up to
    4096 / 8192 rows, 16 columns with four up to 16384 rows, ragged last leaves), the shared-memory cluster
    leaf, and the cooperative grid leaf (40000, 70001 rows: the C3 regime, ragged row count)."""
    bq = _bq()
    L = inputs.gaussian(w, d, seed=w + d)
    _, ipiv_o, margin = oracle.getf2(L)
    _, ipiv_g = bq.debug_lu_pivots(_dev(L))
    ipiv_g = _host(ipiv_g)
    if margin.min() > 1e-10:
        assert np.array_equal(ipiv_g, ipiv_o)
    else:  # compare up to the first near-tie
        first = int(np.argmax(margin <= 1e-10))
        assert np.array_equal(ipiv_g[:first], ipiv_o[:first])


@pytest.mark.parametrize("w", [3000, 7000, 15000])
def test_lu_exact_ties_across_ctas(gpu, w):
    """IDAMAX's first-index rule (Z19) when the largest |value| of a column is held by rows in different CTAs of
    the cluster (and with opposite signs): the first of them is the pivot, here and after two eliminations."""
    bq = _bq()
    rng = np.random.default_rng(w)
    L = rng.integers(-3, 4, size=(w, 24)).astype(np.float64)
    L[:, 0] = 1.0
    for r, v in ((w // 3, -8.0), (w // 2, 8.0), (w - 5, 8.0)):
        L[r, 0] = v
    _, ipiv_o, _ = oracle.getf2(L)
    _, ipiv_g = bq.debug_lu_pivots(_dev(L))
    ipiv_g = _host(ipiv_g)
    assert ipiv_g[0] == ipiv_o[0] == w // 3 + 1
    assert np.array_equal(ipiv_g[:3], ipiv_o[:3])


def test_lu_zero_and_tied_columns(gpu):
    bq = _bq()
    L = np.zeros((40, 8))
    L[5, 0] = 3.0
    L[7, 0] = -3.0  # tie: first index wins (Z19)
    L[:, 3] = 0.0   # zero column after elimination handled per Z18
    rng = np.random.default_rng(0)
    L[:, 4:] = rng.integers(-3, 4, size=(40, 4))
    _, ipiv_o, _ = oracle.getf2(L)
    _, ipiv_g = bq.debug_lu_pivots(_dev(L))
    assert np.array_equal(_host(ipiv_g), ipiv_o)


# ----------------------------------------------------------------------------- a2 sketch QR
@pytest.mark.parametrize("w,d", [(1000, 160), (64, 64), (300, 100), (50, 80), (4000, 512), (3000, 1500),
                                 (2100, 2048)])
def test_sketch_qr_matches_oracle(gpu, w, d):
    """K-SQR up to the C3 sketch depth (d = 2048: the full recursion over register cluster leaves) and a
    ragged d = 1500."""
    bq = _bq()
    WT = inputs.gaussian(w, d, seed=w * d)
    F, _ = oracle.house_qr(WT.T)  # d x w, convention H
    p = min(d, w)
    R_o = np.triu(F)  # upper trapezoid
    got = _host(bq.debug_sketch_qr(_dev(WT))).T  # R_sk (d x w)
    assert np.linalg.norm(got - R_o) <= 1e-12 * np.linalg.norm(R_o)
    assert np.all(np.tril(got, -1) == 0.0)


# ----------------------------------------------------------------------------- a3 permutation
@pytest.mark.parametrize("rows,w,nlu", [(100, 50, 20), (1024, 1000, 160), (7, 3000, 300), (33, 5, 5)])
def test_permute_bitexact(gpu, rows, w, nlu):
    import torch

    bq = _bq()
    rng = np.random.default_rng(rows + w)
    ipiv = np.array([rng.integers(j, w) + 1 for j in range(nlu)], dtype=np.int64)  # valid LU swap list
    X = rng.standard_normal((rows, w))
    Jqr_o = oracle.piv_transform(w, ipiv)
    ref = oracle.col_gather(X, Jqr_o)
    Xg, Jqr_g = bq.debug_permute(_dev(X), torch.tensor(ipiv, device="cuda"))
    assert np.array_equal(_host(Jqr_g), Jqr_o)
    assert np.array_equal(_host(Xg), ref)


# ----------------------------------------------------------------------------- a4/a5 panel
@pytest.mark.parametrize("h,k,t", [(256, 32, 40), (1000, 100, 0), (3000, 128, 200), (129, 129, 3), (8192, 1024, 64),
                                   (65536, 256, 0), (4096, 2048, 64)])
@pytest.mark.parametrize("passes", [0, 1, 2])
def test_panel_matches_householder_oracle(gpu, h, k, t, passes):
    """c.1: CholQR + reconstruction gives the unique (V, tau, R) with tau in [1,2] = convention-H QR."""
    bq = _bq()
    rng = np.random.default_rng(h + k + t)
    P = rng.standard_normal((h, k + t))
    # a genuine preconditioner: R of a sketch of the panel (d = k)
    Sk = rng.standard_normal((k + k // 4 + 1, h)) @ P[:, :k]
    Rsk = np.linalg.qr(Sk, mode="r")[:k, :k]
    F_o, tau_o = oracle.house_qr(P, kref=k)
    Pg, taug = bq.debug_panel(_dev(P), k, _dev(Rsk), cholqr_passes=passes)
    F_g = _host(Pg)
    tol = 1e-9 if passes == 1 else 1e-12  # 0 = Householder panel (BQRRP_HQR), 2 = CholQR2
    # per column: R11, the reflectors, tau; the trailing block (R12 on top of the updated rows) per column
    _parity.compare_factors(F_g[:, :k], _host(taug), F_o[:, :k], tau_o, k, tol)
    if t > 0:
        _parity.assert_colwise(F_g[:, k:], F_o[:, k:], tol, "trailing block")


# ----------------------------------------------------------------------------- end to end
def _run_both(A, b, d, seed=0, rank_tol=None, passes=2):
    bq = _bq()
    out_o = oracle.bqrrp(A, b, d, seed=seed, rank_tol=rank_tol)
    Ag, taug, Jg, rk = bq.factor(_dev(A), b, d, seed=seed, rank_tol=rank_tol, cholqr_passes=passes)
    return out_o, (_host(Ag), _host(taug), _host(Jg), rk)


def _compare(out_o, g, exact_j=True):
    """Per column (tests/_parity.py): R(:, j) and v_j relative 1e-12, tau per entry 1e-12.
    exact_j: J identical.  Otherwise (rank-deficient inputs: the pivots after l are decided on
    rounding noise, so only J(:l) is unique) J(:l) identical, J a permutation, and R(:l, :) compared
    column by column through the original column index it holds."""
    Ag, taug, Jg, rk = g
    l = out_o.rank
    assert rk == l
    if exact_j:
        assert np.array_equal(Jg, out_o.J)
        _parity.compare_factors(Ag, taug, out_o.A, out_o.tau, l)
    else:
        assert np.array_equal(Jg[:l], out_o.J[:l])
        assert sorted(Jg) == list(range(1, len(Jg) + 1))
        Ro = _parity.r_cols(out_o.A, l)[:, np.argsort(out_o.J)]
        Rg = _parity.r_cols(Ag, l)[:, np.argsort(Jg)]
        _parity.assert_colwise(Rg, Ro, what="R (by original column)")
        _parity.assert_colwise(_parity.v_cols(Ag, l), _parity.v_cols(out_o.A, l), what="V")
        assert np.max(np.abs(taug[:l] - out_o.tau[:l]), initial=0.0) <= _parity.TOL
    assert np.all(Ag[l:, l:] == 0) and np.all(taug[l:] == 0)


@pytest.mark.parametrize("shape,b,d", [((1024, 1024), 128, 160), ((256, 256), 32, 32), ((1000, 1000), 128, 128),
                                       ((2048, 512), 128, 160), ((512, 2048), 128, 128), ((700, 450), 64, 80),
                                       ((300, 300), 300, 300), ((4096, 4096), 256, 256)])
def test_factor_matches_oracle(gpu, shape, b, d):
    m, n = shape
    A = inputs.gaussian(m, n, seed=m + 3 * n + b)
    out_o, g = _run_both(A, b, d, seed=0)
    assert out_o.min_margin > 1e-10
    _compare(out_o, g)
    res = oracle.residual(A, oracle.OracleResult(g[0], g[1], g[2], g[3], None, 0, None))
    assert res <= 1e-13


@pytest.mark.parametrize("shape,b,d", [((1024, 1024), 128, 160), ((2048, 512), 128, 160), ((700, 450), 64, 80)])
def test_factor_hqr_variant_matches_oracle(gpu, shape, b, d):
    """BQRRP_HQR: the Householder panel gives the same (V, tau, R) as the oracle."""
    m, n = shape
    A = inputs.gaussian(m, n, seed=m + n)
    out_o, g = _run_both(A, b, d, seed=0, passes=0)
    _compare(out_o, g)


@pytest.mark.parametrize("seed", [1, 2, 3, 4])
def test_factor_c1_seeds(gpu, seed):
    A = inputs.gaussian(1024, 1024, seed=seed)
    out_o, g = _run_both(A, 128, 160, seed=seed)
    _compare(out_o, g)


def test_factor_residual_orthogonality(gpu):
    A = inputs.gaussian(1024, 1024, seed=0)
    _, g = _run_both(A, 128, 160)
    res = oracle.OracleResult(g[0], g[1], g[2], g[3], None, 0, None)
    assert oracle.residual(A, res) <= 1e-13
    assert oracle.orthogonality(res) <= 1e-13


@pytest.mark.parametrize("k_true", [64, 128, 199])
def test_rank_recovery(gpu, k_true):
    A = inputs.low_rank(512, 512, k_true, seed=k_true)
    out_o, g = _run_both(A, 128, 160)
    assert g[3] == k_true == out_o.rank
    _compare(out_o, g, exact_j=False)
    res = oracle.residual(A, oracle.OracleResult(g[0], g[1], g[2], g[3], None, 0, None))
    assert res <= 1e-13


def test_zero_and_empty(gpu):
    import torch

    bq = _bq()
    A = torch.zeros((64, 64), dtype=torch.float64, device="cuda").t().contiguous().t()
    Ag, tau, J, rk = bq.factor(A, 16, 16)
    assert rk == 0 and np.array_equal(_host(J), np.arange(1, 65)) and not _host(tau).any()
    E = torch.zeros((5, 0), dtype=torch.float64, device="cuda").t().contiguous().t()
    _, _, J, rk = bq.factor(E, 2, 2)
    assert rk == 0


def test_nonfinite_input_is_flagged(gpu):
    bq = _bq()
    A = inputs.gaussian(128, 128, seed=0)
    A[5, 7] = np.nan
    with pytest.raises(bq.BqrrpError) as e:
        bq.factor(_dev(A), 32, 32)
    assert e.value.status == 1


def test_deterministic_bitwise(gpu):
    bq = _bq()
    A = inputs.gaussian(1500, 1300, seed=9)
    r1 = bq.factor(_dev(A), 128, 160, seed=4)
    r2 = bq.factor(_dev(A), 128, 160, seed=4)
    for x, y in zip(r1[:3], r2[:3]):
        assert np.array_equal(_host(x), _host(y))


def test_factor_host_e2e_matches_device(gpu):
    import torch

    bq = _bq()
    A = inputs.gaussian(600, 500, seed=2)
    Ad, taud, Jd, rkd = bq.factor(_dev(A), 64, 80, seed=1)
    Ah = torch.tensor(np.ascontiguousarray(A.T)).t()
    Ah2, tauh, Jh, rkh = bq.factor_host(Ah, 64, 80, seed=1)
    assert rkh == rkd
    assert np.array_equal(Ah2.numpy(), _host(Ad))
    assert np.array_equal(tauh.numpy(), _host(taud)) and np.array_equal(Jh.numpy(), _host(Jd))


def _compare_ill_conditioned(A, out_o, g):
    """Ill-conditioned inputs: the pivots J(:l), the rank and R are well determined (R normwise to 1e-12),
    but the Householder vectors of the late columns are not — their forward error is ~ u ||A|| / sigma_i
    (the trailing matrices they come from are tiny) — so V and tau are checked through backward
    stability instead: residual and orthogonality of the GPU factors at the 1e-13 level (reading Z24)."""
    Ag, taug, Jg, rk = g
    l = out_o.rank
    assert rk == l
    if out_o.min_margin > 1e-8:
        assert np.array_equal(Jg[:l], out_o.J[:l])
        Ro = np.triu(out_o.A)[:l][:, np.argsort(out_o.J)]
        Rg = np.triu(Ag)[:l][:, np.argsort(Jg)]
        _parity.assert_colwise(Rg, Ro, what="R (by original column)")
    res = oracle.OracleResult(Ag, taug, Jg, rk, None, 0, None)
    assert oracle.residual(A, res) <= 1e-13
    assert oracle.orthogonality(res) <= 1e-13


@pytest.mark.parametrize("n,sigma_last", [(512, 1e-10), (768, 1e-7)])
def test_factor_graded_spectrum_matches_oracle(gpu, n, sigma_last):
    """C5-style graded spectrum (geometric decay to sigma_last, BASELINE C5 / reading Z30): ill-conditioned
    panels (kappa(R_sk11) up to 1/sigma_last) through the preconditioned CholQR2 path."""
    A, _ = inputs.graded(n, n, n, sigma_last=sigma_last, seed=n)
    A = np.asfortranarray(A)
    out_o, g = _run_both(A, 64, 80, seed=3)
    _compare_ill_conditioned(A, out_o, g)


def test_factor_kahan_matches_oracle(gpu):
    """Kahan matrix (reading Z27): the adversarial case for column pivoting."""
    n = 384
    A = np.asfortranarray(inputs.kahan(n))
    out_o, g = _run_both(A, 64, 64, seed=1)
    _compare_ill_conditioned(A, out_o, g)


def test_cholqr_breakdown_falls_back_to_householder(gpu):
    """CholQR breakdown handling: a panel whose POTRF reports a non-positive pivot is
    re-factored by Householder QR and the factorization stays backward stable — with the same pivots and
    R as the oracle, since the HQR panel and CholQR2 + reconstruction give the same (V, tau, R) (SURVEY
    c.1).  Without the fallback the call reports BQRRP_ENUMERIC.  Whether a given ill-conditioned input
    breaks POTRF down depends on rounding, so the breakdown is forced through the library's test hook."""
    bq = _bq()
    A = np.asfortranarray(inputs.gaussian(1000, 1000, seed=4))
    out_o = oracle.bqrrp(A, 128, 160, seed=0)
    Ag, taug, Jg, rk = bq.factor(_dev(A), 128, 160, seed=0, debug_force_breakdown=True)
    assert bq.panel_fallbacks() == 8  # every panel of the 8 iterations
    _compare(out_o, (_host(Ag), _host(taug), _host(Jg), rk))
    with pytest.raises(bq.BqrrpError) as e:
        bq.factor(_dev(A), 128, 160, seed=0, hqr_fallback=False, debug_force_breakdown=True)
    assert e.value.status == 1
    bq.factor(_dev(A), 128, 160, seed=0)
    assert bq.panel_fallbacks() == 0


@pytest.mark.parametrize("h,k,t", [(131072, 64, 16), (300000, 40, 8)])
def test_tall_householder_panel(gpu, h, k, t):
    """the Householder panel (BQRRP_HQR, and the CholQR-breakdown fallback) on panels taller than
    the 32-column grid leaf holds (94 720 rows): narrower leaves (16 / 8 columns), same (V, tau, R)."""
    bq = _bq()
    rng = np.random.default_rng(h + k)
    P = rng.standard_normal((h, k + t))
    F_o, tau_o = oracle.house_qr(P, kref=k)
    Pg, taug = bq.debug_panel(_dev(P), k, _dev(np.eye(k)), cholqr_passes=0)
    F_g = _host(Pg)
    _parity.compare_factors(F_g[:, :k], _host(taug), F_o[:, :k], tau_o, k)
    _parity.assert_colwise(F_g[:, k:], F_o[:, k:], what="trailing block")


def test_tall_breakdown_fallback_matches_oracle(gpu):
    """The CholQR-breakdown fallback on a C4-like tall matrix (h > 94 720 rows) end to end."""
    bq = _bq()
    A = inputs.gaussian(131072, 192, seed=11)
    out_o = oracle.bqrrp(A, 64, 64, seed=2)
    Ag, taug, Jg, rk = bq.factor(_dev(A), 64, 64, seed=2, debug_force_breakdown=True)
    assert bq.panel_fallbacks() == 3
    _compare(out_o, (_host(Ag), _host(taug), _host(Jg), rk))


def test_numerically_singular_panels_stay_backward_stable(gpu):
    """A Kahan matrix (kappa ~ 1e20 at n = 4096) with rank_tol far below the default keeps numerically
    dependent columns in the blocks; whether or not POTRF then breaks down (rounding-dependent; the
    fallback takes over if it does), the factorization is backward stable and Q orthonormal."""
    bq = _bq()
    A = np.asfortranarray(inputs.kahan(4096))
    Ag, taug, Jg, rk = bq.factor(_dev(A), 1024, 1024, seed=0, rank_tol=1e-300)
    res = oracle.OracleResult(_host(Ag), _host(taug), _host(Jg), rk, None, 0, None)
    assert oracle.residual(A, res) <= 1e-13
    assert oracle.orthogonality(res) <= 1e-12


@pytest.mark.parametrize("n", [200, 1000, 2048])
def test_kxk_cholesky_and_sign_lu(gpu, n):
    """The k x k factorizations of the panel (persistent kernel for n >= 256, blocked below): POTRF of an SPD
    Gram matrix against LAPACK's Cholesky (numpy), and the sign-choosing no-pivot LU of the reconstruction
    (bqrrp_debug_recon_lu with C = I): L U = W - diag(S), S_j = -sgn of the running pivot (reading Z20),
    unit-lower L with |L| <= 1 (the pivots |a - S| >= 1 for orthonormal columns, BD2015)."""
    import ctypes

    import torch

    import paper_2507_00976_b200 as bq

    L = bq.lib()
    rng = np.random.default_rng(n)
    X = rng.standard_normal((3 * n, n))
    G = X.T @ X
    Gd = _dev(G)
    st = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
    assert L.bqrrp_debug_potrf(n, ctypes.c_void_p(Gd.data_ptr()), n, st) == 0
    Lg = np.tril(_host(Gd))
    Lref = np.linalg.cholesky(G)
    assert np.linalg.norm(Lg - Lref) <= 1e-12 * np.linalg.norm(Lref)
    assert np.all(np.triu(_host(Gd), 1) == 0)
    # sign LU of the top n x n of an orthonormal Q (C = I)
    Q, _ = np.linalg.qr(rng.standard_normal((2 * n, n)))
    Qd = _dev(Q)
    C = _dev(np.eye(n))
    Wr = torch.empty((n, n), dtype=torch.float64, device="cuda").t()
    S = torch.empty(n, dtype=torch.float64, device="cuda")
    assert L.bqrrp_debug_recon_lu(n, ctypes.c_void_p(Qd.data_ptr()), 2 * n, ctypes.c_void_p(C.data_ptr()),
                                  ctypes.c_void_p(Wr.data_ptr()), ctypes.c_void_p(S.data_ptr()), st) == 0
    W, s_ = _host(Wr), _host(S)
    Lw = np.tril(W, -1) + np.eye(n)
    Uw = np.triu(W)
    A = Q[:n] - np.diag(s_)
    assert np.linalg.norm(Lw @ Uw - A) <= 1e-12 * np.linalg.norm(A)
    assert np.all(np.abs(Lw) <= 1 + 1e-12)
    assert np.all(np.isin(s_, [-1.0, 1.0]))


def test_lookahead_and_serial_schedules_agree(gpu):
    """The lookahead schedule (bulk rows, the sample update's X, the R_sk GEMM and the k x k panel finish on
    a second stream) and the single-stream schedule compute the same factorization: J and rank identical,
    R / tau to rounding (split-K choices differ between the streams), and the host-buffer entry (overlapped
    copies) is bitwise the device entry."""
    import torch

    bq = _bq()
    A = inputs.gaussian(1500, 1500, seed=11)
    Ag1, tau1, J1, r1 = bq.factor(_dev(A), 256, 256, seed=2)
    Ag0, tau0, J0, r0 = bq.factor(_dev(A), 256, 256, seed=2, lookahead=False)
    assert r1 == r0 == 1500
    assert torch.equal(J1, J0)
    R1, R0 = np.triu(_host(Ag1)), np.triu(_host(Ag0))
    assert np.linalg.norm(R1 - R0) <= 1e-12 * np.linalg.norm(R0)
    assert np.max(np.abs(_host(tau1) - _host(tau0))) <= 1e-12
    Ahost = torch.from_numpy(np.asfortranarray(A).copy(order="F"))  # column-major host tensor
    assert Ahost.stride(0) == 1
    Ah_out, tauh, Jh, rh = bq.factor_host(Ahost, 256, 256, seed=2)
    assert rh == r1
    assert np.array_equal(Ah_out.numpy(), _host(Ag1)) and np.array_equal(tauh.numpy(), _host(tau1))
    assert np.array_equal(Jh.numpy(), _host(J1))
    # the overlapped panel lookahead (panel i+1 factored from a gathered copy while the bulk GEMM of iteration i
    # runs) is bitwise the default schedule's factorization
    for pl in (1,):
        Ag2, tau2, J2, r2 = bq.factor(_dev(A), 256, 256, seed=2, panel_lookahead=pl)
        assert r2 == r1 and torch.equal(J2, J1) and torch.equal(tau2, tau1) and torch.equal(Ag2, Ag1), pl


@pytest.mark.parametrize("shape,b,d", [((3000, 2500), 256, 256), ((2048, 2048), 512, 512), ((1000, 1500), 96, 160),
                                       ((700, 450), 64, 80), ((9000, 9000), 1024, 1024)])
@pytest.mark.parametrize("lu_la", [True, False])
def test_pipelined_sketch_qr_matches_recursive(gpu, shape, b, d, lu_la):
    """K-SQR pipelined with K-LU (left-looking blocks on a third stream, the default) — with K-LU either the
    recursive LU (default) or the lookahead blocked LU (option) — against the recursive K-SQR after the recursive K-LU: the
    same pivots (J(:l), rank identical) and the same factorization to rounding, per column; and against the oracle
    on the smaller shapes."""
    import torch

    bq = _bq()
    A = inputs.gaussian(*shape, seed=3)
    Ag1, tau1, J1, r1 = bq.factor(_dev(A), b, d, seed=4, lu_lookahead=lu_la)
    Ag0, tau0, J0, r0 = bq.factor(_dev(A), b, d, seed=4, sqr_pipeline=False)
    assert r1 == r0 == min(shape)
    # wide inputs: the columns past l = m are ordered on rounding noise, so J(:l) and the first l
    # columns are compared there
    l = r0

    def same(Ja, Fa, ta, Jb, Fb, tb):
        Ja, Jb = np.asarray(Ja), np.asarray(Jb)
        assert np.array_equal(Ja[:l], Jb[:l])
        if not np.array_equal(Ja, Jb):
            Fa, Fb = Fa[:, :l], Fb[:, :l]
        _parity.compare_factors(Fa, ta, Fb, tb, l)

    same(_host(J1), _host(Ag1), _host(tau1), _host(J0), _host(Ag0), _host(tau0))
    if shape[0] * shape[1] <= 1500 * 1500:
        o = oracle.bqrrp(A, b, d, seed=4)
        assert r1 == o.rank
        same(_host(J1), _host(Ag1), _host(tau1), o.J, o.A, o.tau)


def test_sqr_merge_stream_is_bitwise_neutral(gpu):
    """The pipelined K-SQR's T merges on their own stream (default) or on the pipeline's stream: the same GEMMs in
    the same order per element, so the factorization is bitwise identical."""
    import torch

    bq = _bq()
    A = inputs.gaussian(3000, 2600, seed=9)
    Ag0, tau0, J0, r0 = bq.factor(_dev(A), 512, 512, seed=1)
    Ag1, tau1, J1, r1 = bq.factor(_dev(A), 512, 512, seed=1, sqr_merge_stream=False)
    assert r0 == r1 == 2600
    assert torch.equal(J1, J0) and torch.equal(tau1, tau0) and torch.equal(Ag1, Ag0)


@pytest.mark.parametrize("ctas", [32, 148, 16])
def test_lu_grid_leaf_cap_same_factorization(gpu, ctas):
    """A wide input whose sketch transpose needs K-LU's cooperative grid leaf (w > 25.6k rows): capping that leaf at
    16 / 32 CTAs (narrower leaves, more rows per CTA) or running it on every SM gives the same pivots, hence bitwise
    the same factorization (J(:l), tau, the first l columns) as the default schedule (lookahead: the cap applies
    where the bulk GEMM is the long pole)."""
    import torch

    bq = _bq()
    A = inputs.gaussian(640, 30000, seed=13)
    Ag0, tau0, J0, r0 = bq.factor(_dev(A), 256, 256, seed=3)
    Ag1, tau1, J1, r1 = bq.factor(_dev(A), 256, 256, seed=3, lu_grid_ctas=ctas)
    assert r0 == r1 == 640
    # m < n: the pivots past l = m are decided on rounding noise (the last iteration has h < d rows)
    assert torch.equal(J1[:r0], J0[:r0]) and torch.equal(tau1, tau0) and torch.equal(Ag1[:, :r0], Ag0[:, :r0])


@pytest.mark.parametrize("bulk_sms", [-1, 100, 24])
def test_bulk_partition_is_bitwise_neutral(gpu, bulk_sms):
    """The bulk trailing GEMM on a green-context SM partition (bqrrp_options.bulk_sms: every iteration on a
    partition of ~100 or 24 SMs) or on the whole device (-1) gives bitwise the default (auto) factorization: the
    bulk runs in fixed tiles with no split-K, so only its placement changes."""
    import torch

    bq = _bq()
    A = inputs.gaussian(3000, 2500, seed=5)
    Ag0, tau0, J0, r0 = bq.factor(_dev(A), 256, 256, seed=1)
    Ag1, tau1, J1, r1 = bq.factor(_dev(A), 256, 256, seed=1, bulk_sms=bulk_sms)
    assert r1 == r0 == 2500
    assert torch.equal(J1, J0) and torch.equal(tau1, tau0) and torch.equal(Ag1, Ag0)


@pytest.mark.parametrize("shape,b,d,exact_j", [((1, 100), 1, 1, True), ((100, 1), 8, 8, True), ((40, 300), 16, 40, False),
                                               ((333, 77), 100, 120, True), ((257, 257), 64, 64, True),
                                               ((130, 129), 128, 130, True), ((64, 1000), 64, 64, True)])
def test_factor_degenerate_shapes_match_oracle(gpu, shape, b, d, exact_j):
    """Degenerate and ragged shapes (P:241-242 notation): a single row (d = m = 1), a single column (n < b),
    d = m (the sketch is the whole row space), b > n (one ragged block), a last block of ONE column
    (257 = 4 * 64 + 1, 129 = 128 + 1), and a wide matrix whose loop ends after one block (m = b).
    40 x 300 with d = 40: the last iteration has h = 8 trailing rows, so the updated sketch has rank <= 8 and
    its LU pivots 9..40 are decided on rounding noise; they only permute columns beyond l = m, so there J(:l)
    and R(:l, :) column by column are what is unique (GEQP3 format leaves the order after l free)."""
    m, n = shape
    A = inputs.gaussian(m, n, seed=m + 7 * n)
    out_o, g = _run_both(A, b, d, seed=0)
    assert out_o.min_margin > 1e-10
    _compare(out_o, g, exact_j=exact_j)
    res = oracle.residual(A, oracle.OracleResult(g[0], g[1], g[2], g[3], None, 0, None))
    assert res <= 1e-13


def test_factor_duplicate_and_zero_columns(gpu):
    """Exactly dependent columns (a duplicate, a multiple, a zero column): the rank is n - 3 on both sides,
    J(:l) and R(:l, :) agree (the order of the three dependent columns after l is decided on rounding noise,
    so only its being a permutation is checked)."""
    A = inputs.gaussian(300, 200, seed=5)
    A[:, 17] = A[:, 5]
    A[:, 9] = 0.0
    A[:, 150] = 2.0 * A[:, 40]
    out_o, g = _run_both(A, 64, 80, seed=0)
    assert out_o.rank == 197
    _compare(out_o, g, exact_j=False)
    res = oracle.residual(A, oracle.OracleResult(g[0], g[1], g[2], g[3], None, 0, None))
    assert res <= 1e-13


@pytest.mark.parametrize("pad", [1, 37])
def test_factor_padded_lda_matches_unpadded(gpu, pad):
    """The C ABI takes A with a leading dimension lda >= m (GEQP3 argument convention): a view
    into a taller column-major buffer (lda = m + pad; odd lda also disables the 16-byte vector loads of the
    GEMM engine) gives the bitwise-same factorization as the dense lda = m call, and the padding rows are
    left untouched."""
    import torch

    bq = _bq()
    m, n, b, d = 700, 650, 128, 160
    A = inputs.gaussian(m, n, seed=21)
    Ad, taud, Jd, rd = bq.factor(_dev(A), b, d, seed=3)
    big = np.full((m + pad, n), 7.25)
    big[:m] = A
    Bt = _dev(big)
    view = Bt[:m]
    assert view.stride() == (1, m + pad)
    Ap, taup, Jp, rp = bq.factor(view, b, d, seed=3)
    assert rp == rd
    assert torch.equal(Jp, Jd) and torch.equal(taup, taud)
    assert np.array_equal(_host(Ap), _host(Ad))
    assert np.all(_host(Bt)[m:] == 7.25)


def test_factor_on_caller_stream(gpu):
    """The C ABI runs on the caller's stream (its internal streams fork from and join back to it): a
    factorization issued on a non-default torch stream, with the input produced on that same stream just
    before the call, equals the default-stream result bitwise."""
    import torch

    bq = _bq()
    A = inputs.gaussian(900, 900, seed=5)
    Ad, taud, Jd, rd = bq.factor(_dev(A), 128, 128, seed=1)
    src = _dev(A)
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        X = src.t().contiguous().t()  # produced on s, consumed by the library on s
        Xs, taus, Js, rs = bq.factor(X, 128, 128, seed=1)
    s.synchronize()
    assert rs == rd and torch.equal(Js, Jd) and torch.equal(taus, taud)
    assert torch.equal(Xs, Ad)
