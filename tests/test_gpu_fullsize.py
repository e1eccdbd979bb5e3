"""Full-size GPU checks in the launch configuration bench.py times (same API, same workspace, same
b and d), where the oracle cannot run end to end:

  * sampled sketch entries against the oracle's generator evaluated one entry at a time;
  * properties that hold at any size: J a permutation, rank = min(m, n) on Gaussian inputs, tau in [1, 2],
    residual ||A(:,J) X - Q R X|| / ||A(:,J) X|| and orthogonality ||Q^T Q X - X|| / ||X|| for random X
    (estimators of the north-star bounds, readings Z24/Z25);
  * column norms: ||R(0:j+1, j)|| = ||A(:, J(j))|| at sampled j (Q orthogonal), each side summed exactly;
  * bitwise determinism of two full factorizations.
"""
import math

import numpy as np
import pytest

import inputs
import oracle

pytestmark = pytest.mark.gpu


def _apply_q(A, tau, Y, transpose=False):
    """Q Y (or Q^T Y) from GEQP3-format reflectors, one reflector at a time (torch on the GPU)."""
    import torch

    m = A.shape[0]
    l = tau.numel()
    th = tau.cpu().tolist()
    order = range(l) if transpose else range(l - 1, -1, -1)
    for j in order:
        t = th[j]
        if t == 0.0:
            continue
        v = torch.empty(m - j, dtype=A.dtype, device=A.device)
        v[0] = 1.0
        v[1:] = A[j + 1:, j]
        w = v @ Y[j:]
        Y[j:] -= t * torch.outer(v, w)
    return Y


def _check_properties(A0, A, tau, J, rank, nvec=4, tol_res=1e-13, tol_orth=None):
    import torch

    m, n = A0.shape
    assert rank == min(m, n)
    Jh = J.cpu().numpy()
    assert np.array_equal(np.sort(Jh), np.arange(1, n + 1))
    t = tau[:rank]
    assert float(t.min()) >= 1.0 - 1e-12 and float(t.max()) <= 2.0 + 1e-12
    g = torch.Generator(device=A.device)
    g.manual_seed(123)
    X = torch.randn((n, nvec), generator=g, device=A.device, dtype=torch.float64)
    AX = A0[:, J - 1] @ X
    R = torch.triu(A[:rank, :])
    QRX = _apply_q(A, t, torch.cat([R @ X, torch.zeros((m - rank, nvec), dtype=A.dtype, device=A.device)]))
    res = float(torch.linalg.norm(AX - QRX) / torch.linalg.norm(AX))
    assert res <= tol_res, res
    Z = torch.randn((m, nvec), generator=g, device=A.device, dtype=torch.float64)
    QZ = _apply_q(A, t, Z.clone())
    QtQZ = _apply_q(A, t, QZ, transpose=True)
    orth = float(torch.linalg.norm(QtQZ - Z) / torch.linalg.norm(Z))
    if tol_orth is None:
        tol_orth = 1e-13 * max(1.0, rank / 1024.0)  # Z24: literal up to 1024, size-scaled beyond
    assert orth <= tol_orth, orth
    # column by column (sampled): Q is orthogonal, so ||R(0:j+1, j)|| = ||A(:, J(j))|| for every j of a
    # full-rank factorization -- each side summed exactly (fsum) from its own column
    if rank == m:
        rng = np.random.default_rng(7)
        for j in sorted(set(int(x) for x in rng.integers(0, n, 24)) | {0, n - 1}):
            rj = A[:min(j + 1, m), j].cpu().numpy()
            aj = A0[:, int(Jh[j]) - 1].cpu().numpy()
            nr, na = math.sqrt(math.fsum(rj * rj)), math.sqrt(math.fsum(aj * aj))
            assert abs(nr - na) <= 1e-12 * na, (j, nr, na)
    return res, orth


def _factor_bench_config(m, n, b, d, seed=0):
    import torch

    import paper_2507_00976_b200 as bq

    A0 = inputs.gaussian_cuda(m, n, seed=seed)
    A = torch.empty_like(A0.t()).t()
    A.copy_(A0)
    ws = torch.empty(bq.workspace_query(m, n, b, d), dtype=torch.uint8, device="cuda")
    out = bq.factor(A, b, d, seed=seed, workspace=ws)
    torch.cuda.synchronize()
    return A0, out, ws


def test_c2_sampled_sketch_entries(gpu):
    """a1 at C2 size: 64 sampled entries of M_sk = S A against the oracle generator, entry by entry."""
    import torch

    import paper_2507_00976_b200 as bq

    m, n, d = 16384, 16384, 1024
    A0 = inputs.gaussian_cuda(m, n, seed=0)
    _, MskT = bq.debug_sketch(A0, d, seed=0, want_S=False)
    rng = np.random.default_rng(0)
    js = rng.integers(0, n, 8)
    is_ = rng.integers(0, d, 8)
    S = oracle.sketch_operator(d, m, seed=0)  # the oracle's own generator (bit-exact with the GPU's, tested)
    for j in js:
        col = A0[:, int(j)].cpu().numpy()
        for i in is_:
            s = S[int(i)]
            ref = math.fsum(s * col)
            got = float(MskT[int(j), int(i)])
            assert abs(got - ref) <= 1e-13 * (np.linalg.norm(s) * np.linalg.norm(col)), (j, i, got, ref)


def test_c2_full_factorization_properties(gpu):
    A0, (A, tau, J, rank), _ = _factor_bench_config(16384, 16384, 1024, 1024)
    res, orth = _check_properties(A0, A, tau, J, rank)
    print(f"C2 residual {res:.2e} orthogonality {orth:.2e}")


def test_c2_bitwise_deterministic(gpu):
    import torch

    import paper_2507_00976_b200 as bq

    A0, (A, tau, J, rank), ws = _factor_bench_config(8192, 8192, 1024, 1024, seed=3)
    A2 = torch.empty_like(A0.t()).t()
    A2.copy_(A0)
    _, tau2, J2, rank2 = bq.factor(A2, 1024, 1024, seed=3, workspace=ws)
    assert rank2 == rank and torch.equal(J, J2) and torch.equal(tau, tau2) and torch.equal(A, A2)


@pytest.mark.slow
def test_c3_full_factorization_properties(gpu):
    """The bench workload itself (65536^2, b = d = 2048): residual and orthogonality estimators."""
    A0, (A, tau, J, rank), _ = _factor_bench_config(65536, 65536, 2048, 2048)
    res, orth = _check_properties(A0, A, tau, J, rank, nvec=2)
    print(f"C3 residual {res:.2e} orthogonality {orth:.2e}")
