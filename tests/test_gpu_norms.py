"""K-NORM parity (bqrrp_column_norms / bqrrp_trailing_norms through the C ABI) against the oracle's definitions
(oracle.column_norms / trailing_norms, pinned in test_oracle_norms.py) on the same seeded inputs.

Bar: relative 1e-13 per entry, derived from the summation trees: both sides sum positive terms (error <= chain
length x u relative); the GPU's longest chain is <= ~460 additions at C3 (256 per accumulator in a 1024-column
chunk, 64 chunks, a 64-row scan segment, 10 scan levels, the segment back-accumulation), the oracle's BLAS dot a
few dozen, so |Delta| <= ~500 u ~ 5.6e-14 on the squares and half that on the norms.  Exact zeros, bitwise
run-to-run determinism.  Shapes span several 256-row blocks and 1024-column chunks with ragged tails, odd /
padded leading dimensions (the 8-byte path), and the extremes the scaling handles (1e-200, 1e200 columns;
squares that under- or overflow)."""
import numpy as np
import pytest

import inputs
import oracle

pytestmark = pytest.mark.gpu


def _dev(A, lda=None):
    import torch

    m, n = A.shape
    lda = lda or m
    buf = torch.zeros((n, lda), dtype=torch.float64, device="cuda")
    buf[:, :m] = torch.from_numpy(np.ascontiguousarray(A.T)).cuda()
    return buf.t()[:m, :]


TOL = 1e-13


@pytest.mark.parametrize("m,n,pad", [(1, 1, 0), (7, 3, 0), (1000, 37, 0), (4097, 129, 0), (3000, 50, 1), (2048, 300, 37),
                                     (65536, 4, 0)])
def test_column_norms_parity(gpu, m, n, pad):
    import torch

    import paper_2507_00976_b200 as bq

    A = inputs.gaussian(m, n, seed=m + n)
    dA = _dev(A, m + pad)
    got = bq.column_norms(dA).cpu().numpy()
    want = oracle.column_norms(A)
    assert np.all(np.abs(got - want) <= TOL * want), np.max(np.abs(got - want) / want)
    again = bq.column_norms(dA).cpu().numpy()
    assert np.array_equal(got, again)
    torch.cuda.synchronize()


def test_column_norms_extremes_and_zeros(gpu):
    import paper_2507_00976_b200 as bq

    A = inputs.gaussian(5000, 6, seed=2)
    A[:, 1] *= 1e-200
    A[:, 2] *= 1e200
    A[:, 3] = 0.0
    A[:, 4] *= 1e-160  # squares underflow to subnormals: the rescaled path
    A[:, 5] *= 1e155  # squares overflow: the rescaled path
    got = bq.column_norms(_dev(A)).cpu().numpy()
    want = oracle.column_norms(A)
    assert got[3] == 0.0
    nz = [0, 1, 2, 4, 5]
    assert np.all(np.abs(got[nz] - want[nz]) <= TOL * want[nz]), got / np.where(want > 0, want, 1)


@pytest.mark.parametrize("m,n,pad", [(1, 1, 0), (5, 9, 0), (300, 200, 0), (1500, 1300, 3), (2100, 2500, 0),
                                     (700, 3000, 0), (2600, 1100, 1)])
def test_trailing_norms_parity(gpu, m, n, pad):
    import paper_2507_00976_b200 as bq

    A = inputs.gaussian(m, n, seed=3 * m + n)
    got = bq.trailing_norms(_dev(A, m + pad)).cpu().numpy()
    mn = min(m, n)
    if mn <= 1500:
        want = oracle.trailing_norms(A)
    else:  # sampled: each entry by its definition
        idx = sorted(set([0, 1, 255, 256, 1023, 1024, mn // 2, mn - 2, mn - 1]))
        want = oracle.trailing_norms_at(A, idx)
        got = got[idx]
    assert np.all(np.abs(got - want) <= TOL * want), np.max(np.abs(got - want) / want)


def test_trailing_norms_of_a_factorization(gpu):
    """On a BQRRP output (reflectors below the diagonal, ignored): ||R(0:, 0:)||_F = ||A||_F (Q orthogonal), and
    the whole vector against the oracle's definition on the downloaded R."""
    import torch

    import paper_2507_00976_b200 as bq

    m, n, b = 1200, 900, 128
    A = inputs.gaussian(m, n, seed=11)
    dA = _dev(A)
    bq.factor(dA, b, b, seed=0)
    tn = bq.trailing_norms(dA).cpu().numpy()
    want = oracle.trailing_norms(dA.cpu().numpy())
    assert np.all(np.abs(tn - want) <= TOL * want)
    assert abs(tn[0] - np.linalg.norm(A)) <= 1e-13 * np.linalg.norm(A)
    torch.cuda.synchronize()


def test_norms_workspace_and_errors(gpu):
    import torch

    import paper_2507_00976_b200 as bq

    A = inputs.gaussian(300, 2100, seed=1)
    dA = _dev(A)
    need = bq.trailing_norms_workspace(300, 2100)
    ws = torch.empty(need, dtype=torch.uint8, device="cuda")
    a = bq.trailing_norms(dA, workspace=ws).cpu().numpy()
    b = bq.trailing_norms(dA).cpu().numpy()
    assert np.array_equal(a, b)
    small = torch.empty(max(need - 8, 1), dtype=torch.uint8, device="cuda")
    with pytest.raises(bq.BqrrpError):
        bq.trailing_norms(dA, workspace=small)


@pytest.mark.parametrize("rows,w,nt,pad", [(1000, 300, 64, 0), (4097, 700, 511, 1), (64, 5000, 4096, 0)])
def test_permute_touched_bitexact(gpu, rows, w, nt, pad):
    """The a3 touched-set move (bqrrp_debug_permute_touched, the kernels the factorization runs) against the oracle's
    column gather with J_qr = identity except J_qr(tq[t]) = tsrc[t] + 1: bit-exact."""
    import torch

    import paper_2507_00976_b200 as bq

    rng = np.random.default_rng(rows + w)
    X = inputs.gaussian(rows, w, seed=rows)
    tq = rng.choice(w, nt, replace=False).astype(np.int32)
    tsrc = tq[rng.permutation(nt)]
    Jqr = np.arange(1, w + 1, dtype=np.int64)
    Jqr[tq] = tsrc.astype(np.int64) + 1
    want = oracle.col_gather(X, Jqr)
    dX = _dev(X, rows + pad)
    bq.debug_permute_touched(dX, torch.from_numpy(tq).cuda(), torch.from_numpy(tsrc).cuda())
    assert np.array_equal(dX.cpu().numpy(), want)
