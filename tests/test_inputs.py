"""The counter-based device input generator (inputs.counter_gaussian): its int64 torch hash equals splitmix64
written in Python's unbounded integers mod 2^64 (so the wrapping multiplies and masked shifts are right), its
values are N(0,1) (moments, KS), and it is chunking-independent and seed-dependent."""
import math

import numpy as np
import torch

import inputs

MASK = (1 << 64) - 1


def _splitmix64_ref(z):
    z &= MASK
    z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & MASK
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & MASK
    return z ^ (z >> 31)


def test_hash_matches_unsigned_reference():
    xs = [0, 1, 2, 12345, (1 << 63) - 1, -1, -(1 << 63), 0x0123456789ABCDEF, -0x0123456789ABCDEF]
    got = inputs._splitmix64_torch(torch.tensor(xs, dtype=torch.int64)).tolist()
    for x, g in zip(xs, got):
        assert g & MASK == _splitmix64_ref(x & MASK), hex(x)


def test_entry_formula_and_distribution():
    m, n, seed = 300, 200, 9
    A = inputs.counter_gaussian(m, n, seed=seed, device="cpu")
    assert A.shape == (m, n) and A.stride() == (1, m)
    key = (seed * 0x632BE59BD9B4E019) & ((1 << 63) - 1)
    for i, j in [(0, 0), (299, 0), (5, 77), (299, 199)]:
        base = ((i + j * m) * 2 * 0x9E3779B97F4A7C15 + key) & MASK
        h1, h2 = _splitmix64_ref(base), _splitmix64_ref(base + 0x9E3779B97F4A7C15)
        u1 = ((h1 >> 11) + 0.5) * 2.0 ** -53
        u2 = (h2 >> 11) * 2.0 ** -53
        z = math.sqrt(-2.0 * math.log(u1)) * math.cos(2.0 * math.pi * u2)
        assert abs(float(A[i, j]) - z) <= 1e-14 * max(1.0, abs(z))
    x = A.numpy().ravel()
    assert abs(x.mean()) < 0.02 and abs(x.std() - 1.0) < 0.02
    from scipy import stats

    assert stats.kstest(x, "norm").pvalue > 1e-3


def test_chunking_and_seed():
    A = inputs.counter_gaussian(123, 45, seed=1, device="cpu")
    B = inputs.counter_gaussian(123, 45, seed=1, device="cpu", chunk=1000)
    C = inputs.counter_gaussian(123, 45, seed=2, device="cpu")
    assert torch.equal(A, B) and not torch.equal(A, C)
    assert np.all(np.isfinite(A.numpy()))
