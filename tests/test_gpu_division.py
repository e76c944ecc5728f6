"""The engine's inline double division (fg_device.cuh qdiv, used by the
weighted SVM chain) against the CUDA runtime's IEEE division, bitwise; and
the device weighted null-space projection (fg_wproj, the three-weight
mpc_dyn_prox) against the reference's formula (operators.py:86-96)."""

import numpy as np
import pytest

import paper_1603_02526_b200 as fg
from paper_1603_02526_b200 import _native

pytestmark = pytest.mark.gpu


def bits(a):
    return np.ascontiguousarray(a, dtype=np.float64).view(np.uint64)


def assert_same(x, y):
    q, ref = _native.selftest_div(x, y)
    nan = np.isnan(ref)
    assert np.array_equal(np.isnan(q), nan)
    bad = np.flatnonzero((bits(q) != bits(ref)) & ~nan)
    assert bad.size == 0, [(x[i], y[i], q[i], ref[i]) for i in bad[:5]]


def test_qdiv_random_bit_patterns(gpu):
    rng = np.random.default_rng(0)
    n = 1 << 22
    x = rng.integers(0, 1 << 64, n, dtype=np.uint64, endpoint=False).view(np.float64)
    y = rng.integers(0, 1 << 64, n, dtype=np.uint64, endpoint=False).view(np.float64)
    assert_same(x, y)


def test_qdiv_moderate_values(gpu):
    """The common case: magnitudes the kernels see (fast sequence)."""
    rng = np.random.default_rng(1)
    n = 1 << 22
    x = rng.standard_normal(n) * 10.0 ** rng.uniform(-8, 8, n)
    y = rng.uniform(0.05, 20.0, n) * rng.choice([-1.0, 1.0], n)
    assert_same(x, y)
    # weights as users write them, including exact ties of the quotient
    w = np.array([0.1, 0.3, 0.7, 1.3, 1.5, 2.5, 3.0, 5.0, 7.0, 1.0 / 3.0])
    xs = rng.standard_normal(1 << 16)
    assert_same(np.repeat(xs, w.size), np.tile(w, xs.size))


def test_qdiv_edges_and_specials(gpu):
    sp = np.array([0.0, -0.0, np.inf, -np.inf, np.nan, 1.0, -1.0, 5e-324, -5e-324,
                   2.2250738585072014e-308, 2.225073858507201e-308, 1.7976931348623157e308,
                   -1.7976931348623157e308, 1e-300, 1e300, 3.0, 0.1, 2.0 ** -1022,
                   2.0 ** 1023, 2.0 ** -1074 * 3, 1.5 * 2.0 ** -1060])
    x = np.repeat(sp, sp.size)
    y = np.tile(sp, sp.size)
    assert_same(x, y)


@pytest.mark.parametrize("lo,hi", [(-1080, -1015), (-1120, -900), (880, 1030), (-200, 200)])
def test_qdiv_exponent_bands(gpu, lo, hi):
    """Quotients around the subnormal and overflow thresholds, and operands
    outside the fast sequence's range (the exact-rescale path), with
    quotients that tie on the subnormal grid."""
    rng = np.random.default_rng(abs(lo) + 7 * abs(hi))
    n = 1 << 21
    ey = rng.integers(-600, 600, n)
    eq = rng.integers(lo, hi, n)
    my = rng.uniform(1.0, 2.0, n)
    mq = rng.uniform(1.0, 2.0, n)
    y = np.ldexp(my, ey) * rng.choice([-1.0, 1.0], n)
    x = np.ldexp(mq, eq) * np.abs(y)          # x / y ~ 2^eq (rounded products)
    assert_same(x, y)
    # exact subnormal ties: x = (k + 0.5) * 2^-1074 * y with y a small odd integer
    k = rng.integers(0, 1 << 40, n).astype(np.float64)
    yy = rng.choice([3.0, 5.0, 7.0, 9.0], n)
    xx = np.ldexp((k + 0.5) * yy, -1074 + 1)
    assert_same(xx, np.ldexp(yy, 1))


def reference_projection(M, nv, w):
    """operators.py:86-96 for one shared M (NumPy, as the reference)."""
    winv = 1.0 / w
    S = (M * winv) @ M.T
    lam = np.linalg.solve(S, M @ nv)
    return nv - winv * (M.T @ lam)


def test_wproj_matches_reference_formula(gpu):
    rng = np.random.default_rng(3)
    for d, k in ((1, 1), (4, 2), (16, 4)):
        A = 0.3 * rng.standard_normal((d, d))
        B = rng.standard_normal((d, k))
        sys_ = fg.LinearSystem(A, B)
        for _ in range(5):
            nv = rng.standard_normal(2 * d + k)
            w = np.concatenate([np.full(d, rng.uniform(0.2, 5)), np.full(k, rng.uniform(0.2, 5)),
                                np.full(d, rng.uniform(0.2, 5))])
            got = _native.wproj(sys_.M, nv, w)[0]
            want = reference_projection(sys_.M, nv, w)
            np.testing.assert_allclose(got, want, rtol=1e-12, atol=1e-12)
            assert np.max(np.abs(sys_.M @ got)) < 1e-10


def test_mpc_dyn_prox_three_weights(gpu):
    """The reference's own checks (test_operators.py:180-193)."""
    sys_ = fg.LinearSystem([[0.5]], [[2.0]])
    a = fg.mpc_dyn_prox([1.0], [-1.0], [0.7], sys_, 1.0, 2.0, 3.0)
    b = fg.mpc_dyn_prox([1.0], [-1.0], [0.7], sys_, 10.0, 20.0, 30.0)
    for x, y in zip(a, b):
        np.testing.assert_allclose(x, y)
    assert abs(float(sys_.residual(*a)[0])) < 1e-12
    want = reference_projection(sys_.M, np.array([1.0, -1.0, 0.7]), np.array([1.0, 2.0, 3.0]))
    np.testing.assert_allclose(np.concatenate(a), want, rtol=1e-13)
    with pytest.raises(ValueError):
        fg.mpc_dyn_prox([1.0], [-1.0], [0.7], sys_, 1.0, 0.0, 3.0)
