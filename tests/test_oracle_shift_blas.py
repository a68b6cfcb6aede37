"""Pins of the oracle's shift (section II-C) and lattice BLAS
(north star) against exact arithmetic: coordinate-encoded fields (bit-exact), group
identities of the circular shift, integer-valued reductions (exact), math.fsum."""
import math

import numpy as np
import pytest

import fieldgen
import oracle


def _code_field(L, nreal):
    """f(x)[k] = exactly representable code of (x, y, z, t, k)."""
    cx = fieldgen.coords(L)
    V = len(cx)
    k = np.arange(nreal)
    base = cx[:, 0] + 100 * cx[:, 1] + 10_000 * cx[:, 2] + 1_000_000 * cx[:, 3]
    return (base[:, None] * 100 + k[None, :]).astype(np.float64).reshape(V, nreal)


@pytest.mark.parametrize("L", [(4, 4, 4, 4), (2, 6, 4, 2), (6, 2, 2, 8)])
@pytest.mark.parametrize("nreal", [24, 72])
def test_shift_coordinate_code(L, nreal):
    f = _code_field(L, nreal)
    cx = fieldgen.coords(L)
    for mu in range(4):
        for sign in (+1, -1):
            out = oracle.shift(f, L, mu, sign)
            n = cx.copy()
            n[:, mu] = (n[:, mu] + sign) % L[mu]
            expect = _code_field(L, nreal)[n[:, 0] + L[0] * (n[:, 1] + L[1] * (n[:, 2] + L[2] * n[:, 3]))]
            assert np.array_equal(out, expect)


def test_shift_group_identities():
    L = (4, 6, 2, 4)
    f = fieldgen.random_spinor(L, 5).reshape(fieldgen.volume(L), 24)
    for mu in range(4):
        assert np.array_equal(oracle.shift(oracle.shift(f, L, mu, +1), L, mu, -1), f)
        g = f
        for _ in range(L[mu]):
            g = oracle.shift(g, L, mu, +1)
        assert np.array_equal(g, f)


def test_reductions_exact_integers():
    L = (4, 4, 4, 8)
    V = fieldgen.volume(L)
    rng = np.random.default_rng(1)
    a = rng.integers(-1000, 1000, size=(V, 4, 3, 2)).astype(np.float64)
    b = rng.integers(-1000, 1000, size=(V, 4, 3, 2)).astype(np.float64)
    par = fieldgen.parity(L)
    for sub in (-1, 0, 1):
        m = np.ones(V, bool) if sub < 0 else par == sub
        ai = a[m].astype(np.int64)
        bi = b[m].astype(np.int64)
        assert oracle.norm2(a, L, sub) == float((ai ** 2).sum())
        re = (ai[..., 0] * bi[..., 0] + ai[..., 1] * bi[..., 1]).sum()
        im = (ai[..., 0] * bi[..., 1] - ai[..., 1] * bi[..., 0]).sum()
        assert oracle.inner(a, b, L, sub) == complex(re, im)


def test_reductions_vs_fsum_and_linearity():
    L = (4, 4, 4, 4)
    a = fieldgen.random_spinor(L, 8)
    b = fieldgen.random_spinor(L, 9)
    n2 = oracle.norm2(a, L)
    assert abs(n2 - math.fsum((a.ravel() ** 2).tolist())) <= 1e-15 * n2
    # norm2(a) = <a,a>; conjugate-linear in the first argument
    assert abs(oracle.inner(a, a, L) - n2) <= 1e-14 * n2
    ia = np.stack([-a[..., 1], a[..., 0]], axis=-1)          # i*a
    ab = oracle.inner(a, b, L)
    assert abs(oracle.inner(ia, b, L) - (-1j) * ab) <= 1e-13 * abs(ab)
    assert abs(oracle.inner(b, a, L) - np.conj(ab)) <= 1e-13 * abs(ab)


def test_axpy_exact():
    L = (4, 4, 4, 4)
    V = fieldgen.volume(L)
    rng = np.random.default_rng(2)
    x = rng.integers(-64, 64, size=(V, 4, 3, 2)).astype(np.float64)
    y = rng.integers(-64, 64, size=(V, 4, 3, 2)).astype(np.float64)
    par = fieldgen.parity(L)
    out = oracle.axpy(0.5 - 2j, x, y, L, 1)
    xc = x[..., 0] + 1j * x[..., 1]
    yc = y[..., 0] + 1j * y[..., 1]
    e = (0.5 - 2j) * xc + yc
    odd = par == 1
    assert np.array_equal(out[odd][..., 0], e[odd].real)
    assert np.array_equal(out[odd][..., 1], e[odd].imag)
    assert np.array_equal(out[~odd], y[~odd])
