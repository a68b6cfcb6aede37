"""Pins of the oracle hopping term (section VIII-C) against facts that do
not come from the oracle itself: the Clifford algebra of the independently typed basis,
the free-field plane-wave closed form and spectrum, gauge covariance,
gamma5-hermiticity (reading R15), the checkerboard structure, and the matrix-element
(delta) form of PAPER.md:282 assembled densely on tiny lattices (incl. L_mu = 2)."""
import numpy as np
import pytest

import fieldgen
import oracle
from _physics import GAMMA, GAMMA5, c, r, neighbour, gauge_transform, colour_rotate, spin_apply, cdot


def test_basis_clifford_and_oracle_table():
    for a in range(4):
        assert np.allclose(GAMMA[a], GAMMA[a].conj().T)
        for b in range(4):
            assert np.allclose(GAMMA[a] @ GAMMA[b] + GAMMA[b] @ GAMMA[a], 2 * (a == b) * np.eye(4))
        # the oracle's own table must equal the independently typed one
        assert np.array_equal(oracle.gamma(a), GAMMA[a])
    # chiral basis: gamma5 = diag(1,1,-1,-1) -> clover is block diagonal
    assert np.allclose(GAMMA5, np.diag([1, 1, -1, -1]))


@pytest.mark.parametrize("L", [(4, 4, 4, 4), (6, 4, 2, 8)])
def test_free_field_plane_wave(L):
    """U = 1, psi(x) = exp(i p.x) u  ->  H psi = [2 sum cos p_mu - 2i sum sin p_mu gamma_mu] psi."""
    rng = np.random.default_rng(7)
    cx = fieldgen.coords(L)
    U = fieldgen.unit_gauge(L)
    for _ in range(4):
        n = rng.integers(0, 8, size=4)
        p = 2 * np.pi * n / np.array(L)
        u = rng.normal(size=(4, 3)) + 1j * rng.normal(size=(4, 3))
        phase = np.exp(1j * (cx @ p))
        psi = phase[:, None, None] * u[None]
        K = 2 * np.sum(np.cos(p)) * np.eye(4) - 2j * sum(np.sin(p[m]) * GAMMA[m] for m in range(4))
        expect = phase[:, None, None] * (K @ u)[None]
        got = c(oracle.hopping(U, r(psi), L))
        assert np.max(np.abs(got - expect)) < 1e-12 * np.max(np.abs(expect))


def test_constant_field_gives_eight():
    L = (4, 4, 4, 4)
    psi = np.broadcast_to(fieldgen.random_spinor((1, 1, 1, 1), 3), (256, 4, 3, 2)).copy()
    out = oracle.hopping(fieldgen.unit_gauge(L), psi, L)
    assert np.max(np.abs(out - 8 * psi)) < 1e-14 * np.max(np.abs(psi))


def _oracle_dense(U, L):
    V = fieldgen.volume(L)
    N = 12 * V
    D = np.zeros((N, N), dtype=complex)
    e = np.zeros((V, 4, 3, 2))
    for k in range(N):
        e.reshape(-1, 2)[k, 0] = 1.0
        D[:, k] = c(oracle.hopping(U, e, L)).ravel()
        e.reshape(-1, 2)[k, 0] = 0.0
    return D


def test_free_field_spectrum_closed_form():
    """Eigenvalues of H at U=1: 2 sum cos p -/+ 2i sqrt(sum sin^2 p), six-fold each."""
    L = (4, 4, 2, 2)
    D = _oracle_dense(fieldgen.unit_gauge(L), L)
    ev = np.linalg.eigvals(D)
    expect = []
    for n in np.ndindex(*L):
        p = 2 * np.pi * np.array(n) / np.array(L)
        a = 2 * np.cos(p).sum()
        b = 2 * np.sqrt((np.sin(p) ** 2).sum())
        expect += [a + 1j * b] * 6 + [a - 1j * b] * 6
    expect = np.array(expect)
    key = lambda z: np.lexsort((np.round(z.imag, 8), np.round(z.real, 8)))
    assert np.allclose(ev[key(ev)], expect[key(expect)], atol=1e-10)


@pytest.mark.parametrize("L", [(2, 2, 2, 2), (4, 2, 2, 2)])
def test_delta_form_dense(L):
    """Assemble H(x,x') exactly as written in PAPER.md:282 (delta form; += so that the
    two terms add when L_mu = 2) and compare with the oracle's stencil."""
    U = fieldgen.random_gauge(L, 11)
    Uc = c(U)
    V = fieldgen.volume(L)
    H = np.zeros((12 * V, 12 * V), dtype=complex)
    one = np.eye(4)
    for x in range(V):
        for mu in range(4):
            xp = neighbour(L, mu, +1)[x]
            xm = neighbour(L, mu, -1)[x]
            H[12 * x:12 * x + 12, 12 * xp:12 * xp + 12] += np.kron(one - GAMMA[mu], Uc[x, mu])
            H[12 * x:12 * x + 12, 12 * xm:12 * xm + 12] += np.kron(one + GAMMA[mu], Uc[xm, mu].conj().T)
    psi = fieldgen.random_spinor(L, 12)
    got = c(oracle.hopping(U, psi, L)).ravel()
    assert np.max(np.abs(got - H @ c(psi).ravel())) < 1e-13


def test_gauge_covariance():
    L = (4, 4, 4, 6)
    U = fieldgen.random_gauge(L, 21)
    g = fieldgen.random_gauge_transform(L, 22)
    psi = fieldgen.random_spinor(L, 23)
    lhs = oracle.hopping(gauge_transform(U, g, L), colour_rotate(psi, g), L)
    rhs = colour_rotate(oracle.hopping(U, psi, L), g)
    assert np.max(np.abs(lhs - rhs)) < 1e-12


def test_gamma5_hermiticity():
    """<chi, H psi> = <gamma5 H gamma5 chi, psi>  (gamma5 H gamma5 = H^dag; reading R15)."""
    L = (4, 4, 4, 4)
    U = fieldgen.random_gauge(L, 31)
    psi = fieldgen.random_spinor(L, 32)
    chi = fieldgen.random_spinor(L, 33)
    lhs = cdot(chi, oracle.hopping(U, psi, L))
    g5Hg5chi = spin_apply(GAMMA5, oracle.hopping(U, spin_apply(GAMMA5, chi), L))
    rhs = cdot(g5Hg5chi, psi)
    assert abs(lhs - rhs) < 1e-10 * abs(lhs)
    # the literal north-star form with a complex conjugate is false (R15): imaginary part flips
    assert abs(lhs - np.conj(rhs)) > 1e-3 * abs(lhs)


def test_checkerboard_structure():
    """H connects only opposite parities; out_parity restricts the output sites."""
    L = (4, 4, 4, 4)
    U = fieldgen.random_gauge(L, 41)
    psi = fieldgen.random_spinor(L, 42)
    par = fieldgen.parity(L)
    full = oracle.hopping(U, psi, L, -1)
    for p in (0, 1):
        part = oracle.hopping(U, psi, L, p)
        assert np.array_equal(part[par == p], full[par == p])
        assert not part[par != p].any()
        only = psi * (par == 1 - p)[:, None, None, None]
        h = oracle.hopping(U, only, L, -1)
        assert not h[par == 1 - p].any()       # H_pp = 0
        assert np.array_equal(h[par == p], full[par == p])


def test_point_source_neighbours():
    """psi = delta_y u: (H psi)(y - mu) = (1 - g_mu) U_mu(y - mu) u, (H psi)(y + mu) = (1 + g_mu) U_mu(y)^dag u,
    zero elsewhere (the delta form of PAPER.md:282 read column-wise)."""
    L = (6, 4, 4, 4)
    U = fieldgen.random_gauge(L, 51)
    V = fieldgen.volume(L)
    y = 37
    u = c(fieldgen.random_spinor((1, 1, 1, 1), 52))[0]
    psi = np.zeros((V, 4, 3), dtype=complex)
    psi[y] = u
    out = c(oracle.hopping(U, r(psi), L))
    Uc = c(U)
    touched = set()
    for mu in range(4):
        ym = neighbour(L, mu, -1)[y]
        yp = neighbour(L, mu, +1)[y]
        e_m = (np.eye(4) - GAMMA[mu]) @ (u @ Uc[ym, mu].T)
        e_p = (np.eye(4) + GAMMA[mu]) @ (u @ Uc[y, mu].conj())
        assert np.allclose(out[ym], e_m, atol=1e-14)
        assert np.allclose(out[yp], e_p, atol=1e-14)
        touched |= {ym, yp}
    rest = np.ones(V, bool)
    rest[list(touched)] = False
    assert not out[rest].any()


def test_thread_count_independent():
    L = (4, 4, 4, 8)
    U = fieldgen.random_gauge(L, 61)
    psi = fieldgen.random_spinor(L, 62)
    n = oracle.max_threads()
    oracle.set_threads(1)
    a = oracle.hopping(U, psi, L)
    oracle.set_threads(n)
    b = oracle.hopping(U, psi, L)
    assert np.array_equal(a, b)
