"""Pins of the oracle clover term (eq. (1); reading R10) and of the
even-odd CGNR solve (readings R12-R14).

Clover: Hermitian, block-diagonal in chirality, U = 1 -> (4+m) 1,
trace, gauge covariance, and the closed-form spectrum (4+m) +/- (c_SW/2) f_c of a
constant abelian field strength embedded in SU(3).  The overall sign of c_SW is a
convention and stays "parity unpinned" (R10).

CG: the reconstructed full solution equals numpy.linalg.solve of the dense M = A - H/2,
the true residual respects the stopping tolerance, and the history does not depend on
the thread count."""
import numpy as np
import pytest

import fieldgen
import oracle
from _physics import GAMMA5, c, r, gauge_transform


def _dense_clover(A):
    return c(A)  # [V,12,12]


def test_clover_unit_gauge_is_mass():
    L = (4, 4, 4, 4)
    A = oracle.clover_build(fieldgen.unit_gauge(L), L, 0.1, 1.3)
    expect = np.zeros_like(A)
    for i in range(12):
        expect[:, i, i, 0] = 4.1
    assert np.array_equal(A, expect)


def test_clover_hermitian_chiral_blocks_trace():
    L = (4, 4, 4, 4)
    U = fieldgen.random_gauge(L, 71)
    Ac = _dense_clover(oracle.clover_build(U, L, 0.1, 1.0))
    assert np.max(np.abs(Ac - np.conj(np.swapaxes(Ac, 1, 2)))) < 1e-15
    g5 = np.kron(GAMMA5, np.eye(3))
    assert np.max(np.abs(Ac @ g5 - g5 @ Ac)) == 0.0          # two 6x6 blocks
    assert np.max(np.abs(np.trace(Ac, axis1=1, axis2=2) - 12 * 4.1)) < 1e-13
    assert np.max(np.abs(Ac - 4.1 * np.eye(12))) > 0.1        # a real clover term is present


def test_clover_gauge_covariance():
    L = (4, 4, 4, 4)
    U = fieldgen.random_gauge(L, 72)
    g = fieldgen.random_gauge_transform(L, 73)
    A = _dense_clover(oracle.clover_build(U, L, -0.2, 1.7))
    Ag = _dense_clover(oracle.clover_build(gauge_transform(U, g, L), L, -0.2, 1.7))
    G = np.einsum("ij,sab->siajb", np.eye(4), c(g)).reshape(-1, 12, 12)
    assert np.max(np.abs(Ag - G @ A @ np.conj(np.swapaxes(G, 1, 2)))) < 1e-13


@pytest.mark.parametrize("csw", [1.0, 2.5])
def test_clover_constant_abelian_field_spectrum(csw):
    """U_y(x) = diag(e^{i phi_c x}), U_x = diag(e^{-i phi_c Lx y}) on the last x slice,
    phi_c = 2 pi n_c / (Lx Ly), n = (1, 2, -3): every xy plaquette is e^{i phi_c}, so
    F_xy = sin(phi_c) - mean(sin phi) (Hermitian, traceless) and
    A = (4+m) + (c_SW/2) sigma_xy F_xy has eigenvalues (4+m) +/- (c_SW/2) f_c, doubly."""
    L = (4, 6, 2, 2)
    m = 0.05
    cx = fieldgen.coords(L)
    V = len(cx)
    phi = 2 * np.pi * np.array([1, 2, -3]) / (L[0] * L[1])
    U = np.zeros((V, 4, 3, 3), dtype=complex)
    for mu in range(4):
        U[:, mu] = np.eye(3)
    for a in range(3):
        U[:, 1, a, a] = np.exp(1j * phi[a] * cx[:, 0])
        last = cx[:, 0] == L[0] - 1
        U[last, 0, a, a] = np.exp(-1j * phi[a] * L[0] * cx[last, 1])
    f = np.sin(phi) - np.sin(phi).mean()
    expect = np.sort(np.concatenate([4 + m + 0.5 * csw * f, 4 + m + 0.5 * csw * f,
                                     4 + m - 0.5 * csw * f, 4 + m - 0.5 * csw * f]))
    A = _dense_clover(oracle.clover_build(r(U), L, m, csw))
    for s in range(V):
        ev = np.sort(np.linalg.eigvalsh(A[s]))
        assert np.max(np.abs(ev - expect)) < 1e-13


def test_clover_invert_and_apply():
    L = (4, 4, 4, 4)
    U = fieldgen.random_gauge(L, 74)
    A = oracle.clover_build(U, L, 0.1, 1.0)
    Ai = oracle.clover_invert(A, L)
    Ac, Aic = c(A), c(Ai)
    assert np.max(np.abs(Ac @ Aic - np.eye(12))) < 1e-13
    assert np.max(np.abs(Aic - np.linalg.inv(Ac))) < 1e-13
    psi = fieldgen.random_spinor(L, 75)
    out = c(oracle.clover_apply(A, psi, L)).reshape(-1, 12)
    assert np.max(np.abs(out - np.einsum("sij,sj->si", Ac, c(psi).reshape(-1, 12)))) < 1e-12


def _dense_M(U, A, m, L):
    V = fieldgen.volume(L)
    N = 12 * V
    M = np.zeros((N, N), dtype=complex)
    e = np.zeros((V, 4, 3, 2))
    for k in range(N):
        e.reshape(-1, 2)[k, 0] = 1.0
        M[:, k] = c(oracle.wilson_apply(U, A, m, e, L)).ravel()
        e.reshape(-1, 2)[k, 0] = 0.0
    return M


@pytest.mark.parametrize("clover", [False, True])
def test_cg_matches_dense_solve(clover):
    L = (4, 4, 2, 4)
    m = 0.1
    U = fieldgen.random_gauge(L, 81)
    A = oracle.clover_build(U, L, m, 1.0) if clover else None
    b = fieldgen.random_spinor(L, 82)
    res = oracle.cg_solve(U, b, L, m, A=A, tol=1e-12, maxit=1000)
    assert res["status"] == 0
    M = _dense_M(U, A, m, L)
    # the full operator itself: H part pinned in test_oracle_dslash, A part above
    xd = np.linalg.solve(M, c(b).ravel())
    x = c(res["x"]).ravel()
    assert np.linalg.norm(x - xd) / np.linalg.norm(xd) < 1e-9
    assert res["true_resid"] < 1e-10
    h = res["hist"]
    assert len(h) == res["iters"] + 1 and h[0] == 1.0 and h[-1] <= 1e-12


def test_cg_tolerance_and_determinism():
    L = (4, 4, 4, 4)
    U = fieldgen.random_gauge(L, 83)
    A = oracle.clover_build(U, L, 0.1, 1.0)
    b = fieldgen.random_spinor(L, 84)
    n = oracle.max_threads()
    oracle.set_threads(1)
    r1 = oracle.cg_solve(U, b, L, 0.1, A=A, tol=1e-10, maxit=500)
    oracle.set_threads(n)
    r2 = oracle.cg_solve(U, b, L, 0.1, A=A, tol=1e-10, maxit=500)
    assert r1["iters"] == r2["iters"] and np.array_equal(r1["hist"], r2["hist"])
    assert r1["hist"][-1] <= 1e-10 and r1["hist"][-2] > 1e-10
    assert r1["true_resid"] < 5e-10
    # maxit cap: status 1, x holds the last iterate
    r3 = oracle.cg_solve(U, b, L, 0.1, A=A, tol=1e-10, maxit=5)
    assert r3["status"] == 1 and r3["iters"] == 5
    assert np.array_equal(r3["hist"], r1["hist"][:6])
