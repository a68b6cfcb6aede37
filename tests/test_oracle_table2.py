"""Pins of the oracle's Table II test functions (section VI): algebraic facts
that do not come from the oracle -- SU(3) closure and norm preservation, associativity
between lcm and upsi, linearity of matvec, and gamma-matrix products typed by hand."""
import numpy as np

import fieldgen
import oracle
from _physics import GAMMA, c, r


def test_lcm_su3_closure_and_associativity():
    n = 64
    a = fieldgen.random_su3(n, 1)
    b = fieldgen.random_su3(n, 2)
    d = fieldgen.random_su3(n, 3)
    ab = c(oracle.lcm(a, b))
    # product of SU(3) matrices is SU(3)
    assert np.max(np.abs(ab @ np.conj(np.swapaxes(ab, 1, 2)) - np.eye(3))) < 1e-14
    assert np.max(np.abs(np.linalg.det(ab) - 1)) < 1e-14
    # (a b) d = a (b d)
    lhs = oracle.lcm(oracle.lcm(a, b), d)
    rhs = oracle.lcm(a, oracle.lcm(b, d))
    assert np.max(np.abs(lhs - rhs)) < 1e-14
    # identity
    one = np.zeros((n, 3, 3, 2))
    one[:, [0, 1, 2], [0, 1, 2], 0] = 1.0
    assert np.array_equal(oracle.lcm(a, one), a)


def test_lcm_hand_example():
    """diag(1, i, -1) times the cyclic permutation P (P e_j = e_{j+1}) = rows of P scaled."""
    a = np.zeros((1, 3, 3), dtype=complex)
    a[0] = np.diag([1, 1j, -1])
    p = np.zeros((1, 3, 3), dtype=complex)
    p[0, 1, 0] = p[0, 2, 1] = p[0, 0, 2] = 1
    out = c(oracle.lcm(r(a), r(p)))[0]
    expect = np.array([[0, 0, 1], [1j, 0, 0], [0, -1, 0]])
    assert np.array_equal(out, expect)


def test_upsi_norm_and_consistency():
    n = 50
    u = fieldgen.random_su3(n, 4)
    v = fieldgen.random_su3(n, 5)
    psi = fieldgen.random_spinor((n, 1, 1, 1), 6)
    out = oracle.upsi(u, psi)
    # unitary colour rotation preserves each spin component's colour norm
    assert np.allclose(np.sum(out ** 2, axis=(2, 3)), np.sum(psi ** 2, axis=(2, 3)), rtol=1e-14, atol=0)
    # (u v) psi = u (v psi)
    assert np.max(np.abs(oracle.upsi(oracle.lcm(u, v), psi) - oracle.upsi(u, oracle.upsi(v, psi)))) < 1e-14
    # a hand case: u = P (cyclic), psi = e_0 on spin 2 -> e_1 on spin 2
    p = np.zeros((1, 3, 3), dtype=complex)
    p[0, 1, 0] = p[0, 2, 1] = p[0, 0, 2] = 1
    e = np.zeros((1, 4, 3), dtype=complex)
    e[0, 2, 0] = 2 - 1j
    got = c(oracle.upsi(r(p), r(e)))
    assert got[0, 2, 1] == 2 - 1j and np.count_nonzero(got) == 1


def test_adj_upsi_inverts_upsi():
    """For SU(3) u: adj(u) (u psi) = psi; and adj(u) differs from u (a transposition bug would not)."""
    n = 30
    u = fieldgen.random_su3(n, 10)
    psi = fieldgen.random_spinor((n, 1, 1, 1), 11)
    assert np.max(np.abs(oracle.adj_upsi(u, oracle.upsi(u, psi)) - psi)) < 1e-14
    assert np.max(np.abs(oracle.adj_upsi(u, psi) - oracle.upsi(u, psi))) > 0.1
    # hand case: u = i * identity -> adj(u) psi = -i psi
    ui = np.zeros((1, 3, 3), dtype=complex)
    ui[0] = 1j * np.eye(3)
    p = c(fieldgen.random_spinor((1, 1, 1, 1), 12))
    assert np.allclose(c(oracle.adj_upsi(r(ui), r(p))), -1j * p, atol=0, rtol=1e-15)


def test_matvec_linearity():
    n = 40
    u = fieldgen.random_su3(n, 7)
    p1 = fieldgen.random_spinor((n, 1, 1, 1), 8)
    p2 = fieldgen.random_spinor((n, 1, 1, 1), 9)
    assert np.max(np.abs(oracle.matvec(u, p1, p2) - oracle.upsi(u, p1 + p2))) < 1e-14


def _spm(M, n=2):
    return r(np.broadcast_to(M, (n, 4, 4)).copy())


def test_spmat_gamma_products():
    """Clifford algebra through spmat, and one hand-computed non-symmetric product
    (gamma_x gamma_z = [[0,-1],[1,0]] in each chiral block of the DeGrand-Rossi basis)."""
    for mu in range(4):
        for nu in range(4):
            s = c(oracle.spmat(_spm(GAMMA[mu]), _spm(GAMMA[nu]))) + c(oracle.spmat(_spm(GAMMA[nu]), _spm(GAMMA[mu])))
            assert np.array_equal(s[0], 2 * (mu == nu) * np.eye(4))
    xz = c(oracle.spmat(_spm(GAMMA[0]), _spm(GAMMA[2])))[0]
    blk = np.array([[0, -1], [1, 0]])
    expect = np.zeros((4, 4), dtype=complex)
    expect[:2, :2] = blk
    expect[2:, 2:] = blk
    assert np.array_equal(xz, expect)
    g5 = _spm(GAMMA[0])
    for mu in (1, 2, 3):
        g5 = oracle.spmat(g5, _spm(GAMMA[mu]))
    assert np.array_equal(c(g5)[0], np.diag([1, 1, -1, -1]).astype(complex))
