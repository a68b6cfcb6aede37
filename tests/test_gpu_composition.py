"""The paper's Fig. 1 evaluated with the library's own data-parallel
building blocks -- shift(), colour-matrix x fermion and adj(colour matrix) x fermion site
expressions, axpy -- and checked (1) against the oracle's literal Fig. 1 expression and (2)
assembled into the Wilson hopping term of PAPER.md:282, against the fused dslash kernel:
  D+_mu = u[mu] * shift(phi, mu, FORWARD),  D-_mu = shift(adj(u[mu]) * phi, mu, BACKWARD)
  H phi = sum_mu (D+_mu + D-_mu) - gamma_mu (D+_mu - D-_mu)
(the gamma_mu products are applied on the host with the independently typed basis)."""
import numpy as np
import pytest

import fieldgen
import oracle
from _physics import GAMMA, c, r, rel_site_err

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def q():
    from paper_1408_5925_b200 import qdpb
    qdpb.lib()
    return qdpb


@pytest.mark.parametrize("mask", [0, 12])
def test_fig1_composition_equals_fused_dslash(q, mask):
    L = (6, 4, 4, 8)
    V = fieldgen.volume(L)
    U = fieldgen.random_gauge(L, 2201)
    phi = fieldgen.random_spinor(L, 3201)
    c_ = q.qdp_init(L)
    q.qdp_set_option(c_, q.QDP_OPT_SELF_HALO, mask)
    try:
        F = lambda kind: q.qdp_field_alloc(c_, kind, 0, q.QDP_ALL)
        fphi, fs, fa, fb, fbs = (F(q.QDP_FERMION) for _ in range(5))
        q.qdp_field_import(fphi, phi)
        fu = F(q.QDP_COLORMATRIX)
        H = np.zeros((V, 4, 3), dtype=complex)
        for mu in range(4):
            q.qdp_field_import(fu, np.ascontiguousarray(U[:, mu]))
            q.qdp_shift(fs, fphi, mu, q.QDP_FORWARD)             # phi(x+mu)
            q.qdp_expr(q.QDP_EXPR_UPSI, fa, fu, fs)                # D+ = u[mu] shift(phi, +)
            q.qdp_expr(q.QDP_EXPR_ADJ_UPSI, fb, fu, fphi)          # adj(u[mu]) phi
            q.qdp_shift(fbs, fb, mu, q.QDP_BACKWARD)             # D- = shift(adj(u) phi, -)
            dp = q.qdp_field_export(fa)
            dm = q.qdp_field_export(fbs)
            # Fig. 1's psi against the oracle's literal expression
            q.qdp_axpy(1.0, fbs, fa)
            ref = oracle.upsi(U[:, mu], oracle.shift(phi.reshape(V, -1), L, mu, +1).reshape(phi.shape)) + \
                oracle.shift(oracle.adj_upsi(U[:, mu], phi).reshape(V, -1), L, mu, -1).reshape(phi.shape)
            assert rel_site_err(q.qdp_field_export(fa), ref) <= 1e-14
            # assemble the hopping term: (1 - g) D+ + (1 + g) D-
            Dp, Dm = c(dp), c(dm)
            H += (Dp + Dm) - np.einsum("ij,sjc->sic", GAMMA[mu], Dp - Dm)
        fo = F(q.QDP_FERMION)
        q.qdp_dslash(fo, q_gauge(q, c_, U), fphi, q.QDP_ALL)
        assert rel_site_err(q.qdp_field_export(fo), r(H)) <= 1e-13
    finally:
        q.qdp_finalize(c_)


def q_gauge(q, c_, U):
    f = q.qdp_field_alloc(c_, q.QDP_GAUGE, 0, q.QDP_ALL)
    q.qdp_field_import(f, U)
    return f
