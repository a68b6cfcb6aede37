"""Pins of the oracle multi-shift CG (orc_cg_multishift; reading R25): the solver of the
RHMC runs the paper's production lattice is used for (ref. [14]).

The even-odd operator is pinned independently of the oracle's own Mhat code: the dense
Schur complement Mhat = M_oo - M_oe M_ee^-1 M_eo of the dense full M = A - H/2 (whose hopping
and clover parts are pinned in test_oracle_dslash / test_oracle_clover_cg), computed with
numpy; each shifted solution must equal numpy.linalg.solve((Mhat^dag Mhat + sigma_i), phi_o)."""
import numpy as np
import pytest

import fieldgen
import oracle
from _physics import c


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


def _schur(U, A, m, L):
    """dense Mhat on the odd sites (index order: odd sites in lexicographic order, 12 each)"""
    M = _dense_M(U, A, m, L)
    par = fieldgen.parity(L)
    ev = np.repeat(par == 0, 12)
    od = ~ev
    Mee, Meo, Moe, Moo = M[np.ix_(ev, ev)], M[np.ix_(ev, od)], M[np.ix_(od, ev)], M[np.ix_(od, od)]
    return Moo - Moe @ np.linalg.solve(Mee, Meo), od


L0 = (4, 4, 2, 4)


@pytest.fixture(scope="module", params=[False, True], ids=["wilson", "clover"])
def setup(request):
    m = 0.1
    U = fieldgen.random_gauge(L0, 91)
    A = oracle.clover_build(U, L0, m, 1.0) if request.param else None
    Mh, od = _schur(U, A, m, L0)
    return U, A, m, Mh, od


def test_mhat_apply_is_the_schur_complement(setup):
    U, A, m, Mh, od = setup
    v = fieldgen.random_spinor(L0, 92)
    vo = c(v).ravel()[od]
    got = c(oracle.mhat_apply(U, A, m, v, L0)).ravel()
    gotd = c(oracle.mhat_apply(U, A, m, v, L0, dagger=True)).ravel()
    assert np.max(np.abs(got[~od])) == 0.0
    assert np.linalg.norm(got[od] - Mh @ vo) <= 1e-13 * np.linalg.norm(Mh @ vo)
    assert np.linalg.norm(gotd[od] - Mh.conj().T @ vo) <= 1e-13 * np.linalg.norm(vo)


def test_multishift_matches_dense_solves(setup):
    U, A, m, Mh, od = setup
    phi = fieldgen.random_spinor(L0, 93)
    sigma = [0.0, 0.01, 0.1, 0.5, 2.0, 10.0]
    res = oracle.cg_multishift(U, phi, L0, m, sigma, A=A, tol=1e-12, maxit=2000)
    assert res["status"] == 0
    K = Mh.conj().T @ Mh
    b = c(phi).ravel()[od]
    for i, s in enumerate(sigma):
        xd = np.linalg.solve(K + s * np.eye(len(b)), b)
        xi = c(res["x"][i]).ravel()
        assert np.max(np.abs(xi[~od])) == 0.0
        assert np.linalg.norm(xi[od] - xd) <= 1e-9 * np.linalg.norm(xd), (i, s)
        # true residual is the independently computed one
        tr = np.linalg.norm(b - (K + s * np.eye(len(b))) @ xi[od]) / np.linalg.norm(b)
        assert abs(tr - res["true_resid"][i]) <= 1e-14 and tr <= 5e-12
    # larger shifts are better conditioned: they stop no later than smaller ones
    assert all(np.diff(res["conv_iter"]) <= 0) and res["conv_iter"][0] == res["iters"]


def test_multishift_base_is_plain_cg_and_order_free(setup):
    """sigma = [s] alone is plain CG on Mhat^dag Mhat + s (same Krylov iteration as any
    base); the non-base shifts can be listed in any order."""
    U, A, m, Mh, od = setup
    phi = fieldgen.random_spinor(L0, 94)
    one = oracle.cg_multishift(U, phi, L0, m, [0.05], A=A, tol=1e-10, maxit=2000)
    many = oracle.cg_multishift(U, phi, L0, m, [0.05, 0.3, 1.0], A=A, tol=1e-10, maxit=2000)
    perm = oracle.cg_multishift(U, phi, L0, m, [0.05, 1.0, 0.3], A=A, tol=1e-10, maxit=2000)
    assert one["iters"] == many["iters"] and np.array_equal(one["hist"], many["hist"])
    assert np.array_equal(one["x"][0], many["x"][0])
    assert np.array_equal(many["x"][1], perm["x"][2]) and np.array_equal(many["x"][2], perm["x"][1])


def test_multishift_collinear_residuals_and_maxit(setup):
    """|r_i| = zeta_i |r|: a shift's true residual at its stop is <= tol; maxit caps."""
    U, A, m, Mh, od = setup
    phi = fieldgen.random_spinor(L0, 95)
    res = oracle.cg_multishift(U, phi, L0, m, [0.0, 0.2, 4.0], A=A, tol=1e-8, maxit=2000)
    assert np.all(res["true_resid"] <= 2e-8)
    cap = oracle.cg_multishift(U, phi, L0, m, [0.0, 0.2, 4.0], A=A, tol=1e-8, maxit=3)
    assert cap["status"] == 1 and cap["iters"] == 3 and np.array_equal(cap["hist"], res["hist"][:4])
    with pytest.raises(ValueError):
        oracle.cg_multishift(U, phi, L0, m, [0.5, 0.1], A=A)
