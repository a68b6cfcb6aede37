"""Mixed-precision CGNR with reliable updates (qdp_cg_solve_mixed; the paper's ref. [2]).
The iteration history is not the oracle's (a different algorithm); what is pinned is the
answer: the solution agrees with the oracle's fp64 even-odd CG solution of the same system
within the solver tolerance, the true residual meets it, and convergence was declared on an
fp64 residual (at least one reliable update)."""
import numpy as np
import pytest

import fieldgen
import oracle
from _physics import rel_site_err

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def q():
    from paper_1408_5925_b200 import qdpb
    qdpb.lib()
    return qdpb


def _field(q, c, kind, prec, subset, host):
    f = q.qdp_field_alloc(c, kind, prec, subset)
    q.qdp_field_import(f, np.ascontiguousarray(host, dtype=np.float64 if prec == 0 else np.float32))
    return f


@pytest.mark.parametrize("clover,gk", [(False, 1), (True, 1), (True, 3)])
@pytest.mark.parametrize("L", [(8, 8, 8, 8), (16, 16, 16, 16)])
def test_mixed_cg_solution(q, clover, gk, L):
    m = 0.1
    U = fieldgen.random_gauge(L, 1901)
    b = fieldgen.random_spinor(L, 2901)
    A = oracle.clover_build(U, L, m, 1.0) if clover else None
    ref = oracle.cg_solve(U, b, L, m, A=A, tol=1e-11, maxit=2000)
    c = q.qdp_init(L)
    try:
        fU = _field(q, c, gk, 0, q.QDP_ALL, U)
        fUs = _field(q, c, gk, 1, q.QDP_ALL, U)
        fb = _field(q, c, q.QDP_FERMION, 0, q.QDP_ALL, b)
        fx = q.qdp_field_alloc(c, q.QDP_FERMION, 0, q.QDP_ALL)
        fA = fAi = fAs = fAis = None
        if clover:
            fA = q.qdp_field_alloc(c, q.QDP_CLOVER, 0, q.QDP_ALL)
            fAi = q.qdp_field_alloc(c, q.QDP_CLOVER, 0, q.QDP_EVEN)
            fAs = q.qdp_field_alloc(c, q.QDP_CLOVER, 1, q.QDP_ODD)
            fAis = q.qdp_field_alloc(c, q.QDP_CLOVER, 1, q.QDP_EVEN)
            q.qdp_clover_build(fA, fAi, fU, m, 1.0)
            q.qdp_clover_build(fAs, fAis, fUs, m, 1.0)
        res = q.qdp_cg_solve_mixed(fx, fb, fU, fA, fAi, fUs, fAs, fAis, mass=m, tol=1e-10, delta=0.1, maxit=2000)
        assert res["status"] == q.QDP_OK
        assert res["reliable"] >= 1 and res["hist"][-1] <= 1e-10
        assert res["true_resid"] <= 1e-9
        assert res["iters"] <= 2 * ref["iters"] + 10
        assert rel_site_err(q.qdp_field_export(fx), ref["x"]) <= 1e-8
        # same system in plain fp64: the answers agree with each other too
        fy = q.qdp_field_alloc(c, q.QDP_FERMION, 0, q.QDP_ALL)
        r64 = q.qdp_cg_solve(fy, fb, fU, fA, fAi, mass=m, tol=1e-10, maxit=2000)
        assert r64["iters"] == oracle.cg_solve(U, b, L, m, A=A, tol=1e-10, maxit=2000)["iters"]
        assert rel_site_err(q.qdp_field_export(fx), q.qdp_field_export(fy)) <= 1e-8
    finally:
        q.qdp_finalize(c)


@pytest.mark.parametrize("clover,gk", [(False, 1), (True, 1), (True, 3)])
def test_fp32_cg_solution(q, clover, gk):
    """qdp_cg_solve with all-fp32 fields (the sloppy operator on its own) reaches 1e-5 and
    agrees with the oracle's fp64 solution of the fp32-rounded system to fp32 accuracy."""
    L = (8, 8, 8, 8)
    m = 0.1
    U = fieldgen.random_gauge(L, 1911).astype(np.float32).astype(np.float64)
    b = fieldgen.random_spinor(L, 2911).astype(np.float32).astype(np.float64)
    A = oracle.clover_build(U, L, m, 1.0) if clover else None
    ref = oracle.cg_solve(U, b, L, m, A=A, tol=1e-12, maxit=2000)
    c = q.qdp_init(L)
    try:
        fU = _field(q, c, gk, 1, q.QDP_ALL, U)
        fb = _field(q, c, q.QDP_FERMION, 1, q.QDP_ALL, b)
        fx = q.qdp_field_alloc(c, q.QDP_FERMION, 1, q.QDP_ALL)
        fA = fAi = None
        if clover:
            fA = q.qdp_field_alloc(c, q.QDP_CLOVER, 1, q.QDP_ALL)
            fAi = q.qdp_field_alloc(c, q.QDP_CLOVER, 1, q.QDP_EVEN)
            q.qdp_clover_build(fA, fAi, fU, m, 1.0)
        res = q.qdp_cg_solve(fx, fb, fU, fA, fAi, mass=m, tol=1e-5, maxit=2000)
        assert res["status"] == q.QDP_OK and res["true_resid"] <= 1e-4
        assert rel_site_err(q.qdp_field_export(fx).astype(np.float64), ref["x"]) <= 1e-4
    finally:
        q.qdp_finalize(c)


def test_mixed_cg_argument_checks(q):
    L = (4, 4, 4, 4)
    c = q.qdp_init(L)
    try:
        U = q.qdp_field_alloc(c, q.QDP_GAUGE, 0, q.QDP_ALL)
        x = q.qdp_field_alloc(c, q.QDP_FERMION, 0, q.QDP_ALL)
        b = q.qdp_field_alloc(c, q.QDP_FERMION, 0, q.QDP_ALL)
        for Us, delta, st in ((U, 0.1, q.QDP_EPREC), (q.qdp_field_alloc(c, q.QDP_GAUGE, 1, q.QDP_ALL), 1.5, q.QDP_EINVAL)):
            with pytest.raises(q.QdpError) as e:
                q.qdp_cg_solve_mixed(x, b, U, U_s=Us, delta=delta)
            assert e.value.status == st
    finally:
        q.qdp_finalize(c)


@pytest.mark.parametrize("self_halo,p2p", [(0, 0), (8, 1), (12, 1), (12, 0)])
@pytest.mark.parametrize("clover,gk", [(False, 1), (True, 1), (True, 3)])
def test_mixed16_cg_solution(q, clover, gk, self_halo, p2p):
    """16-bit sloppy level (qdp_cg_solve_mixed16): int16 links / clover / search directions, fp32
    residual, fp64 reliable updates.  The answer is pinned like the fp32 variant's: within the
    tolerance of the oracle's fp64 solution, true residual met, convergence declared on an fp64
    residual; also through the halo path (self-halo dims, peer-to-peer fused or separate kernels)."""
    L = (8, 8, 8, 8)
    m = 0.1
    U = fieldgen.random_gauge(L, 1921)
    b = fieldgen.random_spinor(L, 2921)
    A = oracle.clover_build(U, L, m, 1.0) if clover else None
    ref = oracle.cg_solve(U, b, L, m, A=A, tol=1e-11, maxit=2000)
    c = q.qdp_init(L)
    if self_halo:
        q.qdp_set_option(c, q.QDP_OPT_SELF_HALO, self_halo)
        q.qdp_set_option(c, q.QDP_OPT_P2P, p2p)
    try:
        fU = _field(q, c, gk, 0, q.QDP_ALL, U)
        fb = _field(q, c, q.QDP_FERMION, 0, q.QDP_ALL, b)
        fx = q.qdp_field_alloc(c, q.QDP_FERMION, 0, q.QDP_ALL)
        fA = fAi = None
        if clover:
            fA = q.qdp_field_alloc(c, q.QDP_CLOVER, 0, q.QDP_ALL)
            fAi = q.qdp_field_alloc(c, q.QDP_CLOVER, 0, q.QDP_EVEN)
            q.qdp_clover_build(fA, fAi, fU, m, 1.0)
        for delta in (0.1, 0.01):
            res = q.qdp_cg_solve_mixed16(fx, fb, fU, fA, fAi, mass=m, tol=1e-10, delta=delta, maxit=3000)
            assert res["status"] == q.QDP_OK
            assert res["reliable"] >= 1 and res["hist"][-1] <= 1e-10
            assert res["true_resid"] <= 1e-9
            assert res["iters"] <= 3 * ref["iters"] + 20
            assert rel_site_err(q.qdp_field_export(fx), ref["x"]) <= 1e-8
    finally:
        q.qdp_finalize(c)


def test_h16_dslash_accuracy(q):
    """The 16-bit operator itself: one sloppy Mhat^dag Mhat application inside the solver is not
    exposed, so check through the solver's first residual history entry -- with delta close to 1
    every iteration is a reliable update, i.e. the run is fp64 CG steered by 16-bit directions,
    and it must still converge to the oracle's answer."""
    L = (6, 4, 4, 8)
    m = 0.2
    U = fieldgen.random_gauge(L, 1931)
    b = fieldgen.random_spinor(L, 2931)
    ref = oracle.cg_solve(U, b, L, m, tol=1e-11, maxit=2000)
    c = q.qdp_init(L)
    try:
        fU = _field(q, c, q.QDP_GAUGE, 0, q.QDP_ALL, U)
        fb = _field(q, c, q.QDP_FERMION, 0, q.QDP_ALL, b)
        fx = q.qdp_field_alloc(c, q.QDP_FERMION, 0, q.QDP_ALL)
        res = q.qdp_cg_solve_mixed16(fx, fb, fU, mass=m, tol=1e-10, delta=0.999, maxit=2000)
        assert res["status"] == q.QDP_OK and res["reliable"] >= res["iters"] - 1
        assert rel_site_err(q.qdp_field_export(fx), ref["x"]) <= 1e-8
    finally:
        q.qdp_finalize(c)
