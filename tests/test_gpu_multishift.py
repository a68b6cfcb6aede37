"""GPU multi-shift CG (qdp_cg_solve_multishift; reading R25, ref. [14])
against the oracle's orc_cg_multishift on the same seeded fields: same iteration count, same
per-shift stopping iterations, base residual history within 1e-10, every shifted solution
within 1e-9 per site, and the true residuals of every shift."""
import numpy as np
import pytest

import fieldgen
import oracle
from _physics import rel_site_err

pytestmark = pytest.mark.gpu

SIGMA = [0.0, 0.004, 0.03, 0.2, 1.1, 6.0]  # RHMC-like spread of shifts


@pytest.fixture(scope="module")
def q():
    from paper_1408_5925_b200 import qdpb
    qdpb.lib()
    return qdpb


def _odd(a, L):
    """odd sites of a full-lattice host field"""
    return a[fieldgen.parity(L) == 1]


def _run(q, L, clover, prec=0, self_halo=0, subset=-1, sigma=SIGMA, tol=1e-10, maxit=1000, seeds=(1901, 2901)):
    m = 0.1
    U = fieldgen.random_gauge(L, seeds[0])
    phi = fieldgen.random_spinor(L, seeds[1])
    if prec:
        U, phi = (fieldgen.to_fp32(a).astype(np.float64) for a in (U, phi))
    dt = np.float64 if prec == 0 else np.float32
    c = q.qdp_init(L)
    try:
        if self_halo:
            q.qdp_set_option(c, q.QDP_OPT_SELF_HALO, self_halo)
        fU = q.qdp_field_alloc(c, q.QDP_GAUGE, prec, q.QDP_ALL)
        q.qdp_field_import(fU, U.astype(dt))
        fphi = q.qdp_field_alloc(c, q.QDP_FERMION, prec, subset)
        q.qdp_field_import(fphi, np.ascontiguousarray((phi if subset == -1 else _odd(phi, L)).astype(dt)))
        xs = [q.qdp_field_alloc(c, q.QDP_FERMION, prec, subset) for _ in sigma]
        for x in xs:
            q.qdp_field_zero(x)
        fA = fAi = None
        if clover:
            fA = q.qdp_field_alloc(c, q.QDP_CLOVER, prec, q.QDP_ALL)
            fAi = q.qdp_field_alloc(c, q.QDP_CLOVER, prec, q.QDP_EVEN)
            q.qdp_clover_build(fA, fAi, fU, m, 1.0)
        res = q.qdp_cg_solve_multishift(xs, sigma, fphi, fU, fA, fAi, mass=m, tol=tol, maxit=maxit)
        got = [q.qdp_field_export(x).astype(np.float64) for x in xs]
    finally:
        q.qdp_finalize(c)
    A = oracle.clover_build(U, L, m, 1.0) if clover else None
    ref = oracle.cg_multishift(U, phi, L, m, sigma, A=A, tol=tol, maxit=maxit)
    return res, got, ref


@pytest.mark.parametrize("clover", [False, True])
@pytest.mark.parametrize("L", [(4, 4, 4, 4), (8, 6, 4, 10)])
def test_multishift_parity_fp64(q, L, clover):
    res, got, ref = _run(q, L, clover)
    assert res["status"] == q.QDP_OK and ref["status"] == 0
    assert res["iters"] == ref["iters"]
    assert np.array_equal(res["conv_iter"], ref["conv_iter"])
    assert np.max(np.abs(res["hist"] - ref["hist"]) / ref["hist"]) <= 1e-10
    for i in range(len(SIGMA)):
        assert rel_site_err(_odd(got[i], L), _odd(ref["x"][i], L)) <= 1e-9, i
        assert np.max(np.abs(got[i][fieldgen.parity(L) == 0])) == 0.0  # the even block is not written
    assert np.all(res["true_resid"] <= 3e-10)
    assert np.allclose(res["true_resid"], ref["true_resid"], rtol=0, atol=1e-11)


def test_multishift_odd_subset_fields_and_halo_path(q):
    """QDP_ODD solution / source fields, and the whole solve through the halo code path."""
    L = (4, 4, 4, 8)
    res, got, ref = _run(q, L, True, self_halo=12, subset=q.QDP_ODD)
    assert res["iters"] == ref["iters"] and np.array_equal(res["conv_iter"], ref["conv_iter"])
    assert np.max(np.abs(res["hist"] - ref["hist"]) / ref["hist"]) <= 1e-10
    for i in range(len(SIGMA)):
        assert rel_site_err(got[i], _odd(ref["x"][i], L)) <= 1e-9


def test_multishift_fp32(q):
    L = (8, 8, 8, 8)
    res, got, ref = _run(q, L, True, prec=1, tol=1e-5)
    assert abs(res["iters"] - ref["iters"]) <= 2
    assert np.all(res["true_resid"] <= 5e-5)
    for i in range(len(SIGMA)):
        assert rel_site_err(_odd(got[i], L), _odd(ref["x"][i], L)) <= 2e-4


def test_multishift_single_shift_is_cg_and_maxit(q):
    L = (4, 4, 4, 4)
    res, got, ref = _run(q, L, False, sigma=[0.05])
    assert res["iters"] == ref["iters"]
    cap, _, refcap = _run(q, L, False, maxit=4)
    assert cap["status"] == q.QDP_NOT_CONVERGED and cap["iters"] == 4
    assert np.array_equal(cap["conv_iter"], refcap["conv_iter"])
    assert np.max(np.abs(cap["hist"] - refcap["hist"]) / refcap["hist"]) <= 1e-12


def test_multishift_argument_errors(q):
    L = (4, 4, 4, 4)
    c = q.qdp_init(L)
    try:
        fU = q.qdp_field_alloc(c, q.QDP_GAUGE, 0, q.QDP_ALL)
        fphi = q.qdp_field_alloc(c, q.QDP_FERMION, 0, q.QDP_ALL)
        x0, x1 = (q.qdp_field_alloc(c, q.QDP_FERMION, 0, q.QDP_ALL) for _ in range(2))
        xe = q.qdp_field_alloc(c, q.QDP_FERMION, 0, q.QDP_EVEN)
        for xs, sg, st in [([x0, x1], [0.5, 0.1], q.QDP_EINVAL),     # sigma_0 not the smallest
                           ([x0, x0], [0.0, 0.1], q.QDP_EALIAS),     # two shifts share a solution
                           ([x0, xe], [0.0, 0.1], q.QDP_EINVAL),     # even-only solution field
                           ([fphi, x1], [0.0, 0.1], q.QDP_EALIAS)]:  # solution aliases the source
            with pytest.raises(q.QdpError) as e:
                q.qdp_cg_solve_multishift(xs, sg, fphi, fU)
            assert e.value.status == st
    finally:
        q.qdp_finalize(c)


def test_multishift_zero_source_and_positive_base(q):
    """phi = 0: converged at iteration 0 with x_i = 0; a positive base shift (sigma_0 > 0)."""
    L = (4, 4, 4, 4)
    c = q.qdp_init(L)
    try:
        fU = q.qdp_field_alloc(c, q.QDP_GAUGE, 0, q.QDP_ALL)
        q.qdp_field_import(fU, fieldgen.random_gauge(L, 1902))
        fphi = q.qdp_field_alloc(c, q.QDP_FERMION, 0, q.QDP_ODD)
        q.qdp_field_zero(fphi)
        xs = [q.qdp_field_alloc(c, q.QDP_FERMION, 0, q.QDP_ODD) for _ in range(2)]
        res = q.qdp_cg_solve_multishift(xs, [0.0, 1.0], fphi, fU)
        assert res["status"] == q.QDP_OK and res["iters"] == 0
        assert all(np.max(np.abs(q.qdp_field_export(x))) == 0.0 for x in xs)
    finally:
        q.qdp_finalize(c)
    res, got, ref = _run(q, L, True, sigma=[0.3, 0.7, 5.0])
    assert res["iters"] == ref["iters"] and np.array_equal(res["conv_iter"], ref["conv_iter"])
    for i in range(3):
        assert rel_site_err(_odd(got[i], L), _odd(ref["x"][i], L)) <= 1e-9
