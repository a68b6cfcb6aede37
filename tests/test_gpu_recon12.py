"""QDP_GAUGE12: links stored as their first two rows, the third rebuilt as conj(row0 x row1)
("reconstruction of SU(3) matrices from ... 12 real numbers").
The oracle always uses the full 3x3 links; for SU(3) inputs the rebuilt row equals the stored
one to rounding, so the fp64 / fp32 tolerances are unchanged."""
import numpy as np
import pytest

import fieldgen
import oracle
from _physics import rel_site_err

pytestmark = pytest.mark.gpu
TOL = {0: 1e-13, 1: 2e-6}


@pytest.fixture(scope="module")
def q():
    from paper_1408_5925_b200 import qdpb
    qdpb.lib()
    return qdpb


def _host(a, prec):
    return np.ascontiguousarray(a, dtype=np.float64 if prec == 0 else np.float32)


def _field(q, c, kind, prec, subset, host):
    f = q.qdp_field_alloc(c, kind, prec, subset)
    q.qdp_field_import(f, _host(host, prec))
    return f


def _round(a, prec):
    return a if prec == 0 else a.astype(np.float32).astype(np.float64)


@pytest.mark.parametrize("prec", [0, 1])
def test_gauge12_round_trip_and_validation(q, prec):
    L = (4, 4, 6, 4)
    U = _round(fieldgen.random_gauge(L, 1801), prec)
    c = q.qdp_init(L)
    try:
        hb, db = q.qdp_field_bytes(c, q.QDP_GAUGE12, prec, q.QDP_ALL)
        _, db18 = q.qdp_field_bytes(c, q.QDP_GAUGE, prec, q.QDP_ALL)
        assert 3 * db == 2 * db18
        f = _field(q, c, q.QDP_GAUGE12, prec, q.QDP_ALL, U)
        got = q.qdp_field_export(f).astype(np.float64)
        assert np.array_equal(got[:, :, :2], U[:, :, :2])               # stored rows: bit-exact
        assert np.max(np.abs(got[:, :, 2] - U[:, :, 2])) <= (1e-15 if prec == 0 else 1e-6)
        bad = U.copy()
        bad[7, 3] *= -1.0                                                # det = -1: not SU(3)
        with pytest.raises(q.QdpError) as e:
            q.qdp_field_import(f, _host(bad, prec))
        assert e.value.status == q.QDP_EINVAL
    finally:
        q.qdp_finalize(c)


@pytest.mark.parametrize("prec", [0, 1])
@pytest.mark.parametrize("mask", [0, 12])
def test_dslash_gauge12(q, prec, mask):
    L = (6, 4, 4, 8)
    U = _round(fieldgen.random_gauge(L, 1802), prec)
    psi = _round(fieldgen.random_spinor(L, 2802), prec)
    ref = oracle.hopping(U, psi, L, -1)
    c = q.qdp_init(L)
    q.qdp_set_option(c, q.QDP_OPT_SELF_HALO, mask)
    try:
        fU = _field(q, c, q.QDP_GAUGE12, prec, q.QDP_ALL, U)
        fp = _field(q, c, q.QDP_FERMION, prec, q.QDP_ALL, psi)
        fo = q.qdp_field_alloc(c, q.QDP_FERMION, prec, q.QDP_ALL)
        q.qdp_dslash(fo, fU, fp, q.QDP_ALL)
        assert rel_site_err(q.qdp_field_export(fo).astype(np.float64), ref) <= TOL[prec]
    finally:
        q.qdp_finalize(c)


@pytest.mark.parametrize("mask", [0, 15])
def test_shift_and_clover_gauge12(q, mask):
    L = (4, 4, 4, 6)
    U = fieldgen.random_gauge(L, 1803)
    c = q.qdp_init(L)
    q.qdp_set_option(c, q.QDP_OPT_SELF_HALO, mask)
    try:
        fU = _field(q, c, q.QDP_GAUGE12, 0, q.QDP_ALL, U)
        fo = q.qdp_field_alloc(c, q.QDP_GAUGE12, 0, q.QDP_ALL)
        for mu in range(4):
            q.qdp_shift(fo, fU, mu, -1)
            got = q.qdp_field_export(fo)
            ref = oracle.shift(U.reshape(len(U), -1), L, mu, -1).reshape(U.shape)
            assert np.array_equal(got[:, :, :2], ref[:, :, :2])
            assert np.max(np.abs(got - ref)) <= 1e-15
        A = oracle.clover_build(U, L, 0.1, 1.0)
        fA = q.qdp_field_alloc(c, q.QDP_CLOVER, 0, q.QDP_ALL)
        q.qdp_clover_build(fA, None, fU, 0.1, 1.0)
        assert np.max(np.abs(q.qdp_field_export(fA) - A)) <= 1e-13 * np.max(np.abs(A))
    finally:
        q.qdp_finalize(c)


def test_cg_gauge12_history(q):
    L = (8, 8, 8, 8)
    U = fieldgen.random_gauge(L, 1804)
    b = fieldgen.random_spinor(L, 2804)
    A = oracle.clover_build(U, L, 0.1, 1.0)
    ref = oracle.cg_solve(U, b, L, 0.1, A=A, tol=1e-10, maxit=1000)
    c = q.qdp_init(L)
    try:
        fU = _field(q, c, q.QDP_GAUGE12, 0, q.QDP_ALL, U)
        fb = _field(q, c, q.QDP_FERMION, 0, q.QDP_ALL, b)
        fx = q.qdp_field_alloc(c, q.QDP_FERMION, 0, q.QDP_ALL)
        fA = q.qdp_field_alloc(c, q.QDP_CLOVER, 0, q.QDP_ALL)
        fAi = q.qdp_field_alloc(c, q.QDP_CLOVER, 0, q.QDP_EVEN)
        q.qdp_clover_build(fA, fAi, fU, 0.1, 1.0)
        res = q.qdp_cg_solve(fx, fb, fU, fA, fAi, mass=0.1, tol=1e-10, maxit=1000)
        assert res["iters"] == ref["iters"]
        assert np.max(np.abs(res["hist"] - ref["hist"]) / ref["hist"]) <= 1e-10
        assert rel_site_err(q.qdp_field_export(fx), ref["x"]) <= 1e-9
    finally:
        q.qdp_finalize(c)
