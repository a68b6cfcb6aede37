"""The NCCL halo path on one GPU: self-halo dims routed through a one-rank NCCL communicator
(QDP_OPT_SELF_NCCL), i.e. pack -> ncclSend/ncclRecv (comm stream, overlapped or not) ->
interior + exterior, with the same same-peer message order a P_mu = 2 run uses."""
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


def _ctx(q, L, mask, overlap=1):
    c = q.qdp_init(L)
    q.qdp_set_option(c, q.QDP_OPT_SELF_HALO, mask)
    q.qdp_set_option(c, q.QDP_OPT_SELF_NCCL, 1)
    q.qdp_set_option(c, q.QDP_OPT_OVERLAP, overlap)
    return c


def _field(q, c, kind, prec, subset, host):
    f = q.qdp_field_alloc(c, kind, prec, subset)
    q.qdp_field_import(f, np.ascontiguousarray(host, dtype=np.float64 if prec == 0 else np.float32))
    return f


@pytest.mark.parametrize("prec", [0, 1])
@pytest.mark.parametrize("mask,overlap", [(8, 1), (8, 0), (12, 1), (15, 1)])
def test_dslash_nccl_self(q, mask, overlap, prec):
    L = (4, 6, 4, 8)
    U = fieldgen.random_gauge(L, 1701)
    psi = fieldgen.random_spinor(L, 2701)
    if prec:
        U, psi = U.astype(np.float32).astype(np.float64), psi.astype(np.float32).astype(np.float64)
    ref = oracle.hopping(U, psi, L, -1)
    c = _ctx(q, L, mask, overlap)
    try:
        fU = _field(q, c, q.QDP_GAUGE, prec, q.QDP_ALL, U)
        fp = _field(q, c, q.QDP_FERMION, prec, q.QDP_ALL, psi)
        fo = q.qdp_field_alloc(c, q.QDP_FERMION, prec, q.QDP_ALL)
        for _ in range(3):  # repeated exchanges reuse the same buffers and streams
            q.qdp_dslash(fo, fU, fp, q.QDP_ALL)
        got = q.qdp_field_export(fo).astype(np.float64)
        assert rel_site_err(got, ref) <= (1e-13 if prec == 0 else 2e-6)
    finally:
        q.qdp_finalize(c)


def test_shift_nccl_self(q):
    L = (4, 4, 2, 6)
    psi = fieldgen.random_spinor(L, 2702)
    U = fieldgen.random_gauge(L, 1702)
    c = _ctx(q, L, 15)
    try:
        fp = _field(q, c, q.QDP_FERMION, 0, q.QDP_ALL, psi)
        fo = q.qdp_field_alloc(c, q.QDP_FERMION, 0, q.QDP_ALL)
        fU = _field(q, c, q.QDP_GAUGE, 0, q.QDP_ALL, U)
        fUo = q.qdp_field_alloc(c, q.QDP_GAUGE, 0, q.QDP_ALL)
        for mu in range(4):
            for sign in (1, -1):
                q.qdp_shift(fo, fp, mu, sign)
                assert np.array_equal(q.qdp_field_export(fo),
                                      oracle.shift(psi.reshape(len(psi), -1), L, mu, sign).reshape(psi.shape))
                q.qdp_shift(fUo, fU, mu, sign)
                assert np.array_equal(q.qdp_field_export(fUo),
                                      oracle.shift(U.reshape(len(U), -1), L, mu, sign).reshape(U.shape))
    finally:
        q.qdp_finalize(c)


def test_cg_clover_nccl_self(q):
    L = (4, 4, 4, 8)
    U = fieldgen.random_gauge(L, 1703)
    b = fieldgen.random_spinor(L, 2703)
    A = oracle.clover_build(U, L, 0.1, 1.0)
    ref = oracle.cg_solve(U, b, L, 0.1, A=A, tol=1e-10, maxit=1000)
    c = _ctx(q, L, 12)
    try:
        fU = _field(q, c, q.QDP_GAUGE, 0, q.QDP_ALL, U)
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
