"""Peer-to-peer halo protocol (QDP_OPT_P2P) on one GPU: with self-halo dims the pack kernel
stores into this rank's double-buffered ghost slots and release-signals the ready flags, the
exterior kernels acquire them and acknowledge; results must equal the oracle over many calls
(both slots, both precisions, with the fused inner product of the CG)."""
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


def _ctx(q, L, mask):
    c = q.qdp_init(L)
    q.qdp_set_option(c, q.QDP_OPT_SELF_HALO, mask)
    q.qdp_set_option(c, q.QDP_OPT_P2P, 1)
    return c


@pytest.mark.timeout(120)
@pytest.mark.parametrize("overlap", [1, 0])
@pytest.mark.parametrize("prec", [0, 1])
@pytest.mark.parametrize("mask", [8, 4, 12, 15])
def test_dslash_p2p_self(q, prec, mask, overlap):
    L = (4, 6, 4, 8)
    U = fieldgen.random_gauge(L, 2101)
    psi = fieldgen.random_spinor(L, 3101)
    if prec:
        U, psi = U.astype(np.float32).astype(np.float64), psi.astype(np.float32).astype(np.float64)
    ref = oracle.hopping(U, psi, L, -1)
    c = _ctx(q, L, mask)
    q.qdp_set_option(c, q.QDP_OPT_OVERLAP, overlap)  # 0: every block waits for the ghosts
    try:
        fU = _field(q, c, q.QDP_GAUGE, prec, q.QDP_ALL, U)
        fp = _field(q, c, q.QDP_FERMION, prec, q.QDP_ALL, psi)
        fo = q.qdp_field_alloc(c, q.QDP_FERMION, prec, q.QDP_ALL)
        for _ in range(5):  # 10 EO calls: both slots several times, acks gate the reuse
            q.qdp_dslash(fo, fU, fp, q.QDP_ALL)
            q.qdp_synchronize(c)  # also raises if a flag wait had timed out
            got = q.qdp_field_export(fo).astype(np.float64)
            assert rel_site_err(got, ref) <= (1e-13 if prec == 0 else 2e-6)
        n_pack, _ = q.qdp_profile_query(c, q.QDP_PK_PACK)
        n_ext, _ = q.qdp_profile_query(c, q.QDP_PK_DSLASH_EXT)
        n_main, _ = q.qdp_profile_query(c, q.QDP_PK_DSLASH)
        # every split: packing, interior and the remote hops in ONE kernel per EO dslash
        assert (n_pack, n_ext, n_main) == (0, 0, 10)
    finally:
        q.qdp_finalize(c)


@pytest.mark.timeout(120)
@pytest.mark.parametrize("mask", [8, 12])
def test_dslash_p2p_separate_kernels(q, mask):
    """QDP_OPT_FUSE = 0: separate pack / interior / exterior kernels, same result."""
    L = (4, 6, 4, 8)
    U = fieldgen.random_gauge(L, 2101)
    psi = fieldgen.random_spinor(L, 3101)
    ref = oracle.hopping(U, psi, L, -1)
    c = _ctx(q, L, mask)
    q.qdp_set_option(c, q.QDP_OPT_FUSE, 0)
    try:
        fU = _field(q, c, q.QDP_GAUGE, 0, q.QDP_ALL, U)
        fp = _field(q, c, q.QDP_FERMION, 0, q.QDP_ALL, psi)
        fo = q.qdp_field_alloc(c, q.QDP_FERMION, 0, q.QDP_ALL)
        for _ in range(3):
            q.qdp_dslash(fo, fU, fp, q.QDP_ALL)
            q.qdp_synchronize(c)
            assert rel_site_err(q.qdp_field_export(fo), ref) <= 1e-13
        n_pack, _ = q.qdp_profile_query(c, q.QDP_PK_PACK)
        assert n_pack == 6 * bin(mask).count("1")
        for fuse in (1, 0, 1, 1, 0, 0, 1):  # switching modes mid-sequence keeps the protocol (both queue sets)
            q.qdp_set_option(c, q.QDP_OPT_FUSE, fuse)
            q.qdp_dslash(fo, fU, fp, q.QDP_ALL)
            q.qdp_synchronize(c)
            assert rel_site_err(q.qdp_field_export(fo), ref) <= 1e-13
    finally:
        q.qdp_finalize(c)


@pytest.mark.timeout(120)
def test_p2p_partition_change(q):
    """Changing the self-halo mask after the first peer-to-peer dslash (4 -> 8 -> 12) rebuilds the
    ghost slots of a one-rank context (stale slot pointers for the new dim)."""
    L = (4, 6, 4, 8)
    U = fieldgen.random_gauge(L, 2103)
    psi = fieldgen.random_spinor(L, 3103)
    ref = oracle.hopping(U, psi, L, -1)
    c = _ctx(q, L, 4)
    try:
        fU = _field(q, c, q.QDP_GAUGE, 0, q.QDP_ALL, U)
        fp = _field(q, c, q.QDP_FERMION, 0, q.QDP_ALL, psi)
        fo = q.qdp_field_alloc(c, q.QDP_FERMION, 0, q.QDP_ALL)
        for mask in (4, 8, 12, 8):
            q.qdp_set_option(c, q.QDP_OPT_SELF_HALO, mask)
            for _ in range(3):
                q.qdp_dslash(fo, fU, fp, q.QDP_ALL)
                q.qdp_synchronize(c)
                assert rel_site_err(q.qdp_field_export(fo), ref) <= 1e-13, mask
    finally:
        q.qdp_finalize(c)


@pytest.mark.timeout(120)
def test_cg_clover_p2p_self(q):
    L = (4, 4, 6, 4)
    U = fieldgen.random_gauge(L, 2102)
    b = fieldgen.random_spinor(L, 3102)
    A = oracle.clover_build(U, L, 0.1, 1.0)
    ref = oracle.cg_solve(U, b, L, 0.1, A=A, tol=1e-10, maxit=500)
    c = _ctx(q, L, 12)
    try:
        fU = _field(q, c, q.QDP_GAUGE, 0, q.QDP_ALL, U)
        fb = _field(q, c, q.QDP_FERMION, 0, q.QDP_ALL, b)
        fx = q.qdp_field_alloc(c, q.QDP_FERMION, 0, q.QDP_ALL)
        fA = q.qdp_field_alloc(c, q.QDP_CLOVER, 0, q.QDP_ALL)
        fAi = q.qdp_field_alloc(c, q.QDP_CLOVER, 0, q.QDP_EVEN)
        q.qdp_clover_build(fA, fAi, fU, 0.1, 1.0)
        res = q.qdp_cg_solve(fx, fb, fU, fA, fAi, mass=0.1, tol=1e-10, maxit=500)
        assert res["iters"] == ref["iters"]
        assert np.max(np.abs(res["hist"] - ref["hist"]) / ref["hist"]) <= 1e-10
        assert rel_site_err(q.qdp_field_export(fx), ref["x"]) <= 1e-9
    finally:
        q.qdp_finalize(c)


@pytest.mark.timeout(300)
@pytest.mark.parametrize("overlap", [1, 0])
@pytest.mark.parametrize("mask", [8, 12, 15])
def test_fused_boundary_stress(q, mask, overlap):
    """Many fused peer-to-peer calls in a row (both slots, both parities, the acknowledgement of each
    call's ghosts written by the next call, PDL on the reductions in between): every output must be
    bit-identical to the first, which equals the oracle.  A stale ghost (a slot overwritten before
    it was consumed, or read before it was written) changes the face sites' bits."""
    L = (6, 4, 8, 8)
    U = fieldgen.random_gauge(L, 2111)
    psi = fieldgen.random_spinor(L, 3111)
    ref = oracle.hopping(U, psi, L, -1)
    c = _ctx(q, L, mask)
    q.qdp_set_option(c, q.QDP_OPT_OVERLAP, overlap)
    try:
        fU = _field(q, c, q.QDP_GAUGE, 0, q.QDP_ALL, U)
        fp = _field(q, c, q.QDP_FERMION, 0, q.QDP_ALL, psi)
        fo = q.qdp_field_alloc(c, q.QDP_FERMION, 0, q.QDP_ALL)
        q.qdp_dslash(fo, fU, fp, q.QDP_ALL)
        first = q.qdp_field_export(fo)
        assert rel_site_err(first, ref) <= 1e-13
        n0 = q.qdp_norm2(fo)
        for i in range(40):
            q.qdp_field_zero(fo)
            q.qdp_dslash(fo, fU, fp, q.QDP_ALL)
            n = q.qdp_norm2(fo)  # a one-launch reduction between the dslash calls
            assert n == n0, i
            if i % 8 == 7:
                assert np.array_equal(q.qdp_field_export(fo), first), i
        q.qdp_synchronize(c)
    finally:
        q.qdp_finalize(c)
