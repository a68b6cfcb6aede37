"""Edge and degenerate cases of the hot path on the GPU: zero sources, zero iterations, an
exactly singular clover term, a convergence tolerance that is already met, the smallest
lattice (2^4, every neighbour pair coincident), and the per-rank sub-lattice of config 5
(48^3 x 96 over 8 GPUs as z2 x t4 -> 48 x 48 x 24 x 24 per GPU) run through the halo code
path (self-halo in z and t) against the oracle."""
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


def test_zero_source_and_zero_iterations(q):
    L = (4, 4, 4, 4)
    U = fieldgen.random_gauge(L, 31)
    c = q.qdp_init(L)
    try:
        fU = _field(q, c, q.QDP_GAUGE, 0, q.QDP_ALL, U)
        fb = q.qdp_field_alloc(c, q.QDP_FERMION, 0, q.QDP_ALL)          # b = 0
        fx = _field(q, c, q.QDP_FERMION, 0, q.QDP_ALL, fieldgen.random_spinor(L, 32))
        res = q.qdp_cg_solve(fx, fb, fU, mass=0.1, tol=1e-10, maxit=100)
        assert res["status"] == q.QDP_OK and res["iters"] == 0
        assert not q.qdp_field_export(fx).any()                       # x = 0 exactly
        assert q.qdp_norm2(fx) == 0.0
        b = fieldgen.random_spinor(L, 33)
        q.qdp_field_import(fb, b)
        res = q.qdp_cg_solve(fx, fb, fU, mass=0.1, tol=1e-10, maxit=0)
        ref = oracle.cg_solve(U, b, L, 0.1, tol=1e-10, maxit=0)
        assert res["status"] == q.QDP_NOT_CONVERGED and res["iters"] == 0 == ref["iters"]
        assert rel_site_err(q.qdp_field_export(fx), ref["x"]) <= 1e-13  # x_o = 0, x_e = A^-1 b_e
        res = q.qdp_cg_solve(fx, fb, fU, mass=0.1, tol=2.0, maxit=100)   # tolerance already met
        assert res["status"] == q.QDP_OK and res["iters"] == 1
    finally:
        q.qdp_finalize(c)


def test_singular_clover(q):
    """m = -4, c_SW = 0 makes A = 0 on every site: the build must report QDP_ESINGULAR."""
    L = (4, 4, 4, 4)
    c = q.qdp_init(L)
    try:
        fU = _field(q, c, q.QDP_GAUGE, 0, q.QDP_ALL, fieldgen.random_gauge(L, 34))
        fA = q.qdp_field_alloc(c, q.QDP_CLOVER, 0, q.QDP_ALL)
        fAi = q.qdp_field_alloc(c, q.QDP_CLOVER, 0, q.QDP_EVEN)
        with pytest.raises(q.QdpError) as e:
            q.qdp_clover_build(fA, fAi, fU, -4.0, 0.0)
        assert e.value.status == q.QDP_ESINGULAR
        q.qdp_clover_build(fA, None, fU, -4.0, 0.0)  # A alone is fine (and zero)
        assert not q.qdp_field_export(fA).any()
    finally:
        q.qdp_finalize(c)


@pytest.mark.parametrize("mask", [0, 15])
def test_smallest_lattice_everything(q, mask):
    """2^4: x+mu = x-mu for every mu, so every hop pair lands on one neighbour."""
    L = (2, 2, 2, 2)
    U = fieldgen.random_gauge(L, 35)
    b = fieldgen.random_spinor(L, 36)
    A = oracle.clover_build(U, L, 0.2, 1.0)
    ref = oracle.cg_solve(U, b, L, 0.2, A=A, tol=1e-12, maxit=200)
    c = q.qdp_init(L)
    q.qdp_set_option(c, q.QDP_OPT_SELF_HALO, mask)
    try:
        fU = _field(q, c, q.QDP_GAUGE, 0, q.QDP_ALL, U)
        fb = _field(q, c, q.QDP_FERMION, 0, q.QDP_ALL, b)
        fo = q.qdp_field_alloc(c, q.QDP_FERMION, 0, q.QDP_ALL)
        q.qdp_dslash(fo, fU, fb, q.QDP_ALL)
        assert rel_site_err(q.qdp_field_export(fo), oracle.hopping(U, b, L)) <= 1e-13
        fA = q.qdp_field_alloc(c, q.QDP_CLOVER, 0, q.QDP_ALL)
        fAi = q.qdp_field_alloc(c, q.QDP_CLOVER, 0, q.QDP_EVEN)
        q.qdp_clover_build(fA, fAi, fU, 0.2, 1.0)
        assert np.max(np.abs(q.qdp_field_export(fA) - A)) <= 1e-13 * np.max(np.abs(A))
        res = q.qdp_cg_solve(fo, fb, fU, fA, fAi, mass=0.2, tol=1e-12, maxit=200)
        assert res["iters"] == ref["iters"]
        assert np.max(np.abs(res["hist"] - ref["hist"]) / ref["hist"]) <= 1e-10
    finally:
        q.qdp_finalize(c)


def test_config5_rank_sublattice_through_halo_path(q):
    """Config 5 split z2 x t4: one rank's 48 x 48 x 24 x 24 sub-lattice with the z and t
    neighbours reached through the halo path (self-halo), Wilson CG history vs the oracle."""
    L = (48, 48, 24, 24)
    U = fieldgen.random_gauge(L, 1005)
    b = fieldgen.random_spinor(L, 2006)
    ref = oracle.cg_solve(U, b, L, 0.1, tol=0.0, maxit=3)
    c = q.qdp_init(L)
    q.qdp_set_option(c, q.QDP_OPT_SELF_HALO, 12)
    try:
        fU = _field(q, c, q.QDP_GAUGE, 0, q.QDP_ALL, U)
        fb = _field(q, c, q.QDP_FERMION, 0, q.QDP_ALL, b)
        fx = q.qdp_field_alloc(c, q.QDP_FERMION, 0, q.QDP_ALL)
        res = q.qdp_cg_solve(fx, fb, fU, mass=0.1, tol=0.0, maxit=3)
        assert res["iters"] == 3
        assert np.max(np.abs(res["hist"] - ref["hist"]) / ref["hist"]) <= 1e-10
        assert rel_site_err(q.qdp_field_export(fx), ref["x"]) <= 1e-11
        n_ext, _ = q.qdp_profile_query(c, q.QDP_PK_DSLASH_EXT)
        assert n_ext > 0
    finally:
        q.qdp_finalize(c)


@pytest.mark.parametrize("prec", [0, 1])
def test_device_buffer_import_export(q, prec):
    """qdp_field_import_device / export_device: the host canonical layout in a CUDA tensor,
    converted on the context stream; bit-exact against the host-buffer path."""
    import torch
    L = (4, 6, 4, 4)
    psi = fieldgen.random_spinor(L, 41)
    U = fieldgen.random_gauge(L, 42)
    dt = torch.float64 if prec == 0 else torch.float32
    c = q.qdp_init(L)
    try:
        f = q.qdp_field_alloc(c, q.QDP_FERMION, prec, q.QDP_ALL)
        g = q.qdp_field_alloc(c, q.QDP_GAUGE, prec, q.QDP_ALL)
        q.qdp_field_import_device(f, torch.tensor(psi, dtype=dt, device="cuda"))
        q.qdp_field_import_device(g, torch.tensor(U, dtype=dt, device="cuda"))
        hp = psi.astype(np.float64 if prec == 0 else np.float32)
        assert np.array_equal(q.qdp_field_export(f), hp)
        out = torch.empty(psi.shape, dtype=dt, device="cuda")
        q.qdp_field_export_device(f, out)
        q.qdp_synchronize(c)
        assert np.array_equal(out.cpu().numpy(), hp)
        with pytest.raises(q.QdpError) as e:
            q.qdp_field_import_device(f, torch.zeros(7, dtype=dt, device="cuda"))
        assert e.value.status == q.QDP_ESHAPE
    finally:
        q.qdp_finalize(c)


def test_dslash_production_lattice(q):
    """The paper's production lattice 40^3 x 256 (16.4M sites, 9.4 GB of links) on
    one GPU: every output site of one EO dslash (fp64) against the oracle -- 64-bit offsets and
    large-grid indexing at the largest size in BASELINE.json."""
    L = (40, 40, 40, 256)
    U = fieldgen.random_gauge(L, 1004)
    psi = fieldgen.random_spinor(L, 2005)
    ref = oracle.hopping(U, psi, L, 1)
    odd = fieldgen.cb_sites(L, 1)
    c = q.qdp_init(L)
    try:
        fU = _field(q, c, q.QDP_GAUGE, 0, q.QDP_ALL, U)
        del U
        fp = _field(q, c, q.QDP_FERMION, 0, 0, np.ascontiguousarray(psi[fieldgen.cb_sites(L, 0)]))
        fo = q.qdp_field_alloc(c, q.QDP_FERMION, 0, 1)
        q.qdp_dslash(fo, fU, fp, 1)
        assert rel_site_err(q.qdp_field_export(fo), ref[odd]) <= 1e-13
    finally:
        q.qdp_finalize(c)


def test_init_limits(q):
    with pytest.raises(q.QdpError) as e:
        q.qdp_init((2048, 2048, 2048, 2))      # V/2 > 2^30 sites per parity
    assert e.value.status == q.QDP_ESHAPE
    with pytest.raises(q.QdpError) as e:
        q.qdp_init((4, 4, 4, 4), (1, 1, 1, 2), 0, 2, None)  # nranks > 1 needs an NCCL id
    assert e.value.status == q.QDP_EINVAL
