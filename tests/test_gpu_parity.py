"""GPU parity: the CUDA path (through the C ABI) against the oracle on the same seeded
inputs.  Tolerances (north star): per-site relative L2 error
<= 1e-13 (fp64) / 2e-6 (fp32, oracle run in double on the fp32-rounded inputs); integer /
index work (shift, layout round trip) bit-exact; CG residual history within 1e-10 with
the same iteration count."""
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


def _ctx(q, L, self_halo=0, overlap=1):
    c = q.qdp_init(L)
    if self_halo:
        q.qdp_set_option(c, q.QDP_OPT_SELF_HALO, self_halo)
    q.qdp_set_option(c, q.QDP_OPT_OVERLAP, overlap)
    return c


def _round(a, prec):
    return a if prec == 0 else a.astype(np.float32).astype(np.float64)


def _host(a, prec):
    return np.ascontiguousarray(a, dtype=np.float64 if prec == 0 else np.float32)


def _field(q, c, kind, prec, subset, host):
    f = q.qdp_field_alloc(c, kind, prec, subset)
    q.qdp_field_import(f, _host(host, prec))
    return f


LATTICES = [(4, 4, 4, 4), (6, 4, 2, 8), (2, 2, 2, 2), (8, 6, 4, 10), (16, 16, 16, 32)]


@pytest.mark.parametrize("prec", [0, 1])
@pytest.mark.parametrize("L", LATTICES)
def test_dslash_full_lattice(q, L, prec):
    U = _round(fieldgen.random_gauge(L, 1001), prec)
    psi = _round(fieldgen.random_spinor(L, 2001), prec)
    ref = oracle.hopping(U, psi, L, -1)
    c = _ctx(q, L)
    try:
        fU = _field(q, c, q.QDP_GAUGE, prec, q.QDP_ALL, U)
        fp = _field(q, c, q.QDP_FERMION, prec, q.QDP_ALL, psi)
        fo = q.qdp_field_alloc(c, q.QDP_FERMION, prec, q.QDP_ALL)
        q.qdp_dslash(fo, fU, fp, q.QDP_ALL)
        got = q.qdp_field_export(fo).astype(np.float64)
        assert rel_site_err(got, ref) <= TOL[prec]
        # single parity into an ALL field: only that block written
        for p in (0, 1):
            q.qdp_field_zero(fo)
            q.qdp_dslash(fo, fU, fp, p)
            got = q.qdp_field_export(fo).astype(np.float64)
            par = fieldgen.parity(L)
            assert rel_site_err(got[par == p], ref[par == p]) <= TOL[prec]
            assert not got[par != p].any()
    finally:
        q.qdp_finalize(c)


@pytest.mark.parametrize("prec", [0, 1])
def test_dslash_checkerboard_fields(q, prec):
    L = (8, 4, 6, 4)
    U = _round(fieldgen.random_gauge(L, 1101), prec)
    psi = _round(fieldgen.random_spinor(L, 2101), prec)
    c = _ctx(q, L)
    try:
        fU = _field(q, c, q.QDP_GAUGE, prec, q.QDP_ALL, U)
        for p in (0, 1):
            src_sites = fieldgen.cb_sites(L, 1 - p)
            out_sites = fieldgen.cb_sites(L, p)
            fin = _field(q, c, q.QDP_FERMION, prec, 1 - p, psi[src_sites])
            fout = q.qdp_field_alloc(c, q.QDP_FERMION, prec, p)
            q.qdp_dslash(fout, fU, fin, p)
            got = q.qdp_field_export(fout).astype(np.float64)
            ref = oracle.hopping(U, psi, L, p)[out_sites]
            assert rel_site_err(got, ref) <= TOL[prec]
            with pytest.raises(q.QdpError) as e:
                q.qdp_dslash(fout, fU, fin, 1 - p)
            assert e.value.status == q.QDP_EINVAL
    finally:
        q.qdp_finalize(c)


@pytest.mark.parametrize("prec", [0, 1])
@pytest.mark.parametrize("mask,overlap", [(8, 1), (12, 1), (15, 0), (15, 1), (1, 1), (6, 0)])
def test_dslash_self_halo(q, mask, overlap, prec):
    """The multi-GPU code path (pack -> exchange -> interior + exterior) with this rank as
    its own neighbour in every dim of `mask`."""
    L = (4, 6, 4, 8)
    U = _round(fieldgen.random_gauge(L, 1201), prec)
    psi = _round(fieldgen.random_spinor(L, 2201), prec)
    ref = oracle.hopping(U, psi, L, -1)
    c = _ctx(q, L, self_halo=mask, overlap=overlap)
    try:
        fU = _field(q, c, q.QDP_GAUGE, prec, q.QDP_ALL, U)
        fp = _field(q, c, q.QDP_FERMION, prec, q.QDP_ALL, psi)
        fo = q.qdp_field_alloc(c, q.QDP_FERMION, prec, q.QDP_ALL)
        q.qdp_dslash(fo, fU, fp, q.QDP_ALL)
        got = q.qdp_field_export(fo).astype(np.float64)
        assert rel_site_err(got, ref) <= TOL[prec]
        n_pack, _ = q.qdp_profile_query(c, q.QDP_PK_PACK)
        assert n_pack == 2 * bin(mask).count("1")
    finally:
        q.qdp_finalize(c)


@pytest.mark.parametrize("prec", [0, 1])
@pytest.mark.parametrize("self_halo", [0, 15])
def test_shift_bit_exact(q, prec, self_halo):
    L = (4, 6, 2, 8)
    psi = _round(fieldgen.random_spinor(L, 2301), prec)
    U = _round(fieldgen.random_gauge(L, 1301), prec)
    c = _ctx(q, L, self_halo=self_halo)
    try:
        fp = _field(q, c, q.QDP_FERMION, prec, q.QDP_ALL, psi)
        fo = q.qdp_field_alloc(c, q.QDP_FERMION, prec, q.QDP_ALL)
        fU = _field(q, c, q.QDP_GAUGE, prec, q.QDP_ALL, U)
        fUo = q.qdp_field_alloc(c, q.QDP_GAUGE, prec, q.QDP_ALL)
        for mu in range(4):
            for sign in (1, -1):
                q.qdp_shift(fo, fp, mu, sign)
                got = q.qdp_field_export(fo).astype(np.float64)
                assert np.array_equal(got, oracle.shift(psi.reshape(len(psi), -1), L, mu, sign).reshape(psi.shape))
                q.qdp_shift(fUo, fU, mu, sign)
                got = q.qdp_field_export(fUo).astype(np.float64)
                assert np.array_equal(got, oracle.shift(U.reshape(len(U), -1), L, mu, sign).reshape(U.shape))
        # checkerboard: parity p in -> parity 1-p out
        for p in (0, 1):
            fin = _field(q, c, q.QDP_FERMION, prec, p, psi[fieldgen.cb_sites(L, p)])
            fout = q.qdp_field_alloc(c, q.QDP_FERMION, prec, 1 - p)
            full = psi * (fieldgen.parity(L) == p)[:, None, None, None]
            for mu in range(4):
                for sign in (1, -1):
                    q.qdp_shift(fout, fin, mu, sign)
                    got = q.qdp_field_export(fout).astype(np.float64)
                    ref = oracle.shift(full.reshape(len(psi), -1), L, mu, sign).reshape(psi.shape)
                    assert np.array_equal(got, ref[fieldgen.cb_sites(L, 1 - p)])
        with pytest.raises(q.QdpError) as e:
            q.qdp_shift(fp, fp, 0, 1)
        assert e.value.status == q.QDP_EALIAS
    finally:
        q.qdp_finalize(c)


@pytest.mark.parametrize("prec", [0, 1])
def test_layout_round_trip(q, prec):
    L = (6, 4, 4, 2)
    V = fieldgen.volume(L)
    rng = np.random.default_rng(5)
    c = _ctx(q, L)
    try:
        for kind, shape in ((q.QDP_FERMION, (4, 3, 2)), (q.QDP_GAUGE, (4, 3, 3, 2))):
            subsets = [q.QDP_ALL] if kind == q.QDP_GAUGE else [q.QDP_ALL, 0, 1]
            for s in subsets:
                n = V if s == q.QDP_ALL else V // 2
                a = _host(rng.normal(size=(n,) + shape), prec)
                f = _field(q, c, kind, prec, s, a)
                assert np.array_equal(q.qdp_field_export(f), a)
                q.qdp_field_free(f)
        # clover: only the two Hermitian 6x6 blocks survive
        A = oracle.clover_build(fieldgen.random_gauge(L, 7), L, 0.1, 1.0)
        A = _host(_round(A, prec), prec)
        for s in (q.QDP_ALL, 0, 1):
            a = A if s == q.QDP_ALL else np.ascontiguousarray(A[fieldgen.cb_sites(L, s)])
            f = _field(q, c, q.QDP_CLOVER, prec, s, a)
            assert np.array_equal(q.qdp_field_export(f), a)
            q.qdp_field_free(f)
        with pytest.raises(q.QdpError) as e:
            f = q.qdp_field_alloc(c, q.QDP_FERMION, prec, q.QDP_ALL)
            q.qdp_field_import(f, np.zeros(10, dtype=np.float64 if prec == 0 else np.float32))
        assert e.value.status == q.QDP_ESHAPE
    finally:
        q.qdp_finalize(c)


@pytest.mark.parametrize("prec", [0, 1])
def test_blas(q, prec):
    L = (16, 16, 16, 32)
    a = _round(fieldgen.random_spinor(L, 2002), prec)
    b = _round(fieldgen.random_spinor(L, 2003), prec)
    c = _ctx(q, L)
    try:
        fa = _field(q, c, q.QDP_FERMION, prec, q.QDP_ALL, a)
        fb = _field(q, c, q.QDP_FERMION, prec, q.QDP_ALL, b)
        n2 = q.qdp_norm2(fa)
        assert abs(n2 - oracle.norm2(a, L)) <= 1e-13 * n2
        ip = q.qdp_inner_product(fa, fb)
        ref = oracle.inner(a, b, L)
        assert abs(ip - ref) <= 1e-13 * np.sqrt(n2 * oracle.norm2(b, L))
        for p in (0, 1):
            sites = fieldgen.cb_sites(L, p)
            fpa = _field(q, c, q.QDP_FERMION, prec, p, a[sites])
            fpb = _field(q, c, q.QDP_FERMION, prec, p, b[sites])
            assert abs(q.qdp_norm2(fpa) - oracle.norm2(a, L, p)) <= 1e-13 * n2
            assert abs(q.qdp_inner_product(fpa, fpb) - oracle.inner(a, b, L, p)) <= 1e-13 * n2
            q.qdp_axpy(0.25 - 1.5j, fpa, fpb)
            got = q.qdp_field_export(fpb).astype(np.float64)
            refy = oracle.axpy(0.25 - 1.5j, a, b, L, p)[sites]
            assert rel_site_err(got, refy) <= TOL[prec]
        q.qdp_axpy(2.0 + 0.5j, fa, fb)
        got = q.qdp_field_export(fb).astype(np.float64)
        assert rel_site_err(got, oracle.axpy(2.0 + 0.5j, a, b, L)) <= TOL[prec]
    finally:
        q.qdp_finalize(c)


def test_blas_exact_integers(q):
    """Integer-valued fp64 inputs: both sides' sums are exact, so they agree bit for bit."""
    L = (8, 8, 8, 8)
    V = fieldgen.volume(L)
    rng = np.random.default_rng(9)
    a = rng.integers(-500, 500, size=(V, 4, 3, 2)).astype(np.float64)
    b = rng.integers(-500, 500, size=(V, 4, 3, 2)).astype(np.float64)
    c = _ctx(q, L)
    try:
        fa = _field(q, c, q.QDP_FERMION, 0, q.QDP_ALL, a)
        fb = _field(q, c, q.QDP_FERMION, 0, q.QDP_ALL, b)
        assert q.qdp_norm2(fa) == oracle.norm2(a, L)
        assert q.qdp_inner_product(fa, fb) == oracle.inner(a, b, L)
    finally:
        q.qdp_finalize(c)


@pytest.mark.parametrize("prec", [0, 1])
def test_clover_build_apply(q, prec):
    L = (4, 4, 6, 4)
    U = _round(fieldgen.random_gauge(L, 1401), prec)
    psi = _round(fieldgen.random_spinor(L, 2401), prec)
    A = oracle.clover_build(U, L, 0.1, 1.0)
    Ai = oracle.clover_invert(A, L)
    c = _ctx(q, L)
    try:
        fU = _field(q, c, q.QDP_GAUGE, prec, q.QDP_ALL, U)
        fA = q.qdp_field_alloc(c, q.QDP_CLOVER, prec, q.QDP_ALL)
        fAi = q.qdp_field_alloc(c, q.QDP_CLOVER, prec, q.QDP_ALL)
        q.qdp_clover_build(fA, fAi, fU, 0.1, 1.0)
        gA = q.qdp_field_export(fA).astype(np.float64)
        gAi = q.qdp_field_export(fAi).astype(np.float64)
        tolm = 1e-13 if prec == 0 else 2e-6
        assert np.max(np.abs(gA - A)) <= tolm * np.max(np.abs(A))
        assert np.max(np.abs(gAi - Ai)) <= tolm * np.max(np.abs(Ai)) * (1 if prec == 0 else 4)
        fp = _field(q, c, q.QDP_FERMION, prec, q.QDP_ALL, psi)
        fo = q.qdp_field_alloc(c, q.QDP_FERMION, prec, q.QDP_ALL)
        q.qdp_clover_apply(fo, fA, fp, q.QDP_ALL)
        Ar = _round(A, prec)  # the device holds A in the field precision
        got = q.qdp_field_export(fo).astype(np.float64)
        assert rel_site_err(got, oracle.clover_apply(Ar, psi, L)) <= TOL[prec]
    finally:
        q.qdp_finalize(c)


@pytest.mark.parametrize("clover", [False, True])
@pytest.mark.parametrize("L", [(4, 4, 4, 4), (8, 8, 8, 8)])
def test_cg_history_parity(q, L, clover):
    m = 0.1
    U = fieldgen.random_gauge(L, 1003)
    b = fieldgen.random_spinor(L, 2004)
    A = oracle.clover_build(U, L, m, 1.0) if clover else None
    ref = oracle.cg_solve(U, b, L, m, A=A, tol=1e-10, maxit=1000)
    c = _ctx(q, L)
    try:
        fU = _field(q, c, q.QDP_GAUGE, 0, q.QDP_ALL, U)
        fb = _field(q, c, q.QDP_FERMION, 0, q.QDP_ALL, b)
        fx = q.qdp_field_alloc(c, q.QDP_FERMION, 0, q.QDP_ALL)
        fA = fAi = None
        if clover:
            fA = q.qdp_field_alloc(c, q.QDP_CLOVER, 0, q.QDP_ALL)
            fAi = q.qdp_field_alloc(c, q.QDP_CLOVER, 0, q.QDP_EVEN)
            q.qdp_clover_build(fA, fAi, fU, m, 1.0)
        res = q.qdp_cg_solve(fx, fb, fU, fA, fAi, mass=m, tol=1e-10, maxit=1000)
        assert res["status"] == q.QDP_OK
        assert res["iters"] == ref["iters"]
        assert np.max(np.abs(res["hist"] - ref["hist"]) / ref["hist"]) <= 1e-10
        assert res["true_resid"] <= 5e-10 and abs(res["true_resid"] - ref["true_resid"]) <= 1e-11
        x = q.qdp_field_export(fx)
        assert rel_site_err(x, ref["x"]) <= 1e-9
    finally:
        q.qdp_finalize(c)


def test_cg_self_halo_matches(q):
    """The CG through the halo code path gives the oracle history too."""
    L = (4, 4, 4, 8)
    U = fieldgen.random_gauge(L, 1005)
    b = fieldgen.random_spinor(L, 2006)
    ref = oracle.cg_solve(U, b, L, 0.1, tol=1e-10, maxit=1000)
    c = _ctx(q, L, self_halo=12)
    try:
        fU = _field(q, c, q.QDP_GAUGE, 0, q.QDP_ALL, U)
        fb = _field(q, c, q.QDP_FERMION, 0, q.QDP_ALL, b)
        fx = q.qdp_field_alloc(c, q.QDP_FERMION, 0, q.QDP_ALL)
        res = q.qdp_cg_solve(fx, fb, fU, mass=0.1, tol=1e-10, maxit=1000)
        assert res["iters"] == ref["iters"]
        assert np.max(np.abs(res["hist"] - ref["hist"]) / ref["hist"]) <= 1e-10
    finally:
        q.qdp_finalize(c)


def test_errors(q):
    L = (4, 4, 4, 4)
    c = _ctx(q, L)
    try:
        f64 = q.qdp_field_alloc(c, q.QDP_FERMION, 0, q.QDP_ALL)
        f32 = q.qdp_field_alloc(c, q.QDP_FERMION, 1, q.QDP_ALL)
        U = q.qdp_field_alloc(c, q.QDP_GAUGE, 0, q.QDP_ALL)
        for fn, st in ((lambda: q.qdp_dslash(f64, U, f64, q.QDP_ALL), q.QDP_EALIAS),
                       (lambda: q.qdp_dslash(f32, U, f64, q.QDP_ALL), q.QDP_EPREC),
                       (lambda: q.qdp_dslash(f64, U, U, 0), q.QDP_EINVAL),
                       (lambda: q.qdp_shift(f64, f64, 4, 1), q.QDP_EINVAL),
                       (lambda: q.qdp_inner_product(f64, f32), q.QDP_EPREC),
                       (lambda: q.qdp_set_option(c, q.QDP_OPT_SELF_HALO, 99), q.QDP_EINVAL)):
            with pytest.raises(q.QdpError) as e:
                fn()
            assert e.value.status == st
    finally:
        q.qdp_finalize(c)


def test_wrap_torch_tensor(q):
    """Fields can live in torch-allocated device memory (PyTorch as the allocator)."""
    import torch
    L = (4, 4, 4, 8)
    c = _ctx(q, L)
    try:
        _, db = q.qdp_field_bytes(c, q.QDP_FERMION, 0, q.QDP_ALL)
        t = torch.zeros(db // 8, dtype=torch.float64, device="cuda")
        f = q.qdp_field_wrap(c, q.QDP_FERMION, 0, q.QDP_ALL, t)
        psi = fieldgen.random_spinor(L, 3)
        q.qdp_field_import(f, psi)
        assert np.array_equal(q.qdp_field_export(f), psi)
        assert abs(q.qdp_norm2(f) - oracle.norm2(psi, L)) <= 1e-13 * oracle.norm2(psi, L)
        assert float(t.abs().sum()) > 0
    finally:
        q.qdp_finalize(c)


@pytest.mark.parametrize("mask", [8, 15])
def test_clover_build_shifts_of_shifts(q, mask):
    """Partitioned build path (leaves from shifted gauge fields) via self-halo."""
    L = (4, 6, 4, 4)
    U = fieldgen.random_gauge(L, 1501)
    A = oracle.clover_build(U, L, -0.1, 1.3)
    Ai = oracle.clover_invert(A, L)
    c = _ctx(q, L, self_halo=mask)
    try:
        fU = _field(q, c, q.QDP_GAUGE, 0, q.QDP_ALL, U)
        fA = q.qdp_field_alloc(c, q.QDP_CLOVER, 0, q.QDP_ALL)
        fAi = q.qdp_field_alloc(c, q.QDP_CLOVER, 0, q.QDP_ALL)
        q.qdp_clover_build(fA, fAi, fU, -0.1, 1.3)
        assert np.max(np.abs(q.qdp_field_export(fA) - A)) <= 1e-13 * np.max(np.abs(A))
        assert np.max(np.abs(q.qdp_field_export(fAi) - Ai)) <= 1e-13 * np.max(np.abs(Ai))
        n_shift, _ = q.qdp_profile_query(c, q.QDP_PK_SHIFT)
        assert n_shift == 6 * 7
    finally:
        q.qdp_finalize(c)


def test_cg_clover_self_halo(q):
    L = (4, 4, 6, 4)
    U = fieldgen.random_gauge(L, 1601)
    b = fieldgen.random_spinor(L, 2601)
    A = oracle.clover_build(U, L, 0.1, 1.0)
    ref = oracle.cg_solve(U, b, L, 0.1, A=A, tol=1e-10, maxit=1000)
    c = _ctx(q, L, self_halo=12)
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


@pytest.mark.parametrize("prec", [0, 1])
def test_dslash_bench_size(q, prec):
    """The bench's per-GPU lattice (40^3 x 32) and launch configuration: every output site of
    one EO dslash against the oracle."""
    L = (40, 40, 40, 32)
    U = _round(fieldgen.random_gauge(L, 1004), prec)
    psi = _round(fieldgen.random_spinor(L, 2005), prec)
    ref = oracle.hopping(U, psi, L, 0)
    c = _ctx(q, L)
    try:
        fU = _field(q, c, q.QDP_GAUGE, prec, q.QDP_ALL, U)
        fp = _field(q, c, q.QDP_FERMION, prec, 1, psi[fieldgen.cb_sites(L, 1)])
        fo = q.qdp_field_alloc(c, q.QDP_FERMION, prec, 0)
        q.qdp_dslash(fo, fU, fp, 0)
        got = q.qdp_field_export(fo).astype(np.float64)
        assert rel_site_err(got, ref[fieldgen.cb_sites(L, 0)]) <= TOL[prec]
    finally:
        q.qdp_finalize(c)


def test_cg_bench_config_history(q):
    """The bench step (40^3 x 32 clover CGNR, m = 0.1, c_SW = 1) for 3 iterations: history,
    solution and true residual against the oracle."""
    L = (40, 40, 40, 32)
    U = fieldgen.random_gauge(L, 1004)
    b = fieldgen.random_spinor(L, 2005)
    A = oracle.clover_build(U, L, 0.1, 1.0)
    ref = oracle.cg_solve(U, b, L, 0.1, A=A, tol=0.0, maxit=3)
    del A
    c = _ctx(q, L)
    try:
        fU = _field(q, c, q.QDP_GAUGE, 0, q.QDP_ALL, U)
        fb = _field(q, c, q.QDP_FERMION, 0, q.QDP_ALL, b)
        fx = q.qdp_field_alloc(c, q.QDP_FERMION, 0, q.QDP_ALL)
        fA = q.qdp_field_alloc(c, q.QDP_CLOVER, 0, q.QDP_ALL)
        fAi = q.qdp_field_alloc(c, q.QDP_CLOVER, 0, q.QDP_EVEN)
        q.qdp_clover_build(fA, fAi, fU, 0.1, 1.0)
        res = q.qdp_cg_solve(fx, fb, fU, fA, fAi, mass=0.1, tol=0.0, maxit=3)
        assert res["status"] == q.QDP_NOT_CONVERGED and res["iters"] == 3
        assert np.max(np.abs(res["hist"] - ref["hist"]) / ref["hist"]) <= 1e-10
        assert abs(res["true_resid"] - ref["true_resid"]) <= 1e-10 * ref["true_resid"]
        assert rel_site_err(q.qdp_field_export(fx), ref["x"]) <= 1e-11
    finally:
        q.qdp_finalize(c)


@pytest.mark.timeout(1200)
def test_cg_config3_converges(q):
    """Config 3: 32^3 x 64 Wilson-clover CG to 1e-10 (hot field): the FULL residual history and
    the iteration count against the oracle's solve of the same system (reading R14: every entry
    within 1e-10 relative, same number of iterations), the solution site by site and the true
    residual.  The oracle needs about a minute on 16 host cores for this."""
    L = (32, 32, 32, 64)
    m = 0.1
    U = fieldgen.random_gauge(L, 1003)
    b = fieldgen.random_spinor(L, 2004)
    A = oracle.clover_build(U, L, m, 1.0)
    ref = oracle.cg_solve(U, b, L, m, A=A, tol=1e-10, maxit=2000)
    del A
    c = _ctx(q, L)
    try:
        fU = _field(q, c, q.QDP_GAUGE, 0, q.QDP_ALL, U)
        fb = _field(q, c, q.QDP_FERMION, 0, q.QDP_ALL, b)
        fx = q.qdp_field_alloc(c, q.QDP_FERMION, 0, q.QDP_ALL)
        fA = q.qdp_field_alloc(c, q.QDP_CLOVER, 0, q.QDP_ALL)
        fAi = q.qdp_field_alloc(c, q.QDP_CLOVER, 0, q.QDP_EVEN)
        q.qdp_clover_build(fA, fAi, fU, m, 1.0)
        res = q.qdp_cg_solve(fx, fb, fU, fA, fAi, mass=m, tol=1e-10, maxit=2000)
        assert res["status"] == q.QDP_OK
        assert res["iters"] == ref["iters"]
        assert len(res["hist"]) == len(ref["hist"]) == ref["iters"] + 1
        assert np.max(np.abs(res["hist"] - ref["hist"]) / ref["hist"]) <= 1e-10
        assert res["hist"][-1] <= 1e-10 < res["hist"][-2]
        assert res["true_resid"] <= 1e-9
        # |b - M x| / |b| ~ 5e-11 is a difference of nearly equal vectors: compare it absolutely
        # (its relative rounding error is ~eps / 5e-11)
        assert abs(res["true_resid"] - ref["true_resid"]) <= 1e-14
        assert rel_site_err(q.qdp_field_export(fx), ref["x"]) <= 1e-10
    finally:
        q.qdp_finalize(c)
