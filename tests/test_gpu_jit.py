"""Run-time generated site expressions (qdp_jit_eval, PAPER.md sections III-IV) against the oracle.

Every expression is compared element by element with the oracle's functions (Table II kernels,
shift, the hopping term of PAPER.md:282) or with plain numpy on the oracle's gamma matrices:
fp64 per-site relative L2 error <= 1e-13 (1e-14 for single products), fp32 <= 2e-6 against the
oracle in double on the fp32-rounded inputs, shifts bit-exact."""
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


def _dt(prec):
    return np.float64 if prec == 0 else np.float32


def _round(a, prec):
    return a if prec == 0 else a.astype(np.float32).astype(np.float64)


def _field(q, c, kind, prec, subset, host):
    f = q.qdp_field_alloc(c, kind, prec, subset)
    q.qdp_field_import(f, np.ascontiguousarray(host, dtype=_dt(prec)))
    return f


def _gauss(seed, shape, prec):
    return _round(fieldgen.gaussian(seed, int(np.prod(shape))).reshape(shape), prec)


def _err(got, ref):
    return rel_site_err(got.reshape(len(got), -1).astype(np.float64), ref.reshape(len(ref), -1))


def _cx(a):
    return a[..., 0] + 1j * a[..., 1]


def _re(z):
    return np.stack([z.real, z.imag], axis=-1)


def hopping_expr(gauge="$0", psi="$1", grouped=True):
    """PAPER.md:282 in the expression language (paper_1408_5925_b200/exprs.py)."""
    from paper_1408_5925_b200 import exprs
    return exprs.hopping(gauge, psi, grouped)


@pytest.mark.parametrize("prec", [0, 1])
@pytest.mark.parametrize("subset", [-1, 0])
def test_table2_products_vs_oracle(q, prec, subset):
    L = (8, 6, 4, 10)
    V = fieldgen.volume(L)
    u, v = _gauss(11, (V, 3, 3, 2), prec), _gauss(12, (V, 3, 3, 2), prec)
    s, t = _gauss(13, (V, 4, 4, 2), prec), _gauss(14, (V, 4, 4, 2), prec)
    p1, p2 = _gauss(15, (V, 4, 3, 2), prec), _gauss(16, (V, 4, 3, 2), prec)
    sites = np.arange(V) if subset < 0 else fieldgen.cb_sites(L, subset)
    c = q.qdp_init(L)
    try:
        F = lambda kind, arr: _field(q, c, kind, prec, subset, arr[sites])
        fu, fv = F(q.QDP_COLORMATRIX, u), F(q.QDP_COLORMATRIX, v)
        fs, ft = F(q.QDP_SPINMATRIX, s), F(q.QDP_SPINMATRIX, t)
        f1, f2 = F(q.QDP_FERMION, p1), F(q.QDP_FERMION, p2)
        oc = q.qdp_field_alloc(c, q.QDP_COLORMATRIX, prec, subset)
        osm = q.qdp_field_alloc(c, q.QDP_SPINMATRIX, prec, subset)
        of = q.qdp_field_alloc(c, q.QDP_FERMION, prec, subset)
        tol = 1e-14 if prec == 0 else 2e-6
        cases = [
            (oc, "$0*$1", (fu, fv), oracle.lcm(u, v)),                       # Table II lcm
            (of, "$0*$1", (fu, f1), oracle.upsi(u, p1)),                     # upsi
            (osm, "$0*$1", (fs, ft), oracle.spmat(s, t)),                    # spmat
            (of, "$0*$1 + $0*$2", (fu, f1, f2), oracle.matvec(u, p1, p2)),   # matvec
            (of, "adj($0)*$1", (fu, f1), oracle.adj_upsi(u, p1)),            # Fig. 1's adj(u)*phi
            (oc, "$0*adj($1) - 0.5*$1", (fu, fv), _re(_cx(oracle.lcm(u, _re(np.conj(np.swapaxes(_cx(v), 1, 2)))))
                                                      - 0.5 * _cx(v))),
            (of, "timesI($0) + 2*$1", (f1, f2), _re(1j * _cx(p1) + 2 * _cx(p2))),
        ]
        for out, expr, ops, ref in cases:
            q.qdp_jit_eval(out, expr, *ops)
            e = _err(q.qdp_field_export(out), ref[sites])
            assert e <= tol, (expr, e)
    finally:
        q.qdp_finalize(c)


@pytest.mark.parametrize("prec", [0, 1])
def test_gamma_and_spin_products(q, prec):
    """gamma(mu) and gamma5 as left factors, spin matrix x spinor, against numpy on the oracle's
    DeGrand-Rossi matrices (pinned in test_oracle_dslash: hermitian, anticommuting, gamma5 diagonal)."""
    L = (4, 4, 4, 6)
    V = fieldgen.volume(L)
    p = _gauss(21, (V, 4, 3, 2), prec)
    s = _gauss(22, (V, 4, 4, 2), prec)
    G = [oracle.gamma(m) for m in range(4)]
    g5 = G[0] @ G[1] @ G[2] @ G[3]
    c = q.qdp_init(L)
    try:
        fp = _field(q, c, q.QDP_FERMION, prec, -1, p)
        fs = _field(q, c, q.QDP_SPINMATRIX, prec, -1, s)
        of = q.qdp_field_alloc(c, q.QDP_FERMION, prec, -1)
        osm = q.qdp_field_alloc(c, q.QDP_SPINMATRIX, prec, -1)
        tol = 1e-15 if prec == 0 else 2e-7
        for m in range(5):
            gm = G[m] if m < 4 else g5
            name = f"gamma({m})" if m < 4 else "gamma5"
            q.qdp_jit_eval(of, f"{name}*$0", fp)
            assert _err(q.qdp_field_export(of), _re(np.einsum("st,vtc->vsc", gm, _cx(p)))) <= tol, name
            q.qdp_jit_eval(osm, f"{name}*$0", fs)
            assert _err(q.qdp_field_export(osm), _re(np.einsum("st,vtu->vsu", gm, _cx(s)))) <= tol, name
        # (1 - gamma_mu) projection written out, and gamma_mu^2 = 1 exactly
        q.qdp_jit_eval(of, "$0 - gamma(2)*$0", fp)
        assert _err(q.qdp_field_export(of), _re(_cx(p) - np.einsum("st,vtc->vsc", G[2], _cx(p)))) <= tol
        q.qdp_jit_eval(of, "gamma(1)*(gamma(1)*$0)", fp)
        assert np.array_equal(q.qdp_field_export(of), p.astype(_dt(prec)))
        q.qdp_jit_eval(of, "$1*$0", fp, fs)
        ref = _re(np.einsum("vst,vtc->vsc", _cx(s), _cx(p)))
        assert _err(q.qdp_field_export(of), ref) <= (1e-14 if prec == 0 else 2e-6)
    finally:
        q.qdp_finalize(c)


@pytest.mark.parametrize("prec", [0, 1])
def test_shift_bit_exact(q, prec):
    """shift(e, mu, s) evaluated in place equals the oracle's circular shift bit for bit
    (PAPER.md:111-126), on full fields and from one parity to the other; shifts of shifts."""
    L = (6, 4, 8, 4)
    V = fieldgen.volume(L)
    p = _gauss(31, (V, 4, 3, 2), prec)
    u = _gauss(32, (V, 3, 3, 2), prec)
    c = q.qdp_init(L)
    try:
        fp = _field(q, c, q.QDP_FERMION, prec, -1, p)
        fu = _field(q, c, q.QDP_COLORMATRIX, prec, -1, u)
        of = q.qdp_field_alloc(c, q.QDP_FERMION, prec, -1)
        oc = q.qdp_field_alloc(c, q.QDP_COLORMATRIX, prec, -1)
        for mu in range(4):
            for s in (1, -1):
                q.qdp_jit_eval(of, f"shift($0,{mu},{s:+d})", fp)
                assert np.array_equal(q.qdp_field_export(of), oracle.shift(p, L, mu, s).astype(_dt(prec)))
                q.qdp_jit_eval(oc, f"shift($0,{mu},{s:+d})", fu)
                assert np.array_equal(q.qdp_field_export(oc), oracle.shift(u, L, mu, s).astype(_dt(prec)))
        # diagonal neighbour (shift of a shift) and a full circle (L_mu shifts)
        q.qdp_jit_eval(of, "shift(shift($0,0,+1),3,-1)", fp)
        assert np.array_equal(q.qdp_field_export(of),
                              oracle.shift(oracle.shift(p, L, 0, 1), L, 3, -1).astype(_dt(prec)))
        q.qdp_jit_eval(of, "shift(shift(shift(shift($0,3,1),3,1),3,1),3,1)", fp)
        assert np.array_equal(q.qdp_field_export(of), p.astype(_dt(prec)))
        # checkerboard: odd input -> even output
        odd, even = fieldgen.cb_sites(L, 1), fieldgen.cb_sites(L, 0)
        fo = _field(q, c, q.QDP_FERMION, prec, 1, p[odd])
        oe = q.qdp_field_alloc(c, q.QDP_FERMION, prec, 0)
        q.qdp_jit_eval(oe, "shift($0,2,-1)", fo)
        assert np.array_equal(q.qdp_field_export(oe), oracle.shift(p, L, 2, -1)[even].astype(_dt(prec)))
    finally:
        q.qdp_finalize(c)


@pytest.mark.parametrize("prec", [0, 1])
def test_fig1_derivative(q, prec):
    """Fig. 1: psi = u[mu]*shift(phi, FORWARD, mu) + shift(adj(u[mu])*phi,
    BACKWARD, mu) as ONE generated kernel, vs the oracle's shift / upsi / adj_upsi."""
    L = (4, 6, 4, 8)
    U = _round(fieldgen.random_gauge(L, 41), prec)
    phi = _round(fieldgen.random_spinor(L, 42), prec)
    c = q.qdp_init(L)
    try:
        fU = _field(q, c, q.QDP_GAUGE, prec, -1, U)
        fphi = _field(q, c, q.QDP_FERMION, prec, -1, phi)
        out = q.qdp_field_alloc(c, q.QDP_FERMION, prec, -1)
        for mu in range(4):
            q.qdp_jit_eval(out, f"$0[{mu}]*shift($1,{mu},+1) + shift(adj($0[{mu}])*$1,{mu},-1)", fU, fphi)
            ref = (oracle.upsi(U[:, mu], oracle.shift(phi, L, mu, 1))
                   + oracle.shift(oracle.adj_upsi(U[:, mu], phi), L, mu, -1))
            assert _err(q.qdp_field_export(out), ref) <= TOL[prec], mu
    finally:
        q.qdp_finalize(c)


@pytest.mark.parametrize("prec", [0, 1])
@pytest.mark.parametrize("L", [(4, 4, 4, 4), (8, 6, 4, 10), (2, 2, 2, 2)])
@pytest.mark.parametrize("gauge_kind", ["r18", "r12"])
def test_hopping_expression_vs_oracle(q, prec, L, gauge_kind):
    """The hopping term of PAPER.md:282 written as an expression and generated at run time equals
    the oracle's H (full lattice and even-odd) and the hand-written fused dslash."""
    U = _round(fieldgen.random_gauge(L, 51), prec)
    psi = _round(fieldgen.random_spinor(L, 52), prec)
    gk = q.QDP_GAUGE if gauge_kind == "r18" else q.QDP_GAUGE12
    c = q.qdp_init(L)
    try:
        fU = _field(q, c, gk, prec, -1, U)
        fp = _field(q, c, q.QDP_FERMION, prec, -1, psi)
        out = q.qdp_field_alloc(c, q.QDP_FERMION, prec, -1)
        ref = oracle.hopping(U, psi, L, -1)
        tol = TOL[prec]
        for grouped in (True, False):  # grouped and left-associated forms (both spin-projected)
            q.qdp_jit_eval(out, hopping_expr(grouped=grouped), fU, fp)
            assert _err(q.qdp_field_export(out), ref) <= tol, grouped
        # the literal sum (no projection): "1*(A)" is not the same text as A, so no term pairs up
        lit = " + ".join(f"(1*($0[{m}]*shift($1,{m},+1)) - gamma({m})*($0[{m}]*shift($1,{m},+1)))"
                         f" + (1*shift(adj($0[{m}])*$1,{m},-1) + gamma({m})*shift(adj($0[{m}])*$1,{m},-1))"
                         for m in range(4))
        q.qdp_jit_eval(out, lit, fU, fp)
        assert _err(q.qdp_field_export(out), ref) <= tol
        # even-odd: out_e = H_eo psi_o, compared with the fused kernel too
        even, odd = fieldgen.cb_sites(L, 0), fieldgen.cb_sites(L, 1)
        fo = _field(q, c, q.QDP_FERMION, prec, 1, psi[odd])
        oe = q.qdp_field_alloc(c, q.QDP_FERMION, prec, 0)
        q.qdp_jit_eval(oe, hopping_expr(), fU, fo)
        got = q.qdp_field_export(oe)
        assert _err(got, ref[even]) <= tol
        od = q.qdp_field_alloc(c, q.QDP_FERMION, prec, 0)
        q.qdp_dslash(od, fU, fo, 0)
        assert _err(got, q.qdp_field_export(od).astype(np.float64)) <= tol
    finally:
        q.qdp_finalize(c)


def test_cache_accounting_and_errors(q):
    L = (4, 4, 4, 8)
    V = fieldgen.volume(L)
    U = fieldgen.random_gauge(L, 61)
    psi = fieldgen.random_spinor(L, 62)
    c = q.qdp_init(L)
    try:
        fU = _field(q, c, q.QDP_GAUGE, 0, -1, U)
        fp = _field(q, c, q.QDP_FERMION, 0, -1, psi)
        out = q.qdp_field_alloc(c, q.QDP_FERMION, 0, -1)
        fo = _field(q, c, q.QDP_FERMION, 0, 1, psi[fieldgen.cb_sites(L, 1)])
        oe = q.qdp_field_alloc(c, q.QDP_FERMION, 0, 0)
        n0, _ = q.qdp_jit_stats(c)
        q.qdp_profile_reset(c)
        for _ in range(3):
            q.qdp_jit_eval(oe, hopping_expr(), fU, fo)
        n1, secs = q.qdp_jit_stats(c)
        assert n1 == n0 + 1 and secs > 0  # compiled once, then cached
        fl, by = q.qdp_profile_work(c, q.QDP_PK_BLAS)
        src, work = q.qdp_jit_source(hopping_expr(), q.QDP_FERMION, 0, [q.QDP_GAUGE, q.QDP_FERMION], out_subset=0)
        assert by == 3 * (V // 2) * work["bytes"] == 3 * (V // 2) * 1536  # EO compulsory = dslash's
        assert fl == 3 * (V // 2) * work["flops"]
        with pytest.raises(q.QdpError) as e:  # odd operand read at even sites
            q.qdp_jit_eval(oe, "2*$0", fo)
        assert e.value.status == q.QDP_EINVAL
        with pytest.raises(q.QdpError) as e:
            q.qdp_jit_eval(out, "$0*$0", fp)
        assert e.value.status == q.QDP_EINVAL
        with pytest.raises(q.QdpError) as e:
            q.qdp_jit_eval(fp, "2*$0", fp)
        assert e.value.status == q.QDP_EALIAS
        f32 = q.qdp_field_alloc(c, q.QDP_FERMION, 1, -1)
        with pytest.raises(q.QdpError) as e:
            q.qdp_jit_eval(out, "$0", f32)
        assert e.value.status == q.QDP_EPREC
    finally:
        q.qdp_finalize(c)
    # shifts along dimensions reached through the halo path: those leaves are materialised with
    # qdp_shift (face exchange), the rest stays in the kernel; same results as the whole lattice
    for mask in (8, 12, 15):
        c = q.qdp_init(L)
        try:
            q.qdp_set_option(c, q.QDP_OPT_SELF_HALO, mask)
            fU = _field(q, c, q.QDP_GAUGE, 0, -1, U)
            fp = _field(q, c, q.QDP_FERMION, 0, -1, psi)
            out = q.qdp_field_alloc(c, q.QDP_FERMION, 0, -1)
            for expr, ref in (("shift($0,3,+1)", oracle.shift(psi, L, 3, 1)),
                              ("shift(shift($0,2,-1),3,-1)", oracle.shift(oracle.shift(psi, L, 2, -1), L, 3, -1))):
                q.qdp_jit_eval(out, expr, fp)
                assert np.array_equal(q.qdp_field_export(out), ref), (mask, expr)
            for _ in range(2):
                q.qdp_jit_eval(out, hopping_expr(), fU, fp)
            assert _err(q.qdp_field_export(out), oracle.hopping(U, psi, L, -1)) <= 1e-13, mask
            # even-odd through the halo path
            fo = _field(q, c, q.QDP_FERMION, 0, 1, psi[fieldgen.cb_sites(L, 1)])
            oe = q.qdp_field_alloc(c, q.QDP_FERMION, 0, 0)
            q.qdp_jit_eval(oe, hopping_expr(), fU, fo)
            ref = oracle.hopping(U, psi, L, 0)[fieldgen.cb_sites(L, 0)]
            assert _err(q.qdp_field_export(oe), ref) <= 1e-13, mask
        finally:
            q.qdp_finalize(c)


def _plaq_ref(U, L, mu, nu):
    """sum_x Re tr U_mu(x) U_nu(x+mu) U_mu(x+nu)^dag U_nu(x)^dag from the oracle's products and shifts"""
    Umu, Unu = U[:, mu], U[:, nu]
    adj = lambda m: _re(np.conj(np.swapaxes(_cx(m), 1, 2)))
    t = oracle.lcm(oracle.lcm(Umu, oracle.shift(Unu, L, mu, 1)), adj(oracle.shift(Umu, L, nu, 1)))
    t = oracle.lcm(t, adj(Unu))
    return float(np.sum(np.trace(_cx(t), axis1=1, axis2=2).real))


def plaq_expr(mu, nu):
    return f"real(trace($0[{mu}]*shift($0[{nu}],{mu},+1)*adj(shift($0[{mu}],{nu},+1))*adj($0[{nu}])))"


@pytest.mark.parametrize("prec", [0, 1])
def test_sums_plaquette_norms(q, prec):
    """qdp_jit_sum: the plaquette (QDP++ sum(real(trace(...))) over shifted links) against the
    oracle's products / shifts, its closed form on the unit gauge field (3 per site) and its gauge
    invariance; localNorm2 / localInnerProduct sums against the oracle's norm2 / inner, exact on
    integer-valued inputs; determinism."""
    from _physics import gauge_transform
    L = (4, 6, 4, 8)
    V = fieldgen.volume(L)
    U = _round(fieldgen.random_gauge(L, 71), prec)
    c = q.qdp_init(L)
    try:
        fU = _field(q, c, q.QDP_GAUGE, prec, -1, U)
        tol = 1e-12 if prec == 0 else 1e-5
        for mu, nu in ((0, 1), (2, 3), (1, 3)):
            got = q.qdp_jit_sum(c, plaq_expr(mu, nu), fU)
            ref = _plaq_ref(U, L, mu, nu)
            assert abs(got.real - ref) <= tol * 3 * V and got.imag == 0.0, (mu, nu, got, ref)
            assert q.qdp_jit_sum(c, plaq_expr(mu, nu), fU) == got  # deterministic
            # even + odd = all
            e = q.qdp_jit_sum(c, plaq_expr(mu, nu), fU, subset=0)
            o = q.qdp_jit_sum(c, plaq_expr(mu, nu), fU, subset=1)
            assert abs(e.real + o.real - got.real) <= tol * 3 * V
        # gauge invariance: U_mu(x) -> g(x) U_mu(x) g(x+mu)^dag leaves the plaquette unchanged
        Ug = _round(gauge_transform(U, fieldgen.random_gauge_transform(L, 72), L), prec)
        fUg = _field(q, c, q.QDP_GAUGE, prec, -1, Ug)
        assert abs(q.qdp_jit_sum(c, plaq_expr(0, 3), fUg).real - q.qdp_jit_sum(c, plaq_expr(0, 3), fU).real) \
            <= (1e-11 if prec == 0 else 1e-4) * 3 * V
        # unit gauge field: exactly 3 per site
        f1 = _field(q, c, q.QDP_GAUGE, prec, -1, fieldgen.unit_gauge(L))
        assert q.qdp_jit_sum(c, plaq_expr(1, 2), f1) == complex(3 * V, 0)
        # norms and inner products: integer-valued spinors give exact sums
        a = np.round(4 * fieldgen.random_spinor(L, 73))
        b = np.round(4 * fieldgen.random_spinor(L, 74))
        fa, fb = _field(q, c, q.QDP_FERMION, prec, -1, a), _field(q, c, q.QDP_FERMION, prec, -1, b)
        assert q.qdp_jit_sum(c, "localNorm2($0)", fa) == complex(oracle.norm2(a, L), 0)
        assert q.qdp_jit_sum(c, "localInnerProduct($0, $1)", fa, fb) == oracle.inner(a, b, L)
        for sub in (0, 1):
            assert q.qdp_jit_sum(c, "localNorm2($0)", fa, subset=sub) == complex(oracle.norm2(a, L, sub), 0)
        # complex-scalar algebra: <a, b> + i |a|^2 - 2 tr(U_0)
        ref = oracle.inner(a, b, L) + 1j * oracle.norm2(a, L) - 2 * np.sum(np.trace(_cx(U[:, 0]), axis1=1, axis2=2))
        got = q.qdp_jit_sum(c, "localInnerProduct($0,$1) + timesI(localNorm2($0)) - 2*trace($2[0])", fa, fb, fU)
        assert abs(got - ref) <= (1e-12 if prec == 0 else 1e-5) * abs(ref)
        with pytest.raises(q.QdpError) as e:
            q.qdp_jit_sum(c, "$0", fa)
        assert e.value.status == q.QDP_EINVAL
    finally:
        q.qdp_finalize(c)
