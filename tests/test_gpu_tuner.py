"""The paper's autotuner on the whole-lattice EO dslash: the first payload
launches probe the launch variants (four threads per site, then the main kernel with 64 and 32
threads per block) and keep the fastest.  Every probed variant must give the oracle's answer, on
ragged volumes (a partial last block) in both precisions, and the Wilson CG built on them (PLAIN
and XPAY launches tuned separately) must keep the oracle's residual history."""
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


@pytest.mark.parametrize("prec", [0, 1])
@pytest.mark.parametrize("L", [(4, 6, 2, 4), (6, 4, 6, 10), (16, 16, 16, 8)])
def test_tuned_variants_match_oracle(q, prec, L):
    U = fieldgen.random_gauge(L, 4101)
    psi = fieldgen.random_spinor(L, 4201)
    if prec:
        U, psi = U.astype(np.float32).astype(np.float64), psi.astype(np.float32).astype(np.float64)
    par = fieldgen.parity(L)
    ref = oracle.hopping(U, psi, L, -1)
    c = q.qdp_init(L)
    try:
        dt = np.float64 if prec == 0 else np.float32
        fU = q.qdp_field_alloc(c, q.QDP_GAUGE, prec, q.QDP_ALL)
        q.qdp_field_import(fU, U.astype(dt))
        for p in (0, 1):
            fi = q.qdp_field_alloc(c, q.QDP_FERMION, prec, 1 - p)
            q.qdp_field_import(fi, np.ascontiguousarray(psi[par == 1 - p]).astype(dt))
            fo = q.qdp_field_alloc(c, q.QDP_FERMION, prec, p)
            for _ in range(6):  # probes every variant, then the chosen one
                q.qdp_field_zero(fo)
                q.qdp_dslash(fo, fU, fi, p)
                got = q.qdp_field_export(fo).astype(np.float64)
                assert rel_site_err(got, ref[par == p]) <= TOL[prec]
    finally:
        q.qdp_finalize(c)


def test_tuned_wilson_cg_history(q):
    L = (6, 6, 4, 8)
    U = fieldgen.random_gauge(L, 4102)
    b = fieldgen.random_spinor(L, 4202)
    ref = oracle.cg_solve(U, b, L, 0.1, tol=1e-10, maxit=500)
    c = q.qdp_init(L)
    try:
        fU = q.qdp_field_alloc(c, q.QDP_GAUGE, 0, q.QDP_ALL)
        q.qdp_field_import(fU, U)
        fb = q.qdp_field_alloc(c, q.QDP_FERMION, 0, q.QDP_ALL)
        q.qdp_field_import(fb, b)
        fx = q.qdp_field_alloc(c, q.QDP_FERMION, 0, q.QDP_ALL)
        for _ in range(2):  # the first solve runs through the probes, the second on the choice
            res = q.qdp_cg_solve(fx, fb, fU, mass=0.1, tol=1e-10, maxit=500)
            assert res["iters"] == ref["iters"]
            assert np.max(np.abs(res["hist"] - ref["hist"]) / ref["hist"]) <= 1e-10
            assert rel_site_err(q.qdp_field_export(fx), ref["x"]) <= 1e-9
    finally:
        q.qdp_finalize(c)


def test_cg_chunked_stop_is_exact(q):
    """The device-side CG stops at the same iteration whatever the chunking (QDPB_CG_CHUNK = 1:
    a host read every iteration, like the oracle) -- run in a subprocess for the environment."""
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    code = ("import sys, json; sys.path[:0] = ['.']; import fieldgen; from paper_1408_5925_b200 import qdpb as q; "
            "L = (6, 6, 4, 8); U = fieldgen.random_gauge(L, 4102); b = fieldgen.random_spinor(L, 4202); "
            "c = q.qdp_init(L); fU = q.qdp_field_alloc(c, q.QDP_GAUGE, 0, q.QDP_ALL); q.qdp_field_import(fU, U); "
            "fb = q.qdp_field_alloc(c, q.QDP_FERMION, 0, q.QDP_ALL); q.qdp_field_import(fb, b); "
            "fx = q.qdp_field_alloc(c, q.QDP_FERMION, 0, q.QDP_ALL); "
            "r = q.qdp_cg_solve(fx, fb, fU, mass=0.1, tol=1e-10, maxit=500); "
            "print(json.dumps([r['iters'], list(r['hist'])]))")
    out = {}
    for ch in ("1", "16"):
        r = subprocess.run([sys.executable, "-c", code], cwd=root, env=dict(os.environ, QDPB_CG_CHUNK=ch),
                           capture_output=True, text=True, timeout=200)
        assert r.returncode == 0, r.stderr
        out[ch] = __import__("json").loads(r.stdout.strip().splitlines()[-1])
    assert out["1"][0] == out["16"][0]
    assert np.max(np.abs(np.array(out["1"][1]) - np.array(out["16"][1]))) <= 1e-13


@pytest.mark.parametrize("recon", [18, 12])
@pytest.mark.parametrize("L", [(4, 6, 2, 4), (6, 4, 6, 10), (8, 8, 8, 16)])
def test_forced_variants_fp64_bit_identical(q, L, recon):
    """Every fp64 launch variant (QDP_OPT_DSLASH_VARIANT) but the four-threads-per-site one, including
    the asynchronously pipelined one (4: cp.async hop stages), computes exactly the main kernel's
    arithmetic in the same order: the plain EO hopping term is the oracle's and bit-identical across variants, and so is a
    clover CG (its non-fused dslash launches -- the A^-1 and A x + b D epilogues -- take the forced
    variant): same residual history and solution bits."""
    U = fieldgen.random_gauge(L, 4103)
    psi = fieldgen.random_spinor(L, 4203)
    par = fieldgen.parity(L)
    ref = oracle.hopping(U, psi, L, -1)
    c = q.qdp_init(L)
    try:
        fU = q.qdp_field_alloc(c, q.QDP_GAUGE12 if recon == 12 else q.QDP_GAUGE, 0, q.QDP_ALL)
        q.qdp_field_import(fU, U)
        fA = q.qdp_field_alloc(c, q.QDP_CLOVER, 0, q.QDP_ALL)
        fAi = q.qdp_field_alloc(c, q.QDP_CLOVER, 0, q.QDP_EVEN)
        q.qdp_clover_build(fA, fAi, fU, 0.1, 1.0)
        fi = q.qdp_field_alloc(c, q.QDP_FERMION, 0, q.QDP_ODD)
        q.qdp_field_import(fi, np.ascontiguousarray(psi[par == 1]))
        fo = q.qdp_field_alloc(c, q.QDP_FERMION, 0, q.QDP_EVEN)
        fb = q.qdp_field_alloc(c, q.QDP_FERMION, 0, q.QDP_ALL)
        q.qdp_field_import(fb, psi)
        fx = q.qdp_field_alloc(c, q.QDP_FERMION, 0, q.QDP_ALL)
        q.qdp_set_option(c, q.QDP_OPT_AUTOTUNE, 0)  # fixed reduction launches: identical sums
        base = None
        for v in (1, 0, 2, 3, 4, 5):
            q.qdp_set_option(c, q.QDP_OPT_DSLASH_VARIANT, v)
            q.qdp_field_zero(fo)
            q.qdp_dslash(fo, fU, fi, q.QDP_EVEN)
            got = q.qdp_field_export(fo)
            r = q.qdp_cg_solve(fx, fb, fU, fA, fAi, mass=0.1, tol=1e-30, maxit=8)
            now = (got, r["hist"].copy(), q.qdp_field_export(fx))
            if base is None:
                base = now
                assert rel_site_err(got, ref[par == 0]) <= 1e-13
            elif v == 0:  # four threads per site: the directions' partial sums meet in another order
                assert rel_site_err(got, base[0]) <= 1e-14
                assert np.max(np.abs(now[1] - base[1]) / base[1]) <= 1e-12
            else:
                for a, b in zip(now, base):
                    assert np.array_equal(a, b), v
    finally:
        q.qdp_finalize(c)
