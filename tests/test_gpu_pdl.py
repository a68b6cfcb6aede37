"""Programmatic dependent launch (QDP_OPT_PDL) and the fused boundary's visiting order.

PDL only changes when a solver kernel may become resident, never what it computes: the CG with
PDL on and off must give bit-identical residual histories and solutions, and both must match the
oracle (PAPER.md:31 north star: the even-odd CG).  The fused peer-to-peer boundary visits its face
sites halfway through the interior by default (QDPB_FACE_AT, read once per process): faces first
(every block waits at once) and faces last must give the oracle's hopping term too."""
import os
import subprocess
import sys

import numpy as np
import pytest

import fieldgen
import oracle
from _physics import rel_site_err

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def q():
    from paper_1408_5925_b200 import qdpb
    qdpb.lib()
    return qdpb


def _field(q, c, kind, subset, host):
    f = q.qdp_field_alloc(c, kind, q.QDP_F64, subset)
    q.qdp_field_import(f, np.ascontiguousarray(host, dtype=np.float64))
    return f


@pytest.mark.timeout(300)
@pytest.mark.parametrize("mask", [0, 8, 12])
@pytest.mark.parametrize("clover", [False, True])
def test_cg_pdl_on_off_identical(q, clover, mask):
    L = (8, 8, 4, 8)
    U = fieldgen.random_gauge(L, 4101)
    b = fieldgen.random_spinor(L, 4201)
    A = oracle.clover_build(U, L, 0.1, 1.0) if clover else None
    orc = oracle.cg_solve(U, b, L, 0.1, A=A, tol=1e-30, maxit=12)
    c = q.qdp_init(L)
    try:
        if mask:
            q.qdp_set_option(c, q.QDP_OPT_SELF_HALO, mask)
            q.qdp_set_option(c, q.QDP_OPT_P2P, 1)
        assert q.qdp_get_option(c, q.QDP_OPT_PDL) == 1  # the default
        # fixed launch configurations: the tuner's probes change reduction block sizes (and with
        # them the summation order) between payload launches
        q.qdp_set_option(c, q.QDP_OPT_AUTOTUNE, 0)
        fU = _field(q, c, q.QDP_GAUGE, q.QDP_ALL, U)
        fb = _field(q, c, q.QDP_FERMION, q.QDP_ALL, b)
        fx = q.qdp_field_alloc(c, q.QDP_FERMION, q.QDP_F64, q.QDP_ALL)
        fA = fAi = None
        if clover:
            fA = q.qdp_field_alloc(c, q.QDP_CLOVER, q.QDP_F64, q.QDP_ALL)
            fAi = q.qdp_field_alloc(c, q.QDP_CLOVER, q.QDP_F64, q.QDP_EVEN)
            q.qdp_clover_build(fA, fAi, fU, 0.1, 1.0)
        out = {}
        for pdl in (1, 0, 1):
            q.qdp_set_option(c, q.QDP_OPT_PDL, pdl)
            r = q.qdp_cg_solve(fx, fb, fU, fA, fAi, mass=0.1, tol=1e-30, maxit=12)
            out.setdefault(pdl, []).append((r["hist"].copy(), q.qdp_field_export(fx)))
        for hist, x in out[1] + out[0]:
            assert np.array_equal(hist, out[1][0][0]) and np.array_equal(x, out[1][0][1])
        hist, x = out[1][0]
        assert len(hist) == len(orc["hist"])
        assert np.max(np.abs(hist - orc["hist"]) / orc["hist"]) <= 1e-10
        assert rel_site_err(x, orc["x"]) <= 1e-10
    finally:
        q.qdp_finalize(c)


_WORKER = r"""
import sys
import numpy as np
sys.path.insert(0, {root!r}); sys.path.insert(0, {tests!r})
import fieldgen, oracle
from _physics import rel_site_err
from paper_1408_5925_b200 import qdpb as q
L = (4, 6, 4, 8)
U = fieldgen.random_gauge(L, 2101)
psi = fieldgen.random_spinor(L, 3101)
ref = oracle.hopping(U, psi, L, -1)
worst = 0.0
for mask in (8, 4, 12, 15):
    c = q.qdp_init(L)
    q.qdp_set_option(c, q.QDP_OPT_SELF_HALO, mask)
    q.qdp_set_option(c, q.QDP_OPT_P2P, 1)
    fU = q.qdp_field_alloc(c, q.QDP_GAUGE, 0, q.QDP_ALL); q.qdp_field_import(fU, U)
    fp = q.qdp_field_alloc(c, q.QDP_FERMION, 0, q.QDP_ALL); q.qdp_field_import(fp, psi)
    fo = q.qdp_field_alloc(c, q.QDP_FERMION, 0, q.QDP_ALL)
    for _ in range(4):
        q.qdp_dslash(fo, fU, fp, q.QDP_ALL)
        q.qdp_synchronize(c)
        worst = max(worst, rel_site_err(q.qdp_field_export(fo), ref))
    q.qdp_finalize(c)
print(worst)
sys.exit(0 if worst <= 1e-13 else 1)
"""


@pytest.mark.timeout(300)
@pytest.mark.parametrize("face_at", ["0", "1", "0.3"])
def test_fused_face_position(face_at):
    code = _WORKER.format(root=ROOT, tests=os.path.join(ROOT, "tests"))
    env = dict(os.environ, QDPB_FACE_AT=face_at)
    r = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True, timeout=280)
    assert r.returncode == 0, r.stdout + r.stderr
