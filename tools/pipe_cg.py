"""fp64 clover CG at 40^3 x 32 (32 iterations, tol = 0) with the non-fused dslash launches (the A^-1 and
A x + b D epilogues) forced to the register-path kernel (variant 1) or the cp.async hop pipeline (4),
and tuned; 18- and 12-real links.  Interleaved rounds, best of 4: CG it/s and the dslash class's
live GB/s (per-launch events)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tools"))
from pdl_cg import its, q  # noqa: E402
import fieldgen  # noqa: E402
from pdl_cg import stream  # noqa: E402

L = (40, 40, 40, 32)
for kind, rec in ((q.QDP_GAUGE, 18), (q.QDP_GAUGE12, 12)):
    c = q.qdp_init(L, stream=stream)
    fU = q.qdp_field_alloc(c, kind, q.QDP_F64, q.QDP_ALL)
    q.qdp_field_import_device(fU, fieldgen.random_gauge_torch(L, 5))
    fb = q.qdp_field_alloc(c, q.QDP_FERMION, q.QDP_F64, q.QDP_ALL)
    q.qdp_field_import(fb, fieldgen.random_spinor(L, 7))
    fx = q.qdp_field_alloc(c, q.QDP_FERMION, q.QDP_F64, q.QDP_ALL)
    fA = q.qdp_field_alloc(c, q.QDP_CLOVER, q.QDP_F64, q.QDP_ALL)
    fAi = q.qdp_field_alloc(c, q.QDP_CLOVER, q.QDP_F64, q.QDP_EVEN)
    q.qdp_clover_build(fA, fAi, fU, 0.1, 1.0)
    f = (fx, fb, fU, fA, fAi)
    best = {}
    for v in (1, 4, -1):
        q.qdp_set_option(c, q.QDP_OPT_DSLASH_VARIANT, v)
        its(c, f, 32, 2)
    for _ in range(4):
        for v in (1, 4, -1):
            q.qdp_set_option(c, q.QDP_OPT_DSLASH_VARIANT, v)
            best[v] = max(best.get(v, 0.0), its(c, f, 32, 2))
    gbs = {}
    for v in (1, 4):
        q.qdp_set_option(c, q.QDP_OPT_DSLASH_VARIANT, v)
        q.qdp_profile_reset(c)
        q.qdp_set_option(c, q.QDP_OPT_PROFILE, 1)
        its(c, f, 32, 1)
        n, ms = q.qdp_profile_query(c, q.QDP_PK_DSLASH)
        _, by = q.qdp_profile_work(c, q.QDP_PK_DSLASH)
        q.qdp_set_option(c, q.QDP_OPT_PROFILE, 0)
        gbs[v] = by / (ms * 1e-3) * 1e-9
    print(f"r{rec}: CG it/s  v1 {best[1]:7.1f} (dslash {gbs[1]:6.0f} GB/s)  v4 {best[4]:7.1f} (dslash {gbs[4]:6.0f} GB/s)"
          f"  tuned {best[-1]:7.1f}", flush=True)
    q.qdp_finalize(c)
