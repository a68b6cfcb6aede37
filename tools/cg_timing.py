"""Development aid: where does a CG iteration's time go?  Wall time of qdp_cg_solve vs the
sum of its kernels' event times, with and without per-launch profiling."""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import fieldgen  # noqa: E402
from paper_1408_5925_b200 import qdpb as q  # noqa: E402

L = tuple(int(v) for v in (sys.argv[1] if len(sys.argv) > 1 else "40,40,40,32").split(","))
clover = "--wilson" not in sys.argv
GK = q.QDP_GAUGE12 if "--recon12" in sys.argv else q.QDP_GAUGE
U = fieldgen.random_gauge(L, 1004)
b = fieldgen.random_spinor(L, 2005)
c = q.qdp_init(L)
fU = q.qdp_field_alloc(c, GK, 0, q.QDP_ALL)
fb = q.qdp_field_alloc(c, q.QDP_FERMION, 0, q.QDP_ALL)
fx = q.qdp_field_alloc(c, q.QDP_FERMION, 0, q.QDP_ALL)
q.qdp_field_import(fU, U)
q.qdp_field_import(fb, b)
fA = fAi = None
if clover:
    fA = q.qdp_field_alloc(c, q.QDP_CLOVER, 0, q.QDP_ALL)
    fAi = q.qdp_field_alloc(c, q.QDP_CLOVER, 0, q.QDP_EVEN)
    q.qdp_clover_build(fA, fAi, fU, 0.1, 1.0)
for it in (0, 8, 32):
    q.qdp_cg_solve(fx, fb, fU, fA, fAi, mass=0.1, tol=0, maxit=it)
for prof in (0, 1):
    q.qdp_set_option(c, q.QDP_OPT_PROFILE, prof)
    for it in (0, 8, 32):
        q.qdp_profile_reset(c)
        t0 = time.perf_counter()
        q.qdp_cg_solve(fx, fb, fU, fA, fAi, mass=0.1, tol=0, maxit=it)
        wall = (time.perf_counter() - t0) * 1e3
        n, ms = q.qdp_profile_query(c, -1)
        print(f"profile={prof} iters={it:3d}: wall {wall:8.2f} ms, {n} launches, kernel sum {ms:8.2f} ms", flush=True)
        if prof and it == 32:
            for k, name in enumerate(q.PK_NAMES):
                nk, mk = q.qdp_profile_query(c, k)
                if nk:
                    print(f"    {name:11s} {nk:5d} launches {mk:8.2f} ms  avg {mk / nk * 1e3:8.1f} us")
q.qdp_finalize(c)
