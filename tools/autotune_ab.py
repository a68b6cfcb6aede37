"""CG it/s with the paper's autotuner on (tuned launch configurations) vs off (128-thread BLAS, the main dslash kernel)."""
import os, sys, statistics
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__))); sys.path.insert(0, ROOT); sys.path.insert(0, os.path.join(ROOT, "tools"))
from pdl_cg import its, q, setup
for L, clover in (((40, 40, 40, 32), True), ((48, 48, 24, 24), False)):
    c, f = setup(L, clover, 0)
    r = {0: [], 1: []}
    for at in (1, 0):
        q.qdp_set_option(c, q.QDP_OPT_AUTOTUNE, at); its(c, f, 32, 3)
    for _ in range(4):
        for at in (1, 0):
            q.qdp_set_option(c, q.QDP_OPT_AUTOTUNE, at); r[at].append(its(c, f, 32, 2))
    print(L, clover, "tuned", statistics.median(r[1]), "untuned(128, main kernel)", statistics.median(r[0]), flush=True)
    q.qdp_finalize(c)
