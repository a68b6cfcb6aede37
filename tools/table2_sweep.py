"""B200 analogue of the paper's Figs. 4/5: sustained bandwidth of the
Table II test functions vs the local volume, fp32 and fp64, with the paper's block-size
autotuner.  Bandwidth uses the paper's byte convention (every leaf load + the store; matvec
counts U1 twice) and, beside it, the compulsory bytes; fractions are of the measured HBM copy
bandwidth (MEASURED_PEAKS.json).  Inputs are synthetic (timing does not depend on values)."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402

from paper_1408_5925_b200 import qdpb as q  # noqa: E402

peak = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"] if os.path.exists(
    os.path.join(ROOT, "MEASURED_PEAKS.json")) else 6650.0
# (expr, out kind, a kind, b kind, c kind, paper reals/site, compulsory reals/site)
EXPRS = {
    "lcm": (q.QDP_EXPR_LCM, q.QDP_COLORMATRIX, q.QDP_COLORMATRIX, q.QDP_COLORMATRIX, None, 54, 54),
    "upsi": (q.QDP_EXPR_UPSI, q.QDP_FERMION, q.QDP_COLORMATRIX, q.QDP_FERMION, None, 66, 66),
    "spmat": (q.QDP_EXPR_SPMAT, q.QDP_SPINMATRIX, q.QDP_SPINMATRIX, q.QDP_SPINMATRIX, None, 96, 96),
    "matvec": (q.QDP_EXPR_MATVEC, q.QDP_FERMION, q.QDP_COLORMATRIX, q.QDP_FERMION, q.QDP_FERMION, 108, 90),
    "clover": (q.QDP_EXPR_CLOVER, q.QDP_FERMION, q.QDP_CLOVER, q.QDP_FERMION, None, 120, 120),
}
dims = [(4, 4, 4, 4), (6, 6, 6, 6), (8, 8, 8, 8), (10, 10, 10, 10), (12, 12, 12, 12), (16, 16, 16, 16),
        (20, 20, 20, 20), (24, 24, 24, 24), (32, 32, 32, 32), (40, 40, 40, 40)]
print(f"# measured HBM peak {peak} GB/s; bandwidth = paper-convention bytes / kernel time (compulsory in brackets)")
print(f"# {'V':>12} {'prec':>4} " + " ".join(f"{n:>22}" for n in EXPRS))
for L in dims:
    V = int(np.prod(L))
    for prec in (1, 0):
        c = q.qdp_init(L)
        isz = 8 if prec == 0 else 4
        row = []
        for name, (e, ko, ka, kb, kc, paper_r, comp_r) in EXPRS.items():
            # rotate through enough operand sets that consecutive launches cannot hit the 126 MB L2
            set_bytes = comp_r * isz * V
            nsets = int(min(64, max(1, np.ceil(3 * 126e6 / set_bytes))))
            sets = [[q.qdp_field_alloc(c, k, prec, q.QDP_ALL) if k is not None else None for k in (ko, ka, kb, kc)]
                    for _ in range(nsets)]
            for i in range(12):  # autotune on the payload launches
                q.qdp_expr(e, *sets[i % nsets])
            q.qdp_synchronize(c)
            q.qdp_set_option(c, q.QDP_OPT_PROFILE, 1)
            q.qdp_profile_reset(c)
            n = max(30, 2 * nsets) if V < 1e6 else 10
            for i in range(n):
                q.qdp_expr(e, *sets[i % nsets])
            nl, ms = q.qdp_profile_query(c, q.QDP_PK_BLAS)
            q.qdp_set_option(c, q.QDP_OPT_PROFILE, 0)
            t = ms / nl * 1e-3
            gbs = paper_r * isz * V / t * 1e-9
            blk, _ = q.qdp_expr_block(c, e, prec)
            row.append(f"{gbs:7.0f} ({100 * gbs / peak:3.0f}%) b{blk:<4d}")
            for fs in sets:
                for f in fs:
                    if f is not None:
                        q.qdp_field_free(f)
        q.qdp_finalize(c)
        print(f"  {'x'.join(map(str, L)):>12} {'f64' if prec == 0 else 'f32':>4} " + " ".join(f"{r:>22}" for r in row),
              flush=True)
