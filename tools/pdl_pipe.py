"""Wilson CG it/s on config 5's rank sub-lattice (48x48x24x24, no halo) with the plain / xpay dslash
launches forced to the main kernel (variant 1) or the hop pipeline (4), PDL off / on, and tuned:
interleaved rounds, median."""
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tools"))
from pdl_cg import its, q, setup  # noqa: E402

L = tuple(int(v) for v in (sys.argv[1] if len(sys.argv) > 1 else "48,48,24,24").split(","))
c, f = setup(L, False, 0)
combos = [(v, pdl) for v in (1, 4, -1) for pdl in (0, 1)]
r = {k: [] for k in combos}
for v, pdl in combos:
    q.qdp_set_option(c, q.QDP_OPT_DSLASH_VARIANT, v)
    q.qdp_set_option(c, q.QDP_OPT_PDL, pdl)
    its(c, f, 32, 2)
for _ in range(5):
    for v, pdl in combos:
        q.qdp_set_option(c, q.QDP_OPT_DSLASH_VARIANT, v)
        q.qdp_set_option(c, q.QDP_OPT_PDL, pdl)
        r[(v, pdl)].append(its(c, f, 32, 2))
for (v, pdl), x in r.items():
    print(f"{'x'.join(map(str, L))} wilson  variant {v:2d}  PDL {pdl}: CG it/s median {statistics.median(x):7.1f}  best {max(x):7.1f}", flush=True)
q.qdp_finalize(c)
