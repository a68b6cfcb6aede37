"""Config 5's rank sub-lattice (48 x 48 x 24 x 24) through the z x t self-halo path: Wilson CG it/s
with PDL off / on, interleaved over many rounds (median and best).  Run under QDPB_PDL_HALO=0 to
launch the fused boundary kernel without PDL (the other solver kernels keep it)."""
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tools"))
from pdl_cg import its, q, setup  # noqa: E402

for mask in (12, 0):
    c, f = setup((48, 48, 24, 24), False, mask)
    r = {0: [], 1: []}
    for pdl in (0, 1):
        q.qdp_set_option(c, q.QDP_OPT_PDL, pdl)
        its(c, f, 32, 2)
    for _ in range(8):
        for pdl in (0, 1):
            q.qdp_set_option(c, q.QDP_OPT_PDL, pdl)
            r[pdl].append(its(c, f, 32, 3))
    print(f"mask {mask:2d} PDL_HALO={os.environ.get('QDPB_PDL_HALO', '1')}: it/s PDL off median {statistics.median(r[0]):7.1f} "
          f"best {max(r[0]):7.1f} | on median {statistics.median(r[1]):7.1f} best {max(r[1]):7.1f}", flush=True)
    q.qdp_finalize(c)
