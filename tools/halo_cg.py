"""CG it/s through the fused peer-to-peer boundary (self-halo) vs the whole lattice, for the bench's
weak-scaling rank volume (40^3 x 32 clover, t split) and config 5's rank sub-lattice (48x48x24x24 Wilson,
z x t): the on-GPU cost of the multi-GPU code path, interleaved rounds, median."""
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tools"))
from pdl_cg import its, q, setup  # noqa: E402

for L, clover, masks in (((40, 40, 40, 32), True, (0, 8)), ((48, 48, 24, 24), False, (0, 12))):
    ctx = {m: setup(L, clover, m) for m in masks}
    r = {m: [] for m in masks}
    for m in masks:
        its(*ctx[m], 32, 2)
    for _ in range(4):
        for m in masks:
            r[m].append(its(*ctx[m], 32, 2))
    base = statistics.median(r[0])
    print(f"{'x'.join(map(str, L))} {'clover' if clover else 'wilson'}: " + "  ".join(
        f"mask {m:2d} {statistics.median(r[m]):7.1f} it/s ({statistics.median(r[m]) / base:.3f})" for m in masks), flush=True)
    for m in masks:
        q.qdp_finalize(ctx[m][0])
