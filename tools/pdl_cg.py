"""CG iterations per second with and without programmatic dependent launch (QDP_OPT_PDL), at the
BASELINE volumes: config 2 (16^3 x 32), the weak-scaling rank volume (40^3 x 32), config 5's rank
sub-lattice through the z x t halo path (48 x 48 x 24 x 24, self-halo), fp64 clover / Wilson CG
with a fixed iteration count (tol = 0).  PDL off / on alternate over several rounds (the power
cap moves the clocks during a run), best of the rounds reported."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch

import fieldgen
from paper_1408_5925_b200 import qdpb as q

stream = torch.cuda.Stream()
torch.cuda.set_stream(stream)


def setup(L, clover, mask=0):
    c = q.qdp_init(L, stream=stream)
    if mask:
        q.qdp_set_option(c, q.QDP_OPT_SELF_HALO, mask)
        q.qdp_set_option(c, q.QDP_OPT_P2P, 1)
    fU = q.qdp_field_alloc(c, q.QDP_GAUGE, q.QDP_F64, q.QDP_ALL)
    q.qdp_field_import_device(fU, fieldgen.random_gauge_torch(L, 5))
    fb = q.qdp_field_alloc(c, q.QDP_FERMION, q.QDP_F64, q.QDP_ALL)
    fx = q.qdp_field_alloc(c, q.QDP_FERMION, q.QDP_F64, q.QDP_ALL)
    q.qdp_field_import(fb, fieldgen.random_spinor(L, 7))
    fA = fAi = None
    if clover:
        fA = q.qdp_field_alloc(c, q.QDP_CLOVER, q.QDP_F64, q.QDP_ALL)
        fAi = q.qdp_field_alloc(c, q.QDP_CLOVER, q.QDP_F64, q.QDP_EVEN)
        q.qdp_clover_build(fA, fAi, fU, 0.1, 1.0)
    return c, (fx, fb, fU, fA, fAi)


def its(c, f, iters, n):
    fx, fb, fU, fA, fAi = f
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record(stream)
    for _ in range(n):
        q.qdp_cg_solve(fx, fb, fU, fA, fAi, mass=0.1, tol=0.0, maxit=iters)
    e1.record(stream)
    torch.cuda.synchronize()
    return iters * n / (e0.elapsed_time(e1) * 1e-3)


if __name__ != "__main__":
    cases = []
else:
    cases = [((16, 16, 16, 32), True, 0, 64, 10), ((40, 40, 40, 32), True, 0, 32, 4),
             ((48, 48, 24, 24), False, 12, 32, 4), ((48, 48, 24, 24), False, 0, 32, 4)]
for L, clover, mask, iters, n in cases:
    c, f = setup(L, clover, mask)
    best = {0: 0.0, 1: 0.0}
    for pdl in (0, 1):  # warm-up (and the tuner's probes) in both modes
        q.qdp_set_option(c, q.QDP_OPT_PDL, pdl)
        its(c, f, iters, 2)
    for _ in range(4):
        for pdl in (0, 1):
            q.qdp_set_option(c, q.QDP_OPT_PDL, pdl)
            best[pdl] = max(best[pdl], its(c, f, iters, n))
    tag = f"{'x'.join(map(str, L))} {'clover' if clover else 'wilson'}{' self-halo z,t' if mask else ''}"
    print(f"{tag:>40}: CG it/s  PDL off {best[0]:8.1f}  on {best[1]:8.1f}  ({best[1] / best[0]:.3f}x)", flush=True)
    q.qdp_finalize(c)
