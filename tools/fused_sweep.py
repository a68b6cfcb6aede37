"""Cost of the fused peer-to-peer boundary kernel on one GPU (self-halo: the whole protocol with
this rank as its own neighbour): fp64 EO dslash us per launch for the whole lattice (no halo), the
t split and the z x t split (fused, and with QDP_OPT_FUSE = 0), at the weak-scaling local volume
and at config 5's rank sub-lattice.  QDPB_PACK_BLOCKS (env) sets the cap on packing blocks."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch

import fieldgen
from paper_1408_5925_b200 import qdpb as q

stream = torch.cuda.Stream()
torch.cuda.set_stream(stream)


def eo_us(L, mask, fuse=1, n=40):
    c = q.qdp_init(L, stream=stream)
    if mask:
        q.qdp_set_option(c, q.QDP_OPT_SELF_HALO, mask)
        q.qdp_set_option(c, q.QDP_OPT_P2P, 1)
        q.qdp_set_option(c, q.QDP_OPT_FUSE, fuse)
    fU = q.qdp_field_alloc(c, q.QDP_GAUGE, q.QDP_F64, q.QDP_ALL)
    q.qdp_field_import_device(fU, fieldgen.random_gauge_torch(L, 5))
    fi = q.qdp_field_alloc(c, q.QDP_FERMION, q.QDP_F64, q.QDP_ODD)
    fo = q.qdp_field_alloc(c, q.QDP_FERMION, q.QDP_F64, q.QDP_EVEN)
    for _ in range(10):
        q.qdp_dslash(fo, fU, fi, q.QDP_EVEN)
    q.qdp_synchronize(c)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(n):
        q.qdp_dslash(fo, fU, fi, q.QDP_EVEN)
    e1.record(stream)
    torch.cuda.synchronize()
    q.qdp_synchronize(c)
    q.qdp_finalize(c)
    return e0.elapsed_time(e1) / n * 1e3


pb = os.environ.get("QDPB_PACK_BLOCKS", "default(296)")
for L in [(40, 40, 40, 32), (48, 48, 24, 24)]:
    r = [eo_us(L, 0), eo_us(L, 8), eo_us(L, 12), eo_us(L, 12, fuse=0)]
    print(f"{'x'.join(map(str, L)):>12} pack_blocks={pb:>12}: whole {r[0]:7.1f}  t-fused {r[1]:7.1f}  "
          f"zt-fused {r[2]:7.1f}  zt-separate {r[3]:7.1f} us", flush=True)
