"""Config 5's rank sub-lattice (48x48x24x24, Wilson CG, fp64): per-class kernel times per CG iteration
with no halo and with z x t through the fused peer-to-peer halo path (self-halo), marginal it/s."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch

import fieldgen
from paper_1408_5925_b200 import qdpb as q

L = (48, 48, 24, 24)
stream = torch.cuda.Stream()
torch.cuda.set_stream(stream)
Ut = fieldgen.random_gauge_torch(L, 41)
bt = fieldgen.random_spinor_torch(L, 42)
for mask in (0, 8, 12):
    c = q.qdp_init(L, stream=stream)
    if mask:
        q.qdp_set_option(c, q.QDP_OPT_SELF_HALO, mask)
        q.qdp_set_option(c, q.QDP_OPT_P2P, 1)
    fU = q.qdp_field_alloc(c, q.QDP_GAUGE, q.QDP_F64, q.QDP_ALL)
    q.qdp_field_import_device(fU, Ut)
    fb = q.qdp_field_alloc(c, q.QDP_FERMION, q.QDP_F64, q.QDP_ALL)
    q.qdp_field_import_device(fb, bt)
    fx = q.qdp_field_alloc(c, q.QDP_FERMION, q.QDP_F64, q.QDP_ALL)
    res = {}
    for n in (16, 32):
        for _ in range(2):
            q.qdp_cg_solve(fx, fb, fU, mass=0.1, tol=0.0, maxit=n)
        q.qdp_synchronize(c)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(3):
            q.qdp_cg_solve(fx, fb, fU, mass=0.1, tol=0.0, maxit=n)
        e1.record(stream)
        torch.cuda.synchronize()
        res[n] = e0.elapsed_time(e1) / 3
    it_s = 16 / ((res[32] - res[16]) * 1e-3)
    q.qdp_profile_reset(c)
    q.qdp_set_option(c, q.QDP_OPT_PROFILE, 1)
    q.qdp_cg_solve(fx, fb, fU, mass=0.1, tol=0.0, maxit=32)
    parts = []
    for cn, cl in (("dslash", q.QDP_PK_DSLASH), ("blas", q.QDP_PK_BLAS), ("reduce", q.QDP_PK_REDUCE)):
        nl, ms = q.qdp_profile_query(c, cl)
        if nl:
            parts.append(f"{cn} {nl} x {ms / nl * 1e3:.1f} us")
    q.qdp_set_option(c, q.QDP_OPT_PROFILE, 0)
    print(f"mask {mask:2d}: {it_s:7.1f} it/s ({1e3 / it_s:.3f} ms/it) | " + " | ".join(parts), flush=True)
    q.qdp_finalize(c)
