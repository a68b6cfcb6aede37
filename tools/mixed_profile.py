"""Where the time of the mixed-precision solvers goes (40^3 x 32 clover, fixed iterations, tol = 0):
live per-class kernel times (QDP_OPT_PROFILE) for fp64 CG, the fp32 and the 16-bit sloppy levels."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch

import fieldgen
from paper_1408_5925_b200 import qdpb as q

L = (40, 40, 40, 32)
Vh = L[0] * L[1] * L[2] * L[3] // 2
stream = torch.cuda.Stream()
torch.cuda.set_stream(stream)
c = q.qdp_init(L, stream=stream)
Ut = fieldgen.random_gauge_torch(L, 31)
fU = q.qdp_field_alloc(c, q.QDP_GAUGE, q.QDP_F64, q.QDP_ALL)
q.qdp_field_import_device(fU, Ut)
fU32 = q.qdp_field_alloc(c, q.QDP_GAUGE12, q.QDP_F32, q.QDP_ALL)
q.qdp_field_import_device(fU32, Ut.float())
fb = q.qdp_field_alloc(c, q.QDP_FERMION, q.QDP_F64, q.QDP_ALL)
q.qdp_field_import_device(fb, fieldgen.random_spinor_torch(L, 32))
fx = q.qdp_field_alloc(c, q.QDP_FERMION, q.QDP_F64, q.QDP_ALL)
fA = q.qdp_field_alloc(c, q.QDP_CLOVER, q.QDP_F64, q.QDP_ALL)
fAi = q.qdp_field_alloc(c, q.QDP_CLOVER, q.QDP_F64, q.QDP_EVEN)
q.qdp_clover_build(fA, fAi, fU, 0.1, 1.0)
fA32 = q.qdp_field_alloc(c, q.QDP_CLOVER, q.QDP_F32, q.QDP_ODD)
fAi32 = q.qdp_field_alloc(c, q.QDP_CLOVER, q.QDP_F32, q.QDP_EVEN)
q.qdp_clover_build(fA32, fAi32, fU32, 0.1, 1.0)
N = 40
solvers = {
    "fp64": lambda: q.qdp_cg_solve(fx, fb, fU, fA, fAi, mass=0.1, tol=0.0, maxit=N),
    "mixed_fp32_r12": lambda: q.qdp_cg_solve_mixed(fx, fb, fU, fA, fAi, fU32, fA32, fAi32, mass=0.1, tol=0.0,
                                                   delta=1e-30, maxit=N),
    "mixed_h16": lambda: q.qdp_cg_solve_mixed16(fx, fb, fU, fA, fAi, mass=0.1, tol=0.0, delta=1e-30, maxit=N),
}
classes = [("dslash", q.QDP_PK_DSLASH), ("blas", q.QDP_PK_BLAS), ("reduce", q.QDP_PK_REDUCE),
           ("clover", q.QDP_PK_CLOVER), ("layout", q.QDP_PK_LAYOUT)]
print(f"# {N} iterations, delta -> 0 (one reliable update at the end); per class: launches, ms, GB/s")
for name, fn in solvers.items():
    fn()
    q.qdp_synchronize(c)
    q.qdp_profile_reset(c)
    q.qdp_set_option(c, q.QDP_OPT_PROFILE, 1)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    fn()
    e1.record(stream)
    torch.cuda.synchronize()
    tot = e0.elapsed_time(e1)
    parts = []
    for cn, cl in classes:
        n, ms = q.qdp_profile_query(c, cl)
        _, b = q.qdp_profile_work(c, cl)
        if n:
            parts.append(f"{cn} {n} {ms:.2f} ms {b / (ms * 1e-3) * 1e-9:.0f} GB/s")
    q.qdp_set_option(c, q.QDP_OPT_PROFILE, 0)
    print(f"{name:>16}: {tot:8.2f} ms ({tot / N:.3f} ms/it) | " + " | ".join(parts), flush=True)
q.qdp_finalize(c)
