"""Small single-GPU workloads for `ncu --set full` captures (tools/gpu_profile_r02.sh):
  zt     fp64 EO dslash at 40^3x32 with z and t through the peer-to-peer halo path (self-halo,
         the fused boundary kernel: pack + interior + remote hops in one kernel)
  t      the same with only t partitioned (the weak-scaling bench's split)
  h16    a few iterations of qdp_cg_solve_mixed16 (the 16-bit sloppy dslash launches)
  r12    fp64 reconstruct-12 plain EO dslash (tuned; r12main / r12pipe / r12tma: variant 1 / 4 / 3 forced)
  blas   norm2 / CG vector updates at 40^3x32
  cgblas the fp64 clover CG's vector updates at 40^3x32 (cg_r: r -= alpha q with |r|^2; cg_xp)
  c5zt / c5whole  plain fp64 EO dslash on config 5's rank sub-lattice 48x48x24x24: the fused z x t
         boundary kernel (self-halo) / the register-path main kernel without a halo
  t40cg / t40cg0  clover CG at 40^3x32 with t through the fused peer-to-peer halo path / without
  c5cg / c5cg0  Wilson CG on config 5's rank sub-lattice 48x48x24x24 with z x t through the fused
         peer-to-peer halo path (self-halo) / without a halo
Each case warms up, then runs the launches to capture (select them with ncu -k / -s / -c)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch

import fieldgen
from paper_1408_5925_b200 import qdpb as q

case = sys.argv[1]
L = (16, 16, 16, 32) if case == "blas16" else (48, 48, 24, 24) if case.startswith("c5") else (40, 40, 40, 32)
stream = torch.cuda.Stream()
torch.cuda.set_stream(stream)
c = q.qdp_init(L, stream=stream)
Ut = fieldgen.random_gauge_torch(L, 21)


def gauge(kind=q.QDP_GAUGE):
    f = q.qdp_field_alloc(c, kind, q.QDP_F64, q.QDP_ALL)
    q.qdp_field_import_device(f, Ut)
    return f


if case in ("zt", "t", "c5cg", "c5zt", "t40cg"):
    q.qdp_set_option(c, q.QDP_OPT_SELF_HALO, 8 if case in ("t", "t40cg") else 12)
    q.qdp_set_option(c, q.QDP_OPT_P2P, 1)
if case in ("r12tma", "r12pipe", "r12main"):  # fp64 reconstruct-12 dslash, one forced launch variant:
    # bulk-copy staged forward links / cp.async hop pipeline / the register-path main kernel
    q.qdp_set_option(c, q.QDP_OPT_DSLASH_VARIANT, {"r12tma": 3, "r12pipe": 4, "r12main": 1}[case])
    case = "r12"
if case == "c5whole":  # the register-path main kernel on the same sub-lattice, no halo
    q.qdp_set_option(c, q.QDP_OPT_DSLASH_VARIANT, 1)
if case in ("c5zt", "c5whole"):
    case = "zt"
if case in ("zt", "t", "r12"):
    fU = gauge(q.QDP_GAUGE12 if case == "r12" else q.QDP_GAUGE)
    fi = q.qdp_field_alloc(c, q.QDP_FERMION, q.QDP_F64, q.QDP_ODD)
    fo = q.qdp_field_alloc(c, q.QDP_FERMION, q.QDP_F64, q.QDP_EVEN)
    for _ in range(12):
        q.qdp_dslash(fo, fU, fi, q.QDP_EVEN)
    q.qdp_synchronize(c)
elif case == "h16":
    fU = gauge()
    fb = q.qdp_field_alloc(c, q.QDP_FERMION, q.QDP_F64, q.QDP_ALL)
    q.qdp_field_import_device(fb, fieldgen.random_spinor_torch(L, 22))
    fx = q.qdp_field_alloc(c, q.QDP_FERMION, q.QDP_F64, q.QDP_ALL)
    fA = q.qdp_field_alloc(c, q.QDP_CLOVER, q.QDP_F64, q.QDP_ALL)
    fAi = q.qdp_field_alloc(c, q.QDP_CLOVER, q.QDP_F64, q.QDP_EVEN)
    q.qdp_clover_build(fA, fAi, fU, 0.1, 1.0)
    q.qdp_cg_solve_mixed16(fx, fb, fU, fA, fAi, mass=0.1, tol=0.0, delta=0.1, maxit=6)
elif case in ("t40cg", "t40cg0"):
    fU = gauge()
    fb = q.qdp_field_alloc(c, q.QDP_FERMION, q.QDP_F64, q.QDP_ALL)
    q.qdp_field_import_device(fb, fieldgen.random_spinor_torch(L, 22))
    fx = q.qdp_field_alloc(c, q.QDP_FERMION, q.QDP_F64, q.QDP_ALL)
    fA = q.qdp_field_alloc(c, q.QDP_CLOVER, q.QDP_F64, q.QDP_ALL)
    fAi = q.qdp_field_alloc(c, q.QDP_CLOVER, q.QDP_F64, q.QDP_EVEN)
    q.qdp_clover_build(fA, fAi, fU, 0.1, 1.0)
    for _ in range(3):
        q.qdp_cg_solve(fx, fb, fU, fA, fAi, mass=0.1, tol=0.0, maxit=8)
elif case == "cgblas":
    fU = gauge()
    fb = q.qdp_field_alloc(c, q.QDP_FERMION, q.QDP_F64, q.QDP_ALL)
    q.qdp_field_import_device(fb, fieldgen.random_spinor_torch(L, 22))
    fx = q.qdp_field_alloc(c, q.QDP_FERMION, q.QDP_F64, q.QDP_ALL)
    fA = q.qdp_field_alloc(c, q.QDP_CLOVER, q.QDP_F64, q.QDP_ALL)
    fAi = q.qdp_field_alloc(c, q.QDP_CLOVER, q.QDP_F64, q.QDP_EVEN)
    q.qdp_clover_build(fA, fAi, fU, 0.1, 1.0)
    for _ in range(3):
        q.qdp_cg_solve(fx, fb, fU, fA, fAi, mass=0.1, tol=0.0, maxit=12)
elif case in ("c5cg", "c5cg0"):
    fU = gauge()
    fb = q.qdp_field_alloc(c, q.QDP_FERMION, q.QDP_F64, q.QDP_ALL)
    q.qdp_field_import_device(fb, fieldgen.random_spinor_torch(L, 22))
    fx = q.qdp_field_alloc(c, q.QDP_FERMION, q.QDP_F64, q.QDP_ALL)
    for _ in range(3):
        q.qdp_cg_solve(fx, fb, fU, mass=0.1, tol=0.0, maxit=8)
elif case in ("blas", "blas16"):
    a = q.qdp_field_alloc(c, q.QDP_FERMION, q.QDP_F64, q.QDP_ALL)
    q.qdp_field_import_device(a, fieldgen.random_spinor_torch(L, 23))
    b = q.qdp_field_alloc(c, q.QDP_FERMION, q.QDP_F64, q.QDP_ALL)
    for _ in range(30):
        q.qdp_norm2(a)
        q.qdp_inner_product(a, b)
        q.qdp_axpy(0.5, a, b)
q.qdp_synchronize(c)
q.qdp_finalize(c)
print("done", case)
