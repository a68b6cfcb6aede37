"""Cost of the multi-GPU code path on one GPU (development aid for DESIGN.md section 9):
EO dslash and a 32-iteration clover CG at 40^3 x 32 with the t (and z) neighbours reached
through the halo path -- faces written directly (self), through NCCL send/recv to self, or by
the peer-to-peer flag protocol -- against the whole-lattice kernel."""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import fieldgen  # noqa: E402
from paper_1408_5925_b200 import qdpb as q  # noqa: E402

L = (40, 40, 40, 32)
U = fieldgen.random_gauge(L, 1004)
b = fieldgen.random_spinor(L, 2005)
modes = [("whole lattice", 0, 0, 0, 1), ("t halo: direct", 8, 0, 0, 1), ("t halo: NCCL overlap", 8, 1, 0, 1),
         ("t halo: NCCL no-overlap", 8, 1, 0, 0), ("t halo: P2P flags", 8, 0, 1, 1), ("zt halo: direct", 12, 0, 0, 1),
         ("zt halo: NCCL overlap", 12, 1, 0, 1), ("zt halo: P2P flags", 12, 0, 1, 1)]
for name, mask, nccl, p2p, overlap in modes:
    c = q.qdp_init(L)
    q.qdp_set_option(c, q.QDP_OPT_SELF_HALO, mask)
    if nccl:
        q.qdp_set_option(c, q.QDP_OPT_SELF_NCCL, 1)
    q.qdp_set_option(c, q.QDP_OPT_P2P, p2p)
    q.qdp_set_option(c, q.QDP_OPT_OVERLAP, overlap)
    fU = q.qdp_field_alloc(c, q.QDP_GAUGE, 0, q.QDP_ALL)
    fb = q.qdp_field_alloc(c, q.QDP_FERMION, 0, q.QDP_ALL)
    fx = q.qdp_field_alloc(c, q.QDP_FERMION, 0, q.QDP_ALL)
    fA = q.qdp_field_alloc(c, q.QDP_CLOVER, 0, q.QDP_ALL)
    fAi = q.qdp_field_alloc(c, q.QDP_CLOVER, 0, q.QDP_EVEN)
    q.qdp_field_import(fU, U)
    q.qdp_field_import(fb, b)
    q.qdp_clover_build(fA, fAi, fU, 0.1, 1.0)
    for _ in range(5):
        q.qdp_dslash(fx, fU, fb, q.QDP_ALL)
    q.qdp_synchronize(c)
    t0 = time.perf_counter()
    n = 40
    for _ in range(n):
        q.qdp_dslash(fx, fU, fb, q.QDP_ALL)
    q.qdp_synchronize(c)
    us = (time.perf_counter() - t0) / (2 * n) * 1e6
    q.qdp_cg_solve(fx, fb, fU, fA, fAi, mass=0.1, tol=0.0, maxit=32)
    t0 = time.perf_counter()
    res = q.qdp_cg_solve(fx, fb, fU, fA, fAi, mass=0.1, tol=0.0, maxit=32)
    ms = (time.perf_counter() - t0) * 1e3
    print(f"{name:26s} EO dslash {us:7.1f} us (wall, incl. pack/exchange/exterior)   CG(32 it) {ms:7.2f} ms  "
          f"hist[-1] {res['hist'][-1]:.6e}", flush=True)
    q.qdp_finalize(c)
