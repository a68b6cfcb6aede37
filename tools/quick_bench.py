"""Quick dslash timing (development aid): EO dslash at a given local volume, both precisions,
CUDA-event timed through the library's profiling option."""
import argparse
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402

import fieldgen  # noqa: E402
from paper_1408_5925_b200 import qdpb as q  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--dims", default="40,40,40,32")
ap.add_argument("--iters", type=int, default=50)
ap.add_argument("--block", type=int, default=0)
ap.add_argument("--self-halo", type=int, default=0)
ap.add_argument("--recon", type=int, default=18, choices=[12, 18])
args = ap.parse_args()
L = tuple(int(v) for v in args.dims.split(","))
V = fieldgen.volume(L)
t0 = time.time()
U = fieldgen.random_gauge(L, 1004)
psi = fieldgen.random_spinor(L, 2005)
print(f"gen {time.time() - t0:.1f}s", flush=True)
for prec in (0, 1):
    c = q.qdp_init(L)
    q.qdp_set_option(c, q.QDP_OPT_BLOCK, args.block)
    q.qdp_set_option(c, q.QDP_OPT_SELF_HALO, args.self_halo)
    fU = q.qdp_field_alloc(c, q.QDP_GAUGE12 if args.recon == 12 else q.QDP_GAUGE, prec, q.QDP_ALL)
    fp = q.qdp_field_alloc(c, q.QDP_FERMION, prec, 1)
    fo = q.qdp_field_alloc(c, q.QDP_FERMION, prec, 0)
    dt = np.float64 if prec == 0 else np.float32
    q.qdp_field_import(fU, U.astype(dt))
    q.qdp_field_import(fp, np.ascontiguousarray(psi[fieldgen.cb_sites(L, 1)], dtype=dt))
    for _ in range(5):
        q.qdp_dslash(fo, fU, fp, 0)
    q.qdp_synchronize(c)
    q.qdp_set_option(c, q.QDP_OPT_PROFILE, 1)
    q.qdp_profile_reset(c)
    for _ in range(args.iters):
        q.qdp_dslash(fo, fU, fp, 0)
    n, ms = q.qdp_profile_query(c, q.QDP_PK_DSLASH)
    us = ms / n * 1e3
    Vh = V // 2
    b = (8 * args.recon + 48) * (8 if prec == 0 else 4)
    print(f"prec {'f64' if prec == 0 else 'f32'} recon={args.recon} L={L} block={args.block}: {us:.1f} us/launch, "
          f"{Vh / us * 1e-3:.3f} Gsite/s, {1320 * Vh / us * 1e-3:.1f} GFLOPS, {b * Vh / us * 1e-3:.1f} GB/s compulsory",
          flush=True)
    q.qdp_finalize(c)
