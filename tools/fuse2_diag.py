"""QDPB_FUSE=2 diagnostic: which output sites of the fused z x t boundary kernel are wrong."""
import os, sys
sys.path.insert(0, os.path.join(os.path.dirname(__file__), "..")); sys.path.insert(0, os.path.join(os.path.dirname(__file__), "..", "tests"))
import numpy as np
import fieldgen, oracle
from paper_1408_5925_b200 import qdpb as q

L = tuple(int(v) for v in (sys.argv[1] if len(sys.argv) > 1 else "4,6,4,8").split(","))
mask = int(sys.argv[2]) if len(sys.argv) > 2 else 12
U = fieldgen.random_gauge(L, 2101); psi = fieldgen.random_spinor(L, 3101)
ref = oracle.hopping(U, psi, L, -1)
c = q.qdp_init(L); q.qdp_set_option(c, q.QDP_OPT_SELF_HALO, mask); q.qdp_set_option(c, q.QDP_OPT_P2P, 1)
fU = q.qdp_field_alloc(c, q.QDP_GAUGE, 0, q.QDP_ALL); q.qdp_field_import(fU, U)
fp = q.qdp_field_alloc(c, q.QDP_FERMION, 0, q.QDP_ALL); q.qdp_field_import(fp, psi)
fo = q.qdp_field_alloc(c, q.QDP_FERMION, 0, q.QDP_ALL)
co = fieldgen.coords(L)
for it in range(3):
    q.qdp_dslash(fo, fU, fp, q.QDP_ALL); q.qdp_synchronize(c)
    got = q.qdp_field_export(fo)
    d = got - ref
    # is the error a missing/extra remote hop?  compare against the local-only sum
    err = np.linalg.norm(d.reshape(len(d), -1), axis=1) / np.linalg.norm(ref.reshape(len(ref), -1), axis=1)
    bad = np.nonzero(err > 1e-12)[0]
    print(f"call {it}: {len(bad)} bad sites of {len(err)}")
    from collections import Counter
    cnt = Counter()
    for s in bad:
        x = co[s]; par = int(x.sum()) & 1
        tag = ("z0" if x[2] == 0 else "zL" if x[2] == L[2]-1 else "") + ("t0" if x[3] == 0 else "tL" if x[3] == L[3]-1 else "")
        cnt[(par, tag or "int")] += 1
    print("  ", sorted(cnt.items()))
    tot = Counter()
    for s in range(len(err)):
        x = co[s]; par = int(x.sum()) & 1
        tag = ("z0" if x[2] == 0 else "zL" if x[2] == L[2]-1 else "") + ("t0" if x[3] == 0 else "tL" if x[3] == L[3]-1 else "")
        tot[(par, tag or "int")] += 1
    print("  all", sorted(tot.items()))
q.qdp_finalize(c)
