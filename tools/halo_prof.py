import sys, os
sys.path.insert(0, os.getcwd())
import numpy as np, fieldgen
from paper_1408_5925_b200 import qdpb as q
L=(40,40,40,32)
U=fieldgen.random_gauge(L,1004); psi=fieldgen.random_spinor(L,2005)
for mode in ("whole","p2p"):
    c=q.qdp_init(L)
    if mode=="p2p":
        q.qdp_set_option(c,q.QDP_OPT_SELF_HALO,8); q.qdp_set_option(c,q.QDP_OPT_P2P,1)
    fU=q.qdp_field_alloc(c,q.QDP_GAUGE,0,-1); q.qdp_field_import(fU,U)
    fp=q.qdp_field_alloc(c,q.QDP_FERMION,0,1); q.qdp_field_import(fp,np.ascontiguousarray(psi[fieldgen.cb_sites(L,1)]))
    fo=q.qdp_field_alloc(c,q.QDP_FERMION,0,0)
    for _ in range(5): q.qdp_dslash(fo,fU,fp,0)
    q.qdp_synchronize(c); q.qdp_set_option(c,q.QDP_OPT_PROFILE,1); q.qdp_profile_reset(c)
    for _ in range(30): q.qdp_dslash(fo,fU,fp,0)
    out=[]
    for k,name in enumerate(q.PK_NAMES):
        n,ms=q.qdp_profile_query(c,k)
        if n: out.append(f"{name} {ms/n*1e3:.1f}us x{n//30}")
    print(mode, os.environ.get("QDPB_FUSE","1"), " | ".join(out), flush=True)
    q.qdp_finalize(c)
