"""ncu driver (development aid): the generated hopping term (qdp_jit_eval) at 40^3x32 EO, 14 calls
(the paper's autotuner settles in the first ones; capture with ncu -s 12 -c 2), precision from argv."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402

import fieldgen  # noqa: E402
from paper_1408_5925_b200 import qdpb as q  # noqa: E402
from paper_1408_5925_b200.exprs import hopping  # noqa: E402

prec = int(sys.argv[1]) if len(sys.argv) > 1 else 0
L = (40, 40, 40, 32)
dt = np.float64 if prec == 0 else np.float32
U = fieldgen.random_gauge(L, 1004).astype(dt)
psi = fieldgen.random_spinor(L, 2005)
c = q.qdp_init(L)
fU = q.qdp_field_alloc(c, q.QDP_GAUGE, prec, q.QDP_ALL)
q.qdp_field_import(fU, U)
fo = q.qdp_field_alloc(c, q.QDP_FERMION, prec, 1)
q.qdp_field_import(fo, np.ascontiguousarray(psi[fieldgen.cb_sites(L, 1)], dtype=dt))
oe = q.qdp_field_alloc(c, q.QDP_FERMION, prec, 0)
for _ in range(14):
    q.qdp_jit_eval(oe, hopping(), fU, fo)
q.qdp_synchronize(c)
q.qdp_finalize(c)
