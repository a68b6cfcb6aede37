"""fp64 EO dslash (PLAIN) us per launch for the register-path kernel (variant 1) and the cp.async hop
pipeline (4: operands through L2; 5: spinors through L1, links evict-first; 6: spinors through L1), both
gauge storages, interleaved over rounds (best of 3) -- fraction of MEASURED_PEAKS hbm_gbs."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import fieldgen  # noqa: E402
from paper_1408_5925_b200 import qdpb as q  # noqa: E402

PEAK = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"]
stream = torch.cuda.Stream()
torch.cuda.set_stream(stream)


def eo_us(c, fU, prec, n=40):
    fi = q.qdp_field_alloc(c, q.QDP_FERMION, prec, q.QDP_ODD)
    fo = q.qdp_field_alloc(c, q.QDP_FERMION, prec, q.QDP_EVEN)
    for _ in range(5):
        q.qdp_dslash(fo, fU, fi, q.QDP_EVEN)
    q.qdp_synchronize(c)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(n):
        q.qdp_dslash(fo, fU, fi, q.QDP_EVEN)
    e1.record(stream)
    torch.cuda.synchronize()
    q.qdp_field_free(fi)
    q.qdp_field_free(fo)
    return e0.elapsed_time(e1) / n * 1e3

VARS = (1, 4)
print(f"# fp64 EO dslash us (frac of {PEAK} GB/s): variants " + ", ".join(map(str, VARS)))
for L in [(24, 24, 24, 32), (32, 32, 32, 32), (40, 40, 40, 32)]:
    Vh = L[0] * L[1] * L[2] * L[3] // 2
    Ut = fieldgen.random_gauge_torch(L, 11)
    for kind, rec in ((q.QDP_GAUGE, 18), (q.QDP_GAUGE12, 12)):
        c = q.qdp_init(L, stream=stream)
        fU = q.qdp_field_alloc(c, kind, q.QDP_F64, q.QDP_ALL)
        q.qdp_field_import_device(fU, Ut)
        best = {v: 1e30 for v in VARS}
        for _ in range(3):
            for v in VARS:
                q.qdp_set_option(c, q.QDP_OPT_DSLASH_VARIANT, v)
                best[v] = min(best[v], eo_us(c, fU, q.QDP_F64))
        bps = (8 * rec + 48) * 8
        print(f"{'x'.join(map(str, L)):>12} r{rec}: " + "  ".join(
            f"v{v} {best[v]:7.2f} ({bps * Vh / (best[v] * 1e-6) * 1e-9 / PEAK:.3f})" for v in VARS), flush=True)
        q.qdp_finalize(c)
    del Ut
