"""shift() bandwidth (bytes = read + write of one field) at 40^3 x 32:
fermion (full and checkerboard) and gauge fields, every mu and direction, fp64 and fp32."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_1408_5925_b200 import qdpb as q  # noqa: E402

peak = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"] if os.path.exists(
    os.path.join(ROOT, "MEASURED_PEAKS.json")) else 6650.0
L = (40, 40, 40, 32)
for prec in (0, 1):
    c = q.qdp_init(L)
    for kind, sub_in, sub_out, name in ((q.QDP_FERMION, -1, -1, "fermion ALL"), (q.QDP_FERMION, 1, 0, "fermion odd->even"),
                                        (q.QDP_GAUGE, -1, -1, "gauge")):
        fi = q.qdp_field_alloc(c, kind, prec, sub_in)
        fo = q.qdp_field_alloc(c, kind, prec, sub_out)
        row = []
        for mu in range(4):
            for sign in (1, -1):
                q.qdp_shift(fo, fi, mu, sign)
                q.qdp_synchronize(c)
                q.qdp_profile_reset(c)
                q.qdp_set_option(c, q.QDP_OPT_PROFILE, 1)
                for _ in range(10):
                    q.qdp_shift(fo, fi, mu, sign)
                n, ms = q.qdp_profile_query(c, q.QDP_PK_SHIFT)
                _, nbytes = q.qdp_profile_work(c, q.QDP_PK_SHIFT)
                q.qdp_set_option(c, q.QDP_OPT_PROFILE, 0)
                row.append(nbytes / (ms * 1e-3) * 1e-9)
        q.qdp_field_free(fi)
        q.qdp_field_free(fo)
        print(f"{'f64' if prec == 0 else 'f32'} {name:18s} GB/s per (mu,sign): " + " ".join(f"{v:6.0f}" for v in row) +
              f"   mean {sum(row) / len(row):6.0f} = {100 * sum(row) / len(row) / peak:4.1f}% of measured HBM", flush=True)
    q.qdp_finalize(c)
