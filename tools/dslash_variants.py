"""Launch-variant sweep of the whole-lattice EO dslash (QDP_OPT_DSLASH_VARIANT) over local volumes
below and above the bandwidth shoulder, both precisions and gauge storages,
plus what the tuner picks and norm2 latency including the host readback.
Usage (GPU): python tools/dslash_variants.py > profiles/rNN_dslash_variants.txt"""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import json

import numpy as np
import torch

import fieldgen
from paper_1408_5925_b200 import qdpb as q

PEAK = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"]
torch.cuda.init()
stream = torch.cuda.Stream()
torch.cuda.set_stream(stream)


def eo_us(c, fU, prec, n=50):
    fi = q.qdp_field_alloc(c, q.QDP_FERMION, prec, q.QDP_ODD)
    fo = q.qdp_field_alloc(c, q.QDP_FERMION, prec, q.QDP_EVEN)
    for _ in range(12):  # the tuner reads its probes' events without waiting: let them complete
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


print(f"# EO dslash (PLAIN) us per launch and fraction of measured HBM ({PEAK} GB/s); variants: "
      "0 = four threads per site, 1 = one thread per site / 64-thread blocks, 2 = one / 32, "
      "3 = forward links staged by the bulk-copy engine (fp64 r12 only), 4 = cp.async hop pipeline, two stages (fp64 only); "
      "5 = one thread per site at 128 registers (8 x 64 threads per SM); rows where a variant does not apply repeat variant 1; tuned = the autotuner")
print(f"{'lattice':>14} {'prec':>4} {'rec':>3} | {'v0 us':>8} {'frac':>5} | {'v1 us':>8} {'frac':>5} | "
      f"{'v2 us':>8} {'frac':>5} | {'v3 us':>8} {'frac':>5} | {'v4 us':>8} {'frac':>5} | {'v5 us':>8} {'frac':>5} | "
      f"{'tuned':>8} {'frac':>5}")
for L in [(8, 8, 8, 16), (16, 16, 16, 16), (16, 16, 16, 32), (24, 24, 24, 32), (32, 32, 32, 32), (40, 40, 40, 32)]:
    Vh = L[0] * L[1] * L[2] * L[3] // 2
    Ut = fieldgen.random_gauge_torch(L, 11)
    for prec in (q.QDP_F64, q.QDP_F32):
        for kind, rec in ((q.QDP_GAUGE, 18), (q.QDP_GAUGE12, 12)):
            c = q.qdp_init(L, stream=stream)
            fU = q.qdp_field_alloc(c, kind, prec, q.QDP_ALL)
            q.qdp_field_import_device(fU, Ut if prec == q.QDP_F64 else Ut.float())
            bps = (8 * rec + 48) * (8 if prec == q.QDP_F64 else 4)
            row = []
            for v in (0, 1, 2, 3, 4, 5, -1):
                q.qdp_set_option(c, q.QDP_OPT_DSLASH_VARIANT, v)
                us = eo_us(c, fU, prec)
                row.append((us, bps * Vh / (us * 1e-6) * 1e-9 / PEAK))
            q.qdp_field_free(fU)
            q.qdp_finalize(c)
            print(f"{'x'.join(map(str, L)):>14} {'f64' if prec == 0 else 'f32':>4} {rec:>3} | " +
                  " | ".join(f"{u:8.2f} {f:5.3f}" for u, f in row), flush=True)
    del Ut

print("\n# norm2 (one launch, result in mapped host memory) incl. host readback: wall us per call;"
      " kernel = CUDA-event time of the launch; ctypes = wall time of a no-op library call (qdp_get_option)")
for L in [(16, 16, 16, 32), (40, 40, 40, 32)]:
    c = q.qdp_init(L, stream=stream)
    f = q.qdp_field_alloc(c, q.QDP_FERMION, q.QDP_F64, q.QDP_ALL)
    q.qdp_field_import_device(f, fieldgen.random_spinor_torch(L, 3))
    for _ in range(20):
        q.qdp_norm2(f)
    n = 200
    t0 = time.perf_counter()
    for _ in range(n):
        q.qdp_norm2(f)
    t = (time.perf_counter() - t0) / n
    fe = q.qdp_field_alloc(c, q.QDP_FERMION, q.QDP_F64, q.QDP_EVEN)
    t0 = time.perf_counter()
    for _ in range(n):
        q.qdp_norm2(fe)
    te = (time.perf_counter() - t0) / n
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    q.qdp_synchronize(c)
    e0.record(stream)
    for _ in range(n):
        q.qdp_norm2(fe)
    e1.record(stream)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(n):
        q.qdp_get_option(c, q.QDP_OPT_OVERLAP)
    tc = (time.perf_counter() - t0) / n
    print(f"{'x'.join(map(str, L)):>14}: full field {t * 1e6:8.2f} us   one parity {te * 1e6:8.2f} us   "
          f"(one parity, stream time per call {e0.elapsed_time(e1) / n * 1e3:6.2f} us; ctypes no-op {tc * 1e6:5.2f} us)")
    q.qdp_finalize(c)
