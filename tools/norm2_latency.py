"""norm2 latency from Python including the host readback, by lattice size (median of 400 calls), and
the floor: a no-op library call (ctypes) and a 2^4 lattice (the GPU work is negligible)."""
import os
import statistics
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_1408_5925_b200 import qdpb as q  # noqa: E402

for L in [(2, 2, 2, 2), (8, 8, 8, 8), (16, 16, 16, 32), (40, 40, 40, 32)]:
    c = q.qdp_init(L)
    f = q.qdp_field_alloc(c, q.QDP_FERMION, q.QDP_F64, q.QDP_EVEN)
    q.qdp_field_zero(f)
    for _ in range(50):
        q.qdp_norm2(f)
    t = []
    for _ in range(400):
        t0 = time.perf_counter()
        q.qdp_norm2(f)
        t.append(time.perf_counter() - t0)
    t2 = []
    for _ in range(400):
        t0 = time.perf_counter()
        q.qdp_get_option(c, q.QDP_OPT_PDL)
        t2.append(time.perf_counter() - t0)
    print(f"{'x'.join(map(str, L)):>12} one parity: norm2 median {statistics.median(t) * 1e6:6.2f} us  "
          f"(min {min(t) * 1e6:6.2f});  no-op call {statistics.median(t2) * 1e6:5.2f} us", flush=True)
    q.qdp_finalize(c)
