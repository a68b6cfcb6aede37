"""Generated vs hand-written kernels on one B200 (the paper's own comparison, PAPER.md:292:
QDP-JIT's generated hopping term against QUDA's hand-tuned one on the same hardware).

  * the hopping term of PAPER.md:282 written as a site expression (tests/test_gpu_jit.py's
    hopping_expr) and generated at run time by qdp_jit_eval, against the fused hand-written
    qdp_dslash: EO application at 40^3x32, fp64 / fp32, 18- and 12-real links;
  * the Table II functions (lcm, upsi, spmat, matvec) generated from "$0*$1"-style expressions,
    against the hand-written qdp_expr kernels, at 32^4;
  * the generate + NVRTC compile + load time of each kernel (the paper: 0.05-0.22 s).

Bandwidth = compulsory bytes per output site (the library's work counters) / CUDA-event time.
"""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import fieldgen  # noqa: E402
from paper_1408_5925_b200 import qdpb as q  # noqa: E402
from paper_1408_5925_b200.exprs import hopping as hopping_expr  # noqa: E402  (grouped: spin-projected)


def timed(stream, fn, n=30, warm=5):
    for _ in range(warm):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(n):
        fn()
    e1.record(stream)
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / n * 1e3


def main():
    stream = torch.cuda.Stream()
    torch.cuda.set_stream(stream)
    print(f"# {torch.cuda.get_device_name()}  ({time.strftime('%Y-%m-%d %H:%M:%S')})", flush=True)
    L = (40, 40, 40, 32)
    U = fieldgen.random_gauge(L, 1004)
    psi = fieldgen.random_spinor(L, 2005)
    odd = fieldgen.cb_sites(L, 1)
    Vh = fieldgen.volume(L) // 2
    print("== EO hopping term out_e = H_eo psi_o at 40^3x32: generated (qdp_jit_eval) vs hand-written (qdp_dslash)")
    for prec in (0, 1):
        dt = np.float64 if prec == 0 else np.float32
        for gk, tag in ((q.QDP_GAUGE, "18-real links"), (q.QDP_GAUGE12, "12-real links")):
            c = q.qdp_init(L, stream=stream)
            fU = q.qdp_field_alloc(c, gk, prec, q.QDP_ALL)
            q.qdp_field_import(fU, U.astype(dt))
            fo = q.qdp_field_alloc(c, q.QDP_FERMION, prec, 1)
            q.qdp_field_import(fo, np.ascontiguousarray(psi[odd], dtype=dt))
            oj = q.qdp_field_alloc(c, q.QDP_FERMION, prec, 0)
            oh = q.qdp_field_alloc(c, q.QDP_FERMION, prec, 0)
            t0 = time.perf_counter()
            q.qdp_jit_eval(oj, hopping_expr(), fU, fo)
            torch.cuda.synchronize()
            first = time.perf_counter() - t0
            n, secs = q.qdp_jit_stats(c)
            for _ in range(12):  # let the autotuner finish
                q.qdp_jit_eval(oj, hopping_expr(), fU, fo)
                q.qdp_jit_eval(oj, hopping_expr(literal=True), fU, fo)
            q.qdp_profile_reset(c)
            q.qdp_jit_eval(oj, hopping_expr(), fU, fo)
            fl, by = q.qdp_profile_work(c, -1)
            us_u = timed(stream, lambda: q.qdp_jit_eval(oj, hopping_expr(literal=True), fU, fo))
            us_j = timed(stream, lambda: q.qdp_jit_eval(oj, hopping_expr(), fU, fo))
            us_h = timed(stream, lambda: q.qdp_dslash(oh, fU, fo, 0))
            a, b = q.qdp_field_export(oj).astype(np.float64), q.qdp_field_export(oh).astype(np.float64)
            diff = np.max(np.abs(a - b)) / np.max(np.abs(b))
            pname = "fp64" if prec == 0 else "fp32"
            print(f"   {pname} {tag}: generated {us_j:8.1f} us ({by / us_j * 1e-3:7.1f} GB/s, "
                  f"{1320 * Vh / us_j * 1e-3:7.1f} GFLOPS at 1320/site; executes {fl / Vh:.0f} flop/site)   "
                  f"hand-written {us_h:8.1f} us ({by / us_h * 1e-3:7.1f} GB/s)   ratio {us_h / us_j:.3f}   "
                  f"max|diff|/max {diff:.1e}   compile {secs:.2f} s (first call {first:.2f} s);   "
                  f"literal form (no spin projection, 2664 flop/site) {us_u:8.1f} us", flush=True)
            q.qdp_finalize(c)
    print("== Table II functions at 32^4 (full lattice): generated vs hand-written qdp_expr (autotuned, PAPER.md:238)")
    L = (32, 32, 32, 32)
    V = fieldgen.volume(L)
    rng = lambda seed, shape: fieldgen.gaussian(seed, int(np.prod(shape))).reshape(shape)
    host = dict(u=rng(1, (V, 3, 3, 2)), v=rng(2, (V, 3, 3, 2)), s=rng(3, (V, 4, 4, 2)), t=rng(4, (V, 4, 4, 2)),
                p1=rng(5, (V, 4, 3, 2)), p2=rng(6, (V, 4, 3, 2)))
    C, F, S = q.QDP_COLORMATRIX, q.QDP_FERMION, q.QDP_SPINMATRIX
    cases = [("lcm", q.QDP_EXPR_LCM, C, "$0*$1", [(C, "u"), (C, "v")]),
             ("upsi", q.QDP_EXPR_UPSI, F, "$0*$1", [(C, "u"), (F, "p1")]),
             ("spmat", q.QDP_EXPR_SPMAT, S, "$0*$1", [(S, "s"), (S, "t")]),
             ("matvec", q.QDP_EXPR_MATVEC, F, "$0*$1 + $0*$2", [(C, "u"), (F, "p1"), (F, "p2")])]
    for prec in (0, 1):
        dt = np.float64 if prec == 0 else np.float32
        c = q.qdp_init(L, stream=stream)
        for name, code, ok, expr, ops in cases:
            fs = []
            for kind, key in ops:
                f = q.qdp_field_alloc(c, kind, prec, q.QDP_ALL)
                q.qdp_field_import(f, host[key].astype(dt))
                fs.append(f)
            oj = q.qdp_field_alloc(c, ok, prec, q.QDP_ALL)
            oh = q.qdp_field_alloc(c, ok, prec, q.QDP_ALL)
            for _ in range(12):  # let both autotuners finish
                q.qdp_jit_eval(oj, expr, *fs)
                q.qdp_expr(code, oh, *fs, *([None] * (3 - len(fs))))
            q.qdp_profile_reset(c)
            q.qdp_jit_eval(oj, expr, *fs)
            _, by = q.qdp_profile_work(c, -1)
            us_j = timed(stream, lambda: q.qdp_jit_eval(oj, expr, *fs))
            us_h = timed(stream, lambda: q.qdp_expr(code, oh, *fs, *([None] * (3 - len(fs)))))
            same = np.array_equal(q.qdp_field_export(oj), q.qdp_field_export(oh))
            print(f"   {'fp64' if prec == 0 else 'fp32'} {name:7s} generated {us_j:8.1f} us ({by / us_j * 1e-3:7.1f} GB/s)"
                  f"   hand-written {us_h:8.1f} us ({by / us_h * 1e-3:7.1f} GB/s)   ratio {us_h / us_j:.3f}"
                  f"   bit-identical {same}", flush=True)
            for f in fs + [oj, oh]:
                q.qdp_field_free(f)
        n, secs = q.qdp_jit_stats(c)
        print(f"   ({n} kernels generated, {secs:.2f} s total = {secs / max(n, 1):.2f} s per kernel)")
        q.qdp_finalize(c)


if __name__ == "__main__":
    main()
