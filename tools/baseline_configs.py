"""Every BASELINE.json config measured on one B200, plus a Fig. 6 analogue.

  --part configs : configs 1-5 of BASELINE.json on one GPU.
      1  4^4           full H (both parities), fp64: parity vs the oracle + latency per application
      2  16^3x32       EO dslash fp64/fp32 (GFLOPS, compulsory GB/s), norm2 / innerProduct (GB/s),
                       dslash parity vs the oracle
      3  32^3x64       Wilson-clover EO CGNR to 1e-10, fp64 and mixed fp32/fp64 (+ reconstruct-12):
                       iterations, time, iterations/s, algorithmic GFLOPS, true residual
      4  40^3x256      the whole production lattice on ONE GPU (the strong-scaling N = 1 point):
                       EO dslash fp64/fp32, clover CG iterations/s
      5  48^3x96       Wilson EO CGNR to 1e-10 fp64 on one GPU (N = 1 of the 8-GPU config), and the
                       per-rank sub-lattice of the z2 x t4 split (48x48x24x24) with its z and t
                       neighbours reached through the halo path (NCCL to self, overlapped)
  --part fig6    : the hopping term H (both parities, global volume V) vs V in fp32 and fp64 --
                   whole lattice, and with the t neighbour reached through the halo path (the code
                   path of a 2-GPU t split: pack -> NCCL send/recv -> exterior) with overlap on and off.
                   The paper's points: 2 x K20m, DP V = 32^4: 90 GFLOPS, SP V = 40^4: 197 GFLOPS.

Timing: CUDA events on the library's stream (qdp_set_stream), warm-up first; dslash numbers are
whole applications including any halo kernels.  Flops: 1320 per output site;
compulsory bytes: 8 links + input + output spinor per EO output site.
"""
import argparse
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import fieldgen  # noqa: E402
from paper_1408_5925_b200 import qdpb as q  # noqa: E402

PREC = {q.QDP_F64: ("fp64", np.float64, 8), q.QDP_F32: ("fp32", np.float32, 4)}


def out(msg):
    print(msg, flush=True)


class Timer:
    def __init__(self, stream):
        self.s = stream

    def __call__(self, fn, n, warm=12):
        for _ in range(warm):  # the tuners' probes finish here: they read their events
            fn()               # only once those completed, so synchronise between the warm-up calls
            torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(self.s)
        for _ in range(n):
            fn()
        e1.record(self.s)
        torch.cuda.synchronize()
        return e0.elapsed_time(e1) / n * 1e3  # us per call


def make_ctx(L, stream, halo_mask=0, nccl=0, overlap=1):
    """nccl = 1: faces through NCCL send/recv to self (separate pack / interior / exterior kernels);
    nccl = 0 with a halo mask: the peer-to-peer protocol with the fused boundary kernel (one launch)"""
    c = q.qdp_init(L, stream=stream)
    if halo_mask:
        q.qdp_set_option(c, q.QDP_OPT_SELF_HALO, halo_mask)
        q.qdp_set_option(c, q.QDP_OPT_SELF_NCCL, nccl)
        if not nccl:
            q.qdp_set_option(c, q.QDP_OPT_P2P, 1)
        q.qdp_set_option(c, q.QDP_OPT_OVERLAP, overlap)
    return c


def site_err(got, ref):
    g = got.reshape(len(got), -1)
    r = ref.reshape(len(ref), -1)
    nr = np.linalg.norm(r, axis=1)
    rms = np.sqrt(np.mean(nr ** 2))
    return float(np.max(np.linalg.norm(g - r, axis=1) / np.maximum(nr, 1e-12 * rms)))


def dslash_line(tag, L, prec, us, recon=18, per_app_sites=None):
    Vh = fieldgen.volume(L) // 2
    sites = per_app_sites if per_app_sites is not None else Vh
    b = (8 * recon + 48) * PREC[prec][2]
    return (f"{tag:44s} {us:9.1f} us  {sites / us * 1e-3:7.3f} Gsite/s  {1320 * sites / us * 1e-3:8.1f} GFLOPS  "
            f"{b * sites / us * 1e-3:7.1f} GB/s compulsory")


def eo_dslash(stream, L, U, psi, prec, n=20, recon=18):
    c = make_ctx(L, stream)
    try:
        dt = PREC[prec][1]
        fU = q.qdp_field_alloc(c, q.QDP_GAUGE12 if recon == 12 else q.QDP_GAUGE, prec, q.QDP_ALL)
        fp = q.qdp_field_alloc(c, q.QDP_FERMION, prec, q.QDP_ODD)
        fo = q.qdp_field_alloc(c, q.QDP_FERMION, prec, q.QDP_EVEN)
        q.qdp_field_import(fU, U.astype(dt))
        q.qdp_field_import(fp, np.ascontiguousarray(psi[fieldgen.cb_sites(L, 1)], dtype=dt))
        us = Timer(stream)(lambda: q.qdp_dslash(fo, fU, fp, q.QDP_EVEN), n)
        return us, q.qdp_field_export(fo)
    finally:
        q.qdp_finalize(c)


def cg_run(stream, L, U, b, clover, tol, maxit, mixed=False, recon12=False, halo_mask=0, nccl=0):
    c = make_ctx(L, stream, halo_mask, nccl)
    try:
        F = q.QDP_F64
        fU = q.qdp_field_alloc(c, q.QDP_GAUGE, F, q.QDP_ALL)
        fb = q.qdp_field_alloc(c, q.QDP_FERMION, F, q.QDP_ALL)
        fx = q.qdp_field_alloc(c, q.QDP_FERMION, F, q.QDP_ALL)
        q.qdp_field_import(fU, U)
        q.qdp_field_import(fb, b)
        fA = fAi = None
        if clover:
            fA = q.qdp_field_alloc(c, q.QDP_CLOVER, F, q.QDP_ALL)
            fAi = q.qdp_field_alloc(c, q.QDP_CLOVER, F, q.QDP_EVEN)
            q.qdp_clover_build(fA, fAi, fU, 0.1, 1.0)
        if mixed:
            Us = U.astype(np.float32)
            fUs = q.qdp_field_alloc(c, q.QDP_GAUGE12 if recon12 else q.QDP_GAUGE, q.QDP_F32, q.QDP_ALL)
            q.qdp_field_import(fUs, Us)
            fAs = fAis = None
            if clover:
                fAs = q.qdp_field_alloc(c, q.QDP_CLOVER, q.QDP_F32, q.QDP_ALL)
                fAis = q.qdp_field_alloc(c, q.QDP_CLOVER, q.QDP_F32, q.QDP_EVEN)
                q.qdp_clover_build(fAs, fAis, fUs, 0.1, 1.0)

            def solve():
                return q.qdp_cg_solve_mixed(fx, fb, fU, fA, fAi, fUs, fAs, fAis, mass=0.1, tol=tol, maxit=maxit)
        else:
            def solve():
                return q.qdp_cg_solve(fx, fb, fU, fA, fAi, mass=0.1, tol=tol, maxit=maxit)
        solve()
        torch.cuda.synchronize()
        q.qdp_profile_reset(c)  # algorithmic work counters (always on; per-launch events stay off)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        r = solve()
        e1.record(stream)
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1)
        flops, _ = q.qdp_profile_work(c, -1)
        return r, ms, flops
    finally:
        q.qdp_finalize(c)


def cg_line(tag, r, ms, flops):
    it = r["iters"]
    rel = f", {r['reliable']} reliable updates" if "reliable" in r else ""
    return (f"{tag:44s} {it:4d} iterations {ms:9.2f} ms  {it / ms * 1e3:7.1f} it/s  {flops / ms * 1e-6:7.1f} GFLOPS  "
            f"true residual {r['true_resid']:.2e}{rel}")


def part_configs(stream):
    import oracle
    t0 = time.time()
    T = Timer(stream)
    # ---- config 1
    L = (4, 4, 4, 4)
    U = fieldgen.random_gauge(L, 1001)
    psi = fieldgen.random_spinor(L, 2001)
    c = make_ctx(L, stream)
    fU = q.qdp_field_alloc(c, q.QDP_GAUGE, q.QDP_F64, q.QDP_ALL)
    fp = q.qdp_field_alloc(c, q.QDP_FERMION, q.QDP_F64, q.QDP_ALL)
    fo = q.qdp_field_alloc(c, q.QDP_FERMION, q.QDP_F64, q.QDP_ALL)
    q.qdp_field_import(fU, U)
    q.qdp_field_import(fp, psi)
    us = T(lambda: q.qdp_dslash(fo, fU, fp, q.QDP_ALL), 200)
    err = site_err(q.qdp_field_export(fo), oracle.hopping(U, psi, L, -1))
    q.qdp_finalize(c)
    out("== config 1: 4^4, random SU(3), one fp64 Wilson dslash application (full H, both parities)")
    out(f"   parity vs oracle: max per-site relative L2 error {err:.2e} (bar 1e-13)")
    out(f"   {us:.2f} us per application (two EO launches; launch-latency bound at 128 sites per parity)")

    # ---- config 2
    L = (16, 16, 16, 32)
    U = fieldgen.random_gauge(L, 1002)
    psi = fieldgen.random_spinor(L, 2002)
    chi = fieldgen.random_spinor(L, 2003)
    out("== config 2: 16^3x32 EO Wilson dslash + norm2/innerProduct, fp64 and fp32")
    ref = oracle.hopping(U, psi, L, 0)
    for prec in (q.QDP_F64, q.QDP_F32):
        name, dt, _ = PREC[prec]
        Uin = U.astype(dt).astype(np.float64)
        us, got = eo_dslash(stream, L, U, psi, prec, 200)
        refp = ref if prec == q.QDP_F64 else oracle.hopping(Uin, psi.astype(dt).astype(np.float64), L, 0)
        e = site_err(got.astype(np.float64), refp[fieldgen.cb_sites(L, 0)] if len(refp) != len(got) else refp)
        out("   " + dslash_line(f"EO dslash {name}", L, prec, us) + f"  parity {e:.2e}")
        c = make_ctx(L, stream)
        fa = q.qdp_field_alloc(c, q.QDP_FERMION, prec, q.QDP_ALL)
        fb = q.qdp_field_alloc(c, q.QDP_FERMION, prec, q.QDP_ALL)
        q.qdp_field_import(fa, psi.astype(dt))
        q.qdp_field_import(fb, chi.astype(dt))
        V = fieldgen.volume(L)
        us_n = T(lambda: q.qdp_norm2(fa), 200)
        us_i = T(lambda: q.qdp_inner_product(fa, fb), 200)
        eb = PREC[prec][2] * 24
        out(f"   norm2 {name} (full lattice, incl. host readback) {us_n:8.1f} us  {eb * V / us_n * 1e-3:7.1f} GB/s;  "
            f"innerProduct {us_i:8.1f} us  {2 * eb * V / us_i * 1e-3:7.1f} GB/s")
        q.qdp_finalize(c)

    # ---- config 3
    L = (32, 32, 32, 64)
    U = fieldgen.random_gauge(L, 1003)
    b = fieldgen.random_spinor(L, 2004)
    out("== config 3: 32^3x64 Wilson-clover (m = 0.1, c_SW = 1) EO CGNR to 1e-10")
    for tag, mixed, r12 in (("fp64", False, False), ("mixed fp32/fp64", True, False),
                            ("mixed fp32 (reconstruct-12) / fp64", True, True)):
        r, ms, fl = cg_run(stream, L, U, b, True, 1e-10, 10000, mixed, r12)
        out("   " + cg_line(tag, r, ms, fl))
    del U, b

    # ---- config 4 (whole production lattice on one GPU)
    L = (40, 40, 40, 256)
    t1 = time.time()
    U = fieldgen.random_gauge(L, 1004)
    psi = fieldgen.random_spinor(L, 2005)
    out(f"== config 4: 40^3x256 on ONE GPU (strong-scaling N = 1 point; fields generated in {time.time() - t1:.0f} s)")
    for prec in (q.QDP_F64, q.QDP_F32):
        us, _ = eo_dslash(stream, L, U, psi, prec, 10)
        out("   " + dslash_line(f"EO dslash {PREC[prec][0]}", L, prec, us))
    r, ms, fl = cg_run(stream, L, U, psi, True, 0.0, 16)
    out("   " + cg_line("clover CG fp64, 16 fixed iterations", r, ms, fl))
    del U, psi

    # ---- config 5
    L = (48, 48, 48, 96)
    t1 = time.time()
    U = fieldgen.random_gauge(L, 1005)
    b = fieldgen.random_spinor(L, 2006)
    out(f"== config 5: 48^3x96 Wilson (m = 0.1) EO CGNR to 1e-10 fp64 (fields generated in {time.time() - t1:.0f} s)")
    r, ms, fl = cg_run(stream, L, U, b, False, 1e-10, 10000)
    out("   " + cg_line("whole lattice on one GPU", r, ms, fl))
    del U, b
    Ls = (48, 48, 24, 24)
    U = fieldgen.random_gauge(Ls, 1005)
    b = fieldgen.random_spinor(Ls, 2006)
    for tag, mask, nccl in (("rank sub-lattice 48x48x24x24, no halo", 0, 0),
                            ("same, z+t fused peer-to-peer boundary", 12, 0),
                            ("same, z+t halo path (NCCL to self)", 12, 1)):
        r, ms, fl = cg_run(stream, Ls, U, b, False, 0.0, 50, halo_mask=mask, nccl=nccl)
        out("   " + cg_line(tag + ", 50 it", r, ms, fl))
    out(f"(total {time.time() - t0:.0f} s)")


def part_fig6(stream):
    out("Fig. 6 analogue: hopping term H on the global volume V (both parities = 2 EO launches + halo kernels),")
    out("GFLOPS at 1320 flop/site.  'halo t' = the code path of a 2-GPU t split on one GPU (pack -> NCCL send/recv")
    out("to self -> exterior); overlap on = interior kernel concurrent with the exchange (PAPER.md:212, 288).")
    out("'p2p t' = the fused peer-to-peer boundary kernel (one launch per EO application; overlap off = every block")
    out("waits for the ghosts first).")
    out(f"{'V':>6s} {'prec':>5s} {'whole lattice':>22s} {'halo t, overlap on':>22s} {'halo t, overlap off':>22s} "
        f"{'p2p t, overlap on':>22s} {'p2p t, overlap off':>22s}")
    for n in (8, 12, 16, 20, 24, 32, 40, 48):
        L = (n, n, n, n)
        U = fieldgen.random_gauge(L, 1004)
        psi = fieldgen.random_spinor(L, 2005)
        V = fieldgen.volume(L)
        for prec in (q.QDP_F32, q.QDP_F64):
            name, dt, _ = PREC[prec]
            cols = []
            for mask, nccl, ov in ((0, 0, 1), (8, 1, 1), (8, 1, 0), (8, 0, 1), (8, 0, 0)):
                c = make_ctx(L, stream, mask, nccl, ov)
                fU = q.qdp_field_alloc(c, q.QDP_GAUGE, prec, q.QDP_ALL)
                fp = q.qdp_field_alloc(c, q.QDP_FERMION, prec, q.QDP_ALL)
                fo = q.qdp_field_alloc(c, q.QDP_FERMION, prec, q.QDP_ALL)
                q.qdp_field_import(fU, U.astype(dt))
                q.qdp_field_import(fp, psi.astype(dt))
                reps = max(10, min(400, int(2e8 / V)))
                us = Timer(stream)(lambda: q.qdp_dslash(fo, fU, fp, q.QDP_ALL), reps)
                cols.append(f"{1320 * V / us * 1e-3:9.1f} ({us:8.1f} us)")
                q.qdp_finalize(c)
            out(f"{n:>4d}^4 {name:>5s} " + " ".join(f"{s:>22s}" for s in cols))
    out("paper (2 x K20m over PCIe + InfiniBand, overlap on): DP V = 32^4: 90 GFLOPS; SP V = 40^4: 197 GFLOPS")


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--part", choices=["configs", "fig6"], default="configs")
    args = ap.parse_args()
    torch.cuda.init()
    stream = torch.cuda.Stream()
    torch.cuda.set_stream(stream)
    out(f"# {torch.cuda.get_device_name()}  ({time.strftime('%Y-%m-%d %H:%M:%S')})")
    if args.part == "configs":
        part_configs(stream)
    else:
        part_fig6(stream)


if __name__ == "__main__":
    main()
