#!/usr/bin/env python3
"""Benchmark of the B200-native QDP hot path (arXiv:1408.5925) -- one JSON line on rank 0.

Step = one even-odd preconditioned Wilson-clover CGNR solve (fp64) with a fixed number of
iterations (tol = 0), through the C ABI (qdp_cg_solve): every row of SURVEY.md 8(a) runs in
it -- SoA fields (A1), fused EO dslash with clover epilogues (A4, A5), reductions (A6), fused
CG updates (A7), the CG driver (A8) and, for N > 1, face packing + NCCL halo exchange
overlapped with the interior kernel (A2, A9).  Workload: config 4 of BASELINE.json read as
weak scaling (R20): 40^3 x 32 sites per GPU, split along t, so N = 8 is the
paper's 40^3 x 256 production lattice.

value    = whole-job algorithmic GFLOPS of the step (Table II convention, 1320 flop per
           dslash output site), fields resident in HBM;
e2e      = the same with b imported from pinned host memory and x exported every step;
roofline = the dslash kernel: compulsory bytes per launch / live CUDA-event launch time;
cpu_baseline = the C oracle timed on the host cores on a bounded sample of the workload.

--impl reference times the oracle (the tier's reference arm) on the same config and metric.
"""
from __future__ import annotations

import argparse
import json
import os
import shutil
import statistics
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "Wilson dslash GFLOPS & HBM GB/s (fp64/fp32) at 1/2/4/8 B200; CG iters/s"
LOCAL = (40, 40, 40, 32)
MASS, CSW = 0.1, 1.0
HBM_FALLBACK = 6650.0  # GB/s, B200_PROFILING.md fallback (used only without MEASURED_PEAKS.json)


# ---------------------------------------------------------------- accounting
def cg_flops(Vh: int, iters: int, clover: bool = True) -> float:
    """Algorithmic flops of one qdp_cg_solve (same count the library's counters produce).

    clover: per iteration 2 x Mhat (dslash+A^-1: 1320+504+24; dslash+A x xpay: 1320+504+48)
            + Re<p,q> 96 (fused into the last dslash) + r update with |r|^2 96
            + x and p update 96                                        = 7728 / odd site
            (the last iteration skips the p update: -48)
            setup: A^-1 b_e 504, bhat 1392, r0 = Mhat^dag bhat 3720, |r0|^2 48 = 5664
            finish: x_e 1896, true residual 2 x 1872 + 96 + 2 x 96     = 5928
    Wilson: 5712 / iteration, setup 4176, finish 4464."""
    last = -48 if iters > 0 else 0
    if clover:
        return Vh * (5664 + 5928 + 7728 * iters + last)
    return Vh * (4176 + 4464 + 5712 * iters + last)


def dslash_bytes_per_site(prec_bytes: int = 8) -> int:
    """Compulsory bytes of one EO dslash output site: 8 links + input + output = 192 reals."""
    return (8 * 18 + 24 + 24) * prec_bytes


# ---------------------------------------------------------------- helpers
def measured_peak():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "MEASURED_PEAKS.json hbm_gbs (torch copy, measured)"
    return HBM_FALLBACK, "B200_PROFILING.md fallback 6.65 TB/s"


class Clocks:
    """nvidia-smi sampling during the timed region (B200_PROFILING.md clocks line)."""

    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.path = os.path.join(ROOT, "gpurun_out", f"clocks_rank{index}.csv")

    def __enter__(self):
        if shutil.which("nvidia-smi"):
            os.makedirs(os.path.dirname(self.path), exist_ok=True)
            self.f = open(self.path, "w")
            self.proc = subprocess.Popen(["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.Q}",
                                          "--format=csv,noheader,nounits", "-lms", "100"],
                                         stdout=self.f, stderr=subprocess.DEVNULL)
            time.sleep(0.3)
        return self

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            self.proc.wait()
            self.f.close()

    def summary(self):
        if not self.proc:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        sm, smax, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in open(self.path):
            f = [x.strip() for x in line.split(",")]
            if len(f) < 9:
                continue
            try:
                sm.append(float(f[1]))
                smax = float(f[2])
            except ValueError:
                continue
            for n, v in zip(names, f[5:9]):
                if v.lower().startswith("active"):
                    reasons.add(n)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": smax,
                "samples": len(sm), "reasons": sorted(reasons)}


def gen_fields(L, rank):
    import fieldgen
    U = fieldgen.random_gauge(L, 1004 + 7919 * rank)
    b = fieldgen.random_spinor(L, 2005 + 7919 * rank)
    return U, b


# ---------------------------------------------------------------- oracle (reference arm / cpu baseline)
def oracle_solve_timed(U, b, L, iters, A=None):
    import oracle
    if A is None:
        A = oracle.clover_build(U, L, MASS, CSW)  # setup, outside the timed region (as on the GPU)
    t0 = time.perf_counter()
    res = oracle.cg_solve(U, b, L, MASS, A=A, tol=0.0, maxit=iters)
    dt = time.perf_counter() - t0
    assert res["iters"] == iters
    return dt, res


def run_reference(args, rank, world):
    """The tier's reference arm: the C oracle as it stands, on the host cores, same metric."""
    if rank != 0:
        return
    import oracle
    # the other ranks exit without work, so rank 0 has the host's cores (torchrun sets
    # OMP_NUM_THREADS=1 per rank, which would otherwise pin the oracle to one thread)
    oracle.set_threads(len(os.sched_getaffinity(0)))
    L = LOCAL
    Vh = L[0] * L[1] * L[2] * L[3] // 2
    U, b = gen_fields(L, 0)
    A = oracle.clover_build(U, L, MASS, CSW)
    times = []
    for i in range(args.warmup + args.steps):
        dt, _ = oracle_solve_timed(U, b, L, args.ref_iters, A)
        if i >= args.warmup:
            times.append(dt)
    t = sum(times)
    flops = cg_flops(Vh, args.ref_iters) * args.steps
    v = flops / t * 1e-9
    sample = (f"oracle/oracle.c even-odd clover CGNR on one 40^3x32 sub-lattice, {args.ref_iters} iteration(s) "
              f"per step incl. its clover inversion, setup, reconstruction and true residual; fp64")
    out = {"metric": METRIC, "value": v, "unit": "GFLOPS", "impl": "reference", "n_gpus": args.gpus,
           "steps": args.steps, "warmup": args.warmup, "ms_per_step": t / args.steps * 1e3,
           "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
           "config": config_dict(args, world=1),
           "cpu_baseline": {"value": v, "unit": "GFLOPS", "cores": oracle.max_threads(), "kind": "oracle",
                            "sample": sample},
           "e2e": {"value": v, "unit": "GFLOPS", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(out), flush=True)


def config_dict(args, world):
    gl = (LOCAL[0], LOCAL[1], LOCAL[2], LOCAL[3] * world)
    return {"workload": "BASELINE config 4 (40^3x256 production lattice) as weak scaling: 40^3x32 sites per GPU, "
                        "t-split; even-odd Wilson-clover CGNR solve, fixed iterations",
            "global_lattice": "x".join(map(str, gl)), "local_lattice": "x".join(map(str, LOCAL)),
            "operator": f"Wilson-clover m={MASS} c_SW={CSW}, hot random SU(3) gauge field",
            "gauge_storage": "reconstruct-12" if getattr(args, "recon", 18) == 12 else "full 3x3 (18 reals)",
            "cg_iters_per_step": args.iters, "parallelism": f"t-split x{world}" if world > 1 else "single GPU",
            "l2": "inputs larger than L2 (gauge 1.18 GB + clover 1.2 GB + 6 fermion vectors per GPU), no flush"}


# ---------------------------------------------------------------- native arm
def run_native(args, rank, world, local_rank):
    import numpy as np
    import torch
    import torch.distributed as dist

    import fieldgen
    from paper_1408_5925_b200 import dist as qdist
    from paper_1408_5925_b200 import exprs as qexprs
    from paper_1408_5925_b200 import qdpb as q

    # QDPB_BENCH_ONE_GPU=1: every rank on cuda:0 (functional test of the N > 1 path on a one-GPU
    # box; peer communicator only, torch.distributed over gloo -- the timings mean nothing)
    one_gpu = os.environ.get("QDPB_BENCH_ONE_GPU") == "1"
    dev = 0 if one_gpu else local_rank
    torch.cuda.set_device(dev)
    if world > 1:
        if one_gpu:
            if args.comm != "peer":
                raise SystemExit("QDPB_BENCH_ONE_GPU needs --comm peer (NCCL refuses two ranks on one GPU)")
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
    # one explicit stream shared by the library (its context stream) and torch's timing events,
    # so the events are ordered with the kernels they bracket
    stream = torch.cuda.Stream()
    torch.cuda.set_stream(stream)
    gdims = (LOCAL[0], LOCAL[1], LOCAL[2], LOCAL[3] * world)
    P = qdist.proc_grid_for(world, gdims, split=(3,))
    if args.comm == "peer":  # no NCCL on the data path: halos, sums, shifts through peer memory
        ctx = qdist.bootstrap_peer(gdims, P, stream=stream)
    else:
        ctx = qdist.bootstrap(gdims, P, stream=stream)
        q.qdp_set_option(ctx, q.QDP_OPT_P2P, 1 if args.p2p else 0)
    q.qdp_set_option(ctx, q.QDP_OPT_OVERLAP, 0 if args.no_overlap else 1)
    L = LOCAL
    Vh = L[0] * L[1] * L[2] * L[3] // 2

    U, b = gen_fields(L, rank)
    fU = q.qdp_field_alloc(ctx, q.QDP_GAUGE12 if args.recon == 12 else q.QDP_GAUGE, q.QDP_F64, q.QDP_ALL)
    fb = q.qdp_field_alloc(ctx, q.QDP_FERMION, q.QDP_F64, q.QDP_ALL)
    fx = q.qdp_field_alloc(ctx, q.QDP_FERMION, q.QDP_F64, q.QDP_ALL)
    fA = q.qdp_field_alloc(ctx, q.QDP_CLOVER, q.QDP_F64, q.QDP_ALL)
    fAi = q.qdp_field_alloc(ctx, q.QDP_CLOVER, q.QDP_F64, q.QDP_EVEN)
    q.qdp_field_import(fU, U)
    q.qdp_field_import(fb, b)
    q.qdp_clover_build(fA, fAi, fU, MASS, CSW)

    def step():
        return q.qdp_cg_solve(fx, fb, fU, fA, fAi, mass=MASS, tol=0.0, maxit=args.iters)

    # parity spot check of this exact configuration (rank 0, N = 1): first solve's history vs oracle
    parity = None
    for _ in range(args.warmup):
        r = step()
    if args.check and world == 1:
        import oracle
        _, ref = oracle_solve_timed(U, b, L, 2)
        got = q.qdp_cg_solve(fx, fb, fU, fA, fAi, mass=MASS, tol=0.0, maxit=2)
        parity = {"cg_hist_max_rel_diff_2it": float(np.max(np.abs(got["hist"] - ref["hist"]) / ref["hist"])),
                  "x_max_site_rel_err_2it": _site_err(q.qdp_field_export(fx), ref["x"])}

    # ---- timed region: K solves, fields resident in HBM
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    q.qdp_profile_reset(ctx)
    q.qdp_set_option(ctx, q.QDP_OPT_PROFILE, 1)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with Clocks(dev) as clk:
        e0.record(stream)
        for _ in range(args.steps):
            r = step()
        e1.record(stream)
        torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    ms = e0.elapsed_time(e1)
    n_dsl, ms_dsl = q.qdp_profile_query(ctx, q.QDP_PK_DSLASH)
    f_dsl, b_dsl = q.qdp_profile_work(ctx, q.QDP_PK_DSLASH)
    f_all, _ = q.qdp_profile_work(ctx, -1)
    n_all, ms_all = q.qdp_profile_query(ctx, -1)
    q.qdp_set_option(ctx, q.QDP_OPT_PROFILE, 0)
    assert abs(f_all - cg_flops(Vh, args.iters) * args.steps) <= 1e-9 * f_all, (f_all, cg_flops(Vh, args.iters))
    ms_max = qdist.max_over_ranks(ms)
    flops_job = qdist.sum_over_ranks(f_all)
    value = flops_job / (ms_max * 1e-3) * 1e-9

    # ---- e2e: the same solves through the C ABI from pinned host memory, every step's source
    # uploaded and every step's solution downloaded inside the timed region.  Pipelined: on a copy
    # stream the upload of b_{k+1} and the download of x_{k-1} run while solve k runs; the layout
    # conversions (qdp_field_import_device / export_device) run on the compute stream.
    k2 = args.e2e_steps if args.e2e_steps > 0 else args.steps
    hb = [torch.from_numpy(b).pin_memory() for _ in range(2)]          # host sources
    hx = [torch.empty_like(hb[0]).pin_memory() for _ in range(2)]       # host solutions
    d_in = [torch.empty_like(hb[0], device="cuda") for _ in range(2)]   # device staging (host layout)
    d_out = [torch.empty_like(hb[0], device="cuda") for _ in range(2)]
    fbs, fxs = [fb, q.qdp_field_alloc(ctx, q.QDP_FERMION, q.QDP_F64, q.QDP_ALL)], [fx, fx]
    fxs[1] = q.qdp_field_alloc(ctx, q.QDP_FERMION, q.QDP_F64, q.QDP_ALL)
    cs = torch.cuda.Stream()
    ev_in = [torch.cuda.Event() for _ in range(2)]
    ev_out = [torch.cuda.Event() for _ in range(2)]
    ev_dl = [torch.cuda.Event() for _ in range(2)]

    def e2e_run(n):
        for e in ev_dl:
            e.record(cs)
        with torch.cuda.stream(cs):
            d_in[0].copy_(hb[0], non_blocking=True)
            ev_in[0].record(cs)
        for k in range(n):
            s = k % 2
            if k + 1 < n:  # upload the next step's source while this step solves
                with torch.cuda.stream(cs):
                    d_in[1 - s].copy_(hb[1 - s], non_blocking=True)
                    ev_in[1 - s].record(cs)
            stream.wait_event(ev_in[s])
            q.qdp_field_import_device(fbs[s], d_in[s])
            q.qdp_cg_solve(fxs[s], fbs[s], fU, fA, fAi, mass=MASS, tol=0.0, maxit=args.iters)
            stream.wait_event(ev_dl[s])  # d_out[s] was downloaded (step k-2)
            q.qdp_field_export_device(fxs[s], d_out[s])
            ev_out[s].record(stream)
            with torch.cuda.stream(cs):  # download this step's solution during the next solve
                cs.wait_event(ev_out[s])
                hx[s].copy_(d_out[s], non_blocking=True)
                ev_dl[s].record(cs)

    e2e_run(2)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    e2, e3 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e2.record(stream)
    cs.wait_event(e2)
    e2e_run(k2)
    e3.record(cs)  # after the last download (cs is ordered after every compute step)
    torch.cuda.synchronize()
    assert np.array_equal(hx[(k2 - 1) % 2].numpy(), q.qdp_field_export(fxs[(k2 - 1) % 2]))
    ms_e2e = qdist.max_over_ranks(e2.elapsed_time(e3))
    e2e_flops = qdist.sum_over_ranks(cg_flops(Vh, args.iters) * k2)
    e2e_value = e2e_flops / (ms_e2e * 1e-3) * 1e-9
    bytes_b = hb[0].numel() * hb[0].element_size()
    q.qdp_field_free(fbs[1])
    q.qdp_field_free(fxs[1])

    # ---- the metric's plain Wilson dslash in both precisions (not the step): one EO application
    # (out_e = H_eo psi_o) on the same lattice, uncompressed links, live CUDA events
    dsl = {}
    for prec, tag in ((q.QDP_F64, "fp64"), (q.QDP_F32, "fp32")):
        fUp = fU if prec == q.QDP_F64 and args.recon == 18 else q.qdp_field_alloc(ctx, q.QDP_GAUGE, prec, q.QDP_ALL)
        if fUp is not fU:
            q.qdp_field_import(fUp, U.astype(np.float64 if prec == q.QDP_F64 else np.float32))
        fi = q.qdp_field_alloc(ctx, q.QDP_FERMION, prec, q.QDP_ODD)
        fo = q.qdp_field_alloc(ctx, q.QDP_FERMION, prec, q.QDP_EVEN)
        for _ in range(5):
            q.qdp_dslash(fo, fUp, fi, q.QDP_EVEN)
        q.qdp_synchronize(ctx)
        q.qdp_profile_reset(ctx)
        q.qdp_set_option(ctx, q.QDP_OPT_PROFILE, 1)
        for _ in range(20):
            q.qdp_dslash(fo, fUp, fi, q.QDP_EVEN)
        n_d, ms_d = q.qdp_profile_query(ctx, q.QDP_PK_DSLASH)
        f_d, b_d = q.qdp_profile_work(ctx, q.QDP_PK_DSLASH)
        q.qdp_set_option(ctx, q.QDP_OPT_PROFILE, 0)
        t_d = ms_d / n_d * 1e-3
        eff = 2880 if prec == q.QDP_F64 else 1440  # Table II convention: every leaf load, no reuse (R17)
        dsl[tag] = {"us_per_launch": t_d * 1e6, "gsites_per_s": Vh / t_d * 1e-9, "gflops_per_gpu": f_d / n_d / t_d * 1e-9,
                    "gbs_compulsory_per_gpu": b_d / n_d / t_d * 1e-9, "bytes_per_site": b_d / n_d / Vh,
                    "gbs_effective_per_gpu": eff * Vh / t_d * 1e-9,
                    "frac_of_measured_hbm": b_d / n_d / t_d * 1e-9 / measured_peak()[0],
                    "frac_of_8TBs": b_d / n_d / t_d * 1e-9 / 8000.0}
        # the same operator generated at run time from its expression (qdp_jit_eval; PAPER.md
        # sections III-IV): the paper's generated-vs-hand-tuned comparison
        if world == 1:
            expr = qexprs.hopping()
            for _ in range(12):  # compile once, then let the paper's autotuner settle
                q.qdp_jit_eval(fo, expr, fUp, fi)
            q.qdp_synchronize(ctx)
            q.qdp_profile_reset(ctx)
            q.qdp_set_option(ctx, q.QDP_OPT_PROFILE, 1)
            for _ in range(20):
                q.qdp_jit_eval(fo, expr, fUp, fi)
            n_j, ms_j = q.qdp_profile_query(ctx, q.QDP_PK_BLAS)
            f_j, b_j = q.qdp_profile_work(ctx, q.QDP_PK_BLAS)
            q.qdp_set_option(ctx, q.QDP_OPT_PROFILE, 0)
            t_j = ms_j / n_j * 1e-3
            dsl[tag]["generated"] = {"us_per_launch": t_j * 1e6, "flop_per_site": f_j / n_j / Vh,
                                     "gbs_compulsory_per_gpu": b_j / n_j / t_j * 1e-9,
                                     "speed_vs_handwritten": t_d / t_j}
        for f in (fi, fo) + (() if fUp is fU else (fUp,)):
            q.qdp_field_free(f)

    # ---- time to solution at tol 1e-10 (not the step): fp64 CG vs the mixed-precision CG
    tts = None
    if args.tts:
        fU32 = q.qdp_field_alloc(ctx, q.QDP_GAUGE, q.QDP_F32, q.QDP_ALL)
        fU32r = q.qdp_field_alloc(ctx, q.QDP_GAUGE12, q.QDP_F32, q.QDP_ALL)
        fA32 = q.qdp_field_alloc(ctx, q.QDP_CLOVER, q.QDP_F32, q.QDP_ODD)
        fAi32 = q.qdp_field_alloc(ctx, q.QDP_CLOVER, q.QDP_F32, q.QDP_EVEN)
        U32 = U.astype(np.float32)
        q.qdp_field_import(fU32, U32)
        q.qdp_field_import(fU32r, U32)
        q.qdp_clover_build(fA32, fAi32, fU32, MASS, CSW)
        q.qdp_field_import(fb, b)
        solvers = {
            "fp64": lambda: q.qdp_cg_solve(fx, fb, fU, fA, fAi, mass=MASS, tol=1e-10, maxit=5000),
            "mixed_fp32": lambda: q.qdp_cg_solve_mixed(fx, fb, fU, fA, fAi, fU32, fA32, fAi32, mass=MASS, tol=1e-10,
                                                       delta=0.1, maxit=5000),
            "mixed_fp32_recon12": lambda: q.qdp_cg_solve_mixed(fx, fb, fU, fA, fAi, fU32r, fA32, fAi32, mass=MASS,
                                                               tol=1e-10, delta=0.1, maxit=5000),
            # fewer reliable updates: each costs an fp64 Mhat^dag Mhat (4 fp64 dslash launches)
            "mixed_fp32_recon12_delta1e-2": lambda: q.qdp_cg_solve_mixed(fx, fb, fU, fA, fAi, fU32r, fA32, fAi32,
                                                                         mass=MASS, tol=1e-10, delta=1e-2, maxit=5000),
            "mixed_fp32_recon12_delta1e-3": lambda: q.qdp_cg_solve_mixed(fx, fb, fU, fA, fAi, fU32r, fA32, fAi32,
                                                                         mass=MASS, tol=1e-10, delta=1e-3, maxit=5000),
        }
        tts = {}
        for name, fn in solvers.items():
            fn()  # warm
            if world > 1:
                dist.barrier()
            torch.cuda.synchronize()
            e4, e5 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e4.record(stream)
            r = fn()
            e5.record(stream)
            torch.cuda.synchronize()
            tts[name] = {"ms": qdist.max_over_ranks(e4.elapsed_time(e5)), "iters": r["iters"],
                         "true_resid": r["true_resid"], "reliable_updates": r.get("reliable")}
        for f in (fU32, fU32r, fA32, fAi32):
            q.qdp_field_free(f)

    # ---- multi-shift CG (the RHMC solver; not the step): all shifts kept active (tol = 0)
    msh = None
    if args.ms_shifts > 0:
        sig = [0.0] + [0.002 * 4.0 ** i for i in range(args.ms_shifts - 1)]
        fphi = q.qdp_field_alloc(ctx, q.QDP_FERMION, q.QDP_F64, q.QDP_ODD)
        q.qdp_field_import(fphi, np.ascontiguousarray(b[fieldgen.parity(L) == 1]))
        xs = [q.qdp_field_alloc(ctx, q.QDP_FERMION, q.QDP_F64, q.QDP_ODD) for _ in sig]
        q.qdp_cg_solve_multishift(xs, sig, fphi, fU, fA, fAi, mass=MASS, tol=0.0, maxit=2, true_resid=False)
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        q.qdp_profile_reset(ctx)
        q.qdp_set_option(ctx, q.QDP_OPT_PROFILE, 1)
        e6, e7 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e6.record(stream)
        r = q.qdp_cg_solve_multishift(xs, sig, fphi, fU, fA, fAi, mass=MASS, tol=0.0, maxit=args.ms_iters,
                                      true_resid=False)
        e7.record(stream)
        torch.cuda.synchronize()
        n_u, ms_u = q.qdp_profile_query(ctx, q.QDP_PK_MSHIFT)
        _, b_u = q.qdp_profile_work(ctx, q.QDP_PK_MSHIFT)
        f_t, _ = q.qdp_profile_work(ctx, -1)
        q.qdp_set_option(ctx, q.QDP_OPT_PROFILE, 0)
        t_ms = qdist.max_over_ranks(e6.elapsed_time(e7))
        msh = {"shifts": len(sig), "sigma": sig, "iters": r["iters"], "ms_per_iter": t_ms / r["iters"],
               "gflops_per_gpu": f_t / (t_ms * 1e-3) * 1e-9,
               "update_pass": {"us_per_launch": ms_u / n_u * 1e3, "bytes_per_site": b_u / n_u / Vh,
                               "gbs": b_u / (ms_u * 1e-3) * 1e-9,
                               "frac_of_measured_hbm": b_u / (ms_u * 1e-3) * 1e-9 / measured_peak()[0],
                               "share_of_solve": ms_u / t_ms}}
        for f in xs + [fphi]:
            q.qdp_field_free(f)

    # ---- CPU baseline (oracle, rank 0 at N = 1 only)
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        import oracle
        dt, _ = oracle_solve_timed(U, b, L, args.cpu_iters)
        cpu = {"value": cg_flops(Vh, args.cpu_iters) / dt * 1e-9, "unit": "GFLOPS", "cores": oracle.max_threads(),
               "kind": "oracle", "seconds": dt,
               "sample": f"oracle/oracle.c even-odd clover CGNR, same 40^3x32 lattice and fields, {args.cpu_iters} "
                         f"iterations incl. its clover inversion, setup, reconstruction and true residual"}

    peak, peak_src = measured_peak()
    us_dsl = ms_dsl / n_dsl * 1e3
    gbs = (b_dsl / n_dsl) / (us_dsl * 1e-6) * 1e-9
    traffic = None
    tp = os.path.join(ROOT, "profiles", "dslash_ncu_traffic.json")
    if os.path.exists(tp):
        with open(tp) as f:
            traffic = json.load(f).get("dram_bytes_per_launch")
    out = {
        "metric": METRIC, "value": value, "unit": "GFLOPS", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms_max / args.steps, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic (seeded hot random SU(3) gauge field, Gaussian source)",
        "config": config_dict(args, world),
        "cg_iters_per_s": args.iters * args.steps / (ms_max * 1e-3),
        "dslash": {"launches": n_dsl, "us_per_launch": us_dsl, "gflops_per_gpu": f_dsl / n_dsl / (us_dsl * 1e-6) * 1e-9,
                   "gbs_compulsory_per_gpu": gbs, "bytes_per_site": (b_dsl / n_dsl) / Vh,
                   "share_of_step": ms_dsl / ms, "frac_of_8TBs": gbs / 8000.0},
        "roofline": {"bound": "hbm", "achieved": gbs, "peak": peak, "unit": "GB/s", "frac": gbs / peak,
                     "traffic": traffic, "kernel": "dslash_kernel<double> (fused EO hopping term + clover epilogue)",
                     "peak_source": peak_src},
        "e2e": {"value": e2e_value, "unit": "GFLOPS", "h2d_bytes_per_step": bytes_b, "d2h_bytes_per_step": bytes_b,
                "steps": k2},
        "gpu_launches": n_all,
        "clocks": clk.summary(),
        "cpu_baseline": cpu,
        "parity": parity,
        "time_to_solution_1e-10": tts,
        "multishift_cg": msh,
        "eo_dslash_plain": dsl,
        "overlap": not args.no_overlap,
        "halo": ("peer (IPC ghost slots + flags, no NCCL)" if args.comm == "peer" else
                 "p2p" if args.p2p else "nccl") if world > 1 else "none (one GPU, periodic wrap in-kernel)",
    }
    if rank == 0:
        print(json.dumps(out), flush=True)
    for f in (fU, fb, fx, fA, fAi):
        q.qdp_field_free(f)
    q.qdp_finalize(ctx)
    if world > 1:
        dist.destroy_process_group()


def _site_err(got, ref):
    import numpy as np
    g = got.reshape(len(got), -1)
    o = ref.reshape(len(ref), -1)
    return float(np.max(np.linalg.norm(g - o, axis=1) / np.linalg.norm(o, axis=1)))


def main():
    ap = argparse.ArgumentParser(description=__doc__, formatter_class=argparse.RawDescriptionHelpFormatter)
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["native", "reference"], default="native")
    ap.add_argument("--iters", type=int, default=32, help="CG iterations per step (tol = 0)")
    ap.add_argument("--e2e-steps", type=int, default=0, help="e2e steps (0: the same K as the timed region)")
    ap.add_argument("--cpu-iters", type=int, default=2)
    ap.add_argument("--ref-iters", type=int, default=1)
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-overlap", action="store_true")
    ap.add_argument("--p2p", action="store_true", help="with --comm nccl: peer-to-peer (CUDA IPC) halos")
    ap.add_argument("--comm", choices=["peer", "nccl"], default="peer",
                    help="N > 1: peer-memory communicator (qdp_init_peer, default) or NCCL")
    ap.add_argument("--ms-shifts", type=int, default=12, help="multi-shift CG measurement: shifts (0: skip)")
    ap.add_argument("--ms-iters", type=int, default=20)
    ap.add_argument("--recon", type=int, choices=[18, 12], default=18,
                    help="gauge storage of the solve: 18 (default, uncompressed as in PAPER.md:292) or 12")
    ap.add_argument("--no-tts", dest="tts", action="store_false", help="skip the time-to-solution comparison")
    ap.add_argument("--check", action="store_true", default=True)
    ap.add_argument("--no-check", dest="check", action="store_false")
    args = ap.parse_args()
    if args.warmup < 3:
        ap.error("--warmup must be >= 3")
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if world != args.gpus:
        ap.error(f"--gpus {args.gpus} but WORLD_SIZE={world} (launch N > 1 with torch.distributed.run)")
    if args.impl == "reference":
        run_reference(args, rank, world)
    else:
        run_native(args, rank, world, local_rank)


if __name__ == "__main__":
    main()
