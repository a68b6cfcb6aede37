#!/usr/bin/env python3
"""Benchmark of the B200-native QDP hot path (arXiv:1408.5925) -- one JSON line on rank 0.

Step = one even-odd preconditioned Wilson-clover CGNR solve (fp64) with a fixed number of
iterations (tol = 0), through the C ABI (qdp_cg_solve): every row of SURVEY.md 8(a) runs in
it -- SoA fields (A1), fused EO dslash with clover epilogues (A4, A5), reductions (A6), fused
CG updates (A7), the CG driver (A8) and, for N > 1, face packing + peer-to-peer halo exchange
overlapped with the interior sites inside the same kernel (A2, A9).  Workload: config 4 of
BASELINE.json read as weak scaling (R20): 40^3 x 32 sites per GPU, split along t, so
N = 8 is the paper's 40^3 x 256 production lattice.

value    = whole-job algorithmic GFLOPS of the step (Table II convention, 1320 flop per
           dslash output site), fields resident in HBM;
e2e      = the same with b imported from pinned host memory and x exported every step;
roofline = the dslash kernel: compulsory bytes per launch / live CUDA-event launch time;
cpu_baseline = the C oracle timed on the host cores on a bounded sample of the workload.
Further keys (not the step): the plain EO dslash fp64/fp32, halo bytes and NVLink rates,
overlap on/off (Fig. 6), the NCCL arm next to the peer-memory arm, strong scaling of
the fixed 40^3 x 256 lattice, config 5 (48^3 x 96 Wilson CG, t x z split), time to solution,
the multi-shift CG, and parity against the oracle (every site of one global dslash, the full
CG residual history).

`python bench.py --gpus N` without torchrun re-launches itself through torch.distributed.run
(one process per GPU).  QDPB_BENCH_ONE_GPU=1 puts every rank on cuda:0 (a functional check of
the N > 1 path on a one-GPU box: peer communicator, torch.distributed over gloo; its timings
mean nothing).

--impl reference times the oracle (the tier's reference arm) on the same config and metric.
"""
from __future__ import annotations

import argparse
import json
import os
import shutil
import socket
import statistics
import subprocess
import sys
import time
import traceback

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "Wilson dslash GFLOPS & HBM GB/s (fp64/fp32) at 1/2/4/8 B200; CG iters/s"
LOCAL = (40, 40, 40, 32)
STRONG_GLOBAL = (40, 40, 40, 256)
MASS, CSW = 0.1, 1.0
HBM_FALLBACK = 6650.0  # GB/s, B200_PROFILING.md fallback (used only without MEASURED_PEAKS.json)
NVLINK_GBS = 900.0     # NVLink 5 per GPU per direction (task statement)
SEED_U, SEED_B, SEED_RANK = 1004, 2005, 7919


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


def halo_bytes_per_eo_dslash(L, P, prec_bytes: int = 8) -> int:
    """Bytes one rank sends per EO dslash: both faces of every dim with more than one rank, one
    half spinor (12 reals) per face site of the input parity (SURVEY.md 8(d) "halo")."""
    V = L[0] * L[1] * L[2] * L[3]
    return sum(2 * (V // L[mu] // 2) * 12 * prec_bytes for mu in range(4) if P[mu] > 1)


# ---------------------------------------------------------------- helpers
def measured_peak():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "MEASURED_PEAKS.json hbm_gbs (torch copy, measured)"
    return HBM_FALLBACK, "B200_PROFILING.md fallback 6.65 TB/s"


def host_cores() -> int:
    return len(os.sched_getaffinity(0))


class Clocks:
    """nvidia-smi sampling during the timed region (B200_PROFILING.md clocks line)."""

    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int, rank: int):
        self.index = index
        self.proc = None
        self.path = os.path.join(ROOT, "gpurun_out", f"clocks_rank{rank}.csv")

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
    U = fieldgen.random_gauge(L, SEED_U + SEED_RANK * rank)
    b = fieldgen.random_spinor(L, SEED_B + SEED_RANK * rank)
    return U, b


def _site_err(got, ref):
    import numpy as np
    g = got.reshape(len(got), -1)
    o = ref.reshape(len(ref), -1)
    return float(np.max(np.linalg.norm(g - o, axis=1) / np.linalg.norm(o, axis=1)))


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
    oracle.set_threads(host_cores())
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
    sample = (f"oracle/oracle.c even-odd clover CGNR on one {'x'.join(map(str, L))} sub-lattice, {args.ref_iters} iteration(s) "
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
    tag = "x".join(map(str, LOCAL))
    return {"workload": f"BASELINE config 4 (40^3x256 production lattice) as weak scaling: {tag} sites per GPU, "
                        "t-split; even-odd Wilson-clover CGNR solve, fixed iterations",
            "global_lattice": "x".join(map(str, gl)), "local_lattice": "x".join(map(str, LOCAL)),
            "operator": f"Wilson-clover m={MASS} c_SW={CSW}, hot random SU(3) gauge field",
            "gauge_storage": "reconstruct-12" if getattr(args, "recon", 18) == 12 else "full 3x3 (18 reals)",
            "cg_iters_per_step": args.iters,
            "parallelism": f"t-split x{world} ({getattr(args, 'comm', 'peer')} halos)" if world > 1 else "single GPU",
            "l2": "inputs larger than L2 (gauge 1.18 GB + clover 1.2 GB + 6 fermion vectors per GPU), no flush"}


# ---------------------------------------------------------------- native arm
class Bench:
    """State shared by the measurements of one rank."""

    def __init__(self, args, rank, world, local_rank):
        import torch
        import torch.distributed as dist
        from paper_1408_5925_b200 import dist as qdist
        from paper_1408_5925_b200 import qdpb as q
        self.args, self.rank, self.world = args, rank, world
        self.q, self.qdist, self.torch, self.dist = q, qdist, torch, dist
        # QDPB_BENCH_ONE_GPU=1: every rank on cuda:0 (functional test of the N > 1 path on a
        # one-GPU box; peer communicator only, torch.distributed over gloo -- timings mean nothing)
        self.one_gpu = os.environ.get("QDPB_BENCH_ONE_GPU") == "1"
        self.dev = 0 if self.one_gpu else local_rank
        torch.cuda.set_device(self.dev)
        if world > 1:
            if self.one_gpu:
                if args.comm != "peer":
                    raise SystemExit("QDPB_BENCH_ONE_GPU needs --comm peer (NCCL refuses two ranks on one GPU)")
                dist.init_process_group("gloo")
            else:
                dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
        # one explicit stream shared by the library (its context stream) and torch's timing events,
        # so the events are ordered with the kernels they bracket
        self.stream = torch.cuda.Stream()
        torch.cuda.set_stream(self.stream)
        self.notes = []

    # ---- small utilities
    def barrier(self):
        if self.world > 1:
            self.dist.barrier()

    def sync(self):
        self.barrier()
        self.torch.cuda.synchronize()

    def max_all(self, v):
        return self.qdist.max_over_ranks(v)

    def sum_all(self, v):
        return self.qdist.sum_over_ranks(v)

    def all_ok(self, ok: bool) -> bool:
        return self.qdist.max_over_ranks(0.0 if ok else 1.0) == 0.0

    def make_ctx(self, gdims, P, comm):
        q = self.q
        if comm == "peer":  # no NCCL on the data path: halos, sums, shifts through peer memory
            return self.qdist.bootstrap_peer(gdims, P, stream=self.stream)
        ctx = self.qdist.bootstrap(gdims, P, stream=self.stream)
        q.qdp_set_option(ctx, q.QDP_OPT_P2P, 0)
        return ctx

    def event_time(self, fn, n=1):
        """max over ranks of the CUDA-event time (ms) of fn() run n times, synchronised on both sides"""
        torch = self.torch
        self.sync()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(self.stream)
        for _ in range(n):
            fn()
        e1.record(self.stream)
        torch.cuda.synchronize()
        return self.max_all(e0.elapsed_time(e1))

    def profiled(self, ctx, fn, n, cls):
        """(launches, ms) of kernel class `cls` over n calls of fn (CUDA events per launch)"""
        q = self.q
        q.qdp_synchronize(ctx)
        q.qdp_profile_reset(ctx)
        q.qdp_set_option(ctx, q.QDP_OPT_PROFILE, 1)
        for _ in range(n):
            fn()
        nl, ms = q.qdp_profile_query(ctx, cls)
        f, b = q.qdp_profile_work(ctx, cls)
        q.qdp_set_option(ctx, q.QDP_OPT_PROFILE, 0)
        return nl, ms, f, b

    def eo_dslash_us(self, ctx, fU, prec, n=20):
        """mean live launch time (us) of one EO dslash out_e = H_eo psi_o (max over ranks)"""
        q = self.q
        fi = q.qdp_field_alloc(ctx, q.QDP_FERMION, prec, q.QDP_ODD)
        fo = q.qdp_field_alloc(ctx, q.QDP_FERMION, prec, q.QDP_EVEN)
        try:
            for _ in range(12):  # let the tuner's probes finish before the timing
                q.qdp_dslash(fo, fU, fi, q.QDP_EVEN)
                q.qdp_synchronize(ctx)
            self.sync()
            ms = self.event_time(lambda: q.qdp_dslash(fo, fU, fi, q.QDP_EVEN), n)
            q.qdp_synchronize(ctx)
            return ms / n * 1e3
        finally:
            q.qdp_field_free(fi)
            q.qdp_field_free(fo)


def _section(b, name, fn):
    """run an optional measurement; a failure is reported in the line, not fatal (all ranks)"""
    try:
        return fn()
    except Exception as e:  # noqa: BLE001 -- any failure of an extra must not lose the main line
        b.notes.append(f"{name}: {type(e).__name__}: {e}")
        if os.environ.get("QDPB_BENCH_DEBUG"):
            traceback.print_exc()
        return {"error": f"{type(e).__name__}: {e}"}


def run_native(args, rank, world, local_rank):
    import numpy as np

    import fieldgen
    from paper_1408_5925_b200 import exprs as qexprs

    b = Bench(args, rank, world, local_rank)
    q, qdist, torch, stream = b.q, b.qdist, b.torch, b.stream
    L = LOCAL
    Vh = L[0] * L[1] * L[2] * L[3] // 2
    gdims = (L[0], L[1], L[2], L[3] * world)
    P = qdist.proc_grid_for(world, gdims, split=(3,))
    comm = args.comm
    try:
        ctx = b.make_ctx(gdims, P, comm)
        ok = True
    except Exception as e:  # noqa: BLE001
        ok, err = False, e
    if world > 1 and not b.all_ok(ok):  # every rank switches together
        if comm == "peer" and not b.one_gpu:
            b.notes.append(f"peer communicator unavailable ({err if not ok else 'on another rank'}); NCCL arm is main")
            if ok:
                q.qdp_finalize(ctx)
            comm = args.comm = "nccl"
            ctx = b.make_ctx(gdims, P, comm)
        else:
            raise SystemExit(f"context creation failed: {err if not ok else 'on another rank'}")
    elif not ok:
        raise err
    q.qdp_set_option(ctx, q.QDP_OPT_OVERLAP, 0 if args.no_overlap else 1)

    U, bsrc = gen_fields(L, rank)
    fU = q.qdp_field_alloc(ctx, q.QDP_GAUGE12 if args.recon == 12 else q.QDP_GAUGE, q.QDP_F64, q.QDP_ALL)
    fb = q.qdp_field_alloc(ctx, q.QDP_FERMION, q.QDP_F64, q.QDP_ALL)
    fx = q.qdp_field_alloc(ctx, q.QDP_FERMION, q.QDP_F64, q.QDP_ALL)
    fA = q.qdp_field_alloc(ctx, q.QDP_CLOVER, q.QDP_F64, q.QDP_ALL)
    fAi = q.qdp_field_alloc(ctx, q.QDP_CLOVER, q.QDP_F64, q.QDP_EVEN)
    q.qdp_field_import(fU, U)
    q.qdp_field_import(fb, bsrc)
    q.qdp_clover_build(fA, fAi, fU, MASS, CSW)

    def step():
        return q.qdp_cg_solve(fx, fb, fU, fA, fAi, mass=MASS, tol=0.0, maxit=args.iters)

    for k in range(args.warmup):
        if k == args.warmup - 1:  # fills the library's CUDA-event pool before the profiled timed region
            q.qdp_set_option(ctx, q.QDP_OPT_PROFILE, 1)
        step()
    q.qdp_set_option(ctx, q.QDP_OPT_PROFILE, 0)

    # ---- timed region: K solves, fields resident in HBM, a CUDA-event pair around every launch on
    # the launching stream (the roofline's live launch durations and the breakdown by kernel class)
    b.sync()
    q.qdp_profile_reset(ctx)
    q.qdp_set_option(ctx, q.QDP_OPT_PROFILE, 1)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with Clocks(b.dev, rank) as clk:
        e0.record(stream)
        for _ in range(args.steps):
            r = step()
        e1.record(stream)
        torch.cuda.synchronize()
    b.barrier()
    ms = e0.elapsed_time(e1)
    f_all, b_all = q.qdp_profile_work(ctx, -1)
    n_all, ms_all = q.qdp_profile_query(ctx, -1)
    n_dsl, ms_dsl = q.qdp_profile_query(ctx, q.QDP_PK_DSLASH)
    f_dsl, b_dsl = q.qdp_profile_work(ctx, q.QDP_PK_DSLASH)
    assert abs(f_all - cg_flops(Vh, args.iters) * args.steps) <= 1e-9 * f_all, (f_all, cg_flops(Vh, args.iters))
    ms_max = b.max_all(ms)
    flops_job = b.sum_all(f_all)
    ms_p = ms
    breakdown = {}
    for name, cls in (("dslash", q.QDP_PK_DSLASH), ("dslash_exterior", q.QDP_PK_DSLASH_EXT), ("pack", q.QDP_PK_PACK),
                      ("blas", q.QDP_PK_BLAS), ("reduce", q.QDP_PK_REDUCE), ("clover", q.QDP_PK_CLOVER),
                      ("layout", q.QDP_PK_LAYOUT)):
        n_c, ms_c = q.qdp_profile_query(ctx, cls)
        if n_c:
            _, b_c = q.qdp_profile_work(ctx, cls)
            breakdown[name] = {"launches": n_c, "ms": ms_c, "share_of_step": ms_c / ms,
                               "gbs": b_c / (ms_c * 1e-3) * 1e-9 if ms_c > 0 else None}
    breakdown["gaps_and_other"] = {"ms": ms - ms_all, "share_of_step": (ms - ms_all) / ms}
    breakdown["step_algorithmic_gbs"] = b_all / (ms * 1e-3) * 1e-9
    breakdown["step_frac_of_measured_hbm"] = breakdown["step_algorithmic_gbs"] / measured_peak()[0]
    q.qdp_set_option(ctx, q.QDP_OPT_PROFILE, 0)
    # the same K solves once more without the per-launch events (their cost on the step, for reference)
    b.sync()
    e2, e3 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e2.record(stream)
    for _ in range(args.steps):
        step()
    e3.record(stream)
    torch.cuda.synchronize()
    ms_u = b.max_all(e2.elapsed_time(e3))
    breakdown["without_per_launch_events"] = {"ms_per_step": ms_u / args.steps,
                                             "value": flops_job / (ms_u * 1e-3) * 1e-9, "unit": "GFLOPS"}
    value = flops_job / (ms_max * 1e-3) * 1e-9

    # ---- parity of this exact configuration against the oracle
    parity = {}
    if args.check:
        parity["dslash_every_site"] = _section(b, "parity_dslash", lambda: parity_dslash(b, ctx, fU, fb, U, bsrc, P))
        if world == 1:
            parity["cg_full_history"] = _section(
                b, "parity_cg", lambda: parity_cg_full(b, ctx, fx, fb, fU, fA, fAi, U, bsrc, L))
        else:
            parity["cg_full_history_small"] = _section(b, "parity_cg_small", lambda: parity_cg_small(b, comm))

    # ---- e2e: the same solves through the C ABI from pinned host memory
    e2e = _section(b, "e2e", lambda: measure_e2e(b, ctx, fU, fA, fAi, fb, fx, bsrc, Vh))

    # ---- the metric's plain Wilson dslash in both precisions (not the step)
    dsl = _section(b, "eo_dslash_plain", lambda: measure_plain_dslash(b, ctx, fU, U, Vh, qexprs))

    # ---- halo: bytes, NVLink rates, overlap on / off (Fig. 6), local-only kernel
    halo = None
    if world > 1:
        halo = _section(b, "halo", lambda: measure_halo(b, ctx, fU, U, P, comm))

    # ---- the other communicator as a second arm (NCCL send/recv + allreduce vs peer memory)
    arms = None
    if world > 1 and not args.no_arms:
        arms = {comm: {"value": value, "unit": "GFLOPS", "ms_per_step": ms_max / args.steps,
                       "cg_iters_per_s": args.iters * args.steps / (ms_max * 1e-3)}}
        other = "nccl" if comm == "peer" else "peer"
        if not (b.one_gpu and other == "nccl"):
            arms[other] = _section(b, f"arm_{other}", lambda: measure_arm(b, other, gdims, P, U, bsrc, Vh))

    # ---- strong scaling of the fixed 40^3 x 256 lattice, config 5 (48^3 x 96, t x z)
    strong = None if args.no_strong else _section(b, "strong", lambda: measure_strong(b, comm))
    cfg5 = None if args.no_config5 else _section(b, "config5", lambda: measure_config5(b, comm))

    # ---- time to solution at tol 1e-10 (not the step): fp64 CG vs the mixed-precision CG
    tts = _section(b, "tts", lambda: measure_tts(b, ctx, fU, fA, fAi, fb, fx, U, bsrc)) if args.tts else None

    # ---- multi-shift CG (the RHMC solver; not the step): all shifts kept active (tol = 0)
    msh = _section(b, "multishift", lambda: measure_multishift(b, ctx, fU, fA, fAi, bsrc, L, Vh)) \
        if args.ms_shifts > 0 else None

    # ---- CPU baseline (oracle on rank 0's sub-lattice, all host cores)
    cpu = None
    if not args.no_cpu:
        cpu = _section(b, "cpu_baseline", lambda: measure_cpu(b, U, bsrc, L, Vh))

    peak, peak_src = measured_peak()
    us_dsl = ms_dsl / n_dsl * 1e3
    gbs = (b_dsl / n_dsl) / (us_dsl * 1e-6) * 1e-9
    traffic, traffic_note = None, None
    tp = os.path.join(ROOT, "profiles", "dslash_ncu_traffic.json")
    if os.path.exists(tp) and world == 1:
        with open(tp) as f:
            traffic = json.load(f).get("dram_bytes_per_launch")
        traffic_note = "ncu --set full capture of the same kernel on one GPU (profiles/)"
    elif world > 1:
        traffic_note = "null at N > 1: ncu captures are single-GPU (see profiles/ for the N = 1 capture)"
    out = {
        "metric": METRIC, "value": value, "unit": "GFLOPS", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms_max / args.steps, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic (seeded hot random SU(3) gauge field, Gaussian source)",
        "config": config_dict(args, world),
        "cg_iters_per_s": args.iters * args.steps / (ms_max * 1e-3),
        "dslash": {"launches": n_dsl, "us_per_launch": us_dsl, "gflops_per_gpu": f_dsl / n_dsl / (us_dsl * 1e-6) * 1e-9,
                   "gbs_compulsory_per_gpu": gbs, "bytes_per_site": (b_dsl / n_dsl) / Vh,
                   "share_of_step": ms_dsl / ms_p, "frac_of_8TBs": gbs / 8000.0},
        "roofline": {"bound": "hbm", "achieved": gbs, "peak": peak, "unit": "GB/s", "frac": gbs / peak,
                     "traffic": traffic, "traffic_note": traffic_note,
                     "kernel": "dslash_kernel<double> (fused EO hopping term + clover epilogue)",
                     "peak_source": peak_src},
        "e2e": e2e,
        "gpu_launches": n_all,
        "step_breakdown": breakdown,
        "clocks": clk.summary(),
        "cpu_baseline": cpu,
        "parity": parity,
        "eo_dslash_plain": dsl,
        "halo": halo if world > 1 else "none (one GPU, periodic wrap in-kernel)",
        "overlap": (halo or {}).get("overlap") if isinstance(halo, dict) else (not args.no_overlap),
        "arms": arms,
        "strong_40x40x40x256": strong,
        "config5_48x48x48x96": cfg5,
        "time_to_solution_1e-10": tts,
        "multishift_cg": msh,
    }
    if b.notes:
        out["notes"] = b.notes
    if rank == 0:
        print(json.dumps(out), flush=True)
    for f in (fU, fb, fx, fA, fAi):
        q.qdp_field_free(f)
    q.qdp_finalize(ctx)
    if world > 1:
        b.dist.destroy_process_group()


# ---------------------------------------------------------------- measurements
def parity_dslash(b, ctx, fU, fb, U, bsrc, P):
    """Every site of one full-lattice dslash of the timed configuration against the oracle.
    Each rank checks its own sub-lattice: the oracle runs on the rank's sites plus the
    neighbours' adjacent time slices (regenerated from their counter-based seeds), i.e. a
    lattice of extent L_t + 2 whose inner slices are exactly this rank's part of the global
    hopping term (t split: x, y, z are not partitioned).  Ranks run concurrently."""
    import numpy as np

    import fieldgen
    import oracle
    q = b.q
    assert P[0] == P[1] == P[2] == 1
    L = LOCAL
    V3 = L[0] * L[1] * L[2]
    rm, rp = (b.rank - 1) % b.world, (b.rank + 1) % b.world
    lo_U = fieldgen.random_gauge_sites(SEED_U + SEED_RANK * rm, (L[3] - 1) * V3, V3)
    lo_b = fieldgen.random_spinor_sites(SEED_B + SEED_RANK * rm, (L[3] - 1) * V3, V3)
    hi_U = fieldgen.random_gauge_sites(SEED_U + SEED_RANK * rp, 0, V3)
    hi_b = fieldgen.random_spinor_sites(SEED_B + SEED_RANK * rp, 0, V3)
    Lx = (L[0], L[1], L[2], L[3] + 2)
    oracle.set_threads(max(1, host_cores() // b.world))
    t0 = time.perf_counter()
    ref = oracle.hopping(np.concatenate([lo_U, U, hi_U]), np.concatenate([lo_b, bsrc, hi_b]), Lx, -1)[V3:V3 * (L[3] + 1)]
    t_orc = time.perf_counter() - t0
    fo = q.qdp_field_alloc(ctx, q.QDP_FERMION, q.QDP_F64, q.QDP_ALL)
    try:
        q.qdp_dslash(fo, fU, fb, q.QDP_ALL)
        err = _site_err(q.qdp_field_export(fo), ref)
    finally:
        q.qdp_field_free(fo)
    err = b.max_all(err)
    return {"max_site_rel_err": err, "tol": 1e-13, "pass": err <= 1e-13, "sites": V3 * L[3] * b.world,
            "what": "full-lattice H psi of the bench fields, every site of the global lattice (each rank vs the "
                    "oracle on its sub-lattice + the neighbours' adjacent slices)",
            "oracle_seconds": t_orc}


def parity_cg_full(b, ctx, fx, fb, fU, fA, fAi, U, bsrc, L):
    """N = 1: the step's solve (all args.iters iterations) vs oracle.cg_solve: every residual
    history entry (reading R14: |h_gpu - h_orc| / h_orc <= 1e-10) and every site of x."""
    import numpy as np

    import oracle
    q = b.q
    oracle.set_threads(host_cores())
    n = b.args.iters
    t0 = time.perf_counter()
    _, ref = oracle_solve_timed(U, bsrc, L, n)
    t_orc = time.perf_counter() - t0
    got = q.qdp_cg_solve(fx, fb, fU, fA, fAi, mass=MASS, tol=0.0, maxit=n)
    hd = float(np.max(np.abs(got["hist"] - ref["hist"]) / ref["hist"]))
    xe = _site_err(q.qdp_field_export(fx), ref["x"])
    return {"iters": n, "iters_gpu": got["iters"], "iters_oracle": ref["iters"], "hist_max_rel_diff": hd,
            "x_max_site_rel_err": xe, "tol_hist": 1e-10,
            "pass": hd <= 1e-10 and got["iters"] == ref["iters"] == n, "oracle_seconds": t_orc,
            "lattice": "x".join(map(str, L))}


def parity_cg_small(b, comm):
    """N > 1: the full residual history of a clover CG (32 iterations) on a reduced global lattice
    16^3 x (4N), split along t over the same communicator and kernels as the step, vs the oracle
    on the global lattice (run by every rank; the full-size global solve would take the oracle
    minutes per rank)."""
    import numpy as np

    import fieldgen
    import oracle
    q, qdist = b.q, b.qdist
    G = (16, 16, 16, 4 * b.world)
    P = (1, 1, 1, b.world)
    Ug = fieldgen.random_gauge(G, 1104)
    bg = fieldgen.random_spinor(G, 2105)
    n = b.args.iters
    oracle.set_threads(max(1, host_cores() // b.world))
    A = oracle.clover_build(Ug, G, MASS, CSW)
    ref = oracle.cg_solve(Ug, bg, G, MASS, A=A, tol=0.0, maxit=n)
    c = b.make_ctx(G, P, comm)
    fs = []
    try:
        def field(kind, subset, host=None):
            f = q.qdp_field_alloc(c, kind, q.QDP_F64, subset)
            fs.append(f)
            if host is not None:
                q.qdp_field_import(f, np.ascontiguousarray(qdist.local_slice(host, G, P, b.rank)))
            return f
        fU = field(q.QDP_GAUGE, q.QDP_ALL, Ug)
        fb = field(q.QDP_FERMION, q.QDP_ALL, bg)
        fx = field(q.QDP_FERMION, q.QDP_ALL)
        fA = field(q.QDP_CLOVER, q.QDP_ALL)
        fAi = field(q.QDP_CLOVER, q.QDP_EVEN)
        q.qdp_clover_build(fA, fAi, fU, MASS, CSW)
        got = q.qdp_cg_solve(fx, fb, fU, fA, fAi, mass=MASS, tol=0.0, maxit=n)
        hd = float(np.max(np.abs(got["hist"] - ref["hist"]) / ref["hist"]))
        xe = _site_err(q.qdp_field_export(fx), qdist.local_slice(ref["x"], G, P, b.rank))
    finally:
        for f in fs:
            q.qdp_field_free(f)
        q.qdp_finalize(c)
    hd, xe = b.max_all(hd), b.max_all(xe)
    return {"global_lattice": "x".join(map(str, G)), "proc_grid": list(P), "iters": n, "hist_max_rel_diff": hd,
            "x_max_site_rel_err": xe, "tol_hist": 1e-10, "pass": hd <= 1e-10 and got["iters"] == ref["iters"] == n}


def measure_e2e(b, ctx, fU, fA, fAi, fb, fx, bsrc, Vh):
    """The same solves through the C ABI from pinned host memory, every step's source uploaded
    and every step's solution downloaded inside the timed region.  Pipelined: on a copy stream
    the upload of b_{k+1} and the download of x_{k-1} run while solve k runs; the layout
    conversions (qdp_field_import_device / export_device) run on the compute stream."""
    import numpy as np
    q, torch, stream, args = b.q, b.torch, b.stream, b.args
    k2 = args.e2e_steps if args.e2e_steps > 0 else args.steps
    hb = [torch.from_numpy(bsrc).pin_memory() for _ in range(2)]        # host sources
    hx = [torch.empty_like(hb[0]).pin_memory() for _ in range(2)]       # host solutions
    d_in = [torch.empty_like(hb[0], device="cuda") for _ in range(2)]   # device staging (host layout)
    d_out = [torch.empty_like(hb[0], device="cuda") for _ in range(2)]
    fbs = [fb, q.qdp_field_alloc(ctx, q.QDP_FERMION, q.QDP_F64, q.QDP_ALL)]
    fxs = [fx, q.qdp_field_alloc(ctx, q.QDP_FERMION, q.QDP_F64, q.QDP_ALL)]
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

    try:
        e2e_run(2)
        b.sync()
        e2, e3 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e2.record(stream)
        cs.wait_event(e2)
        e2e_run(k2)
        e3.record(cs)  # after the last download (cs is ordered after every compute step)
        torch.cuda.synchronize()
        assert np.array_equal(hx[(k2 - 1) % 2].numpy(), q.qdp_field_export(fxs[(k2 - 1) % 2]))
        ms_e2e = b.max_all(e2.elapsed_time(e3))
    finally:
        q.qdp_field_free(fbs[1])
        q.qdp_field_free(fxs[1])
    e2e_flops = b.sum_all(cg_flops(Vh, args.iters) * k2)
    nbytes = hb[0].numel() * hb[0].element_size()
    # per-solve latency through the library's host-pointer calls, nothing overlapped: qdp_field_import
    # (host -> device + layout conversion), the solve, qdp_field_export (layout + device -> host)
    hxs = np.empty_like(bsrc)
    n3 = max(2, k2 // 2)
    b.sync()
    t0 = time.perf_counter()
    for _ in range(n3):
        q.qdp_field_import(fb, bsrc)
        q.qdp_cg_solve(fx, fb, fU, fA, fAi, mass=MASS, tol=0.0, maxit=args.iters)
        q.qdp_field_export(fx, hxs)
    ms_seq = b.max_all((time.perf_counter() - t0) * 1e3)
    seq = {"value": b.sum_all(cg_flops(Vh, args.iters) * n3) / (ms_seq * 1e-3) * 1e-9, "unit": "GFLOPS",
           "ms_per_solve": ms_seq / n3, "steps": n3,
           "how": "qdp_field_import(host b) + qdp_cg_solve + qdp_field_export(host x) per step, synchronous (wall clock)"}
    return {"value": e2e_flops / (ms_e2e * 1e-3) * 1e-9, "unit": "GFLOPS", "h2d_bytes_per_step": nbytes,
            "d2h_bytes_per_step": nbytes, "steps": k2,
            "how": "pinned host b -> device every step, x -> pinned host every step, copies on a second stream "
                   "pipelined against the solves (throughput with copies hidden, not per-solve latency)",
            "unpipelined_library_calls": seq}


def measure_plain_dslash(b, ctx, fU, U, Vh, qexprs):
    """One EO application (out_e = H_eo psi_o) on the step's lattice, uncompressed links, live
    CUDA events; fp64 and fp32.  At N > 1 it includes the halo (fused peer-to-peer kernel)."""
    import numpy as np
    q, args = b.q, b.args
    dsl = {}
    for prec, tag in ((q.QDP_F64, "fp64"), (q.QDP_F32, "fp32")):
        fUp = fU if prec == q.QDP_F64 and args.recon == 18 else q.qdp_field_alloc(ctx, q.QDP_GAUGE, prec, q.QDP_ALL)
        if fUp is not fU:
            q.qdp_field_import(fUp, U.astype(np.float64 if prec == q.QDP_F64 else np.float32))
        fi = q.qdp_field_alloc(ctx, q.QDP_FERMION, prec, q.QDP_ODD)
        fo = q.qdp_field_alloc(ctx, q.QDP_FERMION, prec, q.QDP_EVEN)
        try:
            for _ in range(12):  # the tuner's probes finish on these launches, not in the timing
                q.qdp_dslash(fo, fUp, fi, q.QDP_EVEN)
                q.qdp_synchronize(ctx)
            b.sync()
            n_d, ms_d, f_d, b_d = b.profiled(ctx, lambda: q.qdp_dslash(fo, fUp, fi, q.QDP_EVEN), 20, q.QDP_PK_DSLASH)
            t_d = b.max_all(ms_d / n_d) * 1e-3
            eff = 2880 if prec == q.QDP_F64 else 1440  # Table II convention: every leaf load, no reuse (R17)
            gbs = b_d / n_d / t_d * 1e-9
            dsl[tag] = {"us_per_launch": t_d * 1e6, "gsites_per_s": Vh / t_d * 1e-9,
                        "gflops_per_gpu": f_d / n_d / t_d * 1e-9, "gflops_job": b.world * f_d / n_d / t_d * 1e-9,
                        "gbs_compulsory_per_gpu": gbs, "bytes_per_site": b_d / n_d / Vh,
                        "gbs_effective_per_gpu": eff * Vh / t_d * 1e-9,
                        "frac_of_measured_hbm": gbs / measured_peak()[0], "frac_of_8TBs": gbs / 8000.0}
            # the same operator generated at run time from its expression (qdp_jit_eval; PAPER.md
            # sections III-IV): the paper's generated-vs-hand-tuned comparison
            if b.world == 1:
                expr = qexprs.hopping()
                for _ in range(12):  # compile once, then let the paper's autotuner settle
                    q.qdp_jit_eval(fo, expr, fUp, fi)
                n_j, ms_j, f_j, b_j = b.profiled(ctx, lambda: q.qdp_jit_eval(fo, expr, fUp, fi), 20, q.QDP_PK_BLAS)
                t_j = ms_j / n_j * 1e-3
                dsl[tag]["generated"] = {"us_per_launch": t_j * 1e6, "flop_per_site": f_j / n_j / Vh,
                                         "gbs_compulsory_per_gpu": b_j / n_j / t_j * 1e-9,
                                         "speed_vs_handwritten": t_d / t_j}
        finally:
            for f in (fi, fo) + (() if fUp is fU else (fUp,)):
                q.qdp_field_free(f)
    return dsl


def measure_halo(b, ctx, fU, U, P, comm):
    """N > 1: what the halo costs.  bytes each rank sends per fp64 EO dslash; the fused kernel
    with overlap on and off (QDP_OPT_OVERLAP = 0: every block waits for the ghosts; PAPER.md
    Fig. 6); the same rank's sub-lattice in a one-rank context (no halo) for the exposed cost;
    and, with separate kernels (QDP_OPT_FUSE = 0), the packing kernel whose stores cross NVLink
    into the neighbours' ghost slots: its bytes / launch time is the achieved NVLink write rate."""
    q = b.q
    L = LOCAL
    hb = halo_bytes_per_eo_dslash(L, P)
    out = {"comm": comm, "proc_grid": list(P), "bytes_per_eo_dslash_per_gpu": hb}
    t_on = b.eo_dslash_us(ctx, fU, q.QDP_F64)
    q.qdp_set_option(ctx, q.QDP_OPT_OVERLAP, 0)
    try:
        t_off = b.eo_dslash_us(ctx, fU, q.QDP_F64)
    finally:
        q.qdp_set_option(ctx, q.QDP_OPT_OVERLAP, 0 if b.args.no_overlap else 1)
    out["overlap"] = {"on_us": t_on, "off_us": t_off, "speedup_on_vs_off": t_off / t_on,
                      "what": "fp64 EO dslash, max over ranks; off = no interior/halo overlap"}
    out["demand_gbs_while_overlapped"] = hb / (t_on * 1e-6) * 1e-9
    out["demand_frac_of_nvlink_900"] = out["demand_gbs_while_overlapped"] / NVLINK_GBS
    # local-only: this rank's sub-lattice with periodic wrap, no halo (same GPU, same kernel)
    c1 = b.q.qdp_init(L, stream=b.stream)
    try:
        fU1 = q.qdp_field_alloc(c1, q.QDP_GAUGE, q.QDP_F64, q.QDP_ALL)
        q.qdp_field_import(fU1, U)
        t_loc = b.eo_dslash_us(c1, fU1, q.QDP_F64)
        q.qdp_field_free(fU1)
    finally:
        q.qdp_finalize(c1)
    out["local_only_us"] = t_loc
    out["exposed_halo_us"] = t_on - t_loc
    out["efficiency_vs_local"] = t_loc / t_on
    if comm == "peer" or q.qdp_get_option(ctx, q.QDP_OPT_P2P):
        q.qdp_set_option(ctx, q.QDP_OPT_FUSE, 0)
        fi = q.qdp_field_alloc(ctx, q.QDP_FERMION, q.QDP_F64, q.QDP_ODD)
        fo = q.qdp_field_alloc(ctx, q.QDP_FERMION, q.QDP_F64, q.QDP_EVEN)
        try:
            for _ in range(5):
                q.qdp_dslash(fo, fU, fi, q.QDP_EVEN)
            b.sync()
            n_p, ms_p, _, _ = b.profiled(ctx, lambda: q.qdp_dslash(fo, fU, fi, q.QDP_EVEN), 20, q.QDP_PK_PACK)
            t_sep = b.eo_dslash_us(ctx, fU, q.QDP_F64)
        finally:
            q.qdp_set_option(ctx, q.QDP_OPT_FUSE, 1)
            q.qdp_field_free(fi)
            q.qdp_field_free(fo)
        t_pack = b.max_all(ms_p / n_p) * 1e-3  # one pack launch per partitioned dim
        per_launch = hb / max(1, sum(1 for m in range(4) if P[m] > 1))
        out["separate_kernels"] = {"eo_dslash_us": t_sep, "pack_us_per_launch": t_pack * 1e6,
                                   "pack_nvlink_store_gbs": per_launch / t_pack * 1e-9,
                                   "pack_frac_of_nvlink_900": per_launch / t_pack * 1e-9 / NVLINK_GBS}
    return out


def measure_arm(b, comm, gdims, P, U, bsrc, Vh):
    """The CG step through the other communicator: a second context with its own fields."""
    q, args = b.q, b.args
    c = b.make_ctx(gdims, P, comm)
    fs = []
    try:
        def field(kind, subset, host=None):
            f = q.qdp_field_alloc(c, kind, q.QDP_F64, subset)
            fs.append(f)
            if host is not None:
                q.qdp_field_import(f, host)
            return f
        fU = field(q.QDP_GAUGE, q.QDP_ALL, U)
        fb = field(q.QDP_FERMION, q.QDP_ALL, bsrc)
        fx = field(q.QDP_FERMION, q.QDP_ALL)
        fA = field(q.QDP_CLOVER, q.QDP_ALL)
        fAi = field(q.QDP_CLOVER, q.QDP_EVEN)
        q.qdp_clover_build(fA, fAi, fU, MASS, CSW)

        def step():
            q.qdp_cg_solve(fx, fb, fU, fA, fAi, mass=MASS, tol=0.0, maxit=args.iters)
        for _ in range(2):
            step()
        n = max(3, args.steps // 2)
        ms = b.event_time(step, n)
        t_on = b.eo_dslash_us(c, fU, q.QDP_F64)
        q.qdp_set_option(c, q.QDP_OPT_OVERLAP, 0)
        t_off = b.eo_dslash_us(c, fU, q.QDP_F64)
    finally:
        for f in fs:
            q.qdp_field_free(f)
        q.qdp_finalize(c)
    flops = b.sum_all(cg_flops(Vh, args.iters) * n)
    return {"value": flops / (ms * 1e-3) * 1e-9, "unit": "GFLOPS", "ms_per_step": ms / n,
            "cg_iters_per_s": args.iters * n / (ms * 1e-3),
            "eo_dslash_fp64_us": {"overlap_on": t_on, "overlap_off": t_off},
            "how": ("NCCL: pack kernel -> ncclSend/ncclRecv on a comm stream || interior kernel -> exterior "
                    "kernels; global sums by ncclAllGather + rank-ordered sum" if comm == "nccl" else
                    "peer memory: one fused kernel per EO dslash, sums by one peer kernel")}


def _device_fields(b, c, L, seed, clover):
    """fields of a timing-only workload generated on the GPU (fieldgen.random_gauge_torch)"""
    import fieldgen
    q = b.q
    fU = q.qdp_field_alloc(c, q.QDP_GAUGE, q.QDP_F64, q.QDP_ALL)
    t = fieldgen.random_gauge_torch(L, seed + SEED_RANK * b.rank)
    q.qdp_field_import_device(fU, t)
    q.qdp_synchronize(c)
    del t
    fb = q.qdp_field_alloc(c, q.QDP_FERMION, q.QDP_F64, q.QDP_ALL)
    t = fieldgen.random_spinor_torch(L, seed + 1 + SEED_RANK * b.rank)
    q.qdp_field_import_device(fb, t)
    q.qdp_synchronize(c)
    del t
    b.torch.cuda.empty_cache()
    fx = q.qdp_field_alloc(c, q.QDP_FERMION, q.QDP_F64, q.QDP_ALL)
    fA = fAi = None
    if clover:
        fA = q.qdp_field_alloc(c, q.QDP_CLOVER, q.QDP_F64, q.QDP_ALL)
        fAi = q.qdp_field_alloc(c, q.QDP_CLOVER, q.QDP_F64, q.QDP_EVEN)
        q.qdp_clover_build(fA, fAi, fU, MASS, CSW)
    return [f for f in (fU, fb, fx, fA, fAi)]


def _cg_rate(b, c, fields, iters, Vh, clover, reps=3):
    """CG throughput: solves of `iters` and of 2 x `iters` iterations (tol = 0); iterations/s is the
    marginal rate (iters / (t(2 iters) - t(iters))), so the per-solve set-up and the solution's
    reconstruction + true residual do not count as iterations."""
    q = b.q
    fU, fb, fx, fA, fAi = fields

    def solve(n):
        return lambda: q.qdp_cg_solve(fx, fb, fU, fA, fAi, mass=MASS, tol=0.0, maxit=n)
    solve(iters)()
    q.qdp_profile_reset(c)
    ms1 = b.event_time(solve(iters), reps) / reps
    f_w, b_w = q.qdp_profile_work(c, -1)
    ms2 = b.event_time(solve(2 * iters), reps) / reps
    flops = b.sum_all(cg_flops(Vh, iters, clover))
    rate = iters / ((ms2 - ms1) * 1e-3)
    return {"cg_iters": iters, "ms_per_solve": ms1, "ms_per_solve_2x": ms2, "cg_iters_per_s": rate,
            "ms_per_iter": 1e3 / rate, "gflops_job": flops / (ms1 * 1e-3) * 1e-9,
            "algorithmic_gbs_per_gpu_whole_solve": b_w / reps / (ms1 * 1e-3) * 1e-9,
            "frac_of_measured_hbm_whole_solve": b_w / reps / (ms1 * 1e-3) * 1e-9 / measured_peak()[0]}


def measure_strong(b, comm):
    """Strong scaling: the fixed 40^3 x 256 lattice (config 4 as stated) split along t over the N
    ranks; fp64 EO dslash and a clover CG with a fixed iteration count.  Timing-only fields
    generated on the GPU."""
    q, qdist = b.q, b.qdist
    G = STRONG_GLOBAL
    P = qdist.proc_grid_for(b.world, G, split=(3,))
    L = tuple(G[m] // P[m] for m in range(4))
    Vh = L[0] * L[1] * L[2] * L[3] // 2
    c = b.make_ctx(G, P, comm)
    fields = []
    try:
        fields = _device_fields(b, c, L, 3004, clover=True)
        t_d = b.eo_dslash_us(c, fields[0], q.QDP_F64)
        cg = _cg_rate(b, c, fields, b.args.strong_iters, Vh, True)
    finally:
        for f in fields:
            if f is not None:
                q.qdp_field_free(f)
        q.qdp_finalize(c)
    gflops = b.world * 1320.0 * Vh / (t_d * 1e-6) * 1e-9
    return {"global_lattice": "x".join(map(str, G)), "proc_grid": list(P), "local_lattice": "x".join(map(str, L)),
            "eo_dslash_fp64": {"us": t_d, "gflops_job": gflops,
                               "gbs_compulsory_per_gpu": 1536.0 * Vh / (t_d * 1e-6) * 1e-9},
            "clover_cg": cg, "scaling": "strong (total work fixed)", "fields": "generated on the GPU (timing only)"}


def measure_config5(b, comm):
    """BASELINE config 5: 48^3 x 96 even-odd Wilson CG (fp64) over the N ranks with the t x z
    decomposition of dist.config5_grid (8 ranks: P = (1,1,2,4), local 48 x 48 x 24 x 24), halos
    overlapped inside the fused kernel, global sums every iteration.  Timing-only fields."""
    q, qdist = b.q, b.qdist
    G = qdist.CONFIG5_DIMS
    P = qdist.config5_grid(b.world)
    L = tuple(G[m] // P[m] for m in range(4))
    Vh = L[0] * L[1] * L[2] * L[3] // 2
    c = b.make_ctx(G, P, comm)
    fields = []
    out = {"global_lattice": "x".join(map(str, G)), "proc_grid": list(P), "local_lattice": "x".join(map(str, L)),
           "operator": f"Wilson m={MASS}", "fields": "generated on the GPU (timing only)"}
    try:
        fields = _device_fields(b, c, L, 5005, clover=False)
        out["eo_dslash_fp64_us"] = b.eo_dslash_us(c, fields[0], q.QDP_F64)
        out.update(_cg_rate(b, c, fields, b.args.c5_iters, Vh, False))
    finally:
        for f in fields:
            if f is not None:
                q.qdp_field_free(f)
        q.qdp_finalize(c)
    if b.world == 1:  # one rank's sub-lattice of the 8-GPU run, through the halo path (self-halo z x t)
        out["rank_sublattice_selfhalo_zt"] = _section(b, "c5_sublattice", lambda: _c5_sublattice(b))
    return out


def _c5_sublattice(b):
    q = b.q
    L = (48, 48, 24, 24)
    Vh = L[0] * L[1] * L[2] * L[3] // 2
    c = q.qdp_init(L, stream=b.stream)
    q.qdp_set_option(c, q.QDP_OPT_SELF_HALO, 12)
    q.qdp_set_option(c, q.QDP_OPT_P2P, 1)
    fields = []
    try:
        fields = _device_fields(b, c, L, 5105, clover=False)
        out = {"lattice": "48x48x24x24", "self_halo": "z,t (peer-to-peer protocol with this rank as neighbour)",
               "eo_dslash_fp64_us": b.eo_dslash_us(c, fields[0], q.QDP_F64)}
        out.update(_cg_rate(b, c, fields, b.args.c5_iters, Vh, False))
    finally:
        for f in fields:
            if f is not None:
                q.qdp_field_free(f)
        q.qdp_finalize(c)
    return out


def measure_tts(b, ctx, fU, fA, fAi, fb, fx, U, bsrc):
    import numpy as np
    q = b.q
    fU32 = q.qdp_field_alloc(ctx, q.QDP_GAUGE, q.QDP_F32, q.QDP_ALL)
    fU32r = q.qdp_field_alloc(ctx, q.QDP_GAUGE12, q.QDP_F32, q.QDP_ALL)
    fA32 = q.qdp_field_alloc(ctx, q.QDP_CLOVER, q.QDP_F32, q.QDP_ODD)
    fAi32 = q.qdp_field_alloc(ctx, q.QDP_CLOVER, q.QDP_F32, q.QDP_EVEN)
    fU12 = q.qdp_field_alloc(ctx, q.QDP_GAUGE12, q.QDP_F64, q.QDP_ALL)
    try:
        q.qdp_field_import(fU12, U)
        U32 = U.astype(np.float32)
        q.qdp_field_import(fU32, U32)
        q.qdp_field_import(fU32r, U32)
        q.qdp_clover_build(fA32, fAi32, fU32, MASS, CSW)
        q.qdp_field_import(fb, bsrc)
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
            # 16-bit sloppy level (int16 links / clover / directions, built from the fp64 fields in the call)
            "mixed_h16_delta1e-1": lambda: q.qdp_cg_solve_mixed16(fx, fb, fU, fA, fAi, mass=MASS, tol=1e-10,
                                                                  delta=0.1, maxit=5000),
            "mixed_h16_delta1e-2": lambda: q.qdp_cg_solve_mixed16(fx, fb, fU, fA, fAi, mass=MASS, tol=1e-10,
                                                                  delta=1e-2, maxit=5000),
            "mixed_h16_delta1e-3": lambda: q.qdp_cg_solve_mixed16(fx, fb, fU, fA, fAi, mass=MASS, tol=1e-10,
                                                                  delta=1e-3, maxit=5000),
            # the same with fp64 reconstruct-12 links for the reliable updates (and the 16-bit copy)
            "mixed_h16_u12_delta1e-2": lambda: q.qdp_cg_solve_mixed16(fx, fb, fU12, fA, fAi, mass=MASS, tol=1e-10,
                                                                      delta=1e-2, maxit=5000),
            "mixed_h16_u12_delta1e-3": lambda: q.qdp_cg_solve_mixed16(fx, fb, fU12, fA, fAi, mass=MASS, tol=1e-10,
                                                                      delta=1e-3, maxit=5000),
        }
        tts = {}
        for name, fn in solvers.items():
            fn()  # warm
            res = {}
            ms = b.event_time(lambda: res.update(fn()), 1)
            tts[name] = {"ms": ms, "iters": res["iters"], "true_resid": res["true_resid"],
                         "reliable_updates": res.get("reliable")}
    finally:
        for f in (fU32, fU32r, fA32, fAi32, fU12):
            q.qdp_field_free(f)
    return tts


def measure_multishift(b, ctx, fU, fA, fAi, bsrc, L, Vh):
    import numpy as np

    import fieldgen
    q, args = b.q, b.args
    sig = [0.0] + [0.002 * 4.0 ** i for i in range(args.ms_shifts - 1)]
    fphi = q.qdp_field_alloc(ctx, q.QDP_FERMION, q.QDP_F64, q.QDP_ODD)
    xs = [q.qdp_field_alloc(ctx, q.QDP_FERMION, q.QDP_F64, q.QDP_ODD) for _ in sig]
    try:
        q.qdp_field_import(fphi, np.ascontiguousarray(bsrc[fieldgen.parity(L) == 1]))
        q.qdp_cg_solve_multishift(xs, sig, fphi, fU, fA, fAi, mass=MASS, tol=0.0, maxit=2, true_resid=False)
        res = {}
        b.sync()
        q.qdp_profile_reset(ctx)
        q.qdp_set_option(ctx, q.QDP_OPT_PROFILE, 1)
        t_ms = b.event_time(lambda: res.update(q.qdp_cg_solve_multishift(
            xs, sig, fphi, fU, fA, fAi, mass=MASS, tol=0.0, maxit=args.ms_iters, true_resid=False)), 1)
        n_u, ms_u = q.qdp_profile_query(ctx, q.QDP_PK_MSHIFT)
        _, b_u = q.qdp_profile_work(ctx, q.QDP_PK_MSHIFT)
        f_t, _ = q.qdp_profile_work(ctx, -1)
        q.qdp_set_option(ctx, q.QDP_OPT_PROFILE, 0)
    finally:
        for f in xs + [fphi]:
            q.qdp_field_free(f)
    return {"shifts": len(sig), "sigma": sig, "iters": res["iters"], "ms_per_iter": t_ms / res["iters"],
            "gflops_per_gpu": f_t / (t_ms * 1e-3) * 1e-9,
            "update_pass": {"us_per_launch": ms_u / n_u * 1e3, "bytes_per_site": b_u / n_u / Vh,
                            "gbs": b_u / (ms_u * 1e-3) * 1e-9,
                            "frac_of_measured_hbm": b_u / (ms_u * 1e-3) * 1e-9 / measured_peak()[0],
                            "share_of_solve": ms_u / t_ms}}


def measure_cpu(b, U, bsrc, L, Vh):
    """The oracle on rank 0's sub-lattice with all host cores while the other ranks wait."""
    cpu = None
    if b.rank == 0:
        import oracle
        oracle.set_threads(host_cores())
        dt, _ = oracle_solve_timed(U, bsrc, L, b.args.cpu_iters)
        cpu = {"value": cg_flops(Vh, b.args.cpu_iters) / dt * 1e-9, "unit": "GFLOPS", "cores": oracle.max_threads(),
               "kind": "oracle", "seconds": dt,
               "sample": f"oracle/oracle.c even-odd clover CGNR, same 40^3x32 (sub-)lattice and fields as rank 0, "
                         f"{b.args.cpu_iters} iterations incl. its clover inversion, setup, reconstruction and true "
                         f"residual"}
    b.barrier()
    return cpu


# ---------------------------------------------------------------- launcher
def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def relaunch(n: int) -> int:
    """`bench.py --gpus N` run without torchrun: one process per GPU through torch.distributed.run."""
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr", "127.0.0.1", "--master-port", str(_free_port()), os.path.abspath(__file__)] + sys.argv[1:]
    env = dict(os.environ, QDPB_BENCH_CHILD="1")
    return subprocess.call(cmd, env=env)


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
    ap.add_argument("--strong-iters", type=int, default=8)
    ap.add_argument("--c5-iters", type=int, default=16)
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-overlap", action="store_true")
    ap.add_argument("--no-arms", action="store_true", help="N > 1: skip the second communicator arm")
    ap.add_argument("--no-strong", action="store_true")
    ap.add_argument("--no-config5", action="store_true")
    ap.add_argument("--comm", choices=["peer", "nccl"], default="peer",
                    help="N > 1: peer-memory communicator (qdp_init_peer, default) or NCCL")
    ap.add_argument("--ms-shifts", type=int, default=12, help="multi-shift CG measurement: shifts (0: skip)")
    ap.add_argument("--ms-iters", type=int, default=20)
    ap.add_argument("--recon", type=int, choices=[18, 12], default=18,
                    help="gauge storage of the solve: 18 (default, uncompressed as in PAPER.md:292) or 12")
    ap.add_argument("--no-tts", dest="tts", action="store_false", help="skip the time-to-solution comparison")
    ap.add_argument("--check", action="store_true", default=True)
    ap.add_argument("--no-check", dest="check", action="store_false")
    ap.add_argument("--lattice", default="40,40,40,32",
                    help="per-GPU lattice of the step (default: the weak-scaling reading of config 4)")
    args = ap.parse_args()
    global LOCAL
    LOCAL = tuple(int(v) for v in args.lattice.split(","))
    assert len(LOCAL) == 4
    if args.warmup < 3:
        ap.error("--warmup must be >= 3")
    if "WORLD_SIZE" not in os.environ and args.gpus > 1:
        sys.exit(relaunch(args.gpus))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if world != args.gpus:
        ap.error(f"--gpus {args.gpus} but WORLD_SIZE={world}")
    if args.impl == "reference":
        run_reference(args, rank, world)
    else:
        run_native(args, rank, world, local_rank)


if __name__ == "__main__":
    main()
