"""Turn gpurun_out/ ncu artefacts into the committed profiles/ summaries.

  python tools/make_profiles.py r01
writes
  profiles/<tag>_launches_bench.txt   per-kernel totals and shares of the ncu launch list of
                                       `bench.py --steps 1 --warmup 3 --iters 8` (cold-cache,
                                       serialised: compare SHARES, not absolute times)
  profiles/<tag>_ncu_full_<name>.txt  --set full summaries of the captured dslash launches
  profiles/dslash_ncu_traffic.json    DRAM bytes per launch of the CG-iteration dslash mix
                                       (read by bench.py for roofline.traffic)
"""
import collections
import csv
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
OUT = os.path.join(ROOT, "gpurun_out")
PROF = os.environ.get("PROF_OUT", os.path.join(ROOT, "profiles"))
tag = sys.argv[1] if len(sys.argv) > 1 else "r01"
os.makedirs(PROF, exist_ok=True)


def launches():
    path = os.path.join(OUT, "launches.csv")
    if not os.path.exists(path):
        return
    rows = list(csv.reader(open(path)))
    hdr, data = None, []
    for r in rows:
        if "Kernel Name" in r:
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            data.append(dict(zip(hdr, r)))
    agg = collections.defaultdict(lambda: [0, 0.0])
    scale = {"nsecond": 1.0, "usecond": 1e3, "msecond": 1e6, "second": 1e9}
    for d in data:
        if d["Metric Name"] != "gpu__time_duration.sum":
            continue
        v = float(d["Metric Value"].replace(",", "")) * scale.get(d["Metric Unit"], 1.0)
        n = d["Kernel Name"].split("(")[0]
        agg[n][0] += 1
        agg[n][1] += v
    tot = sum(v[1] for v in agg.values())
    lines = [f"# ncu launch list (gpu__time_duration.sum, --clock-control none) of",
             f"#   python bench.py --steps 1 --warmup 3 --iters 8 --no-cpu --no-check",
             f"# {sum(v[0] for v in agg.values())} launches, {tot / 1e6:.3f} ms total; cold-cache and serialised",
             f"# {'launches':>8} {'total ms':>10} {'share':>7} {'avg us':>9}  kernel"]
    for n, (c, t) in sorted(agg.items(), key=lambda x: -x[1][1]):
        lines.append(f"  {c:8d} {t / 1e6:10.3f} {100 * t / tot:6.1f}% {t / c / 1e3:9.1f}  {n}")
    open(os.path.join(PROF, f"{tag}_launches_bench.txt"), "w").write("\n".join(lines) + "\n")
    print("\n".join(lines))


METRICS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
           "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "launch__registers_per_thread",
           "launch__block_size", "launch__grid_size", "launch__occupancy_limit_registers",
           "sm__warps_active.avg.pct_of_peak_sustained_active", "lts__t_sector_hit_rate.pct",
           "l1tex__t_sector_hit_rate.pct", "smsp__issue_active.avg.pct_of_peak_sustained_active",
           "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
           "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
           "smsp__warp_issue_stalled_long_scoreboard_per_warp_active.pct",
           "smsp__warp_issue_stalled_lg_throttle_per_warp_active.pct",
           "smsp__warp_issue_stalled_wait_per_warp_active.pct"]


def full(name):
    rep = os.path.join(OUT, f"prof_{name}.ncu-rep")
    if not os.path.exists(rep):
        return []
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    hdr, units, data = rows[0], rows[1], rows[2:]
    idx = {h: i for i, h in enumerate(hdr)}
    recs, lines = [], [f"# ncu --set full --clock-control none summaries: {os.path.basename(rep)}"]
    for d in data:
        name_k = d[idx["Kernel Name"]].split("(")[0]
        rec = {"kernel": name_k}
        lines.append(f"\n{name_k}")
        for m in METRICS:
            if m in idx:
                lines.append(f"  {m:64s} {d[idx[m]]:>16s} {units[idx[m]]}")
                rec[m] = (d[idx[m]], units[idx[m]])
        recs.append(rec)
    open(os.path.join(PROF, f"{tag}_ncu_full_{name}.txt"), "w").write("\n".join(lines) + "\n")
    return recs


def to_bytes(v, u):
    v = float(v.replace(",", ""))
    return v * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(u, 1)


launches()
cg = full("dslash_cg")
for rep in sorted(os.listdir(OUT)):
    if rep.startswith("prof_") and rep.endswith(".ncu-rep") and rep != "prof_dslash_cg.ncu-rep":
        full(rep[len("prof_"):-len(".ncu-rep")])
if cg:
    per = [to_bytes(*r["dram__bytes_read.sum"]) + to_bytes(*r["dram__bytes_write.sum"]) for r in cg]
    json.dump({"dram_bytes_per_launch": sum(per) / len(per),
               "per_launch": [{"kernel": r["kernel"], "dram_bytes": b} for r, b in zip(cg, per)],
               "source": f"profiles/{tag}_ncu_full_dslash_cg.txt (dram__bytes_read.sum + dram__bytes_write.sum, "
                         "mean over the captured CG-solve dslash launches)"},
              open(os.path.join(PROF, "dslash_ncu_traffic.json"), "w"), indent=1)
