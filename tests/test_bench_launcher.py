"""bench.py's launcher on CPU: `bench.py --gpus 2` without torchrun re-launches itself through
torch.distributed.run (one process per rank, 127.0.0.1 rendezvous); the reference arm then runs
on rank 0 only and prints one JSON line; the other rank exits 0 without work."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_bench_self_launch_reference_arm():
    env = {k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK")}
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "2", "--impl", "reference",
                        "--lattice", "4,4,4,4", "--steps", "2", "--warmup", "3"],
                       cwd=ROOT, env=env, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout + r.stderr
    lines = [json.loads(x) for x in r.stdout.splitlines() if x.startswith("{")]
    assert len(lines) == 1, r.stdout
    d = lines[0]
    assert d["impl"] == "reference" and d["n_gpus"] == 2 and d["steps"] == 2 and d["value"] > 0
    assert d["config"]["local_lattice"] == "4x4x4x4" and d["cpu_baseline"]["kind"] == "oracle"
    assert d["e2e"]["h2d_bytes_per_step"] == 0


def test_bench_cli_guards():
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--warmup", "2"], cwd=ROOT,
                       capture_output=True, text=True, timeout=120)
    assert r.returncode != 0 and "warmup" in r.stderr


def test_halo_and_flop_accounting():
    sys.path.insert(0, ROOT)
    import bench
    # t split of 40^3 x 32: 2 faces x 32000 face sites x 12 reals x 8 B = 6.144 MB per EO dslash
    assert bench.halo_bytes_per_eo_dslash((40, 40, 40, 32), (1, 1, 1, 8)) == 2 * 32000 * 96
    assert bench.halo_bytes_per_eo_dslash((40, 40, 40, 32), (1, 1, 1, 1)) == 0
    # config 5 at 8 ranks: z and t faces of 48 x 48 x 24 x 24, 27648 sites each
    assert bench.halo_bytes_per_eo_dslash((48, 48, 24, 24), (1, 1, 2, 4)) == 2 * 2 * 27648 * 96
    assert bench.dslash_bytes_per_site() == 1536
