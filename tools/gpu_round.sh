# One GPU call: tests, smoke, bench, ncu launch list, one ncu --set full capture of the CG dslash launches.
# (gpurun copies back at most 64 MiB of gpurun_out/: keep a single full report.)
set -x
python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests.log 2>&1
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1
python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv \
    python bench.py --steps 1 --warmup 3 --iters 8 --no-cpu --no-check --no-tts > gpurun_out/ncu_launches_bench.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:dslash_kernel -s 45 -c 4 -o gpurun_out/prof_dslash_cg \
    python bench.py --steps 1 --warmup 3 --iters 2 --no-cpu --no-check --no-tts > gpurun_out/ncu_full.log 2>&1
