# One GPU call: tests, bench, ncu launch list, ncu full capture of the dslash kernels.
set -x
python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests.log 2>&1
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1
python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv \
    python bench.py --steps 1 --warmup 3 --iters 8 --no-cpu --no-check > gpurun_out/ncu_launches_bench.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:dslash_kernel -s 12 -c 4 -o gpurun_out/prof_dslash_cg \
    python bench.py --steps 1 --warmup 3 --iters 2 --no-cpu --no-check > gpurun_out/ncu_full.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:dslash_kernel -s 10 -c 2 -o gpurun_out/prof_dslash_plain \
    python tools/quick_bench.py --iters 3 > gpurun_out/ncu_full_plain.log 2>&1
