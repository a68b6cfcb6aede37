set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 1500 python -m pytest tests -m gpu -q -x --durations=15 > gpurun_out/gpu_tests.log 2>&1; echo tests_rc=$?
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke_rc=$?
timeout 600 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo bench_rc=$?
timeout 600 python bench.py --impl reference --steps 2 --warmup 3 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; echo ref_rc=$?
cat gpurun_out/bench.json
tail -3 gpurun_out/gpu_tests.log
