# One GPU call: the whole GPU suite, smoke, the default bench, the reference arm, and the ncu launch list of a
# short bench run (profiles/r01_launches_bench.txt).
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 1800 python -m pytest tests -m gpu -q -x --durations=10 > gpurun_out/gpu_tests.log 2>&1; echo tests_rc=$?
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke_rc=$?
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo bench_rc=$?
timeout 600 python bench.py --impl reference --steps 2 --warmup 3 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; echo ref_rc=$?
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv \
    python bench.py --steps 1 --warmup 3 --iters 8 --no-cpu --no-check --no-tts --ms-shifts 0 > gpurun_out/ncu_launches_bench.log 2>&1; echo ncu_rc=$?
tail -3 gpurun_out/gpu_tests.log
cat gpurun_out/smoke.log
timeout 900 bash tools/sanitize.sh > gpurun_out/sanitize.txt 2>&1; echo san_rc=$?
QDPB_BENCH_ONE_GPU=1 timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 2 --steps 2 --warmup 3 --iters 4 --ms-iters 3 --no-tts > gpurun_out/bench_2rank_onegpu.json 2> gpurun_out/bench_2rank_onegpu.err; echo b2_rc=$?
cat gpurun_out/sanitize.txt | grep -E "===|SUMMARY|passed|failed"
