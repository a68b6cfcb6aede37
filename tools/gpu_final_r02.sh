# One GPU call at the end of round 2: the GPU suite, smoke, the default bench, the reference arm, the
# N = 2 functional run on one GPU, the sanitizers over the halo / reduction / CG tests, and the
# measurement tools.  Outputs in gpurun_out/ (copied into profiles/ by hand).
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -q > gpurun_out/gpu_tests.log 2>&1; echo tests_rc=$?
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke_rc=$?
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo bench_rc=$?
timeout 900 python bench.py --impl reference --steps 2 --warmup 3 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; echo ref_rc=$?
QDPB_BENCH_ONE_GPU=1 timeout 900 python bench.py --gpus 2 --steps 3 > gpurun_out/bench_n2.json 2> gpurun_out/bench_n2.err; echo n2_rc=$?
timeout 300 python tools/fused_sweep.py > gpurun_out/fused_sweep.txt 2>&1
timeout 600 python tools/mixed_profile.py > gpurun_out/mixed_profile.txt 2>&1
for tool in racecheck synccheck synccheck memcheck; do
  echo "=== $tool" >> gpurun_out/sanitize.txt
  timeout 900 compute-sanitizer --tool $tool --error-exitcode 99 python -m pytest tests/test_gpu_p2p.py \
    tests/test_gpu_tuner.py -m gpu -q >> gpurun_out/sanitize.txt 2>&1
  echo rc=$? >> gpurun_out/sanitize.txt
done
grep -E "===|SUMMARY|passed|failed|rc=" gpurun_out/sanitize.txt
tail -3 gpurun_out/gpu_tests.log
