# after the per-thread acquire in block_wait_flags: GPU suite, smoke, sanitizers (synccheck x4) on the halo tests, bench
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/f2_tests.log 2>&1; echo rc=$? >> gpurun_out/f2_tests.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/f2_smoke.log 2>&1; echo rc=$? >> gpurun_out/f2_smoke.log
for tool in synccheck synccheck synccheck synccheck racecheck memcheck; do
  echo "=== $tool" >> gpurun_out/f2_sanitize.log
  timeout 600 compute-sanitizer --tool $tool --error-exitcode 99 --target-processes all \
    python -m pytest tests/test_gpu_p2p.py tests/test_gpu_parity.py::test_dslash_self_halo -m gpu -q -k "not L4 and not bench_size and not 16" 2>&1 | grep -E "passed|failed|FAILED|SUMMARY" >> gpurun_out/f2_sanitize.log
done
timeout 600 python bench.py > gpurun_out/f2_bench.log 2>&1
