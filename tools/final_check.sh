# round-end check: GPU suite, smoke, sanitizers on the halo tests, bench
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/fc_tests.log 2>&1; echo rc=$? >> gpurun_out/fc_tests.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/fc_smoke.log 2>&1; echo rc=$? >> gpurun_out/fc_smoke.log
for tool in racecheck synccheck memcheck; do
  echo "=== $tool" >> gpurun_out/fc_sanitize.log
  timeout 900 compute-sanitizer --tool $tool --error-exitcode 99 --target-processes all \
    python -m pytest tests/test_gpu_p2p.py tests/test_gpu_parity.py::test_dslash_self_halo -m gpu -x -q -k "not L4 and not bench_size and not 16" >> gpurun_out/fc_sanitize.log 2>&1
  echo rc=$? >> gpurun_out/fc_sanitize.log
done
timeout 600 python bench.py > gpurun_out/fc_bench.log 2>&1
