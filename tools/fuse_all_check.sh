# fused boundary for every split (default QDPB_FUSE=2): GPU suite, sanitizers on the halo tests, halo cost
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/fa_tests.log 2>&1; echo rc=$? >> gpurun_out/fa_tests.log
for tool in racecheck synccheck memcheck; do
  echo "=== $tool" >> gpurun_out/fa_sanitize.log
  timeout 900 compute-sanitizer --tool $tool --error-exitcode 99 --target-processes all \
    python -m pytest tests/test_gpu_p2p.py tests/test_gpu_parity.py::test_dslash_self_halo -m gpu -x -q -k "not L4 and not bench_size and not 16" >> gpurun_out/fa_sanitize.log 2>&1
  echo rc=$? >> gpurun_out/fa_sanitize.log
done
for f in 0 1 2; do QDPB_FUSE=$f timeout 300 python tools/halo_overhead.py > gpurun_out/fa_halo_$f.log 2>&1; done
