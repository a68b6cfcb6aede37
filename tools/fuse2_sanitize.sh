# QDPB_FUSE=2 (site-table fused boundary for every split) under the sanitizers, after the per-thread acquire
mkdir -p gpurun_out
for tool in synccheck synccheck racecheck racecheck memcheck; do
  echo "=== $tool" >> gpurun_out/f2s.log
  QDPB_FUSE=2 timeout 600 compute-sanitizer --tool $tool --error-exitcode 99 --target-processes all \
    python -m pytest tests/test_gpu_p2p.py -m gpu -q -k "not L4 and not bench_size and not 16" 2>&1 | grep -E "passed|failed|FAILED|SUMMARY|assert 0" >> gpurun_out/f2s.log
done
