# compute-sanitizer (memcheck, racecheck, synccheck) over the run-time generated kernels (qdp_jit_eval / qdp_jit_sum).
for tool in memcheck racecheck synccheck; do
  echo "=== $tool"
  compute-sanitizer --tool $tool --error-exitcode 99 --target-processes all \
    python -m pytest tests/test_gpu_jit.py -m gpu -x -q -k "not _never_" 2>&1 | tail -4
done
