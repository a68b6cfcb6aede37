# compute-sanitizer over a small subset of the GPU tests (memcheck, racecheck, synccheck).
for tool in memcheck racecheck synccheck; do
  echo "=== $tool"
  compute-sanitizer --tool $tool --error-exitcode 99 --target-processes all \
    python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "dslash_full_lattice and L0 or self_halo and 15-1 or test_blas and 0 or cg_history_parity and L0 or shifts_of_shifts and 8 or shift_bit_exact" 2>&1 | tail -4
done
