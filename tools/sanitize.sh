# compute-sanitizer (memcheck, racecheck, synccheck) over small-lattice GPU tests of every kernel family.
SEL='tests/test_gpu_p2p.py tests/test_gpu_parity.py::test_dslash_full_lattice tests/test_gpu_parity.py::test_dslash_self_halo tests/test_gpu_parity.py::test_blas_exact_integers tests/test_gpu_parity.py::test_clover_build_shifts_of_shifts tests/test_gpu_parity.py::test_shift_bit_exact tests/test_gpu_expr.py tests/test_gpu_recon12.py tests/test_gpu_comm.py tests/test_gpu_edge.py::test_smallest_lattice_everything tests/test_gpu_edge.py::test_zero_source_and_zero_iterations tests/test_gpu_pdl.py tests/test_gpu_tuner.py::test_forced_variants_fp64_bit_identical'
for tool in memcheck racecheck synccheck; do
  echo "=== $tool"
  compute-sanitizer --tool $tool --error-exitcode 99 --target-processes all \
    python -m pytest $SEL -m gpu -x -q -k "not L4 and not bench_size and not 16" 2>&1 | tail -4
done
