# GPU calls of round 2's second session (one `gpurun` call per section; outputs in gpurun_out/, the
# summaries copied into profiles/ by hand).  Usage: bash tools/gpu_r02b.sh SECTION
#   check   the GPU suite, smoke, the default bench
#   evidence  the bench's ncu launch list, the reference arm, the N = 2 functional run on one GPU
#   fused   fused boundary: face position in the visiting order (QDPB_FACE_AT) x ack before the
#           output stores; halo tests under the non-default setting  -> profiles/r02_fused_face_position.txt
#   pdl     programmatic dependent launch off / on (CG it/s), z x t with / without PDL on the fused
#           kernel (QDPB_PDL_HALO)                                    -> profiles/r02_pdl.txt
#   pipe    the cp.async hop pipeline: variant sweep, CG with forced variants, ncu --set full of the
#           fp64 reconstruct-12 dslash as register-path kernel and as pipeline -> profiles/r02_dslash_pipeline.txt
#   c5      config 5's rank sub-lattice CG: per-class times with no halo / t / z x t, and the per-launch
#           dslash times (ncu) of the CG with and without the z x t halo (and of the 40^3x32 clover CG
#           with and without the t halo)                              -> profiles/r02_halo_cg_cost.txt
#   zt      ncu --set full (+ SASS source page) of the fused z x t boundary kernel and of the main kernel
#           on config 5's rank sub-lattice
#   ack     the fused boundary with the acknowledgement by the next call and block-uniform halo
#           tests: halo / peer / PDL / mixed tests, fused sweep, config 5's CG
#   cgblas  ncu --set full of the CG's vector updates (cg_r, cg_xp)
#   h16     the 16-bit dslash with packed fp32 arithmetic vs scalar (A/B in one call), mixed-solver tests
#   compact the fused boundary kernel with one copy of its packing / face-site code: tests, sweep, config 5
#   small   the launch-variant sweep incl. the 128-register variant, tuner tests, CG it/s PDL off / on
#                                                                     -> profiles/r02_dslash_variants_pdl.txt
#   clovt   ncu --set full of the clover-xpay dslash of the 40^3x32 CG with and without the t boundary
#                                                                     -> profiles/r02_ncu_clover_xpay_t_halo.txt
set -u
mkdir -p gpurun_out/prof_txt
case "$1" in
check)
  timeout 2400 python -m pytest tests -m gpu -q > gpurun_out/gpu_tests.log 2>&1; echo tests_rc=$?
  timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke_rc=$?
  timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo bench_rc=$?
  tail -3 gpurun_out/gpu_tests.log; cat gpurun_out/smoke.log ;;
evidence)
  # the bench's ncu launch list (cold, serialised: shares), the reference arm, the N = 2 path on one GPU
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv \
    python bench.py --steps 1 --warmup 3 --iters 8 --no-cpu --no-check --no-tts --ms-shifts 0 --no-strong --no-config5 \
    > gpurun_out/ncu_launches_bench.log 2>&1; echo launches_rc=$?
  timeout 900 python bench.py --impl reference --steps 2 --warmup 3 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; echo ref_rc=$?
  QDPB_BENCH_ONE_GPU=1 timeout 900 python bench.py --gpus 2 --steps 3 > gpurun_out/bench_n2.json 2> gpurun_out/bench_n2.err; echo n2_rc=$?
  tail -c 600 gpurun_out/bench_n2.json ;;
fused)
  for cfg in "1" "0.5" "0.25" "0.75"; do
    echo "FACE_AT=$cfg" >> gpurun_out/fused_exp.txt
    QDPB_FACE_AT=$cfg timeout 300 python tools/fused_sweep.py >> gpurun_out/fused_exp.txt 2>&1
  done
  timeout 900 python -m pytest tests/test_gpu_p2p.py tests/test_gpu_peer.py tests/test_gpu_pdl.py -m gpu -q \
    > gpurun_out/fused_exp_tests.log 2>&1; echo tests_rc=$?
  cat gpurun_out/fused_exp.txt; tail -3 gpurun_out/fused_exp_tests.log ;;
pdl)
  timeout 600 python tools/pdl_cg.py > gpurun_out/pdl_cg.txt 2>&1; echo pdl_rc=$?
  timeout 600 python tools/pdl_zt.py > gpurun_out/pdl_zt.txt 2>&1
  QDPB_PDL_HALO=1 timeout 600 python tools/pdl_zt.py >> gpurun_out/pdl_zt.txt 2>&1
  cat gpurun_out/pdl_cg.txt gpurun_out/pdl_zt.txt ;;
pipe)
  timeout 900 python tools/pipe_variants.py > gpurun_out/pipe_variants.txt 2>&1; echo pipe_rc=$?
  timeout 900 python tools/pipe_cg.py > gpurun_out/pipe_cg.txt 2>&1; echo pipecg_rc=$?
  timeout 900 python tools/dslash_variants.py > gpurun_out/dslash_variants.txt 2>&1; echo var_rc=$?
  F="ncu --clock-control none --set full --import-source on"
  for c in r12main r12pipe; do
    timeout 600 $F -k regex:dslash -s 10 -c 1 -o gpurun_out/prof_$c -f python tools/ncu_cases.py $c > gpurun_out/ncu_$c.log 2>&1
    python tools/ncu_summary.py gpurun_out/prof_$c.ncu-rep > gpurun_out/prof_txt/prof_${c}_detail.txt 2>&1
  done
  rm -f gpurun_out/*.ncu-rep
  cat gpurun_out/pipe_variants.txt gpurun_out/pipe_cg.txt ;;
small)
  timeout 900 python -m pytest tests/test_gpu_tuner.py -m gpu -q > gpurun_out/o8_tests.log 2>&1; echo tests_rc=$?
  timeout 900 python tools/dslash_variants.py > gpurun_out/dslash_variants.txt 2>&1; echo var_rc=$?
  timeout 600 python tools/pdl_cg.py > gpurun_out/pdl_cg.txt 2>&1; echo pdl_rc=$?
  cat gpurun_out/dslash_variants.txt gpurun_out/pdl_cg.txt; tail -3 gpurun_out/o8_tests.log ;;
c5)
  timeout 600 python tools/c5_profile.py > gpurun_out/c5_profile.txt 2>&1; echo c5_rc=$?
  for c in c5cg c5cg0 t40cg t40cg0; do
    timeout 600 ncu --clock-control none --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
      -k regex:dslash -s 40 -c 16 --csv --log-file gpurun_out/ncu_$c.csv python tools/ncu_cases.py $c > gpurun_out/ncu_$c.log 2>&1
    echo ${c}_rc=$?
  done
  cat gpurun_out/c5_profile.txt ;;
zt)
  F="ncu --clock-control none --set full --import-source on"
  for c in c5zt c5whole; do
    timeout 600 $F -k regex:dslash -s 10 -c 1 -o gpurun_out/prof_$c -f python tools/ncu_cases.py $c > gpurun_out/ncu_$c.log 2>&1; echo ${c}_rc=$?
    python tools/ncu_summary.py gpurun_out/prof_$c.ncu-rep > gpurun_out/prof_txt/prof_${c}_detail.txt 2>&1
    ncu -i gpurun_out/prof_$c.ncu-rep --page source --csv --print-source sass > gpurun_out/prof_txt/src_$c.csv 2>&1
  done
  rm -f gpurun_out/*.ncu-rep
  grep -E "gpu__time|dram__bytes|warps_active|long_scoreboard_per|issue_active|l1tex__t_sector_hit|lts__t_sector_hit" gpurun_out/prof_txt/prof_c5*_detail.txt ;;
ack)
  timeout 900 python -m pytest tests/test_gpu_p2p.py tests/test_gpu_peer.py tests/test_gpu_pdl.py tests/test_gpu_mixed.py -m gpu -q \
    > gpurun_out/ack_tests.log 2>&1; echo tests_rc=$?
  timeout 300 python tools/fused_sweep.py > gpurun_out/ack.txt 2>&1
  timeout 300 python tools/c5_profile.py >> gpurun_out/ack.txt 2>&1
  timeout 600 python tools/pdl_zt.py >> gpurun_out/ack.txt 2>&1
  cat gpurun_out/ack.txt; tail -2 gpurun_out/ack_tests.log ;;
cgblas)
  F="ncu --clock-control none --set full --import-source on"
  timeout 600 $F -k "regex:cg_r_kernel|cg_xp_kernel" -s 40 -c 2 -o gpurun_out/prof_cgblas -f python tools/ncu_cases.py cgblas > gpurun_out/ncu_cgblas.log 2>&1; echo cgblas_rc=$?
  python tools/ncu_summary.py gpurun_out/prof_cgblas.ncu-rep > gpurun_out/prof_txt/prof_cgblas_detail.txt 2>&1
  rm -f gpurun_out/*.ncu-rep
  grep -E "Kernel Name|gpu__time|dram__bytes|warps_active|long_scoreboard_per|issue_active|registers|block_size|grid_size|barrier_per|membar_per" gpurun_out/prof_txt/prof_cgblas_detail.txt ;;
h16)
  # the 16-bit dslash with packed fp32 pairs (FFMA2) vs the scalar build (variants/libqdpb_h16_scalar.so)
  timeout 900 python -m pytest tests/test_gpu_mixed.py -m gpu -q > gpurun_out/h16_tests.log 2>&1; echo tests_rc=$?
  for v in scalar f32x2 scalar f32x2; do
    echo "== $v" >> gpurun_out/h16.txt
    if [ $v = scalar ]; then QDPB_LIB=variants/libqdpb_h16_scalar.so timeout 600 python tools/mixed_profile.py >> gpurun_out/h16.txt 2>&1
    else timeout 600 python tools/mixed_profile.py >> gpurun_out/h16.txt 2>&1; fi
  done
  cat gpurun_out/h16.txt; tail -2 gpurun_out/h16_tests.log ;;
compact)
  # the fused boundary kernel with one copy of its packing / face-site code (run-time mu)
  timeout 1500 python -m pytest tests/test_gpu_p2p.py tests/test_gpu_peer.py tests/test_gpu_pdl.py tests/test_gpu_parity.py \
    tests/test_gpu_mixed.py tests/test_gpu_recon12.py tests/test_gpu_comm.py -m gpu -q > gpurun_out/compact_tests.log 2>&1; echo tests_rc=$?
  timeout 300 python tools/fused_sweep.py > gpurun_out/compact.txt 2>&1
  timeout 300 python tools/c5_profile.py >> gpurun_out/compact.txt 2>&1
  timeout 600 python tools/pdl_zt.py >> gpurun_out/compact.txt 2>&1
  cat gpurun_out/compact.txt; tail -2 gpurun_out/compact_tests.log ;;
clovt)
  # ncu --set full of the clover-xpay dslash of the 40^3x32 clover CG with t through the fused boundary and without
  F="ncu --clock-control none --set full --import-source on"
  timeout 600 $F -k "regex:dslash_kernel<double, .int.18, .int.3, .bool.0, .bool.0, .bool.1, .bool.0>" --kernel-name-base demangled -s 2 -c 1 -o gpurun_out/prof_clovt -f python tools/ncu_cases.py t40cg > gpurun_out/ncu_clovt.log 2>&1; echo t_rc=$?
  timeout 600 $F -k "regex:dslash_kernel<double, .int.18, .int.3, .bool.0, .bool.0, .bool.0, .bool.0>" --kernel-name-base demangled -s 2 -c 1 -o gpurun_out/prof_clov0 -f python tools/ncu_cases.py t40cg0 > gpurun_out/ncu_clov0.log 2>&1; echo w_rc=$?
  for c in clovt clov0; do
    python tools/ncu_summary.py gpurun_out/prof_$c.ncu-rep > gpurun_out/prof_txt/prof_${c}_detail.txt 2>&1
    ncu -i gpurun_out/prof_$c.ncu-rep --page source --csv --print-source sass > gpurun_out/prof_txt/src_$c.csv 2>&1
  done
  rm -f gpurun_out/*.ncu-rep
  grep -E "gpu__time|dram__bytes|no_instruction_per|long_scoreboard_per|membar_per|barrier_per|wait_per|issue_active" gpurun_out/prof_txt/prof_clov*_detail.txt ;;
esac
