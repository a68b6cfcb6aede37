# One GPU call: the ncu launch list of a short bench run and --set full captures of the CG dslash
# launches, the fused z x t / t boundary kernels, the 16-bit sloppy dslash, the fp64 reconstruct-12
# dslash and the BLAS kernels.  Summaries: python tools/make_profiles.py r02 (run here afterwards).
mkdir -p gpurun_out
N="ncu --clock-control none"
timeout 900 $N --metrics gpu__time_duration.sum --csv --log-file gpurun_out/launches.csv \
  python bench.py --steps 1 --warmup 3 --iters 8 --no-cpu --no-check --no-tts --ms-shifts 0 --no-strong --no-config5 \
  > gpurun_out/ncu_launches_bench.log 2>&1; echo launches_rc=$?
F="$N --set full --import-source on"
timeout 900 $F -k regex:dslash_kernel -s 12 -c 4 -o gpurun_out/prof_dslash_cg -f \
  python bench.py --steps 1 --warmup 3 --iters 2 --no-cpu --no-check --no-tts --ms-shifts 0 --no-strong --no-config5 \
  > gpurun_out/ncu_cg.log 2>&1; echo cg_rc=$?
for c in zt t r12; do
  timeout 600 $F -k regex:dslash_kernel -s 10 -c 1 -o gpurun_out/prof_$c -f python tools/ncu_cases.py $c > gpurun_out/ncu_$c.log 2>&1; echo ${c}_rc=$?
done
timeout 600 $F --kernel-name-base demangled -k "regex:dslash_kernel<qdpb::h16" -s 4 -c 4 -o gpurun_out/prof_h16 -f python tools/ncu_cases.py h16 > gpurun_out/ncu_h16.log 2>&1; echo h16_rc=$?
timeout 600 $F -k "regex:norm2|inner|axpy" -s 30 -c 3 -o gpurun_out/prof_blas -f python tools/ncu_cases.py blas > gpurun_out/ncu_blas.log 2>&1; echo blas_rc=$?
timeout 600 $F -k "regex:norm2" -s 20 -c 2 -o gpurun_out/prof_blas16 -f python tools/ncu_cases.py blas16 > gpurun_out/ncu_blas16.log 2>&1; echo blas16_rc=$?
ls -la gpurun_out/*.ncu-rep
# summarise here (gpurun copies back at most 64 MiB): text into gpurun_out/prof_txt, reports removed
mkdir -p gpurun_out/prof_txt
PROF_OUT=gpurun_out/prof_txt python tools/make_profiles.py r02 > gpurun_out/prof_txt/make_profiles.log 2>&1
for r in gpurun_out/prof_*.ncu-rep; do python tools/ncu_summary.py $r > gpurun_out/prof_txt/$(basename $r .ncu-rep)_detail.txt 2>&1; done
rm -f gpurun_out/*.ncu-rep
