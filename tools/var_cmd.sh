for v in base occ_a occ_b occ_c occ_d; do
  echo "=== $v" >> gpurun_out/variants.log
  for r in 18 12; do QDPB_LIB=variants/libqdpb_$v.so python tools/quick_bench.py --recon $r --iters 30 >> gpurun_out/variants.log 2>&1; done
  QDPB_LIB=variants/libqdpb_$v.so python tools/cg_timing.py 40,40,40,32 --recon12 >> gpurun_out/variants.log 2>&1
done
