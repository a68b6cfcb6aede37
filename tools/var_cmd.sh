for v in base b128m3 b128m4 b256m2 b64m6; do
  echo "=== $v" >> gpurun_out/variants.log
  QDPB_LIB=variants/libqdpb_$v.so python tools/quick_bench.py >> gpurun_out/variants.log 2>&1
  QDPB_LIB=variants/libqdpb_$v.so python tools/cg_timing.py >> gpurun_out/variants.log 2>&1
done
