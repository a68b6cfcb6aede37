for v in async_d async_df async_d3; do
  echo "=== $v" >> gpurun_out/pf.log
  for r in 18 12; do QDPB_LIB=variants/libqdpb_$v.so python tools/quick_bench.py --recon $r --iters 30 2>&1 | grep prec >> gpurun_out/pf.log; done
  QDPB_LIB=variants/libqdpb_$v.so python tools/cg_timing.py 40,40,40,32 >> gpurun_out/pf.log 2>&1
  QDPB_LIB=variants/libqdpb_$v.so python tools/cg_timing.py 40,40,40,32 --recon12 >> gpurun_out/pf.log 2>&1
done
QDPB_LIB=variants/libqdpb_async_df.so timeout 600 python -m pytest tests/test_gpu_recon12.py -x -q 2>&1 | tail -3 >> gpurun_out/pf.log
