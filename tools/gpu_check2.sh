timeout 300 python -m pytest tests/test_gpu_multishift.py -x -q > gpurun_out/ms2.log 2>&1; tail -3 gpurun_out/ms2.log
QDPB_BENCH_ONE_GPU=1 timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 2 --steps 2 --warmup 3 --iters 4 --ms-iters 3 --no-tts > gpurun_out/bench_2rank_onegpu.json 2> gpurun_out/bench_2rank_onegpu.err
echo rc=$?; tail -5 gpurun_out/bench_2rank_onegpu.err
