# repeated runs of the peer-to-peer halo tests: plain (10x) and under synccheck (3x)
mkdir -p gpurun_out
for i in $(seq 10); do timeout 300 python -m pytest tests/test_gpu_p2p.py tests/test_gpu_peer.py -m gpu -q 2>&1 | tail -1; done > gpurun_out/rep_plain.log
for i in 1 2 3; do timeout 600 compute-sanitizer --tool synccheck --target-processes all python -m pytest tests/test_gpu_p2p.py -m gpu -q -k "not L4 and not bench_size and not 16" 2>&1 | grep -E "passed|failed|FAILED"; done > gpurun_out/rep_sync.log
