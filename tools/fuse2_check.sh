# QDPB_FUSE=2 (fused boundary with a per-parity site table, any split): repeated parity runs and
# one racecheck pass, to locate the first-call failure noted in DESIGN.md §9.
mkdir -p gpurun_out
for i in 1 2 3; do
  QDPB_FUSE=2 timeout 600 python -m pytest tests/test_gpu_p2p.py tests/test_gpu_peer.py -m gpu -q -x 2>&1 | tail -3
done > gpurun_out/fuse2_plain.log
QDPB_FUSE=2 timeout 1200 compute-sanitizer --tool racecheck --target-processes all \
  python -m pytest tests/test_gpu_p2p.py -m gpu -x -q -k "not L4 and not bench_size and not 16" > gpurun_out/fuse2_race.log 2>&1
echo rc=$? >> gpurun_out/fuse2_race.log
QDPB_FUSE=1 timeout 1200 compute-sanitizer --tool racecheck --target-processes all \
  python -m pytest tests/test_gpu_p2p.py -m gpu -x -q -k "not L4 and not bench_size and not 16" > gpurun_out/fuse1_race.log 2>&1
echo rc=$? >> gpurun_out/fuse1_race.log
