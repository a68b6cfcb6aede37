timeout 1200 python -m pytest tests/test_gpu_p2p.py tests/test_gpu_peer.py tests/test_gpu_parity.py tests/test_gpu_edge.py tests/test_gpu_multishift.py -x -q 2>&1 | tail -2
python tools/halo_overhead.py 2>&1 | grep -E "whole|P2P"
QDPB_FUSE=0 python tools/halo_overhead.py 2>&1 | grep -E "P2P" | sed "s/^/(separate) /"
