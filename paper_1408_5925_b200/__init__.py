"""B200-native QDP hot path (arXiv:1408.5925): Wilson(-clover) hopping term, shift, lattice
BLAS and even-odd CG as hand-written sm_100a CUDA behind the C ABI of include/qdpb.h.

`qdpb` is the thin ctypes binding (same names as the C functions); `dist` bootstraps the
NCCL communicator of a multi-GPU run over torch.distributed.
"""
from . import qdpb  # noqa: F401
from .qdpb import *  # noqa: F401,F403

__all__ = [n for n in dir(qdpb) if n.startswith(("qdp_", "QDP_"))] + ["Ctx", "Field", "QdpError", "lib"]
