"""Several ranks of a peer-memory context (qdp_init_peer) as separate processes sharing one
GPU: the real multi-process path of the NVSwitch-native design -- IPC
mappings between processes, dslash halos written into the neighbour's ghost slots with
release/acquire flags, shift faces through the neighbour's mailbox, and global sums by one
peer kernel -- checked against the oracle on the global lattice.  NCCL is never loaded
(it refuses two ranks on one GPU); the IPC handles travel over a gloo group."""
import os
import socket

import pytest

pytestmark = pytest.mark.gpu


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _spawn(case, G, P):
    import torch.multiprocessing as mp

    import _peer_worker
    world = P[0] * P[1] * P[2] * P[3]
    mp.spawn(_peer_worker.run, args=(world, _free_port(), case, G, P), nprocs=world, join=True)


@pytest.mark.timeout(600)
@pytest.mark.parametrize("G,P", [((4, 4, 4, 8), (1, 1, 1, 2)),   # t split (SURVEY 8(e) first split)
                                 ((4, 4, 8, 8), (1, 1, 2, 2)),   # z x t, four ranks
                                 ((8, 4, 4, 4), (2, 1, 1, 1))])  # x split: the checkerboarded dim
def test_peer_dslash_and_sums(G, P):
    _spawn("dslash", G, P)


@pytest.mark.timeout(600)
def test_peer_shift():
    _spawn("shift", (4, 4, 4, 8), (1, 1, 2, 2))


@pytest.mark.timeout(600)
@pytest.mark.parametrize("G, P", [((4, 4, 4, 8), (1, 1, 1, 2)), ((4, 4, 4, 8), (1, 1, 2, 2))])
def test_peer_jit(G, P):
    _spawn("jit", G, P)


@pytest.mark.timeout(600)
@pytest.mark.parametrize("case", ["cg", "cg_clover", "multishift"])
def test_peer_cg(case):
    _spawn(case, (4, 4, 4, 8), (1, 1, 1, 2))


@pytest.mark.timeout(900)
@pytest.mark.parametrize("case", ["cg", "cg_clover"])
def test_peer_cg_zt(case):
    """The config-5 decomposition shape (z x t, here 2 x 2 ranks; dist.config5_grid gives 2 x 4 on
    eight GPUs): fused z x t boundary kernels, one-launch global sums, device-side CG."""
    _spawn(case, (4, 4, 8, 8), (1, 1, 2, 2))
