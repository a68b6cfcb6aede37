"""Multi-process (world_size 2, gloo, CPU) tests of the sub-grid decomposition logic the
multi-GPU path relies on: rank grid and neighbours, the face index
convention shared by sender and receiver, the same-peer message ordering of the halo
exchange when P_mu = 2 (comm.cpp), and a distributed circular shift assembled from those
pieces, checked against the oracle's global shift."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import fieldgen
import oracle
from paper_1408_5925_b200 import dist as qd


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _run(fn, world=2):
    port = _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(fn, r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(120)
    res = [q.get(timeout=5) for _ in procs]
    for r in res:
        assert r == "ok", r


def _worker(fn, rank, world, port, q):
    try:
        os.environ["MASTER_ADDR"] = "127.0.0.1"
        dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
        globals()[fn](rank, world)
        dist.barrier()
        dist.destroy_process_group()
        q.put("ok")
    except Exception as e:  # report to the parent
        import traceback
        q.put(traceback.format_exc())


def test_proc_grid_and_neighbours():
    assert qd.proc_grid_for(8, (40, 40, 40, 256)) == (1, 1, 1, 8)
    assert qd.proc_grid_for(8, (48, 48, 48, 96)) == (1, 1, 1, 8)
    assert qd.proc_grid_for(4, (8, 8, 8, 4)) == (1, 1, 2, 2)   # t runs out (local t must stay even)
    # config 5: the t x z decomposition of BASELINE.json (at most 4 ranks along t)
    assert [qd.config5_grid(n) for n in (1, 2, 4, 8)] == [(1, 1, 1, 1), (1, 1, 1, 2), (1, 1, 1, 4), (1, 1, 2, 4)]
    assert qd.proc_grid_for(8, (48, 48, 48, 96), caps={3: 2}) == (1, 1, 4, 2)
    with pytest.raises(ValueError):
        qd.proc_grid_for(3, (4, 4, 4, 4))
    P = (1, 1, 2, 4)
    for r in range(8):
        assert qd.coords_rank(qd.rank_coords(r, P), P) == r
        nb = qd.neighbours(r, P)
        for mu in range(4):
            m, p = nb[mu]
            assert qd.neighbours(p, P)[mu][0] == r and qd.neighbours(m, P)[mu][1] == r
        assert nb[0] == (r, r) and nb[1] == (r, r)


def test_local_slices_tile_the_lattice():
    L = (4, 4, 6, 8)
    P = (1, 1, 2, 2)
    f = np.arange(fieldgen.volume(L) * 2, dtype=np.float64).reshape(-1, 2)
    parts = [qd.local_slice(f, L, P, r) for r in range(4)]
    assert sorted(np.concatenate(parts)[:, 0].tolist()) == f[:, 0].tolist()


def test_face_index_bijective_per_parity():
    for L in [(4, 4, 4, 8), (2, 6, 4, 2), (6, 2, 2, 4)]:
        for mu in range(4):
            for xmu in (0, L[mu] - 1):
                for p in (0, 1):
                    idx = []
                    for c in np.ndindex(*L[::-1]):
                        c = c[::-1]
                        if c[mu] == xmu and sum(c) % 2 == p:
                            idx.append(qd.face_index(L, mu, c))
                    assert sorted(idx) == list(range(fieldgen.volume(L) // L[mu] // 2))


def _ordering(rank, world):
    """P_mu = 2: both neighbours are the same peer.  Issue sends/recvs in the library's order
    (send +mu, send -mu, recv -mu, recv +mu) and check each message lands in the right buffer."""
    peer = 1 - rank
    to_fwd = torch.full((4,), 10.0 * rank + 1)   # for the peer's backward ghost
    to_bwd = torch.full((4,), 10.0 * rank + 2)   # for the peer's forward ghost
    from_bwd, from_fwd = torch.zeros(4), torch.zeros(4)
    reqs = [dist.isend(to_fwd, peer), dist.isend(to_bwd, peer), dist.irecv(from_bwd, peer), dist.irecv(from_fwd, peer)]
    for r in reqs:
        r.wait()
    # our backward ghost must hold what the peer sent towards its +mu neighbour (us): its "to_fwd"
    assert float(from_bwd[0]) == 10.0 * peer + 1
    assert float(from_fwd[0]) == 10.0 * peer + 2


def test_same_peer_ordering():
    _run("_ordering")


def _dist_shift(rank, world):
    L = (4, 4, 4, 8)
    for P in [(1, 1, 1, 2), (1, 1, 2, 1), (2, 1, 1, 1)]:
        Ll = [L[m] // P[m] for m in range(4)]
        psi = fieldgen.random_spinor(L, 77).reshape(-1, 24)
        loc = qd.local_slice(psi, L, P, rank)
        nb = qd.neighbours(rank, P)
        cl = fieldgen.coords(Ll)
        for mu in range(4):
            for sign in (1, -1):
                ref = qd.local_slice(oracle.shift(psi, L, mu, sign), L, P, rank)
                out = np.empty_like(loc)
                if P[mu] == 1:
                    src = cl.copy()
                    src[:, mu] = (src[:, mu] + sign) % Ll[mu]
                    out[:] = loc[src[:, 0] + Ll[0] * (src[:, 1] + Ll[1] * (src[:, 2] + Ll[2] * src[:, 3]))]
                else:
                    # pack the face the neighbour needs (both parities), in face-index order
                    xmu = 0 if sign > 0 else Ll[mu] - 1
                    nf = fieldgen.volume(Ll) // Ll[mu] // 2
                    send = np.zeros((2, nf, 24))
                    for s_, c in enumerate(cl):
                        if c[mu] == xmu:
                            send[c.sum() % 2, qd.face_index(Ll, mu, c)] = loc[s_]
                    recv = torch.zeros(2 * nf * 24, dtype=torch.float64)
                    to, frm = (nb[mu][0], nb[mu][1]) if sign > 0 else (nb[mu][1], nb[mu][0])
                    reqs = [dist.isend(torch.from_numpy(send.ravel()), to), dist.irecv(recv, frm)]
                    for r in reqs:
                        r.wait()
                    ghost = recv.numpy().reshape(2, nf, 24)
                    for s_, c in enumerate(cl):
                        n = c.copy()
                        n[mu] += sign
                        if 0 <= n[mu] < Ll[mu]:
                            out[s_] = loc[n[0] + Ll[0] * (n[1] + Ll[1] * (n[2] + Ll[2] * n[3]))]
                        else:
                            n[mu] %= Ll[mu]
                            out[s_] = ghost[n.sum() % 2, qd.face_index(Ll, mu, n)]
                assert np.array_equal(out, ref), (P, mu, sign)


def test_distributed_shift_matches_oracle():
    _run("_dist_shift")


def _reductions(rank, world):
    assert qd.max_over_ranks(float(rank + 3)) == 4.0
    assert qd.sum_over_ranks(float(rank + 3)) == 7.0


def test_rank_reductions():
    _run("_reductions")


def _allgather_bytes(rank, world):
    # the set-up callback of qdp_init_peer: equal-sized blocks, concatenated in rank order
    blob = bytes([rank]) * 64 + rank.to_bytes(4, "little") * 16
    out = qd.torch_allgather_bytes(blob)
    assert len(out) == world * len(blob)
    for r in range(world):
        assert out[r * len(blob):(r + 1) * len(blob)] == bytes([r]) * 64 + r.to_bytes(4, "little") * 16


def test_peer_bootstrap_allgather():
    _run("_allgather_bytes", world=3)


def test_peer_ctypes_callback_marshalling():
    """qdp_init_peer's ctypes trampoline: the C side's (send, recv, bytes) buffers round-trip
    through the Python allgather (called here directly, no GPU needed)."""
    import ctypes

    from paper_1408_5925_b200 import qdpb as q
    calls = []

    def fake_allgather(blob):
        calls.append(blob)
        return blob + bytes(reversed(blob))

    captured = {}

    def fake_init(gd, pg, rank, nranks, fn, user, stream, out):
        send = (ctypes.c_ubyte * 8)(*range(8))
        recv = (ctypes.c_ubyte * 16)()
        captured["rc"] = fn(ctypes.addressof(send), ctypes.addressof(recv), 8, None)
        captured["recv"] = bytes(recv)
        return -1  # pretend the device part failed afterwards

    class FakeLib:
        qdp_init_peer = staticmethod(fake_init)

        @staticmethod
        def qdp_strerror(st):
            return b"fake"

        @staticmethod
        def qdp_last_error(c):
            return b""

    real = q._lib
    q._lib = FakeLib()
    try:
        with pytest.raises(q.QdpError):
            q.qdp_init_peer((4, 4, 4, 8), (1, 1, 1, 2), 0, 2, fake_allgather)
    finally:
        q._lib = real
    assert captured["rc"] == 0 and calls == [bytes(range(8))]
    assert captured["recv"] == bytes(range(8)) + bytes(reversed(range(8)))
