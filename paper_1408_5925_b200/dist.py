"""Multi-process plumbing for the C ABI (one process per GPU): the sub-grid decomposition of
PAPER.md:93-95 (t first, then z: SURVEY.md 8(e)), NCCL-id bootstrap over torch.distributed,
and host-side helpers that the halo code path relies on (neighbour ranks, face index
maps), kept in Python so they can be tested with gloo on CPU.
"""
from __future__ import annotations

import numpy as np


def proc_grid_for(n: int, global_dims, split=(3, 2), caps=None):
    """Rank grid P (P0,P1,P2,P3) for n ranks: factor n over the dims in `split` order
    (t first, then z), keeping every local extent even and P[mu] <= caps[mu] where given.
    Raises if impossible."""
    P = [1, 1, 1, 1]
    rem = n
    caps = caps or {}
    for mu in split:
        while rem > 1:
            f = next((k for k in range(2, rem + 1) if rem % k == 0), rem)
            loc = global_dims[mu] // (P[mu] * f)
            if global_dims[mu] % (P[mu] * f) or loc < 2 or loc % 2 or P[mu] * f > caps.get(mu, n):
                break
            P[mu] *= f
            rem //= f
    if rem != 1:
        raise ValueError(f"cannot split {global_dims} over {n} ranks along dims {split}")
    return tuple(P)


CONFIG5_DIMS = (48, 48, 48, 96)


def config5_grid(n: int):
    """Rank grid of BASELINE.json config 5 (48^3 x 96 even-odd CG, "t x z decomposition"):
    t first, at most 4 ranks along t, then z -- so 8 ranks give P = (1,1,2,4) (local
    48 x 48 x 24 x 24); 2 and 4 ranks split t only."""
    return proc_grid_for(n, CONFIG5_DIMS, split=(3, 2), caps={3: 4})


def rank_coords(rank: int, P):
    """Processor coordinates of `rank`: r = p0 + P0(p1 + P1(p2 + P2 p3)) (qdpb.h convention)."""
    c = []
    for mu in range(4):
        c.append(rank % P[mu])
        rank //= P[mu]
    return tuple(c)


def coords_rank(c, P):
    return c[0] + P[0] * (c[1] + P[1] * (c[2] + P[2] * c[3]))


def neighbours(rank: int, P):
    """[(rank of -mu neighbour, rank of +mu neighbour) for mu in 0..3], periodic."""
    c = rank_coords(rank, P)
    out = []
    for mu in range(4):
        pair = []
        for d in (-1, 1):
            n = list(c)
            n[mu] = (n[mu] + d) % P[mu]
            pair.append(coords_rank(n, P))
        out.append(tuple(pair))
    return out


def local_slice(global_array: np.ndarray, global_dims, P, rank: int) -> np.ndarray:
    """The local sub-lattice of a host canonical array [V_global, ...] (lexicographic sites)."""
    c = rank_coords(rank, P)
    L = [global_dims[mu] // P[mu] for mu in range(4)]
    g = global_array.reshape(global_dims[3], global_dims[2], global_dims[1], global_dims[0], *global_array.shape[1:])
    sl = g[c[3] * L[3]:(c[3] + 1) * L[3], c[2] * L[2]:(c[2] + 1) * L[2],
           c[1] * L[1]:(c[1] + 1) * L[1], c[0] * L[0]:(c[0] + 1) * L[0]]
    return np.ascontiguousarray(sl.reshape(-1, *global_array.shape[1:]))


def face_index(L, mu, coords):
    """Face index of a site on the face orthogonal to mu (qdpb internal.h face_index)."""
    lex, mul = 0, 1
    for d in range(4):
        if d == mu:
            continue
        lex += coords[d] * mul
        mul *= L[d]
    return lex >> 1


def bootstrap(global_dims, P, stream=None):
    """Create this rank's qdp context.  torch.distributed must be initialised when the world
    size is > 1: rank 0 draws the NCCL id and broadcasts it."""
    import torch.distributed as dist

    from . import qdpb as q
    if dist.is_available() and dist.is_initialized() and dist.get_world_size() > 1:
        rank, world = dist.get_rank(), dist.get_world_size()
        obj = [q.qdp_get_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        return q.qdp_init(global_dims, P, rank, world, obj[0], stream)
    return q.qdp_init(global_dims, P, 0, 1, None, stream)


def torch_allgather_bytes(blob: bytes) -> bytes:
    """Host allgather of equal-sized byte blocks over the default torch.distributed group
    (gloo or nccl), concatenated in rank order: the set-up callback of qdp_init_peer."""
    import torch.distributed as dist
    out = [None] * dist.get_world_size()
    dist.all_gather_object(out, bytes(blob))
    return b"".join(out)


def bootstrap_peer(global_dims, P, stream=None):
    """Create this rank's peer-memory context (qdp_init_peer: halos, shift faces and global
    sums through IPC-mapped device memory, no NCCL); IPC handles travel over the default
    torch.distributed group, which may be gloo."""
    import torch.distributed as dist

    from . import qdpb as q
    if dist.is_available() and dist.is_initialized() and dist.get_world_size() > 1:
        return q.qdp_init_peer(global_dims, P, dist.get_rank(), dist.get_world_size(), torch_allgather_bytes, stream)
    return q.qdp_init(global_dims, P, 0, 1, None, stream)


def max_over_ranks(value: float) -> float:
    import torch
    import torch.distributed as dist
    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size() == 1:
        return value
    dev = "cuda" if dist.get_backend() == "nccl" else "cpu"
    t = torch.tensor([value], dtype=torch.float64, device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def sum_over_ranks(value: float) -> float:
    import torch
    import torch.distributed as dist
    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size() == 1:
        return value
    dev = "cuda" if dist.get_backend() == "nccl" else "cpu"
    t = torch.tensor([value], dtype=torch.float64, device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.SUM)
    return float(t.item())
