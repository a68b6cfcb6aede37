"""Worker of tests/test_gpu_peer.py: one process = one rank of a peer-memory context
(qdp_init_peer), all ranks on cuda:0.  The ranks exchange IPC handles over a gloo group and
from then on talk only through each other's mapped device memory: dslash halos (pack ->
neighbour's ghost slot + flags), shift faces (mailbox + flags) and global sums (one kernel
per sum).  Rank 0 assembles the global result and checks it against the oracle on the global
lattice (oracle = test infrastructure)."""
from __future__ import annotations

import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
for p in (ROOT, os.path.dirname(os.path.abspath(__file__))):
    if p not in sys.path:
        sys.path.insert(0, p)


def place_local(glob: np.ndarray, loc: np.ndarray, G, P, rank: int) -> None:
    """inverse of dist.local_slice: write a rank's sub-lattice into the global array"""
    from paper_1408_5925_b200.dist import rank_coords
    c = rank_coords(rank, P)
    L = [G[mu] // P[mu] for mu in range(4)]
    g = glob.reshape(G[3], G[2], G[1], G[0], *glob.shape[1:])
    g[c[3] * L[3]:(c[3] + 1) * L[3], c[2] * L[2]:(c[2] + 1) * L[2],
      c[1] * L[1]:(c[1] + 1) * L[1], c[0] * L[0]:(c[0] + 1) * L[0]] = loc.reshape(L[3], L[2], L[1], L[0], *loc.shape[1:])


def run(rank: int, world: int, port: int, case: str, G, P) -> None:
    import torch
    import torch.distributed as dist

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    torch.cuda.set_device(0)
    try:
        _run(rank, world, case, tuple(G), tuple(P))
    finally:
        dist.barrier()
        dist.destroy_process_group()


def _gather(arr: np.ndarray, G, P, per_site_shape):
    """all ranks' local arrays -> the global array (on every rank)"""
    import torch.distributed as dist
    parts = [None] * dist.get_world_size()
    dist.all_gather_object(parts, arr)
    out = np.zeros((int(np.prod(G)),) + tuple(per_site_shape), dtype=arr.dtype)
    for r, a in enumerate(parts):
        place_local(out, a, G, P, r)
    return out


def _same_on_all_ranks(v) -> None:
    import torch.distributed as dist
    vals = [None] * dist.get_world_size()
    dist.all_gather_object(vals, v)
    assert all(x == vals[0] for x in vals), f"global sums differ between ranks: {vals}"


def _run(rank, world, case, G, P):
    import fieldgen
    import oracle
    from _physics import rel_site_err
    from paper_1408_5925_b200 import dist as qd
    from paper_1408_5925_b200 import qdpb as q

    U = fieldgen.random_gauge(G, 1801)
    psi = fieldgen.random_spinor(G, 2801)
    chi = fieldgen.random_spinor(G, 2802)
    Ul, pl, cl = (qd.local_slice(a, G, P, rank) for a in (U, psi, chi))
    c = qd.bootstrap_peer(G, P)
    try:
        assert q.qdp_get_option(c, q.QDP_OPT_P2P) == 1

        def field(kind, prec, subset, host):
            f = q.qdp_field_alloc(c, kind, prec, subset)
            q.qdp_field_import(f, np.ascontiguousarray(host, dtype=np.float64 if prec == 0 else np.float32))
            return f

        if case == "dslash":
            for prec in (0, 1):
                Uh, ph = (U, psi) if prec == 0 else (fieldgen.to_fp32(U).astype(np.float64),
                                                     fieldgen.to_fp32(psi).astype(np.float64))
                fU = field(q.QDP_GAUGE, prec, q.QDP_ALL, qd.local_slice(Uh, G, P, rank))
                fp = field(q.QDP_FERMION, prec, q.QDP_ALL, qd.local_slice(ph, G, P, rank))
                fo = q.qdp_field_alloc(c, q.QDP_FERMION, prec, q.QDP_ALL)
                for overlap in (1, 0):
                    q.qdp_set_option(c, q.QDP_OPT_OVERLAP, overlap)
                    for _ in range(3):  # cycles both ghost slots
                        q.qdp_dslash(fo, fU, fp, q.QDP_ALL)
                    got = _gather(q.qdp_field_export(fo).astype(np.float64), G, P, (4, 3, 2))
                    if rank == 0:
                        ref = oracle.hopping(Uh, ph, G, -1)
                        err = rel_site_err(got, ref)
                        assert err <= (1e-13 if prec == 0 else 2e-6), (prec, overlap, err)
                # global sums: one peer kernel each, identical bits on every rank
                n2 = q.qdp_norm2(fp)
                fc = field(q.QDP_FERMION, prec, q.QDP_ALL, qd.local_slice(chi if prec == 0 else fieldgen.to_fp32(chi).astype(np.float64), G, P, rank))
                ip = q.qdp_inner_product(fc, fp)
                _same_on_all_ranks((n2, ip))
                if rank == 0 and prec == 0:
                    assert abs(n2 - oracle.norm2(psi, G)) <= 1e-13 * n2
                    ref_ip = oracle.inner(chi, psi, G)
                    assert abs(ip - ref_ip) <= 1e-13 * abs(n2)
                for f in (fU, fp, fo, fc):
                    q.qdp_field_free(f)
        elif case == "shift":
            fp = field(q.QDP_FERMION, 0, q.QDP_ALL, pl)
            fo = q.qdp_field_alloc(c, q.QDP_FERMION, 0, q.QDP_ALL)
            fU = field(q.QDP_GAUGE, 0, q.QDP_ALL, Ul)
            fUo = q.qdp_field_alloc(c, q.QDP_GAUGE, 0, q.QDP_ALL)
            for mu in range(4):
                for sign in (1, -1):
                    q.qdp_shift(fo, fp, mu, sign)
                    got = _gather(q.qdp_field_export(fo), G, P, (4, 3, 2))
                    q.qdp_shift(fUo, fU, mu, sign)
                    gotU = _gather(q.qdp_field_export(fUo), G, P, (4, 3, 3, 2))
                    if rank == 0:
                        assert np.array_equal(got, oracle.shift(psi, G, mu, sign)), (mu, sign)
                        assert np.array_equal(gotU, oracle.shift(U, G, mu, sign)), (mu, sign)
        elif case in ("cg", "cg_clover"):
            m = 0.1
            clover = case == "cg_clover"
            fU = field(q.QDP_GAUGE, 0, q.QDP_ALL, Ul)
            fb = field(q.QDP_FERMION, 0, q.QDP_ALL, pl)
            fx = q.qdp_field_alloc(c, q.QDP_FERMION, 0, q.QDP_ALL)
            fA = fAi = None
            if clover:  # partitioned clover build: "shifts of shifts" through the peer mailbox
                fA = q.qdp_field_alloc(c, q.QDP_CLOVER, 0, q.QDP_ALL)
                fAi = q.qdp_field_alloc(c, q.QDP_CLOVER, 0, q.QDP_EVEN)
                q.qdp_clover_build(fA, fAi, fU, m, 1.0)
            res = q.qdp_cg_solve(fx, fb, fU, fA, fAi, mass=m, tol=1e-10, maxit=1000)
            _same_on_all_ranks((res["iters"], tuple(res["hist"]), res["true_resid"]))
            x = _gather(q.qdp_field_export(fx), G, P, (4, 3, 2))
            if rank == 0:
                A = oracle.clover_build(U, G, m, 1.0) if clover else None
                ref = oracle.cg_solve(U, psi, G, m, A=A, tol=1e-10, maxit=1000)
                assert res["status"] == q.QDP_OK
                assert res["iters"] == ref["iters"]
                assert np.max(np.abs(res["hist"] - ref["hist"]) / ref["hist"]) <= 1e-10
                assert res["true_resid"] <= 5e-10
                assert rel_site_err(x, ref["x"]) <= 1e-9
        elif case == "multishift":
            m, sigma = 0.1, [0.0, 0.02, 0.5, 3.0]
            fU = field(q.QDP_GAUGE, 0, q.QDP_ALL, Ul)
            fphi = field(q.QDP_FERMION, 0, q.QDP_ALL, pl)
            xs = [q.qdp_field_alloc(c, q.QDP_FERMION, 0, q.QDP_ALL) for _ in sigma]
            fA = q.qdp_field_alloc(c, q.QDP_CLOVER, 0, q.QDP_ALL)
            fAi = q.qdp_field_alloc(c, q.QDP_CLOVER, 0, q.QDP_EVEN)
            q.qdp_clover_build(fA, fAi, fU, m, 1.0)
            res = q.qdp_cg_solve_multishift(xs, sigma, fphi, fU, fA, fAi, mass=m, tol=1e-10, maxit=1000)
            _same_on_all_ranks((res["iters"], tuple(res["hist"]), tuple(res["conv_iter"])))
            got = [_gather(q.qdp_field_export(x), G, P, (4, 3, 2)) for x in xs]
            if rank == 0:
                ref = oracle.cg_multishift(U, psi, G, m, sigma, A=oracle.clover_build(U, G, m, 1.0), tol=1e-10,
                                           maxit=1000)
                odd = fieldgen.parity(G) == 1
                assert res["iters"] == ref["iters"] and np.array_equal(res["conv_iter"], ref["conv_iter"])
                assert np.max(np.abs(res["hist"] - ref["hist"]) / ref["hist"]) <= 1e-10
                for i in range(len(sigma)):
                    assert rel_site_err(got[i][odd], ref["x"][i][odd]) <= 1e-9
        elif case == "jit":
            # run-time generated expressions whose shifts cross rank boundaries: the halo'd leaves are
            # materialised through qdp_shift (faces via the peer mailbox), the rest is in-kernel
            from paper_1408_5925_b200.exprs import hopping as hopping_expr
            fU = field(q.QDP_GAUGE, 0, q.QDP_ALL, Ul)
            fp = field(q.QDP_FERMION, 0, q.QDP_ALL, pl)
            fo = q.qdp_field_alloc(c, q.QDP_FERMION, 0, q.QDP_ALL)
            for _ in range(2):  # second call: cached kernel and temporaries
                q.qdp_jit_eval(fo, hopping_expr(), fU, fp)
            got = _gather(q.qdp_field_export(fo), G, P, (4, 3, 2))
            # Fig. 1 along t and a diagonal shift of a shift
            q.qdp_jit_eval(fo, "$0[3]*shift($1,3,+1) + shift(adj($0[3])*$1,3,-1)", fU, fp)
            fig1 = _gather(q.qdp_field_export(fo), G, P, (4, 3, 2))
            q.qdp_jit_eval(fo, "shift(shift($0,2,-1),3,+1)", fp)
            diag = _gather(q.qdp_field_export(fo), G, P, (4, 3, 2))
            # global sums of site expressions: the plaquette across rank boundaries, identical on every rank
            plaq = "real(trace($0[2]*shift($0[3],2,+1)*adj(shift($0[2],3,+1))*adj($0[3])))"
            pv = q.qdp_jit_sum(c, plaq, fU)
            nv = q.qdp_jit_sum(c, "localNorm2($0)", fp)
            _same_on_all_ranks((pv, nv))
            if rank == 0:
                Uc = U[..., 0] + 1j * U[..., 1]
                sh = lambda a, mu: oracle.shift(a, G, mu, 1)
                Un = sh(U, 2)[:, 3]
                Un = Un[..., 0] + 1j * Un[..., 1]
                Um = sh(U, 3)[:, 2]
                Um = Um[..., 0] + 1j * Um[..., 1]
                H = lambda m: np.conj(np.swapaxes(m, 1, 2))
                ref = np.sum(np.trace(Uc[:, 2] @ Un @ H(Um) @ H(Uc[:, 3]), axis1=1, axis2=2).real)
                assert abs(pv.real - ref) <= 1e-12 * 3 * np.prod(G)
                assert abs(nv.real - oracle.norm2(psi, G)) <= 1e-13 * nv.real
                assert rel_site_err(got, oracle.hopping(U, psi, G, -1)) <= 1e-13
                ref = (oracle.upsi(U[:, 3], oracle.shift(psi, G, 3, 1))
                       + oracle.shift(oracle.adj_upsi(U[:, 3], psi), G, 3, -1))
                assert rel_site_err(fig1, ref) <= 1e-13
                assert np.array_equal(diag, oracle.shift(oracle.shift(psi, G, 2, -1), G, 3, 1))
        else:
            raise ValueError(case)
    finally:
        q.qdp_finalize(c)
