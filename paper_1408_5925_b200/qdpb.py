"""Thin ctypes binding of include/qdpb.h (libqdpb.so, built in-tree for sm_100a).

Functions carry the C names and only marshal arguments: numpy arrays / torch tensors to
pointers, status codes to exceptions.  Every computation happens in the library's CUDA
kernels.  There is no fallback: if libqdpb.so is missing, `lib()` raises.
"""
from __future__ import annotations

import ctypes
import os
import re

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
# QDPB_LIB selects a tuning-variant build of the same library (development only)
LIB_PATH = os.environ.get("QDPB_LIB") or os.path.join(_HERE, "libqdpb.so")
HEADER = os.path.join(os.path.dirname(_HERE), "include", "qdpb.h")

QDP_F64, QDP_F32 = 0, 1
QDP_FERMION, QDP_GAUGE, QDP_CLOVER, QDP_GAUGE12, QDP_COLORMATRIX, QDP_SPINMATRIX = range(6)
QDP_EXPR_LCM, QDP_EXPR_UPSI, QDP_EXPR_SPMAT, QDP_EXPR_MATVEC, QDP_EXPR_CLOVER, QDP_EXPR_ADJ_UPSI = range(6)
QDP_ALL, QDP_EVEN, QDP_ODD = -1, 0, 1
QDP_FORWARD, QDP_BACKWARD = 1, -1
QDP_OK, QDP_NOT_CONVERGED = 0, 1
QDP_EINVAL, QDP_ESHAPE, QDP_EPREC, QDP_EALIAS, QDP_ENOMEM = -1, -2, -3, -4, -5
QDP_ECUDA, QDP_ENCCL, QDP_ESINGULAR, QDP_EUNSUPPORTED = -6, -7, -8, -9
(QDP_OPT_OVERLAP, QDP_OPT_SELF_HALO, QDP_OPT_PROFILE, QDP_OPT_BLOCK, QDP_OPT_DET_REDUCE, QDP_OPT_SELF_NCCL,
 QDP_OPT_AUTOTUNE, QDP_OPT_P2P, QDP_OPT_FUSE, QDP_OPT_DSLASH_VARIANT, QDP_OPT_PDL) = range(11)
(QDP_PK_DSLASH, QDP_PK_DSLASH_EXT, QDP_PK_PACK, QDP_PK_BLAS, QDP_PK_REDUCE, QDP_PK_CLOVER,
 QDP_PK_SHIFT, QDP_PK_LAYOUT, QDP_PK_MSHIFT, QDP_PK_COUNT) = range(10)
PK_NAMES = ["dslash", "dslash_ext", "pack", "blas", "reduce", "clover", "shift", "layout", "mshift"]

_lib = None
_vp = ctypes.c_void_p
# int (*qdp_allgather_fn)(const void *send, void *recv, size_t bytes, void *user)
ALLGATHER_FN = ctypes.CFUNCTYPE(ctypes.c_int, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_size_t, ctypes.c_void_p)
_ip = ctypes.POINTER(ctypes.c_int)
_dp = ctypes.POINTER(ctypes.c_double)
_SIGS = {
    "qdp_get_unique_id": [ctypes.c_char_p],
    "qdp_init": [_ip, _ip, ctypes.c_int, ctypes.c_int, ctypes.c_char_p, _vp, ctypes.POINTER(_vp)],
    "qdp_init_peer": [_ip, _ip, ctypes.c_int, ctypes.c_int, ALLGATHER_FN, _vp, _vp, ctypes.POINTER(_vp)],
    "qdp_finalize": [_vp],
    "qdp_set_stream": [_vp, _vp],
    "qdp_synchronize": [_vp],
    "qdp_get_geometry": [_vp, _ip, _ip],
    "qdp_set_option": [_vp, ctypes.c_int, ctypes.c_long],
    "qdp_get_option": [_vp, ctypes.c_int, ctypes.POINTER(ctypes.c_long)],
    "qdp_field_alloc": [_vp, ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.POINTER(_vp)],
    "qdp_field_wrap": [_vp, ctypes.c_int, ctypes.c_int, ctypes.c_int, _vp, ctypes.c_size_t, ctypes.POINTER(_vp)],
    "qdp_field_free": [_vp],
    "qdp_field_bytes": [_vp, ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.POINTER(ctypes.c_size_t),
                        ctypes.POINTER(ctypes.c_size_t)],
    "qdp_field_info": [_vp, _ip, _ip, _ip, ctypes.POINTER(_vp)],
    "qdp_field_import": [_vp, _vp, ctypes.c_size_t],
    "qdp_field_export": [_vp, _vp, ctypes.c_size_t],
    "qdp_field_import_device": [_vp, _vp, ctypes.c_size_t],
    "qdp_field_export_device": [_vp, _vp, ctypes.c_size_t],
    "qdp_field_zero": [_vp],
    "qdp_field_copy": [_vp, _vp],
    "qdp_shift": [_vp, _vp, ctypes.c_int, ctypes.c_int],
    "qdp_dslash": [_vp, _vp, _vp, ctypes.c_int],
    "qdp_norm2": [_vp, _dp],
    "qdp_inner_product": [_vp, _vp, _dp],
    "qdp_axpy": [ctypes.c_double, ctypes.c_double, _vp, _vp],
    "qdp_clover_build": [_vp, _vp, _vp, ctypes.c_double, ctypes.c_double],
    "qdp_clover_apply": [_vp, _vp, _vp, ctypes.c_int],
    "qdp_cg_solve": [_vp, _vp, _vp, _vp, _vp, ctypes.c_double, ctypes.c_double, ctypes.c_int, _ip, _dp,
                     ctypes.c_int, _dp],
    "qdp_cg_solve_mixed": [_vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, ctypes.c_double, ctypes.c_double, ctypes.c_double,
                           ctypes.c_int, _ip, _ip, _dp, ctypes.c_int, _dp],
    "qdp_cg_solve_mixed16": [_vp, _vp, _vp, _vp, _vp, ctypes.c_double, ctypes.c_double, ctypes.c_double,
                             ctypes.c_int, _ip, _ip, _dp, ctypes.c_int, _dp],
    "qdp_cg_solve_multishift": [ctypes.POINTER(_vp), ctypes.c_int, _dp, _vp, _vp, _vp, _vp, ctypes.c_double,
                                ctypes.c_double, ctypes.c_int, _ip, _ip, _dp, ctypes.c_int, _dp],
    "qdp_expr": [ctypes.c_int, _vp, _vp, _vp, _vp],
    "qdp_expr_block": [_vp, ctypes.c_int, ctypes.c_int, _ip, _ip],
    "qdp_jit_eval": [_vp, ctypes.c_char_p, ctypes.POINTER(_vp), ctypes.c_int],
    "qdp_jit_source": [ctypes.c_char_p, ctypes.c_int, ctypes.c_int, ctypes.c_int, _ip, ctypes.c_int, ctypes.c_char_p,
                       ctypes.c_size_t, ctypes.POINTER(ctypes.c_size_t), _dp, ctypes.c_int],
    "qdp_jit_stats": [_vp, _ip, _dp],
    "qdp_jit_sum": [_vp, ctypes.c_char_p, ctypes.POINTER(_vp), ctypes.c_int, ctypes.c_int, _dp],
    "qdp_strerror": [ctypes.c_int],
    "qdp_last_error": [_vp],
    "qdp_profile_query": [_vp, ctypes.c_int, ctypes.POINTER(ctypes.c_long), _dp],
    "qdp_profile_work": [_vp, ctypes.c_int, _dp, _dp],
    "qdp_profile_reset": [_vp],
}


class QdpError(RuntimeError):
    def __init__(self, status, msg):
        super().__init__(f"{msg} (status {status})")
        self.status = status


def header_symbols():
    """Names of the functions declared in include/qdpb.h."""
    txt = open(HEADER).read()
    return sorted(set(re.findall(r"^\s*(?:const\s+)?\w+\s*\*?\s*(qdp_\w+)\s*\(", txt, flags=re.M)))


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} is missing: build it with `python -c 'import __graft_entry__ as g; g.build()'` "
                              "(there is no CPU fallback)")
        L = ctypes.CDLL(LIB_PATH)
        for name, args in _SIGS.items():
            fn = getattr(L, name)
            fn.argtypes = args
            fn.restype = ctypes.c_int
        L.qdp_strerror.restype = ctypes.c_char_p
        L.qdp_last_error.restype = ctypes.c_char_p
        _lib = L
    return _lib


class Ctx:
    """Opaque context handle (qdp_ctx)."""

    def __init__(self, ptr, global_dims, proc_grid, rank, nranks):
        self.ptr = ptr
        self.global_dims = tuple(global_dims)
        self.proc_grid = tuple(proc_grid)
        self.rank, self.nranks = rank, nranks

    @property
    def _as_parameter_(self):
        return self.ptr


class Field:
    """Opaque field handle (qdp_field); keeps a reference to wrapped memory."""

    def __init__(self, ptr, ctx, kind, prec, subset, keep=None):
        self.ptr, self.ctx, self.kind, self.prec, self.subset, self._keep = ptr, ctx, kind, prec, subset, keep

    @property
    def _as_parameter_(self):
        return self.ptr


def _check(st, ctx=None):
    if st < 0:
        L = lib()
        detail = L.qdp_last_error(ctx.ptr if ctx is not None else None) if ctx is not None else b""
        msg = L.qdp_strerror(st).decode()
        if detail:
            msg += ": " + detail.decode()
        raise QdpError(st, msg)
    return st


def _i4(v):
    return (ctypes.c_int * 4)(*[int(x) for x in v])


def _ptr_bytes(a):
    """(pointer, nbytes, keepalive) of a contiguous numpy array or torch tensor."""
    if isinstance(a, np.ndarray):
        if not a.flags["C_CONTIGUOUS"]:
            raise ValueError("array must be C-contiguous")
        return a.ctypes.data, a.nbytes, a
    if hasattr(a, "data_ptr"):
        if not a.is_contiguous():
            raise ValueError("tensor must be contiguous")
        return a.data_ptr(), a.numel() * a.element_size(), a
    raise TypeError(f"unsupported buffer type {type(a)}")


def _stream_ptr(stream):
    if stream is None:
        return None
    if hasattr(stream, "cuda_stream"):
        return stream.cuda_stream
    return int(stream)


# ------------------------------------------------------------------ context
def qdp_get_unique_id() -> bytes:
    buf = ctypes.create_string_buffer(128)
    _check(lib().qdp_get_unique_id(buf))
    return buf.raw


def qdp_init(global_dims, proc_grid=(1, 1, 1, 1), rank=0, nranks=1, nccl_id=None, stream=None) -> Ctx:
    out = _vp()
    idb = None if nccl_id is None else ctypes.create_string_buffer(bytes(nccl_id), 128)
    st = lib().qdp_init(_i4(global_dims), _i4(proc_grid), int(rank), int(nranks), idb, _stream_ptr(stream),
                        ctypes.byref(out))
    _check(st)
    return Ctx(out.value, global_dims, proc_grid, rank, nranks)


def qdp_init_peer(global_dims, proc_grid, rank, nranks, allgather, stream=None) -> Ctx:
    """Peer-memory context (no NCCL).  `allgather(bytes) -> bytes` is the caller's host
    allgather (all ranks' blocks concatenated in rank order); it runs only inside this call."""
    err = []

    def _cb(send, recv, nbytes, _user):
        try:
            out = allgather(ctypes.string_at(send, nbytes))
            if len(out) != nbytes * int(nranks):
                raise ValueError(f"allgather returned {len(out)} bytes, expected {nbytes * nranks}")
            ctypes.memmove(recv, out, len(out))
            return 0
        except Exception as e:  # reported after the call; the C side sees a failure status
            err.append(e)
            return 1

    fn = ALLGATHER_FN(_cb)
    out = _vp()
    st = lib().qdp_init_peer(_i4(global_dims), _i4(proc_grid), int(rank), int(nranks), fn, None,
                             _stream_ptr(stream), ctypes.byref(out))
    if err:
        raise err[0]
    _check(st)
    return Ctx(out.value, global_dims, proc_grid, rank, nranks)


def qdp_finalize(ctx: Ctx) -> None:
    if ctx.ptr:
        _check(lib().qdp_finalize(ctx.ptr))
        ctx.ptr = None


def qdp_set_stream(ctx: Ctx, stream) -> None:
    _check(lib().qdp_set_stream(ctx, _stream_ptr(stream)), ctx)


def qdp_synchronize(ctx: Ctx) -> None:
    _check(lib().qdp_synchronize(ctx), ctx)


def qdp_get_geometry(ctx: Ctx):
    ld, pc = (ctypes.c_int * 4)(), (ctypes.c_int * 4)()
    _check(lib().qdp_get_geometry(ctx, ld, pc), ctx)
    return tuple(ld), tuple(pc)


def qdp_set_option(ctx: Ctx, option: int, value: int) -> None:
    _check(lib().qdp_set_option(ctx, int(option), int(value)), ctx)


def qdp_get_option(ctx: Ctx, option: int) -> int:
    v = ctypes.c_long()
    _check(lib().qdp_get_option(ctx, int(option), ctypes.byref(v)), ctx)
    return v.value


# ------------------------------------------------------------------ fields
def qdp_field_bytes(ctx: Ctx, kind: int, prec: int, subset: int):
    hb, db = ctypes.c_size_t(), ctypes.c_size_t()
    _check(lib().qdp_field_bytes(ctx, kind, prec, subset, ctypes.byref(hb), ctypes.byref(db)), ctx)
    return hb.value, db.value


def qdp_field_alloc(ctx: Ctx, kind: int, prec: int, subset: int = QDP_ALL) -> Field:
    out = _vp()
    _check(lib().qdp_field_alloc(ctx, kind, prec, subset, ctypes.byref(out)), ctx)
    return Field(out.value, ctx, kind, prec, subset)


def qdp_field_wrap(ctx: Ctx, kind: int, prec: int, subset: int, tensor) -> Field:
    """Borrow a CUDA tensor's memory (>= qdp_field_bytes device bytes, 256-byte aligned)."""
    p, n, keep = _ptr_bytes(tensor)
    out = _vp()
    _check(lib().qdp_field_wrap(ctx, kind, prec, subset, p, n, ctypes.byref(out)), ctx)
    return Field(out.value, ctx, kind, prec, subset, keep)


def qdp_field_free(f: Field) -> None:
    if f.ptr:
        _check(lib().qdp_field_free(f))
        f.ptr = None


def qdp_field_info(f: Field):
    """(kind, prec, subset, device pointer)"""
    k, p, s, d = ctypes.c_int(), ctypes.c_int(), ctypes.c_int(), _vp()
    _check(lib().qdp_field_info(f, ctypes.byref(k), ctypes.byref(p), ctypes.byref(s), ctypes.byref(d)), f.ctx)
    return k.value, p.value, s.value, d.value


def qdp_field_import(f: Field, host) -> None:
    p, n, _ = _ptr_bytes(host)
    _check(lib().qdp_field_import(f, p, n), f.ctx)


def _host_shape(f: Field):
    hb, _ = qdp_field_bytes(f.ctx, f.kind, f.prec, f.subset)
    per = {QDP_FERMION: (4, 3, 2), QDP_GAUGE: (4, 3, 3, 2), QDP_CLOVER: (12, 12, 2), QDP_GAUGE12: (4, 3, 3, 2),
           QDP_COLORMATRIX: (3, 3, 2), QDP_SPINMATRIX: (4, 4, 2)}[f.kind]
    isz = 8 if f.prec == QDP_F64 else 4
    n = hb // (isz * int(np.prod(per)))
    return (n,) + per, (np.float64 if f.prec == QDP_F64 else np.float32)


def qdp_field_export(f: Field, out=None):
    if out is None:
        shape, dt = _host_shape(f)
        out = np.empty(shape, dtype=dt)
    p, n, _ = _ptr_bytes(out)
    _check(lib().qdp_field_export(f, p, n), f.ctx)
    return out


def qdp_field_import_device(f: Field, dev) -> None:
    """Enqueue the layout conversion from a CUDA tensor holding the host canonical layout."""
    p, n, _ = _ptr_bytes(dev)
    _check(lib().qdp_field_import_device(f, p, n), f.ctx)


def qdp_field_export_device(f: Field, dev) -> None:
    """Enqueue the layout conversion into a CUDA tensor (host canonical layout)."""
    p, n, _ = _ptr_bytes(dev)
    _check(lib().qdp_field_export_device(f, p, n), f.ctx)


def qdp_field_zero(f: Field) -> None:
    _check(lib().qdp_field_zero(f), f.ctx)


def qdp_field_copy(dst: Field, src: Field) -> None:
    _check(lib().qdp_field_copy(dst, src), dst.ctx)


# ------------------------------------------------------------------ operations
def qdp_shift(out: Field, inp: Field, mu: int, sign: int) -> None:
    _check(lib().qdp_shift(out, inp, int(mu), int(sign)), out.ctx)


def qdp_dslash(out: Field, U: Field, psi: Field, out_parity: int) -> None:
    _check(lib().qdp_dslash(out, U, psi, int(out_parity)), out.ctx)


def qdp_norm2(a: Field) -> float:
    v = ctypes.c_double()
    _check(lib().qdp_norm2(a, ctypes.byref(v)), a.ctx)
    return v.value


def qdp_inner_product(a: Field, b: Field) -> complex:
    v = (ctypes.c_double * 2)()
    _check(lib().qdp_inner_product(a, b, v), a.ctx)
    return complex(v[0], v[1])


def qdp_axpy(a: complex, x: Field, y: Field) -> None:
    a = complex(a)
    _check(lib().qdp_axpy(a.real, a.imag, x, y), y.ctx)


def qdp_clover_build(A, Ainv, U: Field, mass: float, csw: float) -> None:
    _check(lib().qdp_clover_build(A, Ainv, U, float(mass), float(csw)), U.ctx)


def qdp_clover_apply(out: Field, A: Field, inp: Field, parity: int) -> None:
    _check(lib().qdp_clover_apply(out, A, inp, int(parity)), out.ctx)


def qdp_cg_solve(x: Field, b: Field, U: Field, A=None, Ainv=None, mass=0.1, tol=1e-10, maxit=10000,
                 hist_cap=None, true_resid=True):
    hist_cap = maxit + 1 if hist_cap is None else hist_cap
    hist = (ctypes.c_double * max(hist_cap, 1))()
    iters = ctypes.c_int()
    tr = ctypes.c_double()
    st = lib().qdp_cg_solve(x, b, U, A, Ainv, float(mass), float(tol), int(maxit), ctypes.byref(iters), hist,
                            int(hist_cap), ctypes.byref(tr) if true_resid else None)
    _check(st, x.ctx)
    n = iters.value
    return dict(status=st, iters=n, hist=np.array(hist[:min(n + 1, hist_cap)]),
                true_resid=tr.value if true_resid else None)


def qdp_cg_solve_mixed(x: Field, b: Field, U: Field, A=None, Ainv=None, U_s: Field = None, A_s=None, Ainv_s=None,
                       mass=0.1, tol=1e-10, delta=0.1, maxit=10000, hist_cap=None, true_resid=True):
    hist_cap = maxit + 1 if hist_cap is None else hist_cap
    hist = (ctypes.c_double * max(hist_cap, 1))()
    iters, rel = ctypes.c_int(), ctypes.c_int()
    tr = ctypes.c_double()
    st = lib().qdp_cg_solve_mixed(x, b, U, A, Ainv, U_s, A_s, Ainv_s, float(mass), float(tol), float(delta),
                                  int(maxit), ctypes.byref(iters), ctypes.byref(rel), hist, int(hist_cap),
                                  ctypes.byref(tr) if true_resid else None)
    _check(st, x.ctx)
    n = iters.value
    return dict(status=st, iters=n, reliable=rel.value, hist=np.array(hist[:min(n + 1, hist_cap)]),
                true_resid=tr.value if true_resid else None)


def qdp_cg_solve_mixed16(x: Field, b: Field, U: Field, A=None, Ainv=None, mass=0.1, tol=1e-10, delta=0.1,
                         maxit=10000, hist_cap=None, true_resid=True):
    """Mixed-precision CG with a 16-bit sloppy level built from the fp64 U, A, Ainv (qdpb.h)."""
    hist_cap = maxit + 1 if hist_cap is None else hist_cap
    hist = (ctypes.c_double * max(hist_cap, 1))()
    iters, rel = ctypes.c_int(), ctypes.c_int()
    tr = ctypes.c_double()
    st = lib().qdp_cg_solve_mixed16(x, b, U, A, Ainv, float(mass), float(tol), float(delta), int(maxit),
                                    ctypes.byref(iters), ctypes.byref(rel), hist, int(hist_cap),
                                    ctypes.byref(tr) if true_resid else None)
    _check(st, x.ctx)
    n = iters.value
    return dict(status=st, iters=n, reliable=rel.value, hist=np.array(hist[:min(n + 1, hist_cap)]),
                true_resid=tr.value if true_resid else None)


def qdp_cg_solve_multishift(x, sigma, phi: Field, U: Field, A=None, Ainv=None, mass=0.1, tol=1e-10, maxit=10000,
                            hist_cap=None, true_resid=True):
    """(Mhat^dag Mhat + sigma_i) x_i = phi_o for every shift (x: list of fields, one per shift)."""
    n = len(sigma)
    if len(x) != n:
        raise ValueError("one solution field per shift")
    hist_cap = maxit + 1 if hist_cap is None else hist_cap
    hist = (ctypes.c_double * max(hist_cap, 1))()
    xs = (_vp * n)(*[f.ptr for f in x])
    sg = (ctypes.c_double * n)(*[float(v) for v in sigma])
    conv = (ctypes.c_int * n)()
    tr = (ctypes.c_double * n)()
    iters = ctypes.c_int()
    st = lib().qdp_cg_solve_multishift(xs, n, sg, phi, U, A, Ainv, float(mass), float(tol), int(maxit),
                                       ctypes.byref(iters), conv, hist, int(hist_cap), tr if true_resid else None)
    _check(st, phi.ctx)
    k = iters.value
    return dict(status=st, iters=k, conv_iter=np.array(conv[:]), hist=np.array(hist[:min(k + 1, hist_cap)]),
                true_resid=np.array(tr[:]) if true_resid else None)


def qdp_expr(expr: int, out: Field, a: Field, b: Field, c: Field = None) -> None:
    """Table II site expression on out's subset."""
    _check(lib().qdp_expr(int(expr), out, a, b, c), out.ctx)


def qdp_expr_block(ctx: Ctx, expr: int, prec: int):
    """(block size, tuned) of the paper's autotuner for (expr, prec)."""
    b, t = ctypes.c_int(), ctypes.c_int()
    _check(lib().qdp_expr_block(ctx, int(expr), int(prec), ctypes.byref(b), ctypes.byref(t)), ctx)
    return b.value, bool(t.value)


# ------------------------------------------------------------------ run-time generated expressions
def qdp_jit_eval(out: Field, expr: str, *operands: Field) -> None:
    """out = expr($0, $1, ...) on out's subset: one generated kernel (include/qdpb.h, PAPER.md III-IV)."""
    arr = (_vp * max(1, len(operands)))(*[f.ptr for f in operands])
    _check(lib().qdp_jit_eval(out, expr.encode(), arr, len(operands)), out.ctx)


def qdp_jit_sum(ctx: Ctx, expr: str, *operands: Field, subset: int = QDP_ALL) -> complex:
    """Global sum over `subset` of a complex-scalar site expression (trace / localNorm2 /
    localInnerProduct / real; include/qdpb.h)."""
    arr = (_vp * max(1, len(operands)))(*[f.ptr for f in operands])
    v = (ctypes.c_double * 2)()
    _check(lib().qdp_jit_sum(ctx, expr.encode(), arr, len(operands), int(subset), v), ctx)
    return complex(v[0], v[1])


QDP_JIT_SUM = -1


def qdp_jit_source(expr: str, out_kind: int, prec: int, operand_kinds, compile: bool = False, out_subset: int = -1):
    """(generated CUDA source, {flops, bytes, table2_bytes} per site) -- no context or GPU needed."""
    kinds = (ctypes.c_int * max(1, len(operand_kinds)))(*[int(k) for k in operand_kinds])
    need = ctypes.c_size_t()
    work = (ctypes.c_double * 3)()
    L = lib()
    for attempt in range(2):
        buf = ctypes.create_string_buffer(max(1, need.value))
        st = L.qdp_jit_source(expr.encode(), int(out_kind), int(out_subset), int(prec), kinds, len(operand_kinds), buf, len(buf),
                              ctypes.byref(need), work, 1 if (compile and attempt) else 0)
        if st < 0:  # the reason is in buf (once it is large enough)
            if need.value > len(buf):
                continue
            raise QdpError(st, L.qdp_strerror(st).decode() + f": {buf.value.decode()} in {expr!r}")
    return buf.value.decode(), dict(flops=work[0], bytes=work[1], table2_bytes=work[2])


def qdp_jit_stats(ctx: Ctx):
    """(kernels compiled on ctx, seconds spent generating + compiling + loading them)."""
    n, s = ctypes.c_int(), ctypes.c_double()
    _check(lib().qdp_jit_stats(ctx, ctypes.byref(n), ctypes.byref(s)), ctx)
    return n.value, s.value


# ------------------------------------------------------------------ diagnostics
def qdp_strerror(status: int) -> str:
    return lib().qdp_strerror(int(status)).decode()


def qdp_last_error(ctx: Ctx) -> str:
    return lib().qdp_last_error(ctx).decode()


def qdp_profile_query(ctx: Ctx, kernel_class: int = -1):
    n, ms = ctypes.c_long(), ctypes.c_double()
    _check(lib().qdp_profile_query(ctx, int(kernel_class), ctypes.byref(n), ctypes.byref(ms)), ctx)
    return n.value, ms.value


def qdp_profile_work(ctx: Ctx, kernel_class: int = -1):
    """(algorithmic flops, compulsory bytes) of the launches counted since the last reset."""
    f, b = ctypes.c_double(), ctypes.c_double()
    _check(lib().qdp_profile_work(ctx, int(kernel_class), ctypes.byref(f), ctypes.byref(b)), ctx)
    return f.value, b.value


def qdp_profile_reset(ctx: Ctx) -> None:
    _check(lib().qdp_profile_reset(ctx), ctx)
