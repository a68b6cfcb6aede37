"""ctypes wrapper around oracle/liboracle.so (the plain C reference, oracle/oracle.c).

TEST INFRASTRUCTURE ONLY: imported by tests/, __graft_entry__.smoke() and bench.py's
cpu_baseline / `--impl reference` legs, never by the product package
(paper_1408_5925_b200/).  The product path fails loudly when its CUDA library is
missing; it never falls back to this module.

All arrays are numpy float64 in the host canonical layouts of fieldgen/:
fermion [V,4,3,2], gauge [V,4,3,3,2], clover dense [V,12,12,2].
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")
_lib = None


def build(force: bool = False) -> str:
    """Compile oracle.c with gcc (IEEE double, no fast-math)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        tmp = _LIB + f".tmp{os.getpid()}"
        subprocess.check_call(["gcc", "-O2", "-std=gnu99", "-fopenmp", "-fPIC", "-shared",
                               "-fno-fast-math", "-ffp-contract=off", _SRC, "-o", tmp, "-lm"])
        os.replace(tmp, _LIB)
    return _LIB


def lib():
    global _lib
    if _lib is None:
        build()
        _lib = ctypes.CDLL(_LIB)
        dp = ctypes.POINTER(ctypes.c_double)
        ip = ctypes.POINTER(ctypes.c_int)
        _lib.orc_norm2.restype = ctypes.c_double
        _lib.orc_cg_solve.restype = ctypes.c_int
        _lib.orc_cg_multishift.restype = ctypes.c_int
        _lib.orc_clover_invert.restype = ctypes.c_int
        _lib.orc_max_threads.restype = ctypes.c_int
        del dp, ip
    return _lib


def _p(a: np.ndarray):
    assert a.dtype == np.float64 and a.flags["C_CONTIGUOUS"], (a.dtype, a.flags)
    return a.ctypes.data_as(ctypes.POINTER(ctypes.c_double))


def _L(L):
    return (ctypes.c_int * 4)(*[int(v) for v in L])


def _f64(a):
    return np.ascontiguousarray(a, dtype=np.float64)


def max_threads() -> int:
    return int(lib().orc_max_threads())


def set_threads(n: int) -> None:
    lib().orc_set_threads(int(n))


def gamma(mu: int) -> np.ndarray:
    out = np.zeros((4, 4, 2))
    lib().orc_gamma(int(mu), _p(out))
    return out[..., 0] + 1j * out[..., 1]


def shift(field: np.ndarray, L, mu: int, sign: int) -> np.ndarray:
    """out(x) = in(x + sign*mu^), periodic."""
    f = _f64(field)
    V = int(np.prod(L))
    out = np.empty_like(f)
    lib().orc_shift(_p(out), _p(f), _L(L), int(f.size // V), int(mu), int(sign))
    return out


def hopping(U, psi, L, out_parity: int = -1) -> np.ndarray:
    """(H psi)(x) of PAPER.md:282 on sites of out_parity (-1: all); other sites 0."""
    U = _f64(U)
    psi = _f64(psi)
    out = np.empty_like(psi)
    lib().orc_hopping(_p(out), _p(U), _p(psi), _L(L), int(out_parity))
    return out


def norm2(a, L, subset: int = -1) -> float:
    return float(lib().orc_norm2(_p(_f64(a)), _L(L), int(subset)))


def inner(a, b, L, subset: int = -1) -> complex:
    out = np.zeros(2)
    lib().orc_inner(_p(_f64(a)), _p(_f64(b)), _L(L), int(subset), _p(out))
    return complex(out[0], out[1])


def axpy(a: complex, x, y, L, subset: int = -1) -> np.ndarray:
    """returns a*x + y on the subset (y copied; other sites of y unchanged)."""
    y2 = _f64(y).copy()
    a = complex(a)
    lib().orc_axpy(ctypes.c_double(a.real), ctypes.c_double(a.imag), _p(_f64(x)), _p(y2), _L(L), int(subset))
    return y2


def clover_build(U, L, mass: float, csw: float) -> np.ndarray:
    """Dense A(x) = (4+m) + 1/4 c_SW sigma F (eq. 1, reading R10). [V,12,12,2]"""
    V = int(np.prod(L))
    A = np.empty((V, 12, 12, 2))
    lib().orc_clover_build(_p(A), _p(_f64(U)), _L(L), ctypes.c_double(mass), ctypes.c_double(csw))
    return A


def clover_invert(A, L, subset: int = -1) -> np.ndarray:
    out = np.empty_like(_f64(A))
    st = lib().orc_clover_invert(_p(out), _p(_f64(A)), _L(L), int(subset))
    if st != 0:
        raise ZeroDivisionError("singular clover block")
    return out


def clover_apply(A, psi, L, subset: int = -1) -> np.ndarray:
    out = _f64(psi).copy()
    lib().orc_clover_apply(_p(out), _p(_f64(A)), _p(_f64(psi)), _L(L), int(subset))
    return out


def wilson_apply(U, A, mass: float, v, L) -> np.ndarray:
    """M v = A v - H v / 2 (full lattice); A=None -> Wilson A = 4+m."""
    v = _f64(v)
    out = np.empty_like(v)
    Ap = _p(_f64(A)) if A is not None else None
    lib().orc_wilson_apply(_p(out), _p(_f64(U)), Ap, ctypes.c_double(mass), _p(v), _L(L))
    return out


def cg_solve(U, b, L, mass: float, A=None, tol: float = 1e-10, maxit: int = 10000):
    """Even-odd CGNR.  Returns dict(x, iters, hist, true_resid, status)."""
    b = _f64(b)
    x = np.zeros_like(b)
    hist = np.zeros(maxit + 1)
    iters = ctypes.c_int(0)
    tr = ctypes.c_double(0.0)
    Ap = _p(_f64(A)) if A is not None else None
    st = lib().orc_cg_solve(_p(x), _p(b), _p(_f64(U)), Ap, ctypes.c_double(mass), _L(L),
                            ctypes.c_double(tol), int(maxit), ctypes.byref(iters), _p(hist),
                            int(maxit + 1), ctypes.byref(tr))
    if st < 0:
        raise ZeroDivisionError("singular clover block")
    n = iters.value
    return dict(x=x, iters=n, hist=hist[:n + 1].copy(), true_resid=tr.value, status=st)


def mhat_apply(U, A, mass: float, v, L, dagger: bool = False) -> np.ndarray:
    """Mhat v (or Mhat^dag v) on the odd sites, Mhat = A_oo - 1/4 H_oe A_ee^-1 H_eo; even sites 0."""
    v = _f64(v)
    out = np.zeros_like(v)
    Ap = _p(_f64(A)) if A is not None else None
    lib().orc_mhat_apply(_p(out), _p(_f64(U)), Ap, ctypes.c_double(mass), _p(v), _L(L), int(bool(dagger)))
    return out


def cg_multishift(U, phi, L, mass: float, sigma, A=None, tol: float = 1e-10, maxit: int = 10000):
    """Multi-shift CG for (Mhat^dag Mhat + sigma_i) x_i = phi_o (oracle.c orc_cg_multishift).
    Returns dict(x [n,V,4,3,2], iters, conv_iter [n], hist, true_resid [n], status)."""
    phi = _f64(phi)
    sigma = np.ascontiguousarray(sigma, dtype=np.float64)
    n = len(sigma)
    x = np.zeros((n,) + phi.shape)
    hist = np.zeros(maxit + 1)
    conv = (ctypes.c_int * n)()
    tr = np.zeros(n)
    iters = ctypes.c_int(0)
    Ap = _p(_f64(A)) if A is not None else None
    st = lib().orc_cg_multishift(_p(x), _p(phi), _p(_f64(U)), Ap, ctypes.c_double(mass), _L(L), int(n), _p(sigma),
                                 ctypes.c_double(tol), int(maxit), ctypes.byref(iters), conv, _p(hist),
                                 int(maxit + 1), _p(tr))
    if st == -1:
        raise ZeroDivisionError("singular clover block")
    if st == -2:
        raise ValueError("shifts: sigma[0] must be the smallest")
    k = iters.value
    return dict(x=x, iters=k, conv_iter=np.array(conv[:]), hist=hist[:k + 1].copy(), true_resid=tr, status=st)


def _n(a, per):
    return int(np.asarray(a).size // per)


def lcm(a, b) -> np.ndarray:
    """Table II lcm: site-wise 3x3 product.  a, b: [n,3,3,2]."""
    a, b = _f64(a), _f64(b)
    out = np.empty_like(a)
    lib().orc_lcm(_p(out), _p(a), _p(b), ctypes.c_long(_n(a, 18)))
    return out


def upsi(u, psi) -> np.ndarray:
    """Table II upsi: colour matrix times the colour vector of each spin.  u [n,3,3,2], psi [n,4,3,2]."""
    u, psi = _f64(u), _f64(psi)
    out = np.empty_like(psi)
    lib().orc_upsi(_p(out), _p(u), _p(psi), ctypes.c_long(_n(u, 18)))
    return out


def adj_upsi(u, psi) -> np.ndarray:
    """adj(u) * psi on every spin (Fig. 1's adj(u[mu])*phi)."""
    u, psi = _f64(u), _f64(psi)
    out = np.empty_like(psi)
    lib().orc_adj_upsi(_p(out), _p(u), _p(psi), ctypes.c_long(_n(u, 18)))
    return out


def spmat(a, b) -> np.ndarray:
    """Table II spmat: site-wise 4x4 product.  a, b: [n,4,4,2]."""
    a, b = _f64(a), _f64(b)
    out = np.empty_like(a)
    lib().orc_spmat(_p(out), _p(a), _p(b), ctypes.c_long(_n(a, 32)))
    return out


def matvec(u, p1, p2) -> np.ndarray:
    """Table II matvec: u psi1 + u psi2."""
    u, p1, p2 = _f64(u), _f64(p1), _f64(p2)
    out = np.empty_like(p1)
    lib().orc_matvec(_p(out), _p(u), _p(p1), _p(p2), ctypes.c_long(_n(u, 18)))
    return out
