"""Test-side helpers written independently of oracle/ and of the CUDA path.

The gamma matrices are typed here from DESIGN.md reading R1 (DeGrand-Rossi) and are
checked against the Clifford algebra in tests/test_oracle_dslash.py, so a typo in
the oracle's own table cannot hide behind a shared constant.
"""
import numpy as np

import fieldgen

_i = 1j
GAMMA = [
    np.array([[0, 0, 0, _i], [0, 0, _i, 0], [0, -_i, 0, 0], [-_i, 0, 0, 0]]),
    np.array([[0, 0, 0, -1], [0, 0, 1, 0], [0, 1, 0, 0], [-1, 0, 0, 0]], dtype=complex),
    np.array([[0, 0, _i, 0], [0, 0, 0, -_i], [-_i, 0, 0, 0], [0, _i, 0, 0]]),
    np.array([[0, 0, 1, 0], [0, 0, 0, 1], [1, 0, 0, 0], [0, 1, 0, 0]], dtype=complex),
]
GAMMA5 = GAMMA[0] @ GAMMA[1] @ GAMMA[2] @ GAMMA[3]


def c(a):
    """real [...,2] -> complex [...]"""
    return a[..., 0] + 1j * a[..., 1]


def r(z):
    """complex [...] -> real [...,2]"""
    return np.stack([z.real, z.imag], axis=-1)


def site_index(cx, L):
    return cx[..., 0] + L[0] * (cx[..., 1] + L[1] * (cx[..., 2] + L[2] * cx[..., 3]))


def neighbour(L, mu, sign):
    """int[V]: lexicographic index of x + sign*mu^ (periodic)."""
    cx = fieldgen.coords(L).copy()
    cx[:, mu] = (cx[:, mu] + sign) % L[mu]
    return site_index(cx, L)


def gauge_transform(U, g, L):
    """U^g_mu(x) = g(x) U_mu(x) g(x+mu)^dag."""
    Uc, gc = c(U), c(g)
    out = np.empty_like(Uc)
    for mu in range(4):
        f = neighbour(L, mu, +1)
        out[:, mu] = gc @ Uc[:, mu] @ np.conj(np.swapaxes(gc[f], 1, 2))
    return r(out)


def colour_rotate(psi, g):
    """(g psi)(x) = g(x) psi(x) on colour."""
    return r(np.einsum("sab,sib->sia", c(g), c(psi)))


def spin_apply(M, psi):
    """(M psi)(x) = M psi(x) on spin, M a 4x4 complex matrix."""
    return r(np.einsum("ij,sjc->sic", M, c(psi)))


def cdot(a, b):
    """<a, b> = sum conj(a) b (plain numpy, for invariants)."""
    return np.vdot(c(a).ravel(), c(b).ravel())


def rel_site_err(got, ref):
    """max_x |got(x) - ref(x)|_2 / |ref(x)|_2 (reading R18; rms floor for tiny sites)."""
    g = got.reshape(got.shape[0], -1)
    o = ref.reshape(ref.shape[0], -1)
    d = np.linalg.norm(g - o, axis=1)
    n = np.linalg.norm(o, axis=1)
    rms = np.sqrt(np.mean(n ** 2)) if n.size else 0.0
    n = np.where(n < 1e-12 * rms, rms, n)
    if rms == 0.0:
        return float(np.max(d)) if d.size else 0.0
    return float(np.max(d / n))
