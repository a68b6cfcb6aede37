"""Seeded synthetic input fields shared by the oracle tests, the CUDA-path tests and bench.py.

This module holds NONE of the method's arithmetic (no hopping term, no clover, no
BLAS, no solver).  It only produces inputs in the *host canonical layout* that the
C ABI (`include/qdpb.h`) and the oracle (`oracle/`) both accept:

  fermion  float64[V, 4 spin, 3 colour, 2 re/im]           (full lattice, lexicographic site)
  gauge    float64[V, 4 mu, 3 row, 3 col, 2 re/im]          (U_mu(x), row-major 3x3)

Site order (reading R7): s = x + Lx*(y + Ly*(z + Lz*t)), mu = 0,1,2,3 <-> x,y,z,t.

Random numbers: counter-based splitmix64 (value k of stream `seed` is
mix64(seed*PHI + (k+1)*GAMMA)), uniforms from the top 53 bits, one Box-Muller
cosine branch per Gaussian (uniforms 2k, 2k+1 -> Gaussian k).  The Gaussian
counter runs over the components in the fixed order of the host layout
(site, mu, row, col, re/im), SURVEY.md section 8(c) item 7.

Gauge links (reading R21): SU(3) by Gram-Schmidt of a complex Gaussian 3x3 with
row2 = conj(row0 x row1), so det = 1 to rounding.  "Warm" links are exp(i*eps*H)
with H a traceless Hermitian Gaussian matrix (exponentiated by eigendecomposition).
"""
from __future__ import annotations

import numpy as np

__all__ = [
    "volume", "coords", "parity", "gaussian", "uniform", "random_spinor",
    "random_su3", "random_gauge", "warm_gauge", "unit_gauge", "random_gauge_transform",
    "to_fp32", "cb_sites", "apply_antiperiodic_t", "random_gauge_sites", "random_spinor_sites",
    "random_gauge_torch", "random_spinor_torch",
]

_GAMMA = np.uint64(0x9E3779B97F4A7C15)
_PHI = np.uint64(0xD1B54A32D192ED03)
_M1 = np.uint64(0xBF58476D1CE4E5B9)
_M2 = np.uint64(0x94D049BB133111EB)


def _mix64(z: np.ndarray) -> np.ndarray:
    z = (z ^ (z >> np.uint64(30))) * _M1
    z = (z ^ (z >> np.uint64(27))) * _M2
    return z ^ (z >> np.uint64(31))


def _raw(seed: int, start: int, n: int) -> np.ndarray:
    with np.errstate(over="ignore"):
        base = np.uint64(seed & 0xFFFFFFFFFFFFFFFF) * _PHI
        k = np.arange(start + 1, start + n + 1, dtype=np.uint64)
        return _mix64(base + k * _GAMMA)


def uniform(seed: int, n: int, start: int = 0) -> np.ndarray:
    """n uniforms in (0, 1], counter positions start..start+n-1 of stream `seed`."""
    r = _raw(seed, start, n)
    return ((r >> np.uint64(11)).astype(np.float64) + 1.0) * (2.0 ** -53)


def gaussian(seed: int, n: int, start: int = 0, chunk: int = 1 << 24) -> np.ndarray:
    """n standard normals; Gaussian k uses uniforms 2k, 2k+1 (Box-Muller, cosine branch)."""
    out = np.empty(n, dtype=np.float64)
    for lo in range(0, n, chunk):
        m = min(chunk, n - lo)
        u = uniform(seed, 2 * m, 2 * (start + lo)).reshape(m, 2)
        out[lo:lo + m] = np.sqrt(-2.0 * np.log(u[:, 0])) * np.cos(2.0 * np.pi * u[:, 1])
    return out


def volume(L) -> int:
    L = tuple(int(v) for v in L)
    assert len(L) == 4
    return L[0] * L[1] * L[2] * L[3]


def coords(L) -> np.ndarray:
    """int64[V, 4] coordinates (x, y, z, t) of lexicographic sites."""
    V = volume(L)
    s = np.arange(V, dtype=np.int64)
    x = s % L[0]
    r = s // L[0]
    y = r % L[1]
    r //= L[1]
    z = r % L[2]
    t = r // L[2]
    return np.stack([x, y, z, t], axis=1)


def parity(L, origin=(0, 0, 0, 0)) -> np.ndarray:
    """int64[V] parity of each site, (X+Y+Z+T) mod 2 in global coordinates."""
    c = coords(L) + np.asarray(origin, dtype=np.int64)
    return c.sum(axis=1) & 1


def cb_sites(L, p: int) -> np.ndarray:
    """Lexicographic indices of the parity-p sites in checkerboard order (cb = s >> 1)."""
    par = parity(L)
    s = np.nonzero(par == p)[0]
    assert np.array_equal(s >> 1, np.arange(len(s)))
    return s


def random_spinor(L, seed: int) -> np.ndarray:
    """Gaussian fermion: every real component N(0,1).  float64[V,4,3,2]."""
    V = volume(L)
    return gaussian(seed, V * 24).reshape(V, 4, 3, 2)


def _su3_from_gaussian(g: np.ndarray) -> np.ndarray:
    """g: complex[N,3,3] -> SU(3) by Gram-Schmidt rows, row2 = conj(row0 x row1)."""
    r0 = g[:, 0, :]
    r0 = r0 / np.linalg.norm(r0, axis=1, keepdims=True)
    r1 = g[:, 1, :]
    r1 = r1 - np.sum(np.conj(r0) * r1, axis=1, keepdims=True) * r0
    r1 = r1 / np.linalg.norm(r1, axis=1, keepdims=True)
    r2 = np.conj(np.cross(r0, r1))
    return np.stack([r0, r1, r2], axis=1)


def random_su3(n: int, seed: int, chunk: int = 1 << 20, first: int = 0) -> np.ndarray:
    """n random SU(3) matrices as float64[n,3,3,2]: matrices first .. first+n-1 of stream `seed`."""
    out = np.empty((n, 3, 3, 2), dtype=np.float64)
    for lo in range(0, n, chunk):
        m = min(chunk, n - lo)
        g = gaussian(seed, m * 18, start=(first + lo) * 18).reshape(m, 3, 3, 2)
        c = _su3_from_gaussian(g[..., 0] + 1j * g[..., 1])
        out[lo:lo + m, ..., 0] = c.real
        out[lo:lo + m, ..., 1] = c.imag
    return out


def random_gauge(L, seed: int) -> np.ndarray:
    """Hot random SU(3) gauge field float64[V,4,3,3,2]."""
    V = volume(L)
    return random_su3(V * 4, seed).reshape(V, 4, 3, 3, 2)


def random_gauge_sites(seed: int, site_lo: int, n_sites: int) -> np.ndarray:
    """Sites site_lo .. site_lo+n_sites-1 of random_gauge(L, seed) (the counter-based stream makes
    any contiguous site range cheap: e.g. one time slice of a neighbouring rank's sub-lattice)."""
    return random_su3(n_sites * 4, seed, first=site_lo * 4).reshape(n_sites, 4, 3, 3, 2)


def random_spinor_sites(seed: int, site_lo: int, n_sites: int) -> np.ndarray:
    """Sites site_lo .. site_lo+n_sites-1 of random_spinor(L, seed)."""
    return gaussian(seed, n_sites * 24, start=site_lo * 24).reshape(n_sites, 4, 3, 2)


def random_gauge_torch(L, seed: int, device="cuda"):
    """Hot random SU(3) gauge field generated on `device` with torch's generator (float64 tensor
    [V,4,3,3,2], host canonical layout).  Same Gram-Schmidt construction as random_gauge, but NOT
    the same numbers: for timing-only workloads whose fields are too large to generate on the host
    in reasonable time (no parity claim rests on them)."""
    import torch
    V = volume(L)
    gen = torch.Generator(device=device)
    gen.manual_seed(int(seed))
    out = torch.empty((V * 4, 3, 3, 2), dtype=torch.float64, device=device)
    chunk = 1 << 22
    for lo in range(0, V * 4, chunk):
        m = min(chunk, V * 4 - lo)
        g = torch.randn((m, 3, 3, 2), dtype=torch.float64, device=device, generator=gen)
        a = torch.complex(g[..., 0], g[..., 1])
        r0 = a[:, 0, :] / torch.linalg.vector_norm(a[:, 0, :], dim=1, keepdim=True)
        r1 = a[:, 1, :] - torch.sum(torch.conj(r0) * a[:, 1, :], dim=1, keepdim=True) * r0
        r1 = r1 / torch.linalg.vector_norm(r1, dim=1, keepdim=True)
        r2 = torch.conj(torch.linalg.cross(r0, r1, dim=1))
        c = torch.stack([r0, r1, r2], dim=1)
        out[lo:lo + m, ..., 0] = c.real
        out[lo:lo + m, ..., 1] = c.imag
    return out.reshape(V, 4, 3, 3, 2)


def random_spinor_torch(L, seed: int, device="cuda"):
    """Gaussian fermion generated on `device` (float64 tensor [V,4,3,2]); see random_gauge_torch."""
    import torch
    gen = torch.Generator(device=device)
    gen.manual_seed(int(seed))
    return torch.randn((volume(L), 4, 3, 2), dtype=torch.float64, device=device, generator=gen)


def warm_gauge(L, seed: int, eps: float, chunk: int = 1 << 20) -> np.ndarray:
    """U = exp(i eps H), H traceless Hermitian with Gaussian entries.  float64[V,4,3,3,2]."""
    V = volume(L)
    n = V * 4
    out = np.empty((n, 3, 3, 2), dtype=np.float64)
    for lo in range(0, n, chunk):
        m = min(chunk, n - lo)
        g = gaussian(seed, m * 18, start=lo * 18).reshape(m, 3, 3, 2)
        a = g[..., 0] + 1j * g[..., 1]
        h = 0.5 * (a + np.conj(np.swapaxes(a, 1, 2)))
        tr = np.trace(h, axis1=1, axis2=2).real / 3.0
        h = h - tr[:, None, None] * np.eye(3)[None]
        w, v = np.linalg.eigh(h)
        e = np.exp(1j * eps * w)
        u = np.einsum("nij,nj,nkj->nik", v, e, np.conj(v))
        out[lo:lo + m, ..., 0] = u.real
        out[lo:lo + m, ..., 1] = u.imag
    return out.reshape(V, 4, 3, 3, 2)


def unit_gauge(L) -> np.ndarray:
    V = volume(L)
    U = np.zeros((V, 4, 3, 3, 2))
    U[:, :, 0, 0, 0] = U[:, :, 1, 1, 0] = U[:, :, 2, 2, 0] = 1.0
    return U


def random_gauge_transform(L, seed: int) -> np.ndarray:
    """One random SU(3) matrix per site: float64[V,3,3,2]."""
    return random_su3(volume(L), seed)


def apply_antiperiodic_t(U: np.ndarray, L) -> np.ndarray:
    """Reading R5: antiperiodic fermion BC in t as a sign flip of U_t on the last time slice."""
    U = U.copy()
    c = coords(L)
    U[c[:, 3] == L[3] - 1, 3] *= -1.0
    return U


def to_fp32(a: np.ndarray) -> np.ndarray:
    """Round to float32 (SP inputs); the oracle then runs in double on these rounded values."""
    return np.ascontiguousarray(a, dtype=np.float32)
