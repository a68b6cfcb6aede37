// dslash_impl.cuh -- fused even-odd Wilson hopping term (section VIII-C) with
// face packing and interior/exterior split for the halo overlap of section V
// (PAPER.md:208-214).
//
//   (H psi)(x) = sum_mu [(1 - gamma_mu) U_mu(x) psi(x+mu) + (1 + gamma_mu) U_mu(x-mu)^dag psi(x-mu)]
//
// One thread per output site.  Per direction: load the neighbour spinor, spin-project to a
// half spinor with (1 -/+ gamma_mu) (12 flop), multiply by U or U^dag (2 x 66 flop),
// reconstruct rows 2,3 from rows 0,1 and accumulate (24 flop) -> 1320 flop per site
// (DESIGN.md "Flop and byte accounting").  Projection/reconstruction follow the
// DeGrand-Rossi basis (reading R1); the derivation is in DESIGN.md "Spin projection".
//
// Included by one translation unit per (precision, gauge storage) -- dslash_{d18,d12,f18,f12,h16}.cu --
// so the kernel instantiations compile in parallel; dslash.cu dispatches.
//
// Epilogues (fused into the same kernel, so the hopping result never round-trips HBM):
//   EPI_PLAIN    out = b [g5] H psi
//   EPI_XPAY     out = a x + b [g5] H psi
//   EPI_CLOVINV  out = A^{-1} (a x + b [g5] H psi)         (x optional)
//   EPI_CLOVXPAY out = A x + b [g5] H psi
// g5_in applies gamma5 to psi as it is loaded (Mhat^dag = g5 Mhat g5).
#pragma once
#include <type_traits>

#ifndef QDPB_H16_F32X2
#define QDPB_H16_F32X2 1  // 16-bit dslash: SU(3) products and accumulation in packed fp32 pairs (FFMA2)
#endif
#ifndef QDPB_TUNE_O8
#define QDPB_TUNE_O8 1  // offer the 128-register small-volume variant (5) to the tuner
#endif

#include "internal.h"

namespace qdpb {

template <typename R> struct HalfGhost;  // ghost half-spinor SoA: 6 complex per face site
template <> struct HalfGhost<double> {
  static __device__ __forceinline__ void store(void *buf, int n, int f, const Half<double> &h) {
    double2 *q = (double2 *)buf;
#pragma unroll
    for (int k = 0; k < 6; k++) q[(size_t)k * n + f] = make_double2(h.c[k].re, h.c[k].im);
  }
  // Ghosts may be written by other blocks of the same kernel or by a peer GPU while this kernel
  // runs (peer-to-peer halo): coherent L2 loads (ld.global.cg) after the acquire, never the
  // non-coherent read-only path.
  static __device__ __forceinline__ Half<double> load(const void *buf, int n, int f) {
    const double2 *q = (const double2 *)buf;
    Half<double> h;
#pragma unroll
    for (int k = 0; k < 6; k++) {
      double2 v = __ldcg(q + (size_t)k * n + f);
      h.c[k] = {v.x, v.y};
    }
    return h;
  }
};
template <> struct HalfGhost<float> {
  static __device__ __forceinline__ void store(void *buf, int n, int f, const Half<float> &h) {
    float4 *q = (float4 *)buf;
#pragma unroll
    for (int k = 0; k < 3; k++)
      q[(size_t)k * n + f] = make_float4(h.c[2 * k].re, h.c[2 * k].im, h.c[2 * k + 1].re, h.c[2 * k + 1].im);
  }
  static __device__ __forceinline__ Half<float> load(const void *buf, int n, int f) {
    const float4 *q = (const float4 *)buf;
    Half<float> h;
#pragma unroll
    for (int k = 0; k < 3; k++) {
      float4 v = __ldcg(q + (size_t)k * n + f);  // coherent: see HalfGhost<double>::load
      h.c[2 * k] = {v.x, v.y};
      h.c[2 * k + 1] = {v.z, v.w};
    }
    return h;
  }
};

// rows 0,1 of (1 + S gamma_mu) psi  (S = -1: forward hop, S = +1: backward hop)
template <int MU, int S, typename R>
__device__ __forceinline__ Half<R> project(const Spinor<R> &p) {
  Half<R> h;
#pragma unroll
  for (int c = 0; c < 3; c++) {
    const cx<R> p0 = p.c[c], p1 = p.c[3 + c], p2 = p.c[6 + c], p3 = p.c[9 + c];
    if (MU == 0) {        // h0 = p0 + S i p3, h1 = p1 + S i p2
      h.c[c] = S > 0 ? p0 + times_i(p3) : p0 - times_i(p3);
      h.c[3 + c] = S > 0 ? p1 + times_i(p2) : p1 - times_i(p2);
    } else if (MU == 1) { // h0 = p0 - S p3, h1 = p1 + S p2
      h.c[c] = S > 0 ? p0 - p3 : p0 + p3;
      h.c[3 + c] = S > 0 ? p1 + p2 : p1 - p2;
    } else if (MU == 2) { // h0 = p0 + S i p2, h1 = p1 - S i p3
      h.c[c] = S > 0 ? p0 + times_i(p2) : p0 - times_i(p2);
      h.c[3 + c] = S > 0 ? p1 - times_i(p3) : p1 + times_i(p3);
    } else {              // h0 = p0 + S p2, h1 = p1 + S p3
      h.c[c] = S > 0 ? p0 + p2 : p0 - p2;
      h.c[3 + c] = S > 0 ? p1 + p3 : p1 - p3;
    }
  }
  return h;
}

// acc += (1 + S gamma_mu) reconstructed from its rows 0,1 (h already colour-multiplied)
template <int MU, int S, typename R>
__device__ __forceinline__ void accum_recon(Spinor<R> &acc, const Half<R> &h) {
#pragma unroll
  for (int c = 0; c < 3; c++) {
    const cx<R> h0 = h.c[c], h1 = h.c[3 + c];
    acc.c[c] = acc.c[c] + h0;
    acc.c[3 + c] = acc.c[3 + c] + h1;
    if (MU == 0) {        // r2 = -S i h1, r3 = -S i h0
      acc.c[6 + c] = S > 0 ? acc.c[6 + c] - times_i(h1) : acc.c[6 + c] + times_i(h1);
      acc.c[9 + c] = S > 0 ? acc.c[9 + c] - times_i(h0) : acc.c[9 + c] + times_i(h0);
    } else if (MU == 1) { // r2 = S h1, r3 = -S h0
      acc.c[6 + c] = S > 0 ? acc.c[6 + c] + h1 : acc.c[6 + c] - h1;
      acc.c[9 + c] = S > 0 ? acc.c[9 + c] - h0 : acc.c[9 + c] + h0;
    } else if (MU == 2) { // r2 = -S i h0, r3 = S i h1
      acc.c[6 + c] = S > 0 ? acc.c[6 + c] - times_i(h0) : acc.c[6 + c] + times_i(h0);
      acc.c[9 + c] = S > 0 ? acc.c[9 + c] + times_i(h1) : acc.c[9 + c] - times_i(h1);
    } else {              // r2 = S h0, r3 = S h1
      acc.c[6 + c] = S > 0 ? acc.c[6 + c] + h0 : acc.c[6 + c] - h0;
      acc.c[9 + c] = S > 0 ? acc.c[9 + c] + h1 : acc.c[9 + c] - h1;
    }
  }
}

// Runtime-mu forms of project / accum_recon for the boundary code (face packing, remote hops): one
// copy of the code for every direction instead of four, so the fused boundary kernel's packing and
// face-site regions stay small next to the interior's hop code in the instruction cache.  Same
// arithmetic as the compile-time forms (a unit factor +-1 / +-i is exact), so results are identical.
template <typename T>
__device__ __forceinline__ cx<T> mul_unit(cx<T> p, bool im, T sgn) {  // sgn * p or sgn * i p
  return im ? cx<T>{-sgn * p.im, sgn * p.re} : cx<T>{sgn * p.re, sgn * p.im};
}
// rows 0,1 of (1 + S gamma_mu) psi: h0 = p0 + a0 p[k0], h1 = p1 + a1 p[k1] (table of project)
template <typename T>
__device__ __forceinline__ Half<T> project_rt(const Spinor<T> &p, int mu, int S) {
  const bool lo = mu < 2;  // k0 = 3, k1 = 2 (else k0 = 2, k1 = 3); selects, not run-time indices
  const bool im = (mu & 1) == 0;
  const T a0 = (T)(mu == 1 ? -S : S), a1 = (T)(mu == 2 ? -S : S);
  Half<T> h;
#pragma unroll
  for (int c = 0; c < 3; c++) {
    h.c[c] = p.c[c] + mul_unit(lo ? p.c[9 + c] : p.c[6 + c], im, a0);
    h.c[3 + c] = p.c[3 + c] + mul_unit(lo ? p.c[6 + c] : p.c[9 + c], im, a1);
  }
  return h;
}
// acc += (1 + S gamma_mu) reconstructed from h: rows 2,3 = b2 h[j2], b3 h[j3] (table of accum_recon)
template <typename T>
__device__ __forceinline__ void accum_recon_rt(Spinor<T> &acc, const Half<T> &h, int mu, int S) {
  const bool im = (mu & 1) == 0;
  const bool lo = mu < 2;  // rows 2,3 from h1, h0 (else from h0, h1)
  const T b2 = (T)((mu & 1) == 0 ? -S : S), b3 = (T)(lo ? -S : S);
#pragma unroll
  for (int c = 0; c < 3; c++) {
    acc.c[c] = acc.c[c] + h.c[c];
    acc.c[3 + c] = acc.c[3 + c] + h.c[3 + c];
    acc.c[6 + c] = acc.c[6 + c] + mul_unit(lo ? h.c[3 + c] : h.c[c], im, b2);
    acc.c[9 + c] = acc.c[9 + c] + mul_unit(lo ? h.c[c] : h.c[3 + c], im, b3);
  }
}

// acc += f x (the reconstruction of accum_recon), with every scaled term one fused multiply-add:
// the 16-bit dslash applies its operands' scales here instead of to every stored value
template <int K, typename R>
__device__ __forceinline__ void add_f(cx<R> &a, cx<R> h, R f) {  // K: 0 +h, 1 -h, 2 +i h, 3 -i h
  if (K == 0) { a.re = fma(f, h.re, a.re); a.im = fma(f, h.im, a.im); }
  else if (K == 1) { a.re = fma(-f, h.re, a.re); a.im = fma(-f, h.im, a.im); }
  else if (K == 2) { a.re = fma(-f, h.im, a.re); a.im = fma(f, h.re, a.im); }
  else { a.re = fma(f, h.im, a.re); a.im = fma(-f, h.re, a.im); }
}
template <int MU, int S, typename R>
__device__ __forceinline__ void accum_recon_f(Spinor<R> &acc, const Half<R> &h, R f) {
#pragma unroll
  for (int c = 0; c < 3; c++) {
    const cx<R> h0 = h.c[c], h1 = h.c[3 + c];
    add_f<0>(acc.c[c], h0, f);
    add_f<0>(acc.c[3 + c], h1, f);
    if (MU == 0) {        // r2 = -S i h1, r3 = -S i h0
      add_f<(S > 0 ? 3 : 2)>(acc.c[6 + c], h1, f);
      add_f<(S > 0 ? 3 : 2)>(acc.c[9 + c], h0, f);
    } else if (MU == 1) { // r2 = S h1, r3 = -S h0
      add_f<(S > 0 ? 0 : 1)>(acc.c[6 + c], h1, f);
      add_f<(S > 0 ? 1 : 0)>(acc.c[9 + c], h0, f);
    } else if (MU == 2) { // r2 = -S i h0, r3 = S i h1
      add_f<(S > 0 ? 3 : 2)>(acc.c[6 + c], h0, f);
      add_f<(S > 0 ? 2 : 3)>(acc.c[9 + c], h1, f);
    } else {              // r2 = S h0, r3 = S h1
      add_f<(S > 0 ? 0 : 1)>(acc.c[6 + c], h0, f);
      add_f<(S > 0 ? 0 : 1)>(acc.c[9 + c], h1, f);
    }
  }
}

// ---- packed fp32 pairs (FFMA2 / FMUL2, sm_100): the 16-bit dslash is issue-bound,
// and a complex multiply-add is two packed fused multiply-adds with one operand a broadcast scalar:
// a * h = a.re (h.re, h.im) + a.im (-h.im, h.re), the second vector i h formed once per h and reused
// across the three rows of the SU(3) product.  Same products and the same summation order as the
// scalar code (acc.re: + a.re h.re, then - a.im h.im; acc.im: + a.re h.im, then + a.im h.re).
typedef unsigned long long f2_t;
__device__ __forceinline__ f2_t f2pk(float x, float y) {
  f2_t d;
  asm("mov.b64 %0, {%1, %2};" : "=l"(d) : "f"(x), "f"(y));
  return d;
}
__device__ __forceinline__ f2_t f2pk(cx<float> a) { return f2pk(a.re, a.im); }
__device__ __forceinline__ cx<float> f2up(f2_t d) {
  cx<float> r;
  asm("mov.b64 {%0, %1}, %2;" : "=f"(r.re), "=f"(r.im) : "l"(d));
  return r;
}
__device__ __forceinline__ f2_t ffma2(f2_t a, f2_t b, f2_t c) {
  f2_t d;
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(a), "l"(b), "l"(c));
  return d;
}
__device__ __forceinline__ f2_t fmul2(f2_t a, f2_t b) {
  f2_t d;
  asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b));
  return d;
}
__device__ __forceinline__ f2_t splat(float x) { return f2pk(x, x); }
__device__ __forceinline__ f2_t times_i2(cx<float> h) { return f2pk(-h.im, h.re); }  // i h

__device__ __forceinline__ Half<float> mul_link2(const Link<float> &u, const Half<float> &h) {  // U h
  Half<float> r;
#pragma unroll
  for (int s = 0; s < 2; s++) {
    f2_t hv[3], ih[3];
#pragma unroll
    for (int b = 0; b < 3; b++) {
      hv[b] = f2pk(h.c[3 * s + b]);
      ih[b] = times_i2(h.c[3 * s + b]);
    }
#pragma unroll
    for (int a = 0; a < 3; a++) {
      f2_t acc = fmul2(splat(u.m[3 * a].re), hv[0]);
      acc = ffma2(splat(u.m[3 * a].im), ih[0], acc);
#pragma unroll
      for (int b = 1; b < 3; b++) {
        acc = ffma2(splat(u.m[3 * a + b].re), hv[b], acc);
        acc = ffma2(splat(u.m[3 * a + b].im), ih[b], acc);
      }
      r.c[3 * s + a] = f2up(acc);
    }
  }
  return r;
}
__device__ __forceinline__ Half<float> mul_link_dag2(const Link<float> &u, const Half<float> &h) {  // U^dag h
  Half<float> r;
#pragma unroll
  for (int s = 0; s < 2; s++) {
    f2_t hv[3], ih[3];
#pragma unroll
    for (int b = 0; b < 3; b++) {
      hv[b] = f2pk(h.c[3 * s + b]);
      ih[b] = times_i2(h.c[3 * s + b]);
    }
#pragma unroll
    for (int a = 0; a < 3; a++) {  // conj(u) h = u.re h - u.im (i h)
      f2_t acc = fmul2(splat(u.m[a].re), hv[0]);
      acc = ffma2(splat(-u.m[a].im), ih[0], acc);
#pragma unroll
      for (int b = 1; b < 3; b++) {
        acc = ffma2(splat(u.m[3 * b + a].re), hv[b], acc);
        acc = ffma2(splat(-u.m[3 * b + a].im), ih[b], acc);
      }
      r.c[3 * s + a] = f2up(acc);
    }
  }
  return r;
}
// acc += f x (the reconstruction of accum_recon) in packed pairs: +-h by +-f, +-i h by +-f on i h
template <int K>
__device__ __forceinline__ void add_f2(cx<float> &a, f2_t h, f2_t ih, float f) {  // K: 0 +h, 1 -h, 2 +i h, 3 -i h
  if (K == 0) a = f2up(ffma2(splat(f), h, f2pk(a)));
  else if (K == 1) a = f2up(ffma2(splat(-f), h, f2pk(a)));
  else if (K == 2) a = f2up(ffma2(splat(f), ih, f2pk(a)));
  else a = f2up(ffma2(splat(-f), ih, f2pk(a)));
}
template <int MU, int S>
__device__ __forceinline__ void accum_recon_f2(Spinor<float> &acc, const Half<float> &h, float f) {
#pragma unroll
  for (int c = 0; c < 3; c++) {
    const f2_t h0 = f2pk(h.c[c]), h1 = f2pk(h.c[3 + c]);
    const f2_t i0 = (MU == 0 || MU == 2) ? times_i2(h.c[c]) : h0, i1 = (MU == 0 || MU == 2) ? times_i2(h.c[3 + c]) : h1;
    add_f2<0>(acc.c[c], h0, i0, f);
    add_f2<0>(acc.c[3 + c], h1, i1, f);
    if (MU == 0) {        // r2 = -S i h1, r3 = -S i h0
      add_f2<(S > 0 ? 3 : 2)>(acc.c[6 + c], h1, i1, f);
      add_f2<(S > 0 ? 3 : 2)>(acc.c[9 + c], h0, i0, f);
    } else if (MU == 1) { // r2 = S h1, r3 = -S h0
      add_f2<(S > 0 ? 0 : 1)>(acc.c[6 + c], h1, i1, f);
      add_f2<(S > 0 ? 1 : 0)>(acc.c[9 + c], h0, i0, f);
    } else if (MU == 2) { // r2 = -S i h0, r3 = S i h1
      add_f2<(S > 0 ? 3 : 2)>(acc.c[6 + c], h0, i0, f);
      add_f2<(S > 0 ? 2 : 3)>(acc.c[9 + c], h1, i1, f);
    } else {              // r2 = S h0, r3 = S h1
      add_f2<(S > 0 ? 0 : 1)>(acc.c[6 + c], h0, i0, f);
      add_f2<(S > 0 ? 0 : 1)>(acc.c[9 + c], h1, i1, f);
    }
  }
}

template <typename R>
__device__ __forceinline__ Half<R> mul_link(const Link<R> &u, const Half<R> &h) {  // U h
  Half<R> r;
#pragma unroll
  for (int s = 0; s < 2; s++)
#pragma unroll
    for (int a = 0; a < 3; a++) {
      cx<R> acc = cmul(u.m[3 * a], h.c[3 * s]);
      acc = cmadd(u.m[3 * a + 1], h.c[3 * s + 1], acc);
      acc = cmadd(u.m[3 * a + 2], h.c[3 * s + 2], acc);
      r.c[3 * s + a] = acc;
    }
  return r;
}
template <typename R>
__device__ __forceinline__ Half<R> mul_link_dag(const Link<R> &u, const Half<R> &h) {  // U^dag h
  Half<R> r;
#pragma unroll
  for (int s = 0; s < 2; s++)
#pragma unroll
    for (int a = 0; a < 3; a++) {
      cx<R> acc = {u.m[a].re * h.c[3 * s].re + u.m[a].im * h.c[3 * s].im,
                   u.m[a].re * h.c[3 * s].im - u.m[a].im * h.c[3 * s].re};
      acc = cjmadd(u.m[3 + a], h.c[3 * s + 1], acc);
      acc = cjmadd(u.m[6 + a], h.c[3 * s + 2], acc);
      r.c[3 * s + a] = acc;
    }
  return r;
}

template <typename R>
__device__ __forceinline__ void g5(Spinor<R> &s) {
#pragma unroll
  for (int k = 6; k < 12; k++) s.c[k] = -s.c[k];
}

template <typename R, int REC = 18> struct KParams {
  FermView<R> out, psi, x;
  GaugeView<R, REC> U;
  CloverView<R> A;
  int parity;
  Arith_t<R> a, b;  // arithmetic type (fp32 for the 16-bit storage)
  // ghost buffers (exterior): [mu][dir], dir 0 = from -mu (already U^dag P+ psi), 1 = from +mu (P- psi)
  const void *ghost[4][2];
  // pack destinations: [mu][dir], dir 0 = to -mu neighbour, 1 = to +mu neighbour
  void *dst[4][2];
  // fused Re<dotx, out>: per-block partials
  FermView<R> dotx;
  double *dot_part;
  Arith_t<R> dot_shift;  // with a fused dot: out += dot_shift * dotx first
  // peer-to-peer halo (QDP_OPT_P2P; p2p.cu): pack waits war >= seq-2, stores, and its last
  // block release-stores seq into sig; the exterior waits ready >= seq and its last block
  // release-stores seq into ack_to.  pack_counter == nullptr: NCCL / direct halo.
  unsigned *pack_counter[4], *ext_counter[4];
  unsigned *sig[4][2], *ack_to[4][2];
  const unsigned *war[4][2], *ready[4][2];
  unsigned *err;
  unsigned seq;
  // fused boundary (peer-to-peer): leading blocks pack every partitioned face into the
  // neighbours' ghost slots; the rest visit the output sites interior first, then the sites on a
  // partitioned face, then the rest of the interior; the blocks holding face sites acquire the
  // ghosts and add the remote hops themselves (no exterior kernels, no read-modify-write of the
  // output); the NEXT call acknowledges the consumed ghosts to the senders as it starts
  int fuse;
  int fuse_npack;   // leading pack blocks
  int fuse_nin;     // interior sites: perm[0, nin) interior, perm[nin, Vh) on a partitioned face
  // the face sites are visited after the first fuse_kin interior sites (a multiple of blockDim;
  // fuse_nin: after every interior site), then the rest of the interior
  int fuse_kin;
  const int *perm;  // visiting order of the output parity's sites (nullptr: by arithmetic, below)
  // z or z x t partitioned: the sites come in (z,t) slabs of S = L0/2 x L1 consecutive cb indices;
  // interior slabs (z in [sz0, sz0 + nzi), t in [st0, ...)) first, then the face slabs listed here
  const int *face_slab;
  int sz0, nzi, st0;
  int pack_off[5];  // cumulative pack threads per dim (2 faceVh for a partitioned dim, else 0)
  // face packing as a work queue of pack_chunks chunks (blockDim items each): the leading blocks
  // and every block that is about to wait for a ghost take chunks until none is left, so a wait
  // never depends on a block that has not started (CUDA does not promise in-order dispatch)
  unsigned *pack_q;  // set seq & 1: {next chunk, chunks done}; the other set is reset by block 0
  int pack_chunks;
  int wait_all;     // QDP_OPT_OVERLAP = 0: every block waits for the ghosts (no overlap; Fig. 6)
  // fused inner product finished inside this kernel (reduce.cuh; whole-lattice or fused boundary)
  int red_fin;
  RedArgs red;
};

template <typename R, int MU, typename KP>
__device__ __forceinline__ void hop_dir(const Geom &g, const KP &P, const int c[4], int cb, int p,
                                        bool G5IN, bool halo, Spinor<Arith_t<R>> &acc) {
  using T = Arith_t<R>;
  // forward: (1 - gamma_mu) U_mu(x) psi(x + mu)
  {
    const bool remote = halo && ((g.part >> MU) & 1) && c[MU] == g.L[MU] - 1;
    if (!remote) {
      int n[4] = {c[0], c[1], c[2], c[3]};
      n[MU] = (c[MU] + 1 == g.L[MU]) ? 0 : c[MU] + 1;
      if constexpr (is_h16<R>()) {  // stored integers; both scales applied once, in the accumulation
        float sc;
        Spinor<T> s = P.psi.load_raw(coords_cb(g, n), sc);
        if (G5IN) g5(s);
#if QDPB_H16_F32X2
        accum_recon_f2<MU, -1>(acc, mul_link2(P.U.load_raw(MU, p, cb), project<MU, -1>(s)), sc * P.U.raw_scale);
#else
        accum_recon_f<MU, -1>(acc, mul_link(P.U.load_raw(MU, p, cb), project<MU, -1>(s)), sc * P.U.raw_scale);
#endif
      } else {
        Spinor<T> s = P.psi.load(coords_cb(g, n));
        if (G5IN) g5(s);
        Half<T> h = project<MU, -1>(s);
        Link<T> u = P.U.load(MU, p, cb);
        accum_recon<MU, -1>(acc, mul_link(u, h));
      }
    }
  }
  // backward: (1 + gamma_mu) U_mu(x - mu)^dag psi(x - mu)
  {
    const bool remote = halo && ((g.part >> MU) & 1) && c[MU] == 0;
    if (!remote) {
      int n[4] = {c[0], c[1], c[2], c[3]};
      n[MU] = (c[MU] == 0) ? g.L[MU] - 1 : c[MU] - 1;
      const int ncb = coords_cb(g, n);
      if constexpr (is_h16<R>()) {
        float sc;
        Spinor<T> s = P.psi.load_raw(ncb, sc);
        if (G5IN) g5(s);
#if QDPB_H16_F32X2
        accum_recon_f2<MU, +1>(acc, mul_link_dag2(P.U.load_raw(MU, 1 - p, ncb), project<MU, +1>(s)),
                               sc * P.U.raw_scale);
#else
        accum_recon_f<MU, +1>(acc, mul_link_dag(P.U.load_raw(MU, 1 - p, ncb), project<MU, +1>(s)),
                              sc * P.U.raw_scale);
#endif
      } else {
        Spinor<T> s = P.psi.load(ncb);
        if (G5IN) g5(s);
        Half<T> h = project<MU, +1>(s);
        Link<T> u = P.U.load(MU, 1 - p, ncb);
        accum_recon<MU, +1>(acc, mul_link_dag(u, h));
      }
    }
  }
}

template <typename R, int EPI, typename KP>
__device__ __forceinline__ Spinor<Arith_t<R>> epilogue(const KP &P, int cb, Spinor<Arith_t<R>> &acc, bool G5OUT) {
  using T = Arith_t<R>;
  if (G5OUT) g5(acc);
  Spinor<T> o;
  if (EPI == EPI_PLAIN) {
#pragma unroll
    for (int k = 0; k < 12; k++) o.c[k] = P.b * acc.c[k];
  } else if (EPI == EPI_XPAY) {
    Spinor<T> xv = P.x.load_stream(cb);
#pragma unroll
    for (int k = 0; k < 12; k++) o.c[k] = P.a * xv.c[k] + P.b * acc.c[k];
  } else if (EPI == EPI_CLOVINV) {
    if (P.x.p) {
      Spinor<T> xv = P.x.load_stream(cb);
#pragma unroll
      for (int k = 0; k < 12; k++) acc.c[k] = P.a * xv.c[k] + P.b * acc.c[k];
    } else {
#pragma unroll
      for (int k = 0; k < 12; k++) acc.c[k] = P.b * acc.c[k];
    }
    o = clover_mul_s(P.A, cb, acc);
  } else {  // EPI_CLOVXPAY
    Spinor<T> xv = P.x.load_stream(cb);
    Spinor<T> ax = clover_mul_s(P.A, cb, xv);
#pragma unroll
    for (int k = 0; k < 12; k++) o.c[k] = ax.c[k] + P.b * acc.c[k];
  }
  return o;
}

// Re<d, o> for the fused inner product (fp64 accumulation)
template <typename R>
__device__ __forceinline__ double re_dot(const Spinor<R> &d, const Spinor<R> &o) {
  double s = 0.0;
#pragma unroll
  for (int k = 0; k < 12; k++) s += (double)d.c[k].re * o.c[k].re + (double)d.c[k].im * o.c[k].im;
  return s;
}

// block sum of v -> part[2 * idx] (re), part[2 * idx + 1] = 0; blockDim <= 256
__device__ __forceinline__ void dot_block_partial(double v, double *part, int idx) {
  __shared__ double sm[8];
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  if (l == 0) sm[w] = v;
  __syncthreads();
  if (w == 0) {
    v = l < (int)(blockDim.x >> 5) ? sm[l] : 0.0;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    if (l == 0) {
      part[2 * idx] = v;
      part[2 * idx + 1] = 0.0;
    }
  }
}

// Whole-lattice (HALO=false) or interior (HALO=true: remote hops skipped) kernel.
// DOT: also accumulate Re<dot, out> per block into dot_part (fused inner product).
// Face packing for dim mu: input psi has parity q = 1 - p.
//   f <  faceVh: my sites at x_mu = 0      -> P^- psi          -> dst[mu][0] (the -mu neighbour's forward ghost)
//   f >= faceVh: my sites at x_mu = L-1    -> U_mu^dag P^+ psi  -> dst[mu][1] (the +mu neighbour's backward ghost)
template <typename R, int REC, bool G5IN, typename KP>
__device__ __forceinline__ void pack_site(const Geom &g, const KP &P, int mu, int f) {
  const int n = sel4(g.faceVh, mu);
  if (f >= 2 * n) return;
  const int q = 1 - P.parity;
  const bool fwd = f >= n;
  if (fwd) f -= n;
  int c[4];
  face_coords(g, mu, fwd ? sel4(g.L, mu) - 1 : 0, f, q, c);
  const int cb = coords_cb(g, c);
  using T = Arith_t<R>;
  Spinor<T> s = P.psi.load(cb);
  if (G5IN) g5(s);
  Half<T> h;
  if (!fwd) {
    h = project_rt(s, mu, -1);
    HalfGhost<T>::store(P.dst[mu][0], n, f, h);
  } else {
    h = project_rt(s, mu, +1);
    Link<T> u = P.U.load(mu, q, cb);
    HalfGhost<T>::store(P.dst[mu][1], n, f, mul_link_dag(u, h));
  }
}

template <typename R, int REC, bool G5IN>
__global__ void __launch_bounds__(128) pack_kernel(const Geom g, const KParams<R, REC> P, int mu) {
  // peer-to-peer: the receivers must have consumed this slot (written two calls ago)
  if (P.pack_counter[mu]) block_wait_flags(P.war[mu][0], P.war[mu][1], P.seq - 2u, P.err);
  pack_site<R, REC, G5IN>(g, P, mu, blockIdx.x * blockDim.x + threadIdx.x);
  // Peer-to-peer halo: the face stores above may target a neighbour's memory over NVLink.
  // Every thread fences them at system scope; the last block to finish publishes `seq` to the
  // two receivers' ready flags with release semantics (they acquire before reading).
  if (P.pack_counter[mu]) grid_signal_last(P.pack_counter[mu], P.sig[mu][0], P.sig[mu][1], P.seq);
}

// Fused boundary: take chunks of the face-packing work until none is left (every thread of the block
// calls it; roles are uniform per block).  Each chunk is blockDim consecutive pack items (pack_off
// order); the block publishes its chunks with one system fence and adds them to the done count; the
// block that completes the last chunk release-stores seq into the receivers' ready flags.
template <typename R, int REC, bool G5IN, typename KP>
__device__ __forceinline__ void pack_help(const Geom &g, const KP &P) {
  __shared__ int s_chunk;
  unsigned *q = P.pack_q + 2 * (P.seq & 1u);
  int mine = 0;
  for (;;) {
    if (threadIdx.x == 0) s_chunk = (int)atomicAdd(q, 1u);
    __syncthreads();
    const int ch = s_chunk;
    __syncthreads();
    if (ch >= P.pack_chunks) break;
    if (!mine) {  // the receivers must have consumed this slot (written two calls ago)
#pragma unroll 1
      for (int mu = 0; mu < 4; mu++)
        if ((g.part >> mu) & 1) block_wait_flags(P.war[mu][0], P.war[mu][1], P.seq - 2u, P.err);
    }
    // the item's dim found at run time: one copy of the packing code (instruction cache; project_rt)
    const int i = ch * (int)blockDim.x + threadIdx.x;
    if (i < P.pack_off[4]) {
      int mu = 0;
#pragma unroll 1
      while (i >= P.pack_off[mu + 1]) mu++;
      pack_site<R, REC, G5IN>(g, P, mu, i - P.pack_off[mu]);
    }
    mine++;
  }
  if (mine) {
    __syncthreads();
    if (threadIdx.x == 0) {
      __threadfence_system();
      const unsigned prev = atomicAdd(q + 1, (unsigned)mine);
      if (prev + (unsigned)mine == (unsigned)P.pack_chunks) {
        __threadfence_system();
        for (int mu = 0; mu < 4; mu++)
          if ((g.part >> mu) & 1) {
            st_release_sys(P.sig[mu][0], P.seq);
            st_release_sys(P.sig[mu][1], P.seq);
          }
      }
    }
  }
}

// Fused boundary: the remote hops of every partitioned dim for a site on its faces, from the ghost
// slots (forward: P^- psi(x + mu) from the +mu neighbour, multiplied here by U_mu(x); backward: the
// neighbour already applied U^dag P^+); runtime mu, one copy of the code (see project_rt)
template <typename R, typename KP>
__device__ __forceinline__ void remote_hops(const Geom &g, const KP &P, const int c[4], int cb, int p,
                                            Spinor<Arith_t<R>> &acc) {
  using T = Arith_t<R>;
#pragma unroll 1
  for (int mu = 0; mu < 4; mu++) {
    if (!((g.part >> mu) & 1)) continue;
    const int n = sel4(g.faceVh, mu), x = sel4(c, mu);
    if (x == sel4(g.L, mu) - 1) {
      const Half<T> h = HalfGhost<T>::load(P.ghost[mu][1], n, face_index(g, mu, c));
      accum_recon_rt(acc, mul_link(P.U.load(mu, p, cb), h), mu, -1);
    }
    if (x == 0) accum_recon_rt(acc, HalfGhost<T>::load(P.ghost[mu][0], n, face_index(g, mu, c)), mu, +1);
  }
}

template <typename R, int REC, int EPI, bool G5IN, bool G5OUT, bool HALO, bool DOT>
__device__ __forceinline__ void dslash_body(const Geom &g, const KParams<R, REC> &P) {
  pdl_enter();
  int cb = blockIdx.x * blockDim.x + threadIdx.x;
  const int vb = blockIdx.x;
  double dot = 0.0;
  bool face = false;  // fused boundary: this block holds sites on a partitioned face
  if (HALO && P.fuse) {
    // the other queue set (used by the previous call, which has completed) is reset for the next one;
    // and the previous call's ghosts are consumed -- that grid has completed (this kernel is launched
    // in plain stream order), so its ghost loads have all returned -- so this call acknowledges them
    // to the senders (release, system scope): no face block of any call fences or counts itself
    if (blockIdx.x == 0 && threadIdx.x == 0) {
      P.pack_q[2 * ((P.seq + 1u) & 1u)] = 0u;
      P.pack_q[2 * ((P.seq + 1u) & 1u) + 1] = 0u;
#pragma unroll
      for (int mu = 0; mu < 4; mu++)
        if ((g.part >> mu) & 1) {
          st_release_sys(P.ack_to[mu][0], P.seq - 1u);
          st_release_sys(P.ack_to[mu][1], P.seq - 1u);
        }
    }
    // leading blocks pack (work queue) and leave; a block about to wait for a ghost takes whatever
    // packing is left first, so a wait never depends on an unstarted block (one call site: one copy)
    const bool packer = (int)blockIdx.x < P.fuse_npack;
    cb -= P.fuse_npack * blockDim.x;
    // visiting position v -> interior sites [0, kin), the face sites, then interior [kin, nin)
    const int nf = g.Vh - P.fuse_nin, b0 = (int)(blockIdx.x - P.fuse_npack) * (int)blockDim.x;
    face = !packer && b0 + (int)blockDim.x > P.fuse_kin && b0 < P.fuse_kin + nf;
    if (packer || face || P.wait_all) pack_help<R, REC, G5IN>(g, P);
    if (packer) {
      if (DOT) {
        if (P.red_fin) red_finish(P.red, gridDim.x, vb, 0.0, 0.0, false);
        else dot_block_partial(0.0, P.dot_part, vb);
      }
      return;
    }
    if (cb >= P.fuse_kin) cb = cb < P.fuse_kin + nf ? P.fuse_nin + (cb - P.fuse_kin) : cb - nf;
    if (face || P.wait_all) {
#pragma unroll 1
      for (int mu = 0; mu < 4; mu++)
        if ((g.part >> mu) & 1) block_wait_flags(P.ready[mu][0], P.ready[mu][1], P.seq, P.err);
    }
    if (cb < g.Vh) {
      if (P.perm) {
        cb = P.perm[cb];
      } else if (P.face_slab) {  // z or z x t: interior (z,t) slabs by arithmetic, then the face slabs
        const int S = g.Lh0 * g.L[1];
        if (cb < P.fuse_nin) {
          const int sl = cb / S, zi = sl % P.nzi, ti = sl / P.nzi;
          cb += S * ((zi + P.sz0 + g.L[2] * (ti + P.st0)) - sl);
        } else {
          const int k = cb - P.fuse_nin, sl = k / S;
          cb = k - sl * S + S * __ldg(P.face_slab + sl);
        }
      } else {  // only t partitioned: interior [F, Vh - F), then the slabs t = 0 and t = L-1, by arithmetic
        const int F = g.faceVh[3];
        cb = cb < P.fuse_nin ? F + cb : (cb - P.fuse_nin < F ? cb - P.fuse_nin : cb);
      }
    }
  }
  Spinor<Arith_t<R>> o;
  bool have = false;
  if (cb < g.Vh) {
    const int p = P.parity;
    int c[4];
    cb_coords(g, cb, p, c);
    if constexpr (sizeof(R) == 4 && REC == 12 && QDPB_PF_F12) {
      // the site's 8 links towards L2 before their first use, without holding registers
#pragma unroll
      for (int mu = 0; mu < 4; mu++) {
        P.U.prefetch(mu, p, cb);
        int n[4] = {c[0], c[1], c[2], c[3]};
        n[mu] = (c[mu] == 0) ? g.L[mu] - 1 : c[mu] - 1;
        P.U.prefetch(mu, 1 - p, coords_cb(g, n));
      }
    }
    using T = Arith_t<R>;
    Spinor<T> acc;
#pragma unroll
    for (int k = 0; k < 12; k++) acc.c[k] = {T(0), T(0)};
    // fused boundary: a block without face sites has only interior sites (block-uniform: no remote hop
    // test per site and hop); the separate-kernel interior pass tests every site
    const bool halo = HALO && (!P.fuse || face);
    hop_dir<R, 0>(g, P, c, cb, p, G5IN, halo, acc);
    hop_dir<R, 1>(g, P, c, cb, p, G5IN, halo, acc);
    hop_dir<R, 2>(g, P, c, cb, p, G5IN, halo, acc);
    hop_dir<R, 3>(g, P, c, cb, p, G5IN, halo, acc);
    if (HALO && P.fuse && face) remote_hops<R>(g, P, c, cb, p, acc);  // from the neighbours' ghosts
    o = epilogue<R, EPI>(P, cb, acc, G5OUT);
    have = true;
    if (DOT) {
      // fused Re<d, out> (and out += dot_shift d: the base shift of the multi-shift CG)
      const Spinor<T> d = P.dotx.load_stream(cb);
      if (P.dot_shift != T(0)) {
#pragma unroll
        for (int k = 0; k < 12; k++) o.c[k] = o.c[k] + P.dot_shift * d.c[k];
      }
      dot = re_dot(d, o);
    }
  }
  // the block's partial of the fused dot goes out BEFORE the output stores (reduce.cuh red_arrive)
  bool red_last = false;
  if (DOT && P.red_fin) red_last = red_arrive(P.red, gridDim.x, vb, dot, 0.0);
  if (have) P.out.store(cb, o);
  if (DOT) {
    if (!P.red_fin) dot_block_partial(dot, P.dot_part, vb);
    else if (red_last) red_complete(P.red, gridDim.x, vb, false);
  }
}

template <typename R, int REC, int EPI, bool G5IN, bool G5OUT, bool HALO, bool DOT>
__global__ void __launch_bounds__(QDPB_DSLASH_MAXT, (dslash_minb<R, REC>()))
    dslash_kernel(const Geom g, const __grid_constant__ KParams<R, REC> P) {
  dslash_body<R, REC, EPI, G5IN, G5OUT, HALO, DOT>(g, P);
}

// Small-volume variant: the same code capped at 128 registers (8 x 64 threads per SM).  Below the
// bandwidth shoulder the whole lattice is little more than one wave of the 168-register kernel
// (16^3 x 32: 65536 sites for 56832 resident threads), so its second, nearly empty wave is the
// tail; at 8 blocks per SM every site is resident at once.  Whole lattice, no fused dot.
template <typename R, int REC, int EPI, bool G5IN, bool G5OUT>
__global__ void __launch_bounds__(64, 8) dslash_o8_kernel(const Geom g, const __grid_constant__ KParams<R, REC> P) {
  dslash_body<R, REC, EPI, G5IN, G5OUT, false, false>(g, P);
}

// Exterior: add the remote hops of dim mu for the output sites on its two faces.  With DOT,
// Re<dotx, increment> is accumulated: by linearity the interior's partial plus these give
// Re<dotx, out> of the final output.
template <typename R, int REC, int EPI, bool G5OUT, bool DOT>
__global__ void __launch_bounds__(128) exterior_kernel(const Geom g, const KParams<R, REC> P, int mu, double *dot_part) {
  const int n = g.faceVh[mu];
  int f = blockIdx.x * blockDim.x + threadIdx.x;
  double dot = 0.0;
  // peer-to-peer: acquire both ghosts of this call before reading them
  if (P.pack_counter[mu]) block_wait_flags(P.ready[mu][0], P.ready[mu][1], P.seq, P.err);
  if (f < 2 * n) {
    const int p = P.parity;
    const bool fwd = f >= n;  // fwd: site at x_mu = L-1 needs psi(x+mu) from the +mu neighbour
    if (fwd) f -= n;
    int c[4];
    face_coords(g, mu, fwd ? g.L[mu] - 1 : 0, f, p, c);
    const int cb = coords_cb(g, c);
    using T = Arith_t<R>;
    Spinor<T> acc;
#pragma unroll
    for (int k = 0; k < 12; k++) acc.c[k] = {T(0), T(0)};
    if (fwd) {
      Half<T> h = HalfGhost<T>::load(P.ghost[mu][1], n, f);
      Link<T> u = P.U.load(mu, p, cb);
      Half<T> uh = mul_link(u, h);
      switch (mu) {
        case 0: accum_recon<0, -1>(acc, uh); break;
        case 1: accum_recon<1, -1>(acc, uh); break;
        case 2: accum_recon<2, -1>(acc, uh); break;
        default: accum_recon<3, -1>(acc, uh); break;
      }
    } else {
      Half<T> uh = HalfGhost<T>::load(P.ghost[mu][0], n, f);
      switch (mu) {
        case 0: accum_recon<0, +1>(acc, uh); break;
        case 1: accum_recon<1, +1>(acc, uh); break;
        case 2: accum_recon<2, +1>(acc, uh); break;
        default: accum_recon<3, +1>(acc, uh); break;
      }
    }
    if (G5OUT) g5(acc);
#pragma unroll
    for (int k = 0; k < 12; k++) acc.c[k] = P.b * acc.c[k];
    if (EPI == EPI_CLOVINV) acc = clover_mul_s(P.A, cb, acc);
    Spinor<T> o = P.out.load_plain(cb);
#pragma unroll
    for (int k = 0; k < 12; k++) o.c[k] = o.c[k] + acc.c[k];
    P.out.store(cb, o);
    if (DOT) dot = re_dot(P.dotx.load_stream(cb), acc);
  }
  if (DOT) dot_block_partial(dot, dot_part, blockIdx.x);
  // peer-to-peer: the last block tells both senders their slot has been consumed
  if (P.pack_counter[mu]) grid_signal_last(P.ext_counter[mu], P.ack_to[mu][0], P.ack_to[mu][1], P.seq);
}

// ------------------------------------------------------------------ small-volume variant
// Below the bandwidth "shoulder" (not enough threads resident to hide the memory
// latency) one thread per output site leaves the SMs short of independent loads: at 16^3 x 32 the
// whole lattice is about one wave of the main kernel.  Here FOUR threads share a site, one per
// direction: warp w of a 128-thread block does the two hops of mu = w for 32 consecutive sites
// (warp-uniform mu, coalesced 32-site loads), the four partial spinors meet in shared memory, and
// thread (w, l) finishes components k = w, w + 4, w + 8 of site l (epilogue and store).  Whole
// lattice, EPI_PLAIN / EPI_XPAY, no fused dot.  Chosen by the tuner below when it is faster.
__device__ __forceinline__ cx<double> comp_load(const FermView<double> &v, int cb, int k) {
  const double2 t = ld_stream(v.p + (size_t)k * v.stride + cb);
  return {t.x, t.y};
}
__device__ __forceinline__ void comp_store(const FermView<double> &v, int cb, int k, cx<double> c) {
  st_stream(v.p + (size_t)k * v.stride + cb, make_double2(c.re, c.im));
}
__device__ __forceinline__ cx<float> comp_load(const FermView<float> &v, int cb, int k) {
  const float2 t = ld_stream((const float2 *)(v.p + (size_t)(k >> 1) * v.stride) + 2 * cb + (k & 1));
  return {t.x, t.y};
}
__device__ __forceinline__ void comp_store(const FermView<float> &v, int cb, int k, cx<float> c) {
  st_stream((float2 *)(v.p + (size_t)(k >> 1) * v.stride) + 2 * cb + (k & 1), make_float2(c.re, c.im));
}

template <typename R, int REC, int EPI, bool G5IN, bool G5OUT>
__global__ void __launch_bounds__(128) dslash4_kernel(const Geom g, const __grid_constant__ KParams<R, REC> P) {
  __shared__ cx<R> part[4][12][33];
  const int mu = threadIdx.x >> 5, l = threadIdx.x & 31;
  const int cb = blockIdx.x * 32 + l;
  const int p = P.parity;
  Spinor<R> acc;
#pragma unroll
  for (int k = 0; k < 12; k++) acc.c[k] = {R(0), R(0)};
  if (cb < g.Vh) {
    int c[4];
    cb_coords(g, cb, p, c);
    switch (mu) {  // warp-uniform
      case 0: hop_dir<R, 0>(g, P, c, cb, p, G5IN, false, acc); break;
      case 1: hop_dir<R, 1>(g, P, c, cb, p, G5IN, false, acc); break;
      case 2: hop_dir<R, 2>(g, P, c, cb, p, G5IN, false, acc); break;
      default: hop_dir<R, 3>(g, P, c, cb, p, G5IN, false, acc); break;
    }
  }
#pragma unroll
  for (int k = 0; k < 12; k++) part[mu][k][l] = acc.c[k];
  __syncthreads();
  if (cb >= g.Vh) return;
#pragma unroll
  for (int j = 0; j < 3; j++) {
    const int k = mu + 4 * j;
    cx<R> h = part[0][k][l] + part[1][k][l];
    h = h + part[2][k][l];
    h = h + part[3][k][l];
    if (G5OUT && k >= 6) h = -h;
    cx<R> o = P.b * h;
    if (EPI == EPI_XPAY) o = P.a * comp_load(P.x, cb, k) + o;
    comp_store(P.out, cb, k, o);
  }
}

// ------------------------------------------------------------------ bulk-copy staged variant
// Latency hiding for the fp64 kernels (the reconstruct-12 one is latency-bound: 12 warps per SM at
// 168 registers, long-scoreboard stalls).  The forward links U_mu(x) of a block's 64 output sites
// are 4 x (REC/2) contiguous 1 KB plane segments: one thread hands them to the bulk-copy (TMA)
// engine at block start (cp.async.bulk global -> shared, completion on an mbarrier), so those bytes
// are in flight without holding registers; the threads start with the mu = 0 backward hop on the
// register path, then wait and take the forward links from shared memory.  Accumulation order:
// bwd0 + fwd0 == fwd0 + bwd0 exactly (the first two terms commute), the rest as the main kernel,
// so the output is bit-identical to it.  Whole lattice, fp64 reconstruct-12, any epilogue, no fused
// dot.  Measured (profiles/r02_dslash_variants.txt, r02_ncu_detail_r12_tma.txt): within 1-2% of the
// register-path kernel (long-scoreboard stalls 6.7 -> 5.3 per issue, same time): the spinor and
// backward-link loads that stay on the register path keep it latency-bound; a candidate of the tuner.
__device__ __forceinline__ unsigned smem_u32(const void *p) { return (unsigned)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(unsigned long long *bar, unsigned n) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(n) : "memory");
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_expect_tx(unsigned long long *bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void bulk_g2s(void *dst, const void *src, unsigned bytes, unsigned long long *bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   smem_u32(dst)),
               "l"(src), "r"(bytes), "r"(smem_u32(bar))
               : "memory");
}
__device__ __forceinline__ bool mbar_try(unsigned long long *bar, unsigned phase) {
  unsigned ok;
  asm volatile(
      "{\n .reg .pred P1;\n mbarrier.try_wait.parity.shared::cta.b64 P1, [%1], %2;\n selp.u32 %0, 1, 0, P1;\n}"
      : "=r"(ok)
      : "r"(smem_u32(bar)), "r"(phase)
      : "memory");
  return ok != 0;
}

template <int MU, int REC>
__device__ __forceinline__ Link<double> smem_link(const double2 *sU) {
  constexpr int NPL = REC / 2;
  Link<double> u;
#pragma unroll
  for (int k = 0; k < NPL; k++) {
    const double2 v = sU[(MU * NPL + k) * 64 + threadIdx.x];
    u.m[k] = {v.x, v.y};
  }
  if (REC == 12) su3_third_row(u);
  return u;
}

template <int MU, int REC, typename KP>
__device__ __forceinline__ void hop_fwd_smem(const Geom &g, const KP &P, const int c[4], bool G5IN, const double2 *sU,
                                             Spinor<double> &acc) {
  int n[4] = {c[0], c[1], c[2], c[3]};
  n[MU] = (c[MU] + 1 == g.L[MU]) ? 0 : c[MU] + 1;
  Spinor<double> s = P.psi.load(coords_cb(g, n));
  if (G5IN) g5(s);
  accum_recon<MU, -1>(acc, mul_link(smem_link<MU, REC>(sU), project<MU, -1>(s)));
}
template <int MU, typename KP>
__device__ __forceinline__ void hop_bwd(const Geom &g, const KP &P, const int c[4], int p, bool G5IN,
                                        Spinor<double> &acc) {
  int n[4] = {c[0], c[1], c[2], c[3]};
  n[MU] = (c[MU] == 0) ? g.L[MU] - 1 : c[MU] - 1;
  const int ncb = coords_cb(g, n);
  Spinor<double> s = P.psi.load(ncb);
  if (G5IN) g5(s);
  accum_recon<MU, +1>(acc, mul_link_dag(P.U.load(MU, 1 - p, ncb), project<MU, +1>(s)));
}

template <typename R, int REC, int EPI, bool G5IN, bool G5OUT>
__global__ void __launch_bounds__(64, (dslash_minb<R, REC>()))
    dslash_tma_kernel(const Geom g, const __grid_constant__ KParams<R, REC> P) {
  if constexpr (sizeof(R) == 8) {
    constexpr int NPL = REC / 2;
    __shared__ __align__(128) double2 sU[4 * NPL * 64];
    __shared__ __align__(8) unsigned long long bar;
    const int cb0 = blockIdx.x * 64;
    const int cb = cb0 + threadIdx.x;
    const int p = P.parity;
    if (threadIdx.x == 0) {
      mbar_init(&bar, 1);
      mbar_expect_tx(&bar, 4 * NPL * 64 * 16);
#pragma unroll
      for (int mu = 0; mu < 4; mu++)
#pragma unroll
        for (int k = 0; k < NPL; k++)  // planes are padded to a multiple of 64 sites: always in bounds
          bulk_g2s(&sU[(mu * NPL + k) * 64], (const double2 *)P.U.p + ((size_t)(mu * 2 + p) * NPL + k) * g.stride + cb0,
                   64 * 16, &bar);
    }
    __syncthreads();
    Spinor<double> acc;
#pragma unroll
    for (int k = 0; k < 12; k++) acc.c[k] = {0.0, 0.0};
    int c[4] = {0, 0, 0, 0};
    if (cb < g.Vh) {
      cb_coords(g, cb, p, c);
      hop_bwd<0>(g, P, c, p, G5IN, acc);  // register path while the links land
    }
    while (!mbar_try(&bar, 0)) {
    }
    if (cb >= g.Vh) return;
    hop_fwd_smem<0, REC>(g, P, c, G5IN, sU, acc);
    hop_fwd_smem<1, REC>(g, P, c, G5IN, sU, acc);
    hop_bwd<1>(g, P, c, p, G5IN, acc);
    hop_fwd_smem<2, REC>(g, P, c, G5IN, sU, acc);
    hop_bwd<2>(g, P, c, p, G5IN, acc);
    hop_fwd_smem<3, REC>(g, P, c, G5IN, sU, acc);
    hop_bwd<3>(g, P, c, p, G5IN, acc);
    P.out.store(cb, epilogue<R, EPI>(P, cb, acc, G5OUT));
  }
}

// ------------------------------------------------------------------ asynchronously pipelined variant
// Latency hiding without registers (fp64): each thread stages the operands of its next hops -- the
// neighbour spinor (12 x 16 B) and the link (REC/2 x 16 B) -- into its own slots of a shared-memory
// ring of NST hop stages with cp.async (LDGSTS), so NST - 1 hops' loads are in flight while it
// computes the current hop from shared memory.  The bytes in flight are held by the async-copy
// unit, not by registers, so the register-path kernel's trade (more loads in flight = more registers
// = fewer warps) does not apply.  Each thread reads only the slots it filled (completion by
// cp.async.wait_group, no barrier).  Hop order and arithmetic are the main kernel's (fwd, bwd per
// mu = 0..3), so the output is bit-identical to it.  Whole lattice, any epilogue, no fused dot.
__device__ __forceinline__ void cp_async16(void *s, const void *gp) {  // L2 only (see the measured note above)
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(s)), "l"(gp) : "memory");
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N> __device__ __forceinline__ void cp_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }

template <int REC> struct PipeHop {
  static constexpr int NPL = REC / 2, NE = 12 + NPL;  // 16-byte slots per hop and thread
  // stage hop H (mu = H / 2, forward if H is even) into ring slot `st` (slot [k][thread])
  template <int H, typename KP>
  static __device__ __forceinline__ void issue(const Geom &g, const KP &P, const int c[4], int cb, int p, double2 *st) {
    constexpr int MU = H / 2;
    int n[4] = {c[0], c[1], c[2], c[3]};
    if (H % 2 == 0) n[MU] = (c[MU] + 1 == g.L[MU]) ? 0 : c[MU] + 1;
    else n[MU] = (c[MU] == 0) ? g.L[MU] - 1 : c[MU] - 1;
    const int ncb = coords_cb(g, n);
    const double2 *sp = P.psi.p + ncb;
#pragma unroll
    for (int k = 0; k < 12; k++) cp_async16(st + k * 64, sp + (size_t)k * g.stride);
    const double2 *lp = (const double2 *)P.U.p + (size_t)(MU * 2 + (H % 2 == 0 ? p : 1 - p)) * NPL * g.stride +
                        (H % 2 == 0 ? cb : ncb);
#pragma unroll
    for (int k = 0; k < NPL; k++) cp_async16(st + (12 + k) * 64, lp + (size_t)k * g.stride);
  }
  template <int H>
  static __device__ __forceinline__ void compute(const double2 *st, bool G5IN, Spinor<double> &acc) {
    constexpr int MU = H / 2;
    Spinor<double> s;
#pragma unroll
    for (int k = 0; k < 12; k++) {
      const double2 v = st[k * 64];
      s.c[k] = {v.x, v.y};
    }
    if (G5IN) g5(s);
    Link<double> u;
#pragma unroll
    for (int k = 0; k < NPL; k++) {
      const double2 v = st[(12 + k) * 64];
      u.m[k] = {v.x, v.y};
    }
    if (REC == 12) su3_third_row(u);
    if (H % 2 == 0) accum_recon<MU, -1>(acc, mul_link(u, project<MU, -1>(s)));
    else accum_recon<MU, +1>(acc, mul_link_dag(u, project<MU, +1>(s)));
  }
};

template <int REC, int EPI, bool G5IN, bool G5OUT, int NST>
__global__ void __launch_bounds__(64) dslash_pipe_kernel(const Geom g, const __grid_constant__ KParams<double, REC> P) {
  using PH = PipeHop<REC>;
  extern __shared__ __align__(16) double2 ring[];  // [NST][NE][64]
  const int cb = blockIdx.x * 64 + threadIdx.x;
  if (cb >= g.Vh) return;  // whole warps only on the last block: no barrier below
  const int p = P.parity;
  int c[4];
  cb_coords(g, cb, p, c);
  double2 *base = ring + threadIdx.x;
#define QDPB_ST(H) (base + ((H) % NST) * PH::NE * 64)
#define QDPB_ISSUE(H) \
  if constexpr ((H) < 8) PH::template issue<((H) < 8 ? (H) : 0)>(g, P, c, cb, p, QDPB_ST(H)); \
  cp_commit();
#define QDPB_HOP(H)                                  \
  QDPB_ISSUE((H) + NST - 1)                          \
  cp_wait<NST - 1>();                                \
  PH::template compute<H>(QDPB_ST(H), G5IN, acc);
  QDPB_ISSUE(0)  // prologue: hops 0 .. NST - 2
  if constexpr (NST > 2) { QDPB_ISSUE(1) }
  if constexpr (NST > 3) { QDPB_ISSUE(2) }
  Spinor<double> acc;
#pragma unroll
  for (int k = 0; k < 12; k++) acc.c[k] = {0.0, 0.0};
  QDPB_HOP(0) QDPB_HOP(1) QDPB_HOP(2) QDPB_HOP(3) QDPB_HOP(4) QDPB_HOP(5) QDPB_HOP(6) QDPB_HOP(7)
#undef QDPB_HOP
#undef QDPB_ISSUE
#undef QDPB_ST
  P.out.store(cb, epilogue<double, EPI>(P, cb, acc, G5OUT));
}

// ------------------------------------------------------------------ host side
template <typename R> static FermView<R> fview(const void *p, int stride);
template <> FermView<double> fview<double>(const void *p, int stride) { return {(double2 *)p, stride}; }
template <> FermView<float> fview<float>(const void *p, int stride) { return {(float4 *)p, stride}; }
template <typename R, int REC> static GaugeView<R, REC> gview(const void *p, int stride) {
  return {(decltype(GaugeView<R, REC>::p))p, stride};
}
template <typename R> static CloverView<R> cview(const void *p, int stride);
template <> CloverView<double> cview<double>(const void *p, int stride) { return {(const double2 *)p, stride}; }
template <> CloverView<float> cview<float>(const void *p, int stride) { return {(const float4 *)p, stride}; }
// 16-bit storage: [3 int4 planes][float norm plane] / [9 int4 planes][float norm plane]
template <> FermView<h16> fview<h16>(const void *p, int stride) {
  return {(int4 *)p, p ? (float *)((char *)p + (size_t)48 * stride) : nullptr, stride};
}
template <> CloverView<h16> cview<h16>(const void *p, int stride) {
  return {(const int4 *)p, p ? (const float *)((const char *)p + (size_t)144 * stride) : nullptr, stride};
}

template <typename R, int REC, int EPI, bool G5IN, bool G5OUT, bool HALO, bool DOT>
static void launch_main(qdp_ctx ctx, const KParams<R, REC> &P, int block) {
  const Geom &g = ctx->geom;
  // the fused boundary kernel keeps plain stream order: with PDL its leading (packing) blocks land
  // on whichever SMs the predecessor frees first, and config 5's z x t rank sub-lattice CG lost 1%
  // (profiles/r02_pdl.txt); QDPB_PDL_HALO=1 for measurements
  static const bool pdl_halo = getenv("QDPB_PDL_HALO") && atoi(getenv("QDPB_PDL_HALO"));
  launch_pdl(ctx->stream, ctx->pdl && (!HALO || pdl_halo), dslash_kernel<R, REC, EPI, G5IN, G5OUT, HALO, DOT>,
             grid_for(g.Vh, block) + P.fuse_npack, block, 0, g, P);
}

template <typename R, int REC, int EPI>
static void launch_four(qdp_ctx ctx, const KParams<R, REC> &P, bool g5i, bool g5o) {
  if constexpr ((EPI == EPI_PLAIN || EPI == EPI_XPAY) && !is_h16<R>()) {
    const int grid = grid_for(ctx->geom.Vh, 32);
#define QDPB_L4(A, B) dslash4_kernel<R, REC, EPI, A, B><<<grid, 128, 0, ctx->stream>>>(ctx->geom, P)
    if (g5i) { if (g5o) QDPB_L4(true, true); else QDPB_L4(true, false); }
    else { if (g5o) QDPB_L4(false, true); else QDPB_L4(false, false); }
#undef QDPB_L4
  }
}

template <typename R, int REC, int EPI>
static void launch_tma(qdp_ctx ctx, const KParams<R, REC> &P, bool g5i, bool g5o) {
  if constexpr (sizeof(R) == 8 && REC == 12) {  // (18 links: 36 KB of staging per block, 30-40% slower)
    const int grid = grid_for(ctx->geom.Vh, 64);
#define QDPB_LT(A, B) dslash_tma_kernel<R, REC, EPI, A, B><<<grid, 64, 0, ctx->stream>>>(ctx->geom, P)
    if (g5i) { if (g5o) QDPB_LT(true, true); else QDPB_LT(true, false); }
    else { if (g5o) QDPB_LT(false, true); else QDPB_LT(false, false); }
#undef QDPB_LT
  }
}

template <typename R, int REC, int EPI>
static void launch_o8(qdp_ctx ctx, const KParams<R, REC> &P, bool g5i, bool g5o) {
  if constexpr (dslash_minb<R, REC>() < 8) {
    const int grid = grid_for(ctx->geom.Vh, 64);
#define QDPB_LO(A, B) launch_k(ctx, dslash_o8_kernel<R, REC, EPI, A, B>, grid, 64, ctx->geom, P)
    if (g5i) { if (g5o) QDPB_LO(true, true); else QDPB_LO(true, false); }
    else { if (g5o) QDPB_LO(false, true); else QDPB_LO(false, false); }
#undef QDPB_LO
  }
}

template <typename R, int REC, int EPI, int NST>
static void launch_pipe(qdp_ctx ctx, const KParams<R, REC> &P, bool g5i, bool g5o) {
  if constexpr (sizeof(R) == 8 && !is_h16<R>()) {
    const int grid = grid_for(ctx->geom.Vh, 64);
    // two stages: 36 KB (12-real links) / 42 KB (18) of dynamic shared memory, within the default 48 KB
    constexpr size_t smem = (size_t)NST * PipeHop<REC>::NE * 64 * 16;
    static_assert(smem <= 48 * 1024, "the hop ring must fit the default dynamic shared-memory limit");
    // plain stream order, no griddepcontrol in the kernel: with PDL a sequence of pipeline launches alone
    // ran faster, but inside the Wilson CG (mixed with the main kernel and the BLAS kernels) the CG lost
    // 13-14% (profiles/r02_dslash_pipeline.txt section 7)
#define QDPB_LP(A, B) launch_pdl(ctx->stream, false, dslash_pipe_kernel<REC, EPI, A, B, NST>, grid, 64, smem, ctx->geom, P)
    if (g5i) { if (g5o) QDPB_LP(true, true); else QDPB_LP(true, false); }
    else { if (g5o) QDPB_LP(false, true); else QDPB_LP(false, false); }
#undef QDPB_LP
  }
}

template <typename R, int REC, int EPI>
static void launch_main_dispatch(qdp_ctx ctx, const KParams<R, REC> &P, bool g5i, bool g5o, bool halo, bool dot,
                                 int block) {
  if (dot) {  // fused inner product: only the Mhat^dag output step (g5_out, no g5_in) uses it
    if constexpr (EPI == EPI_XPAY || EPI == EPI_CLOVXPAY) {
      if (halo) launch_main<R, REC, EPI, false, true, true, true>(ctx, P, block);
      else launch_main<R, REC, EPI, false, true, false, true>(ctx, P, block);
    }
    return;
  }
#define QDPB_L(A, B, C) launch_main<R, REC, EPI, A, B, C, false>(ctx, P, block)
  if (halo) {
    if (g5i) { if (g5o) QDPB_L(true, true, true); else QDPB_L(true, false, true); }
    else { if (g5o) QDPB_L(false, true, true); else QDPB_L(false, false, true); }
  } else {
    if (g5i) { if (g5o) QDPB_L(true, true, false); else QDPB_L(true, false, false); }
    else { if (g5o) QDPB_L(false, true, false); else QDPB_L(false, false, false); }
  }
#undef QDPB_L
}

template <typename R, int REC, int EPI>
static void launch_ext(qdp_ctx ctx, const KParams<R, REC> &P, int mu, bool g5o, double *dot_part) {
  const Geom &g = ctx->geom;
  const int n = 2 * g.faceVh[mu];
  if (dot_part) exterior_kernel<R, REC, EPI, true, true><<<grid_for(n, 128), 128, 0, ctx->stream>>>(g, P, mu, dot_part);
  else if (g5o) exterior_kernel<R, REC, EPI, true, false><<<grid_for(n, 128), 128, 0, ctx->stream>>>(g, P, mu, nullptr);
  else exterior_kernel<R, REC, EPI, false, false><<<grid_for(n, 128), 128, 0, ctx->stream>>>(g, P, mu, nullptr);
}

// Algorithmic work of one EO dslash launch: 1320 flop per output
// site for the hopping term (8 x (12 projection + 132 SU(3) x half spinor) + 7 x 24
// accumulate) plus the epilogue; compulsory bytes 8 links + input + output (+ x, + clover,
// + the fused inner product's second vector).
// 16-bit storage: the bytes the kernel moves (a spinor 52 B, a link 24 B, a clover site 148 B).
template <typename R, int REC>
static void dslash_work(qdp_ctx ctx, const DslashArgs &a) {
  double f = 1320, r = 8 * REC + 24 + 24;
  const double sp = is_h16<R>() ? 52 : 24 * sizeof(R), cl = is_h16<R>() ? 148 : 72 * sizeof(R);
  double bytes = is_h16<R>() ? 8 * 24 + 2 * sp : r * sizeof(R);
  switch (a.epi) {
    case EPI_PLAIN: f += a.b != 1.0 ? 24 : 0; break;
    case EPI_XPAY: f += 72; bytes += sp; break;
    case EPI_CLOVINV: f += 504 + 24 + (a.x ? 48 : 0); bytes += cl + (a.x ? sp : 0); break;
    default: f += 504 + 48; bytes += cl + sp; break;
  }
  if (a.dot_x) { f += 96 + (a.dot_shift != 0.0 ? 48 : 0); bytes += sp; }
  const double vh = ctx->geom.Vh;
  prof_work(ctx, QDP_PK_DSLASH, f * vh, bytes * vh);
}

// The paper's autotuner (section VII) on the launch configuration of the
// whole-lattice EO dslash, on its payload launches: the candidates -- the four-threads-per-site
// kernel (128 threads), the main kernel with 64 threads, the cp.async hop pipeline (fp64), the main
// kernel with 32 threads, the bulk-copy staged links (fp64 r12) -- the first launch takes the first,
// later launches probe the next ones until one is 33% slower than the best, and the best is kept
// for the key (precision, gauge storage, epilogue, volume).
template <typename R, int REC>
static int launch_main_epi(qdp_ctx ctx, const DslashArgs &a, const KParams<R, REC> &P, bool halo, int block) {
  ProfEvent ev;
  prof_begin(ctx, QDP_PK_DSLASH, &ev);
  dslash_work<R, REC>(ctx, a);
  const bool dot = a.dot_x != nullptr;
  auto go = [&](int variant) -> cudaError_t {
    // variant: 0 = four threads per site (PLAIN / XPAY only), 1 = main kernel with `block`
    // threads, 2 = main kernel with 32 threads, 3 = bulk-copy staged forward links (fp64 r12),
    // 4 = cp.async hop pipeline (fp64), 5 = main kernel at 128 registers (8 blocks per SM)
    if (variant == 0) {
      if (a.epi == EPI_PLAIN) launch_four<R, REC, EPI_PLAIN>(ctx, P, a.g5_in, a.g5_out);
      else launch_four<R, REC, EPI_XPAY>(ctx, P, a.g5_in, a.g5_out);
      return cudaGetLastError();
    }
    if (variant == 3) {
      switch (a.epi) {
        case EPI_PLAIN: launch_tma<R, REC, EPI_PLAIN>(ctx, P, a.g5_in, a.g5_out); break;
        case EPI_XPAY: launch_tma<R, REC, EPI_XPAY>(ctx, P, a.g5_in, a.g5_out); break;
        case EPI_CLOVINV: launch_tma<R, REC, EPI_CLOVINV>(ctx, P, a.g5_in, a.g5_out); break;
        default: launch_tma<R, REC, EPI_CLOVXPAY>(ctx, P, a.g5_in, a.g5_out); break;
      }
      return cudaGetLastError();
    }
    if (variant == 5) {
      switch (a.epi) {
        case EPI_PLAIN: launch_o8<R, REC, EPI_PLAIN>(ctx, P, a.g5_in, a.g5_out); break;
        case EPI_XPAY: launch_o8<R, REC, EPI_XPAY>(ctx, P, a.g5_in, a.g5_out); break;
        case EPI_CLOVINV: launch_o8<R, REC, EPI_CLOVINV>(ctx, P, a.g5_in, a.g5_out); break;
        default: launch_o8<R, REC, EPI_CLOVXPAY>(ctx, P, a.g5_in, a.g5_out); break;
      }
      return cudaGetLastError();
    }
    if (variant == 4) {  // cp.async hop pipeline, two stages (fp64)
#define QDPB_PIPE(E) launch_pipe<R, REC, E, 2>(ctx, P, a.g5_in, a.g5_out)
      switch (a.epi) {
        case EPI_PLAIN: QDPB_PIPE(EPI_PLAIN); break;
        case EPI_XPAY: QDPB_PIPE(EPI_XPAY); break;
        case EPI_CLOVINV: QDPB_PIPE(EPI_CLOVINV); break;
        default: QDPB_PIPE(EPI_CLOVXPAY); break;
      }
#undef QDPB_PIPE
      return cudaGetLastError();
    }
    const int b = variant == 1 ? block : 32;
    switch (a.epi) {
      case EPI_PLAIN: launch_main_dispatch<R, REC, EPI_PLAIN>(ctx, P, a.g5_in, a.g5_out, halo, false, b); break;
      case EPI_XPAY: launch_main_dispatch<R, REC, EPI_XPAY>(ctx, P, a.g5_in, a.g5_out, halo, dot, b); break;
      case EPI_CLOVINV: launch_main_dispatch<R, REC, EPI_CLOVINV>(ctx, P, a.g5_in, a.g5_out, halo, false, b); break;
      default: launch_main_dispatch<R, REC, EPI_CLOVXPAY>(ctx, P, a.g5_in, a.g5_out, halo, dot, b); break;
    }
    return cudaGetLastError();
  };
  // the candidates of this call, in the tuner's order (decreasing threads per block, then the
  // staged variant): whole lattice, no fused reduction (its partials follow the block size)
  int vids[7], nv = 0;
  if (!is_h16<R>() && (a.epi == EPI_PLAIN || a.epi == EPI_XPAY)) vids[nv++] = 0;
  vids[nv++] = 1;
  // the hop pipeline right after the main kernel (probed before a slow candidate stops the search):
  // fp64 reconstruct-12, plain / xpay only.  With the clover epilogues it lost inside the CG; with 18-real
  // links it only matches the main kernel in isolation and inside the Wilson CG the main kernel, which
  // overlaps its neighbours under PDL, is 2-4% faster (profiles/r02_dslash_pipeline.txt sections 4, 7)
  if (sizeof(R) == 8 && !is_h16<R>() && REC == 12 && (a.epi == EPI_PLAIN || a.epi == EPI_XPAY)) vids[nv++] = 4;
  if (dslash_minb<R, REC>() < 8 && QDPB_TUNE_O8) vids[nv++] = 5;
  vids[nv++] = 2;
  if (sizeof(R) == 8 && REC == 12) vids[nv++] = 3;
  if (!halo && !dot && ctx->block == 0 && ctx->dslash_variant >= 0) {  // forced (measurements)
    int v = 1;
    for (int i = 0; i < nv; i++)
      if (vids[i] == ctx->dslash_variant) v = vids[i];
    if (sizeof(R) == 8 && !is_h16<R>() && ctx->dslash_variant == 4) v = 4;  // any epilogue (tests)
    if (dslash_minb<R, REC>() < 8 && ctx->dslash_variant == 5) v = 5;
    const cudaError_t e = go(v);
    const int rc = prof_end(ctx, &ev);
    return e != cudaSuccess ? cuda_check(ctx, e, "dslash launch") : rc;
  }
  if (!halo && !dot && ctx->autotune && ctx->block == 0) {
    const long key = ((((long)(is_h16<R>() ? 2 : sizeof(R) == 8) * 2 + (REC == 12)) * 4 + a.epi) << 40) + ctx->geom.Vh;
    int rc = tuned_variant(ctx, key, nv, [&](int i) { return go(vids[i]); });
    if (rc) {
      prof_end(ctx, &ev);
      return rc;
    }
    return prof_end(ctx, &ev);
  }
  const cudaError_t e = go(1);
  const int rc = prof_end(ctx, &ev);
  return e != cudaSuccess ? cuda_check(ctx, e, "dslash launch") : rc;
}

struct KParams_slab {
  const int *face_slab;
  int sz0, nzi, st0, nin;
};
// z or z x t partition (x, y unpartitioned): the face (z,t) slabs, in order, for the fused kernel;
// the interior slabs are enumerated by arithmetic.  Built once per (context, partition).
static int fuse_slabs(qdp_ctx ctx, KParams_slab *out) {
  const Geom &g = ctx->geom;
  const bool pz = (g.part >> 2) & 1, pt = (g.part >> 3) & 1;
  if (ctx->fuse_slab_part != g.part) {
    if (ctx->fuse_slabs) cudaFree(ctx->fuse_slabs);
    ctx->fuse_slabs = nullptr;
    std::vector<int> face;
    int nin = 0;
    for (int t = 0; t < g.L[3]; t++)
      for (int z = 0; z < g.L[2]; z++) {
        const bool onface = (pz && (z == 0 || z == g.L[2] - 1)) || (pt && (t == 0 || t == g.L[3] - 1));
        if (onface) face.push_back(z + g.L[2] * t);
        else nin++;
      }
    QDP_CUDA(ctx, cudaMalloc((void **)&ctx->fuse_slabs, sizeof(int) * std::max<size_t>(1, face.size())));
    QDP_CUDA(ctx, cudaMemcpyAsync(ctx->fuse_slabs, face.data(), sizeof(int) * face.size(), cudaMemcpyHostToDevice,
                                  ctx->stream));
    QDP_CUDA(ctx, cudaStreamSynchronize(ctx->stream));  // `face` is released on return
    ctx->fuse_slab_part = g.part;
    ctx->fuse_nslab_in = nin;
  }
  out->face_slab = ctx->fuse_slabs;
  out->sz0 = pz ? 1 : 0;
  out->nzi = pz ? g.L[2] - 2 : g.L[2];
  out->st0 = pt ? 1 : 0;
  out->nin = ctx->fuse_nslab_in * g.Lh0 * g.L[1];
  return QDP_OK;
}

// Visiting order of the fused boundary kernel for output parity p: sites on no partitioned face
// first (nin of them), then the others; built once per (context, partition, parity), on the host.
static int fuse_order(qdp_ctx ctx, int p, const int **perm, int *nin) {
  const Geom &g = ctx->geom;
  if (ctx->fuse_part != g.part) {
    for (int q = 0; q < 2; q++) {
      if (ctx->fuse_perm[q]) cudaFree(ctx->fuse_perm[q]);
      ctx->fuse_perm[q] = nullptr;
    }
    ctx->fuse_part = g.part;
  }
  for (int pp = 0; pp < 2; pp++) {  // both parities at once (before either kernel runs)
    if (ctx->fuse_perm[pp]) continue;
    std::vector<int> in, out;
    in.reserve(g.Vh);
    for (int cb = 0; cb < g.Vh; cb++) {
      int c[4];
      cb_coords(g, cb, pp, c);
      bool onface = false;
      for (int mu = 0; mu < 4; mu++)
        if (((g.part >> mu) & 1) && (c[mu] == 0 || c[mu] == g.L[mu] - 1)) onface = true;
      (onface ? out : in).push_back(cb);
    }
    ctx->fuse_nin[pp] = (int)in.size();
    in.insert(in.end(), out.begin(), out.end());
    QDP_CUDA(ctx, cudaMalloc((void **)&ctx->fuse_perm[pp], sizeof(int) * g.Vh));
    // on the context stream, ordered before the kernels that read it (a pageable cudaMemcpy may
    // return before its DMA lands, and the context stream need not synchronise with it)
    QDP_CUDA(ctx, cudaMemcpyAsync(ctx->fuse_perm[pp], in.data(), sizeof(int) * g.Vh, cudaMemcpyHostToDevice,
                                  ctx->stream));
    QDP_CUDA(ctx, cudaStreamSynchronize(ctx->stream));  // `in` is released on return
  }
  *perm = ctx->fuse_perm[p];
  *nin = ctx->fuse_nin[p];
  return QDP_OK;
}

template <typename R, int REC>
static int dslash_t(qdp_ctx ctx, const DslashArgs &a) {
  const bool slab_mode = (ctx->geom.part & 3) == 0 && ctx->geom.part != 8;  // z or z x t
  const Geom &g = ctx->geom;
  const int prec = sizeof(R) == 8 ? QDP_F64 : QDP_F32;  // halo buffers (16-bit storage: fp32 ghosts)
  using T = Arith_t<R>;
  constexpr double BPR = is_h16<R>() ? 2.0 : (double)sizeof(R);  // bytes per stored real (accounting)
  KParams<R, REC> P = {};
  P.out = fview<R>(a.out, g.stride);
  P.psi = fview<R>(a.psi, g.stride);
  P.x = fview<R>(a.x, g.stride);
  P.U = gview<R, REC>(a.U, g.stride);
  P.A = cview<R>(a.clov, g.stride);
  P.parity = a.parity;
  P.a = (T)a.a;
  P.b = (T)a.b;
  const int block = ctx->block > 0 ? ctx->block : QDPB_DSLASH_BLOCK;
  const bool halo = g.part != 0;
  const bool dot = a.dot_x != nullptr;
  int rc;
  if (dot && !(a.epi == EPI_XPAY || a.epi == EPI_CLOVXPAY) ) return set_error(ctx, QDP_EINVAL, "fused dot: XPAY epilogues only");
  if (dot && (a.g5_in || !a.g5_out)) return set_error(ctx, QDP_EINVAL, "fused dot: Mhat^dag output step only");
  // peer-to-peer: packing, interior and remote hops in the one main kernel (KParams::fuse), for
  // every split (t: the face sites are the two end slabs of the cb order, found by arithmetic;
  // others: a site table, interior sites first).  Otherwise separate pack / interior /
  // exterior kernels (QDP_OPT_FUSE = 0, kept for comparison).
  const bool fuse = halo && ctx->p2p_on && ctx->fuse;
  // partial-sum layout of the fused inner product: interior blocks, then each exterior's blocks
  int nparts = 0, ext_off[4] = {0, 0, 0, 0};
  int pack_off[5] = {0, 0, 0, 0, 0};
  for (int mu = 0; mu < 4; mu++) pack_off[mu + 1] = pack_off[mu] + (((g.part >> mu) & 1) ? 2 * g.faceVh[mu] : 0);
  // pack blocks: few enough that their per-block system fences stay cheap (grid-stride loop)
  static const int pack_cap =
      std::max(1, getenv("QDPB_PACK_BLOCKS") ? atoi(getenv("QDPB_PACK_BLOCKS")) : 2 * 148);  // measured: 260.0 -> 257.7 us
  const int npack = fuse ? std::min(grid_for(pack_off[4], block), pack_cap) : 0;
  // fused inner product: finished inside the main kernel when every partial is produced there
  // (whole lattice, or the fused boundary); else block partials + a final pass
  const bool red_fin = dot && (!halo || fuse);
  if (dot) {
    nparts = grid_for(g.Vh, block) + npack;
    for (int mu = 0; mu < 4; mu++)
      if (((g.part >> mu) & 1) && !fuse) {
        ext_off[mu] = nparts;
        nparts += grid_for(2 * g.faceVh[mu], 128);
      }
    if ((rc = ensure_reduce(ctx, nparts))) return rc;
    P.dotx = fview<R>(a.dot_x, g.stride);
    P.dot_part = ctx->red_partials;
    P.dot_shift = (T)a.dot_shift;
  }

  unsigned seq = 0;
  if (halo && ctx->p2p_on) {
    // host-side preparation that can fail comes first; the sequence number is taken last, by
    // p2p_prepare, so a failure never leaves this rank a call behind its neighbours
    KParams_slab sl = {};
    if (fuse && slab_mode && (rc = fuse_slabs(ctx, &sl))) return rc;
    if (fuse && g.part != 8 && !slab_mode && (rc = fuse_order(ctx, a.parity, &P.perm, &P.fuse_nin))) return rc;
    if (fuse && slab_mode) {
      P.face_slab = sl.face_slab;
      P.sz0 = sl.sz0;
      P.nzi = sl.nzi;
      P.st0 = sl.st0;
      P.fuse_nin = sl.nin;
    }
    // peer-to-peer: pack straight into the neighbours' ghost slots, flags instead of NCCL (p2p.cu)
    P2PLaunch L;
    if ((rc = p2p_prepare(ctx, prec, &L))) return rc;
    seq = L.seq;
    for (int mu = 0; mu < 4; mu++) {
      P.pack_counter[mu] = L.pack_counter[mu];
      P.ext_counter[mu] = L.ext_counter[mu];
      for (int d = 0; d < 2; d++) {
        P.dst[mu][d] = L.dst[mu][d];
        P.ghost[mu][d] = L.ghost[mu][d];
        P.sig[mu][d] = L.sig[mu][d];
        P.ack_to[mu][d] = L.ack_to[mu][d];
        P.war[mu][d] = L.war[mu][d];
        P.ready[mu][d] = L.ready[mu][d];
      }
    }
    P.err = L.err;
    P.seq = seq;
    if (fuse) {
      if (g.part == 8) {  // t slabs are contiguous in cb: the order is arithmetic
        P.perm = nullptr;
        P.fuse_nin = g.Vh - 2 * g.faceVh[3];
      }
      P.fuse = 1;
      // the face sites halfway through the interior rather than last: they no longer form the
      // kernel's tail (measured, profiles/r02_fused_face_position.txt: 40^3 x 32 t 260 -> 255 us,
      // z x t 270 -> 264 us; 48 x 48 x 24 x 24 z x t 183 -> 177 us), and half the interior still
      // runs before any block waits for a ghost.  QDPB_FACE_AT (fraction of the interior visited
      // first, >= 1: faces last) for measurements.
      static const double face_at = getenv("QDPB_FACE_AT") ? atof(getenv("QDPB_FACE_AT")) : 0.5;
      P.fuse_kin = face_at >= 1.0 ? P.fuse_nin
                                  : std::max(0, (int)(face_at * P.fuse_nin) / block * block);
      P.fuse_npack = npack;
      for (int k = 0; k < 5; k++) P.pack_off[k] = pack_off[k];
      P.pack_q = L.pack_q;
      P.pack_chunks = grid_for(pack_off[4], block);
      P.wait_all = ctx->overlap ? 0 : 1;
    } else {
      // separate kernels: the fused kernel's work-queue sets are not advanced by this call, so a
      // later fused call must not find the counts a fused call left two sequence numbers ago
      QDP_CUDA(ctx, cudaMemsetAsync(L.pack_q, 0, 4 * sizeof(unsigned), ctx->stream));
    }
  }
  if (halo) {
    bool any_comm = false;
    size_t face_bytes[4] = {0, 0, 0, 0};
    if (!seq) {
      if ((rc = ensure_halo(ctx, prec))) return rc;
      // destinations: self-halo dims pack straight into our own ghost buffers (the peer is
      // this rank); communicated dims pack into send buffers for NCCL.
      for (int mu = 0; mu < 4; mu++) {
        if (!((g.part >> mu) & 1)) continue;
        const bool self = direct_self(ctx, mu);
        any_comm |= !self;
        face_bytes[mu] = (size_t)g.faceVh[mu] * 12 * sizeof(T);
        P.dst[mu][0] = self ? ctx->halo_recv[prec][mu][1] : ctx->halo_send[prec][mu][0];
        P.dst[mu][1] = self ? ctx->halo_recv[prec][mu][0] : ctx->halo_send[prec][mu][1];
        P.ghost[mu][0] = ctx->halo_recv[prec][mu][0];
        P.ghost[mu][1] = ctx->halo_recv[prec][mu][1];
      }
    }
    for (int mu = 0; mu < 4; mu++) {
      if (!((g.part >> mu) & 1)) continue;
      if (fuse) {  // packed by the leading blocks of the main kernel: bytes only, no launch
        prof_work(ctx, QDP_PK_DSLASH, 0.0, (double)g.faceVh[mu] * (24 + 12 + 24 + REC + 12) * BPR);
        continue;
      }
      ProfEvent ev;
      prof_begin(ctx, QDP_PK_PACK, &ev);
      // compulsory: psi read on both faces, the forward face's link, the half spinors written
      prof_work(ctx, QDP_PK_PACK, 0.0, (double)g.faceVh[mu] * (24 + 12 + 24 + REC + 12) * BPR);
      const int n = 2 * g.faceVh[mu];
      if (a.g5_in) pack_kernel<R, REC, true><<<grid_for(n, 128), 128, 0, ctx->stream>>>(g, P, mu);
      else pack_kernel<R, REC, false><<<grid_for(n, 128), 128, 0, ctx->stream>>>(g, P, mu);
      if ((rc = prof_end(ctx, &ev))) return rc;
    }
    const bool overlap = ctx->overlap && any_comm;
    if (any_comm) {
      if (overlap) {
        QDP_CUDA(ctx, cudaEventRecord(ctx->ev_packed, ctx->stream));
        QDP_CUDA(ctx, cudaStreamWaitEvent(ctx->comm_stream, ctx->ev_packed, 0));
        if ((rc = comm_exchange(ctx, prec, face_bytes, ctx->comm_stream))) return rc;
        QDP_CUDA(ctx, cudaEventRecord(ctx->ev_comm, ctx->comm_stream));
      } else {
        if ((rc = comm_exchange(ctx, prec, face_bytes, ctx->stream))) return rc;
      }
    }
    bool red_after = false;
    if (red_fin) {  // takes the peer sum's sequence number: right before the launch
      if ((rc = red_setup(ctx, grid_for(g.Vh, block) + npack, a.dot_slot, 2, true, false, &P.red, &red_after))) return rc;
      P.red_fin = 1;
    }
    if ((rc = launch_main_epi<R, REC>(ctx, a, P, true, block))) return rc;
    if (red_fin) return red_after ? reduce_global(ctx, a.dot_slot, 2) : QDP_OK;
    if (overlap) QDP_CUDA(ctx, cudaStreamWaitEvent(ctx->stream, ctx->ev_comm, 0));
    for (int mu = 0; mu < 4; mu++) {
      if (!((g.part >> mu) & 1) || fuse) continue;
      ProfEvent ev;
      prof_begin(ctx, QDP_PK_DSLASH_EXT, &ev);
      // ghost read, forward-face link, output read-modify-write (+ clover on CLOVINV)
      prof_work(ctx, QDP_PK_DSLASH_EXT, 0.0,
                (double)g.faceVh[mu] * (2 * 12 + REC + 2 * 48 + (a.epi == EPI_CLOVINV ? 2 * 72 : 0) + (dot ? 48 : 0)) *
                    BPR);
      double *dp = dot ? ctx->red_partials + 2 * ext_off[mu] : nullptr;
      if (a.epi == EPI_CLOVINV) launch_ext<R, REC, EPI_CLOVINV>(ctx, P, mu, a.g5_out, nullptr);
      else launch_ext<R, REC, EPI_PLAIN>(ctx, P, mu, a.g5_out, dp);
      if ((rc = prof_end(ctx, &ev))) return rc;
    }
  } else {
    bool red_after = false;
    if (red_fin) {
      if ((rc = red_setup(ctx, grid_for(g.Vh, block), a.dot_slot, 2, true, false, &P.red, &red_after))) return rc;
      P.red_fin = 1;
    }
    if ((rc = launch_main_epi<R, REC>(ctx, a, P, false, block))) return rc;
    if (red_fin) return red_after ? reduce_global(ctx, a.dot_slot, 2) : QDP_OK;
  }
  if (dot) {
    if ((rc = reduce_partials(ctx, nparts, a.dot_slot))) return rc;
    return reduce_global(ctx, a.dot_slot, 2);
  }
  return QDP_OK;
}

}  // namespace qdpb
