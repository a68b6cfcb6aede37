// internal.h -- shared declarations of the qdpb CUDA library (not part of the ABI).
//
// Device layout: structure-of-arrays with the
// checkerboard site index fastest, the coalescing condition of PAPER.md:156-160
// (section III-B, layout function I(i_V, i_S, i_C, i_R)), but with re/im interleaved so
// that one 16-byte load moves one complex double (or two complex floats):
//   fermion F64 : double2 plane[parity][12 = 3*spin+colour][stride]
//   fermion F32 : float4  plane[parity][6 = pairs of (spin,colour)][stride]
//   gauge   F64 : double2 plane[mu][parity][9 = 3*row+col][stride]
//   gauge   F32 : per (mu,parity): float4 plane[4][stride] (elements 0..7) + float2 plane[stride] (element 8)
//   clover  F64 : double2 plane[parity][36][stride]   (per chiral block b: 3 diag pairs + 15 off-diag)
//   clover  F32 : float4  plane[parity][18][stride]
// stride = Vh rounded up to a multiple of 64 sites (1 KB-aligned planes).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>
#include <functional>
#include <map>
#include <string>
#include <type_traits>
#include <vector>

#include "../../include/qdpb.h"

// Occupancy target of the main dslash kernel: __launch_bounds__(QDPB_DSLASH_MAXT, QDPB_DSLASH_MINB)
// caps it at 168 registers (6 x 64 threads per SM), measured best on B200.
#ifndef QDPB_DSLASH_MAXT
#define QDPB_DSLASH_MAXT 64
#endif
#ifndef QDPB_DSLASH_MINB
#define QDPB_DSLASH_MINB 6
#endif
// per (precision, gauge storage) overrides of the minimum resident blocks
#ifndef QDPB_MINB_D18
#define QDPB_MINB_D18 QDPB_DSLASH_MINB
#endif
#ifndef QDPB_MINB_D12
#define QDPB_MINB_D12 QDPB_DSLASH_MINB
#endif
#ifndef QDPB_MINB_F18
#define QDPB_MINB_F18 QDPB_DSLASH_MINB
#endif
#ifndef QDPB_MINB_F12
#define QDPB_MINB_F12 8  // fp32 + reconstruct-12: 128 registers, measured 110 -> 101 us at 40^3x32
#endif
template <typename R, int REC> constexpr int dslash_minb() {
  return sizeof(R) == 8 ? (REC == 18 ? QDPB_MINB_D18 : QDPB_MINB_D12)
         : sizeof(R) == 4 ? (REC == 18 ? QDPB_MINB_F18 : QDPB_MINB_F12)
                          : 8;  // 16-bit storage (sizeof(h16) == 1): fp32 arithmetic, 128 registers
}
#ifndef QDPB_MAX_SHIFTS
#define QDPB_MAX_SHIFTS 32  // qdp_cg_solve_multishift
#endif
// fp32 reconstruct-12 dslash: per-thread L2 prefetch of the site's 8 links at kernel entry
// (measured 100.7 -> 97.0 us at 40^3x32; the same prefetch slows every fp64 variant, and
// block-wide bulk prefetch or cp.async staging of the links did not pay either: DESIGN.md §6)
#ifndef QDPB_PF_F12
#define QDPB_PF_F12 1
#endif
#ifndef QDPB_DSLASH_BLOCK
#define QDPB_DSLASH_BLOCK 64
#endif
#define PEER_MAX_RANKS 16

namespace qdpb {

// ------------------------------------------------------------------ geometry
struct Geom {
  int L[4];        // local extents (all even)
  int Lh0;         // L[0] / 2
  int Vh;          // local sites per parity
  int stride;      // plane stride (sites)
  int part;        // bitmask: dims whose neighbours are reached through the halo path
  int faceVh[4];   // sites per parity on a face orthogonal to mu: V / L[mu] / 2
};

// site coordinates of checkerboard index cb on parity p
__host__ __device__ inline void cb_coords(const Geom &g, int cb, int p, int c[4]) {
  int xh = cb % g.Lh0;
  int r = cb / g.Lh0;
  c[1] = r % g.L[1];
  int r2 = r / g.L[1];
  c[2] = r2 % g.L[2];
  c[3] = r2 / g.L[2];
  c[0] = 2 * xh + ((p + c[1] + c[2] + c[3]) & 1);
}
__host__ __device__ inline int coords_cb(const Geom &g, const int c[4]) {
  return (c[0] >> 1) + g.Lh0 * (c[1] + g.L[1] * (c[2] + g.L[2] * c[3]));
}
__host__ __device__ inline int coords_parity(const int c[4]) { return (c[0] + c[1] + c[2] + c[3]) & 1; }

// Face index of a site on the face orthogonal to mu: lexicographic index of the three
// other coordinates (in x,y,z,t order), halved.  Bijective per parity because the first
// remaining extent is even; sender and receiver compute the same index.
__host__ __device__ inline int face_index(const Geom &g, int mu, const int c[4]) {
  int lex = 0, mul = 1;
#pragma unroll
  for (int d = 0; d < 4; d++) {
    if (d == mu) continue;
    lex += c[d] * mul;
    mul *= g.L[d];
  }
  return lex >> 1;
}
// inverse: coordinates of face site f on the face x_mu = xmu with site parity p.  Written without a
// run-time index into c[] (mu may be a run-time value: such an index would put c[] in local memory)
__host__ __device__ inline void face_coords(const Geom &g, int mu, int xmu, int f, int p, int c[4]) {
  // the first two of the other three dims: d0 = (mu == 0 ? 1 : 0), d1 = (mu <= 1 ? 2 : 1)
  const int A = mu == 0 ? g.L[1] : g.L[0], B = mu <= 1 ? g.L[2] : g.L[1];
  const int ah = f % (A >> 1), rest = f / (A >> 1), b = rest % B, cc = rest / B;
  const int x0 = 2 * ah + ((p + xmu + b + cc) & 1);
#pragma unroll
  for (int d = 0; d < 4; d++) {
    const int k = d - (d > mu ? 1 : 0);  // position among the other dims
    c[d] = d == mu ? xmu : (k == 0 ? x0 : (k == 1 ? b : cc));
  }
}
// a[mu] for a run-time mu without a run-time index (keeps a local c[] in registers, and a by-value
// kernel parameter such as Geom out of local memory)
__host__ __device__ inline int sel4(const int a[4], int mu) {
  return mu == 0 ? a[0] : mu == 1 ? a[1] : mu == 2 ? a[2] : a[3];
}

#ifdef __CUDACC__
// ------------------------------------------------------------------ complex helpers
template <typename R> struct cx { R re, im; };
template <typename R> __device__ __forceinline__ cx<R> mk(R a, R b) { return {a, b}; }
template <typename R> __device__ __forceinline__ cx<R> operator+(cx<R> a, cx<R> b) { return {a.re + b.re, a.im + b.im}; }
template <typename R> __device__ __forceinline__ cx<R> operator-(cx<R> a, cx<R> b) { return {a.re - b.re, a.im - b.im}; }
template <typename R> __device__ __forceinline__ cx<R> operator*(R s, cx<R> a) { return {s * a.re, s * a.im}; }
template <typename R> __device__ __forceinline__ cx<R> operator-(cx<R> a) { return {-a.re, -a.im}; }
template <typename R> __device__ __forceinline__ cx<R> cmul(cx<R> a, cx<R> b) {
  return {a.re * b.re - a.im * b.im, a.re * b.im + a.im * b.re};
}
// conj(a) * b
template <typename R> __device__ __forceinline__ cx<R> cjmul(cx<R> a, cx<R> b) {
  return {a.re * b.re + a.im * b.im, a.re * b.im - a.im * b.re};
}
template <typename R> __device__ __forceinline__ cx<R> cmadd(cx<R> a, cx<R> b, cx<R> acc) {  // acc + a*b
  acc.re = fma(a.re, b.re, acc.re);
  acc.re = fma(-a.im, b.im, acc.re);
  acc.im = fma(a.re, b.im, acc.im);
  acc.im = fma(a.im, b.re, acc.im);
  return acc;
}
template <typename R> __device__ __forceinline__ cx<R> cjmadd(cx<R> a, cx<R> b, cx<R> acc) {  // acc + conj(a)*b
  acc.re = fma(a.re, b.re, acc.re);
  acc.re = fma(a.im, b.im, acc.re);
  acc.im = fma(a.re, b.im, acc.im);
  acc.im = fma(-a.im, b.re, acc.im);
  return acc;
}
template <typename R> __device__ __forceinline__ cx<R> times_i(cx<R> a) { return {-a.im, a.re}; }
template <typename R> __device__ __forceinline__ cx<R> times_mi(cx<R> a) { return {a.im, -a.re}; }

// ------------------------------------------------------------------ memory access
// Streaming (read-once) loads: read-only path, no L1 allocation.
__device__ __forceinline__ double2 ld_stream(const double2 *p) {
  double2 r;
  asm("ld.global.nc.L1::no_allocate.v2.f64 {%0,%1}, [%2];" : "=d"(r.x), "=d"(r.y) : "l"(p));
  return r;
}
__device__ __forceinline__ float4 ld_stream(const float4 *p) {
  float4 r;
  asm("ld.global.nc.L1::no_allocate.v4.f32 {%0,%1,%2,%3}, [%4];"
               : "=f"(r.x), "=f"(r.y), "=f"(r.z), "=f"(r.w) : "l"(p));
  return r;
}
__device__ __forceinline__ float2 ld_stream(const float2 *p) {
  float2 r;
  asm("ld.global.nc.L1::no_allocate.v2.f32 {%0,%1}, [%2];" : "=f"(r.x), "=f"(r.y) : "l"(p));
  return r;
}
__device__ __forceinline__ int4 ld_stream(const int4 *p) {
  int4 r;
  asm("ld.global.nc.L1::no_allocate.v4.s32 {%0,%1,%2,%3}, [%4];" : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w) : "l"(p));
  return r;
}
__device__ __forceinline__ int2 ld_stream(const int2 *p) {
  int2 r;
  asm("ld.global.nc.L1::no_allocate.v2.s32 {%0,%1}, [%2];" : "=r"(r.x), "=r"(r.y) : "l"(p));
  return r;
}
__device__ __forceinline__ float ld_stream(const float *p) {
  float r;
  asm("ld.global.nc.L1::no_allocate.f32 %0, [%1];" : "=f"(r) : "l"(p));
  return r;
}
// L2 prefetch of one element (no register, no dependency).
__device__ __forceinline__ void prefetch_l2(const void *p) { asm volatile("prefetch.global.L2 [%0];" ::"l"(p)); }
// Re-used loads (neighbour spinors: 8 readers per site) go through the normal path.
__device__ __forceinline__ double2 ld_reuse(const double2 *p) { return __ldg(p); }
__device__ __forceinline__ float4 ld_reuse(const float4 *p) { return __ldg(p); }
// Streaming stores.
__device__ __forceinline__ void st_stream(double2 *p, double2 v) { __stcs(p, v); }
__device__ __forceinline__ void st_stream(float4 *p, float4 v) { __stcs(p, v); }
__device__ __forceinline__ void st_stream(float2 *p, float2 v) { __stcs(p, v); }

// System-scope release / acquire on 32-bit flags (peer-to-peer halo signalling, p2p.cu).
__device__ __forceinline__ void st_release_sys(unsigned *p, unsigned v) {
  asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ unsigned ld_acquire_sys(const unsigned *p) {
  unsigned v;
  asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

// Block-wide wait until both flags reach `expect` (wrap-safe); thread 0 polls with a bounded
// budget (~10 s) and raises *err instead of hanging.  All threads of the block must call it.
__device__ __forceinline__ void block_wait_flags(const unsigned *f0, const unsigned *f1, unsigned expect, unsigned *err) {
  if (threadIdx.x == 0) {
    long n = 0;
    while ((int)(ld_acquire_sys(f0) - expect) < 0 || (int)(ld_acquire_sys(f1) - expect) < 0) {
      if (++n > (1L << 26)) {
        atomicExch(err, 1u);
        break;
      }
      __nanosleep(128);
    }
  }
  __syncthreads();
  // every thread acquires the flags itself (they only grow, so it reads a value >= expect):
  // its later ghost loads are then ordered after the sender's release without relying on the
  // barrier carrying thread 0's acquire to the rest of the block
  if (threadIdx.x) {
    (void)ld_acquire_sys(f0);
    (void)ld_acquire_sys(f1);
  }
}
// Called by every thread after its stores: the last block of the grid to get here release-
// stores v into f0 and f1 (system scope) and resets the block counter.  The barrier orders the
// block's stores before thread 0's system-scope fence (fences are cumulative), and the fence /
// counter-RMW chain orders every block's stores before the last block's release.
__device__ __forceinline__ void grid_signal_last(unsigned *counter, unsigned *f0, unsigned *f1, unsigned v) {
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence_system();
    const unsigned prev = atomicAdd(counter, 1u);
    if (prev == gridDim.x - 1) {
      *counter = 0u;
      __threadfence_system();
      st_release_sys(f0, v);
      st_release_sys(f1, v);
    }
  }
}

}  // namespace qdpb
#include "reduce.cuh"
namespace qdpb {

// Spinor: 12 complex, index 3*spin + colour.
template <typename R> struct Spinor { cx<R> c[12]; };
// Half spinor: 6 complex, index 3*h + colour (h = 0,1).
template <typename R> struct Half { cx<R> c[6]; };
template <typename R> struct Link { cx<R> m[9]; };  // row-major

template <typename R> struct FermView;
template <> struct FermView<double> {
  double2 *p;  // parity block base
  int stride;
  __device__ __forceinline__ Spinor<double> load(int cb) const {
    Spinor<double> s;
#pragma unroll
    for (int k = 0; k < 12; k++) {
      double2 v = ld_reuse(p + (size_t)k * stride + cb);
      s.c[k] = {v.x, v.y};
    }
    return s;
  }
  __device__ __forceinline__ Spinor<double> load_stream(int cb) const {
    Spinor<double> s;
#pragma unroll
    for (int k = 0; k < 12; k++) {
      double2 v = ld_stream(p + (size_t)k * stride + cb);
      s.c[k] = {v.x, v.y};
    }
    return s;
  }
  __device__ __forceinline__ Spinor<double> load_plain(int cb) const {
    Spinor<double> s;
#pragma unroll
    for (int k = 0; k < 12; k++) {
      double2 v = p[(size_t)k * stride + cb];
      s.c[k] = {v.x, v.y};
    }
    return s;
  }
  __device__ __forceinline__ void store(int cb, const Spinor<double> &s) const {
#pragma unroll
    for (int k = 0; k < 12; k++) st_stream(p + (size_t)k * stride + cb, make_double2(s.c[k].re, s.c[k].im));
  }
};
template <> struct FermView<float> {
  float4 *p;
  int stride;
  __device__ __forceinline__ Spinor<float> load(int cb) const {
    Spinor<float> s;
#pragma unroll
    for (int k = 0; k < 6; k++) {
      float4 v = ld_reuse(p + (size_t)k * stride + cb);
      s.c[2 * k] = {v.x, v.y};
      s.c[2 * k + 1] = {v.z, v.w};
    }
    return s;
  }
  __device__ __forceinline__ Spinor<float> load_stream(int cb) const {
    Spinor<float> s;
#pragma unroll
    for (int k = 0; k < 6; k++) {
      float4 v = ld_stream(p + (size_t)k * stride + cb);
      s.c[2 * k] = {v.x, v.y};
      s.c[2 * k + 1] = {v.z, v.w};
    }
    return s;
  }
  __device__ __forceinline__ Spinor<float> load_plain(int cb) const {
    Spinor<float> s;
#pragma unroll
    for (int k = 0; k < 6; k++) {
      float4 v = p[(size_t)k * stride + cb];
      s.c[2 * k] = {v.x, v.y};
      s.c[2 * k + 1] = {v.z, v.w};
    }
    return s;
  }
  __device__ __forceinline__ void store(int cb, const Spinor<float> &s) const {
#pragma unroll
    for (int k = 0; k < 6; k++)
      st_stream(p + (size_t)k * stride + cb, make_float4(s.c[2 * k].re, s.c[2 * k].im, s.c[2 * k + 1].re, s.c[2 * k + 1].im));
  }
};

// Gauge field: base of the whole field; link (mu, parity, cb).
// Gauge field views.  REC = 18: full 3x3 links.  REC = 12 (QDP_GAUGE12): the first two rows
// are stored and the third is rebuilt as conj(row0 x row1), exact for SU(3) links
// (the "reconstruction from 12 real numbers" of PAPER.md:292).
template <typename R> __device__ __forceinline__ void su3_third_row(Link<R> &u) {
#pragma unroll
  for (int a = 0; a < 3; a++) {
    const int b = (a + 1) % 3, c = (a + 2) % 3;
    const cx<R> t = cmul(u.m[b], u.m[3 + c]) - cmul(u.m[c], u.m[3 + b]);
    u.m[6 + a] = {t.re, -t.im};
  }
}
template <typename R, int REC = 18> struct GaugeView;
template <> struct GaugeView<double, 18> {
  const double2 *p;
  int stride;
  __device__ __forceinline__ const double2 *block(int mu, int par) const { return p + (size_t)(mu * 2 + par) * 9 * stride; }
  __device__ __forceinline__ Link<double> load(int mu, int par, int cb) const {
    const double2 *b = block(mu, par);
    Link<double> u;
#pragma unroll
    for (int k = 0; k < 9; k++) {
      double2 v = ld_stream(b + (size_t)k * stride + cb);
      u.m[k] = {v.x, v.y};
    }
    return u;
  }
};
template <> struct GaugeView<double, 12> {
  const double2 *p;  // double2 [mu][parity][6][stride]
  int stride;
  __device__ __forceinline__ Link<double> load(int mu, int par, int cb) const {
    const double2 *b = p + (size_t)(mu * 2 + par) * 6 * stride;
    Link<double> u;
#pragma unroll
    for (int k = 0; k < 6; k++) {
      double2 v = ld_stream(b + (size_t)k * stride + cb);
      u.m[k] = {v.x, v.y};
    }
    su3_third_row(u);
    return u;
  }
};
template <> struct GaugeView<float, 12> {
  const float4 *p;  // float4 [mu][parity][3][stride]
  int stride;
  __device__ __forceinline__ void prefetch(int mu, int par, int cb) const {
    const float4 *b = p + (size_t)(mu * 2 + par) * 3 * stride + cb;
#pragma unroll
    for (int k = 0; k < 3; k++) prefetch_l2(b + (size_t)k * stride);
  }
  __device__ __forceinline__ Link<float> load(int mu, int par, int cb) const {
    const float4 *b = p + (size_t)(mu * 2 + par) * 3 * stride;
    Link<float> u;
#pragma unroll
    for (int k = 0; k < 3; k++) {
      float4 v = ld_stream(b + (size_t)k * stride + cb);
      u.m[2 * k] = {v.x, v.y};
      u.m[2 * k + 1] = {v.z, v.w};
    }
    su3_third_row(u);
    return u;
  }
};
template <> struct GaugeView<float, 18> {
  const float *p;  // byte layout: per (mu,par) block of stride*(4*16+8) bytes
  int stride;
  __device__ __forceinline__ Link<float> load(int mu, int par, int cb) const {
    const char *b = (const char *)p + (size_t)(mu * 2 + par) * stride * 72;
    const float4 *q = (const float4 *)b;
    const float2 *q2 = (const float2 *)(b + (size_t)stride * 64);
    Link<float> u;
#pragma unroll
    for (int k = 0; k < 4; k++) {
      float4 v = ld_stream(q + (size_t)k * stride + cb);
      u.m[2 * k] = {v.x, v.y};
      u.m[2 * k + 1] = {v.z, v.w};
    }
    float2 v = ld_stream(q2 + cb);
    u.m[8] = {v.x, v.y};
    return u;
  }
};

// Packed Hermitian clover block pair: per chiral block b: d[6] real + off[15] complex
// (strictly lower triangle, row-major: (i,j), i>j -> i(i-1)/2 + j).  36 "complex slots"
// per site: block b occupies slots 18b .. 18b+17 = (d0,d1),(d2,d3),(d4,d5),off[0..14].
template <typename R> struct CloverBlock { R d[6]; cx<R> off[15]; };
template <typename R> struct CloverView;
template <> struct CloverView<double> {
  const double2 *p;  // parity block base
  int stride;
  __device__ __forceinline__ CloverBlock<double> load(int b, int cb) const {
    CloverBlock<double> B;
    const double2 *q = p + (size_t)18 * b * stride + cb;
#pragma unroll
    for (int k = 0; k < 3; k++) {
      double2 v = ld_stream(q + (size_t)k * stride);
      B.d[2 * k] = v.x;
      B.d[2 * k + 1] = v.y;
    }
#pragma unroll
    for (int k = 0; k < 15; k++) {
      double2 v = ld_stream(q + (size_t)(3 + k) * stride);
      B.off[k] = {v.x, v.y};
    }
    return B;
  }
};
template <> struct CloverView<float> {
  const float4 *p;
  int stride;
  __device__ __forceinline__ CloverBlock<float> load(int b, int cb) const {
    // per block: 36 floats = 9 float4: d0..d5, off0.re,off0.im, then off1..off14 (28 floats)
    CloverBlock<float> B;
    const float4 *q = p + (size_t)9 * b * stride + cb;
    float f[36];
#pragma unroll
    for (int k = 0; k < 9; k++) {
      float4 v = ld_stream(q + (size_t)k * stride);
      f[4 * k] = v.x; f[4 * k + 1] = v.y; f[4 * k + 2] = v.z; f[4 * k + 3] = v.w;
    }
#pragma unroll
    for (int k = 0; k < 6; k++) B.d[k] = f[k];
#pragma unroll
    for (int k = 0; k < 15; k++) B.off[k] = {f[6 + 2 * k], f[7 + 2 * k]};
    return B;
  }
};

// y = B v for one packed Hermitian 6x6 block
template <typename R>
__device__ __forceinline__ void clover_block_mul(const CloverBlock<R> &B, const cx<R> v[6], cx<R> y[6]) {
#pragma unroll
  for (int i = 0; i < 6; i++) y[i] = B.d[i] * v[i];
#pragma unroll
  for (int i = 1; i < 6; i++)
#pragma unroll
    for (int j = 0; j < i; j++) {
      const cx<R> o = B.off[i * (i - 1) / 2 + j];
      y[i] = cmadd(o, v[j], y[i]);    // lower: M[i][j] = o
      y[j] = cjmadd(o, v[i], y[j]);   // upper: M[j][i] = conj(o)
    }
}
// out = A in (both chiral blocks: spins {0,1} -> block 0, {2,3} -> block 1)
template <typename R>
__device__ __forceinline__ Spinor<R> clover_mul(const CloverView<R> &A, int cb, const Spinor<R> &in) {
  Spinor<R> out;
#pragma unroll
  for (int b = 0; b < 2; b++) {
    CloverBlock<R> B = A.load(b, cb);
    cx<R> v[6], y[6];
#pragma unroll
    for (int i = 0; i < 6; i++) v[i] = in.c[6 * b + i];
    clover_block_mul(B, v, y);
#pragma unroll
    for (int i = 0; i < 6; i++) out.c[6 * b + i] = y[i];
  }
  return out;
}

// ------------------------------------------------------------------ 16-bit storage (sloppy level)
// The 16-bit sloppy precision of qdp_cg_solve_mixed16 (the reliable-update solvers of the paper's
// ref. [2]): fields stored as int16 fixed point, arithmetic in fp32.
//   spinor : 24 int16 per site, 3 int4 planes [3][stride], value = q * norm / 32767 with a
//            per-site float norm plane [stride] (norm = max |component| of the site)      52 B/site
//   gauge  : reconstruct-12 links, rows 0-1 as 12 int16 (|u_ij| <= 1 for SU(3)), value =
//            q / 32767; per (mu, parity): int4 plane (entries 0-3) + int2 plane (4-5)     24 B/link
//   clover : the 72 reals of both packed blocks (block b: d0..d5, off0 .. off14, the fp32
//            order) as 9 int4 planes + a per-site float norm plane                       148 B/site
struct h16 {};
template <typename S> struct Arith { using T = S; };
template <> struct Arith<h16> { using T = float; };
template <typename S> using Arith_t = typename Arith<S>::T;
constexpr float H16_SCALE = 32767.0f;

// int16 <-> fp32 without the quarter-rate I2F / F2I conversions: a 16-bit value q is stored in
// offset binary u = q + 32768; the float whose bit pattern is 0x4B400000 + u equals 1.5 * 2^23 + u
// exactly, so one byte permute and one add decode it, and adding 1.5 * 2^23 + 32768 to a value
// in [-32767.5, 32767.5] leaves round-to-nearest(q) + 32768 in the low 16 bits of the float.
constexpr float H16_MAGIC = 12615680.0f;  // 1.5 * 2^23 + 32768
__device__ __forceinline__ float h16_lo(int w) { return __int_as_float(__byte_perm(w, 0x4B400000, 0x7610)) - H16_MAGIC; }
__device__ __forceinline__ float h16_hi(int w) { return __int_as_float(__byte_perm(w, 0x4B400000, 0x7632)) - H16_MAGIC; }
// two values already scaled to [-32767, 32767] -> one word (lo in bits 0-15)
__device__ __forceinline__ int h16_pack(float lo, float hi) {
  return __byte_perm(__float_as_int(lo + H16_MAGIC), __float_as_int(hi + H16_MAGIC), 0x5410);
}

template <> struct FermView<h16> {
  int4 *p;      // [3][stride]
  float *norm;  // [stride]
  int stride;
  template <bool STREAM> __device__ __forceinline__ Spinor<float> load_(int cb) const {
    Spinor<float> s;
    const float n = (STREAM ? ld_stream(norm + cb) : __ldg(norm + cb)) * (1.0f / H16_SCALE);
#pragma unroll
    for (int k = 0; k < 3; k++) {
      const int4 v = STREAM ? ld_stream(p + (size_t)k * stride + cb) : __ldg(p + (size_t)k * stride + cb);
      const int w[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
      for (int j = 0; j < 4; j++) s.c[4 * k + j] = {n * h16_lo(w[j]), n * h16_hi(w[j])};
    }
    return s;
  }
  __device__ __forceinline__ Spinor<float> load(int cb) const { return load_<false>(cb); }
  __device__ __forceinline__ Spinor<float> load_stream(int cb) const { return load_<true>(cb); }
  __device__ __forceinline__ Spinor<float> load_plain(int cb) const { return load_<false>(cb); }
  // the stored integers as floats (exact) and the factor that scales them: the dslash applies the
  // factor once, fused into its accumulation, instead of 24 multiplies per spinor
  __device__ __forceinline__ Spinor<float> load_raw(int cb, float &scale) const {
    Spinor<float> s;
    scale = __ldg(norm + cb) * (1.0f / H16_SCALE);
#pragma unroll
    for (int k = 0; k < 3; k++) {
      const int4 v = __ldg(p + (size_t)k * stride + cb);
      const int w[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
      for (int j = 0; j < 4; j++) s.c[4 * k + j] = {h16_lo(w[j]), h16_hi(w[j])};
    }
    return s;
  }
  __device__ __forceinline__ void store(int cb, const Spinor<float> &s) const {
    float m = 0.f;
#pragma unroll
    for (int k = 0; k < 12; k++) m = fmaxf(m, fmaxf(fabsf(s.c[k].re), fabsf(s.c[k].im)));
    const float inv = m > 0.f ? H16_SCALE / m : 0.f;
#pragma unroll
    for (int k = 0; k < 3; k++) {
      int w[4];
#pragma unroll
      for (int j = 0; j < 4; j++)
        w[j] = h16_pack(s.c[4 * k + j].re * inv, s.c[4 * k + j].im * inv);
      __stcs(p + (size_t)k * stride + cb, make_int4(w[0], w[1], w[2], w[3]));
    }
    __stcs(norm + cb, m);
  }
};
template <> struct GaugeView<h16, 12> {
  const char *p;  // per (mu, parity): int4 [stride] then int2 [stride]
  int stride;
  __device__ __forceinline__ Link<float> load(int mu, int par, int cb) const {
    const char *b = p + (size_t)(mu * 2 + par) * 24 * stride;
    const int4 a = ld_stream((const int4 *)b + cb);
    const int2 c = ld_stream((const int2 *)(b + (size_t)16 * stride) + cb);
    const int w[6] = {a.x, a.y, a.z, a.w, c.x, c.y};
    constexpr float s = 1.0f / H16_SCALE;
    Link<float> u;
#pragma unroll
    for (int k = 0; k < 6; k++) u.m[k] = {s * h16_lo(w[k]), s * h16_hi(w[k])};
    su3_third_row(u);
    return u;
  }
  // 32767 x U: rows 0-1 as the stored integers, row 2 = conj(row0 x row1) / 32767 (so the link is
  // uniformly scaled; the dslash folds 1/32767 into its accumulation)
  static constexpr float raw_scale = 1.0f / H16_SCALE;
  __device__ __forceinline__ Link<float> load_raw(int mu, int par, int cb) const {
    const char *b = p + (size_t)(mu * 2 + par) * 24 * stride;
    const int4 a = ld_stream((const int4 *)b + cb);
    const int2 c = ld_stream((const int2 *)(b + (size_t)16 * stride) + cb);
    const int w[6] = {a.x, a.y, a.z, a.w, c.x, c.y};
    Link<float> u;
#pragma unroll
    for (int k = 0; k < 6; k++) u.m[k] = {h16_lo(w[k]), h16_hi(w[k])};
    su3_third_row(u);
#pragma unroll
    for (int k = 6; k < 9; k++) u.m[k] = raw_scale * u.m[k];
    return u;
  }
};
template <> struct CloverView<h16> {
  const int4 *p;      // [9][stride]
  const float *norm;  // [stride]
  int stride;
  __device__ __forceinline__ CloverBlock<float> load(int b, int cb) const {
    float n;
    CloverBlock<float> B = load_raw(b, cb, n);
#pragma unroll
    for (int k = 0; k < 6; k++) B.d[k] *= n;
#pragma unroll
    for (int k = 0; k < 15; k++) B.off[k] = n * B.off[k];
    return B;
  }
  // the stored integers as floats and the factor that scales them
  __device__ __forceinline__ CloverBlock<float> load_raw(int b, int cb, float &scale) const {
    // block b = int16 entries 36b .. 36b+35: int4 planes 4.5b .. (plane 4 shared)
    scale = ld_stream(norm + cb) * (1.0f / H16_SCALE);
    const float n = 1.0f;
    float f[40];
    const int first = b ? 4 : 0;
#pragma unroll
    for (int k = 0; k < 5; k++) {
      const int4 v = ld_stream(p + (size_t)(first + k) * stride + cb);
      const int w[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
      for (int j = 0; j < 4; j++) {
        f[8 * k + 2 * j] = n * h16_lo(w[j]);
        f[8 * k + 2 * j + 1] = n * h16_hi(w[j]);
      }
    }
    const int o = b ? 4 : 0;  // block 1 starts at entry 36 = plane 4, entry 4
    CloverBlock<float> B;
#pragma unroll
    for (int k = 0; k < 6; k++) B.d[k] = f[o + k];
#pragma unroll
    for (int k = 0; k < 15; k++) B.off[k] = {f[o + 6 + 2 * k], f[o + 7 + 2 * k]};
    return B;
  }
};
// out = A in for any storage of A (arithmetic in Arith_t); the 16-bit clover multiplies its stored
// integers and scales the 12 results once (instead of its 72 entries)
template <typename S>
__device__ __forceinline__ Spinor<Arith_t<S>> clover_mul_s(const CloverView<S> &A, int cb, const Spinor<Arith_t<S>> &in) {
  using T = Arith_t<S>;
  Spinor<T> out;
#pragma unroll
  for (int b = 0; b < 2; b++) {
    T sc = T(1);
    CloverBlock<T> B;
    if constexpr (std::is_same<S, h16>::value) B = A.load_raw(b, cb, sc);
    else B = A.load(b, cb);
    cx<T> v[6], y[6];
#pragma unroll
    for (int i = 0; i < 6; i++) v[i] = in.c[6 * b + i];
    clover_block_mul(B, v, y);
#pragma unroll
    for (int i = 0; i < 6; i++) out.c[6 * b + i] = std::is_same<S, h16>::value ? sc * y[i] : y[i];
  }
  return out;
}
template <typename R> constexpr bool is_h16() { return std::is_same<R, h16>::value; }

#endif  // __CUDACC__

// ------------------------------------------------------------------ host-side objects
enum { KIND_FERMION = QDP_FERMION, KIND_GAUGE = QDP_GAUGE, KIND_CLOVER = QDP_CLOVER, KIND_GAUGE12 = QDP_GAUGE12,
       KIND_CMAT = QDP_COLORMATRIX, KIND_SMAT = QDP_SPINMATRIX };

// Block-size autotuner state of one (expression, precision, volume).
struct Tune {
  int state = 0;           // 0 untouched, 1 probing, 2 done
  int block = 1024, best_block = 0;
  float best_ms = 0.f;
  bool pending = false;    // an event pair of the last payload launch awaits reading
  bool warm = true;        // the candidate's next launch is its first: run it untimed
  cudaEvent_t a = nullptr, b = nullptr;
};
struct JitKernel;  // jit.cu
inline bool is_gauge(int kind) { return kind == KIND_GAUGE || kind == KIND_GAUGE12; }

size_t parity_block_bytes(int kind, int prec, int stride);  // bytes of one parity block
size_t host_site_reals(int kind);                           // 24 / 72 / 288

struct Comm;      // comm.cpp
struct P2P;       // p2p.cu
struct PeerComm;  // peer.cu

struct ProfEvent {
  int cls;
  cudaEvent_t a, b;
};

}  // namespace qdpb

struct qdp_field_s {
  qdp_ctx ctx;
  int kind, prec, subset;
  void *data;
  size_t bytes;
  bool owned;
};

struct qdp_ctx_s {
  int gdims[4], pgrid[4], pcoord[4];
  int rank, nranks, device;
  qdpb::Geom geom;
  long V;
  cudaStream_t stream = nullptr, comm_stream = nullptr;
  bool own_stream = false;
  cudaEvent_t ev_packed = nullptr, ev_comm = nullptr;
  // options
  int overlap = 1, self_halo = 0, profiling = 0, block = 0, det_reduce = 1, self_nccl = 0;
  int fuse = 1;  // QDP_OPT_FUSE (default: env QDPB_FUSE, else 1)
  int dslash_variant = -1;  // QDP_OPT_DSLASH_VARIANT: -1 tuned, else the forced launch variant
  int pdl = 1;  // QDP_OPT_PDL (default: env QDPB_PDL, else 1): solver-chain kernels with programmatic dependent launch
  // scratch (device)
  void *staging = nullptr;
  size_t staging_bytes = 0;
  double *red_partials = nullptr;  // per-block partial sums (2 doubles per block)
  double *red_partials2 = nullptr; // per-group partial sums of the one-launch reductions (reduce.cuh)
  unsigned *red_cnt = nullptr;     // their counters: [0] top, [1 + g] groups (zero between launches)
  int red_capacity = 0;            // number of blocks
  double *red_result = nullptr;    // device scalars: [0..7]
  double *red_gather = nullptr;    // [nranks * 2] gathered per-rank sums
  double *host_pinned = nullptr;   // pinned host scratch (64 doubles; [32..40): reduction results)
  double *cg_hist = nullptr;       // mapped pinned |r_k|^2 of the device-side CG bookkeeping
  int cg_hist_cap = 0;
  unsigned red_token = 0;          // token of the last reduction read through read_red_host
  int *cg_stop = nullptr;          // device: first iteration that stops the CG (reduce.cuh CgDev)
  void *cg_work = nullptr;         // persistent CG work vectors
  size_t cg_work_bytes = 0;
  // halo buffers: [prec][mu][dir] for send and recv (dir 0 = to/from -mu, 1 = to/from +mu)
  void *halo_send[2][4][2] = {}, *halo_recv[2][4][2] = {};
  size_t halo_bytes[2] = {0, 0};
  qdpb::Comm *comm = nullptr;
  qdpb::P2P *p2p = nullptr;  // peer-to-peer halo state (QDP_OPT_P2P)
  int p2p_on = 0;
  // fused peer-to-peer boundary (dslash.cu): per output parity, interior sites first, then face sites
  int *fuse_perm[2] = {nullptr, nullptr};
  int fuse_nin[2] = {0, 0};
  int fuse_part = -1;
  // z / z x t partitions: the (z,t) slabs on a partitioned face, after the interior ones (dslash.cu)
  int *fuse_slabs = nullptr;
  int fuse_slab_part = -1, fuse_nslab_in = 0;
  // peer-memory communicator (qdp_init_peer; peer.cu): no NCCL; the host allgather callback
  // exchanges IPC handles at set-up time only
  qdpb::PeerComm *peer = nullptr;
  qdp_allgather_fn allgather = nullptr;
  void *allgather_user = nullptr;
  int neighbour[4][2];  // ranks of -mu / +mu neighbours
  // profiling / counting
  long launches[QDP_PK_COUNT] = {};
  double work_flops[QDP_PK_COUNT] = {}, work_bytes[QDP_PK_COUNT] = {};
  double prof_ms[QDP_PK_COUNT] = {};
  std::vector<qdpb::ProfEvent> pending;
  int autotune = 1;
  std::map<long, qdpb::Tune> tune;
  // run-time generated site-expression kernels (jit.cu), keyed by expression + kinds + precision
  std::map<std::string, qdpb::JitKernel *> jit;
  int jit_compiled = 0;
  double jit_seconds = 0.0;
  std::vector<cudaEvent_t> event_pool;
  std::string last_error;
};

namespace qdpb {
// error helpers (capi.cu)
int set_error(qdp_ctx ctx, int status, const char *fmt, ...);
int cuda_check(qdp_ctx ctx, cudaError_t e, const char *what);
#define QDP_CUDA(ctx, call)                                   \
  do {                                                        \
    cudaError_t _e = (call);                                  \
    if (_e != cudaSuccess) return qdpb::cuda_check(ctx, _e, #call); \
  } while (0)

// launch bookkeeping: call before/after each kernel launch
void prof_begin(qdp_ctx ctx, int cls, ProfEvent *ev);
// algorithmic work of the launch just begun (flops, compulsory bytes)
inline void prof_work(qdp_ctx ctx, int cls, double flops, double bytes) {
  ctx->work_flops[cls] += flops;
  ctx->work_bytes[cls] += bytes;
}
int prof_end(qdp_ctx ctx, ProfEvent *ev);  // checks cudaGetLastError

int ensure_staging(qdp_ctx ctx, size_t bytes);
int ensure_reduce(qdp_ctx ctx, int blocks);
int ensure_halo(qdp_ctx ctx, int prec);
int ensure_cg_work(qdp_ctx ctx, size_t bytes);

// ---- kernels entry points (host wrappers, each enqueues on ctx->stream) ----
// layout.cu
int layout_import(qdp_field f, const void *dev_aos);      // staging (device AoS) -> field
int layout_export(const qdp_field f, void *dev_aos);      // field -> staging
int field_copy_parity(qdp_ctx ctx, int kind, int prec, void *dst, const void *src, size_t bytes);

// blas.cu: operate on parity blocks (n_par = 1 or 2 consecutive blocks)
// y = a x + y
int blas_axpy(qdp_ctx ctx, int prec, double ar, double ai, const void *x, void *y, int nblk);
// partial sums -> red_result[slot] (and slot+1 for the imaginary part)
// GLOBAL sums (over all ranks), one launch with a peer communicator; host: also into
// host_pinned + 32 (read_red_host)
int blas_norm2(qdp_ctx ctx, int prec, const void *a, int nblk, int slot, bool host = false);
int blas_inner(qdp_ctx ctx, int prec, const void *a, const void *b, int nblk, int slot, bool host = false);
// sum nparts block partial pairs in red_partials -> red_result[slot], [slot+1]
int reduce_partials(qdp_ctx ctx, int nparts, int slot);
#ifdef __CUDACC__
// Arguments of a reduction that finishes inside its producing kernel of nblk blocks (reduce.cuh):
// res[slot .. slot+n); global: summed over the ranks -- in the kernel with a peer communicator
// (*after = false), else by reduce_global after the launch (*after = true); host: also store the
// values into ctx->host_pinned + 32 (read them with read_red_host).  Takes the peer sum's
// sequence number: call it right before the launch.
int red_setup(qdp_ctx ctx, int nblk, int slot, int n, bool global, bool host, RedArgs *R, bool *after);
#endif
int read_red_host(qdp_ctx ctx, int n, double *out);  // synchronise, then ctx->host_pinned[32 ..]
// finish a reduction: cross-rank sum of red_result[slot..slot+n-1]
int reduce_global(qdp_ctx ctx, int slot, int n);
// CG helpers (device scalars in red_result)
// r -= alpha q ; red_result[rr_slot] = |r|^2 (global), alpha = res[rho] / res[pq].  cg (optional):
// the device-side bookkeeping of iteration cg->k (skip when *cg->stop < cg->k; record |r_k|^2)
#ifdef __CUDACC__
int blas_cg_update_r(qdp_ctx ctx, int prec, void *r, const void *q, int rho_slot, int pq_slot, int rr_slot,
                     const CgDev *cg = nullptr);
#endif
// x += alpha p ; if update_p: p = r + beta p with beta = res[rr] / res[rho].  stop (optional):
// skip when *stop < iter, no p update when *stop == iter (iteration `iter` is the last)
int blas_cg_update_xp(qdp_ctx ctx, int prec, void *x, void *p, const void *r, int rho_slot, int pq_slot, int rr_slot,
                      bool update_p, const int *stop = nullptr, int iter = 0);
int blas_xpay(qdp_ctx ctx, int prec, const void *x, double a, void *y, int nblk);  // y = x + a y
// p = r + beta p with beta = res[rr] / res[rho]
int blas_cg_update_p(qdp_ctx ctx, int prec, void *p, const void *r, int rho_slot, int rr_slot);
// one fermion parity block fp64 <-> fp32 (dst_prec = precision of dst)
int blas_convert(qdp_ctx ctx, void *dst, int dst_prec, const void *src);
// y64 += x32 ; x32 = 0  (one parity block)
int blas_accum_mixed(qdp_ctx ctx, void *y64, void *x32);
int blas_scale_copy(qdp_ctx ctx, int prec, void *dst, const void *src, double a, int nblk);  // dst = a src
// Copy-engine-free scalar traffic of the solvers: a copy engine busy with a caller's large
// host<->device transfer would otherwise delay every per-iteration scalar readback (e2e).
//   read_scalars: red_result[slot .. slot+n) -> out via a kernel store into the mapped pinned
//                 host buffer, then a stream synchronisation (n <= 64)
//   copy_scalars: red_result[dst .. dst+n) = red_result[src .. src+n) by a kernel
//   copy_blocks:  nblk fermion parity blocks dst = src by a kernel
int read_scalars(qdp_ctx ctx, int slot, int n, double *out);
int copy_scalars(qdp_ctx ctx, int dst, int src, int n);
int copy_blocks(qdp_ctx ctx, int prec, void *dst, const void *src, int nblk);

// dslash.cu
enum Epi { EPI_PLAIN = 0, EPI_XPAY = 1, EPI_CLOVINV = 2, EPI_CLOVXPAY = 3 };
struct DslashArgs {
  void *out;              // output parity block
  const void *psi;        // input parity block (parity 1-p)
  const void *U;          // gauge field base
  const void *x;          // xpay vector (output parity block) or nullptr
  const void *clov;       // clover parity block for output parity (A or A^-1) or nullptr
  int parity;             // output parity p
  double a, b;            // epilogue scalars
  int epi;                // Epi
  bool g5_in, g5_out;
  const void *dot_x;      // if set: red_result[dot_slot] = Re<dot_x, out> (global), [dot_slot+1] = 0
  int dot_slot;
  double dot_shift;       // with dot_x: out += dot_shift * dot_x before the dot (multi-shift CG base shift)
  bool rec12;             // U is a QDP_GAUGE12 field
  bool h16;               // every operand in the 16-bit storage (U reconstruct-12)
};
int dslash(qdp_ctx ctx, int prec, const DslashArgs &a);
// the per-(storage, links) translation units behind dslash()
int dslash_d18(qdp_ctx ctx, const DslashArgs &a);
int dslash_d12(qdp_ctx ctx, const DslashArgs &a);
int dslash_f18(qdp_ctx ctx, const DslashArgs &a);
int dslash_f12(qdp_ctx ctx, const DslashArgs &a);
int dslash_h16(qdp_ctx ctx, const DslashArgs &a);

// clover.cu
int clover_build(qdp_ctx ctx, const qdp_field U, void *A, int A_subset, void *Ainv, int Ainv_subset,
                 double mass, double csw, int *singular_flag_host);
int clover_apply(qdp_ctx ctx, int prec, void *out, const void *A, const void *in, int nblk);

// p2p.cu: peer-to-peer halo.  For dslash call `seq` (1, 2, ...; identical on every rank),
// p2p_prepare makes sure the buffers exist and are mapped (collective on first use) and
// returns everything the pack and exterior kernels need to run the protocol themselves:
//   pack     : wait until war[mu][d] >= seq-2 (the receiver consumed this slot two calls ago),
//              store into dst[mu][d], the last block release-stores seq into sig[mu][d];
//   exterior : wait until ready[mu][d] >= seq, read ghost[mu][d], the last block release-stores
//              seq into ack_to[mu][d] (the senders' WAR flags).
struct P2PLaunch {
  void *dst[4][2];
  const void *ghost[4][2];
  unsigned *pack_counter[4], *ext_counter[4];
  unsigned *sig[4][2], *ack_to[4][2];
  const unsigned *war[4][2], *ready[4][2];
  unsigned *err;
  unsigned seq;               // this call's sequence number (taken after every set-up step succeeded)
  unsigned *pack_q;           // fused boundary: face-packing work queue, 2 sets x {next, done} (device)
};
// set up (collective on first use), then take the next sequence number and fill *out
int p2p_prepare(qdp_ctx ctx, int prec, P2PLaunch *out);
int p2p_check(qdp_ctx ctx);  // QDP_ECUDA if a flag wait timed out
void p2p_destroy(qdp_ctx ctx);

// expr.cu (Table II site expressions)
int expr_eval(qdp_ctx ctx, int expr, qdp_field out, const qdp_field a, const qdp_field b, const qdp_field c);
void tune_release(qdp_ctx ctx);
// the paper's block-size autotuner around go(block), per key (expr.cu)
int tuned_launch(qdp_ctx ctx, long key, const std::function<cudaError_t(int)> &go);
// the same rule over nvar launch variants ordered by decreasing threads per block (dslash.cu)
int tuned_variant(qdp_ctx ctx, long key, int nvar, const std::function<cudaError_t(int)> &go);

// jit.cu: run-time generated site-expression kernels (qdp_jit_eval)
struct JitKernel;
void jit_release(qdp_ctx ctx);
int jit_eval(qdp_field out, const char *expr, const qdp_field *ops, int nops);
// red_result[slot], [slot+1] = global sum of a complex-scalar expression over `subset`
int jit_sum(qdp_ctx ctx, const char *expr, const qdp_field *ops, int nops, int subset, int prec, int slot);
int jit_source(const char *expr, int out_kind, int out_subset, int prec, const int *kinds, int nops, char *src,
               size_t cap, size_t *src_len, double work[3], int compile, std::string &err);

// shift.cu
int shift_field(qdp_ctx ctx, qdp_field out, const qdp_field in, int mu, int sign);

// solver.cu
int cg_solve(qdp_field x, const qdp_field b, const qdp_field U, const qdp_field A,
             const qdp_field Ainv, double mass, double tol, int maxit, int *iters,
             double *hist, int hist_cap, double *true_resid);
int cg_solve_multishift(qdp_field *x, int nshift, const double *sigma, const qdp_field phi, const qdp_field U,
                        const qdp_field A, const qdp_field Ainv, double mass, double tol, int maxit, int *iters,
                        int *conv_iter, double *hist, int hist_cap, double *true_resid);
int cg_solve_mixed(qdp_field x, const qdp_field b, const qdp_field U, const qdp_field A, const qdp_field Ainv,
                   const qdp_field Us, const qdp_field As, const qdp_field Ainvs, double mass, double tol, double delta,
                   int maxit, int *iters, int *nreliable, double *hist, int hist_cap, double *true_resid);

// h16.cu: the 16-bit sloppy level (storage of internal.h "16-bit storage"): bytes per parity
// block of a fermion / per gauge field (8 reconstruct-12 links per site pair) / per clover block
inline size_t h16_fermion_bytes(int stride) { return (size_t)52 * stride; }
inline size_t h16_gauge_bytes(int stride) { return (size_t)8 * 24 * stride; }
inline size_t h16_clover_bytes(int stride) { return (size_t)148 * stride; }
int h16_gauge_from(qdp_ctx ctx, void *dst, const qdp_field U);            // U: F64/F32, 18 or 12
int h16_clover_from(qdp_ctx ctx, void *dst, const void *src_block, int prec);  // one clover parity block
int h16_from_f32(qdp_ctx ctx, void *p16, const void *r32);                 // one fermion parity block
int h16_cg_r(qdp_ctx ctx, void *r32, const void *q16, int rho_slot, int pq_slot, int rr_slot);
int h16_cg_xp(qdp_ctx ctx, void *x32, void *p16, const void *r32, int rho_slot, int pq_slot, int rr_slot, bool upd_p);
int h16_cg_p(qdp_ctx ctx, void *p16, const void *r32, int rho_slot, int rr_slot);
int cg_solve_mixed16(qdp_field x, const qdp_field b, const qdp_field U, const qdp_field A, const qdp_field Ainv,
                     double mass, double tol, double delta, int maxit, int *iters, int *nreliable, double *hist,
                     int hist_cap, double *true_resid);

// peer.cu: the peer-memory communicator of qdp_init_peer
int peer_init(qdp_ctx ctx);
void peer_destroy(qdp_ctx ctx);
int host_allgather(qdp_ctx ctx, const void *send, void *recv, size_t bytes);  // set-up only
int peer_allreduce(qdp_ctx ctx, int slot, int n);  // red_result[slot..slot+n) summed over ranks, rank order
#ifdef __CUDACC__
PeerArgs peer_args(qdp_ctx ctx);
#endif
unsigned peer_next_sum_seq(qdp_ctx ctx);
// copy `bytes` of a packed face into rank `to`'s mailbox and wait for this rank's own
// mailbox to receive the face of the same call; *ghost = the mailbox, *seq for release
int peer_sendrecv(qdp_ctx ctx, const void *send, size_t bytes, int to, void **ghost, unsigned *seq);
int peer_release_mailbox(qdp_ctx ctx, unsigned seq);  // after the mailbox has been read
int peer_check(qdp_ctx ctx);                          // QDP_ECUDA if a flag wait timed out
int p2p_setup_all(qdp_ctx ctx);                       // eager p2p halo set-up, both precisions

// comm.cpp
int comm_get_unique_id(unsigned char id[128]);
int comm_init(qdp_ctx ctx, const unsigned char *id);
void comm_destroy(qdp_ctx ctx);
// exchange halo buffers of `bytes[mu]` per face for every partitioned dim, on `stream`
int comm_exchange(qdp_ctx ctx, int prec, const size_t face_bytes[4], cudaStream_t stream);
int comm_sendrecv(qdp_ctx ctx, const void *send, size_t bytes, int to, void *recv, int from, cudaStream_t stream);
int comm_allgather_f64(qdp_ctx ctx, const double *send, double *recv, int count, cudaStream_t stream);
int comm_allreduce_f64(qdp_ctx ctx, double *buf, int count, cudaStream_t stream);
int comm_allgather_bytes(qdp_ctx ctx, const void *send, void *recv, size_t bytes, cudaStream_t stream);

// A partitioned dim whose neighbour is this rank and whose faces are written straight into
// the local ghost buffers (self-halo without NCCL).
inline bool direct_self(qdp_ctx ctx, int mu) { return ctx->pgrid[mu] == 1 && !ctx->self_nccl; }
// create a one-rank NCCL communicator for QDP_OPT_SELF_NCCL (comm.cpp)
int comm_ensure_self(qdp_ctx ctx);

inline size_t fermion_block_bytes(int prec, int stride) { return (size_t)stride * (prec == QDP_F64 ? 12 * 16 : 6 * 16); }
inline int grid_for(long n, int block) { return (int)((n + block - 1) / block); }

// Programmatic dependent launch (QDP_OPT_PDL).  A kernel of the solver chain (dslash, the BLAS and
// reduction kernels) is launched with programmatic stream serialisation: it may become resident
// while its predecessor in the stream drains its last blocks, so launch processing and block
// dispatch overlap that tail instead of following it.  Every such kernel starts with pdl_enter():
// griddepcontrol.wait blocks until the predecessor grid has completed and its memory is visible
// (a no-op without the attribute), then launch_dependents lets the successor in once every block
// of this grid has started -- so a dependent's blocks only take slots this grid's finished blocks
// free, and waits inside this grid (fused boundary flags, one-launch reductions) never depend on
// an unstarted block.
__device__ __forceinline__ void pdl_enter() {
  asm volatile("griddepcontrol.wait;" ::: "memory");
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}
template <typename... KA, typename... A>
cudaError_t launch_pdl(cudaStream_t stream, bool pdl, void (*kernel)(KA...), int grid, int block, size_t smem,
                       A &&...args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)grid);
  cfg.blockDim = dim3((unsigned)block);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = stream;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = pdl ? 1 : 0;
  return cudaLaunchKernelEx(&cfg, kernel, std::forward<A>(args)...);
}
// on the context stream, with PDL as QDP_OPT_PDL says
template <typename... KA, typename... A>
cudaError_t launch_k(qdp_ctx ctx, void (*kernel)(KA...), int grid, int block, A &&...args) {
  return launch_pdl(ctx->stream, ctx->pdl != 0, kernel, grid, block, 0, std::forward<A>(args)...);
}

}  // namespace qdpb
