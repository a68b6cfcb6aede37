// h16.cu -- the 16-bit sloppy level of qdp_cg_solve_mixed16 (the reliable-update mixed-precision
// solvers of the paper's ref. [2]): conversion of the fp64
// (or fp32) gauge / clover fields into the 16-bit storage of internal.h ("16-bit storage"), and
// the sloppy CG's vector updates between fp32 vectors (r, x) and 16-bit ones (p, q).  Arithmetic
// in fp32 throughout; quantisation is per site (one norm per spinor / clover site, a fixed scale
// for SU(3) links).
#include <string.h>

#include <algorithm>

#include "internal.h"

namespace qdpb {

constexpr int HB = 256;

// links rows 0-1 of U_mu(x) (x of parity par) -> int4 (entries 0-3) + int2 (entries 4-5)
template <typename R, int REC>
__global__ void __launch_bounds__(HB) gauge_h16_kernel(const Geom g, const GaugeView<R, REC> U, char *dst) {
  const int cb = blockIdx.x * blockDim.x + threadIdx.x;
  if (cb >= g.Vh) return;
  constexpr float s = H16_SCALE;
#pragma unroll
  for (int mu = 0; mu < 4; mu++)
#pragma unroll
    for (int par = 0; par < 2; par++) {
      const Link<R> u = U.load(mu, par, cb);
      int w[6];
#pragma unroll
      for (int k = 0; k < 6; k++)
        w[k] = h16_pack((float)u.m[k].re * s, (float)u.m[k].im * s);
      char *b = dst + (size_t)(mu * 2 + par) * 24 * g.stride;
      ((int4 *)b)[cb] = make_int4(w[0], w[1], w[2], w[3]);
      ((int2 *)(b + (size_t)16 * g.stride))[cb] = make_int2(w[4], w[5]);
    }
}

// one clover parity block (both chiral blocks, 72 reals) -> 9 int4 planes + a per-site norm
template <typename R>
__global__ void __launch_bounds__(HB) clover_h16_kernel(const Geom g, const CloverView<R> A, int4 *dst) {
  const int cb = blockIdx.x * blockDim.x + threadIdx.x;
  if (cb >= g.Vh) return;
  float f[72];
#pragma unroll
  for (int b = 0; b < 2; b++) {
    const CloverBlock<R> B = A.load(b, cb);
#pragma unroll
    for (int k = 0; k < 6; k++) f[36 * b + k] = (float)B.d[k];
#pragma unroll
    for (int k = 0; k < 15; k++) {
      f[36 * b + 6 + 2 * k] = (float)B.off[k].re;
      f[36 * b + 7 + 2 * k] = (float)B.off[k].im;
    }
  }
  float m = 0.f;
#pragma unroll
  for (int k = 0; k < 72; k++) m = fmaxf(m, fabsf(f[k]));
  const float inv = m > 0.f ? H16_SCALE / m : 0.f;
#pragma unroll
  for (int k = 0; k < 9; k++) {
    int w[4];
#pragma unroll
    for (int j = 0; j < 4; j++)
      w[j] = h16_pack(f[8 * k + 2 * j] * inv, f[8 * k + 2 * j + 1] * inv);
    dst[(size_t)k * g.stride + cb] = make_int4(w[0], w[1], w[2], w[3]);
  }
  ((float *)(dst + (size_t)9 * g.stride))[cb] = m;
}

__device__ __forceinline__ FermView<h16> hview(void *p, int stride) {
  return {(int4 *)p, (float *)((char *)p + (size_t)48 * stride), stride};
}
__device__ __forceinline__ FermView<float> fview32(void *p, int stride) { return {(float4 *)p, stride}; }

// p16 = (16-bit) r32
__global__ void __launch_bounds__(HB) to_h16_kernel(const Geom g, void *p16, const void *r32) {
  pdl_enter();
  const int cb = blockIdx.x * blockDim.x + threadIdx.x;
  if (cb >= g.Vh) return;
  hview(p16, g.stride).store(cb, fview32(const_cast<void *>(r32), g.stride).load_stream(cb));
}

// r32 -= alpha q16 ; |r|^2 (one launch, reduce.cuh), alpha = res[rho] / res[pq]
__global__ void __launch_bounds__(HB) cg16_r_kernel(const Geom g, void *r32, const void *q16, const double *res,
                                                    int rho_slot, int pq_slot, const __grid_constant__ RedArgs Rd) {
  pdl_enter();
  const float alpha = (float)(res[rho_slot] / res[pq_slot]);
  double acc = 0.0;
  const FermView<float> r = fview32(r32, g.stride);
  const FermView<h16> q = hview(const_cast<void *>(q16), g.stride);
  for (int cb = blockIdx.x * blockDim.x + threadIdx.x; cb < g.Vh; cb += gridDim.x * blockDim.x) {
    Spinor<float> rv = r.load_stream(cb);
    const Spinor<float> qv = q.load_stream(cb);
#pragma unroll
    for (int k = 0; k < 12; k++) {
      rv.c[k] = rv.c[k] - alpha * qv.c[k];
      acc += (double)rv.c[k].re * rv.c[k].re + (double)rv.c[k].im * rv.c[k].im;
    }
    r.store(cb, rv);
  }
  red_finish(Rd, gridDim.x, blockIdx.x, acc, 0.0, false);
}

// x32 += alpha p16 ; (UPD) p16 = r32 + beta p16   (alpha = res[rho]/res[pq], beta = res[rr]/res[rho])
template <bool UPD>
__global__ void __launch_bounds__(HB) cg16_xp_kernel(const Geom g, void *x32, void *p16, const void *r32,
                                                     const double *res, int rho_slot, int pq_slot, int rr_slot) {
  pdl_enter();
  const int cb = blockIdx.x * blockDim.x + threadIdx.x;
  if (cb >= g.Vh) return;
  const float alpha = (float)(res[rho_slot] / res[pq_slot]);
  const float beta = (float)(res[rr_slot] / res[rho_slot]);
  const FermView<float> x = fview32(x32, g.stride);
  const FermView<h16> p = hview(p16, g.stride);
  Spinor<float> xv = x.load_stream(cb);
  Spinor<float> pv = p.load_stream(cb);
#pragma unroll
  for (int k = 0; k < 12; k++) xv.c[k] = xv.c[k] + alpha * pv.c[k];
  x.store(cb, xv);
  if (UPD) {
    const Spinor<float> rv = fview32(const_cast<void *>(r32), g.stride).load_stream(cb);
#pragma unroll
    for (int k = 0; k < 12; k++) pv.c[k] = rv.c[k] + beta * pv.c[k];
    p.store(cb, pv);
  }
}

// p16 = r32 + beta p16, beta = res[rr] / res[rho]
__global__ void __launch_bounds__(HB) cg16_p_kernel(const Geom g, void *p16, const void *r32, const double *res,
                                                    int rho_slot, int rr_slot) {
  pdl_enter();
  const int cb = blockIdx.x * blockDim.x + threadIdx.x;
  if (cb >= g.Vh) return;
  const float beta = (float)(res[rr_slot] / res[rho_slot]);
  const FermView<h16> p = hview(p16, g.stride);
  Spinor<float> pv = p.load_stream(cb);
  const Spinor<float> rv = fview32(const_cast<void *>(r32), g.stride).load_stream(cb);
#pragma unroll
  for (int k = 0; k < 12; k++) pv.c[k] = rv.c[k] + beta * pv.c[k];
  p.store(cb, pv);
}

// ------------------------------------------------------------------ host wrappers
static int launch_end(qdp_ctx ctx, ProfEvent *ev) { return prof_end(ctx, ev); }

int h16_gauge_from(qdp_ctx ctx, void *dst, const qdp_field U) {
  const Geom &g = ctx->geom;
  ProfEvent ev;
  prof_begin(ctx, QDP_PK_LAYOUT, &ev);
  const double in = (U->kind == QDP_GAUGE12 ? 12 : 18) * (U->prec == QDP_F64 ? 8 : 4);
  prof_work(ctx, QDP_PK_LAYOUT, 0.0, 8.0 * (in + 24) * g.Vh);
  const int nb = grid_for(g.Vh, HB);
  const int s = g.stride;
  if (U->prec == QDP_F64) {
    if (U->kind == QDP_GAUGE12)
      gauge_h16_kernel<double, 12><<<nb, HB, 0, ctx->stream>>>(g, GaugeView<double, 12>{(const double2 *)U->data, s}, (char *)dst);
    else
      gauge_h16_kernel<double, 18><<<nb, HB, 0, ctx->stream>>>(g, GaugeView<double, 18>{(const double2 *)U->data, s}, (char *)dst);
  } else {
    if (U->kind == QDP_GAUGE12)
      gauge_h16_kernel<float, 12><<<nb, HB, 0, ctx->stream>>>(g, GaugeView<float, 12>{(const float4 *)U->data, s}, (char *)dst);
    else
      gauge_h16_kernel<float, 18><<<nb, HB, 0, ctx->stream>>>(g, GaugeView<float, 18>{(const float *)U->data, s}, (char *)dst);
  }
  return launch_end(ctx, &ev);
}

int h16_clover_from(qdp_ctx ctx, void *dst, const void *src_block, int prec) {
  const Geom &g = ctx->geom;
  ProfEvent ev;
  prof_begin(ctx, QDP_PK_LAYOUT, &ev);
  prof_work(ctx, QDP_PK_LAYOUT, 0.0, (72.0 * (prec == QDP_F64 ? 8 : 4) + 148) * g.Vh);
  const int nb = grid_for(g.Vh, HB);
  if (prec == QDP_F64)
    clover_h16_kernel<double><<<nb, HB, 0, ctx->stream>>>(g, CloverView<double>{(const double2 *)src_block, g.stride}, (int4 *)dst);
  else
    clover_h16_kernel<float><<<nb, HB, 0, ctx->stream>>>(g, CloverView<float>{(const float4 *)src_block, g.stride}, (int4 *)dst);
  return launch_end(ctx, &ev);
}

int h16_from_f32(qdp_ctx ctx, void *p16, const void *r32) {
  const Geom &g = ctx->geom;
  ProfEvent ev;
  prof_begin(ctx, QDP_PK_BLAS, &ev);
  prof_work(ctx, QDP_PK_BLAS, 0.0, (96.0 + 52.0) * g.Vh);
  launch_k(ctx, to_h16_kernel, grid_for(g.Vh, HB), HB, g, p16, r32);
  return launch_end(ctx, &ev);
}

int h16_cg_r(qdp_ctx ctx, void *r32, const void *q16, int rho_slot, int pq_slot, int rr_slot) {
  const Geom &g = ctx->geom;
  const int nb = std::min(grid_for(g.Vh, HB), 148 * 8);
  int rc;
  RedArgs R;
  bool after;
  if ((rc = red_setup(ctx, nb, rr_slot, 1, true, false, &R, &after))) return rc;
  ProfEvent ev;
  prof_begin(ctx, QDP_PK_BLAS, &ev);
  prof_work(ctx, QDP_PK_BLAS, 96.0 * g.Vh, (2 * 96.0 + 52.0) * g.Vh);
  launch_k(ctx, cg16_r_kernel, nb, HB, g, r32, q16, ctx->red_result, rho_slot, pq_slot, R);
  if ((rc = launch_end(ctx, &ev))) return rc;
  return after ? reduce_global(ctx, rr_slot, 1) : QDP_OK;
}

int h16_cg_xp(qdp_ctx ctx, void *x32, void *p16, const void *r32, int rho_slot, int pq_slot, int rr_slot, bool upd) {
  const Geom &g = ctx->geom;
  ProfEvent ev;
  prof_begin(ctx, QDP_PK_BLAS, &ev);
  prof_work(ctx, QDP_PK_BLAS, (upd ? 96.0 : 48.0) * g.Vh, (upd ? 2 * 96.0 + 2 * 52.0 + 96.0 : 2 * 96.0 + 52.0) * g.Vh);
  const int nb = grid_for(g.Vh, HB);
  if (upd) launch_k(ctx, cg16_xp_kernel<true>, nb, HB, g, x32, p16, r32, ctx->red_result, rho_slot, pq_slot, rr_slot);
  else launch_k(ctx, cg16_xp_kernel<false>, nb, HB, g, x32, p16, r32, ctx->red_result, rho_slot, pq_slot, rr_slot);
  return launch_end(ctx, &ev);
}

int h16_cg_p(qdp_ctx ctx, void *p16, const void *r32, int rho_slot, int rr_slot) {
  const Geom &g = ctx->geom;
  ProfEvent ev;
  prof_begin(ctx, QDP_PK_BLAS, &ev);
  prof_work(ctx, QDP_PK_BLAS, 48.0 * g.Vh, (2 * 52.0 + 96.0) * g.Vh);
  launch_k(ctx, cg16_p_kernel, grid_for(g.Vh, HB), HB, g, p16, r32, ctx->red_result, rho_slot, rr_slot);
  return launch_end(ctx, &ev);
}

}  // namespace qdpb
