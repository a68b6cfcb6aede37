// blas.cu -- lattice BLAS on fermion parity blocks: norm2 / innerProduct reductions
// (warp shuffle -> block partials -> one fixed-order final pass; fp64 accumulation for
// both precisions, deterministic for a fixed launch configuration), axpy, and the fused
// CG updates (north star).
//
// Every kernel runs one thread per checkerboard site (grid-stride), looping over the
// site's planes (12 double2 or 6 float4) and over nblk consecutive parity blocks, so the
// padded tail of each plane (cb >= Vh) is never read or written.
#include <string.h>

#include <algorithm>
#include <atomic>
#include <functional>

#include "internal.h"

namespace qdpb {

template <typename R> struct E;  // one plane element
template <> struct E<double> {
  using T = double2;
  static constexpr int NP = 12;  // planes per parity block
  static constexpr int NR = 2;   // reals per element
  static __device__ __forceinline__ void get(const T &v, double r[2]) { r[0] = v.x; r[1] = v.y; }
  static __device__ __forceinline__ T put(const double r[2]) { return make_double2(r[0], r[1]); }
};
template <> struct E<float> {
  using T = float4;
  static constexpr int NP = 6;
  static constexpr int NR = 4;
  static __device__ __forceinline__ void get(const T &v, float r[4]) { r[0] = v.x; r[1] = v.y; r[2] = v.z; r[3] = v.w; }
  static __device__ __forceinline__ T put(const float r[4]) { return make_float4(r[0], r[1], r[2], r[3]); }
};

constexpr int RB = 256;  // block of the untuned launches
// reductions run one site per thread like the other kernels (a capped grid-stride grid left the
// last stride a third full at 40^3 x 32; the two-level finish of reduce.cuh takes any block count)

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}
// Final pass: one block sums n partial pairs in a fixed order -> res[slot], res[slot+1].
__global__ void __launch_bounds__(1024) final_kernel(const double *partials, int n, double *res, int slot) {
  __shared__ double s0[32], s1[32];
  double v0 = 0.0, v1 = 0.0;
  for (int i = threadIdx.x; i < n; i += blockDim.x) { v0 += partials[2 * i]; v1 += partials[2 * i + 1]; }
  v0 = warp_sum(v0);
  v1 = warp_sum(v1);
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  if (l == 0) { s0[w] = v0; s1[w] = v1; }
  __syncthreads();
  if (w == 0) {
    const int nw = blockDim.x >> 5;
    v0 = l < nw ? s0[l] : 0.0;
    v1 = l < nw ? s1[l] : 0.0;
    v0 = warp_sum(v0);
    v1 = warp_sum(v1);
    if (l == 0) { res[slot] = v0; res[slot + 1] = v1; }
  }
}

// rank-ordered sum of gathered per-rank values: res[slot+k] = sum_r g[r*n + k]
__global__ void rank_sum_kernel(const double *g, int nranks, int n, double *res, int slot) {
  const int k = threadIdx.x;
  if (k >= n) return;
  double s = 0.0;
  for (int r = 0; r < nranks; r++) s += g[r * n + k];
  res[slot + k] = s;
}

template <typename R>
__global__ void __launch_bounds__(1024) norm2_kernel(const Geom g, const typename E<R>::T *a, int nblk, const __grid_constant__ RedArgs Rd) {
  pdl_enter();
  double acc = 0.0;
  const size_t bs = (size_t)E<R>::NP * g.stride;
  for (int cb = blockIdx.x * blockDim.x + threadIdx.x; cb < g.Vh; cb += gridDim.x * blockDim.x)
    for (int b = 0; b < nblk; b++)
#pragma unroll
      for (int k = 0; k < E<R>::NP; k++) {
        R v[E<R>::NR];
        E<R>::get(ld_stream(a + b * bs + (size_t)k * g.stride + cb), v);
#pragma unroll
        for (int j = 0; j < E<R>::NR; j++) acc += (double)v[j] * (double)v[j];
      }
  red_finish(Rd, gridDim.x, blockIdx.x, acc, 0.0, false);
}

template <typename R>
__global__ void __launch_bounds__(1024) inner_kernel(const Geom g, const typename E<R>::T *a, const typename E<R>::T *b_,
                                                   int nblk, const __grid_constant__ RedArgs Rd) {
  pdl_enter();
  double re = 0.0, im = 0.0;
  const size_t bs = (size_t)E<R>::NP * g.stride;
  for (int cb = blockIdx.x * blockDim.x + threadIdx.x; cb < g.Vh; cb += gridDim.x * blockDim.x)
    for (int b = 0; b < nblk; b++)
#pragma unroll
      for (int k = 0; k < E<R>::NP; k++) {
        const size_t i = b * bs + (size_t)k * g.stride + cb;
        R u[E<R>::NR], v[E<R>::NR];
        E<R>::get(ld_stream(a + i), u);
        E<R>::get(ld_stream(b_ + i), v);
#pragma unroll
        for (int j = 0; j < E<R>::NR; j += 2) {
          re += (double)u[j] * v[j] + (double)u[j + 1] * v[j + 1];
          im += (double)u[j] * v[j + 1] - (double)u[j + 1] * v[j];
        }
      }
  red_finish(Rd, gridDim.x, blockIdx.x, re, im, false);
}

template <typename R>
__global__ void __launch_bounds__(1024) axpy_kernel(const Geom g, R ar, R ai, const typename E<R>::T *x,
                                                  typename E<R>::T *y, int nblk) {
  pdl_enter();
  const size_t bs = (size_t)E<R>::NP * g.stride;
  for (int cb = blockIdx.x * blockDim.x + threadIdx.x; cb < g.Vh; cb += gridDim.x * blockDim.x)
    for (int b = 0; b < nblk; b++)
#pragma unroll
      for (int k = 0; k < E<R>::NP; k++) {
        const size_t i = b * bs + (size_t)k * g.stride + cb;
        R u[E<R>::NR], v[E<R>::NR];
        E<R>::get(ld_stream(x + i), u);
        E<R>::get(y[i], v);
#pragma unroll
        for (int j = 0; j < E<R>::NR; j += 2) {
          const R re = ar * u[j] - ai * u[j + 1] + v[j];
          const R im = ar * u[j + 1] + ai * u[j] + v[j + 1];
          v[j] = re;
          v[j + 1] = im;
        }
        st_stream(y + i, E<R>::put(v));
      }
}

// y = x + a y
template <typename R>
__global__ void __launch_bounds__(1024) xpay_kernel(const Geom g, const typename E<R>::T *x, R a, typename E<R>::T *y, int nblk) {
  pdl_enter();
  const size_t bs = (size_t)E<R>::NP * g.stride;
  for (int cb = blockIdx.x * blockDim.x + threadIdx.x; cb < g.Vh; cb += gridDim.x * blockDim.x)
    for (int b = 0; b < nblk; b++)
#pragma unroll
      for (int k = 0; k < E<R>::NP; k++) {
        const size_t i = b * bs + (size_t)k * g.stride + cb;
        R u[E<R>::NR], v[E<R>::NR];
        E<R>::get(ld_stream(x + i), u);
        E<R>::get(y[i], v);
#pragma unroll
        for (int j = 0; j < E<R>::NR; j++) v[j] = u[j] + a * v[j];
        st_stream(y + i, E<R>::put(v));
      }
}

template <typename R>
__global__ void __launch_bounds__(1024) scale_copy_kernel(const Geom g, typename E<R>::T *d, const typename E<R>::T *s, R a, int nblk) {
  pdl_enter();
  const size_t bs = (size_t)E<R>::NP * g.stride;
  for (int cb = blockIdx.x * blockDim.x + threadIdx.x; cb < g.Vh; cb += gridDim.x * blockDim.x)
    for (int b = 0; b < nblk; b++)
#pragma unroll
      for (int k = 0; k < E<R>::NP; k++) {
        const size_t i = b * bs + (size_t)k * g.stride + cb;
        R u[E<R>::NR];
        E<R>::get(ld_stream(s + i), u);
#pragma unroll
        for (int j = 0; j < E<R>::NR; j++) u[j] *= a;
        st_stream(d + i, E<R>::put(u));
      }
}

// r -= alpha q ; |r|^2 (one launch, reduce.cuh)   with alpha = res[rho] / res[pq]  (CG step 5).
// Rd.has_cg: iteration Rd.cg.k of the device-side CG (no work once *stop < k; records |r_k|^2).
template <typename R>
__global__ void __launch_bounds__(256) cg_r_kernel(const Geom g, typename E<R>::T *r, const typename E<R>::T *q,
                                                  const double *res, int rho_slot, int pq_slot,
                                                  const __grid_constant__ RedArgs Rd) {
  pdl_enter();
  // one site per thread (blas_launch sizes the grid); the block's partial of |r|^2 is published
  // BEFORE the r stores, so its fence does not wait for them (reduce.cuh red_arrive).  The new r
  // is held in registers meanwhile: launch bound 256 (1024 would cap it at 64 registers and spill;
  // the tuner's 1024 and 512 launches fail and it halves)
  const bool skip = Rd.has_cg && cg_skip(Rd.cg.stop, Rd.cg.k);
  const int cb = blockIdx.x * blockDim.x + threadIdx.x;
  const bool have = !skip && cb < g.Vh;
  double acc = 0.0;
  typename E<R>::T out[E<R>::NP];
  if (have) {
    const R alpha = (R)(res[rho_slot] / res[pq_slot]);
#pragma unroll
    for (int k = 0; k < E<R>::NP; k++) {
      const size_t i = (size_t)k * g.stride + cb;
      R rv[E<R>::NR], qv[E<R>::NR];
      E<R>::get(r[i], rv);
      E<R>::get(ld_stream(q + i), qv);
#pragma unroll
      for (int j = 0; j < E<R>::NR; j++) {
        rv[j] = rv[j] - alpha * qv[j];
        acc += (double)rv[j] * (double)rv[j];
      }
      out[k] = E<R>::put(rv);
    }
  }
  const bool last = red_arrive(Rd, gridDim.x, blockIdx.x, acc, 0.0);
  if (have) {
#pragma unroll
    for (int k = 0; k < E<R>::NP; k++) st_stream(r + (size_t)k * g.stride + cb, out[k]);
  }
  if (last) red_complete(Rd, gridDim.x, blockIdx.x, skip);
}

// x += alpha p ; p = r + beta p (UPD_P), alpha = res[rho] / res[pq], beta = res[rr] / res[rho].
// stop (device-side CG): no work when *stop < iter; x only when *stop == iter (the last iteration)
template <typename R, bool UPD_P>
__global__ void __launch_bounds__(1024) cg_xp_kernel(const Geom g, typename E<R>::T *x, typename E<R>::T *p,
                                                   const typename E<R>::T *r, const double *res, int rho_slot,
                                                   int pq_slot, int rr_slot, const int *stop, int iter) {
  pdl_enter();
  bool upd_p = UPD_P;
  if (stop) {
    const int s = __ldcg(stop);
    if (s < iter) return;
    if (s == iter) upd_p = false;
  }
  const R alpha = (R)(res[rho_slot] / res[pq_slot]);
  const R beta = (R)(res[rr_slot] / res[rho_slot]);
  for (int cb = blockIdx.x * blockDim.x + threadIdx.x; cb < g.Vh; cb += gridDim.x * blockDim.x)
#pragma unroll
    for (int k = 0; k < E<R>::NP; k++) {
      const size_t i = (size_t)k * g.stride + cb;
      R xv[E<R>::NR], pv[E<R>::NR], rv[E<R>::NR];
      E<R>::get(x[i], xv);
      E<R>::get(p[i], pv);
      if (UPD_P && upd_p) E<R>::get(ld_stream(r + i), rv);
#pragma unroll
      for (int j = 0; j < E<R>::NR; j++) {
        xv[j] = xv[j] + alpha * pv[j];
        if (UPD_P && upd_p) pv[j] = rv[j] + beta * pv[j];
      }
      st_stream(x + i, E<R>::put(xv));
      if (UPD_P && upd_p) st_stream(p + i, E<R>::put(pv));
    }
}

// p = r + beta p, beta = res[rr] / res[rho]
template <typename R>
__global__ void __launch_bounds__(1024) cg_p_kernel(const Geom g, typename E<R>::T *p, const typename E<R>::T *r,
                                                  const double *res, int rho_slot, int rr_slot) {
  pdl_enter();
  const R beta = (R)(res[rr_slot] / res[rho_slot]);
  for (int cb = blockIdx.x * blockDim.x + threadIdx.x; cb < g.Vh; cb += gridDim.x * blockDim.x)
#pragma unroll
    for (int k = 0; k < E<R>::NP; k++) {
      const size_t i = (size_t)k * g.stride + cb;
      R pv[E<R>::NR], rv[E<R>::NR];
      E<R>::get(p[i], pv);
      E<R>::get(ld_stream(r + i), rv);
#pragma unroll
      for (int j = 0; j < E<R>::NR; j++) pv[j] = rv[j] + beta * pv[j];
      st_stream(p + i, E<R>::put(pv));
    }
}

// Precision conversion of one fermion parity block: fp64 double2[12] <-> fp32 float4[6].
template <bool TO32>
__global__ void __launch_bounds__(1024) convert_kernel(const Geom g, double2 *d64, float4 *f32) {
  pdl_enter();
  for (int cb = blockIdx.x * blockDim.x + threadIdx.x; cb < g.Vh; cb += gridDim.x * blockDim.x)
#pragma unroll
    for (int k = 0; k < 6; k++) {
      double2 *a = d64 + (size_t)(2 * k) * g.stride + cb, *b = d64 + (size_t)(2 * k + 1) * g.stride + cb;
      float4 *f = f32 + (size_t)k * g.stride + cb;
      if (TO32) {
        const double2 u = *a, v = *b;
        *f = make_float4((float)u.x, (float)u.y, (float)v.x, (float)v.y);
      } else {
        const float4 w = *f;
        *a = make_double2(w.x, w.y);
        *b = make_double2(w.z, w.w);
      }
    }
}

// y64 += x32 (the reliable update's accumulation of the sloppy solution), then x32 = 0
__global__ void __launch_bounds__(1024) accum_mixed_kernel(const Geom g, double2 *y64, float4 *x32) {
  pdl_enter();
  for (int cb = blockIdx.x * blockDim.x + threadIdx.x; cb < g.Vh; cb += gridDim.x * blockDim.x)
#pragma unroll
    for (int k = 0; k < 6; k++) {
      double2 *a = y64 + (size_t)(2 * k) * g.stride + cb, *b = y64 + (size_t)(2 * k + 1) * g.stride + cb;
      float4 *f = x32 + (size_t)k * g.stride + cb;
      const float4 w = *f;
      double2 u = *a, v = *b;
      u.x += w.x; u.y += w.y; v.x += w.z; v.y += w.w;
      *a = u;
      *b = v;
      *f = make_float4(0.f, 0.f, 0.f, 0.f);
    }
}

// ------------------------------------------------------------------ host wrappers

template <typename R> using T_ = typename E<R>::T;

// The paper's autotuner (expr.cu tuned_launch) on the launch configuration of
// every BLAS kernel, per (kernel, precision, number of parity blocks, volume): the block size
// starts at 1024 and halves on later payload launches until one is 33% slower than the best.
// `launch(grid, block)` enqueues the kernel (one site per thread; the kernels keep a grid-stride loop).
enum { K_NORM2 = 1, K_INNER, K_AXPY, K_XPAY, K_SCALE, K_COPY, K_CGR, K_CGXP, K_CGXP0, K_CGP, K_CONV32, K_CONV64, K_ACCUM };
static int blas_launch(qdp_ctx ctx, int kid, int prec, int nblk, bool red,
                       const std::function<void(int grid, int block)> &launch) {
  const Geom &g = ctx->geom;
  const long key = (1L << 60) | ((long)kid << 44) | ((long)prec << 43) | ((long)nblk << 41) | (long)g.Vh;
  // a block above the kernel's launch bound "fails" up front, without a launch (as the expression
  // kernels do): the tuner halves, and no failed launch reaches the driver
  const int max_block = kid == K_CGR ? 256 : 1024;
  return tuned_launch(ctx, key, [&](int block) -> cudaError_t {
    (void)red;
    if (block > max_block) return cudaErrorLaunchOutOfResources;
    launch(grid_for(g.Vh, block), block);
    return cudaGetLastError();
  });
}
// largest grid a tuned reduction can use (its partial arrays are sized for it)
static int red_grid_max(const Geom &g) { return std::max(1, grid_for(g.Vh, 32)); }

int reduce_partials(qdp_ctx ctx, int nparts, int slot) {
  ProfEvent ev;
  prof_begin(ctx, QDP_PK_REDUCE, &ev);
  final_kernel<<<1, 1024, 0, ctx->stream>>>(ctx->red_partials, nparts, ctx->red_result, slot);
  return prof_end(ctx, &ev);
}

int red_setup(qdp_ctx ctx, int nblk, int slot, int n, bool global, bool host, RedArgs *R, bool *after) {
  int rc;
  if ((rc = ensure_reduce(ctx, nblk))) return rc;
  memset(R, 0, sizeof(*R));
  R->part = ctx->red_partials;
  R->part2 = ctx->red_partials2;
  R->cnt = ctx->red_cnt;
  R->res = ctx->red_result;
  R->slot = slot;
  R->n = n;
  const bool multi = global && ctx->nranks > 1;
  R->peer = multi && ctx->peer;
  *after = multi && !ctx->peer;  // NCCL: reduce_global after the launch
  if (host && !*after) {
    R->host = ctx->host_pinned + 32;
    R->host_flag = (unsigned *)(ctx->host_pinned + 36);
    R->token = ++ctx->red_token;
    *(volatile unsigned *)R->host_flag = 0u;
  }
  if (R->peer) {
    R->pa = peer_args(ctx);
    R->seq = peer_next_sum_seq(ctx);
  }
  return QDP_OK;
}

// The final block of the reduction stores the values and then the call's token into mapped host
// memory: poll for the token (no stream synchronisation -- the kernel's remaining blocks have all
// finished their share), then read.  Falls back to a synchronisation (which also reports a
// failed launch) if the token does not show up within ~2 s.
int read_red_host(qdp_ctx ctx, int n, double *out) {
  const volatile unsigned *flag = (const volatile unsigned *)(ctx->host_pinned + 36);
  const unsigned token = ctx->red_token;
  long spins = 0;
  while (*flag != token) {
    if (++spins > (1L << 27)) {
      QDP_CUDA(ctx, cudaStreamSynchronize(ctx->stream));
      if (*flag != token) return set_error(ctx, QDP_ECUDA, "reduction result never arrived");
      break;
    }
  }
  std::atomic_thread_fence(std::memory_order_acquire);
  for (int i = 0; i < n; i++) out[i] = ((volatile double *)ctx->host_pinned)[32 + i];
  return QDP_OK;
}

int blas_norm2(qdp_ctx ctx, int prec, const void *a, int nblk, int slot, bool host) {
  const Geom &g = ctx->geom;
  int rc;
  RedArgs R;
  bool after;
  if ((rc = red_setup(ctx, red_grid_max(g), slot, 1, true, host, &R, &after))) return rc;
  ProfEvent ev;
  prof_begin(ctx, QDP_PK_REDUCE, &ev);
  prof_work(ctx, QDP_PK_REDUCE, 48.0 * g.Vh * nblk, 24.0 * g.Vh * nblk * (prec == QDP_F64 ? 8 : 4));
  rc = blas_launch(ctx, K_NORM2, prec, nblk, true, [&](int nb, int bs) {
    if (prec == QDP_F64) launch_k(ctx, norm2_kernel<double>, nb, bs, g, (const T_<double> *)a, nblk, R);
    else launch_k(ctx, norm2_kernel<float>, nb, bs, g, (const T_<float> *)a, nblk, R);
  });
  if (rc || (rc = prof_end(ctx, &ev))) return rc;
  return after ? reduce_global(ctx, slot, 1) : QDP_OK;
}

int blas_inner(qdp_ctx ctx, int prec, const void *a, const void *b, int nblk, int slot, bool host) {
  const Geom &g = ctx->geom;
  int rc;
  RedArgs R;
  bool after;
  if ((rc = red_setup(ctx, red_grid_max(g), slot, 2, true, host, &R, &after))) return rc;
  ProfEvent ev;
  prof_begin(ctx, QDP_PK_REDUCE, &ev);
  prof_work(ctx, QDP_PK_REDUCE, 96.0 * g.Vh * nblk, 48.0 * g.Vh * nblk * (prec == QDP_F64 ? 8 : 4));
  rc = blas_launch(ctx, K_INNER, prec, nblk, true, [&](int nb, int bs) {
    if (prec == QDP_F64)
      launch_k(ctx, inner_kernel<double>, nb, bs, g, (const T_<double> *)a, (const T_<double> *)b, nblk, R);
    else
      launch_k(ctx, inner_kernel<float>, nb, bs, g, (const T_<float> *)a, (const T_<float> *)b, nblk, R);
  });
  if (rc || (rc = prof_end(ctx, &ev))) return rc;
  return after ? reduce_global(ctx, slot, 2) : QDP_OK;
}

int reduce_global(qdp_ctx ctx, int slot, int n) {
  if (ctx->nranks == 1) return QDP_OK;
  if (ctx->peer) return peer_allreduce(ctx, slot, n);  // one kernel, deterministic (peer.cu)
  int rc;
  if (ctx->det_reduce) {
    if ((rc = comm_allgather_f64(ctx, ctx->red_result + slot, ctx->red_gather, n, ctx->stream))) return rc;
    ProfEvent ev;
    prof_begin(ctx, QDP_PK_REDUCE, &ev);
    rank_sum_kernel<<<1, 32, 0, ctx->stream>>>(ctx->red_gather, ctx->nranks, n, ctx->red_result, slot);
    return prof_end(ctx, &ev);
  }
  return comm_allreduce_f64(ctx, ctx->red_result + slot, n, ctx->stream);
}

__global__ void scalars_kernel(double *dst, const double *src, int n) {
  for (int i = threadIdx.x; i < n; i += blockDim.x) dst[i] = src[i];
}
template <typename R>
__global__ void __launch_bounds__(1024) copy_kernel(const Geom g, typename E<R>::T *d, const typename E<R>::T *s, int nblk) {
  pdl_enter();
  const size_t bs = (size_t)E<R>::NP * g.stride;
  for (int cb = blockIdx.x * blockDim.x + threadIdx.x; cb < g.Vh; cb += gridDim.x * blockDim.x)
    for (int b = 0; b < nblk; b++)
#pragma unroll
      for (int k = 0; k < E<R>::NP; k++) {
        const size_t i = b * bs + (size_t)k * g.stride + cb;
        st_stream(d + i, ld_stream(s + i));
      }
}

int read_scalars(qdp_ctx ctx, int slot, int n, double *out) {
  // host_pinned comes from cudaMallocHost: mapped, the same address on the device (UVA)
  scalars_kernel<<<1, 64, 0, ctx->stream>>>(ctx->host_pinned, ctx->red_result + slot, n);
  QDP_CUDA(ctx, cudaGetLastError());
  QDP_CUDA(ctx, cudaStreamSynchronize(ctx->stream));
  for (int i = 0; i < n; i++) out[i] = ((volatile double *)ctx->host_pinned)[i];
  return QDP_OK;
}

int copy_scalars(qdp_ctx ctx, int dst, int src, int n) {
  scalars_kernel<<<1, 64, 0, ctx->stream>>>(ctx->red_result + dst, ctx->red_result + src, n);
  QDP_CUDA(ctx, cudaGetLastError());
  return QDP_OK;
}

int copy_blocks(qdp_ctx ctx, int prec, void *dst, const void *src, int nblk) {
  const Geom &g = ctx->geom;
  ProfEvent ev;
  prof_begin(ctx, QDP_PK_BLAS, &ev);
  prof_work(ctx, QDP_PK_BLAS, 0.0, 48.0 * g.Vh * nblk * (prec == QDP_F64 ? 8 : 4));
  int rc = blas_launch(ctx, K_COPY, prec, nblk, false, [&](int nb, int bs) {
    if (prec == QDP_F64) launch_k(ctx, copy_kernel<double>, nb, bs, g, (T_<double> *)dst, (const T_<double> *)src, nblk);
    else launch_k(ctx, copy_kernel<float>, nb, bs, g, (T_<float> *)dst, (const T_<float> *)src, nblk);
  });
  if (rc) return rc;
  return prof_end(ctx, &ev);
}

int blas_axpy(qdp_ctx ctx, int prec, double ar, double ai, const void *x, void *y, int nblk) {
  const Geom &g = ctx->geom;
  ProfEvent ev;
  prof_begin(ctx, QDP_PK_BLAS, &ev);
  prof_work(ctx, QDP_PK_BLAS, 96.0 * g.Vh * nblk, 72.0 * g.Vh * nblk * (prec == QDP_F64 ? 8 : 4));
  int rc = blas_launch(ctx, K_AXPY, prec, nblk, false, [&](int nb, int bs) {
    if (prec == QDP_F64)
      launch_k(ctx, axpy_kernel<double>, nb, bs, g, ar, ai, (const T_<double> *)x, (T_<double> *)y, nblk);
    else
      launch_k(ctx, axpy_kernel<float>, nb, bs, g, (float)ar, (float)ai, (const T_<float> *)x, (T_<float> *)y, nblk);
  });
  if (rc) return rc;
  return prof_end(ctx, &ev);
}

int blas_xpay(qdp_ctx ctx, int prec, const void *x, double a, void *y, int nblk) {
  const Geom &g = ctx->geom;
  ProfEvent ev;
  prof_begin(ctx, QDP_PK_BLAS, &ev);
  prof_work(ctx, QDP_PK_BLAS, 48.0 * g.Vh * nblk, 72.0 * g.Vh * nblk * (prec == QDP_F64 ? 8 : 4));
  int rc = blas_launch(ctx, K_XPAY, prec, nblk, false, [&](int nb, int bs) {
    if (prec == QDP_F64) launch_k(ctx, xpay_kernel<double>, nb, bs, g, (const T_<double> *)x, a, (T_<double> *)y, nblk);
    else launch_k(ctx, xpay_kernel<float>, nb, bs, g, (const T_<float> *)x, (float)a, (T_<float> *)y, nblk);
  });
  if (rc) return rc;
  return prof_end(ctx, &ev);
}

int blas_scale_copy(qdp_ctx ctx, int prec, void *dst, const void *src, double a, int nblk) {
  const Geom &g = ctx->geom;
  ProfEvent ev;
  prof_begin(ctx, QDP_PK_BLAS, &ev);
  prof_work(ctx, QDP_PK_BLAS, 24.0 * g.Vh * nblk, 48.0 * g.Vh * nblk * (prec == QDP_F64 ? 8 : 4));
  int rc = blas_launch(ctx, K_SCALE, prec, nblk, false, [&](int nb, int bs) {
    if (prec == QDP_F64)
      launch_k(ctx, scale_copy_kernel<double>, nb, bs, g, (T_<double> *)dst, (const T_<double> *)src, a, nblk);
    else
      launch_k(ctx, scale_copy_kernel<float>, nb, bs, g, (T_<float> *)dst, (const T_<float> *)src, (float)a, nblk);
  });
  if (rc) return rc;
  return prof_end(ctx, &ev);
}

int blas_cg_update_r(qdp_ctx ctx, int prec, void *r, const void *q, int rho_slot, int pq_slot, int rr_slot,
                     const CgDev *cg) {
  const Geom &g = ctx->geom;
  int rc;
  RedArgs R;
  bool after;
  if ((rc = red_setup(ctx, red_grid_max(g), rr_slot, 1, true, false, &R, &after))) return rc;
  if (cg) {
    if (after) return set_error(ctx, QDP_EINVAL, "device-side CG needs the in-kernel global sum");
    R.has_cg = 1;
    R.cg = *cg;
  }
  ProfEvent ev;
  prof_begin(ctx, QDP_PK_BLAS, &ev);
  prof_work(ctx, QDP_PK_BLAS, 96.0 * g.Vh, 72.0 * g.Vh * (prec == QDP_F64 ? 8 : 4));
  rc = blas_launch(ctx, K_CGR, prec, 1, true, [&](int nb, int bs) {
    if (prec == QDP_F64)
      launch_k(ctx, cg_r_kernel<double>, nb, bs, g, (T_<double> *)r, (const T_<double> *)q, ctx->red_result,
                                                       rho_slot, pq_slot, R);
    else
      launch_k(ctx, cg_r_kernel<float>, nb, bs, g, (T_<float> *)r, (const T_<float> *)q, ctx->red_result,
                                                      rho_slot, pq_slot, R);
  });
  if (rc || (rc = prof_end(ctx, &ev))) return rc;
  return after ? reduce_global(ctx, rr_slot, 1) : QDP_OK;
}

int blas_cg_update_xp(qdp_ctx ctx, int prec, void *x, void *p, const void *r, int rho_slot, int pq_slot, int rr_slot,
                      bool update_p, const int *stop, int iter) {
  const Geom &g = ctx->geom;
  ProfEvent ev;
  prof_begin(ctx, QDP_PK_BLAS, &ev);
  prof_work(ctx, QDP_PK_BLAS, (update_p ? 96.0 : 48.0) * g.Vh,
            (update_p ? 120.0 : 72.0) * g.Vh * (prec == QDP_F64 ? 8 : 4));
#define QDPB_XP(Rt, U)                                                                                              \
  launch_k(ctx, cg_xp_kernel<Rt, U>, nb, bs, g, (T_<Rt> *)x, (T_<Rt> *)p, (const T_<Rt> *)r, ctx->red_result, \
                                                  rho_slot, pq_slot, rr_slot, stop, iter)
  int rc = blas_launch(ctx, update_p ? K_CGXP : K_CGXP0, prec, 1, false, [&](int nb, int bs) {
    if (prec == QDP_F64) { if (update_p) QDPB_XP(double, true); else QDPB_XP(double, false); }
    else { if (update_p) QDPB_XP(float, true); else QDPB_XP(float, false); }
  });
#undef QDPB_XP
  if (rc) return rc;
  return prof_end(ctx, &ev);
}

int blas_cg_update_p(qdp_ctx ctx, int prec, void *p, const void *r, int rho_slot, int rr_slot) {
  const Geom &g = ctx->geom;
  ProfEvent ev;
  prof_begin(ctx, QDP_PK_BLAS, &ev);
  prof_work(ctx, QDP_PK_BLAS, 48.0 * g.Vh, 72.0 * g.Vh * (prec == QDP_F64 ? 8 : 4));
  int rc = blas_launch(ctx, K_CGP, prec, 1, false, [&](int nb, int bs) {
    if (prec == QDP_F64)
      launch_k(ctx, cg_p_kernel<double>, nb, bs, g, (T_<double> *)p, (const T_<double> *)r, ctx->red_result, rho_slot, rr_slot);
    else
      launch_k(ctx, cg_p_kernel<float>, nb, bs, g, (T_<float> *)p, (const T_<float> *)r, ctx->red_result, rho_slot, rr_slot);
  });
  if (rc) return rc;
  return prof_end(ctx, &ev);
}

int blas_convert(qdp_ctx ctx, void *dst, int dst_prec, const void *src) {
  const Geom &g = ctx->geom;
  ProfEvent ev;
  prof_begin(ctx, QDP_PK_BLAS, &ev);
  prof_work(ctx, QDP_PK_BLAS, 0.0, 288.0 * g.Vh);  // 24 reals fp64 + 24 reals fp32 per site
  int rc = blas_launch(ctx, dst_prec == QDP_F32 ? K_CONV32 : K_CONV64, 0, 1, false, [&](int nb, int bs) {
    if (dst_prec == QDP_F32) launch_k(ctx, convert_kernel<true>, nb, bs, g, (double2 *)src, (float4 *)dst);
    else launch_k(ctx, convert_kernel<false>, nb, bs, g, (double2 *)dst, (float4 *)src);
  });
  if (rc) return rc;
  return prof_end(ctx, &ev);
}

int blas_accum_mixed(qdp_ctx ctx, void *y64, void *x32) {
  const Geom &g = ctx->geom;
  ProfEvent ev;
  prof_begin(ctx, QDP_PK_BLAS, &ev);
  prof_work(ctx, QDP_PK_BLAS, 24.0 * g.Vh, (2.0 * 24 * 8 + 2.0 * 24 * 4) * g.Vh);
  int rc = blas_launch(ctx, K_ACCUM, 0, 1, false, [&](int nb, int bs) {
    launch_k(ctx, accum_mixed_kernel, nb, bs, g, (double2 *)y64, (float4 *)x32);
  });
  if (rc) return rc;
  return prof_end(ctx, &ev);
}

}  // namespace qdpb
