// multishift.cu -- multi-shift CG: (Mhat^dag Mhat + sigma_i) x_i = phi_o for all shifts i from
// one Krylov space, the solver of the RHMC gauge generation the paper's production runs use
// (ref. [14]; reading R25 of DESIGN.md): plain CG on
// the base shift sigma_0 <= sigma_i, collinear shifted residuals r_i = zeta_i r:
//   zeta_i' = zeta_i zeta_i^old alpha^old / [alpha beta^old (zeta_i^old - zeta_i) + zeta_i^old alpha^old (1 + s_i alpha)]
//   alpha_i = alpha zeta_i' / zeta_i ; beta_i = beta (zeta_i' / zeta_i)^2
//   x_i += alpha_i p_i ; p_i = zeta_i' r + beta_i p_i         (shift i frozen once zeta_i'^2 rho <= tol^2 rho_0)
// Per iteration:
//   q = (Mhat^dag Mhat + sigma_0) p_0   4 fused dslash launches; the last adds sigma_0 p_0 and forms Re<p_0, q>
//   r -= alpha q, |r|^2                 one pass (cg_r kernel)
//   coefficients                        one thread: the zeta recurrences of every shift, in fp64, on the device
//   x_i += alpha_i p_i, p_i = ...       ONE pass over all active shifts (r read once per site)
// and one device->host read (rho and the active-shift counts).
#include <math.h>
#include <string.h>

#include "internal.h"

namespace qdpb {

namespace {
constexpr int MAXS = QDPB_MAX_SHIFTS;
enum { S_RHO = 0, S_PQ = 2, S_RR = 4, S_NX = 12, S_NP = 13 };

struct MsState {
  double sigma[MAXS], zeta[MAXS], zeta_old[MAXS];
  double ax[MAXS], zp[MAXS], bp[MAXS];  // this iteration's coefficients
  double alpha_old, beta_old;
  int active[MAXS], conv_iter[MAXS];
  int xupd[MAXS], pupd[MAXS];
};

struct MsPtrs {
  void *x[MAXS];
  void *p[MAXS];
};

// One thread; every product / quotient rounded separately (no FMA contraction), evaluated left
// to right as written in R25, so any plain IEEE implementation takes the same freeze decisions.
__global__ void ms_coeff_kernel(MsState *st, double *res, int n, int k, double tol2rho0, int last) {
  pdl_enter();
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  const double rho = res[S_RHO], rho_new = res[S_RR];
  const double alpha = __ddiv_rn(rho, res[S_PQ]);
  const double beta = __ddiv_rn(rho_new, rho);
  int nx = 0, np = 0;
  for (int i = 0; i < n; i++) {
    st->xupd[i] = st->pupd[i] = 0;
    if (!st->active[i]) continue;
    double zn, ai;
    if (i == 0) {
      zn = 1.0;
      ai = alpha;
    } else {
      const double si = __dsub_rn(st->sigma[i], st->sigma[0]);
      const double num = __dmul_rn(__dmul_rn(st->zeta[i], st->zeta_old[i]), st->alpha_old);
      const double d1 = __dmul_rn(__dmul_rn(alpha, st->beta_old), __dsub_rn(st->zeta_old[i], st->zeta[i]));
      const double d2 = __dmul_rn(__dmul_rn(st->zeta_old[i], st->alpha_old), __dadd_rn(1.0, __dmul_rn(si, alpha)));
      zn = __ddiv_rn(num, __dadd_rn(d1, d2));
      ai = __ddiv_rn(__dmul_rn(alpha, zn), st->zeta[i]);
    }
    st->xupd[i] = 1;
    st->ax[i] = ai;
    nx++;
    if (__dmul_rn(__dmul_rn(zn, zn), rho_new) <= tol2rho0) {
      st->active[i] = 0;
      st->conv_iter[i] = k;
      continue;
    }
    const double ratio = __ddiv_rn(zn, st->zeta[i]);
    st->bp[i] = __dmul_rn(__dmul_rn(beta, ratio), ratio);
    st->zp[i] = zn;
    st->pupd[i] = last ? 0 : 1;
    np += st->pupd[i];
    st->zeta_old[i] = st->zeta[i];
    st->zeta[i] = zn;
  }
  st->alpha_old = alpha;
  st->beta_old = beta;
  res[S_NX] = nx;
  res[S_NP] = np;
}

template <typename R> struct MsE;
template <> struct MsE<double> {
  using T = double2;
  static constexpr int NP = 12;
};
template <> struct MsE<float> {
  using T = float4;
  static constexpr int NP = 6;
};
template <typename T> __device__ __forceinline__ T axpy_(double a, T x, T y);
template <> __device__ __forceinline__ double2 axpy_(double a, double2 x, double2 y) {
  return make_double2(fma(a, x.x, y.x), fma(a, x.y, y.y));
}
template <> __device__ __forceinline__ float4 axpy_(double a, float4 x, float4 y) {
  const float f = (float)a;
  return make_float4(fmaf(f, x.x, y.x), fmaf(f, x.y, y.y), fmaf(f, x.z, y.z), fmaf(f, x.w, y.w));
}
template <typename T> __device__ __forceinline__ T lin_(double a, T x, double b, T y);  // a x + b y
template <> __device__ __forceinline__ double2 lin_(double a, double2 x, double b, double2 y) {
  return make_double2(a * x.x + b * y.x, a * x.y + b * y.y);
}
template <> __device__ __forceinline__ float4 lin_(double a, float4 x, double b, float4 y) {
  const float fa = (float)a, fb = (float)b;
  return make_float4(fa * x.x + fb * y.x, fa * x.y + fb * y.y, fa * x.z + fb * y.z, fa * x.w + fb * y.w);
}

// One thread per site: r read once; for every shift updated this iteration x_i += alpha_i p_i,
// then p_i = zeta_i' r + beta_i p_i.  The per-shift flags are uniform across the grid.
template <typename R>
__global__ void __launch_bounds__(256) ms_update_kernel(const Geom g, const MsPtrs P, const typename MsE<R>::T *r,
                                                        const MsState *st, int n) {
  pdl_enter();
  using T = typename MsE<R>::T;
  __shared__ double s_ax[MAXS], s_zp[MAXS], s_bp[MAXS];
  __shared__ int s_x[MAXS], s_p[MAXS];
  for (int i = threadIdx.x; i < n; i += blockDim.x) {
    s_x[i] = st->xupd[i];
    s_p[i] = st->pupd[i];
    s_ax[i] = st->ax[i];
    s_zp[i] = st->zp[i];
    s_bp[i] = st->bp[i];
  }
  __syncthreads();
  const int cb = blockIdx.x * blockDim.x + threadIdx.x;
  if (cb >= g.Vh) return;
#pragma unroll
  for (int k = 0; k < MsE<R>::NP; k++) {
    const size_t o = (size_t)k * g.stride + cb;
    const T rv = r[o];
    for (int i = 0; i < n; i++) {
      if (!s_x[i]) continue;
      T *xp = (T *)P.x[i] + o;
      T *pp = (T *)P.p[i] + o;
      const T pv = *pp;
      *xp = axpy_(s_ax[i], pv, *xp);
      if (s_p[i]) *pp = lin_(s_zp[i], rv, s_bp[i], pv);
    }
  }
}

int read_slots(qdp_ctx ctx, int slot, int n, double *v) { return read_scalars(ctx, slot, n, v); }
}  // namespace

// Mhat_op: the even-odd operator pieces of solver.cu
int mhat_apply(qdp_ctx ctx, const qdp_field U, const qdp_field A, const qdp_field Ainv, double mass, void *t, void *out,
               const void *v, bool dag, const void *dot_x, int dot_slot, double dot_shift);

int cg_solve_multishift(qdp_field *x, int n, const double *sigma, const qdp_field phi, const qdp_field U,
                        const qdp_field A, const qdp_field Ainv, double mass, double tol, int maxit, int *iters_out,
                        int *conv_iter, double *hist, int hist_cap, double *true_resid) {
  qdp_ctx ctx = phi->ctx;
  const Geom &g = ctx->geom;
  const int prec = phi->prec;
  const size_t blk = fermion_block_bytes(prec, g.stride);
  int rc;
  // work: [t | r | q | mp | p_0 .. p_{n-1}] + the coefficient state
  const size_t state_off = (4 + (size_t)n) * blk;
  if ((rc = ensure_cg_work(ctx, state_off + sizeof(MsState)))) return rc;
  char *work = (char *)ctx->cg_work;
  void *t = work, *r = work + blk, *q = work + 2 * blk, *mp = work + 3 * blk;
  MsState *st = (MsState *)(work + state_off);
  MsPtrs P;
  memset(&P, 0, sizeof(P));
  for (int i = 0; i < n; i++) {
    P.x[i] = (char *)x[i]->data + (x[i]->subset == QDP_ALL ? blk : 0);
    P.p[i] = work + (4 + i) * blk;
  }
  const char *phi_o = (const char *)phi->data + (phi->subset == QDP_ALL ? blk : 0);

  MsState h;
  memset(&h, 0, sizeof(h));
  for (int i = 0; i < n; i++) {
    h.sigma[i] = sigma[i];
    h.zeta[i] = h.zeta_old[i] = 1.0;
    h.active[i] = 1;
  }
  h.alpha_old = 1.0;
  h.beta_old = 0.0;
  QDP_CUDA(ctx, cudaMemcpyAsync(st, &h, sizeof(h), cudaMemcpyHostToDevice, ctx->stream));
  // x_i = 0 ; r = p_i = phi_o ; rho0 = |r|^2
  for (int i = 0; i < n; i++) {
    QDP_CUDA(ctx, cudaMemsetAsync(P.x[i], 0, blk, ctx->stream));
    if ((rc = copy_blocks(ctx, prec, P.p[i], phi_o, 1))) return rc;
  }
  if ((rc = copy_blocks(ctx, prec, r, phi_o, 1))) return rc;
  double rho0 = 0.0;
  if ((rc = blas_norm2(ctx, prec, r, 1, S_RHO)) ||
      (rc = read_slots(ctx, S_RHO, 1, &rho0)))
    return rc;
  if (hist_cap > 0 && hist) hist[0] = 1.0;
  int k = 0, status = rho0 == 0.0 ? QDP_OK : QDP_NOT_CONVERGED;
  const double tol2rho0 = tol * tol * rho0;
  const double fb = prec == QDP_F64 ? 8.0 : 4.0;

  while (status == QDP_NOT_CONVERGED && k < maxit) {
    if ((rc = mhat_apply(ctx, U, A, Ainv, mass, t, mp, P.p[0], false, nullptr, 0, 0.0))) return rc;
    if ((rc = mhat_apply(ctx, U, A, Ainv, mass, t, q, mp, true, P.p[0], S_PQ, sigma[0]))) return rc;
    if ((rc = blas_cg_update_r(ctx, prec, r, q, S_RHO, S_PQ, S_RR))) return rc;
    k++;
    launch_k(ctx, ms_coeff_kernel, 1, 32, st, ctx->red_result, n, k, tol2rho0, k == maxit ? 1 : 0);
    QDP_CUDA(ctx, cudaGetLastError());
    ProfEvent ev;
    prof_begin(ctx, QDP_PK_MSHIFT, &ev);
    if (prec == QDP_F64)
      launch_k(ctx, ms_update_kernel<double>, grid_for(g.Vh, 256), 256, g, P, (const double2 *)r, st, n);
    else
      launch_k(ctx, ms_update_kernel<float>, grid_for(g.Vh, 256), 256, g, P, (const float4 *)r, st, n);
    if ((rc = prof_end(ctx, &ev))) return rc;
    double s[10];  // slots S_RR .. S_NP
    if ((rc = read_slots(ctx, S_RR, S_NP - S_RR + 1, s))) return rc;
    const double rho_new = s[0], nx = s[S_NX - S_RR], np = s[S_NP - S_RR];
    // algorithmic work of the update pass: r once, x_i read + write, p_i read (+ write)
    prof_work(ctx, QDP_PK_MSHIFT, (48.0 * nx + 72.0 * np) * g.Vh, (24.0 + 72.0 * nx + 24.0 * np) * g.Vh * fb);
    if (hist && k < hist_cap) hist[k] = sqrt(rho_new / rho0);
    if (rho_new <= tol2rho0) status = QDP_OK;
    if ((rc = copy_scalars(ctx, S_RHO, S_RR, 1))) return rc;
  }
  if (iters_out) *iters_out = k;
  QDP_CUDA(ctx, cudaMemcpyAsync(&h, st, sizeof(h), cudaMemcpyDeviceToHost, ctx->stream));
  QDP_CUDA(ctx, cudaStreamSynchronize(ctx->stream));
  if (conv_iter)
    for (int i = 0; i < n; i++) conv_iter[i] = h.active[i] ? k : h.conv_iter[i];
  if (true_resid) {
    // |phi - (Mhat^dag Mhat + sigma_i) x_i| / |phi|: q = (..) x_i, q = phi - q
    for (int i = 0; i < n; i++) {
      if ((rc = mhat_apply(ctx, U, A, Ainv, mass, t, mp, P.x[i], false, nullptr, 0, 0.0))) return rc;
      if ((rc = mhat_apply(ctx, U, A, Ainv, mass, t, q, mp, true, P.x[i], S_PQ, sigma[i]))) return rc;
      if ((rc = blas_xpay(ctx, prec, phi_o, -1.0, q, 1))) return rc;
      double rr;
      if ((rc = blas_norm2(ctx, prec, q, 1, S_RR)) ||
          (rc = read_slots(ctx, S_RR, 1, &rr)))
        return rc;
      true_resid[i] = rho0 > 0 ? sqrt(rr / rho0) : 0.0;
    }
  }
  QDP_CUDA(ctx, cudaStreamSynchronize(ctx->stream));
  if ((rc = p2p_check(ctx))) return rc;
  return status;
}

}  // namespace qdpb
