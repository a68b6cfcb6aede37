// solver.cu -- even-odd preconditioned CGNR for M x = b, M = A - H/2 (readings R3, R12-R14;
// the linear solves of PAPER.md:31).  Host-driven loop; every vector operation is one of
// this library's kernels and the scalars alpha, beta live on the device, so an iteration
// needs exactly one device->host read (rho, for the convergence test).  Per iteration:
//   q = Mhat^dag Mhat p    4 fused dslash launches; the last also forms Re<p, q>
//   r -= alpha q, |r|^2    one pass (alpha = rho / Re<p,q> read on the device)
//   x += alpha p, p = r + beta p   one pass (beta = |r|^2 / rho)
//
//   Mhat v      = A_oo v - 1/4 H_oe A_ee^-1 H_eo v         (2 fused dslash launches)
//   Mhat^dag v  = gamma5 Mhat gamma5 v                       (gamma5 folded into the kernels)
//   bhat_o      = b_o + 1/2 H_oe A_ee^-1 b_e
//   x_e         = A_ee^-1 (b_e + 1/2 H_eo x_o)
// Wilson: A = (4 + m) 1, applied as scalars inside the dslash epilogues.
#include <math.h>

#include "internal.h"

namespace qdpb {

namespace {
enum { S_RHO = 0, S_PQ = 2, S_RR = 4 };

struct Op {
  qdp_ctx ctx;
  int prec;
  const void *U;
  bool rec12;          // U is QDP_GAUGE12
  const void *A_o;     // clover A on odd sites (nullptr: Wilson)
  const void *Ainv_e;  // clover A^-1 on even sites
  double diag;         // 4 + m
  void *t;             // even scratch block
};

// out_o = Mhat v_o  (dag: Mhat^dag); dot_x: also red_result[dot_slot] = Re<dot_x, out>
int apply_mhat(const Op &op, void *out, const void *v, bool dag, const void *dot_x = nullptr, int dot_slot = 0) {
  DslashArgs a = {};
  int rc;
  a.U = op.U;
  a.rec12 = op.rec12;
  // t_e = [A_ee^-1] H_eo [g5] v
  a.out = op.t;
  a.psi = v;
  a.parity = 0;
  a.g5_in = dag;
  a.b = 1.0;
  if (op.A_o) {
    a.epi = EPI_CLOVINV;
    a.clov = op.Ainv_e;
  } else {
    a.epi = EPI_PLAIN;
  }
  if ((rc = dslash(op.ctx, op.prec, a))) return rc;
  // out_o = A_oo v - 1/4 [g5] H_oe t   (Wilson: (4+m) v - 1/(4(4+m)) [g5] H_oe t)
  DslashArgs c = {};
  c.U = op.U;
  c.rec12 = op.rec12;
  c.out = out;
  c.psi = op.t;
  c.x = v;
  c.parity = 1;
  c.g5_out = dag;
  c.dot_x = dot_x;
  c.dot_slot = dot_slot;
  if (op.A_o) {
    c.epi = EPI_CLOVXPAY;
    c.clov = op.A_o;
    c.b = -0.25;
  } else {
    c.epi = EPI_XPAY;
    c.a = op.diag;
    c.b = -0.25 / op.diag;
  }
  return dslash(op.ctx, op.prec, c);
}
}  // namespace

int cg_solve(qdp_field x, const qdp_field b, const qdp_field U, const qdp_field A, const qdp_field Ainv, double mass,
             double tol, int maxit, int *iters_out, double *hist, int hist_cap, double *true_resid) {
  qdp_ctx ctx = x->ctx;
  const Geom &g = ctx->geom;
  const int prec = x->prec;
  const size_t blk = fermion_block_bytes(prec, g.stride);
  const bool clover = A != nullptr;
  const size_t cbk = parity_block_bytes(KIND_CLOVER, prec, g.stride);
  int rc;

  Op op;
  op.ctx = ctx;
  op.prec = prec;
  op.U = U->data;
  op.rec12 = U->kind == QDP_GAUGE12;
  op.A_o = clover ? (const char *)A->data + (A->subset == QDP_ALL ? cbk : 0) : nullptr;
  op.Ainv_e = clover ? Ainv->data : nullptr;
  op.diag = 4.0 + mass;

  // work: [t | r | p | q | mp | bh], persistent in the context (every block is fully
  // written before it is read, so no clearing is needed)
  if ((rc = ensure_cg_work(ctx, 6 * blk))) return rc;
  char *work = (char *)ctx->cg_work;
  op.t = work;
  void *r = work + blk, *p = work + 2 * blk, *q = work + 3 * blk, *mp = work + 4 * blk, *bh = work + 5 * blk;
  const char *b_e = (const char *)b->data, *b_o = b_e + blk;
  char *x_e = (char *)x->data, *x_o = x_e + blk;
  double *h = ctx->host_pinned;
  int k = 0, status = QDP_NOT_CONVERGED;
  double rho0 = 0.0, rho = 0.0;

  auto fail = [&](int e) { return e; };
  auto read_slot = [&](int slot, double *v) -> int {
    cudaError_t e = cudaMemcpyAsync(h, ctx->red_result + slot, sizeof(double), cudaMemcpyDeviceToHost, ctx->stream);
    if (e == cudaSuccess) e = cudaStreamSynchronize(ctx->stream);
    if (e != cudaSuccess) return cuda_check(ctx, e, "cg: read scalar");
    *v = h[0];
    return QDP_OK;
  };

  // bhat_o = b_o + 1/2 H_oe A_ee^-1 b_e
  if (clover) rc = clover_apply(ctx, prec, op.t, op.Ainv_e, b_e, 1);
  else rc = blas_scale_copy(ctx, prec, op.t, b_e, 1.0 / op.diag, 1);
  if (rc) return fail(rc);
  {
    DslashArgs a = {};
    a.U = op.U;
    a.rec12 = op.rec12;
    a.out = bh;
    a.psi = op.t;
    a.x = b_o;
    a.parity = 1;
    a.epi = EPI_XPAY;
    a.a = 1.0;
    a.b = 0.5;
    if ((rc = dslash(ctx, prec, a))) return fail(rc);
  }
  // x_o = 0 ; r = Mhat^dag bhat ; p = r ; rho0 = |r|^2
  if (cudaMemsetAsync(x_o, 0, blk, ctx->stream) != cudaSuccess) return fail(set_error(ctx, QDP_ECUDA, "cg: memset"));
  if ((rc = apply_mhat(op, r, bh, true))) return fail(rc);
  if (cudaMemcpyAsync(p, r, blk, cudaMemcpyDeviceToDevice, ctx->stream) != cudaSuccess)
    return fail(set_error(ctx, QDP_ECUDA, "cg: copy"));
  if ((rc = blas_norm2(ctx, prec, r, 1, S_RHO)) || (rc = reduce_global(ctx, S_RHO, 1)) || (rc = read_slot(S_RHO, &rho0)))
    return fail(rc);
  rho = rho0;
  if (hist_cap > 0 && hist) hist[0] = 1.0;
  if (rho0 == 0.0) status = QDP_OK;

  while (status == QDP_NOT_CONVERGED && k < maxit) {
    // q = Mhat^dag Mhat p, with Re<p, q> -> S_PQ fused into the last launch
    if ((rc = apply_mhat(op, mp, p, false))) return fail(rc);
    if ((rc = apply_mhat(op, q, mp, true, p, S_PQ))) return fail(rc);
    // r -= alpha q ; rr = |r|^2
    if ((rc = blas_cg_update_r(ctx, prec, r, q, S_RHO, S_PQ, S_RR))) return fail(rc);
    double rho_new;
    if ((rc = read_slot(S_RR, &rho_new))) return fail(rc);
    k++;
    if (hist && k < hist_cap) hist[k] = sqrt(rho_new / rho0);
    const bool done = rho_new <= tol * tol * rho0;
    // x += alpha p ; p = r + beta p (skipped on the last iteration)
    const bool last = done || k == maxit;
    if ((rc = blas_cg_update_xp(ctx, prec, x_o, p, r, S_RHO, S_PQ, S_RR, !last))) return fail(rc);
    if (done) {
      status = QDP_OK;
      rho = rho_new;
      break;
    }
    if (cudaMemcpyAsync(ctx->red_result + S_RHO, ctx->red_result + S_RR, sizeof(double), cudaMemcpyDeviceToDevice,
                        ctx->stream) != cudaSuccess)
      return fail(set_error(ctx, QDP_ECUDA, "cg: scalar copy"));
    rho = rho_new;
  }
  (void)rho;
  if (iters_out) *iters_out = k;

  // x_e = A_ee^-1 (b_e + 1/2 H_eo x_o)
  {
    DslashArgs a = {};
    a.U = op.U;
    a.rec12 = op.rec12;
    a.out = x_e;
    a.psi = x_o;
    a.x = b_e;
    a.parity = 0;
    if (clover) {
      a.epi = EPI_CLOVINV;
      a.clov = op.Ainv_e;
      a.a = 1.0;
      a.b = 0.5;
    } else {
      a.epi = EPI_XPAY;
      a.a = 1.0 / op.diag;
      a.b = 0.5 / op.diag;
    }
    if ((rc = dslash(ctx, prec, a))) return fail(rc);
  }

  if (true_resid) {
    // tmp = M x = A x - 1/2 H x  (per parity), then tmp = b - tmp ; |tmp| / |b|
    char *tmp = (char *)r;  // r | p are adjacent: a full two-block vector
    for (int par = 0; par < 2; par++) {
      DslashArgs a = {};
      a.U = op.U;
      a.rec12 = op.rec12;
      a.out = tmp + par * blk;
      a.psi = par == 0 ? x_o : x_e;
      a.x = par == 0 ? x_e : x_o;
      a.parity = par;
      a.b = -0.5;
      if (clover) {
        a.epi = EPI_CLOVXPAY;
        a.clov = (const char *)A->data + par * cbk;  // A covers ALL sites (checked in capi)
      } else {
        a.epi = EPI_XPAY;
        a.a = op.diag;
      }
      if ((rc = dslash(ctx, prec, a))) return fail(rc);
    }
    if ((rc = blas_xpay(ctx, prec, b->data, -1.0, tmp, 2))) return fail(rc);
    double rr, bb;
    if ((rc = blas_norm2(ctx, prec, tmp, 2, S_RR)) || (rc = reduce_global(ctx, S_RR, 1)) || (rc = read_slot(S_RR, &rr)))
      return fail(rc);
    if ((rc = blas_norm2(ctx, prec, b->data, 2, S_RR)) || (rc = reduce_global(ctx, S_RR, 1)) || (rc = read_slot(S_RR, &bb)))
      return fail(rc);
    *true_resid = bb > 0 ? sqrt(rr / bb) : 0.0;
  }
  QDP_CUDA(ctx, cudaStreamSynchronize(ctx->stream));
  return status;
}

}  // namespace qdpb
