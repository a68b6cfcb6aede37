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
//
// cg_solve_mixed: the same CGNR iterated in fp32 ("sloppy" copies of U, A, A^-1) with fp64
// reliable updates (the mixed-precision solvers of the paper's ref. [2]): whenever the fp32
// residual has dropped by `delta` below its maximum since the last update, the fp32 solution
// is accumulated into the fp64 x and the fp64 residual c - Mhat^dag Mhat x is recomputed.
// Convergence is only ever declared on an fp64 residual.
#include <math.h>
#include <stdlib.h>
#include <string.h>

#include <algorithm>
#include <vector>

#include "internal.h"

namespace qdpb {

namespace {
enum { S_RHO = 0, S_PQ = 2, S_RR = 4, S_TRUE = 6, S_RHO0 = 14 };

struct Op {
  qdp_ctx ctx;
  int prec;
  const void *U;
  bool rec12;          // U is QDP_GAUGE12
  bool h16 = false;    // U, A, Ainv and every vector in the 16-bit storage (cg_solve_mixed16)
  const void *A_o;     // clover A on odd sites (nullptr: Wilson)
  const void *Ainv_e;  // clover A^-1 on even sites
  double diag;         // 4 + m
  void *t;             // even scratch block
};

Op make_op(qdp_ctx ctx, const qdp_field U, const qdp_field A, const qdp_field Ainv, double mass, void *t) {
  const size_t cbk = parity_block_bytes(KIND_CLOVER, U->prec, ctx->geom.stride);
  Op op;
  op.ctx = ctx;
  op.prec = U->prec;
  op.U = U->data;
  op.rec12 = U->kind == QDP_GAUGE12;
  op.A_o = A ? (const char *)A->data + (A->subset == QDP_ALL ? cbk : 0) : nullptr;
  op.Ainv_e = A ? Ainv->data : nullptr;
  op.diag = 4.0 + mass;
  op.t = t;
  return op;
}

DslashArgs args(const Op &op) {
  DslashArgs a = {};
  a.U = op.U;
  a.rec12 = op.rec12;
  a.h16 = op.h16;
  return a;
}

// out_o = Mhat v_o  (dag: Mhat^dag); dot_x: also red_result[dot_slot] = Re<dot_x, out>
int apply_mhat(const Op &op, void *out, const void *v, bool dag, const void *dot_x = nullptr, int dot_slot = 0,
               double dot_shift = 0.0) {
  int rc;
  // t_e = [A_ee^-1] H_eo [g5] v
  DslashArgs a = args(op);
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
  DslashArgs c = args(op);
  c.out = out;
  c.psi = op.t;
  c.x = v;
  c.parity = 1;
  c.g5_out = dag;
  c.dot_x = dot_x;
  c.dot_slot = dot_slot;
  c.dot_shift = dot_shift;
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

int read_slot(qdp_ctx ctx, int slot, double *v) { return read_scalars(ctx, slot, 1, v); }
int copy_slot(qdp_ctx ctx, int dst, int src) { return copy_scalars(ctx, dst, src, 1); }

// bhat_o = b_o + 1/2 H_oe A_ee^-1 b_e
int prepare_source(const Op &op, void *bh, const char *b_e, const char *b_o) {
  int rc;
  if (op.A_o) rc = clover_apply(op.ctx, op.prec, op.t, op.Ainv_e, b_e, 1);
  else rc = blas_scale_copy(op.ctx, op.prec, op.t, b_e, 1.0 / op.diag, 1);
  if (rc) return rc;
  DslashArgs a = args(op);
  a.out = bh;
  a.psi = op.t;
  a.x = b_o;
  a.parity = 1;
  a.epi = EPI_XPAY;
  a.a = 1.0;
  a.b = 0.5;
  return dslash(op.ctx, op.prec, a);
}

// x_e = A_ee^-1 (b_e + 1/2 H_eo x_o), then (if asked) |b - M x| / |b| using `tmp2` (2 blocks)
int finish_solve(const Op &op, const qdp_field x, const qdp_field b, const qdp_field A, void *tmp2,
                 double *true_resid) {
  qdp_ctx ctx = op.ctx;
  const Geom &g = ctx->geom;
  const size_t blk = fermion_block_bytes(op.prec, g.stride);
  const size_t cbk = parity_block_bytes(KIND_CLOVER, op.prec, g.stride);
  char *x_e = (char *)x->data, *x_o = x_e + blk;
  const char *b_e = (const char *)b->data;
  int rc;
  {
    DslashArgs a = args(op);
    a.out = x_e;
    a.psi = x_o;
    a.x = b_e;
    a.parity = 0;
    if (op.A_o) {
      a.epi = EPI_CLOVINV;
      a.clov = op.Ainv_e;
      a.a = 1.0;
      a.b = 0.5;
    } else {
      a.epi = EPI_XPAY;
      a.a = 1.0 / op.diag;
      a.b = 0.5 / op.diag;
    }
    if ((rc = dslash(ctx, op.prec, a))) return rc;
  }
  if (!true_resid) return QDP_OK;
  // tmp = M x = A x - 1/2 H x  (per parity), then tmp = b - tmp ; |tmp| / |b|
  char *tmp = (char *)tmp2;
  for (int par = 0; par < 2; par++) {
    DslashArgs a = args(op);
    a.out = tmp + par * blk;
    a.psi = par == 0 ? x_o : x_e;
    a.x = par == 0 ? x_e : x_o;
    a.parity = par;
    a.b = -0.5;
    if (op.A_o) {
      a.epi = EPI_CLOVXPAY;
      a.clov = (const char *)A->data + par * cbk;  // A covers ALL sites (checked in capi)
    } else {
      a.epi = EPI_XPAY;
      a.a = op.diag;
    }
    if ((rc = dslash(ctx, op.prec, a))) return rc;
  }
  if ((rc = blas_xpay(ctx, op.prec, b->data, -1.0, tmp, 2))) return rc;
  double rr, bb;
  if ((rc = blas_norm2(ctx, op.prec, tmp, 2, S_RR)) || (rc = read_slot(ctx, S_RR, &rr)))
    return rc;
  if ((rc = blas_norm2(ctx, op.prec, b->data, 2, S_RR)) ||
      (rc = read_slot(ctx, S_RR, &bb)))
    return rc;
  *true_resid = bb > 0 ? sqrt(rr / bb) : 0.0;
  return QDP_OK;
}
}  // namespace

// out_o = Mhat v_o (dag: Mhat^dag v_o) for the multi-shift solver (multishift.cu); with dot_x:
// out += dot_shift * dot_x and red_result[dot_slot] = Re<dot_x, out>.  t: an even scratch block.
int mhat_apply(qdp_ctx ctx, const qdp_field U, const qdp_field A, const qdp_field Ainv, double mass, void *t, void *out,
               const void *v, bool dag, const void *dot_x, int dot_slot, double dot_shift) {
  return apply_mhat(make_op(ctx, U, A, Ainv, mass, t), out, v, dag, dot_x, dot_slot, dot_shift);
}

// Iterations per host round trip of cg_solve: all of them up to QDPB_CG_CHUNK (default 16) while
// the residual history says convergence is further away; fewer near the end (so few iterations
// are enqueued past the stopping one -- they run as no-ops); 1 = a host read every iteration.
static int cg_chunk(const double *hist_raw, int k, int maxit, double tol2rho0) {
  static const int cmax = getenv("QDPB_CG_CHUNK") ? std::max(1, atoi(getenv("QDPB_CG_CHUNK"))) : 16;
  int c = std::min(cmax, maxit - k);
  if (tol2rho0 > 0.0) {
    if (k < 2) return std::min(c, 2);
    const int m = std::min(k, 4);
    const double rate = pow(hist_raw[k] / hist_raw[k - m], 1.0 / m);  // per-iteration factor of |r|^2
    if (rate < 1.0 && rate > 0.0) {
      const double left = log(tol2rho0 / hist_raw[k]) / log(rate);
      c = std::min(c, std::max(1, (int)(0.75 * left)));
    } else {
      c = std::min(c, 2);
    }
  }
  return std::max(1, c);
}

int cg_solve(qdp_field x, const qdp_field b, const qdp_field U, const qdp_field A, const qdp_field Ainv, double mass,
             double tol, int maxit, int *iters_out, double *hist, int hist_cap, double *true_resid) {
  qdp_ctx ctx = x->ctx;
  const Geom &g = ctx->geom;
  const int prec = x->prec;
  const size_t blk = fermion_block_bytes(prec, g.stride);
  int rc;

  // work: [t | r | p | q | mp | bh], persistent in the context (every block is fully
  // written before it is read, so no clearing is needed)
  if ((rc = ensure_cg_work(ctx, 6 * blk))) return rc;
  // device-side bookkeeping: |r_k|^2 history in mapped pinned memory, the stop word on the device
  if (ctx->cg_hist_cap < maxit + 1) {
    if (ctx->cg_hist) {
      QDP_CUDA(ctx, cudaStreamSynchronize(ctx->stream));
      cudaFreeHost(ctx->cg_hist);
      ctx->cg_hist = nullptr;
      ctx->cg_hist_cap = 0;
    }
    const int cap = std::max(maxit + 1, 1024);
    QDP_CUDA(ctx, cudaHostAlloc((void **)&ctx->cg_hist, sizeof(double) * cap, cudaHostAllocMapped));
    ctx->cg_hist_cap = cap;
  }
  if (!ctx->cg_stop) QDP_CUDA(ctx, cudaMalloc((void **)&ctx->cg_stop, sizeof(int)));
  char *work = (char *)ctx->cg_work;
  const Op op = make_op(ctx, U, A, Ainv, mass, work);
  void *r = work + blk, *p = work + 2 * blk, *q = work + 3 * blk, *mp = work + 4 * blk, *bh = work + 5 * blk;
  const char *b_e = (const char *)b->data, *b_o = b_e + blk;
  char *x_o = (char *)x->data + blk;
  int k = 0, status = QDP_NOT_CONVERGED;
  double rho0 = 0.0;

  if ((rc = prepare_source(op, bh, b_e, b_o))) return rc;
  // x_o = 0 ; r = Mhat^dag bhat ; p = r ; rho0 = |r|^2
  QDP_CUDA(ctx, cudaMemsetAsync(x_o, 0, blk, ctx->stream));
  if ((rc = apply_mhat(op, r, bh, true))) return rc;
  if ((rc = copy_blocks(ctx, prec, p, r, 1))) return rc;
  if ((rc = blas_norm2(ctx, prec, r, 1, S_RHO)) || (rc = copy_scalars(ctx, S_RHO0, S_RHO, 1)) ||
      (rc = read_slot(ctx, S_RHO, &rho0)))
    return rc;
  if (hist_cap > 0 && hist) hist[0] = 1.0;
  if (rho0 == 0.0) status = QDP_OK;

  // Iterations run in chunks without host round trips: alpha, beta and |r|^2 stay on the device
  // (rho of iteration k in slot S_RHO / S_RR alternately), the final block of the r update
  // records |r_k|^2 and the stopping iteration (reduce.cuh CgDev), and the vector updates of a
  // later iteration do nothing.  The history and the stop are read once per chunk.
  volatile int *stop_host = (volatile int *)(ctx->host_pinned + 40);
  *stop_host = 0x7f7f7f7f;
  ctx->cg_hist[0] = rho0;  // |r_0|^2: the chunk predictor's first rate uses it
  QDP_CUDA(ctx, cudaMemsetAsync(ctx->cg_stop, 0x7f, sizeof(int), ctx->stream));
  const double tol2 = tol * tol;
  const int rs[2] = {S_RHO, S_RR};
  std::vector<double> snap_f((size_t)QDP_PK_COUNT * 17), snap_b((size_t)QDP_PK_COUNT * 17);
  while (status == QDP_NOT_CONVERGED && k < maxit) {
    const int c = cg_chunk(ctx->cg_hist, k, maxit, tol2 * rho0);
    snap_f.resize((size_t)QDP_PK_COUNT * (c + 1));
    snap_b.resize((size_t)QDP_PK_COUNT * (c + 1));
    for (int j = 1; j <= c; j++) {
      const int it = k + j;
      const int rho = rs[(it - 1) & 1], rr = rs[it & 1];
      // q = Mhat^dag Mhat p, with Re<p, q> -> S_PQ fused into the last launch
      // (after the stopping iteration these still run -- the predictor keeps that rare -- but the
      // two updates below do nothing, so x, r and the history stay those of the stopping one)
      if ((rc = apply_mhat(op, mp, p, false))) return rc;
      if ((rc = apply_mhat(op, q, mp, true, p, S_PQ))) return rc;
      // r -= alpha q ; |r|^2 ; records |r_it|^2 and whether it stops here
      const CgDev cg = {ctx->cg_hist, ctx->cg_stop, (int *)stop_host, ctx->red_result + S_RHO0, it, maxit, tol2};
      if ((rc = blas_cg_update_r(ctx, prec, r, q, rho, S_PQ, rr, &cg))) return rc;
      // x += alpha p ; p = r + beta p (not on the stopping iteration)
      if ((rc = blas_cg_update_xp(ctx, prec, x_o, p, r, rho, S_PQ, rr, it < maxit, ctx->cg_stop, it))) return rc;
      memcpy(&snap_f[(size_t)QDP_PK_COUNT * j], ctx->work_flops, sizeof(double) * QDP_PK_COUNT);
      memcpy(&snap_b[(size_t)QDP_PK_COUNT * j], ctx->work_bytes, sizeof(double) * QDP_PK_COUNT);
    }
    QDP_CUDA(ctx, cudaStreamSynchronize(ctx->stream));
    const int s = *stop_host;
    const int last = std::min(s, k + c);
    for (int it = k + 1; it <= last; it++)
      if (hist && it < hist_cap) hist[it] = sqrt(ctx->cg_hist[it] / rho0);
    if (s <= k + c) {  // stopped inside this chunk: the iterations after s did no work
      memcpy(ctx->work_flops, &snap_f[(size_t)QDP_PK_COUNT * (s - k)], sizeof(double) * QDP_PK_COUNT);
      memcpy(ctx->work_bytes, &snap_b[(size_t)QDP_PK_COUNT * (s - k)], sizeof(double) * QDP_PK_COUNT);
      if (s < maxit) prof_work(ctx, QDP_PK_BLAS, -48.0 * g.Vh, -48.0 * g.Vh * (prec == QDP_F64 ? 8 : 4));
      k = s;
      if (ctx->cg_hist[s] <= tol2 * rho0) status = QDP_OK;
      break;
    }
    k += c;
  }
  if (iters_out) *iters_out = k;
  if ((rc = finish_solve(op, x, b, A, r, true_resid))) return rc;  // r | p: a two-block scratch
  QDP_CUDA(ctx, cudaStreamSynchronize(ctx->stream));
  if ((rc = p2p_check(ctx))) return rc;
  return status;
}

int cg_solve_mixed(qdp_field x, const qdp_field b, const qdp_field U, const qdp_field A, const qdp_field Ainv,
                   const qdp_field Us, const qdp_field As, const qdp_field Ainvs, double mass, double tol, double delta,
                   int maxit, int *iters_out, int *nreliable_out, double *hist, int hist_cap, double *true_resid) {
  qdp_ctx ctx = x->ctx;
  const Geom &g = ctx->geom;
  const size_t b64 = fermion_block_bytes(QDP_F64, g.stride), b32 = fermion_block_bytes(QDP_F32, g.stride);
  int rc;
  // fp64 work: [t | r | c | mp | q | bh] ; fp32 work: [t | r | p | q | mp | x]
  if ((rc = ensure_cg_work(ctx, 6 * b64 + 6 * b32))) return rc;
  char *w64 = (char *)ctx->cg_work, *w32 = w64 + 6 * b64;
  const Op op = make_op(ctx, U, A, Ainv, mass, w64);
  const Op ops = make_op(ctx, Us, As, Ainvs, mass, w32);
  void *r = w64 + b64, *c = w64 + 2 * b64, *mp = w64 + 3 * b64, *q = w64 + 4 * b64, *bh = w64 + 5 * b64;
  void *rs = w32 + b32, *ps = w32 + 2 * b32, *qs = w32 + 3 * b32, *mps = w32 + 4 * b32, *xs = w32 + 5 * b32;
  const char *b_e = (const char *)b->data, *b_o = b_e + b64;
  char *x_o = (char *)x->data + b64;
  int k = 0, nrel = 0, status = QDP_NOT_CONVERGED;
  double rho0 = 0.0;

  // c = Mhat^dag bhat (fp64); x_o = 0; r = c; sloppy r_s = p_s = (float) r; x_s = 0
  if ((rc = prepare_source(op, bh, b_e, b_o))) return rc;
  if ((rc = apply_mhat(op, c, bh, true))) return rc;
  QDP_CUDA(ctx, cudaMemsetAsync(x_o, 0, b64, ctx->stream));
  QDP_CUDA(ctx, cudaMemsetAsync(xs, 0, b32, ctx->stream));
  if ((rc = copy_blocks(ctx, QDP_F64, r, c, 1))) return rc;
  if ((rc = blas_norm2(ctx, QDP_F64, r, 1, S_RHO)) ||
      (rc = read_slot(ctx, S_RHO, &rho0)))
    return rc;
  if ((rc = blas_convert(ctx, rs, QDP_F32, r))) return rc;
  if ((rc = copy_blocks(ctx, QDP_F32, ps, rs, 1))) return rc;
  if (hist_cap > 0 && hist) hist[0] = 1.0;
  if (rho0 == 0.0) status = QDP_OK;
  double maxr = sqrt(rho0);

  while (status == QDP_NOT_CONVERGED && k < maxit) {
    if ((rc = apply_mhat(ops, mps, ps, false))) return rc;
    if ((rc = apply_mhat(ops, qs, mps, true, ps, S_PQ))) return rc;
    if ((rc = blas_cg_update_r(ctx, QDP_F32, rs, qs, S_RHO, S_PQ, S_RR))) return rc;
    double rr;
    if ((rc = read_slot(ctx, S_RR, &rr))) return rc;
    k++;
    const bool reliable = sqrt(rr) < delta * maxr || rr <= tol * tol * rho0 || k == maxit;
    if (!reliable) {
      if (hist && k < hist_cap) hist[k] = sqrt(rr / rho0);
      if ((rc = blas_cg_update_xp(ctx, QDP_F32, xs, ps, rs, S_RHO, S_PQ, S_RR, true))) return rc;
      if ((rc = copy_slot(ctx, S_RHO, S_RR))) return rc;
      continue;
    }
    // reliable update: x += x_s (fp64), r = c - Mhat^dag Mhat x (fp64), r_s = (float) r
    if ((rc = blas_cg_update_xp(ctx, QDP_F32, xs, ps, rs, S_RHO, S_PQ, S_RR, false))) return rc;
    if ((rc = blas_accum_mixed(ctx, x_o, xs))) return rc;
    if ((rc = apply_mhat(op, mp, x_o, false)) || (rc = apply_mhat(op, q, mp, true))) return rc;
    if ((rc = copy_blocks(ctx, QDP_F64, r, c, 1))) return rc;
    if ((rc = blas_axpy(ctx, QDP_F64, -1.0, 0.0, q, r, 1))) return rc;
    double rt;
    if ((rc = blas_norm2(ctx, QDP_F64, r, 1, S_TRUE)) ||
        (rc = read_slot(ctx, S_TRUE, &rt)))
      return rc;
    nrel++;
    if (hist && k < hist_cap) hist[k] = sqrt(rt / rho0);
    maxr = sqrt(rt);
    if (rt <= tol * tol * rho0) {
      status = QDP_OK;
      break;
    }
    if (k == maxit) break;
    // p_s = r_s + beta p_s with beta = |r|^2 / rho (the fp64 residual norm), rho <- |r|^2
    if ((rc = blas_convert(ctx, rs, QDP_F32, r))) return rc;
    if ((rc = copy_slot(ctx, S_RR, S_TRUE))) return rc;
    if ((rc = blas_cg_update_p(ctx, QDP_F32, ps, rs, S_RHO, S_RR))) return rc;
    if ((rc = copy_slot(ctx, S_RHO, S_RR))) return rc;
  }
  if (iters_out) *iters_out = k;
  if (nreliable_out) *nreliable_out = nrel;
  if ((rc = finish_solve(op, x, b, A, mp, true_resid))) return rc;  // mp | q: a two-block scratch
  QDP_CUDA(ctx, cudaStreamSynchronize(ctx->stream));
  if ((rc = p2p_check(ctx))) return rc;
  return status;
}


// cg_solve_mixed16: cg_solve_mixed with a 16-bit sloppy level -- U (reconstruct-12), A_oo and
// A_ee^-1 converted to the 16-bit storage at the start of every call (so they can never be stale),
// the search direction p and the operator's vectors (t, Mhat p, Mhat^dag Mhat p) 16-bit with a
// per-site norm, the sloppy residual r and solution x fp32; fp64 reliable updates as before.
int cg_solve_mixed16(qdp_field x, const qdp_field b, const qdp_field U, const qdp_field A, const qdp_field Ainv,
                     double mass, double tol, double delta, int maxit, int *iters_out, int *nreliable_out,
                     double *hist, int hist_cap, double *true_resid) {
  qdp_ctx ctx = x->ctx;
  const Geom &g = ctx->geom;
  const size_t b64 = fermion_block_bytes(QDP_F64, g.stride), b32 = fermion_block_bytes(QDP_F32, g.stride);
  const size_t b16 = h16_fermion_bytes(g.stride), bu = h16_gauge_bytes(g.stride), bc = h16_clover_bytes(g.stride);
  int rc;
  // fp64 work: [t | r | c | mp | q | bh] ; fp32: [r | x] ; 16-bit: [t | p | q | mp] ; U16, A16_o, Ainv16_e
  const size_t need = 6 * b64 + 2 * b32 + 4 * b16 + bu + 2 * bc;
  if ((rc = ensure_cg_work(ctx, need))) return rc;
  char *w64 = (char *)ctx->cg_work, *w32 = w64 + 6 * b64, *w16 = w32 + 2 * b32;
  char *U16 = w16 + 4 * b16, *A16 = U16 + bu, *Ai16 = A16 + bc;
  const Op op = make_op(ctx, U, A, Ainv, mass, w64);
  Op ops = op;
  ops.prec = QDP_F32;
  ops.h16 = true;
  ops.rec12 = true;
  ops.U = U16;
  ops.t = w16;
  if (A) {
    const size_t cbk = parity_block_bytes(KIND_CLOVER, A->prec, g.stride);
    if ((rc = h16_gauge_from(ctx, U16, U)) ||
        (rc = h16_clover_from(ctx, A16, (const char *)A->data + (A->subset == QDP_ALL ? cbk : 0), A->prec)) ||
        (rc = h16_clover_from(ctx, Ai16, Ainv->data, Ainv->prec)))
      return rc;
    ops.A_o = A16;
    ops.Ainv_e = Ai16;
  } else if ((rc = h16_gauge_from(ctx, U16, U))) {
    return rc;
  }
  void *r = w64 + b64, *c = w64 + 2 * b64, *mp = w64 + 3 * b64, *q = w64 + 4 * b64, *bh = w64 + 5 * b64;
  void *rs = w32, *xs = w32 + b32;
  void *ps = w16 + b16, *qs = w16 + 2 * b16, *mps = w16 + 3 * b16;
  const char *b_e = (const char *)b->data, *b_o = b_e + b64;
  char *x_o = (char *)x->data + b64;
  int k = 0, nrel = 0, status = QDP_NOT_CONVERGED;
  double rho0 = 0.0;

  // c = Mhat^dag bhat (fp64); x_o = 0; r = c; r_s = (float) r; p_s = (16-bit) r_s; x_s = 0
  if ((rc = prepare_source(op, bh, b_e, b_o))) return rc;
  if ((rc = apply_mhat(op, c, bh, true))) return rc;
  QDP_CUDA(ctx, cudaMemsetAsync(x_o, 0, b64, ctx->stream));
  QDP_CUDA(ctx, cudaMemsetAsync(xs, 0, b32, ctx->stream));
  if ((rc = copy_blocks(ctx, QDP_F64, r, c, 1))) return rc;
  if ((rc = blas_norm2(ctx, QDP_F64, r, 1, S_RHO)) || (rc = read_slot(ctx, S_RHO, &rho0))) return rc;
  if ((rc = blas_convert(ctx, rs, QDP_F32, r)) || (rc = h16_from_f32(ctx, ps, rs))) return rc;
  if (hist_cap > 0 && hist) hist[0] = 1.0;
  if (rho0 == 0.0) status = QDP_OK;
  double maxr = sqrt(rho0);

  while (status == QDP_NOT_CONVERGED && k < maxit) {
    if ((rc = apply_mhat(ops, mps, ps, false))) return rc;
    if ((rc = apply_mhat(ops, qs, mps, true, ps, S_PQ))) return rc;
    if ((rc = h16_cg_r(ctx, rs, qs, S_RHO, S_PQ, S_RR))) return rc;
    double rr;
    if ((rc = read_slot(ctx, S_RR, &rr))) return rc;
    k++;
    const bool reliable = sqrt(rr) < delta * maxr || rr <= tol * tol * rho0 || k == maxit;
    if (!reliable) {
      if (hist && k < hist_cap) hist[k] = sqrt(rr / rho0);
      if ((rc = h16_cg_xp(ctx, xs, ps, rs, S_RHO, S_PQ, S_RR, true))) return rc;
      if ((rc = copy_slot(ctx, S_RHO, S_RR))) return rc;
      continue;
    }
    // reliable update: x += x_s (fp64), r = c - Mhat^dag Mhat x (fp64), r_s = (float) r
    if ((rc = h16_cg_xp(ctx, xs, ps, rs, S_RHO, S_PQ, S_RR, false))) return rc;
    if ((rc = blas_accum_mixed(ctx, x_o, xs))) return rc;
    if ((rc = apply_mhat(op, mp, x_o, false)) || (rc = apply_mhat(op, q, mp, true))) return rc;
    if ((rc = copy_blocks(ctx, QDP_F64, r, c, 1))) return rc;
    if ((rc = blas_axpy(ctx, QDP_F64, -1.0, 0.0, q, r, 1))) return rc;
    double rt;
    if ((rc = blas_norm2(ctx, QDP_F64, r, 1, S_TRUE)) || (rc = read_slot(ctx, S_TRUE, &rt))) return rc;
    nrel++;
    if (hist && k < hist_cap) hist[k] = sqrt(rt / rho0);
    maxr = sqrt(rt);
    if (rt <= tol * tol * rho0) {
      status = QDP_OK;
      break;
    }
    if (k == maxit) break;
    // p_s = r_s + beta p_s with beta = |r|^2 / rho (the fp64 residual norm), rho <- |r|^2
    if ((rc = blas_convert(ctx, rs, QDP_F32, r))) return rc;
    if ((rc = copy_slot(ctx, S_RR, S_TRUE))) return rc;
    if ((rc = h16_cg_p(ctx, ps, rs, S_RHO, S_RR))) return rc;
    if ((rc = copy_slot(ctx, S_RHO, S_RR))) return rc;
  }
  if (iters_out) *iters_out = k;
  if (nreliable_out) *nreliable_out = nrel;
  if ((rc = finish_solve(op, x, b, A, mp, true_resid))) return rc;  // mp | q: a two-block scratch
  QDP_CUDA(ctx, cudaStreamSynchronize(ctx->stream));
  if ((rc = p2p_check(ctx))) return rc;
  return status;
}

}  // namespace qdpb
