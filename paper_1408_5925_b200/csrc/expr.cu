// expr.cu -- the test functions of PAPER.md Table II (section VI) as fused site-parallel
// streaming kernels, one thread per site (the i_V = thread index mapping of PAPER.md:186),
// with the paper's thread-block autotuner (section VII):
//   lcm    U1 = U2 * U3            198 flop, 432 B/site (fp64)
//   upsi   psi1 = U1 * psi2        264 flop, 528 B
//   spmat  G1 = G2 * G3            480 flop, 768 B
//   matvec psi0 = U1 psi1 + U1 psi2  552 flop, 864 B by the paper's count (U1 "loaded twice"), 720 compulsory
//   clover psi0 = A * psi1         504 flop, 960 B
// Flops and bytes follow Table II's convention (cmul 6, cadd 2; every leaf + the store).
#include <functional>

#include <stdio.h>
#include <stdlib.h>

#include "internal.h"

namespace qdpb {

template <typename R> struct SMat { cx<R> m[16]; };

// colour matrix: fp64 double2[9][stride]; fp32 float4[4][stride] + float2[stride]
template <typename R> struct CMatView;
template <> struct CMatView<double> {
  double2 *p;
  int stride;
  __device__ __forceinline__ Link<double> load(int cb) const {
    Link<double> u;
#pragma unroll
    for (int k = 0; k < 9; k++) {
      double2 v = ld_stream(p + (size_t)k * stride + cb);
      u.m[k] = {v.x, v.y};
    }
    return u;
  }
  __device__ __forceinline__ void store(int cb, const Link<double> &u) const {
#pragma unroll
    for (int k = 0; k < 9; k++) st_stream(p + (size_t)k * stride + cb, make_double2(u.m[k].re, u.m[k].im));
  }
};
template <> struct CMatView<float> {
  float4 *p;
  int stride;
  __device__ __forceinline__ Link<float> load(int cb) const {
    Link<float> u;
#pragma unroll
    for (int k = 0; k < 4; k++) {
      float4 v = ld_stream(p + (size_t)k * stride + cb);
      u.m[2 * k] = {v.x, v.y};
      u.m[2 * k + 1] = {v.z, v.w};
    }
    float2 v = ld_stream((const float2 *)(p + (size_t)4 * stride) + cb);
    u.m[8] = {v.x, v.y};
    return u;
  }
  __device__ __forceinline__ void store(int cb, const Link<float> &u) const {
#pragma unroll
    for (int k = 0; k < 4; k++)
      st_stream(p + (size_t)k * stride + cb, make_float4(u.m[2 * k].re, u.m[2 * k].im, u.m[2 * k + 1].re, u.m[2 * k + 1].im));
    st_stream((float2 *)(p + (size_t)4 * stride) + cb, make_float2(u.m[8].re, u.m[8].im));
  }
};
// spin matrix: fp64 double2[16][stride]; fp32 float4[8][stride]
template <typename R> struct SMatView;
template <> struct SMatView<double> {
  double2 *p;
  int stride;
  __device__ __forceinline__ SMat<double> load(int cb) const {
    SMat<double> s;
#pragma unroll
    for (int k = 0; k < 16; k++) {
      double2 v = ld_stream(p + (size_t)k * stride + cb);
      s.m[k] = {v.x, v.y};
    }
    return s;
  }
  __device__ __forceinline__ void store(int cb, const SMat<double> &s) const {
#pragma unroll
    for (int k = 0; k < 16; k++) st_stream(p + (size_t)k * stride + cb, make_double2(s.m[k].re, s.m[k].im));
  }
};
template <> struct SMatView<float> {
  float4 *p;
  int stride;
  __device__ __forceinline__ SMat<float> load(int cb) const {
    SMat<float> s;
#pragma unroll
    for (int k = 0; k < 8; k++) {
      float4 v = ld_stream(p + (size_t)k * stride + cb);
      s.m[2 * k] = {v.x, v.y};
      s.m[2 * k + 1] = {v.z, v.w};
    }
    return s;
  }
  __device__ __forceinline__ void store(int cb, const SMat<float> &s) const {
#pragma unroll
    for (int k = 0; k < 8; k++)
      st_stream(p + (size_t)k * stride + cb, make_float4(s.m[2 * k].re, s.m[2 * k].im, s.m[2 * k + 1].re, s.m[2 * k + 1].im));
  }
};

// colour matrix x the colour vector of every spin
template <typename R>
__device__ __forceinline__ Spinor<R> mul_spinor(const Link<R> &u, const Spinor<R> &s) {
  Spinor<R> o;
#pragma unroll
  for (int sp = 0; sp < 4; sp++)
#pragma unroll
    for (int a = 0; a < 3; a++) {
      cx<R> acc = cmul(u.m[3 * a], s.c[3 * sp]);
      acc = cmadd(u.m[3 * a + 1], s.c[3 * sp + 1], acc);
      acc = cmadd(u.m[3 * a + 2], s.c[3 * sp + 2], acc);
      o.c[3 * sp + a] = acc;
    }
  return o;
}

struct ExprArgs {
  void *out;
  const void *a, *b, *c;
  int n_blocks;       // parity blocks processed (1 or 2)
  size_t out_blk, a_blk, b_blk, c_blk;  // bytes between consecutive parity blocks of each operand
};

// One thread per (parity block, site).  EXPR selects the Table II function.
template <typename R, int EXPR>
__global__ void expr_kernel(const Geom g, const ExprArgs e) {
  const long i = (long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= (long)e.n_blocks * g.Vh) return;
  const int blk = (int)(i / g.Vh), cb = (int)(i % g.Vh);
  char *out = (char *)e.out + blk * e.out_blk;
  const char *a = (const char *)e.a + blk * e.a_blk, *b = (const char *)e.b + blk * e.b_blk;
  using FV = FermView<R>;
  if (EXPR == QDP_EXPR_LCM) {
    const Link<R> x = CMatView<R>{(decltype(CMatView<R>::p))a, g.stride}.load(cb);
    const Link<R> y = CMatView<R>{(decltype(CMatView<R>::p))b, g.stride}.load(cb);
    Link<R> z;
#pragma unroll
    for (int r = 0; r < 3; r++)
#pragma unroll
      for (int col = 0; col < 3; col++) {
        cx<R> acc = cmul(x.m[3 * r], y.m[col]);
        acc = cmadd(x.m[3 * r + 1], y.m[3 + col], acc);
        acc = cmadd(x.m[3 * r + 2], y.m[6 + col], acc);
        z.m[3 * r + col] = acc;
      }
    CMatView<R>{(decltype(CMatView<R>::p))out, g.stride}.store(cb, z);
  } else if (EXPR == QDP_EXPR_UPSI || EXPR == QDP_EXPR_MATVEC || EXPR == QDP_EXPR_ADJ_UPSI) {
    Link<R> u = CMatView<R>{(decltype(CMatView<R>::p))a, g.stride}.load(cb);
    if (EXPR == QDP_EXPR_ADJ_UPSI) {  // u <- u^dag
      Link<R> t = u;
#pragma unroll
      for (int r = 0; r < 3; r++)
#pragma unroll
        for (int col = 0; col < 3; col++) u.m[3 * r + col] = {t.m[3 * col + r].re, -t.m[3 * col + r].im};
    }
    Spinor<R> o = mul_spinor(u, FV{(decltype(FV::p))b, g.stride}.load_stream(cb));
    if (EXPR == QDP_EXPR_MATVEC) {
      const char *c = (const char *)e.c + blk * e.c_blk;
      const Spinor<R> o2 = mul_spinor(u, FV{(decltype(FV::p))c, g.stride}.load_stream(cb));
#pragma unroll
      for (int k = 0; k < 12; k++) o.c[k] = o.c[k] + o2.c[k];
    }
    FV{(decltype(FV::p))out, g.stride}.store(cb, o);
  } else if (EXPR == QDP_EXPR_SPMAT) {
    const SMat<R> x = SMatView<R>{(decltype(SMatView<R>::p))a, g.stride}.load(cb);
    const SMat<R> y = SMatView<R>{(decltype(SMatView<R>::p))b, g.stride}.load(cb);
    SMat<R> z;
#pragma unroll
    for (int r = 0; r < 4; r++)
#pragma unroll
      for (int col = 0; col < 4; col++) {
        cx<R> acc = cmul(x.m[4 * r], y.m[col]);
#pragma unroll
        for (int k = 1; k < 4; k++) acc = cmadd(x.m[4 * r + k], y.m[4 * k + col], acc);
        z.m[4 * r + col] = acc;
      }
    SMatView<R>{(decltype(SMatView<R>::p))out, g.stride}.store(cb, z);
  } else {  // CLOVER
    const CloverView<R> A{(decltype(CloverView<R>::p))a, g.stride};
    FV{(decltype(FV::p))out, g.stride}.store(cb, clover_mul(A, cb, FV{(decltype(FV::p))b, g.stride}.load_stream(cb)));
  }
}

// Table II accounting (flops, bytes in the paper's convention) per site, fp64 bytes
static void expr_work(int expr, double &flops, double &reals) {
  switch (expr) {
    case QDP_EXPR_LCM: flops = 198; reals = 54; break;        // 3 colour matrices
    case QDP_EXPR_UPSI:
    case QDP_EXPR_ADJ_UPSI: flops = 264; reals = 18 + 48; break;  // U, psi, psi
    case QDP_EXPR_SPMAT: flops = 480; reals = 96; break;      // 3 spin matrices
    case QDP_EXPR_MATVEC: flops = 552; reals = 18 + 72; break;  // U once (compulsory), 3 fermions
    default: flops = 504; reals = 72 + 48; break;             // clover, 2 fermions
  }
}

template <typename R, int EXPR>
static cudaError_t launch(qdp_ctx ctx, const ExprArgs &e, int block) {
  const Geom &g = ctx->geom;
  const long n = (long)e.n_blocks * g.Vh;
  // A launch with more threads than the kernel's register budget allows fails with
  // cudaErrorLaunchOutOfResources; report that outcome without issuing the failing launch.
  static int max_threads = 0;
  if (!max_threads) {
    cudaFuncAttributes attr;
    if (cudaFuncGetAttributes(&attr, expr_kernel<R, EXPR>) != cudaSuccess) return cudaGetLastError();
    max_threads = attr.maxThreadsPerBlock;
  }
  if (block > max_threads) return cudaErrorLaunchOutOfResources;
  expr_kernel<R, EXPR><<<(unsigned)((n + block - 1) / block), block, 0, ctx->stream>>>(g, e);
  return cudaGetLastError();
}

template <typename R>
static cudaError_t launch_expr(qdp_ctx ctx, int expr, const ExprArgs &e, int block) {
  switch (expr) {
    case QDP_EXPR_LCM: return launch<R, QDP_EXPR_LCM>(ctx, e, block);
    case QDP_EXPR_UPSI: return launch<R, QDP_EXPR_UPSI>(ctx, e, block);
    case QDP_EXPR_ADJ_UPSI: return launch<R, QDP_EXPR_ADJ_UPSI>(ctx, e, block);
    case QDP_EXPR_SPMAT: return launch<R, QDP_EXPR_SPMAT>(ctx, e, block);
    case QDP_EXPR_MATVEC: return launch<R, QDP_EXPR_MATVEC>(ctx, e, block);
    default: return launch<R, QDP_EXPR_CLOVER>(ctx, e, block);
  }
}

static long tune_key(int expr, int prec, long sites) { return ((long)expr * 2 + prec) * (1L << 40) + sites; }

void tune_release(qdp_ctx ctx) {
  for (auto &kv : ctx->tune) {
    if (kv.second.a) cudaEventDestroy(kv.second.a);
    if (kv.second.b) cudaEventDestroy(kv.second.b);
  }
  ctx->tune.clear();
}

// start at the largest block (1024), halve while the launch fails; once a launch
// succeeded, every further payload launch probes the next smaller block until its time exceeds
// the best seen by more than 33%; then the best block is used for good.  Only payload launches.
// (A launch "fails" when the block exceeds the kernel's maxThreadsPerBlock -- checked up front
// by `go`, which returns cudaErrorLaunchOutOfResources without launching.)
// Both tuners below time a candidate on its SECOND payload launch (the first one of a kernel may
// include its lazy module load and cold caches); every launch is a payload launch.
static bool tune_log() {  // QDPB_TUNE_LOG=1: report every tuner decision on stderr (measurements)
  static const bool on = getenv("QDPB_TUNE_LOG") && atoi(getenv("QDPB_TUNE_LOG"));
  return on;
}

int tuned_launch(qdp_ctx ctx, long key, const std::function<cudaError_t(int)> &go) {
  if (!ctx->autotune) {
    cudaError_t err = go(128);
    return err != cudaSuccess ? cuda_check(ctx, err, "tuned launch") : QDP_OK;
  }
  Tune &t = ctx->tune[key];
  if (!t.a) {
    cudaEventCreate(&t.a);
    cudaEventCreate(&t.b);
  }
  if (t.pending) {  // time of the previous payload launch at t.block
    // never wait for it: a synchronisation here would leave the GPU idle before the next probe and
    // put the host's launch latency into its timing; until the events complete, launch untimed
    const cudaError_t qe = cudaEventQuery(t.b);
    if (qe == cudaErrorNotReady) {
      const cudaError_t err = go(t.block);
      return err != cudaSuccess ? cuda_check(ctx, err, "tuned launch") : QDP_OK;
    }
    QDP_CUDA(ctx, qe);
    float ms = 0.f;
    QDP_CUDA(ctx, cudaEventElapsedTime(&ms, t.a, t.b));
    t.pending = false;
    if (t.best_block == 0 || ms < t.best_ms) {
      t.best_ms = ms;
      t.best_block = t.block;
    }
    if (ms > 1.33f * t.best_ms || t.block <= 32) {
      t.state = 2;
      t.block = t.best_block;
      if (tune_log()) fprintf(stderr, "qdpb tune: key %lx -> block %d (%.2f us)\n", key, t.block, 1e3 * t.best_ms);
    } else {
      t.block /= 2;
      t.warm = true;
    }
  }
  cudaError_t err = cudaSuccess;
  const bool timed = t.state != 2 && !t.warm;
  if (timed) QDP_CUDA(ctx, cudaEventRecord(t.a, ctx->stream));
  for (;;) {
    err = go(t.block);
    if (err == cudaSuccess || t.state != 0 || t.block <= 32) break;
    t.block /= 2;  // launch failed (too many resources at this block size): halve and retry
  }
  if (err != cudaSuccess) return cuda_check(ctx, err, "tuned launch");
  if (t.state != 2) {
    if (timed) {
      QDP_CUDA(ctx, cudaEventRecord(t.b, ctx->stream));
      t.pending = true;
    }
    t.warm = !timed && t.warm ? false : t.warm;
    t.state = 1;
  }
  return QDP_OK;
}

// The same rule over an ordered list of launch variants (index 0 = the most threads per block):
// variant 0 first (the next one if it fails to launch), then probe 1, 2, ... on later payload
// launches until one is 33% slower than the best or the list ends; keep the best.  For kernels
// whose output does not depend on its old contents (go() may run twice): a probing call launches
// its candidate twice back to back and times the second launch only -- warm, and with no host
// launch latency inside the timed interval (a few-microsecond kernel would otherwise be judged
// by the host's jitter).
int tuned_variant(qdp_ctx ctx, long key, int nvar, const std::function<cudaError_t(int)> &go) {
  Tune &t = ctx->tune[key | (1L << 61)];  // disjoint from expression (< 2^50) and jit (bit 62) keys
  if (!t.a) {
    cudaEventCreate(&t.a);
    cudaEventCreate(&t.b);
    t.block = 0;
  }
  if (t.pending) {
    const cudaError_t qe = cudaEventQuery(t.b);  // never wait (see tuned_launch)
    if (qe == cudaErrorNotReady) {
      const cudaError_t err = go(t.block);
      return err != cudaSuccess ? cuda_check(ctx, err, "tuned launch") : QDP_OK;
    }
    QDP_CUDA(ctx, qe);
    float ms = 0.f;
    QDP_CUDA(ctx, cudaEventElapsedTime(&ms, t.a, t.b));
    t.pending = false;
    if (t.best_ms == 0.f || ms < t.best_ms) {
      t.best_ms = ms;
      t.best_block = t.block;
    }
    if (ms > 1.33f * t.best_ms || t.block + 1 >= nvar) {
      t.state = 2;
      t.block = t.best_block;
      if (tune_log()) fprintf(stderr, "qdpb tune: dslash key %lx -> variant %d (%.2f us)\n", key, t.block, 1e3 * t.best_ms);
    } else {
      t.block++;
    }
  }
  cudaError_t err;
  for (;;) {
    err = go(t.block);
    if (err == cudaSuccess || t.state != 0 || t.block + 1 >= nvar) break;
    t.block++;  // could not launch (resources): the next variant
  }
  if (err != cudaSuccess) return cuda_check(ctx, err, "tuned launch");
  if (t.state != 2) {  // probing: the timed repeat
    QDP_CUDA(ctx, cudaEventRecord(t.a, ctx->stream));
    if ((err = go(t.block)) != cudaSuccess) return cuda_check(ctx, err, "tuned launch");
    QDP_CUDA(ctx, cudaEventRecord(t.b, ctx->stream));
    t.pending = true;
    t.state = 1;
  }
  return QDP_OK;
}

// One Table II expression: the paper's autotuner on its payload launches.
int expr_eval(qdp_ctx ctx, int expr, qdp_field out, const qdp_field a, const qdp_field b, const qdp_field c) {
  const Geom &g = ctx->geom;
  const int prec = out->prec;
  const size_t fb = parity_block_bytes(out->kind, prec, g.stride);
  ExprArgs e;
  e.out = out->data;
  e.a = a->data;
  e.b = b->data;
  e.c = c ? c->data : nullptr;
  e.n_blocks = out->subset == QDP_ALL ? 2 : 1;
  // operands that are QDP_ALL while the output is one parity: start at that parity's block
  auto base = [&](const qdp_field f) -> const char * {
    if (!f) return nullptr;
    if (f->subset == QDP_ALL && out->subset != QDP_ALL)
      return (const char *)f->data + out->subset * parity_block_bytes(f->kind, prec, g.stride);
    return (const char *)f->data;
  };
  e.a = base(a);
  e.b = base(b);
  e.c = base(c);
  e.out_blk = fb;
  e.a_blk = parity_block_bytes(a->kind, prec, g.stride);
  e.b_blk = parity_block_bytes(b->kind, prec, g.stride);
  e.c_blk = c ? parity_block_bytes(c->kind, prec, g.stride) : 0;

  double flops, reals;
  expr_work(expr, flops, reals);
  const long sites = (long)e.n_blocks * g.Vh;
  auto go = [&](int block) {
    return prec == QDP_F64 ? launch_expr<double>(ctx, expr, e, block) : launch_expr<float>(ctx, expr, e, block);
  };

  ProfEvent ev;
  prof_begin(ctx, QDP_PK_BLAS, &ev);
  prof_work(ctx, QDP_PK_BLAS, flops * sites, reals * sites * (prec == QDP_F64 ? 8 : 4));
  const int rc = tuned_launch(ctx, tune_key(expr, prec, sites), go);
  if (rc) {
    prof_end(ctx, &ev);
    return rc;
  }
  return prof_end(ctx, &ev);
}

}  // namespace qdpb
