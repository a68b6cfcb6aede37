// clover.cu -- clover term (section VI-A, eq. (1); reading R10):
//   A(x) = (4 + m) + 1/4 c_SW sum_{mu,nu} sigma_mu,nu F_mu,nu(x)
//        = (4 + m) + c_SW/2 sum_{mu<nu} sigma_mu,nu (x) F_mu,nu(x),
//   sigma_mu,nu = [gamma_mu, gamma_nu]/(2i),  F = traceless part of (Q - Q^dag)/(8i),
// Q the sum of the four clover-leaf plaquettes.  In the chiral (DeGrand-Rossi) basis every
// sigma_mu,nu is block diagonal, so A splits into two Hermitian 6x6 blocks (spins {0,1} and
// {2,3}), stored as 6 real diagonal + 15 complex strictly-lower entries
// (PAPER.md:228-230).  The 2x2 spin blocks of sigma used below:
//   block 0: s01 = diag(-1,1), s23 = diag(1,-1), s02 = s13 = [[0,i],[-i,0]], s03 = [[0,1],[1,0]], s12 = -[[0,1],[1,0]]
//   block 1: s01 = diag(-1,1), s23 = diag(-1,1), s02 = [[0,i],[-i,0]], s13 = -[[0,i],[-i,0]], s03 = s12 = -[[0,1],[1,0]]
// Build (setup, once per gauge field) computes in fp64 and inverts each block by LDL^dag.
// Apply (per CG iteration) is the two packed matvecs, 504 flop / site (Table II "clover").
#include "internal.h"

namespace qdpb {

struct M3 { double2 m[9]; };
template <typename R, int REC> struct ShiftSet { GaugeView<R, REC> s[7]; };

__device__ __forceinline__ double2 c_add(double2 a, double2 b) { return make_double2(a.x + b.x, a.y + b.y); }
__device__ __forceinline__ double2 c_sub(double2 a, double2 b) { return make_double2(a.x - b.x, a.y - b.y); }
__device__ __forceinline__ double2 c_mul(double2 a, double2 b) { return make_double2(a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x); }
__device__ __forceinline__ double2 c_conj(double2 a) { return make_double2(a.x, -a.y); }
__device__ __forceinline__ double2 c_i(double2 a) { return make_double2(-a.y, a.x); }

__device__ __forceinline__ M3 m3_mul(const M3 &a, const M3 &b) {
  M3 r;
#pragma unroll
  for (int i = 0; i < 3; i++)
#pragma unroll
    for (int j = 0; j < 3; j++) {
      double2 s = c_mul(a.m[3 * i], b.m[j]);
      s = c_add(s, c_mul(a.m[3 * i + 1], b.m[3 + j]));
      s = c_add(s, c_mul(a.m[3 * i + 2], b.m[6 + j]));
      r.m[3 * i + j] = s;
    }
  return r;
}
__device__ __forceinline__ M3 m3_dag(const M3 &a) {
  M3 r;
#pragma unroll
  for (int i = 0; i < 3; i++)
#pragma unroll
    for (int j = 0; j < 3; j++) r.m[3 * i + j] = c_conj(a.m[3 * j + i]);
  return r;
}

template <typename GV>
__device__ __forceinline__ M3 link_at(const Geom &g, const GV &U, const int c0[4], int mu, int d1, int a, int d2, int b) {
  int c[4] = {c0[0], c0[1], c0[2], c0[3]};
  c[d1] = (c[d1] + a + g.L[d1]) % g.L[d1];
  c[d2] = (c[d2] + b + g.L[d2]) % g.L[d2];
  const auto l = U.load(mu, coords_parity(c), coords_cb(g, c));
  M3 r;
#pragma unroll
  for (int k = 0; k < 9; k++) r.m[k] = make_double2((double)l.m[k].re, (double)l.m[k].im);
  return r;
}

// Hermitian traceless F_mu,nu at c (reading R10)
template <typename GV>
__device__ M3 field_strength(const Geom &g, const GV &U, const int c[4], int mu, int nu) {
  M3 q, t;
  // U_mu(x) U_nu(x+mu) U_mu(x+nu)^dag U_nu(x)^dag
  q = m3_mul(m3_mul(link_at(g, U, c, mu, mu, 0, nu, 0), link_at(g, U, c, nu, mu, 1, nu, 0)),
             m3_mul(m3_dag(link_at(g, U, c, mu, mu, 0, nu, 1)), m3_dag(link_at(g, U, c, nu, mu, 0, nu, 0))));
  // U_nu(x) U_mu(x-mu+nu)^dag U_nu(x-mu)^dag U_mu(x-mu)
  t = m3_mul(m3_mul(link_at(g, U, c, nu, mu, 0, nu, 0), m3_dag(link_at(g, U, c, mu, mu, -1, nu, 1))),
             m3_mul(m3_dag(link_at(g, U, c, nu, mu, -1, nu, 0)), link_at(g, U, c, mu, mu, -1, nu, 0)));
#pragma unroll
  for (int k = 0; k < 9; k++) q.m[k] = c_add(q.m[k], t.m[k]);
  // U_mu(x-mu)^dag U_nu(x-mu-nu)^dag U_mu(x-mu-nu) U_nu(x-nu)
  t = m3_mul(m3_mul(m3_dag(link_at(g, U, c, mu, mu, -1, nu, 0)), m3_dag(link_at(g, U, c, nu, mu, -1, nu, -1))),
             m3_mul(link_at(g, U, c, mu, mu, -1, nu, -1), link_at(g, U, c, nu, mu, 0, nu, -1)));
#pragma unroll
  for (int k = 0; k < 9; k++) q.m[k] = c_add(q.m[k], t.m[k]);
  // U_nu(x-nu)^dag U_mu(x-nu) U_nu(x-nu+mu) U_mu(x)^dag
  t = m3_mul(m3_mul(m3_dag(link_at(g, U, c, nu, mu, 0, nu, -1)), link_at(g, U, c, mu, mu, 0, nu, -1)),
             m3_mul(link_at(g, U, c, nu, mu, 1, nu, -1), m3_dag(link_at(g, U, c, mu, mu, 0, nu, 0))));
#pragma unroll
  for (int k = 0; k < 9; k++) q.m[k] = c_add(q.m[k], t.m[k]);
  // F = (Q - Q^dag) / (8 i)  = -i (Q - Q^dag) / 8
  M3 f;
#pragma unroll
  for (int i = 0; i < 3; i++)
#pragma unroll
    for (int j = 0; j < 3; j++) {
      double2 d = c_sub(q.m[3 * i + j], c_conj(q.m[3 * j + i]));
      f.m[3 * i + j] = make_double2(d.y / 8.0, -d.x / 8.0);
    }
  const double tr = (f.m[0].x + f.m[4].x + f.m[8].x) / 3.0;  // trace is real
  f.m[0].x -= tr;
  f.m[4].x -= tr;
  f.m[8].x -= tr;
  return f;
}

template <typename R> __device__ __forceinline__ void store_block(char *base, int stride, int b, const double d[6], const double2 off[15]);
template <> __device__ __forceinline__ void store_block<double>(char *base, int stride, int b, const double d[6], const double2 off[15]) {
  double2 *q = (double2 *)base + (size_t)18 * b * stride;
  for (int k = 0; k < 3; k++) q[(size_t)k * stride] = make_double2(d[2 * k], d[2 * k + 1]);
  for (int k = 0; k < 15; k++) q[(size_t)(3 + k) * stride] = off[k];
}
template <> __device__ __forceinline__ void store_block<float>(char *base, int stride, int b, const double d[6], const double2 off[15]) {
  float4 *q = (float4 *)base + (size_t)9 * b * stride;
  float f[36];
  for (int k = 0; k < 6; k++) f[k] = (float)d[k];
  for (int k = 0; k < 15; k++) { f[6 + 2 * k] = (float)off[k].x; f[7 + 2 * k] = (float)off[k].y; }
  for (int k = 0; k < 9; k++) q[(size_t)k * stride] = make_float4(f[4 * k], f[4 * k + 1], f[4 * k + 2], f[4 * k + 3]);
}

// LDL^dag inverse of a Hermitian 6x6 given by d (diag) and off (strict lower, row-major).
// Returns false on a zero / non-finite pivot.
__device__ bool hermitian_inverse6(const double d[6], const double2 off[15], double di[6], double2 oi[15]) {
  double2 Lm[6][6];
  double D[6];
  for (int j = 0; j < 6; j++) {
    double dj = d[j];
    for (int k = 0; k < j; k++) dj -= (Lm[j][k].x * Lm[j][k].x + Lm[j][k].y * Lm[j][k].y) * D[k];
    if (!(fabs(dj) > 1e-300) || !isfinite(dj)) return false;
    D[j] = dj;
    for (int i = j + 1; i < 6; i++) {
      double2 s = off[i * (i - 1) / 2 + j];
      for (int k = 0; k < j; k++) s = c_sub(s, c_mul(c_mul(Lm[i][k], c_conj(Lm[j][k])), make_double2(D[k], 0.0)));
      Lm[i][j] = make_double2(s.x / dj, s.y / dj);
    }
  }
  // columns of the inverse: solve L y = e_c, z = y / D, L^dag x = z
  double2 X[6][6];
  for (int col = 0; col < 6; col++) {
    double2 y[6];
    for (int i = 0; i < 6; i++) {
      double2 s = make_double2(i == col ? 1.0 : 0.0, 0.0);
      for (int k = 0; k < i; k++) s = c_sub(s, c_mul(Lm[i][k], y[k]));
      y[i] = s;
    }
    for (int i = 0; i < 6; i++) y[i] = make_double2(y[i].x / D[i], y[i].y / D[i]);
    for (int i = 5; i >= 0; i--) {
      double2 s = y[i];
      for (int k = i + 1; k < 6; k++) s = c_sub(s, c_mul(c_conj(Lm[k][i]), X[k][col]));
      X[i][col] = s;
    }
  }
  for (int i = 0; i < 6; i++) di[i] = X[i][i].x;
  for (int i = 1; i < 6; i++)
    for (int j = 0; j < i; j++) oi[i * (i - 1) / 2 + j] = X[i][j];
  return true;
}

// Assemble the two packed blocks of A from the six F_mu,nu (01 02 03 12 13 23) of one site,
// store A and / or A^-1 (fp64 arithmetic, stored in the field precision R).
template <typename R>
__device__ void assemble_store(const Geom &g, const M3 F[6], int cb, char *A, char *Ainv, double mass, double csw,
                               int *singular) {
  const double h = 0.5 * csw;
  for (int b = 0; b < 2; b++) {
    // 2x2 spin blocks with 3x3 colour entries: B00, B11, B01 (upper); B10 = B01^dag
    M3 B00, B11, B01;
    const double s23 = b == 0 ? 1.0 : -1.0;   // sign of F23 in B00 (block 0: +, block 1: -)
    const double s03 = b == 0 ? 1.0 : -1.0;
    const double s13 = b == 0 ? 1.0 : -1.0;
    for (int k = 0; k < 9; k++) {
      B00.m[k] = make_double2(-F[0].m[k].x + s23 * F[5].m[k].x, -F[0].m[k].y + s23 * F[5].m[k].y);
      B11.m[k] = make_double2(F[0].m[k].x - s23 * F[5].m[k].x, F[0].m[k].y - s23 * F[5].m[k].y);
      // B01 = i F02 + s03 F03 - F12 + s13 i F13
      double2 v = c_i(F[1].m[k]);
      v = c_add(v, make_double2(s03 * F[2].m[k].x, s03 * F[2].m[k].y));
      v = c_sub(v, F[3].m[k]);
      double2 w = c_i(F[4].m[k]);
      v = c_add(v, make_double2(s13 * w.x, s13 * w.y));
      B01.m[k] = v;
    }
    double d[6];
    double2 off[15];
    // element (i, j), i = 3 s + a
    for (int i = 0; i < 6; i++) {
      const int si = i / 3, a = i % 3;
      const M3 &Bd = si == 0 ? B00 : B11;
      d[i] = 4.0 + mass + h * Bd.m[4 * a].x;
      for (int j = 0; j < i; j++) {
        const int sj = j / 3, bb = j % 3;
        double2 v;
        if (si == sj) v = Bd.m[3 * a + bb];
        else v = c_conj(B01.m[3 * bb + a]);  // B10[a][bb] = conj(B01[bb][a])
        off[i * (i - 1) / 2 + j] = make_double2(h * v.x, h * v.y);
      }
    }
    if (A) store_block<R>(A + (size_t)cb * 16, g.stride, b, d, off);
    if (Ainv) {
      double di[6];
      double2 oi[15];
      if (!hermitian_inverse6(d, off, di, oi)) {
        atomicExch(singular, 1);
        for (int i = 0; i < 6; i++) di[i] = 0.0;
        for (int i = 0; i < 15; i++) oi[i] = make_double2(0.0, 0.0);
      }
      store_block<R>(Ainv + (size_t)cb * 16, g.stride, b, di, oi);
    }
  }
}

// Single-rank build: the leaves read their off-site links directly (periodic wrap).
template <typename R, int REC>
__global__ void __launch_bounds__(128) clover_build_kernel(const Geom g, GaugeView<R, REC> U, int p, char *A, char *Ainv,
                                                           double mass, double csw, int *singular) {
  const int cb = blockIdx.x * blockDim.x + threadIdx.x;
  if (cb >= g.Vh) return;
  int c[4];
  cb_coords(g, cb, p, c);
  M3 F[6];  // 01 02 03 12 13 23
  {
    int k = 0;
    for (int mu = 0; mu < 4; mu++)
      for (int nu = mu + 1; nu < 4; nu++) F[k++] = field_strength(g, U, c, mu, nu);
  }
  assemble_store<R>(g, F, cb, A, Ainv, mass, csw, singular);
}

// Partitioned build ("shifts of shifts"): the seven displaced gauge fields
// S[k](x) = U(x + d_k), d = (+mu, +nu, -mu, -nu, -mu+nu, -mu-nu, +mu-nu), were formed with
// qdp_shift (halo exchange included), so every leaf link is local to x.  Writes F_mu,nu of
// both parities into Fbuf[plane][parity][9][stride] (fp64).
template <typename R, int REC>
__global__ void __launch_bounds__(128) clover_leaf_kernel(const Geom g, GaugeView<R, REC> U, ShiftSet<R, REC> S, int mu,
                                                          int nu, int plane, double2 *Fbuf) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= 2 * g.Vh) return;
  const int p = i / g.Vh, cb = i % g.Vh;
  auto L = [&](const GaugeView<R, REC> &G, int d) {
    Link<R> l = G.load(d, p, cb);
    M3 r;
#pragma unroll
    for (int k = 0; k < 9; k++) r.m[k] = make_double2((double)l.m[k].re, (double)l.m[k].im);
    return r;
  };
  const GaugeView<R, REC> &Pm = S.s[0], &Pn = S.s[1], &Mm = S.s[2], &Mn = S.s[3], &MmPn = S.s[4], &MmMn = S.s[5],
                          &PmMn = S.s[6];
  M3 q, t;
  q = m3_mul(m3_mul(L(U, mu), L(Pm, nu)), m3_mul(m3_dag(L(Pn, mu)), m3_dag(L(U, nu))));
  t = m3_mul(m3_mul(L(U, nu), m3_dag(L(MmPn, mu))), m3_mul(m3_dag(L(Mm, nu)), L(Mm, mu)));
#pragma unroll
  for (int k = 0; k < 9; k++) q.m[k] = c_add(q.m[k], t.m[k]);
  t = m3_mul(m3_mul(m3_dag(L(Mm, mu)), m3_dag(L(MmMn, nu))), m3_mul(L(MmMn, mu), L(Mn, nu)));
#pragma unroll
  for (int k = 0; k < 9; k++) q.m[k] = c_add(q.m[k], t.m[k]);
  t = m3_mul(m3_mul(m3_dag(L(Mn, nu)), L(Mn, mu)), m3_mul(L(PmMn, nu), m3_dag(L(U, mu))));
#pragma unroll
  for (int k = 0; k < 9; k++) q.m[k] = c_add(q.m[k], t.m[k]);
  double2 *Fo = Fbuf + ((size_t)(plane * 2 + p) * 9) * g.stride + cb;
  double tr = 0.0;
  double2 f[9];
#pragma unroll
  for (int a = 0; a < 3; a++)
#pragma unroll
    for (int b = 0; b < 3; b++) {
      double2 d = c_sub(q.m[3 * a + b], c_conj(q.m[3 * b + a]));
      f[3 * a + b] = make_double2(d.y / 8.0, -d.x / 8.0);
    }
  tr = (f[0].x + f[4].x + f[8].x) / 3.0;
  f[0].x -= tr;
  f[4].x -= tr;
  f[8].x -= tr;
#pragma unroll
  for (int k = 0; k < 9; k++) Fo[(size_t)k * g.stride] = f[k];
}

template <typename R>
__global__ void __launch_bounds__(128) clover_assemble_kernel(const Geom g, const double2 *Fbuf, int p, char *A,
                                                              char *Ainv, double mass, double csw, int *singular) {
  const int cb = blockIdx.x * blockDim.x + threadIdx.x;
  if (cb >= g.Vh) return;
  M3 F[6];
  for (int k = 0; k < 6; k++)
    for (int e = 0; e < 9; e++) F[k].m[e] = Fbuf[((size_t)(k * 2 + p) * 9 + e) * g.stride + cb];
  assemble_store<R>(g, F, cb, A, Ainv, mass, csw, singular);
}

template <typename R>
__global__ void __launch_bounds__(128) clover_apply_kernel(const Geom g, FermView<R> out, CloverView<R> A, FermView<R> in) {
  const int cb = blockIdx.x * blockDim.x + threadIdx.x;
  if (cb >= g.Vh) return;
  Spinor<R> s = in.load_stream(cb);
  out.store(cb, clover_mul(A, cb, s));
}

// Partitioned lattice: F_mu,nu from local leaves on shifted gauge fields (see clover_leaf_kernel).
template <typename R, int REC>
static int build_F_by_shifts(qdp_ctx ctx, const qdp_field U, double2 *Fbuf) {
  const Geom &g = ctx->geom;
  const int prec = U->prec;
  const size_t gb = 2 * parity_block_bytes(U->kind, prec, g.stride);
  char *tmp = nullptr;
  QDP_CUDA(ctx, cudaMallocAsync((void **)&tmp, 8 * gb, ctx->stream));
  qdp_field_s f[8];
  for (int k = 0; k < 8; k++) {
    f[k].ctx = ctx;
    f[k].kind = U->kind;
    f[k].prec = prec;
    f[k].subset = QDP_ALL;
    f[k].data = tmp + k * gb;
    f[k].bytes = gb;
    f[k].owned = false;
  }
  // f[0..6] = U(x + d_k) in the order of ShiftSet; f[7] scratch
  int rc = QDP_OK, plane = 0;
  for (int mu = 0; mu < 4 && !rc; mu++)
    for (int nu = mu + 1; nu < 4 && !rc; nu++, plane++) {
      if ((rc = shift_field(ctx, &f[0], U, mu, +1))) break;      // U(x+mu)
      if ((rc = shift_field(ctx, &f[1], U, nu, +1))) break;      // U(x+nu)
      if ((rc = shift_field(ctx, &f[2], U, mu, -1))) break;      // U(x-mu)
      if ((rc = shift_field(ctx, &f[3], U, nu, -1))) break;      // U(x-nu)
      if ((rc = shift_field(ctx, &f[4], &f[1], mu, -1))) break;  // U(x-mu+nu)  (shift of a shift)
      if ((rc = shift_field(ctx, &f[5], &f[3], mu, -1))) break;  // U(x-mu-nu)
      if ((rc = shift_field(ctx, &f[6], &f[3], mu, +1))) break;  // U(x+mu-nu)
      ShiftSet<R, REC> S;
      for (int k = 0; k < 7; k++) S.s[k] = GaugeView<R, REC>{(decltype(S.s[k].p))f[k].data, g.stride};
      ProfEvent ev;
      prof_begin(ctx, QDP_PK_CLOVER, &ev);
      clover_leaf_kernel<R, REC><<<grid_for(2 * g.Vh, 128), 128, 0, ctx->stream>>>(
          g, GaugeView<R, REC>{(decltype(S.s[0].p))U->data, g.stride}, S, mu, nu, plane, Fbuf);
      if ((rc = prof_end(ctx, &ev))) break;
    }
  cudaFreeAsync(tmp, ctx->stream);
  return rc;
}

int clover_build(qdp_ctx ctx, const qdp_field U, void *A, int A_subset, void *Ainv, int Ainv_subset, double mass,
                 double csw, int *singular_host) {
  const Geom &g = ctx->geom;
  const int prec = U->prec;
  const size_t blk = parity_block_bytes(KIND_CLOVER, prec, g.stride);
  int *flag = (int *)(ctx->red_result + 62);  // scratch int in the reduction scalars
  QDP_CUDA(ctx, cudaMemsetAsync(flag, 0, sizeof(int), ctx->stream));
  double2 *Fbuf = nullptr;
  int rc;
  if (g.part) {  // some neighbours live across a rank (or self-halo) boundary: shifts of shifts
    QDP_CUDA(ctx, cudaMallocAsync((void **)&Fbuf, (size_t)6 * 2 * 9 * g.stride * sizeof(double2), ctx->stream));
    if (U->kind == KIND_GAUGE12)
      rc = prec == QDP_F64 ? build_F_by_shifts<double, 12>(ctx, U, Fbuf) : build_F_by_shifts<float, 12>(ctx, U, Fbuf);
    else
      rc = prec == QDP_F64 ? build_F_by_shifts<double, 18>(ctx, U, Fbuf) : build_F_by_shifts<float, 18>(ctx, U, Fbuf);
    if (rc) {
      cudaFreeAsync(Fbuf, ctx->stream);
      return rc;
    }
  }
  for (int p = 0; p < 2; p++) {
    char *a = nullptr, *ai = nullptr;
    if (A && (A_subset == QDP_ALL || A_subset == p)) a = (char *)A + (A_subset == QDP_ALL ? p * blk : 0);
    if (Ainv && (Ainv_subset == QDP_ALL || Ainv_subset == p)) ai = (char *)Ainv + (Ainv_subset == QDP_ALL ? p * blk : 0);
    if (!a && !ai) continue;
    ProfEvent ev;
    prof_begin(ctx, QDP_PK_CLOVER, &ev);
    const int nb = grid_for(g.Vh, 128);
    if (Fbuf) {
      if (prec == QDP_F64) clover_assemble_kernel<double><<<nb, 128, 0, ctx->stream>>>(g, Fbuf, p, a, ai, mass, csw, flag);
      else clover_assemble_kernel<float><<<nb, 128, 0, ctx->stream>>>(g, Fbuf, p, a, ai, mass, csw, flag);
    } else {
#define QDPB_CB(Rt, REC)                                                                                 \
  clover_build_kernel<Rt, REC><<<nb, 128, 0, ctx->stream>>>(                                             \
      g, GaugeView<Rt, REC>{(decltype(GaugeView<Rt, REC>::p))U->data, g.stride}, p, a, ai, mass, csw, flag)
      if (U->kind == KIND_GAUGE12) {
        if (prec == QDP_F64) QDPB_CB(double, 12); else QDPB_CB(float, 12);
      } else {
        if (prec == QDP_F64) QDPB_CB(double, 18); else QDPB_CB(float, 18);
      }
#undef QDPB_CB
    }
    if ((rc = prof_end(ctx, &ev))) return rc;
  }
  if (Fbuf) QDP_CUDA(ctx, cudaFreeAsync(Fbuf, ctx->stream));
  int h = 0;
  QDP_CUDA(ctx, cudaMemcpyAsync(&h, flag, sizeof(int), cudaMemcpyDeviceToHost, ctx->stream));
  QDP_CUDA(ctx, cudaStreamSynchronize(ctx->stream));
  *singular_host = h;
  return QDP_OK;
}

int clover_apply(qdp_ctx ctx, int prec, void *out, const void *A, const void *in, int nblk) {
  const Geom &g = ctx->geom;
  const size_t fb = fermion_block_bytes(prec, g.stride), cbk = parity_block_bytes(KIND_CLOVER, prec, g.stride);
  for (int b = 0; b < nblk; b++) {
    ProfEvent ev;
    prof_begin(ctx, QDP_PK_CLOVER, &ev);
    // Table II "clover": 504 flop, A (72 reals) + psi + out
    prof_work(ctx, QDP_PK_CLOVER, 504.0 * g.Vh, (72.0 + 24 + 24) * g.Vh * (prec == QDP_F64 ? 8 : 4));
    if (prec == QDP_F64)
      clover_apply_kernel<double><<<grid_for(g.Vh, 128), 128, 0, ctx->stream>>>(
          g, {(double2 *)((char *)out + b * fb), g.stride}, {(const double2 *)((const char *)A + b * cbk), g.stride},
          {(double2 *)((char *)in + b * fb), g.stride});
    else
      clover_apply_kernel<float><<<grid_for(g.Vh, 128), 128, 0, ctx->stream>>>(
          g, {(float4 *)((char *)out + b * fb), g.stride}, {(const float4 *)((const char *)A + b * cbk), g.stride},
          {(float4 *)((char *)in + b * fb), g.stride});
    int rc = prof_end(ctx, &ev);
    if (rc) return rc;
  }
  return QDP_OK;
}

}  // namespace qdpb
