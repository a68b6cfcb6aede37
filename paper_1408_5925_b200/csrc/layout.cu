// layout.cu -- host canonical (AoS, Table I order spin->colour->re/im) <->
// device structure-of-arrays conversion (section III-B), done on the
// device: the host array is copied as-is into a device staging buffer, then one thread per
// site scatters / gathers its components.  Also the slot maps shared with shift.cu.
#include <type_traits>

#include "internal.h"
#include "slots.h"

namespace qdpb {

size_t host_site_reals(int kind) {
  switch (kind) {
    case KIND_FERMION: return 24;
    case KIND_CMAT: return 18;
    case KIND_SMAT: return 32;
    case KIND_CLOVER: return 288;
    default: return 72;  // gauge
  }
}

size_t parity_block_bytes(int kind, int prec, int stride) {
  if (kind == KIND_FERMION) return fermion_block_bytes(prec, stride);
  if (kind == KIND_GAUGE) return (size_t)4 * stride * (prec == QDP_F64 ? 9 * 16 : 72);  // 4 mu per parity
  if (kind == KIND_GAUGE12) return (size_t)4 * stride * (prec == QDP_F64 ? 6 * 16 : 3 * 16);
  if (kind == KIND_CMAT) return (size_t)stride * (prec == QDP_F64 ? 9 * 16 : 72);
  if (kind == KIND_SMAT) return (size_t)stride * (prec == QDP_F64 ? 16 * 16 : 8 * 16);
  return (size_t)stride * (prec == QDP_F64 ? 36 * 16 : 18 * 16);
}

SlotMap make_slot_map(int kind, int prec, int stride, int subset) {
  SlotMap m = {};
  const size_t S = (size_t)stride;
  if (kind == KIND_FERMION) {
    m.n = 12;
    const size_t blk = fermion_block_bytes(prec, stride);
    for (int p = 0; p < 2; p++) {
      const long long base = subset == QDP_ALL ? (long long)(p * blk) : (p == subset ? 0 : -1);
      for (int k = 0; k < 12; k++) {
        if (prec == QDP_F64) { m.off[p][k] = base < 0 ? -1 : base + (long long)(k * S * 16); m.step[k] = 16; }
        else { m.off[p][k] = base < 0 ? -1 : base + (long long)((k / 2) * S * 16 + (k & 1) * 8); m.step[k] = 16; }
      }
    }
  } else if (kind == KIND_CMAT || kind == KIND_SMAT) {
    // colour matrix: fp64 double2[9], fp32 float4[4] + float2[1]; spin matrix: double2[16] / float4[8]
    m.n = kind == KIND_CMAT ? 9 : 16;
    const size_t blk = parity_block_bytes(kind, prec, stride);
    for (int p = 0; p < 2; p++) {
      const long long base = subset == QDP_ALL ? (long long)(p * blk) : (p == subset ? 0 : -1);
      for (int k = 0; k < m.n; k++) {
        long long o;
        int st = 16;
        if (prec == QDP_F64) o = (long long)(k * S * 16);
        else if (kind == KIND_CMAT && k == 8) { o = (long long)(S * 64); st = 8; }
        else o = (long long)((k / 2) * S * 16 + (k & 1) * 8);
        m.off[p][k] = base < 0 ? -1 : base + o;
        m.step[k] = st;
      }
    }
  } else if (kind == KIND_GAUGE12) {  // slot = mu*6 + e (rows 0,1)
    m.n = 24;
    for (int p = 0; p < 2; p++)
      for (int mu = 0; mu < 4; mu++)
        for (int e = 0; e < 6; e++) {
          const int k = mu * 6 + e;
          m.step[k] = 16;
          if (prec == QDP_F64) m.off[p][k] = (long long)(((mu * 2 + p) * 6 + e) * S * 16);
          else m.off[p][k] = (long long)(((mu * 2 + p) * 3 + e / 2) * S * 16 + (e & 1) * 8);
        }
  } else {  // gauge: slot = mu*9 + e
    m.n = 36;
    for (int p = 0; p < 2; p++)
      for (int mu = 0; mu < 4; mu++)
        for (int e = 0; e < 9; e++) {
          const int k = mu * 9 + e;
          if (prec == QDP_F64) {
            m.off[p][k] = (long long)(((mu * 2 + p) * 9 + e) * S * 16);
            m.step[k] = 16;
          } else {
            const long long blk = (long long)((mu * 2 + p) * S * 72);
            m.off[p][k] = blk + (long long)(e < 8 ? (e / 2) * S * 16 + (e & 1) * 8 : S * 64);
            m.step[k] = e < 8 ? 16 : 8;
          }
        }
  }
  // fp32: an even slot whose successor fills the other half of the same 16-byte element can be
  // moved together with it in one 16-byte access (both parities share the pattern)
  for (int k = 0; k + 1 < m.n; k++) {
    const int p = m.off[0][k] >= 0 ? 0 : 1;
    m.pair[k] = prec == QDP_F32 && m.step[k] == 16 && m.step[k + 1] == 16 && m.off[p][k] >= 0 &&
                m.off[p][k] % 16 == 0 && m.off[p][k + 1] == m.off[p][k] + 8;
  }
  return m;
}

// host record i -> (parity, cb)
__device__ __forceinline__ void record_site(const Geom &g, int subset, long i, int &p, int &cb) {
  if (subset == QDP_ALL) {
    int c[4];
    long s = i;
    c[0] = (int)(s % g.L[0]); s /= g.L[0];
    c[1] = (int)(s % g.L[1]); s /= g.L[1];
    c[2] = (int)(s % g.L[2]);
    c[3] = (int)(s / g.L[2]);
    p = coords_parity(c);
    cb = (int)(i >> 1);
  } else {
    p = subset;
    cb = (int)i;
  }
}

template <typename R, bool IMPORT>
__global__ void slots_kernel(const Geom g, const SlotMap m, int subset, long nrec, char *data, R *aos) {
  const long i = (long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= nrec) return;
  int p, cb;
  record_site(g, subset, i, p, cb);
  // one complex = one 16-byte (fp64) or 8-byte (fp32) access on both sides
  using C2 = typename std::conditional<sizeof(R) == 8, double2, float2>::type;
  C2 *rec = (C2 *)(aos + i * m.n * 2);
  for (int k = 0; k < m.n; k++) {
    C2 *d = (C2 *)(data + m.off[p][k] + (long long)cb * m.step[k]);
    if (IMPORT) *d = rec[k];
    else rec[k] = *d;
  }
}

// packed clover real j (0..71) of a parity block -> byte offset for cb = 0 (step 16 bytes)
template <typename R>
__device__ __forceinline__ long long clover_real_off(int j, int stride) {
  const int b = j / 36, r = j % 36;
  if (sizeof(R) == 8) {
    if (r < 6) return (long long)(18 * b + r / 2) * stride * 16 + (r & 1) * 8;
    const int k = (r - 6) / 2;
    return (long long)(18 * b + 3 + k) * stride * 16 + ((r - 6) & 1) * 8;
  }
  return (long long)(9 * b + r / 4) * stride * 16 + (r % 4) * 4;
}

// dense (row, col) of block-b packed real r: returns (row, col, part, conj-mirror)
template <typename R, bool IMPORT>
__global__ void clover_kernel(const Geom g, int subset, long nrec, char *data, size_t blk_bytes, R *aos) {
  const long i = (long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= nrec) return;
  int p, cb;
  record_site(g, subset, i, p, cb);
  char *base = data + (subset == QDP_ALL ? p * blk_bytes : 0) + (size_t)cb * 16;
  R *rec = aos + i * 288;  // [12][12][2]
  if (!IMPORT)
    for (int k = 0; k < 288; k++) rec[k] = R(0);
  for (int b = 0; b < 2; b++) {
    for (int ii = 0; ii < 6; ii++) {  // diagonal
      R *d = (R *)(base + clover_real_off<R>(36 * b + ii, g.stride));
      const int row = 6 * b + ii;
      if (IMPORT) *d = rec[(row * 12 + row) * 2];
      else rec[(row * 12 + row) * 2] = *d;
    }
    for (int a = 1; a < 6; a++)
      for (int c = 0; c < a; c++) {
        const int k = a * (a - 1) / 2 + c;
        R *re = (R *)(base + clover_real_off<R>(36 * b + 6 + 2 * k, g.stride));
        R *im = (R *)(base + clover_real_off<R>(36 * b + 7 + 2 * k, g.stride));
        const int row = 6 * b + a, col = 6 * b + c;
        if (IMPORT) {
          *re = rec[(row * 12 + col) * 2];
          *im = rec[(row * 12 + col) * 2 + 1];
        } else {
          rec[(row * 12 + col) * 2] = *re;
          rec[(row * 12 + col) * 2 + 1] = *im;
          rec[(col * 12 + row) * 2] = *re;
          rec[(col * 12 + row) * 2 + 1] = -*im;
        }
      }
  }
}

// QDP_GAUGE12: import keeps rows 0,1 of every link and flags links whose row 2 is not
// conj(row0 x row1) within tol (the compressed field would be wrong); export rebuilds row 2.
template <typename R, bool IMPORT>
__global__ void gauge12_kernel(const Geom g, const SlotMap m, long nrec, char *data, R *aos, double tol, int *bad) {
  const long i = (long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= nrec) return;
  int p, cb;
  record_site(g, QDP_ALL, i, p, cb);
  for (int mu = 0; mu < 4; mu++) {
    R *rec = aos + (i * 4 + mu) * 18;
    double re[6], im[6];
    for (int e = 0; e < 6; e++) {
      R *d = (R *)(data + m.off[p][mu * 6 + e] + (long long)cb * m.step[mu * 6 + e]);
      if (IMPORT) { d[0] = rec[2 * e]; d[1] = rec[2 * e + 1]; }
      re[e] = IMPORT ? (double)rec[2 * e] : (double)d[0];
      im[e] = IMPORT ? (double)rec[2 * e + 1] : (double)d[1];
    }
    double dev = 0.0;
    for (int a = 0; a < 3; a++) {
      const int b = (a + 1) % 3, c = (a + 2) % 3;
      // conj(r0[b] r1[c] - r0[c] r1[b])
      const double tr = re[b] * re[3 + c] - im[b] * im[3 + c] - (re[c] * re[3 + b] - im[c] * im[3 + b]);
      const double ti = re[b] * im[3 + c] + im[b] * re[3 + c] - (re[c] * im[3 + b] + im[c] * re[3 + b]);
      if (IMPORT) {
        dev = fmax(dev, fabs((double)rec[12 + 2 * a] - tr));
        dev = fmax(dev, fabs((double)rec[13 + 2 * a] + ti));
      } else {
        for (int e = 0; e < 6; e++) { rec[2 * e] = (R)re[e]; rec[2 * e + 1] = (R)im[e]; }
        rec[12 + 2 * a] = (R)tr;
        rec[13 + 2 * a] = (R)(-ti);
      }
    }
    if (IMPORT && !(dev <= tol)) atomicExch(bad, 1);
  }
}

static int layout_run(qdp_field f, void *dev_aos, bool import) {
  qdp_ctx ctx = f->ctx;
  const Geom &g = ctx->geom;
  const long nrec = f->subset == QDP_ALL ? ctx->V : g.Vh;
  const int blocks = grid_for(nrec, 128);
  ProfEvent ev;
  prof_begin(ctx, QDP_PK_LAYOUT, &ev);
  prof_work(ctx, QDP_PK_LAYOUT, 0.0, 2.0 * nrec * host_site_reals(f->kind) * (f->prec == QDP_F64 ? 8 : 4));
  if (f->kind == KIND_GAUGE12) {
    int *bad = (int *)(ctx->red_result + 60);
    QDP_CUDA(ctx, cudaMemsetAsync(bad, 0, sizeof(int), ctx->stream));
    SlotMap m = make_slot_map(f->kind, f->prec, g.stride, QDP_ALL);
    const double tol = f->prec == QDP_F64 ? 1e-10 : 1e-5;
    if (f->prec == QDP_F64) {
      if (import) gauge12_kernel<double, true><<<blocks, 128, 0, ctx->stream>>>(g, m, nrec, (char *)f->data, (double *)dev_aos, tol, bad);
      else gauge12_kernel<double, false><<<blocks, 128, 0, ctx->stream>>>(g, m, nrec, (char *)f->data, (double *)dev_aos, tol, bad);
    } else {
      if (import) gauge12_kernel<float, true><<<blocks, 128, 0, ctx->stream>>>(g, m, nrec, (char *)f->data, (float *)dev_aos, tol, bad);
      else gauge12_kernel<float, false><<<blocks, 128, 0, ctx->stream>>>(g, m, nrec, (char *)f->data, (float *)dev_aos, tol, bad);
    }
    int rc = prof_end(ctx, &ev);
    if (rc || !import) return rc;
    int h = 0;
    QDP_CUDA(ctx, cudaMemcpyAsync(&h, bad, sizeof(int), cudaMemcpyDeviceToHost, ctx->stream));
    QDP_CUDA(ctx, cudaStreamSynchronize(ctx->stream));
    if (h) return set_error(ctx, QDP_EINVAL, "import: QDP_GAUGE12 needs SU(3) links (row 2 = conj(row0 x row1))");
    return QDP_OK;
  }
  if (f->kind == KIND_CLOVER) {
    const size_t blk = parity_block_bytes(KIND_CLOVER, f->prec, g.stride);
    if (f->prec == QDP_F64) {
      if (import) clover_kernel<double, true><<<blocks, 128, 0, ctx->stream>>>(g, f->subset, nrec, (char *)f->data, blk, (double *)dev_aos);
      else clover_kernel<double, false><<<blocks, 128, 0, ctx->stream>>>(g, f->subset, nrec, (char *)f->data, blk, (double *)dev_aos);
    } else {
      if (import) clover_kernel<float, true><<<blocks, 128, 0, ctx->stream>>>(g, f->subset, nrec, (char *)f->data, blk, (float *)dev_aos);
      else clover_kernel<float, false><<<blocks, 128, 0, ctx->stream>>>(g, f->subset, nrec, (char *)f->data, blk, (float *)dev_aos);
    }
  } else {
    SlotMap m = make_slot_map(f->kind, f->prec, g.stride, f->subset);
    if (f->prec == QDP_F64) {
      if (import) slots_kernel<double, true><<<blocks, 128, 0, ctx->stream>>>(g, m, f->subset, nrec, (char *)f->data, (double *)dev_aos);
      else slots_kernel<double, false><<<blocks, 128, 0, ctx->stream>>>(g, m, f->subset, nrec, (char *)f->data, (double *)dev_aos);
    } else {
      if (import) slots_kernel<float, true><<<blocks, 128, 0, ctx->stream>>>(g, m, f->subset, nrec, (char *)f->data, (float *)dev_aos);
      else slots_kernel<float, false><<<blocks, 128, 0, ctx->stream>>>(g, m, f->subset, nrec, (char *)f->data, (float *)dev_aos);
    }
  }
  return prof_end(ctx, &ev);
}

int layout_import(qdp_field f, const void *dev_aos) { return layout_run(f, (void *)dev_aos, true); }
int layout_export(const qdp_field f, void *dev_aos) { return layout_run((qdp_field)f, dev_aos, false); }

}  // namespace qdpb
