// shift.cu -- circular shift of QDP++ (section II-C; reading R4):
//   out(x) = in(x + sign * mu^)
// A pure site permutation: one thread per output site copies the site's complex slots.
// When dim mu is partitioned, the face that crosses the rank boundary is gathered into a
// contiguous buffer, exchanged (NCCL, or written straight into this rank's
// ghost buffer in self-halo mode), and read by the main kernel for the boundary sites.
// Ghost layout: [parity][slot][faceVh] complex slots.
#include "internal.h"
#include "slots.h"

namespace qdpb {

template <typename R> struct C2;
template <> struct C2<double> { using T = double2; };
template <> struct C2<float> { using T = float2; };

template <typename R>
__global__ void shift_pack_kernel(const Geom g, const SlotMap m, const char *in, int mu, int xmu, int nq, int q0,
                                  typename C2<R>::T *ghost) {
  using T = typename C2<R>::T;
  const int n = g.faceVh[mu];
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= nq * n) return;
  const int q = q0 + i / n, f = i % n;
  int c[4];
  face_coords(g, mu, xmu, f, q, c);
  const int cb = coords_cb(g, c);
  for (int k = 0; k < m.n; k++)
    ghost[((size_t)q * m.n + k) * n + f] = *(const T *)(in + m.off[q][k] + (long long)cb * m.step[k]);
}

template <typename R>
__global__ void shift_kernel(const Geom g, const SlotMap mo, const SlotMap mi, char *out, const char *in, int mu, int sign,
                             int np, int p0, bool remote_dim, const typename C2<R>::T *ghost) {
  using T = typename C2<R>::T;
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= np * g.Vh) return;
  const int p = p0 + i / g.Vh, cb = i % g.Vh;
  int c[4];
  cb_coords(g, cb, p, c);
  int n = c[mu] + sign;
  const bool wrap = n < 0 || n >= g.L[mu];
  n = n < 0 ? n + g.L[mu] : (n >= g.L[mu] ? n - g.L[mu] : n);
  c[mu] = n;
  const int q = 1 - p;
  if (wrap && remote_dim) {
    const int nf = g.faceVh[mu];
    const int f = face_index(g, mu, c);
    for (int k = 0; k < mo.n; k++)
      *(T *)(out + mo.off[p][k] + (long long)cb * mo.step[k]) = ghost[((size_t)q * mo.n + k) * nf + f];
  } else {
    const int scb = coords_cb(g, c);
    for (int k = 0; k < mo.n; k++) {
      char *d = out + mo.off[p][k] + (long long)cb * mo.step[k];
      const char *s = in + mi.off[q][k] + (long long)scb * mi.step[k];
      if (sizeof(R) == 4 && mo.pair[k]) {  // two fp32 complex in one 16-byte access
        *(float4 *)d = *(const float4 *)s;
        k++;
      } else {
        *(T *)d = *(const T *)s;
      }
    }
  }
}

int shift_field(qdp_ctx ctx, qdp_field out, const qdp_field in, int mu, int sign) {
  const Geom &g = ctx->geom;
  const SlotMap mo = make_slot_map(out->kind, out->prec, g.stride, out->subset);
  const SlotMap mi = make_slot_map(in->kind, in->prec, g.stride, in->subset);
  // output parities: ALL -> both; parity p field -> p
  const int np = out->subset == QDP_ALL ? 2 : 1;
  const int p0 = out->subset == QDP_ALL ? 0 : out->subset;
  const int nq = in->subset == QDP_ALL ? 2 : 1;
  const int q0 = in->subset == QDP_ALL ? 0 : in->subset;
  const bool remote = (g.part >> mu) & 1;
  const size_t cbytes = in->prec == QDP_F64 ? 16 : 8;
  void *ghost = nullptr;
  unsigned peer_seq = 0;
  int rc;
  if (remote) {
    const size_t bytes = (size_t)2 * mi.n * g.faceVh[mu] * cbytes;
    // scratch: [send | recv] in the staging buffer
    if ((rc = ensure_staging(ctx, 2 * bytes))) return rc;
    char *send = (char *)ctx->staging, *recv = send + bytes;
    const bool self = direct_self(ctx, mu);
    // receiver needs in(x + sign mu) for its boundary sites: sign=+1 -> our x_mu=0 face goes to -mu
    const int xmu = sign > 0 ? 0 : g.L[mu] - 1;
    ProfEvent ev;
    prof_begin(ctx, QDP_PK_PACK, &ev);
    prof_work(ctx, QDP_PK_PACK, 0.0, 2.0 * nq * g.faceVh[mu] * mi.n * cbytes);
    const int nth = nq * g.faceVh[mu];
    char *dst = self ? recv : send;
    if (in->prec == QDP_F64)
      shift_pack_kernel<double><<<grid_for(nth, 128), 128, 0, ctx->stream>>>(g, mi, (const char *)in->data, mu, xmu, nq, q0, (double2 *)dst);
    else
      shift_pack_kernel<float><<<grid_for(nth, 128), 128, 0, ctx->stream>>>(g, mi, (const char *)in->data, mu, xmu, nq, q0, (float2 *)dst);
    if ((rc = prof_end(ctx, &ev))) return rc;
    ghost = recv;
    if (!self) {
      const int to = ctx->neighbour[mu][sign > 0 ? 0 : 1], from = ctx->neighbour[mu][sign > 0 ? 1 : 0];
      if (ctx->peer) {  // into the receiver's mapped mailbox (peer.cu); ghost = our own mailbox
        if ((rc = peer_sendrecv(ctx, send, bytes, to, &ghost, &peer_seq))) return rc;
      } else if ((rc = comm_sendrecv(ctx, send, bytes, to, recv, from, ctx->stream))) {
        return rc;
      }
    }
  }
  ProfEvent ev;
  prof_begin(ctx, QDP_PK_SHIFT, &ev);
  prof_work(ctx, QDP_PK_SHIFT, 0.0, 2.0 * np * g.Vh * mo.n * cbytes);
  const int nth = np * g.Vh;
  if (in->prec == QDP_F64)
    shift_kernel<double><<<grid_for(nth, 128), 128, 0, ctx->stream>>>(g, mo, mi, (char *)out->data, (const char *)in->data, mu, sign,
                                                                       np, p0, remote, (const double2 *)ghost);
  else
    shift_kernel<float><<<grid_for(nth, 128), 128, 0, ctx->stream>>>(g, mo, mi, (char *)out->data, (const char *)in->data, mu, sign,
                                                                      np, p0, remote, (const float2 *)ghost);
  if ((rc = prof_end(ctx, &ev))) return rc;
  return peer_seq ? peer_release_mailbox(ctx, peer_seq) : QDP_OK;
}

}  // namespace qdpb
