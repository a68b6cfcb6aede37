// p2p.cu -- peer-to-peer halo exchange over NVLink / NVSwitch ("B200-native
// upgrade"; the face exchange of PAPER.md:208-214 without a separate communication call).
//
// Every rank exports its ghost buffers (two slots per face, alternating by call) and a small
// flag block through CUDA IPC; the neighbours map them.  Per EO dslash call `seq`, inside the
// dslash's own kernels (no extra launches, no communication library):
//   sender (pack kernel): wait until the receiver acknowledged slot seq&1 of call seq-2 (WAR),
//            store the projected faces straight into the receiver's ghost slot over NVLink, the
//            last block release-stores seq into the receiver's ready flag;
//   receiver: the interior kernel runs meanwhile; the exterior kernel acquires ready == seq,
//            reads the ghosts, and its last block release-stores seq into the senders' ack flags.
// A dim with one rank (self-halo) maps "the neighbour" to this rank, so the whole protocol runs
// and is tested on one GPU.  Waits poll with a bounded budget and raise an error flag instead
// of hanging (checked by p2p_check).
#include <string.h>

#include <algorithm>
#include <map>

#include "internal.h"

namespace qdpb {

enum { F_READY = 0, F_ACK = 1, F_COUNT = 2 };
// flag block of one rank: unsigned [2 prec][3 kinds][4 mu][2 dir], then the error word
constexpr int NFLAGS = 2 * 3 * 4 * 2;
inline size_t fidx(int prec, int kind, int mu, int d) { return ((size_t)(prec * 3 + kind) * 4 + mu) * 2 + d; }

// words after the flag block: [NFLAGS] error word, [NFLAGS + 1 + 4 prec ..] the face-packing work
// queue of the fused boundary kernel: two sets (by seq & 1) of {next chunk, chunks done} (local
// only: never written by a peer)
constexpr int NWORDS = NFLAGS + 1 + 8;

struct P2P {
  unsigned *flags = nullptr;  // this rank's flag block (+ error word and packing work queues)
  size_t slot_bytes[2] = {0, 0};
  int part[2] = {-1, -1};             // partition mask the slots of each precision were set up for
  void *recv[2][4][2] = {};           // this rank's ghost buffers (2 slots each)
  void *peer_recv[2][4][2] = {};      // [prec][mu][d]: ghost slots channel d writes into
  unsigned *peer_flags[4][2] = {};    // flag block of the -mu (d = 0) / +mu (d = 1) neighbour
  unsigned seq[2] = {0, 0};
  std::vector<void *> opened;         // IPC mappings
  std::map<int, unsigned *> flag_map;  // rank -> mapped flag block
};

struct HandleMsg {
  cudaIpcMemHandle_t recv[4][2];
  cudaIpcMemHandle_t flags;
};

static bool remote_dim(qdp_ctx ctx, int mu) { return ((ctx->geom.part >> mu) & 1) && ctx->pgrid[mu] > 1; }

static int p2p_setup(qdp_ctx ctx, int prec) {
  const Geom &g = ctx->geom;
  if (!ctx->p2p) {
    P2P *p = new P2P();
    if (cudaMalloc((void **)&p->flags, sizeof(unsigned) * NWORDS) != cudaSuccess) {
      cudaGetLastError();
      delete p;
      return set_error(ctx, QDP_ENOMEM, "p2p flags");
    }
    // on the context stream (non-blocking: a legacy-stream cudaMemset is not ordered before its
    // kernels, and a reused allocation would show the previous context's flags to the first call)
    QDP_CUDA(ctx, cudaMemsetAsync(p->flags, 0, sizeof(unsigned) * NWORDS, ctx->stream));
    QDP_CUDA(ctx, cudaStreamSynchronize(ctx->stream));  // zero before any peer can map and signal it
    ctx->p2p = p;
  }
  P2P *p = ctx->p2p;
  size_t need = 0;
  bool any_remote = false;
  for (int mu = 0; mu < 4; mu++)
    if ((g.part >> mu) & 1) {
      need = std::max(need, (size_t)g.faceVh[mu] * 12 * (prec == QDP_F64 ? 8 : 4));  // half spinors
      any_remote |= remote_dim(ctx, mu);
    }
  if (p->slot_bytes[prec] && p->part[prec] == g.part) return QDP_OK;
  if (p->slot_bytes[prec]) {
    // The partition changed after first use (QDP_OPT_SELF_HALO).  Dims reached through a
    // neighbour's mapped memory cannot be re-negotiated without every rank taking part, so that
    // is refused; a context whose partitioned dims are all self-halo dims rebuilds its slots and
    // restarts its sequence with zeroed flags (a newly partitioned dim's WAR flag would otherwise
    // lag the running sequence and its first pack would wait forever).
    if (any_remote) return set_error(ctx, QDP_EUNSUPPORTED, "p2p: the partition changed after first use");
    QDP_CUDA(ctx, cudaStreamSynchronize(ctx->stream));
    for (int mu = 0; mu < 4; mu++)
      for (int d = 0; d < 2; d++) {
        if (p->recv[prec][mu][d]) cudaFree(p->recv[prec][mu][d]);
        p->recv[prec][mu][d] = p->peer_recv[prec][mu][d] = nullptr;
      }
    const size_t f0 = fidx(prec, 0, 0, 0), nf = fidx(prec + 1, 0, 0, 0) - f0;
    QDP_CUDA(ctx, cudaMemsetAsync(p->flags + f0, 0, sizeof(unsigned) * nf, ctx->stream));
    QDP_CUDA(ctx, cudaMemsetAsync(p->flags + NFLAGS + 1 + 4 * prec, 0, 4 * sizeof(unsigned), ctx->stream));
    p->seq[prec] = 0;
    p->slot_bytes[prec] = 0;
    p->part[prec] = -1;
  }
  if (need == 0) return QDP_OK;
  QDP_CUDA(ctx, cudaStreamSynchronize(ctx->stream));
  for (int mu = 0; mu < 4; mu++)
    if ((g.part >> mu) & 1)
      for (int d = 0; d < 2; d++) {
        if (cudaMalloc(&p->recv[prec][mu][d], 2 * need) != cudaSuccess) {
          cudaGetLastError();
          return set_error(ctx, QDP_ENOMEM, "p2p ghost buffers");
        }
        QDP_CUDA(ctx, cudaMemsetAsync(p->recv[prec][mu][d], 0, 2 * need, ctx->stream));
      }
  QDP_CUDA(ctx, cudaStreamSynchronize(ctx->stream));
  // self dims: "the neighbour" is this rank
  for (int mu = 0; mu < 4; mu++)
    if (((g.part >> mu) & 1) && !remote_dim(ctx, mu)) {
      p->peer_recv[prec][mu][0] = p->recv[prec][mu][1];
      p->peer_recv[prec][mu][1] = p->recv[prec][mu][0];
      p->peer_flags[mu][0] = p->peer_flags[mu][1] = p->flags;
    }
  if (any_remote) {
    // exchange IPC handles of every rank's ghost buffers and flag block (allgather over NCCL)
    HandleMsg mine;
    memset(&mine, 0, sizeof(mine));
    for (int mu = 0; mu < 4; mu++)
      if ((g.part >> mu) & 1)
        for (int d = 0; d < 2; d++) QDP_CUDA(ctx, cudaIpcGetMemHandle(&mine.recv[mu][d], p->recv[prec][mu][d]));
    QDP_CUDA(ctx, cudaIpcGetMemHandle(&mine.flags, p->flags));
    std::vector<HandleMsg> all(ctx->nranks);
    if (ctx->peer) {
      int rc = host_allgather(ctx, &mine, all.data(), sizeof(HandleMsg));
      if (rc) return rc;
    } else {
    char *dev = nullptr;
    QDP_CUDA(ctx, cudaMalloc(&dev, sizeof(HandleMsg) * (ctx->nranks + 1)));
    QDP_CUDA(ctx, cudaMemcpyAsync(dev, &mine, sizeof(HandleMsg), cudaMemcpyHostToDevice, ctx->stream));
    int rc = comm_allgather_bytes(ctx, dev, dev + sizeof(HandleMsg), sizeof(HandleMsg), ctx->stream);
    if (!rc) {
      QDP_CUDA(ctx, cudaMemcpyAsync(all.data(), dev + sizeof(HandleMsg), sizeof(HandleMsg) * ctx->nranks,
                                    cudaMemcpyDeviceToHost, ctx->stream));
      QDP_CUDA(ctx, cudaStreamSynchronize(ctx->stream));
    }
    cudaFree(dev);
    if (rc) return rc;
    }
    int rc;
    auto open = [&](const cudaIpcMemHandle_t &h, void **out) -> int {
      cudaError_t e = cudaIpcOpenMemHandle(out, h, cudaIpcMemLazyEnablePeerAccess);
      if (e != cudaSuccess) return cuda_check(ctx, e, "p2p: cudaIpcOpenMemHandle (peer not reachable?)");
      p->opened.push_back(*out);
      return QDP_OK;
    };
    for (int mu = 0; mu < 4; mu++) {
      if (!remote_dim(ctx, mu)) continue;
      const int nm = ctx->neighbour[mu][0], np = ctx->neighbour[mu][1];
      // channel 0 writes the -mu neighbour's forward ghost, channel 1 the +mu neighbour's backward ghost
      if ((rc = open(all[nm].recv[mu][1], &p->peer_recv[prec][mu][0]))) return rc;
      if ((rc = open(all[np].recv[mu][0], &p->peer_recv[prec][mu][1]))) return rc;
      for (int d = 0; d < 2; d++) {
        const int r = d ? np : nm;
        if (!p->flag_map.count(r)) {
          void *fp = nullptr;
          if ((rc = open(all[r].flags, &fp))) return rc;
          p->flag_map[r] = (unsigned *)fp;
        }
        p->peer_flags[mu][d] = p->flag_map[r];
      }
    }
  }
  p->slot_bytes[prec] = need;
  p->part[prec] = g.part;
  return QDP_OK;
}

int p2p_setup_all(qdp_ctx ctx) {
  int rc;
  if ((rc = p2p_setup(ctx, QDP_F64))) return rc;
  return p2p_setup(ctx, QDP_F32);
}

// Set-up (collective on first use) happens BEFORE the call's sequence number is taken, so every
// launch of a call sees a fresh `seq` (a first call that created the state used to get seq 1 and
// the next call seq 1 again: its face blocks then passed their ready wait on the previous call's
// flag and could read the ghosts before this call's packers wrote them).
int p2p_prepare(qdp_ctx ctx, int prec, P2PLaunch *L) {
  int rc;
  if ((rc = p2p_setup(ctx, prec))) return rc;
  P2P *p = ctx->p2p;
  const Geom &g = ctx->geom;
  const unsigned seq = ++p->seq[prec];
  const size_t off = (seq & 1u) * p->slot_bytes[prec];
  memset(L, 0, sizeof(*L));
  L->seq = seq;
  L->err = p->flags + NFLAGS;
  L->pack_q = p->flags + NFLAGS + 1 + 4 * prec;
  for (int mu = 0; mu < 4; mu++) {
    if (!((g.part >> mu) & 1)) continue;
    for (int d = 0; d < 2; d++) {
      L->dst[mu][d] = (char *)p->peer_recv[prec][mu][d] + off;
      L->ghost[mu][d] = (const char *)p->recv[prec][mu][d] + off;
      // WAR: slot seq&1 of channel d was last read by its receiver in call seq-2
      L->war[mu][d] = p->flags + fidx(prec, F_ACK, mu, d);
      L->ready[mu][d] = p->flags + fidx(prec, F_READY, mu, d);
    }
    L->pack_counter[mu] = p->flags + fidx(prec, F_COUNT, mu, 0);
    L->ext_counter[mu] = p->flags + fidx(prec, F_COUNT, mu, 1);
    L->sig[mu][0] = p->peer_flags[mu][0] + fidx(prec, F_READY, mu, 1);  // -mu neighbour's forward ghost
    L->sig[mu][1] = p->peer_flags[mu][1] + fidx(prec, F_READY, mu, 0);  // +mu neighbour's backward ghost
    // ghost 0 came from the -mu neighbour's channel 1, ghost 1 from the +mu neighbour's channel 0
    L->ack_to[mu][0] = p->peer_flags[mu][0] + fidx(prec, F_ACK, mu, 1);
    L->ack_to[mu][1] = p->peer_flags[mu][1] + fidx(prec, F_ACK, mu, 0);
  }
  return QDP_OK;
}

int p2p_check(qdp_ctx ctx) {
  if (ctx->peer) {
    int rc = peer_check(ctx);
    if (rc) return rc;
  }
  if (!ctx->p2p) return QDP_OK;
  unsigned e = 0;
  QDP_CUDA(ctx, cudaMemcpyAsync(&e, ctx->p2p->flags + NFLAGS, sizeof(unsigned), cudaMemcpyDeviceToHost, ctx->stream));
  QDP_CUDA(ctx, cudaStreamSynchronize(ctx->stream));
  if (e) return set_error(ctx, QDP_ECUDA, "p2p halo: a flag wait timed out (a neighbour stopped calling dslash?)");
  return QDP_OK;
}

void p2p_destroy(qdp_ctx ctx) {
  P2P *p = ctx->p2p;
  if (!p) return;
  for (void *ptr : p->opened) cudaIpcCloseMemHandle(ptr);
  for (int pr = 0; pr < 2; pr++)
    for (int mu = 0; mu < 4; mu++)
      for (int d = 0; d < 2; d++)
        if (p->recv[pr][mu][d]) cudaFree(p->recv[pr][mu][d]);
  if (p->flags) cudaFree(p->flags);
  delete p;
  ctx->p2p = nullptr;
}

}  // namespace qdpb
