// comm.cpp -- inter-rank communication of the sub-grid decomposition (PAPER.md:93-95,
// 208-214): NCCL point-to-point face exchange (the MPI send/recv of section V, here over
// NVLink / NVSwitch) and the global sums of the reductions.
//
// NCCL is loaded with dlopen at qdp_init time (only when nranks > 1), so the library loads
// and its single-rank path runs without NCCL; in a torch process the already-loaded
// libnccl.so.2 is reused.
#include <dlfcn.h>
#include <nccl.h>
#include <string.h>

#include "internal.h"

namespace qdpb {

struct NcclApi {
  void *h = nullptr;
  ncclResult_t (*GetUniqueId)(ncclUniqueId *);
  ncclResult_t (*CommInitRank)(ncclComm_t *, int, ncclUniqueId, int);
  ncclResult_t (*CommDestroy)(ncclComm_t);
  ncclResult_t (*Send)(const void *, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t);
  ncclResult_t (*Recv)(void *, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t);
  ncclResult_t (*GroupStart)();
  ncclResult_t (*GroupEnd)();
  ncclResult_t (*AllGather)(const void *, void *, size_t, ncclDataType_t, ncclComm_t, cudaStream_t);
  ncclResult_t (*AllReduce)(const void *, void *, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t, cudaStream_t);
  const char *(*GetErrorString)(ncclResult_t);
};

static NcclApi g_nccl;

static bool load_nccl() {
  if (g_nccl.h) return true;
  const char *names[] = {"libnccl.so.2", "libnccl.so"};
  void *h = nullptr;
  for (const char *n : names)
    if ((h = dlopen(n, RTLD_NOW | RTLD_GLOBAL))) break;
  if (!h) return false;
#define QDPB_SYM(field, name)                                  \
  *(void **)(&g_nccl.field) = dlsym(h, name);                  \
  if (!g_nccl.field) return false;
  QDPB_SYM(GetUniqueId, "ncclGetUniqueId");
  QDPB_SYM(CommInitRank, "ncclCommInitRank");
  QDPB_SYM(CommDestroy, "ncclCommDestroy");
  QDPB_SYM(Send, "ncclSend");
  QDPB_SYM(Recv, "ncclRecv");
  QDPB_SYM(GroupStart, "ncclGroupStart");
  QDPB_SYM(GroupEnd, "ncclGroupEnd");
  QDPB_SYM(AllGather, "ncclAllGather");
  QDPB_SYM(AllReduce, "ncclAllReduce");
  QDPB_SYM(GetErrorString, "ncclGetErrorString");
#undef QDPB_SYM
  g_nccl.h = h;
  return true;
}

struct Comm {
  ncclComm_t comm;
};

static int nccl_err(qdp_ctx ctx, ncclResult_t r, const char *what) {
  return set_error(ctx, QDP_ENCCL, "%s: %s", what, g_nccl.GetErrorString ? g_nccl.GetErrorString(r) : "nccl error");
}
#define QDPB_NCCL(ctx, call)                                         \
  do {                                                               \
    ncclResult_t _r = (call);                                        \
    if (_r != ncclSuccess) return nccl_err(ctx, _r, #call);          \
  } while (0)

int comm_get_unique_id(unsigned char id[128]) {
  static_assert(sizeof(ncclUniqueId) == 128, "ncclUniqueId size");
  if (!load_nccl()) return QDP_ENCCL;
  ncclUniqueId u;
  if (g_nccl.GetUniqueId(&u) != ncclSuccess) return QDP_ENCCL;
  memcpy(id, &u, 128);
  return QDP_OK;
}

int comm_init(qdp_ctx ctx, const unsigned char *id) {
  if (ctx->nranks == 1) return QDP_OK;
  if (!id) return set_error(ctx, QDP_EINVAL, "qdp_init: NCCL id required for nranks > 1");
  if (!load_nccl()) return set_error(ctx, QDP_ENCCL, "qdp_init: cannot dlopen libnccl.so.2");
  ncclUniqueId u;
  memcpy(&u, id, 128);
  Comm *c = new Comm();
  ncclResult_t r = g_nccl.CommInitRank(&c->comm, ctx->nranks, u, ctx->rank);
  if (r != ncclSuccess) {
    delete c;
    return nccl_err(ctx, r, "ncclCommInitRank");
  }
  ctx->comm = c;
  return QDP_OK;
}

// One-rank communicator: self-halo dims then exchange through ncclSend / ncclRecv to this
// rank (the same message order as P_mu = 2, where both neighbours are one peer).
int comm_ensure_self(qdp_ctx ctx) {
  if (ctx->comm) return QDP_OK;
  if (ctx->nranks != 1) return set_error(ctx, QDP_ENCCL, "no communicator");
  unsigned char id[128];
  if (comm_get_unique_id(id)) return set_error(ctx, QDP_ENCCL, "cannot load NCCL / get a unique id");
  ncclUniqueId u;
  memcpy(&u, id, 128);
  Comm *c = new Comm();
  ncclResult_t r = g_nccl.CommInitRank(&c->comm, 1, u, 0);
  if (r != ncclSuccess) {
    delete c;
    return nccl_err(ctx, r, "ncclCommInitRank(1 rank)");
  }
  ctx->comm = c;
  return QDP_OK;
}

void comm_destroy(qdp_ctx ctx) {
  if (ctx->comm) {
    g_nccl.CommDestroy(ctx->comm->comm);
    delete ctx->comm;
    ctx->comm = nullptr;
  }
}

// For every communicated dim (partitioned with more than one rank):
//   send(+mu: send[mu][1]), send(-mu: send[mu][0]), recv(-mu: recv[mu][0]), recv(+mu: recv[mu][1]).
// With P_mu = 2 both neighbours are the same rank and NCCL matches same-peer messages in
// issue order: our first send (to +mu) pairs with the peer's first recv (from its -mu,
// which is us), so the messages land in the right buffers.
int comm_exchange(qdp_ctx ctx, int prec, const size_t face_bytes[4], cudaStream_t stream) {
  if (!ctx->comm) return set_error(ctx, QDP_ENCCL, "halo exchange without a communicator");
  ncclComm_t cm = ctx->comm->comm;
  QDPB_NCCL(ctx, g_nccl.GroupStart());
  for (int mu = 0; mu < 4; mu++) {
    if (!face_bytes[mu] || direct_self(ctx, mu)) continue;
    const size_t n = face_bytes[mu];
    QDPB_NCCL(ctx, g_nccl.Send(ctx->halo_send[prec][mu][1], n, ncclChar, ctx->neighbour[mu][1], cm, stream));
    QDPB_NCCL(ctx, g_nccl.Send(ctx->halo_send[prec][mu][0], n, ncclChar, ctx->neighbour[mu][0], cm, stream));
    QDPB_NCCL(ctx, g_nccl.Recv(ctx->halo_recv[prec][mu][0], n, ncclChar, ctx->neighbour[mu][0], cm, stream));
    QDPB_NCCL(ctx, g_nccl.Recv(ctx->halo_recv[prec][mu][1], n, ncclChar, ctx->neighbour[mu][1], cm, stream));
  }
  QDPB_NCCL(ctx, g_nccl.GroupEnd());
  return QDP_OK;
}

int comm_sendrecv(qdp_ctx ctx, const void *send, size_t bytes, int to, void *recv, int from, cudaStream_t stream) {
  if (!ctx->comm) return set_error(ctx, QDP_ENCCL, "sendrecv without a communicator");
  ncclComm_t cm = ctx->comm->comm;
  QDPB_NCCL(ctx, g_nccl.GroupStart());
  QDPB_NCCL(ctx, g_nccl.Send(send, bytes, ncclChar, to, cm, stream));
  QDPB_NCCL(ctx, g_nccl.Recv(recv, bytes, ncclChar, from, cm, stream));
  QDPB_NCCL(ctx, g_nccl.GroupEnd());
  return QDP_OK;
}

int comm_allgather_f64(qdp_ctx ctx, const double *send, double *recv, int count, cudaStream_t stream) {
  if (!ctx->comm) return set_error(ctx, QDP_ENCCL, "allgather without a communicator");
  QDPB_NCCL(ctx, g_nccl.AllGather(send, recv, (size_t)count, ncclDouble, ctx->comm->comm, stream));
  return QDP_OK;
}

int comm_allgather_bytes(qdp_ctx ctx, const void *send, void *recv, size_t bytes, cudaStream_t stream) {
  if (!ctx->comm) return set_error(ctx, QDP_ENCCL, "allgather without a communicator");
  QDPB_NCCL(ctx, g_nccl.AllGather(send, recv, bytes, ncclChar, ctx->comm->comm, stream));
  return QDP_OK;
}

int comm_allreduce_f64(qdp_ctx ctx, double *buf, int count, cudaStream_t stream) {
  if (!ctx->comm) return set_error(ctx, QDP_ENCCL, "allreduce without a communicator");
  QDPB_NCCL(ctx, g_nccl.AllReduce(buf, buf, (size_t)count, ncclDouble, ncclSum, ctx->comm->comm, stream));
  return QDP_OK;
}

}  // namespace qdpb
