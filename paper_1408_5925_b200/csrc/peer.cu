// peer.cu -- a communicator made of peer memory only (qdp_init_peer): every collective of the
// sub-grid decomposition -- the dslash face exchange, the shift
// face exchange and the global sums of norm2 / innerProduct -- is done by the library's own
// kernels storing into the other ranks' IPC-mapped device memory over NVLink / NVSwitch
// ("B200-native upgrade"), with release/acquire flags instead of a
// communication library.  The caller's host allgather is used once, inside qdp_init_peer, to
// exchange the IPC handles; no NCCL is loaded.
//
// Each rank owns one "board" (device memory, exported through CUDA IPC and mapped by every
// other rank):
//   header : unsigned sum_flag[2][MAXR]       ready flags of the global-sum slots
//            unsigned shift_arrived           seq of the last shift face written into mailbox
//            unsigned shift_consumed          seq of the last shift face read out of mailbox
//            unsigned put_counter, err
//   vals   : double   sum_val[2][MAXR][8]     per-source partial sums, two alternating slots
//   mailbox: shift faces (2 parities x up to 36 complex slots x the largest remote face)
//
// Global sum of n <= 8 doubles, call `seq` (same sequence on every rank): one thread stores
// its rank's values into slot seq&1 of EVERY rank's board and release-stores seq into that
// board's flag for this source; then it acquires all MAXR flags of its own board and sums the
// values in rank order (deterministic, identical on every rank).  Two slots suffice: a rank can
// only reach call seq+2 after every rank's call seq+1 contribution arrived, and each rank
// writes its seq+1 contribution only after it finished reading call seq.
//
// Shift face, call `seq`: the sender's copy kernel waits until the receiver's shift_consumed
// >= seq-1 (its mailbox is free), copies the packed face into the receiver's mailbox, and its
// last block release-stores seq into the receiver's shift_arrived; the receiver waits for
// shift_arrived >= seq before its shift kernel reads the mailbox and release-stores
// shift_consumed = seq after it.  Every wait is bounded (~10 s) and raises `err` instead of
// hanging (surfaced as QDP_ECUDA by qdp_synchronize and every synchronising call).
#include <string.h>

#include <algorithm>

#include "internal.h"

namespace qdpb {

constexpr int MAXR = PEER_MAX_RANKS;
constexpr size_t HDR_BYTES = PEER_HDR_BYTES;
constexpr size_t VAL_BYTES = PEER_VAL_BYTES;
static_assert(sizeof(unsigned) * (2 * MAXR + 4) <= HDR_BYTES, "peer board header");

struct PeerComm {
  char *board = nullptr;        // this rank's board
  char *peer[MAXR] = {};        // every rank's board as mapped here (peer[rank] = board)
  size_t mailbox_bytes = 0;
  unsigned sum_seq = 0, shift_seq = 0;
  std::vector<void *> opened;
};

__device__ __forceinline__ BoardHdr *hdr(char *b) { return board_hdr(b); }

// One thread: the allgather-and-sum of n <= 8 doubles at res[slot ..] (reduce.cuh peer_sum_dev).
__global__ void peer_sum_kernel(const PeerArgs a, double *res, int slot, int n, unsigned seq) {
  if (threadIdx.x != 0) return;
  double v[8];
  for (int i = 0; i < n; i++) v[i] = res[slot + i];
  peer_sum_dev(a, v, n, seq);
  for (int i = 0; i < n; i++) res[slot + i] = v[i];
}

// Sender side of a shift face: wait for the receiver's mailbox, copy, publish.
__global__ void __launch_bounds__(256) peer_put_kernel(const int4 *src, int4 *dst, size_t n16, char *dst_board,
                                                       unsigned *counter, unsigned seq, unsigned *err) {
  BoardHdr *h = hdr(dst_board);
  block_wait_flags(&h->shift_consumed, &h->shift_consumed, seq - 1u, err);
  for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n16; i += (size_t)gridDim.x * blockDim.x)
    dst[i] = src[i];
  grid_signal_last(counter, &h->shift_arrived, &h->shift_arrived, seq);
}

// Receiver side: wait until the face of call seq is in the mailbox.
__global__ void peer_wait_arrived_kernel(char *board, unsigned seq) {
  BoardHdr *h = hdr(board);
  block_wait_flags(&h->shift_arrived, &h->shift_arrived, seq, &h->err);
}
// Receiver side, after the shift kernel read the mailbox.
__global__ void peer_mark_consumed_kernel(char *board, unsigned seq) {
  if (threadIdx.x == 0) st_release_sys(&hdr(board)->shift_consumed, seq);
}

unsigned peer_next_sum_seq(qdp_ctx ctx) { return ++ctx->peer->sum_seq; }

PeerArgs peer_args(qdp_ctx ctx) {
  PeerArgs a;
  memset(&a, 0, sizeof(a));
  for (int q = 0; q < ctx->nranks; q++) a.board[q] = ctx->peer->peer[q];
  a.nranks = ctx->nranks;
  a.me = ctx->rank;
  return a;
}

// Host allgather through the caller's callback (set up time only).
int host_allgather(qdp_ctx ctx, const void *send, void *recv, size_t bytes) {
  if (!ctx->allgather) return set_error(ctx, QDP_EINVAL, "no host allgather callback");
  if (ctx->allgather(send, recv, bytes, ctx->allgather_user) != 0)
    return set_error(ctx, QDP_ECUDA, "the host allgather callback failed");
  return QDP_OK;
}

int peer_init(qdp_ctx ctx) {
  if (ctx->nranks > MAXR) return set_error(ctx, QDP_EUNSUPPORTED, "peer communicator: at most %d ranks", MAXR);
  PeerComm *p = new PeerComm();
  ctx->peer = p;
  const Geom &g = ctx->geom;
  long face = 0;
  for (int mu = 0; mu < 4; mu++)
    if (ctx->pgrid[mu] > 1) face = std::max(face, (long)g.faceVh[mu]);
  p->mailbox_bytes = (size_t)2 * 36 * face * 16;  // both parities of a gauge field, fp64
  const size_t total = HDR_BYTES + VAL_BYTES + p->mailbox_bytes;
  QDP_CUDA(ctx, cudaMalloc((void **)&p->board, total));
  QDP_CUDA(ctx, cudaMemset(p->board, 0, HDR_BYTES + VAL_BYTES));
  QDP_CUDA(ctx, cudaDeviceSynchronize());
  cudaIpcMemHandle_t mine;
  QDP_CUDA(ctx, cudaIpcGetMemHandle(&mine, p->board));
  std::vector<cudaIpcMemHandle_t> all(ctx->nranks);
  int rc = host_allgather(ctx, &mine, all.data(), sizeof(mine));
  if (rc) return rc;
  for (int q = 0; q < ctx->nranks; q++) {
    if (q == ctx->rank) {
      p->peer[q] = p->board;
      continue;
    }
    void *ptr = nullptr;
    cudaError_t e = cudaIpcOpenMemHandle(&ptr, all[q], cudaIpcMemLazyEnablePeerAccess);
    if (e != cudaSuccess) return cuda_check(ctx, e, "peer: cudaIpcOpenMemHandle (rank not reachable peer to peer?)");
    p->opened.push_back(ptr);
    p->peer[q] = (char *)ptr;
  }
  return QDP_OK;
}

void peer_destroy(qdp_ctx ctx) {
  PeerComm *p = ctx->peer;
  if (!p) return;
  for (void *ptr : p->opened) cudaIpcCloseMemHandle(ptr);
  if (p->board) cudaFree(p->board);
  delete p;
  ctx->peer = nullptr;
}

int peer_allreduce(qdp_ctx ctx, int slot, int n) {
  if (n > 8) return set_error(ctx, QDP_EINVAL, "peer sum: at most 8 scalars");
  ProfEvent ev;
  prof_begin(ctx, QDP_PK_REDUCE, &ev);
  peer_sum_kernel<<<1, 32, 0, ctx->stream>>>(peer_args(ctx), ctx->red_result, slot, n, peer_next_sum_seq(ctx));
  return prof_end(ctx, &ev);
}

int peer_sendrecv(qdp_ctx ctx, const void *send, size_t bytes, int to, void **ghost, unsigned *seq_out) {
  PeerComm *p = ctx->peer;
  if (bytes > p->mailbox_bytes) return set_error(ctx, QDP_EUNSUPPORTED, "peer shift: face larger than the mailbox");
  if (bytes % 16) return set_error(ctx, QDP_EINVAL, "peer shift: face bytes not a multiple of 16");
  const unsigned seq = ++p->shift_seq;
  const size_t n16 = bytes / 16;
  ProfEvent ev;
  prof_begin(ctx, QDP_PK_PACK, &ev);
  prof_work(ctx, QDP_PK_PACK, 0.0, 2.0 * bytes);
  const int blocks = std::max(1, std::min(grid_for((long)n16, 256), 2 * 148));
  char *dst_board = p->peer[to];
  peer_put_kernel<<<blocks, 256, 0, ctx->stream>>>((const int4 *)send, (int4 *)(dst_board + HDR_BYTES + VAL_BYTES), n16,
                                                   dst_board, &((BoardHdr *)p->board)->put_counter, seq,
                                                   &((BoardHdr *)p->board)->err);
  peer_wait_arrived_kernel<<<1, 32, 0, ctx->stream>>>(p->board, seq);
  int rc = prof_end(ctx, &ev);
  if (rc) return rc;
  *ghost = p->board + HDR_BYTES + VAL_BYTES;
  *seq_out = seq;
  return QDP_OK;
}

int peer_release_mailbox(qdp_ctx ctx, unsigned seq) {
  peer_mark_consumed_kernel<<<1, 32, 0, ctx->stream>>>(ctx->peer->board, seq);
  QDP_CUDA(ctx, cudaGetLastError());
  return QDP_OK;
}

int peer_check(qdp_ctx ctx) {
  if (!ctx->peer) return QDP_OK;
  unsigned e = 0;
  QDP_CUDA(ctx, cudaMemcpyAsync(&e, &((BoardHdr *)ctx->peer->board)->err, sizeof(unsigned), cudaMemcpyDeviceToHost,
                                ctx->stream));
  QDP_CUDA(ctx, cudaStreamSynchronize(ctx->stream));
  if (e) return set_error(ctx, QDP_ECUDA, "peer communicator: a flag wait timed out (a rank stopped participating?)");
  return QDP_OK;
}

}  // namespace qdpb
