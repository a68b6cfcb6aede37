// reduce.cuh -- one-launch deterministic grid reductions (norm2 / innerProduct of the north
// star) and the device side of the peer-memory global sum (peer.cu).
//
// A reduction finishes inside the kernel that produces it ("last block done"), in two levels of
// fixed order so the result does not depend on which block finishes last:
//   every block   : its sum (warp shuffles, then one warp) -> part[vb]; fence; counter of its
//                   group of G = blockDim consecutive blocks;
//   last of group : sums the group's G partials (thread i reads partial i) -> part2[g]; fence;
//                   top counter;
//   last of all   : sums part2[] (thread i reads i, i+G, ...) -> the total; with a peer
//                   communicator it then does the rank-ordered global sum over NVLink itself
//                   (peer_sum_dev), writes res[slot..] (and a mapped host copy), and may record
//                   a CG residual (CgDev) -- so a norm2 or the CG's |r|^2 is one launch.
// The counters return to zero after every launch (each level's last block resets its own).
#pragma once

namespace qdpb {

// ---- peer-memory boards (peer.cu): the device side of the global sum
constexpr size_t PEER_HDR_BYTES = 4096;
constexpr size_t PEER_VAL_BYTES = sizeof(double) * 2 * PEER_MAX_RANKS * 8;
struct BoardHdr {
  unsigned sum_flag[2][PEER_MAX_RANKS];
  unsigned shift_arrived, shift_consumed, put_counter, err;
};
struct PeerArgs {
  char *board[PEER_MAX_RANKS];  // every rank's board as mapped in this process
  int nranks, me;
};

#ifdef __CUDACC__
__device__ __forceinline__ BoardHdr *board_hdr(char *b) { return (BoardHdr *)b; }
__device__ __forceinline__ double *board_vals(char *b, int slot, int src) {
  return (double *)(b + PEER_HDR_BYTES) + ((size_t)slot * PEER_MAX_RANKS + src) * 8;
}

// Global sum of v[0..n) (n <= 8) over the ranks, call `seq` (the same sequence on every rank);
// ONE thread.  It stores this rank's values into slot seq&1 of EVERY rank's board and
// release-stores seq into that board's flag for this source, then acquires all flags of its
// own board and sums the values in rank order (deterministic, identical on every rank).  Two
// slots suffice: a rank can only reach call seq+2 after every rank's call seq+1 contribution
// arrived, and each rank writes its seq+1 contribution only after it finished reading call seq.
__device__ inline void peer_sum_dev(const PeerArgs &a, double *v, int n, unsigned seq) {
  const int s = seq & 1;
  for (int q = 0; q < a.nranks; q++) {
    char *b = a.board[q];
    double *d = board_vals(b, s, a.me);
    for (int i = 0; i < n; i++) d[i] = v[i];
    st_release_sys(&board_hdr(b)->sum_flag[s][a.me], seq);  // orders this thread's stores above
  }
  char *mine = a.board[a.me];
  BoardHdr *h = board_hdr(mine);
  for (int q = 0; q < a.nranks; q++) {
    long k = 0;
    while ((int)(ld_acquire_sys(&h->sum_flag[s][q]) - seq) < 0) {
      if (++k > (1L << 26)) {
        atomicExch(&h->err, 1u);
        break;
      }
      __nanosleep(64);
    }
  }
  double acc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  for (int q = 0; q < a.nranks; q++) {
    const volatile double *src = board_vals(mine, s, q);
    for (int i = 0; i < n; i++) acc[i] += src[i];
  }
  for (int i = 0; i < n; i++) v[i] = acc[i];
}
#endif

// Device-side bookkeeping of the CG (solver.cu), applied by the final block of the r update of
// iteration k once |r_k|^2 is known globally: hist[k] = |r_k|^2 (mapped pinned host memory), and
// the first k with |r_k|^2 <= tol2 |r_0|^2 or k == maxit is stored in *stop (device) and
// *stop_host.  Kernels of later iterations see *stop < their iteration and do no work.
struct CgDev {
  double *hist;
  int *stop, *stop_host;
  const double *rho0;  // device scalar |r_0|^2
  int k, maxit;
  double tol2;
};

struct RedArgs {
  double *part, *part2;  // level-1 [2 x blocks], level-2 [2 x groups] partial pairs
  unsigned *cnt;         // [0] top counter, [1 + g] group counters (zero between launches)
  double *res;           // device scalars (red_result)
  int slot, n;           // res[slot .. slot+n), n = 1 or 2
  double *host;          // optional mapped pinned copy of the n values
  unsigned *host_flag;   // with host: `token` is stored here (mapped) after the values
  unsigned token;
  int peer;              // 1: global sum over the peer communicator in the final block
  unsigned seq;          //    its call sequence number
  PeerArgs pa;
  int has_cg;
  CgDev cg;
};

#ifdef __CUDACC__
// sum of (v0, v1) over the block, in thread 0 (fixed order; blockDim a multiple of 32, <= 1024)
__device__ __forceinline__ void block_sum2(double &v0, double &v1) {
  __shared__ double s0[32], s1[32];
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    v0 += __shfl_xor_sync(0xffffffffu, v0, o);
    v1 += __shfl_xor_sync(0xffffffffu, v1, o);
  }
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  if (l == 0) {
    s0[w] = v0;
    s1[w] = v1;
  }
  __syncthreads();
  if (w == 0) {
    const int nw = blockDim.x >> 5;
    v0 = l < nw ? s0[l] : 0.0;
    v1 = l < nw ? s1[l] : 0.0;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      v0 += __shfl_xor_sync(0xffffffffu, v0, o);
      v1 += __shfl_xor_sync(0xffffffffu, v1, o);
    }
  }
  __syncthreads();  // s0 / s1 may be reused by the next call
}

__device__ __forceinline__ void cg_record(const CgDev &c, double rr) {
  c.hist[c.k] = rr;
  const int stop = *c.stop;
  if (stop > c.k && (rr <= c.tol2 * *c.rho0 || c.k >= c.maxit)) {
    *c.stop = c.k;
    *(volatile int *)c.stop_host = c.k;
  }
}

// First half, called by EVERY thread of EVERY block of the grid (nblk blocks) with this thread's
// share (v0, v1); vb = the block's index in the fixed partial order.  Stores the block's partial,
// fences it and counts the block into its group; returns (to every thread) whether this block
// was the group's last, i.e. must call red_complete.  Kernels that also store a large output call
// it BEFORE those stores: the fence then only waits for the partial (a fence after the output
// stores holds each block's SM slot until they are acknowledged -- measured ~16 us per dslash).
__device__ __forceinline__ bool red_arrive(const RedArgs &R, int nblk, int vb, double v0, double v1) {
  __shared__ int s_arrive_last;
  block_sum2(v0, v1);
  const int G = blockDim.x;
  const int g = vb / G;
  if (threadIdx.x == 0) {
    R.part[2 * vb] = v0;
    R.part[2 * vb + 1] = v1;
    __threadfence();
    const int ng = min(G, nblk - g * G);
    s_arrive_last = atomicAdd(&R.cnt[1 + g], 1u) == (unsigned)(ng - 1);
  }
  __syncthreads();
  return s_arrive_last != 0;
}

// Second half, by every thread of a block for which red_arrive returned true: the group's sum,
// then (last group) the total, the peer global sum, the results and the CG bookkeeping.  skip:
// the kernel did no work this launch (a CG iteration after the stopping one): the sum and the peer
// protocol still run, the CG bookkeeping does not.  Out of line, so the main path of the kernels
// that end with it keeps its registers (pass a __grid_constant__ kernel parameter or any other
// addressable RedArgs).
static __device__ __noinline__ void red_complete(const RedArgs &R, int nblk, int vb, bool skip) {
  __shared__ int s_last;
  const int G = blockDim.x;
  const int g = vb / G;
  __threadfence();
  double a0 = 0.0, a1 = 0.0;
  const int i = g * G + threadIdx.x;
  if (i < nblk && threadIdx.x < G) {
    a0 = __ldcg(&R.part[2 * i]);
    a1 = __ldcg(&R.part[2 * i + 1]);
  }
  block_sum2(a0, a1);
  const int ngroups = (nblk + G - 1) / G;
  if (ngroups > 1) {  // (one group: its sum is the total -- no second level, three round trips fewer)
    if (threadIdx.x == 0) {
      R.cnt[1 + g] = 0u;
      R.part2[2 * g] = a0;
      R.part2[2 * g + 1] = a1;
      __threadfence();
      s_last = atomicAdd(&R.cnt[0], 1u) == (unsigned)(ngroups - 1);
    }
    __syncthreads();
    if (!s_last) return;
    __threadfence();
    a0 = a1 = 0.0;
    for (int j = threadIdx.x; j < ngroups; j += G) {
      a0 += __ldcg(&R.part2[2 * j]);
      a1 += __ldcg(&R.part2[2 * j + 1]);
    }
    block_sum2(a0, a1);
  }
  if (threadIdx.x == 0) {
    R.cnt[1 + g] = 0u;
    R.cnt[0] = 0u;
    double v[2] = {a0, a1};
    if (R.peer) peer_sum_dev(R.pa, v, R.n, R.seq);
    R.res[R.slot] = v[0];
    if (R.n > 1) R.res[R.slot + 1] = v[1];
    if (R.host) {
      R.host[0] = v[0];
      if (R.n > 1) R.host[1] = v[1];
      __threadfence_system();
      *(volatile unsigned *)R.host_flag = R.token;
    }
    if (R.has_cg && !skip) cg_record(R.cg, v[0]);
  }
}

// Both halves at the end of a kernel (nothing left to store).
__device__ __forceinline__ void red_finish(const RedArgs &R, int nblk, int vb, double v0, double v1, bool skip) {
  if (red_arrive(R, nblk, vb, v0, v1)) red_complete(R, nblk, vb, skip);
}

// the skip test of a CG kernel of iteration `iter` (stop == nullptr: never skip)
__device__ __forceinline__ bool cg_skip(const int *stop, int iter) { return stop && __ldcg(stop) < iter; }
#endif

}  // namespace qdpb
