// capi.cu -- the extern "C" entry points of include/qdpb.h: argument validation, field
// objects, geometry, scratch management, launch bookkeeping, dispatch to the kernels.
#include <stdarg.h>
#include <stdio.h>
#include <string.h>

#include <algorithm>

#include "internal.h"

using namespace qdpb;

namespace qdpb {

int set_error(qdp_ctx ctx, int status, const char *fmt, ...) {
  if (ctx) {
    char buf[512];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof(buf), fmt, ap);
    va_end(ap);
    ctx->last_error = buf;
  }
  return status;
}

int cuda_check(qdp_ctx ctx, cudaError_t e, const char *what) {
  return set_error(ctx, QDP_ECUDA, "%s: %s", what, cudaGetErrorString(e));
}

static cudaEvent_t pool_event(qdp_ctx ctx) {
  if (!ctx->event_pool.empty()) {
    cudaEvent_t e = ctx->event_pool.back();
    ctx->event_pool.pop_back();
    return e;
  }
  cudaEvent_t e = nullptr;
  cudaEventCreate(&e);
  return e;
}

void prof_begin(qdp_ctx ctx, int cls, ProfEvent *ev) {
  ev->cls = cls;
  ev->a = ev->b = nullptr;
  ctx->launches[cls]++;
  if (ctx->profiling) {
    ev->a = pool_event(ctx);
    ev->b = pool_event(ctx);
    cudaEventRecord(ev->a, ctx->stream);
  }
}

int prof_end(qdp_ctx ctx, ProfEvent *ev) {
  cudaError_t e = cudaGetLastError();
  if (ev->a) {
    cudaEventRecord(ev->b, ctx->stream);
    ctx->pending.push_back(*ev);
  }
  if (e != cudaSuccess) return cuda_check(ctx, e, "kernel launch");
  return QDP_OK;
}

static int resolve_profile(qdp_ctx ctx) {
  if (ctx->pending.empty()) return QDP_OK;
  QDP_CUDA(ctx, cudaStreamSynchronize(ctx->stream));
  for (auto &p : ctx->pending) {
    float ms = 0.f;
    if (cudaEventElapsedTime(&ms, p.a, p.b) == cudaSuccess) ctx->prof_ms[p.cls] += ms;
    ctx->event_pool.push_back(p.a);
    ctx->event_pool.push_back(p.b);
  }
  ctx->pending.clear();
  return QDP_OK;
}

int ensure_staging(qdp_ctx ctx, size_t bytes) {
  if (ctx->staging_bytes >= bytes) return QDP_OK;
  if (ctx->staging) {
    QDP_CUDA(ctx, cudaStreamSynchronize(ctx->stream));
    cudaFree(ctx->staging);
    ctx->staging = nullptr;
    ctx->staging_bytes = 0;
  }
  if (cudaMalloc(&ctx->staging, bytes) != cudaSuccess) {
    cudaGetLastError();
    return set_error(ctx, QDP_ENOMEM, "staging buffer of %zu bytes", bytes);
  }
  ctx->staging_bytes = bytes;
  return QDP_OK;
}

int ensure_reduce(qdp_ctx ctx, int blocks) {
  if (ctx->red_capacity >= blocks) return QDP_OK;
  if (ctx->red_partials) QDP_CUDA(ctx, cudaStreamSynchronize(ctx->stream));
  cudaFree(ctx->red_partials);
  cudaFree(ctx->red_partials2);
  cudaFree(ctx->red_cnt);
  ctx->red_partials = ctx->red_partials2 = nullptr;
  ctx->red_cnt = nullptr;
  ctx->red_capacity = 0;
  blocks = std::max(blocks, 4096);
  if (cudaMalloc((void **)&ctx->red_partials, sizeof(double) * 2 * blocks) != cudaSuccess ||
      cudaMalloc((void **)&ctx->red_partials2, sizeof(double) * 2 * blocks) != cudaSuccess ||
      cudaMalloc((void **)&ctx->red_cnt, sizeof(unsigned) * (1 + blocks)) != cudaSuccess) {
    cudaGetLastError();
    return set_error(ctx, QDP_ENOMEM, "reduction partials");
  }
  QDP_CUDA(ctx, cudaMemsetAsync(ctx->red_cnt, 0, sizeof(unsigned) * (1 + blocks), ctx->stream));
  ctx->red_capacity = blocks;
  return QDP_OK;
}

int ensure_halo(qdp_ctx ctx, int prec) {
  const Geom &g = ctx->geom;
  size_t need = 0;
  for (int mu = 0; mu < 4; mu++)
    if ((g.part >> mu) & 1) {
      size_t b = (size_t)g.faceVh[mu] * 12 * (prec == QDP_F64 ? 8 : 4);
      if (b > need) need = b;
    }
  if (ctx->halo_bytes[prec] >= need) return QDP_OK;
  QDP_CUDA(ctx, cudaStreamSynchronize(ctx->stream));
  for (int mu = 0; mu < 4; mu++)
    for (int d = 0; d < 2; d++) {
      if (ctx->halo_send[prec][mu][d]) cudaFree(ctx->halo_send[prec][mu][d]);
      if (ctx->halo_recv[prec][mu][d]) cudaFree(ctx->halo_recv[prec][mu][d]);
      ctx->halo_send[prec][mu][d] = ctx->halo_recv[prec][mu][d] = nullptr;
    }
  ctx->halo_bytes[prec] = 0;
  for (int mu = 0; mu < 4; mu++)
    for (int d = 0; d < 2; d++) {
      if (cudaMalloc(&ctx->halo_send[prec][mu][d], need) != cudaSuccess ||
          cudaMalloc(&ctx->halo_recv[prec][mu][d], need) != cudaSuccess) {
        cudaGetLastError();
        return set_error(ctx, QDP_ENOMEM, "halo buffers");
      }
    }
  ctx->halo_bytes[prec] = need;
  return QDP_OK;
}

int ensure_cg_work(qdp_ctx ctx, size_t bytes) {
  if (ctx->cg_work_bytes >= bytes) return QDP_OK;
  if (ctx->cg_work) {
    QDP_CUDA(ctx, cudaStreamSynchronize(ctx->stream));
    cudaFree(ctx->cg_work);
  }
  ctx->cg_work = nullptr;
  ctx->cg_work_bytes = 0;
  if (cudaMalloc(&ctx->cg_work, bytes) != cudaSuccess) {
    cudaGetLastError();
    return set_error(ctx, QDP_ENOMEM, "CG work vectors (%zu bytes)", bytes);
  }
  ctx->cg_work_bytes = bytes;
  return QDP_OK;
}

static void update_partition(qdp_ctx ctx) {
  int part = 0;
  for (int mu = 0; mu < 4; mu++)
    if (ctx->pgrid[mu] > 1 || ((ctx->self_halo >> mu) & 1)) part |= 1 << mu;
  ctx->geom.part = part;
}

static size_t field_device_bytes(qdp_ctx ctx, int kind, int prec, int subset) {
  const size_t blk = parity_block_bytes(kind, prec, ctx->geom.stride);
  return (is_gauge(kind) || subset == QDP_ALL) ? 2 * blk : blk;
}
static size_t field_host_bytes(qdp_ctx ctx, int kind, int prec, int subset) {
  const long sites = (is_gauge(kind) || subset == QDP_ALL) ? ctx->V : ctx->geom.Vh;
  return (size_t)sites * host_site_reals(kind) * (prec == QDP_F64 ? 8 : 4);
}

}  // namespace qdpb

static bool valid_kind(int k) { return k >= QDP_FERMION && k <= QDP_SPINMATRIX; }
static bool valid_prec(int p) { return p == QDP_F64 || p == QDP_F32; }
static bool valid_subset(int s) { return s == QDP_ALL || s == QDP_EVEN || s == QDP_ODD; }

// ---------------------------------------------------------------------------- context
extern "C" int qdp_get_unique_id(unsigned char id[128]) {
  if (!id) return QDP_EINVAL;
  return comm_get_unique_id(id);
}

// Everything of a context but its communicator.
static int ctx_create(const int global_dims[4], const int proc_grid[4], int rank, int nranks, void *cuda_stream,
                      qdp_ctx *out) {
  if (!global_dims || !proc_grid || !out) return QDP_EINVAL;
  *out = nullptr;
  if (nranks < 1 || rank < 0 || rank >= nranks) return QDP_EINVAL;
  long prod = 1;
  for (int mu = 0; mu < 4; mu++) {
    if (proc_grid[mu] < 1 || global_dims[mu] < 2) return QDP_ESHAPE;
    if (global_dims[mu] % proc_grid[mu]) return QDP_ESHAPE;
    const int l = global_dims[mu] / proc_grid[mu];
    if (l < 2 || (l & 1)) return QDP_ESHAPE;  // reading R6: every local extent even
    prod *= proc_grid[mu];
  }
  if (prod != nranks) return QDP_ESHAPE;
  long V = 1;
  for (int mu = 0; mu < 4; mu++) V *= global_dims[mu] / proc_grid[mu];
  if (V / 2 > (1L << 30)) return QDP_ESHAPE;

  qdp_ctx c = new qdp_ctx_s();
  memcpy(c->gdims, global_dims, sizeof(c->gdims));
  memcpy(c->pgrid, proc_grid, sizeof(c->pgrid));
  c->rank = rank;
  c->nranks = nranks;
  int r = rank;
  for (int mu = 0; mu < 4; mu++) {
    c->pcoord[mu] = r % proc_grid[mu];
    r /= proc_grid[mu];
  }
  for (int mu = 0; mu < 4; mu++)
    for (int d = 0; d < 2; d++) {
      int pc[4];
      memcpy(pc, c->pcoord, sizeof(pc));
      pc[mu] = (pc[mu] + (d ? 1 : -1) + proc_grid[mu]) % proc_grid[mu];
      c->neighbour[mu][d] = pc[0] + proc_grid[0] * (pc[1] + proc_grid[1] * (pc[2] + proc_grid[2] * pc[3]));
    }
  Geom &g = c->geom;
  for (int mu = 0; mu < 4; mu++) g.L[mu] = global_dims[mu] / proc_grid[mu];
  g.Lh0 = g.L[0] / 2;
  c->V = V;
  g.Vh = (int)(V / 2);
  g.stride = (g.Vh + 63) / 64 * 64;
  for (int mu = 0; mu < 4; mu++) g.faceVh[mu] = (int)(V / g.L[mu] / 2);
  update_partition(c);
  if (const char *fe = getenv("QDPB_FUSE")) c->fuse = atoi(fe) ? 1 : 0;
  if (const char *pe = getenv("QDPB_PDL")) c->pdl = atoi(pe) ? 1 : 0;

  int rc = QDP_OK;
  cudaError_t e = cudaGetDevice(&c->device);
  if (e != cudaSuccess) rc = cuda_check(c, e, "cudaGetDevice");
  if (!rc) {
    if (cuda_stream) {
      c->stream = (cudaStream_t)cuda_stream;
    } else {
      e = cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking);
      c->own_stream = true;
      if (e != cudaSuccess) rc = cuda_check(c, e, "cudaStreamCreate");
    }
  }
  if (!rc && (e = cudaStreamCreateWithFlags(&c->comm_stream, cudaStreamNonBlocking)) != cudaSuccess)
    rc = cuda_check(c, e, "comm stream");
  if (!rc && ((e = cudaEventCreateWithFlags(&c->ev_packed, cudaEventDisableTiming)) != cudaSuccess ||
              (e = cudaEventCreateWithFlags(&c->ev_comm, cudaEventDisableTiming)) != cudaSuccess))
    rc = cuda_check(c, e, "events");
  if (!rc && (e = cudaMalloc((void **)&c->red_result, 64 * sizeof(double))) != cudaSuccess) rc = cuda_check(c, e, "scalars");
  if (!rc && (e = cudaMemsetAsync(c->red_result, 0, 64 * sizeof(double), c->stream)) != cudaSuccess) rc = cuda_check(c, e, "scalars");
  if (!rc && (e = cudaMalloc((void **)&c->red_gather, 8 * sizeof(double) * nranks)) != cudaSuccess) rc = cuda_check(c, e, "gather");
  if (!rc && (e = cudaMallocHost((void **)&c->host_pinned, 64 * sizeof(double))) != cudaSuccess) rc = cuda_check(c, e, "pinned");
  if (rc) {
    qdp_finalize(c);
    return rc;
  }
  *out = c;
  return QDP_OK;
}

extern "C" int qdp_init(const int global_dims[4], const int proc_grid[4], int rank, int nranks, const unsigned char *id,
                        void *cuda_stream, qdp_ctx *out) {
  if (!out) return QDP_EINVAL;
  qdp_ctx c = nullptr;
  int rc = ctx_create(global_dims, proc_grid, rank, nranks, cuda_stream, &c);
  if (rc) return rc;
  if ((rc = comm_init(c, id))) {
    qdp_finalize(c);
    return rc;
  }
  *out = c;
  return QDP_OK;
}

extern "C" int qdp_init_peer(const int global_dims[4], const int proc_grid[4], int rank, int nranks,
                             qdp_allgather_fn allgather, void *user, void *cuda_stream, qdp_ctx *out) {
  if (!out || !allgather) return QDP_EINVAL;
  *out = nullptr;
  qdp_ctx c = nullptr;
  int rc = ctx_create(global_dims, proc_grid, rank, nranks, cuda_stream, &c);
  if (rc) return rc;
  c->allgather = allgather;
  c->allgather_user = user;
  c->p2p_on = 1;
  if (!rc) rc = peer_init(c);
  if (!rc) rc = p2p_setup_all(c);
  c->allgather = nullptr;  // set-up done: the callback is never called again
  c->allgather_user = nullptr;
  if (rc) {
    qdp_finalize(c);
    return rc;
  }
  *out = c;
  return QDP_OK;
}

extern "C" int qdp_finalize(qdp_ctx c) {
  if (!c) return QDP_EINVAL;
  if (c->stream) cudaStreamSynchronize(c->stream);
  resolve_profile(c);
  jit_release(c);
  tune_release(c);
  for (int q = 0; q < 2; q++)
    if (c->fuse_perm[q]) cudaFree(c->fuse_perm[q]);
  if (c->fuse_slabs) cudaFree(c->fuse_slabs);
  p2p_destroy(c);
  peer_destroy(c);
  comm_destroy(c);
  for (auto e : c->event_pool) cudaEventDestroy(e);
  if (c->ev_packed) cudaEventDestroy(c->ev_packed);
  if (c->ev_comm) cudaEventDestroy(c->ev_comm);
  for (int p = 0; p < 2; p++)
    for (int mu = 0; mu < 4; mu++)
      for (int d = 0; d < 2; d++) {
        if (c->halo_send[p][mu][d]) cudaFree(c->halo_send[p][mu][d]);
        if (c->halo_recv[p][mu][d]) cudaFree(c->halo_recv[p][mu][d]);
      }
  if (c->staging) cudaFree(c->staging);
  if (c->cg_work) cudaFree(c->cg_work);
  if (c->red_partials) cudaFree(c->red_partials);
  if (c->red_partials2) cudaFree(c->red_partials2);
  if (c->red_cnt) cudaFree(c->red_cnt);
  if (c->cg_hist) cudaFreeHost(c->cg_hist);
  if (c->cg_stop) cudaFree(c->cg_stop);
  if (c->red_result) cudaFree(c->red_result);
  if (c->red_gather) cudaFree(c->red_gather);
  if (c->host_pinned) cudaFreeHost(c->host_pinned);
  if (c->comm_stream) cudaStreamDestroy(c->comm_stream);
  if (c->own_stream && c->stream) cudaStreamDestroy(c->stream);
  delete c;
  return QDP_OK;
}

extern "C" int qdp_set_stream(qdp_ctx c, void *s) {
  if (!c) return QDP_EINVAL;
  if (c->own_stream) {
    cudaStreamSynchronize(c->stream);
    cudaStreamDestroy(c->stream);
    c->own_stream = false;
  }
  if (!s) {
    QDP_CUDA(c, cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking));
    c->own_stream = true;
  } else {
    c->stream = (cudaStream_t)s;
  }
  return QDP_OK;
}

extern "C" int qdp_synchronize(qdp_ctx c) {
  if (!c) return QDP_EINVAL;
  QDP_CUDA(c, cudaStreamSynchronize(c->stream));
  return p2p_check(c);
}

extern "C" int qdp_get_geometry(qdp_ctx c, int local_dims[4], int proc_coords[4]) {
  if (!c) return QDP_EINVAL;
  if (local_dims) memcpy(local_dims, c->geom.L, 4 * sizeof(int));
  if (proc_coords) memcpy(proc_coords, c->pcoord, 4 * sizeof(int));
  return QDP_OK;
}

extern "C" int qdp_set_option(qdp_ctx c, int opt, long v) {
  if (!c) return QDP_EINVAL;
  switch (opt) {
    case QDP_OPT_OVERLAP: c->overlap = v ? 1 : 0; return QDP_OK;
    case QDP_OPT_SELF_HALO:
      if (v < 0 || v > 15) return set_error(c, QDP_EINVAL, "self-halo mask must be in [0, 15]");
      c->self_halo = (int)v;
      update_partition(c);
      return QDP_OK;
    case QDP_OPT_PROFILE:
      if (!v) resolve_profile(c);
      c->profiling = v ? 1 : 0;
      return QDP_OK;
    case QDP_OPT_BLOCK:
      if (v < 0 || v > QDPB_DSLASH_MAXT || (v % 32))
        return set_error(c, QDP_EINVAL, "block must be a multiple of 32 <= %d", QDPB_DSLASH_MAXT);
      c->block = (int)v;
      return QDP_OK;
    case QDP_OPT_DET_REDUCE: c->det_reduce = v ? 1 : 0; return QDP_OK;
    case QDP_OPT_AUTOTUNE: c->autotune = v ? 1 : 0; return QDP_OK;
    case QDP_OPT_FUSE: c->fuse = v ? 1 : 0; return QDP_OK;
    case QDP_OPT_PDL: c->pdl = v ? 1 : 0; return QDP_OK;
    case QDP_OPT_DSLASH_VARIANT:
      if (v < -1 || v > 5) return set_error(c, QDP_EINVAL, "dslash variant must be -1 (tuned) or 0 .. 5");
      c->dslash_variant = (int)v;
      return QDP_OK;
    case QDP_OPT_P2P:
      if (c->peer) {
        if (!v) return set_error(c, QDP_EUNSUPPORTED, "p2p: always on in a peer-memory context");
        return QDP_OK;
      }
      if (v && c->nranks > 1 && !c->comm) return set_error(c, QDP_ENCCL, "p2p: needs the NCCL communicator for setup");
      c->p2p_on = v ? 1 : 0;
      return QDP_OK;
    case QDP_OPT_SELF_NCCL: {
      if (v && c->peer) return set_error(c, QDP_EUNSUPPORTED, "no NCCL in a peer-memory context");
      if (v) {
        int rc = comm_ensure_self(c);
        if (rc) return rc;
      }
      c->self_nccl = v ? 1 : 0;
      return QDP_OK;
    }
  }
  return set_error(c, QDP_EINVAL, "unknown option %d", opt);
}

extern "C" int qdp_get_option(qdp_ctx c, int opt, long *v) {
  if (!c || !v) return QDP_EINVAL;
  switch (opt) {
    case QDP_OPT_OVERLAP: *v = c->overlap; return QDP_OK;
    case QDP_OPT_SELF_HALO: *v = c->self_halo; return QDP_OK;
    case QDP_OPT_PROFILE: *v = c->profiling; return QDP_OK;
    case QDP_OPT_BLOCK: *v = c->block; return QDP_OK;
    case QDP_OPT_DET_REDUCE: *v = c->det_reduce; return QDP_OK;
    case QDP_OPT_SELF_NCCL: *v = c->self_nccl; return QDP_OK;
    case QDP_OPT_AUTOTUNE: *v = c->autotune; return QDP_OK;
    case QDP_OPT_P2P: *v = c->p2p_on; return QDP_OK;
    case QDP_OPT_FUSE: *v = c->fuse; return QDP_OK;
    case QDP_OPT_PDL: *v = c->pdl; return QDP_OK;
    case QDP_OPT_DSLASH_VARIANT: *v = c->dslash_variant; return QDP_OK;
  }
  return set_error(c, QDP_EINVAL, "unknown option %d", opt);
}

// ---------------------------------------------------------------------------- fields
extern "C" int qdp_field_bytes(qdp_ctx c, int kind, int prec, int subset, size_t *hb, size_t *db) {
  if (!c || !valid_kind(kind) || !valid_prec(prec) || !valid_subset(subset)) return QDP_EINVAL;
  if (is_gauge(kind) && subset != QDP_ALL) return set_error(c, QDP_EINVAL, "gauge fields are QDP_ALL");
  if (hb) *hb = field_host_bytes(c, kind, prec, subset);
  if (db) *db = field_device_bytes(c, kind, prec, subset);
  return QDP_OK;
}

static int make_field(qdp_ctx c, int kind, int prec, int subset, void *ptr, size_t bytes, bool owned, qdp_field *out) {
  qdp_field f = new qdp_field_s();
  f->ctx = c;
  f->kind = kind;
  f->prec = prec;
  f->subset = subset;
  f->data = ptr;
  f->bytes = bytes;
  f->owned = owned;
  *out = f;
  return QDP_OK;
}

extern "C" int qdp_field_alloc(qdp_ctx c, int kind, int prec, int subset, qdp_field *out) {
  if (!c || !out) return QDP_EINVAL;
  *out = nullptr;
  int rc = qdp_field_bytes(c, kind, prec, subset, nullptr, nullptr);
  if (rc) return rc;
  const size_t bytes = field_device_bytes(c, kind, prec, subset);
  void *p = nullptr;
  if (cudaMalloc(&p, bytes) != cudaSuccess) {
    cudaGetLastError();
    return set_error(c, QDP_ENOMEM, "field of %zu bytes", bytes);
  }
  QDP_CUDA(c, cudaMemsetAsync(p, 0, bytes, c->stream));
  return make_field(c, kind, prec, subset, p, bytes, true, out);
}

extern "C" int qdp_field_wrap(qdp_ctx c, int kind, int prec, int subset, void *ptr, size_t bytes, qdp_field *out) {
  if (!c || !out || !ptr) return QDP_EINVAL;
  *out = nullptr;
  int rc = qdp_field_bytes(c, kind, prec, subset, nullptr, nullptr);
  if (rc) return rc;
  if (bytes < field_device_bytes(c, kind, prec, subset))
    return set_error(c, QDP_ESHAPE, "wrap: %zu bytes < required %zu", bytes, field_device_bytes(c, kind, prec, subset));
  if ((uintptr_t)ptr % 256) return set_error(c, QDP_EINVAL, "wrap: pointer not 256-byte aligned");
  return make_field(c, kind, prec, subset, ptr, bytes, false, out);
}

extern "C" int qdp_field_free(qdp_field f) {
  if (!f) return QDP_EINVAL;
  if (f->owned && f->data) {
    cudaStreamSynchronize(f->ctx->stream);
    cudaFree(f->data);
  }
  delete f;
  return QDP_OK;
}

extern "C" int qdp_field_info(const qdp_field f, int *kind, int *prec, int *subset, void **ptr) {
  if (!f) return QDP_EINVAL;
  if (kind) *kind = f->kind;
  if (prec) *prec = f->prec;
  if (subset) *subset = f->subset;
  if (ptr) *ptr = f->data;
  return QDP_OK;
}

extern "C" int qdp_field_import(qdp_field f, const void *host, size_t bytes) {
  if (!f || !host) return QDP_EINVAL;
  qdp_ctx c = f->ctx;
  const size_t hb = field_host_bytes(c, f->kind, f->prec, f->subset);
  if (bytes != hb) return set_error(c, QDP_ESHAPE, "import: %zu bytes, expected %zu", bytes, hb);
  int rc;
  if ((rc = ensure_staging(c, hb))) return rc;
  QDP_CUDA(c, cudaMemcpyAsync(c->staging, host, hb, cudaMemcpyHostToDevice, c->stream));
  if ((rc = layout_import(f, c->staging))) return rc;
  QDP_CUDA(c, cudaStreamSynchronize(c->stream));
  return QDP_OK;
}

extern "C" int qdp_field_export(const qdp_field f, void *host, size_t bytes) {
  if (!f || !host) return QDP_EINVAL;
  qdp_ctx c = f->ctx;
  const size_t hb = field_host_bytes(c, f->kind, f->prec, f->subset);
  if (bytes != hb) return set_error(c, QDP_ESHAPE, "export: %zu bytes, expected %zu", bytes, hb);
  int rc;
  if ((rc = ensure_staging(c, hb))) return rc;
  if ((rc = layout_export(f, c->staging))) return rc;
  QDP_CUDA(c, cudaMemcpyAsync(host, c->staging, hb, cudaMemcpyDeviceToHost, c->stream));
  QDP_CUDA(c, cudaStreamSynchronize(c->stream));
  return QDP_OK;
}

extern "C" int qdp_field_import_device(qdp_field f, const void *dev_aos, size_t bytes) {
  if (!f || !dev_aos) return QDP_EINVAL;
  qdp_ctx c = f->ctx;
  const size_t hb = field_host_bytes(c, f->kind, f->prec, f->subset);
  if (bytes != hb) return set_error(c, QDP_ESHAPE, "import_device: %zu bytes, expected %zu", bytes, hb);
  return layout_import(f, dev_aos);
}

extern "C" int qdp_field_export_device(const qdp_field f, void *dev_aos, size_t bytes) {
  if (!f || !dev_aos) return QDP_EINVAL;
  qdp_ctx c = f->ctx;
  const size_t hb = field_host_bytes(c, f->kind, f->prec, f->subset);
  if (bytes != hb) return set_error(c, QDP_ESHAPE, "export_device: %zu bytes, expected %zu", bytes, hb);
  return layout_export(f, dev_aos);
}

extern "C" int qdp_field_zero(qdp_field f) {
  if (!f) return QDP_EINVAL;
  qdp_ctx c = f->ctx;
  QDP_CUDA(c, cudaMemsetAsync(f->data, 0, field_device_bytes(c, f->kind, f->prec, f->subset), c->stream));
  return QDP_OK;
}

// parity block `par` of field f (nullptr if absent)
static char *block_of(const qdp_field f, int par) {
  if (is_gauge(f->kind)) return nullptr;
  const size_t blk = parity_block_bytes(f->kind, f->prec, f->ctx->geom.stride);
  if (f->subset == QDP_ALL) return (char *)f->data + par * blk;
  return f->subset == par ? (char *)f->data : nullptr;
}

static int check_pair(const qdp_field a, const qdp_field b) {
  if (a->ctx != b->ctx) return set_error(a->ctx, QDP_ESHAPE, "fields on different contexts");
  if (a->prec != b->prec) return set_error(a->ctx, QDP_EPREC, "precision mismatch");
  return QDP_OK;
}

extern "C" int qdp_field_copy(qdp_field dst, const qdp_field src) {
  if (!dst || !src) return QDP_EINVAL;
  int rc;
  if ((rc = check_pair(dst, src))) return rc;
  qdp_ctx c = dst->ctx;
  if (dst->kind != src->kind) return set_error(c, QDP_EINVAL, "copy: kind mismatch");
  if (dst == src || dst->data == src->data) return QDP_OK;
  if (is_gauge(dst->kind) || dst->subset == src->subset) {
    QDP_CUDA(c, cudaMemcpyAsync(dst->data, src->data, field_device_bytes(c, dst->kind, dst->prec, dst->subset),
                                cudaMemcpyDeviceToDevice, c->stream));
    return QDP_OK;
  }
  const int par = dst->subset == QDP_ALL ? src->subset : dst->subset;
  char *d = block_of(dst, par), *s = block_of(src, par);
  if (!d || !s) return set_error(c, QDP_EINVAL, "copy: incompatible subsets");
  QDP_CUDA(c, cudaMemcpyAsync(d, s, parity_block_bytes(dst->kind, dst->prec, c->geom.stride), cudaMemcpyDeviceToDevice,
                              c->stream));
  return QDP_OK;
}

// ---------------------------------------------------------------------------- operations
extern "C" int qdp_shift(qdp_field out, const qdp_field in, int mu, int sign) {
  if (!out || !in) return QDP_EINVAL;
  int rc;
  if ((rc = check_pair(out, in))) return rc;
  qdp_ctx c = out->ctx;
  if (mu < 0 || mu > 3 || (sign != 1 && sign != -1)) return set_error(c, QDP_EINVAL, "shift: bad mu/sign");
  if (out->kind != in->kind || in->kind == QDP_CLOVER)
    return set_error(c, QDP_EINVAL, "shift: fermion, gauge, colour- or spin-matrix fields of one kind");
  if (out == in || out->data == in->data) return set_error(c, QDP_EALIAS, "shift: out aliases in");
  if (!is_gauge(in->kind)) {
    const bool ok = (in->subset == QDP_ALL && out->subset == QDP_ALL) ||
                    (in->subset != QDP_ALL && out->subset == 1 - in->subset);
    if (!ok) return set_error(c, QDP_EINVAL, "shift: parity p input needs a parity 1-p output");
  }
  return shift_field(c, out, in, mu, sign);
}

extern "C" int qdp_dslash(qdp_field out, const qdp_field U, const qdp_field psi, int out_parity) {
  if (!out || !U || !psi) return QDP_EINVAL;
  int rc;
  if ((rc = check_pair(out, psi)) || (rc = check_pair(out, U))) return rc;
  qdp_ctx c = out->ctx;
  if (out->kind != QDP_FERMION || psi->kind != QDP_FERMION || !is_gauge(U->kind))
    return set_error(c, QDP_EINVAL, "dslash: kinds (fermion, gauge, fermion)");
  if (!valid_subset(out_parity)) return set_error(c, QDP_EINVAL, "dslash: bad parity");
  if (out == psi || out->data == psi->data) return set_error(c, QDP_EALIAS, "dslash: out aliases psi");
  const int first = out_parity == QDP_ALL ? 0 : out_parity, last = out_parity == QDP_ALL ? 1 : out_parity;
  if (out_parity == QDP_ALL && (out->subset != QDP_ALL || psi->subset != QDP_ALL))
    return set_error(c, QDP_EINVAL, "dslash: out_parity ALL needs ALL fields");
  for (int p = first; p <= last; p++)
    if (!block_of(out, p) || !block_of(psi, 1 - p)) return set_error(c, QDP_EINVAL, "dslash: subset mismatch");
  for (int p = first; p <= last; p++) {
    DslashArgs a = {};
    a.out = block_of(out, p);
    a.psi = block_of(psi, 1 - p);
    a.U = U->data;
    a.rec12 = U->kind == QDP_GAUGE12;
    a.parity = p;
    a.epi = EPI_PLAIN;
    a.b = 1.0;
    if ((rc = dslash(c, out->prec, a))) return rc;
  }
  return QDP_OK;
}

static int read_result(qdp_ctx c, int slot, int n, double *out) {
  int rc = read_scalars(c, slot, n, out);
  if (rc) return rc;
  return c->peer ? peer_check(c) : QDP_OK;
}

extern "C" int qdp_norm2(const qdp_field a, double *out) {
  if (!a || !out) return QDP_EINVAL;
  qdp_ctx c = a->ctx;
  if (a->kind != QDP_FERMION) return set_error(c, QDP_EINVAL, "norm2: fermion fields");
  int rc;
  if ((rc = blas_norm2(c, a->prec, a->data, a->subset == QDP_ALL ? 2 : 1, 8, true))) return rc;
  if (c->nranks > 1 && !c->peer) return read_result(c, 8, 1, out);  // NCCL sum after the kernel
  if ((rc = read_red_host(c, 1, out))) return rc;  // one launch, result in mapped host memory
  return c->peer ? peer_check(c) : QDP_OK;
}

extern "C" int qdp_inner_product(const qdp_field a, const qdp_field b, double out[2]) {
  if (!a || !b || !out) return QDP_EINVAL;
  int rc;
  if ((rc = check_pair(a, b))) return rc;
  qdp_ctx c = a->ctx;
  if (a->kind != QDP_FERMION || b->kind != QDP_FERMION) return set_error(c, QDP_EINVAL, "inner: fermion fields");
  if (a->subset != b->subset) return set_error(c, QDP_EINVAL, "inner: subsets differ");
  if ((rc = blas_inner(c, a->prec, a->data, b->data, a->subset == QDP_ALL ? 2 : 1, 10, true))) return rc;
  if (c->nranks > 1 && !c->peer) return read_result(c, 10, 2, out);
  if ((rc = read_red_host(c, 2, out))) return rc;
  return c->peer ? peer_check(c) : QDP_OK;
}

extern "C" int qdp_axpy(double ar, double ai, const qdp_field x, qdp_field y) {
  if (!x || !y) return QDP_EINVAL;
  int rc;
  if ((rc = check_pair(x, y))) return rc;
  qdp_ctx c = y->ctx;
  if (x->kind != QDP_FERMION || y->kind != QDP_FERMION) return set_error(c, QDP_EINVAL, "axpy: fermion fields");
  if (x->subset == y->subset) return blas_axpy(c, y->prec, ar, ai, x->data, y->data, y->subset == QDP_ALL ? 2 : 1);
  if (x->subset == QDP_ALL) return blas_axpy(c, y->prec, ar, ai, block_of(x, y->subset), y->data, 1);
  return set_error(c, QDP_EINVAL, "axpy: x must cover y's subset");
}

extern "C" int qdp_clover_build(qdp_field A, qdp_field Ainv, const qdp_field U, double mass, double csw) {
  if (!U || (!A && !Ainv)) return QDP_EINVAL;
  qdp_ctx c = U->ctx;
  int rc;
  if (!is_gauge(U->kind)) return set_error(c, QDP_EINVAL, "clover_build: U must be a gauge field");
  for (qdp_field f : {A, Ainv}) {
    if (!f) continue;
    if ((rc = check_pair(f, U))) return rc;
    if (f->kind != QDP_CLOVER) return set_error(c, QDP_EINVAL, "clover_build: outputs must be clover fields");
  }
  if (A && Ainv && A->data == Ainv->data) return set_error(c, QDP_EALIAS, "clover_build: A aliases Ainv");
  int singular = 0;
  if ((rc = clover_build(c, U, A ? A->data : nullptr, A ? A->subset : 0, Ainv ? Ainv->data : nullptr,
                         Ainv ? Ainv->subset : 0, mass, csw, &singular)))
    return rc;
  if (singular) return set_error(c, QDP_ESINGULAR, "clover_build: zero pivot in a 6x6 block");
  return QDP_OK;
}

extern "C" int qdp_clover_apply(qdp_field out, const qdp_field A, const qdp_field in, int parity) {
  if (!out || !A || !in) return QDP_EINVAL;
  int rc;
  if ((rc = check_pair(out, A)) || (rc = check_pair(out, in))) return rc;
  qdp_ctx c = out->ctx;
  if (out->kind != QDP_FERMION || in->kind != QDP_FERMION || A->kind != QDP_CLOVER)
    return set_error(c, QDP_EINVAL, "clover_apply: kinds (fermion, clover, fermion)");
  if (!valid_subset(parity)) return set_error(c, QDP_EINVAL, "clover_apply: bad parity");
  const int first = parity == QDP_ALL ? 0 : parity, last = parity == QDP_ALL ? 1 : parity;
  for (int p = first; p <= last; p++) {
    char *o = block_of(out, p), *i = block_of(in, p), *a = block_of(A, p);
    if (!o || !i || !a) return set_error(c, QDP_EINVAL, "clover_apply: subset mismatch");
  }
  for (int p = first; p <= last; p++)
    if ((rc = clover_apply(c, out->prec, block_of(out, p), block_of(A, p), block_of(in, p), 1))) return rc;
  return QDP_OK;
}

extern "C" int qdp_cg_solve(qdp_field x, const qdp_field b, const qdp_field U, const qdp_field A, const qdp_field Ainv,
                            double mass, double tol, int maxit, int *iters, double *resid_hist, int hist_cap,
                            double *true_resid) {
  if (!x || !b || !U) return QDP_EINVAL;
  int rc;
  if ((rc = check_pair(x, b)) || (rc = check_pair(x, U))) return rc;
  qdp_ctx c = x->ctx;
  if (x->kind != QDP_FERMION || b->kind != QDP_FERMION || !is_gauge(U->kind))
    return set_error(c, QDP_EINVAL, "cg: kinds (fermion, fermion, gauge)");
  if (x->subset != QDP_ALL || b->subset != QDP_ALL) return set_error(c, QDP_EINVAL, "cg: x and b must be QDP_ALL");
  if (x->data == b->data) return set_error(c, QDP_EALIAS, "cg: x aliases b");
  if ((A == nullptr) != (Ainv == nullptr)) return set_error(c, QDP_EINVAL, "cg: give both A and Ainv, or neither");
  if (A) {
    if ((rc = check_pair(x, A)) || (rc = check_pair(x, Ainv))) return rc;
    if (A->kind != QDP_CLOVER || Ainv->kind != QDP_CLOVER) return set_error(c, QDP_EINVAL, "cg: A, Ainv must be clover");
    if (!block_of(A, 1) || !block_of(Ainv, 0)) return set_error(c, QDP_EINVAL, "cg: A must cover odd, Ainv even sites");
    if (true_resid && A->subset != QDP_ALL) return set_error(c, QDP_EINVAL, "cg: true_resid needs A on all sites");
  }
  if (maxit < 0 || !(tol >= 0)) return set_error(c, QDP_EINVAL, "cg: bad tol/maxit");
  return cg_solve(x, b, U, A, Ainv, mass, tol, maxit, iters, resid_hist, hist_cap, true_resid);
}

extern "C" int qdp_cg_solve_multishift(qdp_field *x, int nshift, const double *sigma, const qdp_field phi,
                                       const qdp_field U, const qdp_field A, const qdp_field Ainv, double mass,
                                       double tol, int maxit, int *iters, int *conv_iter, double *resid_hist,
                                       int hist_cap, double *true_resid) {
  if (!x || !sigma || !phi || !U) return QDP_EINVAL;
  qdp_ctx c = phi->ctx;
  int rc;
  if (nshift < 1 || nshift > QDPB_MAX_SHIFTS)
    return set_error(c, QDP_EINVAL, "multishift: 1 <= nshift <= %d", QDPB_MAX_SHIFTS);
  if ((rc = check_pair(phi, U))) return rc;
  if (phi->kind != QDP_FERMION || !is_gauge(U->kind)) return set_error(c, QDP_EINVAL, "multishift: kinds (fermion, gauge)");
  if (!block_of(phi, 1)) return set_error(c, QDP_EINVAL, "multishift: phi must cover the odd sites");
  for (int i = 0; i < nshift; i++) {
    if (!x[i]) return QDP_EINVAL;
    if ((rc = check_pair(phi, x[i]))) return rc;
    if (x[i]->kind != QDP_FERMION || !block_of(x[i], 1))
      return set_error(c, QDP_EINVAL, "multishift: x[%d] must be a fermion covering the odd sites", i);
    if (x[i]->data == phi->data) return set_error(c, QDP_EALIAS, "multishift: x[%d] aliases phi", i);
    for (int j = 0; j < i; j++)
      if (x[j]->data == x[i]->data) return set_error(c, QDP_EALIAS, "multishift: x[%d] aliases x[%d]", i, j);
    if (!(sigma[i] >= 0.0) || sigma[i] < sigma[0])
      return set_error(c, QDP_EINVAL, "multishift: need 0 <= sigma[0] <= sigma[i]");
  }
  if ((A == nullptr) != (Ainv == nullptr)) return set_error(c, QDP_EINVAL, "multishift: give both A and Ainv, or neither");
  if (A) {
    if ((rc = check_pair(phi, A)) || (rc = check_pair(phi, Ainv))) return rc;
    if (A->kind != QDP_CLOVER || Ainv->kind != QDP_CLOVER) return set_error(c, QDP_EINVAL, "multishift: A, Ainv clover");
    if (!block_of(A, 1) || !block_of(Ainv, 0)) return set_error(c, QDP_EINVAL, "multishift: A odd, Ainv even sites");
  }
  if (maxit < 0 || !(tol >= 0)) return set_error(c, QDP_EINVAL, "multishift: bad tol/maxit");
  return cg_solve_multishift(x, nshift, sigma, phi, U, A, Ainv, mass, tol, maxit, iters, conv_iter, resid_hist,
                             hist_cap, true_resid);
}

extern "C" int qdp_cg_solve_mixed(qdp_field x, const qdp_field b, const qdp_field U, const qdp_field A,
                                  const qdp_field Ainv, const qdp_field Us, const qdp_field As, const qdp_field Ainvs,
                                  double mass, double tol, double delta, int maxit, int *iters, int *reliable,
                                  double *resid_hist, int hist_cap, double *true_resid) {
  if (!x || !b || !U || !Us) return QDP_EINVAL;
  qdp_ctx c = x->ctx;
  int rc;
  if (x->prec != QDP_F64 || b->prec != QDP_F64 || U->prec != QDP_F64)
    return set_error(c, QDP_EPREC, "cg_mixed: x, b, U must be QDP_F64");
  if (Us->prec != QDP_F32) return set_error(c, QDP_EPREC, "cg_mixed: the sloppy fields must be QDP_F32");
  if (Us->ctx != c || !is_gauge(Us->kind)) return set_error(c, QDP_EINVAL, "cg_mixed: U_s must be a gauge field");
  if ((A == nullptr) != (As == nullptr) || (A == nullptr) != (Ainvs == nullptr))
    return set_error(c, QDP_EINVAL, "cg_mixed: give A, Ainv, A_s, Ainv_s together, or none");
  if (As) {
    if (As->prec != QDP_F32 || Ainvs->prec != QDP_F32) return set_error(c, QDP_EPREC, "cg_mixed: A_s, Ainv_s must be F32");
    if (As->kind != QDP_CLOVER || Ainvs->kind != QDP_CLOVER || !block_of(As, 1) || !block_of(Ainvs, 0))
      return set_error(c, QDP_EINVAL, "cg_mixed: A_s must cover odd, Ainv_s even sites");
  }
  if (!(delta > 0 && delta < 1)) return set_error(c, QDP_EINVAL, "cg_mixed: 0 < delta < 1");
  // the fp64 fields obey the rules of qdp_cg_solve
  if ((rc = check_pair(x, b)) || (rc = check_pair(x, U))) return rc;
  if (x->kind != QDP_FERMION || b->kind != QDP_FERMION || !is_gauge(U->kind))
    return set_error(c, QDP_EINVAL, "cg_mixed: kinds (fermion, fermion, gauge)");
  if (x->subset != QDP_ALL || b->subset != QDP_ALL) return set_error(c, QDP_EINVAL, "cg_mixed: x and b must be QDP_ALL");
  if (x->data == b->data) return set_error(c, QDP_EALIAS, "cg_mixed: x aliases b");
  if ((A == nullptr) != (Ainv == nullptr)) return set_error(c, QDP_EINVAL, "cg_mixed: give both A and Ainv, or neither");
  if (A) {
    if ((rc = check_pair(x, A)) || (rc = check_pair(x, Ainv))) return rc;
    if (A->kind != QDP_CLOVER || Ainv->kind != QDP_CLOVER || !block_of(A, 1) || !block_of(Ainv, 0))
      return set_error(c, QDP_EINVAL, "cg_mixed: A must cover odd, Ainv even sites");
    if (true_resid && A->subset != QDP_ALL) return set_error(c, QDP_EINVAL, "cg_mixed: true_resid needs A on all sites");
  }
  if (maxit < 0 || !(tol >= 0)) return set_error(c, QDP_EINVAL, "cg_mixed: bad tol/maxit");
  return cg_solve_mixed(x, b, U, A, Ainv, Us, As, Ainvs, mass, tol, delta, maxit, iters, reliable, resid_hist, hist_cap,
                        true_resid);
}

extern "C" int qdp_cg_solve_mixed16(qdp_field x, const qdp_field b, const qdp_field U, const qdp_field A,
                                    const qdp_field Ainv, double mass, double tol, double delta, int maxit, int *iters,
                                    int *reliable, double *resid_hist, int hist_cap, double *true_resid) {
  if (!x || !b || !U) return QDP_EINVAL;
  qdp_ctx c = x->ctx;
  int rc;
  if (x->prec != QDP_F64 || b->prec != QDP_F64) return set_error(c, QDP_EPREC, "cg_mixed16: x, b must be QDP_F64");
  if (!(delta > 0 && delta < 1)) return set_error(c, QDP_EINVAL, "cg_mixed16: 0 < delta < 1");
  if ((rc = check_pair(x, b))) return rc;
  if (U->ctx != c || !is_gauge(U->kind)) return set_error(c, QDP_EINVAL, "cg_mixed16: U must be a gauge field");
  if (U->prec != QDP_F64) return set_error(c, QDP_EPREC, "cg_mixed16: U must be QDP_F64 (its reliable updates)");
  if (x->kind != QDP_FERMION || b->kind != QDP_FERMION)
    return set_error(c, QDP_EINVAL, "cg_mixed16: kinds (fermion, fermion, gauge)");
  if (x->subset != QDP_ALL || b->subset != QDP_ALL) return set_error(c, QDP_EINVAL, "cg_mixed16: x and b must be QDP_ALL");
  if (x->data == b->data) return set_error(c, QDP_EALIAS, "cg_mixed16: x aliases b");
  if ((A == nullptr) != (Ainv == nullptr)) return set_error(c, QDP_EINVAL, "cg_mixed16: give both A and Ainv, or neither");
  if (A) {
    if ((rc = check_pair(x, A)) || (rc = check_pair(x, Ainv))) return rc;
    if (A->kind != QDP_CLOVER || Ainv->kind != QDP_CLOVER || !block_of(A, 1) || !block_of(Ainv, 0))
      return set_error(c, QDP_EINVAL, "cg_mixed16: A must cover odd, Ainv even sites");
    if (true_resid && A->subset != QDP_ALL) return set_error(c, QDP_EINVAL, "cg_mixed16: true_resid needs A on all sites");
  }
  if (maxit < 0 || !(tol >= 0)) return set_error(c, QDP_EINVAL, "cg_mixed16: bad tol/maxit");
  return cg_solve_mixed16(x, b, U, A, Ainv, mass, tol, delta, maxit, iters, reliable, resid_hist, hist_cap, true_resid);
}

// ---------------------------------------------------------------------------- Table II expressions
extern "C" int qdp_expr(int expr, qdp_field out, const qdp_field a, const qdp_field b, const qdp_field c) {
  if (!out || !a || !b) return QDP_EINVAL;
  qdp_ctx ctx = out->ctx;
  int rc;
  if (expr < QDP_EXPR_LCM || expr > QDP_EXPR_ADJ_UPSI)
    return set_error(ctx, QDP_EINVAL, "expr: unknown expression %d", expr);
  if ((expr == QDP_EXPR_MATVEC) != (c != nullptr)) return set_error(ctx, QDP_EINVAL, "expr: c is used by MATVEC only");
  static const int kinds[6][4] = {{QDP_COLORMATRIX, QDP_COLORMATRIX, QDP_COLORMATRIX, -1},
                                  {QDP_FERMION, QDP_COLORMATRIX, QDP_FERMION, -1},
                                  {QDP_SPINMATRIX, QDP_SPINMATRIX, QDP_SPINMATRIX, -1},
                                  {QDP_FERMION, QDP_COLORMATRIX, QDP_FERMION, QDP_FERMION},
                                  {QDP_FERMION, QDP_CLOVER, QDP_FERMION, -1},
                                  {QDP_FERMION, QDP_COLORMATRIX, QDP_FERMION, -1}};
  const qdp_field f[4] = {out, a, b, c};
  for (int k = 0; k < 4; k++) {
    if (!f[k]) continue;
    if ((rc = check_pair(out, f[k]))) return rc;
    if (f[k]->kind != kinds[expr][k]) return set_error(ctx, QDP_EINVAL, "expr: operand %d has the wrong kind", k);
    if (k && !(f[k]->subset == out->subset || f[k]->subset == QDP_ALL))
      return set_error(ctx, QDP_EINVAL, "expr: operand %d does not cover the output's subset", k);
    if (k && f[k]->data == out->data) return set_error(ctx, QDP_EALIAS, "expr: out aliases operand %d", k);
  }
  return expr_eval(ctx, expr, out, a, b, c);
}

extern "C" int qdp_jit_eval(qdp_field out, const char *expr, const qdp_field *operands, int n_operands) {
  if (!out || !expr || n_operands < 0 || n_operands > QDP_JIT_MAX_OPERANDS || (n_operands && !operands))
    return QDP_EINVAL;
  qdp_ctx ctx = out->ctx;
  int rc;
  for (int k = 0; k < n_operands; k++) {
    if (!operands[k]) return set_error(ctx, QDP_EINVAL, "jit: operand %d is NULL", k);
    if ((rc = check_pair(out, operands[k]))) return rc;
    if (operands[k]->data == out->data) return set_error(ctx, QDP_EALIAS, "jit: out aliases operand %d", k);
  }
  return jit_eval(out, expr, operands, n_operands);
}

extern "C" int qdp_jit_sum(qdp_ctx ctx, const char *expr, const qdp_field *operands, int n_operands, int subset,
                           double out[2]) {
  if (!ctx || !expr || !out || n_operands < 1 || n_operands > QDP_JIT_MAX_OPERANDS || !operands) return QDP_EINVAL;
  if (subset != QDP_ALL && subset != QDP_EVEN && subset != QDP_ODD) return set_error(ctx, QDP_EINVAL, "jit sum: subset");
  int rc;
  for (int k = 0; k < n_operands; k++) {
    if (!operands[k]) return set_error(ctx, QDP_EINVAL, "jit: operand %d is NULL", k);
    if (operands[k]->ctx != ctx) return set_error(ctx, QDP_ESHAPE, "jit: operand %d on another context", k);
    if ((rc = check_pair(operands[0], operands[k]))) return rc;
  }
  if ((rc = jit_sum(ctx, expr, operands, n_operands, subset, operands[0]->prec, 12))) return rc;
  return read_result(ctx, 12, 2, out);
}

extern "C" int qdp_jit_source(const char *expr, int out_kind, int out_subset, int prec, const int *operand_kinds,
                              int n_operands, char *src, size_t src_cap, size_t *src_len, double work[3], int compile) {
  if (!expr || n_operands < 0 || n_operands > QDP_JIT_MAX_OPERANDS || (n_operands && !operand_kinds)) return QDP_EINVAL;
  std::string err;
  const int rc =
      jit_source(expr, out_kind, out_subset, prec, operand_kinds, n_operands, src, src_cap, src_len, work, compile, err);
  if (rc < 0) {  // the reason goes where the source would have
    if (src_len) *src_len = err.size() + 1;
    if (src && src_cap) {
      strncpy(src, err.c_str(), src_cap - 1);
      src[src_cap - 1] = '\0';
    }
  }
  return rc;
}

extern "C" int qdp_jit_stats(qdp_ctx ctx, int *kernels, double *seconds) {
  if (!ctx) return QDP_EINVAL;
  if (kernels) *kernels = ctx->jit_compiled;
  if (seconds) *seconds = ctx->jit_seconds;
  return QDP_OK;
}

extern "C" int qdp_expr_block(qdp_ctx c, int expr, int prec, int *block, int *tuned) {
  if (!c || expr < QDP_EXPR_LCM || expr > QDP_EXPR_ADJ_UPSI || !valid_prec(prec)) return QDP_EINVAL;
  int bl = c->autotune ? 0 : 128, done = c->autotune ? 0 : 1;
  for (const auto &kv : c->tune) {
    if (kv.first / (1L << 40) != (long)expr * 2 + prec) continue;
    bl = kv.second.state == 2 ? kv.second.best_block : kv.second.block;
    done = kv.second.state == 2;
  }
  if (block) *block = bl;
  if (tuned) *tuned = done;
  return QDP_OK;
}

// ---------------------------------------------------------------------------- diagnostics
extern "C" const char *qdp_strerror(int s) {
  switch (s) {
    case QDP_OK: return "ok";
    case QDP_NOT_CONVERGED: return "not converged";
    case QDP_EINVAL: return "invalid argument";
    case QDP_ESHAPE: return "shape mismatch";
    case QDP_EPREC: return "precision mismatch";
    case QDP_EALIAS: return "aliased arguments";
    case QDP_ENOMEM: return "out of memory";
    case QDP_ECUDA: return "CUDA error";
    case QDP_ENCCL: return "NCCL error";
    case QDP_ESINGULAR: return "singular clover block";
    case QDP_EUNSUPPORTED: return "unsupported";
  }
  return "unknown status";
}

extern "C" const char *qdp_last_error(qdp_ctx c) { return c ? c->last_error.c_str() : ""; }

extern "C" int qdp_profile_query(qdp_ctx c, int cls, long *launches, double *ms) {
  if (!c || cls < -1 || cls >= QDP_PK_COUNT) return QDP_EINVAL;
  int rc;
  if ((rc = resolve_profile(c))) return rc;
  long n = 0;
  double t = 0;
  for (int k = 0; k < QDP_PK_COUNT; k++)
    if (cls == -1 || cls == k) {
      n += c->launches[k];
      t += c->prof_ms[k];
    }
  if (launches) *launches = n;
  if (ms) *ms = t;
  return QDP_OK;
}

extern "C" int qdp_profile_work(qdp_ctx c, int cls, double *flops, double *bytes) {
  if (!c || cls < -1 || cls >= QDP_PK_COUNT) return QDP_EINVAL;
  double f = 0, b = 0;
  for (int k = 0; k < QDP_PK_COUNT; k++)
    if (cls == -1 || cls == k) {
      f += c->work_flops[k];
      b += c->work_bytes[k];
    }
  if (flops) *flops = f;
  if (bytes) *bytes = b;
  return QDP_OK;
}

extern "C" int qdp_profile_reset(qdp_ctx c) {
  if (!c) return QDP_EINVAL;
  int rc;
  if ((rc = resolve_profile(c))) return rc;
  for (int k = 0; k < QDP_PK_COUNT; k++) {
    c->launches[k] = 0;
    c->prof_ms[k] = 0;
    c->work_flops[k] = 0;
    c->work_bytes[k] = 0;
  }
  return QDP_OK;
}
