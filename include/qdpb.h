/*
 * qdpb.h -- C ABI of the B200-native QDP hot path (arXiv:1408.5925, "A Framework for
 * Lattice QCD Calculations on GPUs").
 *
 * The library (paper_1408_5925_b200/libqdpb.so) implements, in hand-written sm_100a
 * CUDA kernels, the data-parallel operations the paper's QDP-JIT/PTX layer accelerates:
 * lattice fields in a coalesced structure-of-arrays layout (section
 * III-B), the circular shift (section II-C), the Wilson hopping term
 * (section VIII-C), the clover term (eq. (1)), the
 * lattice BLAS (norm2 / innerProduct / axpy) and an even-odd CG solve of the Wilson(-clover)
 * operator, with the sub-grid decomposition and inner/face overlap of
 * section V.
 *
 * Conventions:
 *  - mu = 0,1,2,3 <-> x,y,z,t (R2); gamma matrices in the DeGrand-Rossi chiral basis (R1).
 *  - All global and local extents are even and >= 2 (R6).  Local site order is
 *    lexicographic s = x + Lx(y + Ly(z + Lz t)) (R7); parity = (X+Y+Z+T) mod 2 of the
 *    GLOBAL coordinates, which equals the local parity (local origins are even); the
 *    checkerboard index of a site of parity p is cb = s >> 1 (R7).
 *  - Boundary conditions are periodic in every direction (R5).
 *  - Rank r has processor coordinates r = p0 + P0(p1 + P1(p2 + P2 p3)) in the grid P.
 *
 * Host canonical layouts (the contract of import/export; the device layout is opaque):
 *  - QDP_FERMION: REAL[sites][4 spin][3 colour][2 re/im]; subset QDP_ALL: all local sites
 *    in lexicographic order; subset QDP_EVEN/QDP_ODD: the sites of that parity in cb order.
 *  - QDP_GAUGE:   REAL[local sites][4 mu][3 row][3 col][2]   (always subset QDP_ALL; U_mu(x)).
 *  - QDP_CLOVER:  REAL[sites][12][12][2] dense, index i = 3*spin + colour; sites as for
 *    fermions.  Only the two chiral 6x6 blocks (spins {0,1}, {2,3}) are stored on the
 *    device, as 6 real diagonal + 15 complex lower-triangle numbers each (PAPER.md:228-230,
 *    Table I lower part); import reads the diagonal and the strictly-lower triangle of each
 *    block and ignores the rest.
 *  REAL is double for QDP_F64 fields and float for QDP_F32 fields.
 *
 * Ownership: fields from qdp_field_alloc own their device memory (released by
 * qdp_field_free); fields from qdp_field_wrap borrow caller memory (never freed by the
 * library; >= 256-byte aligned, at least qdp_field_bytes() device bytes).
 *
 * Streams: every call enqueues its kernels on the context stream (qdp_init / qdp_set_stream)
 * and returns without synchronising, EXCEPT calls that return host values (import, export,
 * norm2, inner_product, cg_solve, clover_build), which return once their values are final:
 * they synchronise the stream, except norm2 / inner_product on a one-rank context, whose
 * reduction kernel stores the result and a completion token into mapped host memory in its
 * final block -- the call polls for the token (a later call is ordered after that kernel on
 * the stream anyway; a launch failure is then reported by the next synchronising call).
 *
 * Errors: every entry point returns a status; 0 = QDP_OK, > 0 = warning, < 0 = error.
 * On error nothing has been enqueued and the outputs are unchanged, except QDP_ECUDA /
 * QDP_ENCCL (a device or communication failure after launch; the context should be
 * finalised).  qdp_last_error(ctx) returns a human-readable message for the last error.
 * One host thread per context.
 */
#ifndef QDPB_H
#define QDPB_H

#include <stddef.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct qdp_ctx_s *qdp_ctx;     /* one per process = one GPU: geometry, streams, comm, scratch */
typedef struct qdp_field_s *qdp_field; /* a lattice field on one context */

enum { QDP_F64 = 0, QDP_F32 = 1 };                             /* precision */
/* kind.  QDP_GAUGE12 is a gauge field stored as the first two rows of each link, the third
 * rebuilt as conj(row0 x row1) on use ("reconstruction of SU(3) matrices from 12 real
 * numbers"): same host layout as QDP_GAUGE; import rejects (QDP_EINVAL) links
 * whose third row differs from conj(row0 x row1) by more than 1e-10 (F64) / 1e-5 (F32), and
 * export returns the rebuilt third row.  Accepted wherever a QDP_GAUGE field is. */
enum { QDP_FERMION = 0, QDP_GAUGE = 1, QDP_CLOVER = 2, QDP_GAUGE12 = 3,
       QDP_COLORMATRIX = 4, /* LatticeColorMatrix (Table I): REAL[sites][3 row][3 col][2] */
       QDP_SPINMATRIX = 5   /* LatticeSpinMatrix  (Table I): REAL[sites][4 row][4 col][2] */ };
enum { QDP_ALL = -1, QDP_EVEN = 0, QDP_ODD = 1 };             /* subset / parity */
enum { QDP_FORWARD = +1, QDP_BACKWARD = -1 };                 /* shift direction */

enum {
  QDP_OK = 0,
  QDP_NOT_CONVERGED = 1, /* cg_solve hit maxit; x holds the last iterate */
  QDP_EINVAL = -1,       /* bad argument (NULL handle, bad enum, bad mu/sign, wrong kind/subset) */
  QDP_ESHAPE = -2,       /* odd / non-divisible dims, byte-count mismatch, fields on different contexts */
  QDP_EPREC = -3,        /* precision mismatch between fields */
  QDP_EALIAS = -4,       /* an output aliases an input where that is not allowed */
  QDP_ENOMEM = -5,       /* device or host allocation failed */
  QDP_ECUDA = -6,        /* CUDA error */
  QDP_ENCCL = -7,        /* NCCL error or NCCL unavailable for nranks > 1 */
  QDP_ESINGULAR = -8,    /* a clover block has a zero pivot */
  QDP_EUNSUPPORTED = -9  /* valid request this build does not implement */
};

/* ---- context ---------------------------------------------------------------------- */

/* NCCL unique id (rank 0 only; the caller broadcasts the 128 bytes to all ranks). */
int qdp_get_unique_id(unsigned char id[128]);

/* Create a context for this rank.  global_dims: the global lattice; proc_grid: ranks per
 * dimension (product == nranks); local dims = global/proc, all even (else QDP_ESHAPE).
 * id: NCCL id from qdp_get_unique_id (ignored, may be NULL, when nranks == 1).
 * cuda_stream: cudaStream_t to enqueue on (NULL: the context creates its own).
 * The current CUDA device at the time of the call is the context's device. */
int qdp_init(const int global_dims[4], const int proc_grid[4], int rank, int nranks,
             const unsigned char *id, void *cuda_stream, qdp_ctx *out);
/* Host allgather supplied by the caller for qdp_init_peer: every rank passes `bytes` bytes
 * in `send`; `recv` (nranks * bytes) receives all ranks' blocks in rank order.  Return 0 on
 * success.  Called collectively, only from inside qdp_init_peer. */
typedef int (*qdp_allgather_fn)(const void *send, void *recv, size_t bytes, void *user);

/* Create a context whose inter-rank communication uses peer memory only, no NCCL
 * (SURVEY.md 8(e) "B200-native upgrade"; the sub-grid decomposition of PAPER.md:93-95,
 * 208-214).  Every rank's GPU must be able to map every other rank's memory through CUDA IPC
 * (GPUs of one NVLink / NVSwitch node, or several processes sharing one GPU).  Arguments as
 * qdp_init; `allgather` (with `user`) exchanges the IPC handles during this call and is not
 * used afterwards.  Then:
 *  - dslash halos always use the peer-to-peer protocol of QDP_OPT_P2P (it cannot be turned off);
 *  - global sums (norm2, inner_product, the CG's) are one kernel per sum: each rank stores its
 *    partial into every rank's mapped board and release-signals a flag, then acquires all
 *    flags and sums in rank order (deterministic, identical on every rank);
 *  - shift faces are copied into the receiving rank's mapped mailbox by a kernel, with
 *    release/acquire flags (the mailbox holds the largest face of a fp64 gauge field).
 * At most 16 ranks (QDP_EUNSUPPORTED).  QDP_OPT_SELF_NCCL returns QDP_EUNSUPPORTED.  A flag
 * wait that exceeds ~10 s sets an error word reported as QDP_ECUDA by the next synchronising
 * call (no hang). */
int qdp_init_peer(const int global_dims[4], const int proc_grid[4], int rank, int nranks,
                  qdp_allgather_fn allgather, void *user, void *cuda_stream, qdp_ctx *out);
int qdp_finalize(qdp_ctx ctx);
int qdp_set_stream(qdp_ctx ctx, void *cuda_stream);
int qdp_synchronize(qdp_ctx ctx);
/* local_dims[4], proc_coords[4] of this rank */
int qdp_get_geometry(qdp_ctx ctx, int local_dims[4], int proc_coords[4]);

/* Options (qdp_set_option / qdp_get_option):
 *  QDP_OPT_OVERLAP    1 (default): overlap face exchange with the interior kernel
 *                     (PAPER.md:212); 0: exchange first, then compute (Fig. 6 "off").
 *  QDP_OPT_SELF_HALO  bitmask of dims with one rank that are nevertheless treated as
 *                     partitioned: faces are packed and the halo path runs, the peer being
 *                     this rank (single-GPU test mode of the multi-GPU code).
 *  QDP_OPT_PROFILE    1: bracket every launch with CUDA events (see qdp_profile_query).
 *  QDP_OPT_BLOCK      threads per block of the main dslash kernel: 0 (the build's default,
 *                     64) or a multiple of 32 up to the build's launch bound (64).
 *  QDP_OPT_DET_REDUCE 1 (default): cross-rank sums by allgather + rank-ordered sum
 *                     (deterministic); 0: ncclAllReduce.
 *  QDP_OPT_SELF_NCCL  1: self-halo dims exchange their faces with ncclSend/ncclRecv to this
 *                     rank (a one-rank communicator is created on first use; QDP_ENCCL if
 *                     NCCL cannot be loaded) instead of packing straight into the ghost
 *                     buffers -- the NCCL code path of a multi-GPU run, on one GPU. */
 /*  QDP_OPT_P2P        1: dslash halos go peer to peer instead of through NCCL: every rank
 *                     maps its neighbours' ghost buffers (CUDA IPC over NVLink / NVSwitch,
 *                     exchanged collectively at first use).  One kernel per EO dslash: the
 *                     face packing is a work queue taken by its leading blocks -- and by every
 *                     block about to wait for a ghost, so no wait depends on an unstarted block --
 *                     which store the faces straight into the neighbours' ghost slots and
 *                     release-signal a flag; the interior blocks run meanwhile; the blocks holding
 *                     face sites acquire the flags and add the remote hops; the next call acknowledges
 *                     the consumed ghosts as it starts (two slots per
 *                     face).  With QDP_OPT_OVERLAP = 0 every block waits for the ghosts first.
 *                     Self-halo dims use the same protocol on this rank.  Changing
 *                     QDP_OPT_SELF_HALO after the first dslash rebuilds the slots when every
 *                     partitioned dim is a self dim, else returns QDP_EUNSUPPORTED from the
 *                     next dslash.  A flag wait that never completes surfaces as QDP_ECUDA at
 *                     the next synchronising call.
 *  QDP_OPT_FUSE       1 (default; environment QDPB_FUSE=0 changes the default): with
 *                     QDP_OPT_P2P, packing, interior and remote hops in the one kernel above;
 *                     0: separate pack / interior / exterior kernels (comparison mode).
 *  QDP_OPT_DSLASH_VARIANT  -1 (default): the whole-lattice EO dslash launch configuration is
 *                     chosen by the paper's autotuner on the payload
 *                     launches, per (precision, gauge storage, epilogue, volume), among:
 *                     0 four threads per site (one per direction, 128-thread blocks; plain
 *                     and xpay epilogues), 1 one thread per site, 64-thread blocks, 2 one thread
 *                     per site, 32-thread blocks, 3 (fp64) one thread per site with the block's
 *                     forward links staged into shared memory by the bulk-copy engine.
 *                     0..3 force that variant where it applies (measurements).
 *  QDP_OPT_PDL        1 (default; environment QDPB_PDL=0 changes the default): the dslash,
 *                     BLAS and reduction kernels of the solvers are launched with programmatic
 *                     dependent launch, so each becomes resident while its predecessor drains
 *                     (it waits for the predecessor's completion before reading anything);
 *                     0: plain stream order.  Results are identical either way. */
enum { QDP_OPT_OVERLAP = 0, QDP_OPT_SELF_HALO = 1, QDP_OPT_PROFILE = 2, QDP_OPT_BLOCK = 3,
       QDP_OPT_DET_REDUCE = 4, QDP_OPT_SELF_NCCL = 5, QDP_OPT_AUTOTUNE = 6 /* see qdp_expr */,
       QDP_OPT_P2P = 7, QDP_OPT_FUSE = 8, QDP_OPT_DSLASH_VARIANT = 9, QDP_OPT_PDL = 10 };
int qdp_set_option(qdp_ctx ctx, int option, long value);
int qdp_get_option(qdp_ctx ctx, int option, long *value);

/* ---- fields (section II-B; Table I) ---------------------------------- */

int qdp_field_alloc(qdp_ctx ctx, int kind, int prec, int subset, qdp_field *out);
int qdp_field_wrap(qdp_ctx ctx, int kind, int prec, int subset, void *dev_ptr, size_t bytes,
                   qdp_field *out);
int qdp_field_free(qdp_field f);
/* host_bytes: size of the host canonical array; device_bytes: device footprint */
int qdp_field_bytes(qdp_ctx ctx, int kind, int prec, int subset, size_t *host_bytes,
                    size_t *device_bytes);
int qdp_field_info(const qdp_field f, int *kind, int *prec, int *subset, void **dev_ptr);
/* copy host canonical data (bytes must equal host_bytes) into the field, converting the
 * layout on the device; export is the inverse.  Host memory may be pageable or pinned. */
int qdp_field_import(qdp_field f, const void *host, size_t bytes);
int qdp_field_export(const qdp_field f, void *host, size_t bytes);
/* The same conversions from / to a DEVICE buffer holding the host canonical layout: enqueued
 * on the context stream, no synchronisation (so the caller can overlap its own host<->device
 * copies on another stream).  dev_aos must stay valid until the stream reaches the call. */
int qdp_field_import_device(qdp_field f, const void *dev_aos, size_t bytes);
int qdp_field_export_device(const qdp_field f, void *dev_aos, size_t bytes);
int qdp_field_zero(qdp_field f);
/* dst <- src (same kind/precision; subsets equal, or dst ALL and src a parity, or
 * src ALL and dst a parity: the matching parity is copied). */
int qdp_field_copy(qdp_field dst, const qdp_field src);

/* ---- data-parallel operations ---------------------------------------------------------- */

/* Circular shift (section II-C, Fig. 1; reading R4):
 *   out(x) = in(x + sign * mu^),  sign = QDP_FORWARD (+1) or QDP_BACKWARD (-1).
 * Fermion fields: in ALL -> out ALL; in parity p -> out parity 1-p.  Gauge fields: ALL.
 * Faces crossing ranks are exchanged (packed, sent, received) by the library.
 * out == in -> QDP_EALIAS. */
int qdp_shift(qdp_field out, const qdp_field in, int mu, int sign);

/* Wilson hopping term H of PAPER.md:282 (reading R3: no kappa, no 1/2):
 *   (H psi)(x) = sum_mu [(1 - gamma_mu) U_mu(x) psi(x+mu) + (1 + gamma_mu) U_mu(x-mu)^dag psi(x-mu)]
 * on the output sites of parity out_parity (QDP_EVEN / QDP_ODD), reading psi on the other
 * parity; out_parity = QDP_ALL applies H on all sites (both parity blocks; out and psi ALL).
 * out: fermion of subset out_parity or ALL (then only out_parity's block is written);
 * psi: fermion of subset 1-out_parity or ALL.  U: gauge.  Same precision (QDP_EPREC).
 * out == psi -> QDP_EALIAS. */
int qdp_dslash(qdp_field out, const qdp_field U, const qdp_field psi, int out_parity);

/* Global sums over the field's subset and all ranks (fp64 accumulation for both precisions;
 * deterministic for a fixed launch configuration and rank count):
 *   norm2(a) = sum_x |a(x)|^2 ; inner_product(a, b) = sum_x conj(a(x)) . b(x) (out[0]=re, out[1]=im). */
int qdp_norm2(const qdp_field a, double *out);
int qdp_inner_product(const qdp_field a, const qdp_field b, double out[2]);
/* y <- a x + y (complex a) on y's subset; x == y allowed. */
int qdp_axpy(double a_re, double a_im, const qdp_field x, qdp_field y);

/* Clover term (eq. (1); reading R10), the Wilson mass folded in:
 *   A(x) = (4 + mass) + 1/4 c_SW sum_{mu,nu} sigma_mu,nu F_mu,nu(x),
 *   sigma_mu,nu = [gamma_mu, gamma_nu] / (2i),  F = traceless part of (Q - Q^dag)/(8i),
 * Q the four clover leaves.  A (nullable) receives A on its subset's sites, Ainv (nullable)
 * A^{-1} on its subset's sites.  Both QDP_CLOVER fields of U's precision.  Computed in fp64
 * internally.  On a partitioned lattice the leaves' off-site links come from shifted copies
 * of U ("shifts of shifts", executed without overlap as in PAPER.md:214; 8 gauge-field
 * temporaries).  Returns QDP_ESINGULAR if a 6x6 block has a zero pivot. */
int qdp_clover_build(qdp_field A, qdp_field Ainv, const qdp_field U, double mass, double csw);
/* out(x) = A(x) in(x) on the sites of `parity` (QDP_ALL: all); out may equal in. */
int qdp_clover_apply(qdp_field out, const qdp_field A, const qdp_field in, int parity);

/* Even-odd preconditioned CGNR for M x = b, M = A - H/2 (readings R3, R12-R14):
 *   Mhat = A_oo - 1/4 H_oe A_ee^-1 H_eo ; bhat_o = b_o + 1/2 H_oe A_ee^-1 b_e ;
 *   CG on Mhat^dag Mhat x_o = Mhat^dag bhat_o from x_o = 0 ; x_e = A_ee^-1 (b_e + 1/2 H_eo x_o).
 * x, b: full (QDP_ALL) fermions; U: gauge.  A / Ainv: clover fields from qdp_clover_build
 * (A covering the odd sites, Ainv the even sites), or both NULL for Wilson (A = 4 + mass).
 * Stops when |r_k|^2 <= tol^2 |r_0|^2 (r the CGNR residual) or after maxit iterations.
 * iters (nullable): iterations done; resid_hist (nullable): resid_hist[k] = |r_k|/|r_0|
 * for k = 0..min(iters, hist_cap-1); true_resid (nullable): |b - M x| / |b|.
 * Returns QDP_OK, QDP_NOT_CONVERGED, or an error. */
int qdp_cg_solve(qdp_field x, const qdp_field b, const qdp_field U, const qdp_field A,
                 const qdp_field Ainv, double mass, double tol, int maxit, int *iters,
                 double *resid_hist, int hist_cap, double *true_resid);

/* Multi-shift CG (the solver of RHMC gauge generation, ref. [14]; reading
 * R25): solves (Mhat^dag Mhat + sigma_i) x_i = phi on the odd sites for i = 0..nshift-1 from
 * ONE Krylov space (Mhat as in qdp_cg_solve).  CG runs on the base shift sigma_0; the shifted
 * residuals are collinear, r_i = zeta_i r, and
 *   zeta_i' = zeta_i zeta_i^old a^old / [a b^old (zeta_i^old - zeta_i) + zeta_i^old a^old (1 + (sigma_i - sigma_0) a)],
 *   x_i += a zeta_i'/zeta_i p_i,  p_i = zeta_i' r + b (zeta_i'/zeta_i)^2 p_i.
 * Shift i stops being updated once zeta_i'^2 |r|^2 <= tol^2 |phi|^2; the solve ends when the
 * base system converges (status QDP_OK) or after maxit iterations (QDP_NOT_CONVERGED).
 * x[i]: nshift distinct fermions covering the odd sites (QDP_ODD or QDP_ALL; only the odd block is
 * written); phi: fermion covering the odd sites (its odd block is the source); U, A, Ainv, mass as
 * qdp_cg_solve (A covering the odd, Ainv the even sites); all one precision.  Requires
 * 1 <= nshift <= 32 and 0 <= sigma[0] <= sigma[i] (QDP_EINVAL).
 * iters: iterations; conv_iter[i] (nullable): the iteration at which shift i stopped;
 * resid_hist[k] (nullable) = |r_k| / |phi| of the base system; true_resid[i] (nullable) =
 * |phi - (Mhat^dag Mhat + sigma_i) x_i| / |phi| (two more operator applications per shift). */
int qdp_cg_solve_multishift(qdp_field *x, int nshift, const double *sigma, const qdp_field phi,
                            const qdp_field U, const qdp_field A, const qdp_field Ainv, double mass,
                            double tol, int maxit, int *iters, int *conv_iter, double *resid_hist,
                            int hist_cap, double *true_resid);

/* Mixed-precision variant of qdp_cg_solve (the reliable-update mixed-precision CG of the
 * paper's ref. [2], Clark et al.): the CGNR iteration runs on the QDP_F32 "sloppy" fields
 * U_s, A_s, Ainv_s (the same operator stored in single precision, e.g. imported from the
 * same data and built with qdp_clover_build); x, b, U, A, Ainv are QDP_F64.  When the fp32
 * residual norm falls below delta times its maximum since the last update (0 < delta < 1,
 * e.g. 0.1), the fp32 solution is added to the fp64 x and the fp64 residual is recomputed.
 * Convergence (|r|^2 <= tol^2 |r_0|^2) is tested only on such fp64 residuals.
 * resid_hist[k] holds the fp32 residual, or the fp64 one after an update; reliable
 * (nullable) returns the number of updates.  Other arguments and returns as qdp_cg_solve. */
int qdp_cg_solve_mixed(qdp_field x, const qdp_field b, const qdp_field U, const qdp_field A,
                       const qdp_field Ainv, const qdp_field U_s, const qdp_field A_s,
                       const qdp_field Ainv_s, double mass, double tol, double delta, int maxit,
                       int *iters, int *reliable, double *resid_hist, int hist_cap,
                       double *true_resid);

/* qdp_cg_solve_mixed with a 16-bit sloppy level (the half-precision reliable-update solver of
 * the paper's ref. [2]): the sloppy operator uses U (as reconstruct-12 links, int16 fixed point),
 * A_oo and A_ee^-1 converted at the start of the call to 16-bit storage (int16 with one float norm
 * per site for the clover blocks), 16-bit search directions and operator vectors (int16 with a
 * per-site norm) and fp32 residual and solution, all arithmetic in fp32; fp64 reliable updates
 * and the convergence test as qdp_cg_solve_mixed.  x, b, U, A, Ainv are QDP_F64 (A, Ainv NULL for
 * Wilson); the 16-bit copies live in the context's work space. */
int qdp_cg_solve_mixed16(qdp_field x, const qdp_field b, const qdp_field U, const qdp_field A,
                         const qdp_field Ainv, double mass, double tol, double delta, int maxit, int *iters,
                         int *reliable, double *resid_hist, int hist_cap, double *true_resid);

/* ---- site-local expressions: the test functions of PAPER.md Table II (section VI) ----------
 * One fused streaming kernel per expression, evaluated on every site of the output's subset
 * (all operands share that subset, or are QDP_ALL when the output is a parity):
 *   QDP_EXPR_LCM     out = a * b            colour matrices                  (Table II "lcm")
 *   QDP_EXPR_UPSI    out = a * b            colour matrix x fermion          ("upsi")
 *   QDP_EXPR_SPMAT   out = a * b            spin matrices                    ("spmat")
 *   QDP_EXPR_MATVEC  out = a * b + a * c    colour matrix x two fermions     ("matvec")
 *   QDP_EXPR_CLOVER  out = a * b            clover (packed blocks) x fermion ("clover")
 *   QDP_EXPR_ADJ_UPSI out = adj(a) * b      colour matrix^dag x fermion (Fig. 1's adj(u[mu])*phi,
 *                                           PAPER.md:121)
 * c is NULL except for MATVEC.  All operands have the output's precision (QDP_EPREC).
 * Block size: the paper's autotuner runs on the payload launches -- first
 * launch at 1024 threads, halved while the launch fails, then each further launch probes the
 * next smaller size until the time grows by more than 33%; the best size is kept per
 * (expression, precision, volume).  QDP_OPT_AUTOTUNE = 0 disables it (128 threads). */
enum { QDP_EXPR_LCM = 0, QDP_EXPR_UPSI = 1, QDP_EXPR_SPMAT = 2, QDP_EXPR_MATVEC = 3, QDP_EXPR_CLOVER = 4,
       QDP_EXPR_ADJ_UPSI = 5 };
int qdp_expr(int expr, qdp_field out, const qdp_field a, const qdp_field b, const qdp_field c);
/* block size the autotuner currently uses for (expr, prec) on this context's volume, and
 * whether its search has finished (1) */
int qdp_expr_block(qdp_ctx ctx, int expr, int prec, int *block, int *tuned);

/* ---- run-time generated site expressions (PAPER.md sections III-IV, 148-206; Figs. 1-3) ------
 * The paper's data-parallel expression evaluation: an expression over lattice fields becomes
 * ONE kernel, one thread per site, generated at run time from the expression's
 * tree, compiled (here by NVRTC to an sm_100a cubin), cached per context and
 * launched with the paper's block-size autotuner (as qdp_expr).
 *
 * Grammar (whitespace free-form):
 *   e := e + e | e - e | e * e | -e | (e) | number | $k | $k[mu]
 *      | adj(e) | timesI(e) | gamma(mu) | gamma5 | shift(e, mu, s)
 *   $k       operands[k]: QDP_FERMION -> spinor, QDP_COLORMATRIX -> colour matrix,
 *            QDP_SPINMATRIX -> spin matrix; QDP_GAUGE / QDP_GAUGE12 only as $k[mu] = U_mu
 *   adj      hermitian conjugate of a colour or spin matrix; timesI: i * e
 *   gamma    gamma_mu in the DeGrand-Rossi basis (reading R1), gamma5 = diag(1,1,-1,-1);
 *            only as a left factor of a spinor or spin matrix
 *   shift    e(x + s mu^), s = +1 (FORWARD) / -1 (BACKWARD) (reading R4),
 *            evaluated at the neighbouring site inside the same kernel (no temporary; shifts of
 *            shifts reach diagonal neighbours); periodic on the local lattice
 *   products: colour x colour, colour x spinor, spin x spin, spin x spinor, real x any
 * Identical subexpressions at the same site are computed once.  Example, Fig. 1:
 *   "$0[0]*shift($1,0,+1) + shift(adj($0[0])*$1,0,-1)"  with $0 a gauge field, $1 a fermion.
 *
 * qdp_jit_eval: out = expr(operands) on every site of out's subset.  All operands have out's
 * precision (QDP_EPREC); a one-parity operand must hold the parity it is read at (out's parity,
 * flipped by each odd shift displacement) and gauge operands must be QDP_ALL (QDP_EINVAL);
 * out must not alias an operand (QDP_EALIAS).  Parse and type errors: QDP_EINVAL with the
 * reason in qdp_last_error.  Shifts along dimensions reached through the halo path (P_mu > 1 or
 * self-halo): every operand read at a displacement with such components is
 * first shifted by those components with qdp_shift (faces exchanged; collective, so every rank
 * must make the same call), into temporaries kept with the cached kernel; more than 16 such
 * (operand, displacement) pairs: QDP_EUNSUPPORTED.  The first
 * call for an (expression, operand kinds, precision) compiles (~0.1-0.5 s); NVRTC missing:
 * QDP_EUNSUPPORTED.  Work counters (qdp_profile_work, class QDP_PK_BLAS): flops by the Table II
 * convention for the operations executed, compulsory bytes (each distinct field once + store).
 *
 * qdp_jit_source: the same front end without a context or GPU: writes the generated CUDA
 * source (NUL-terminated, truncated to src_cap; *src_len = bytes needed; on an error the reason
 * is written there instead; out_kind = QDP_JIT_SUM for a qdp_jit_sum expression) and the work
 * per output site of an output of subset out_subset:
 * work[0] flops, work[1] compulsory bytes (each distinct field -- for a one-parity output each
 * distinct parity block of a field -- read once, plus the store), work[2] bytes by Table II's
 * convention (every leaf occurrence + the store).  compile = 1 also runs NVRTC
 * (no GPU needed).
 * qdp_jit_stats: kernels compiled on this context and the seconds spent generating, compiling
 * and loading them (the paper's JIT overhead). */
#define QDP_JIT_MAX_OPERANDS 8
#define QDP_JIT_SUM (-1) /* qdp_jit_source out_kind of a qdp_jit_sum expression */
int qdp_jit_eval(qdp_field out, const char *expr, const qdp_field *operands, int n_operands);
int qdp_jit_source(const char *expr, int out_kind, int out_subset, int prec, const int *operand_kinds,
                   int n_operands, char *src, size_t src_cap, size_t *src_len, double work[3], int compile);
int qdp_jit_stats(qdp_ctx ctx, int *kernels, double *seconds);
/* Global sums of site expressions (QDP++'s sum(), PAPER.md:95 global sums): out[0] + i out[1] =
 * sum over the sites of `subset` (QDP_ALL / QDP_EVEN / QDP_ODD) of a complex-scalar expression,
 * built with
 *   trace(e)                  trace of a colour or spin matrix
 *   localNorm2(e)             sum of |component|^2 of a field (a complex scalar with zero imaginary part)
 *   localInnerProduct(a, b)   sum of conj(a_i) b_i over the components (conjugate-linear in a)
 *   real(z)                   z with its imaginary part dropped
 * and the operators above (complex scalars add, subtract, multiply, scale, timesI).  E.g. the
 * plaquette: "real(trace($0[0]*shift($0[1],0,+1)*adj(shift($0[0],1,+1))*adj($0[1])))".
 * Accumulated in fp64 (per-thread, block partials, one fixed-order final pass, rank-ordered
 * cross-rank sum: deterministic for a fixed rank count), 256-thread blocks.  Collective across
 * ranks.  Errors as qdp_jit_eval; the output-parity rule applies with out's parity = subset. */
int qdp_jit_sum(qdp_ctx ctx, const char *expr, const qdp_field *operands, int n_operands, int subset, double out[2]);

/* ---- diagnostics ---------------------------------------------------------------------- */

const char *qdp_strerror(int status);
const char *qdp_last_error(qdp_ctx ctx);

/* Kernel classes for profiling and launch counting. */
enum { QDP_PK_DSLASH = 0,  /* interior / whole-lattice dslash */
       QDP_PK_DSLASH_EXT,  /* exterior (face) dslash */
       QDP_PK_PACK,        /* face packing */
       QDP_PK_BLAS,        /* axpy / xpay / fused CG updates */
       QDP_PK_REDUCE,      /* norm2 / inner product (both passes) */
       QDP_PK_CLOVER,      /* clover apply / build */
       QDP_PK_SHIFT,       /* shift */
       QDP_PK_LAYOUT,      /* import / export / copy / zero */
       QDP_PK_MSHIFT,      /* multi-shift CG: the update pass over all shifts */
       QDP_PK_COUNT };
/* launches: kernels launched in this class since the last reset (always counted);
 * total_ms: sum of their CUDA-event durations (only while QDP_OPT_PROFILE = 1; resolving
 * the events synchronises the stream).  kernel_class = -1: totals over all classes. */
int qdp_profile_query(qdp_ctx ctx, int kernel_class, long *launches, double *total_ms);
/* Algorithmic work of the launches counted above (always counted): flops by the paper's
 * Table II convention (complex mul 6, complex add 2, real x complex 2; PAPER.md:71-79;
 * hopping term 1320 per output site, clover apply 504) and compulsory bytes (every
 * operand read once and every result written once; for the dslash: 8 links, the input
 * spinor once, the output once = 1536 B/site fp64, 768 fp32).  DESIGN.md "Accounting". */
int qdp_profile_work(qdp_ctx ctx, int kernel_class, double *flops, double *bytes);
int qdp_profile_reset(qdp_ctx ctx);

#ifdef __cplusplus
}
#endif
#endif /* QDPB_H */
