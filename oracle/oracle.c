/*
 * oracle.c -- plain, slow, obviously-correct CPU reference for the QDP hot path.
 *
 * TEST INFRASTRUCTURE ONLY.  Nothing on the product path (paper_1408_5925_b200/,
 * include/) may include, link or call this file.  Only tests/, __graft_entry__.smoke()
 * and bench.py's cpu_baseline / --impl reference leg use it (through oracle/__init__.py).
 * It shares no code, header, table or constant generator with the CUDA path.
 *
 * Arithmetic: IEEE double, C99 `double complex`.  No blocking, no spin projection,
 * no fusion: every function is the written-out definition it cites.  OpenMP is used
 * only over independent per-site loops; every reduction is a sequential Neumaier sum
 * in lexicographic site order, so results do not depend on the thread count.
 *
 * Citations are to /root/reference/PAPER.md (arXiv:1408.5925) line numbers and to
 * the readings R1..R21 listed in DESIGN.md (same numbering as SURVEY.md section 8(c)).
 *
 * Host canonical layouts:
 *   fermion  double[V][4 spin][3 colour][2]            site s = x + Lx(y + Ly(z + Lz t))
 *   gauge    double[V][4 mu][3 row][3 col][2]          U_mu(x), row-major (R9)
 *   clover   double[V][12][12][2]  dense, index i = 3*spin + colour
 *
 * Parity pins: see tests/test_oracle_*.py.  Functions whose result has no independent
 * pin are marked "parity unpinned" below (only the overall sign convention of the
 * clover term, R10).
 */
#include <complex.h>
#include <math.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

typedef double complex cplx;

#define NS 4
#define NC 3
#define SC 12

/* ---- Dirac matrices, DeGrand-Rossi basis (reading R1); gamma[mu], mu = x,y,z,t (R2) ---- */
static cplx GAM[4][4][4];
static int gam_ready = 0;

static void init_gamma(void) {
    if (gam_ready) return;
    memset(GAM, 0, sizeof(GAM));
    /* gamma_x */
    GAM[0][0][3] = I;  GAM[0][1][2] = I;  GAM[0][2][1] = -I; GAM[0][3][0] = -I;
    /* gamma_y */
    GAM[1][0][3] = -1; GAM[1][1][2] = 1;  GAM[1][2][1] = 1;  GAM[1][3][0] = -1;
    /* gamma_z */
    GAM[2][0][2] = I;  GAM[2][1][3] = -I; GAM[2][2][0] = -I; GAM[2][3][1] = I;
    /* gamma_t */
    GAM[3][0][2] = 1;  GAM[3][1][3] = 1;  GAM[3][2][0] = 1;  GAM[3][3][1] = 1;
    gam_ready = 1;
}

int orc_version(void) { return 1; }

int orc_max_threads(void) {
#ifdef _OPENMP
    return omp_get_max_threads();
#else
    return 1;
#endif
}

void orc_set_threads(int n) {
#ifdef _OPENMP
    if (n > 0) omp_set_num_threads(n);
#else
    (void)n;
#endif
}

void orc_gamma(int mu, double *out /* [4][4][2] */) {
    init_gamma();
    for (int a = 0; a < 4; a++)
        for (int b = 0; b < 4; b++) {
            out[(a * 4 + b) * 2] = creal(GAM[mu][a][b]);
            out[(a * 4 + b) * 2 + 1] = cimag(GAM[mu][a][b]);
        }
}

/* ---- lattice geometry: lexicographic sites, periodic ("circular shift as in HPF",
 *      PAPER.md:113 section II-C; reading R5) ---- */
static long vol(const int L[4]) { return (long)L[0] * L[1] * L[2] * L[3]; }

static void site_coords(long s, const int L[4], int c[4]) {
    c[0] = (int)(s % L[0]); s /= L[0];
    c[1] = (int)(s % L[1]); s /= L[1];
    c[2] = (int)(s % L[2]); s /= L[2];
    c[3] = (int)s;
}

static long site_index(const int c[4], const int L[4]) {
    return c[0] + (long)L[0] * (c[1] + (long)L[1] * (c[2] + (long)L[2] * c[3]));
}

static int site_parity(long s, const int L[4]) {
    int c[4];
    site_coords(s, L, c);
    return (c[0] + c[1] + c[2] + c[3]) & 1;
}

/* index of x + sign*mu^ (periodic) */
static long neighbour(long s, const int L[4], int mu, int sign) {
    int c[4];
    site_coords(s, L, c);
    c[mu] = ((c[mu] + sign) % L[mu] + L[mu]) % L[mu];
    return site_index(c, L);
}

static int in_subset(long s, const int L[4], int subset) {
    return subset < 0 || site_parity(s, L) == subset;
}

/* ---- shift (section II-C, Fig. 1; reading R4):
 *      out(x) = in(x + sign*mu^), FORWARD sign=+1 ---- */
void orc_shift(double *out, const double *in, const int L[4], int nreal, int mu, int sign) {
    long V = vol(L);
#pragma omp parallel for schedule(static)
    for (long s = 0; s < V; s++) {
        long n = neighbour(s, L, mu, sign);
        memcpy(out + s * nreal, in + n * nreal, sizeof(double) * (size_t)nreal);
    }
}

/* ---- hopping term (section VIII-C):
 *   H(x,x') = sum_mu (1 - gamma_mu) U_mu(x) delta_{x+mu,x'} + (1 + gamma_mu) U_mu(x-mu)^dag delta_{x-mu,x'}
 * applied to psi:  (H psi)(x) = sum_mu [(1-g_mu) U_mu(x) psi(x+mu) + (1+g_mu) U_mu(x-mu)^dag psi(x-mu)].
 * Full 4x4 gamma matrices, full 3x3 complex products, no projection trick.
 * Both terms are ACCUMULATED (+=): at L_mu = 2, x+mu = x-mu.
 * out_parity = 0/1: only sites of that parity are computed, all others are set to 0;
 * out_parity = -1: every site. ---- */
void orc_hopping(double *out_, const double *U_, const double *psi_, const int L[4], int out_parity) {
    init_gamma();
    const cplx *U = (const cplx *)U_;
    const cplx *psi = (const cplx *)psi_;
    cplx *out = (cplx *)out_;
    long V = vol(L);
#pragma omp parallel for schedule(static)
    for (long s = 0; s < V; s++) {
        cplx res[NS][NC];
        memset(res, 0, sizeof(res));
        if (in_subset(s, L, out_parity)) {
            for (int mu = 0; mu < 4; mu++) {
                /* forward: (1 - gamma_mu) U_mu(x) psi(x + mu) */
                long f = neighbour(s, L, mu, +1);
                const cplx *Uf = U + (s * 4 + mu) * 9;
                const cplx *pf = psi + f * SC;
                cplx tmp[NS][NC];
                for (int sp = 0; sp < NS; sp++)
                    for (int a = 0; a < NC; a++) {
                        cplx acc = 0;
                        for (int b = 0; b < NC; b++) acc += Uf[a * 3 + b] * pf[sp * 3 + b];
                        tmp[sp][a] = acc;
                    }
                for (int sa = 0; sa < NS; sa++)
                    for (int sb = 0; sb < NS; sb++) {
                        cplx coef = (sa == sb ? 1.0 : 0.0) - GAM[mu][sa][sb];
                        for (int a = 0; a < NC; a++) res[sa][a] += coef * tmp[sb][a];
                    }
                /* backward: (1 + gamma_mu) U_mu(x - mu)^dagger psi(x - mu) */
                long b_ = neighbour(s, L, mu, -1);
                const cplx *Ub = U + (b_ * 4 + mu) * 9;
                const cplx *pb = psi + b_ * SC;
                for (int sp = 0; sp < NS; sp++)
                    for (int a = 0; a < NC; a++) {
                        cplx acc = 0;
                        for (int b = 0; b < NC; b++) acc += conj(Ub[b * 3 + a]) * pb[sp * 3 + b];
                        tmp[sp][a] = acc;
                    }
                for (int sa = 0; sa < NS; sa++)
                    for (int sb = 0; sb < NS; sb++) {
                        cplx coef = (sa == sb ? 1.0 : 0.0) + GAM[mu][sa][sb];
                        for (int a = 0; a < NC; a++) res[sa][a] += coef * tmp[sb][a];
                    }
            }
        }
        memcpy(out + s * SC, res, sizeof(res));
    }
}

/* ---- lattice BLAS (north star).  Neumaier-compensated sums
 *      in lexicographic site order, components in storage order. ---- */
typedef struct { double s, c; } neum;
static void neum_add(neum *n, double v) {
    double t = n->s + v;
    if (fabs(n->s) >= fabs(v)) n->c += (n->s - t) + v;
    else n->c += (v - t) + n->s;
    n->s = t;
}

/* norm2(a) = sum_x sum_{spin,colour} |a(x)|^2 over the subset */
double orc_norm2(const double *a, const int L[4], int subset) {
    long V = vol(L);
    neum n = {0, 0};
    for (long s = 0; s < V; s++) {
        if (!in_subset(s, L, subset)) continue;
        for (int k = 0; k < 2 * SC; k++) neum_add(&n, a[s * 24 + k] * a[s * 24 + k]);
    }
    return n.s + n.c;
}

/* innerProduct(a, b) = sum_x sum conj(a) b  (conjugate-linear in the FIRST argument) */
void orc_inner(const double *a_, const double *b_, const int L[4], int subset, double out[2]) {
    const cplx *a = (const cplx *)a_, *b = (const cplx *)b_;
    long V = vol(L);
    neum re = {0, 0}, im = {0, 0};
    for (long s = 0; s < V; s++) {
        if (!in_subset(s, L, subset)) continue;
        for (int k = 0; k < SC; k++) {
            cplx p = conj(a[s * SC + k]) * b[s * SC + k];
            neum_add(&re, creal(p));
            neum_add(&im, cimag(p));
        }
    }
    out[0] = re.s + re.c;
    out[1] = im.s + im.c;
}

/* axpy: y <- a x + y on the subset (complex a) */
void orc_axpy(double ar, double ai, const double *x_, double *y_, const int L[4], int subset) {
    const cplx *x = (const cplx *)x_;
    cplx *y = (cplx *)y_;
    cplx a = ar + ai * I;
    long V = vol(L);
#pragma omp parallel for schedule(static)
    for (long s = 0; s < V; s++) {
        if (!in_subset(s, L, subset)) continue;
        for (int k = 0; k < SC; k++) y[s * SC + k] = a * x[s * SC + k] + y[s * SC + k];
    }
}

/* ---- 3x3 colour-matrix helpers for the clover leaves ---- */
typedef struct { cplx m[3][3]; } mat3;

static mat3 link(const cplx *U, long s, int mu) {
    mat3 r;
    for (int a = 0; a < 3; a++)
        for (int b = 0; b < 3; b++) r.m[a][b] = U[(s * 4 + mu) * 9 + a * 3 + b];
    return r;
}
static mat3 dag(mat3 x) {
    mat3 r;
    for (int a = 0; a < 3; a++)
        for (int b = 0; b < 3; b++) r.m[a][b] = conj(x.m[b][a]);
    return r;
}
static mat3 mul(mat3 x, mat3 y) {
    mat3 r;
    for (int a = 0; a < 3; a++)
        for (int b = 0; b < 3; b++) {
            cplx acc = 0;
            for (int k = 0; k < 3; k++) acc += x.m[a][k] * y.m[k][b];
            r.m[a][b] = acc;
        }
    return r;
}
static mat3 mul4(mat3 a, mat3 b, mat3 c, mat3 d) { return mul(mul(mul(a, b), c), d); }

/* site index of x + a*mu^ + b*nu^ */
static long nb2(long s, const int L[4], int mu, int a, int nu, int b) {
    int c[4];
    site_coords(s, L, c);
    c[mu] = ((c[mu] + a) % L[mu] + L[mu]) % L[mu];
    c[nu] = ((c[nu] + b) % L[nu] + L[nu]) % L[nu];
    return site_index(c, L);
}

/* Q_mu,nu(x): sum of the four clover-leaf plaquettes at x, all with the same
 * orientation in the (mu,nu) plane (reading R10). */
static mat3 clover_leaves(const cplx *U, long s, const int L[4], int mu, int nu) {
    mat3 q, t;
    /* U_mu(x) U_nu(x+mu) U_mu(x+nu)^dag U_nu(x)^dag */
    q = mul4(link(U, s, mu), link(U, nb2(s, L, mu, 1, nu, 0), nu),
             dag(link(U, nb2(s, L, mu, 0, nu, 1), mu)), dag(link(U, s, nu)));
    /* U_nu(x) U_mu(x-mu+nu)^dag U_nu(x-mu)^dag U_mu(x-mu) */
    t = mul4(link(U, s, nu), dag(link(U, nb2(s, L, mu, -1, nu, 1), mu)),
             dag(link(U, nb2(s, L, mu, -1, nu, 0), nu)), link(U, nb2(s, L, mu, -1, nu, 0), mu));
    for (int a = 0; a < 3; a++) for (int b = 0; b < 3; b++) q.m[a][b] += t.m[a][b];
    /* U_mu(x-mu)^dag U_nu(x-mu-nu)^dag U_mu(x-mu-nu) U_nu(x-nu) */
    t = mul4(dag(link(U, nb2(s, L, mu, -1, nu, 0), mu)), dag(link(U, nb2(s, L, mu, -1, nu, -1), nu)),
             link(U, nb2(s, L, mu, -1, nu, -1), mu), link(U, nb2(s, L, mu, 0, nu, -1), nu));
    for (int a = 0; a < 3; a++) for (int b = 0; b < 3; b++) q.m[a][b] += t.m[a][b];
    /* U_nu(x-nu)^dag U_mu(x-nu) U_nu(x-nu+mu) U_mu(x)^dag */
    t = mul4(dag(link(U, nb2(s, L, mu, 0, nu, -1), nu)), link(U, nb2(s, L, mu, 0, nu, -1), mu),
             link(U, nb2(s, L, mu, 1, nu, -1), nu), dag(link(U, s, mu)));
    for (int a = 0; a < 3; a++) for (int b = 0; b < 3; b++) q.m[a][b] += t.m[a][b];
    return q;
}

/* ---- clover term (section VI-A, eq. (1)):
 *   A(x) = (4 + m) 1 + 1/4 c_SW sum_{mu,nu} sigma_mu,nu F_mu,nu(x)
 * with (reading R10) sigma_mu,nu = [gamma_mu, gamma_nu] / (2i) and the Hermitian,
 * traceless field strength F_mu,nu = traceless part of (Q_mu,nu - Q_mu,nu^dag) / (8i).
 * The (4+m) diagonal is the Wilson mass term of M = A - H/2 (reading R3/R12), folded
 * into A as in the C ABI.  Output: dense 12x12 per site, i = 3*spin + colour.
 * Parity of the overall sign of c_SW: UNPINNED (convention, R10); magnitude, F, the
 * leaves and the sigma algebra are pinned (tests/test_oracle_clover.py). ---- */
void orc_clover_build(double *A_, const double *U_, const int L[4], double mass, double csw) {
    init_gamma();
    const cplx *U = (const cplx *)U_;
    cplx *A = (cplx *)A_;
    long V = vol(L);
    /* sigma_mu,nu = (gamma_mu gamma_nu - gamma_nu gamma_mu) / (2i) */
    static cplx sig[4][4][4][4];
    for (int mu = 0; mu < 4; mu++)
        for (int nu = 0; nu < 4; nu++)
            for (int a = 0; a < 4; a++)
                for (int b = 0; b < 4; b++) {
                    cplx c = 0;
                    for (int k = 0; k < 4; k++) c += GAM[mu][a][k] * GAM[nu][k][b] - GAM[nu][a][k] * GAM[mu][k][b];
                    sig[mu][nu][a][b] = c / (2.0 * I);
                }
#pragma omp parallel for schedule(static)
    for (long s = 0; s < V; s++) {
        cplx *As = A + s * SC * SC;
        for (int i = 0; i < SC * SC; i++) As[i] = 0;
        for (int i = 0; i < SC; i++) As[i * SC + i] = 4.0 + mass;
        for (int mu = 0; mu < 4; mu++)
            for (int nu = 0; nu < 4; nu++) {
                if (mu == nu) continue;
                mat3 q = clover_leaves(U, s, L, mu, nu);
                cplx F[3][3];
                cplx tr = 0;
                for (int a = 0; a < 3; a++)
                    for (int b = 0; b < 3; b++) F[a][b] = (q.m[a][b] - conj(q.m[b][a])) / (8.0 * I);
                for (int a = 0; a < 3; a++) tr += F[a][a];
                for (int a = 0; a < 3; a++) F[a][a] -= tr / 3.0;
                for (int sa = 0; sa < 4; sa++)
                    for (int sb = 0; sb < 4; sb++) {
                        cplx sg = 0.25 * csw * sig[mu][nu][sa][sb];
                        if (sg == 0) continue;
                        for (int a = 0; a < 3; a++)
                            for (int b = 0; b < 3; b++) As[(sa * 3 + a) * SC + sb * 3 + b] += sg * F[a][b];
                    }
            }
    }
}

/* Gaussian elimination with partial pivoting: inverse of one dense 12x12 matrix.
 * Returns 0, or -1 if a pivot is exactly zero (singular). */
static int invert12(cplx *out, const cplx *in) {
    cplx a[SC][2 * SC];
    for (int i = 0; i < SC; i++)
        for (int j = 0; j < SC; j++) {
            a[i][j] = in[i * SC + j];
            a[i][SC + j] = (i == j) ? 1.0 : 0.0;
        }
    for (int col = 0; col < SC; col++) {
        int piv = col;
        for (int r = col + 1; r < SC; r++)
            if (cabs(a[r][col]) > cabs(a[piv][col])) piv = r;
        if (cabs(a[piv][col]) == 0.0) return -1;
        if (piv != col)
            for (int j = 0; j < 2 * SC; j++) { cplx t = a[col][j]; a[col][j] = a[piv][j]; a[piv][j] = t; }
        cplx d = a[col][col];
        for (int j = 0; j < 2 * SC; j++) a[col][j] /= d;
        for (int r = 0; r < SC; r++) {
            if (r == col) continue;
            cplx f = a[r][col];
            if (f == 0) continue;
            for (int j = 0; j < 2 * SC; j++) a[r][j] -= f * a[col][j];
        }
    }
    for (int i = 0; i < SC; i++)
        for (int j = 0; j < SC; j++) out[i * SC + j] = a[i][SC + j];
    return 0;
}

/* inverse of A on the subset's sites (others: zero).  Returns 0 or -1 (singular). */
int orc_clover_invert(double *Ainv_, const double *A_, const int L[4], int subset) {
    const cplx *A = (const cplx *)A_;
    cplx *Ainv = (cplx *)Ainv_;
    long V = vol(L);
    int bad = 0;
#pragma omp parallel for schedule(static) reduction(| : bad)
    for (long s = 0; s < V; s++) {
        if (!in_subset(s, L, subset)) {
            for (int i = 0; i < SC * SC; i++) Ainv[s * SC * SC + i] = 0;
            continue;
        }
        if (invert12(Ainv + s * SC * SC, A + s * SC * SC)) bad = 1;
    }
    return bad ? -1 : 0;
}

/* out(x) = A(x) in(x) on the subset; other sites untouched. */
void orc_clover_apply(double *out_, const double *A_, const double *in_, const int L[4], int subset) {
    const cplx *A = (const cplx *)A_, *in = (const cplx *)in_;
    cplx *out = (cplx *)out_;
    long V = vol(L);
#pragma omp parallel for schedule(static)
    for (long s = 0; s < V; s++) {
        if (!in_subset(s, L, subset)) continue;
        cplx r[SC];
        for (int i = 0; i < SC; i++) {
            cplx acc = 0;
            for (int j = 0; j < SC; j++) acc += A[s * SC * SC + i * SC + j] * in[s * SC + j];
            r[i] = acc;
        }
        memcpy(out + s * SC, r, sizeof(r));
    }
}

/* ================= Wilson(-clover) operator and even-odd CG ===================
 * M = A - H/2 with A = (4+m) 1 (Wilson) or the clover A above (readings R3, R12).
 * Vectors are full-lattice fermions; "_e"/"_o" parts are their parity-0/1 sites. */

typedef struct {
    const int *L;
    const double *U;
    const double *A;     /* dense clover incl. 4+m, or NULL for Wilson */
    const double *Ainv;  /* its inverse on even sites, or NULL */
    double diag;         /* 4 + m (Wilson) */
    long V;
    double *t1, *t2;     /* scratch, full-lattice fermions */
} op_t;

/* out = A v on parity p (Wilson: (4+m) v); other parity untouched */
static void apply_A(const op_t *op, double *out, const double *v, int p) {
    if (op->A) { orc_clover_apply(out, op->A, v, op->L, p); return; }
    for (long s = 0; s < op->V; s++)
        if (in_subset(s, op->L, p))
            for (int k = 0; k < 24; k++) out[s * 24 + k] = op->diag * v[s * 24 + k];
}
/* out = A_ee^{-1} v on even sites */
static void apply_Ainv_e(const op_t *op, double *out, const double *v) {
    if (op->A) { orc_clover_apply(out, op->Ainv, v, op->L, 0); return; }
    for (long s = 0; s < op->V; s++)
        if (in_subset(s, op->L, 0))
            for (int k = 0; k < 24; k++) out[s * 24 + k] = v[s * 24 + k] / op->diag;
}

static void zero_parity(double *v, const int *L, long V, int p) {
    for (long s = 0; s < V; s++)
        if (in_subset(s, L, p)) memset(v + s * 24, 0, sizeof(double) * 24);
}

/* gamma5 = gamma_x gamma_y gamma_z gamma_t = diag(1,1,-1,-1) in this basis: computed from GAM */
static void apply_gamma5(double *out_, const double *in_, const int *L, long V, int p) {
    init_gamma();
    cplx g5[4][4], t[4][4];
    for (int a = 0; a < 4; a++) for (int b = 0; b < 4; b++) {
        cplx c = 0;
        for (int k = 0; k < 4; k++) c += GAM[0][a][k] * GAM[1][k][b];
        t[a][b] = c;
    }
    for (int a = 0; a < 4; a++) for (int b = 0; b < 4; b++) {
        cplx c = 0;
        for (int k = 0; k < 4; k++) c += t[a][k] * GAM[2][k][b];
        g5[a][b] = c;
    }
    for (int a = 0; a < 4; a++) for (int b = 0; b < 4; b++) {
        cplx c = 0;
        for (int k = 0; k < 4; k++) c += g5[a][k] * GAM[3][k][b];
        t[a][b] = c;
    }
    const cplx *in = (const cplx *)in_;
    cplx *out = (cplx *)out_;
    for (long s = 0; s < V; s++) {
        if (!in_subset(s, L, p)) continue;
        cplx r[4][3];
        for (int a = 0; a < 4; a++) for (int c = 0; c < 3; c++) {
            cplx acc = 0;
            for (int b = 0; b < 4; b++) acc += t[a][b] * in[s * SC + b * 3 + c];
            r[a][c] = acc;
        }
        memcpy(out + s * SC, r, sizeof(r));
    }
}

/* Mhat v = A_oo v - 1/4 H_oe A_ee^{-1} H_eo v   (odd sites of out) */
static void apply_Mhat(const op_t *op, double *out, const double *v) {
    orc_hopping(op->t1, op->U, v, op->L, 0);          /* t1_e = H_eo v_o */
    apply_Ainv_e(op, op->t2, op->t1);                 /* t2_e = A_ee^-1 t1_e */
    orc_hopping(op->t1, op->U, op->t2, op->L, 1);     /* t1_o = H_oe t2_e */
    apply_A(op, out, v, 1);                           /* out_o = A_oo v_o */
    orc_axpy(-0.25, 0.0, op->t1, out, op->L, 1);      /* out_o -= 1/4 t1_o */
    zero_parity(out, op->L, op->V, 0);
}

/* Mhat^dag v = gamma5 Mhat gamma5 v (A commutes with gamma5) */
static void apply_Mhat_dag(const op_t *op, double *out, const double *v, double *g) {
    apply_gamma5(g, v, op->L, op->V, 1);
    zero_parity(g, op->L, op->V, 0);
    apply_Mhat(op, out, g);
    apply_gamma5(out, out, op->L, op->V, 1);
}

/* out = M v = A v - H v / 2 (full lattice) */
void orc_wilson_apply(double *out, const double *U, const double *A, double mass,
                      const double *v, const int L[4]) {
    long V = vol(L);
    op_t op = {L, U, A, NULL, 4.0 + mass, V, NULL, NULL};
    double *h = (double *)malloc(sizeof(double) * 24 * (size_t)V);
    orc_hopping(h, U, v, L, -1);
    apply_A(&op, out, v, -1);
    orc_axpy(-0.5, 0.0, h, out, L, -1);
    free(h);
}

/* Even-odd CGNR (SURVEY.md 8(c) item 6, step by step; x0 = 0):
 *   hist[k] = sqrt(rho_k / rho_0) for k = 0..iters (if hist_cap allows).
 * Returns 0 converged, 1 not converged, -1 singular clover. */
int orc_cg_solve(double *x, const double *b, const double *U, const double *A, double mass,
                 const int L[4], double tol, int maxit, int *iters, double *hist, int hist_cap,
                 double *true_resid) {
    long V = vol(L);
    size_t nb = sizeof(double) * 24 * (size_t)V;
    double *Ainv = NULL;
    if (A) {
        Ainv = (double *)malloc(sizeof(double) * 288 * (size_t)V);
        if (orc_clover_invert(Ainv, A, L, 0)) { free(Ainv); return -1; }
    }
    double *t1 = calloc(1, nb), *t2 = calloc(1, nb), *g = calloc(1, nb);
    double *bh = calloc(1, nb), *r = calloc(1, nb), *p = calloc(1, nb), *q = calloc(1, nb), *mp = calloc(1, nb);
    op_t op = {L, U, A, Ainv, 4.0 + mass, V, t1, t2};

    /* step 2: bhat_o = b_o + 1/2 H_oe A_ee^-1 b_e */
    double *tmp = calloc(1, nb), *tmp2 = calloc(1, nb);
    apply_Ainv_e(&op, tmp, b);
    orc_hopping(tmp2, U, tmp, L, 1);
    for (long s = 0; s < V; s++)
        if (in_subset(s, L, 1))
            for (int k = 0; k < 24; k++) bh[s * 24 + k] = b[s * 24 + k] + 0.5 * tmp2[s * 24 + k];

    /* step 4: r0 = Mhat^dag bhat, p0 = r0, rho0 = <r0,r0> */
    memset(x, 0, nb);
    apply_Mhat_dag(&op, r, bh, g);
    memcpy(p, r, nb);
    double rho0 = orc_norm2(r, L, 1), rho = rho0;
    int k = 0, status = 1;
    if (hist_cap > 0) hist[0] = 1.0;
    if (rho0 == 0.0) status = 0;
    /* step 5 */
    while (status == 1 && k < maxit) {
        apply_Mhat(&op, mp, p);
        apply_Mhat_dag(&op, q, mp, g);
        double pq[2];
        orc_inner(p, q, L, 1, pq);
        double alpha = rho / pq[0];
        orc_axpy(alpha, 0.0, p, x, L, 1);
        orc_axpy(-alpha, 0.0, q, r, L, 1);
        double rho_new = orc_norm2(r, L, 1);
        k++;
        if (k < hist_cap) hist[k] = sqrt(rho_new / rho0);
        if (rho_new <= tol * tol * rho0) { rho = rho_new; status = 0; break; }
        double beta = rho_new / rho;
        rho = rho_new;
        for (long s = 0; s < V; s++)
            if (in_subset(s, L, 1))
                for (int c = 0; c < 24; c++) p[s * 24 + c] = r[s * 24 + c] + beta * p[s * 24 + c];
    }
    *iters = k;

    /* step 6: x_e = A_ee^-1 (b_e + 1/2 H_eo x_o) */
    orc_hopping(tmp, U, x, L, 0);
    for (long s = 0; s < V; s++)
        if (in_subset(s, L, 0))
            for (int c = 0; c < 24; c++) tmp[s * 24 + c] = b[s * 24 + c] + 0.5 * tmp[s * 24 + c];
    apply_Ainv_e(&op, tmp2, tmp);
    for (long s = 0; s < V; s++)
        if (in_subset(s, L, 0)) memcpy(x + s * 24, tmp2 + s * 24, sizeof(double) * 24);

    /* step 7: true residual |b - M x| / |b| */
    orc_wilson_apply(tmp, U, A, mass, x, L);
    for (long s = 0; s < V * 24; s++) tmp[s] = b[s] - tmp[s];
    *true_resid = sqrt(orc_norm2(tmp, L, -1) / orc_norm2(b, L, -1));

    free(tmp); free(tmp2); free(t1); free(t2); free(g); free(bh); free(r); free(p); free(q); free(mp);
    free(Ainv);
    return status;
}

/* out_o = Mhat v_o (dagger = 0) or Mhat^dag v_o (dagger = 1); even sites of out zero.
 * Exposed so tests can assemble the dense even-odd operator column by column. */
void orc_mhat_apply(double *out, const double *U, const double *A, double mass, const double *v,
                    const int L[4], int dagger) {
    long V = vol(L);
    size_t nb = sizeof(double) * 24 * (size_t)V;
    double *Ainv = NULL;
    if (A) {
        Ainv = (double *)malloc(sizeof(double) * 288 * (size_t)V);
        orc_clover_invert(Ainv, A, L, 0);
    }
    double *t1 = calloc(1, nb), *t2 = calloc(1, nb), *g = calloc(1, nb), *vo = calloc(1, nb);
    op_t op = {L, U, A, Ainv, 4.0 + mass, V, t1, t2};
    for (long s = 0; s < V; s++)
        if (in_subset(s, L, 1)) memcpy(vo + s * 24, v + s * 24, sizeof(double) * 24);
    if (dagger) apply_Mhat_dag(&op, out, vo, g);
    else apply_Mhat(&op, out, vo);
    free(t1); free(t2); free(g); free(vo); free(Ainv);
}

/* Multi-shift CG (the solver of the paper's RHMC production runs, ref. [14];
 * reading R25): solves (Mhat^dag Mhat + sigma_i) x_i = phi on the odd sites for all i at once,
 * from ONE Krylov space: plain CG on the base system sigma_0 (sigma_0 <= sigma_i), the shifted
 * residuals collinear, r_i = zeta_i r, with (s_i = sigma_i - sigma_0, x_i = 0, p_i = phi):
 *   zeta_i(k+1) = zeta_i(k) zeta_i(k-1) alpha(k-1) /
 *                 [alpha(k) beta(k-1) (zeta_i(k-1) - zeta_i(k)) + zeta_i(k-1) alpha(k-1) (1 + s_i alpha(k))]
 *   alpha_i(k) = alpha(k) zeta_i(k+1) / zeta_i(k),   beta_i(k) = beta(k) (zeta_i(k+1) / zeta_i(k))^2
 *   x_i += alpha_i(k) p_i ;  p_i = zeta_i(k+1) r(k+1) + beta_i(k) p_i
 * with zeta(-1) = zeta(0) = 1, alpha(-1) = 1, beta(-1) = 0.  Shift i stops being updated once
 * zeta_i(k+1)^2 rho(k+1) <= tol^2 rho(0) (its own relative residual); iterations stop when the
 * base system (the slowest) converges.  Step by step, each line of the recurrence one C line.
 * hist[k] = sqrt(rho_k / rho_0) of the base system; conv_iter[i] = iteration at which shift i
 * stopped; true_resid[i] = |phi - (Mhat^dag Mhat + sigma_i) x_i| / |phi|.
 * x: nshift consecutive fermion arrays [nshift][V][24]; only odd sites are written.
 * Returns 0 converged, 1 not converged, -1 singular clover, -2 bad shifts. */
int orc_cg_multishift(double *x, const double *phi, const double *U, const double *A, double mass,
                      const int L[4], int nshift, const double *sigma, double tol, int maxit,
                      int *iters, int *conv_iter, double *hist, int hist_cap, double *true_resid) {
    if (nshift < 1) return -2;
    for (int i = 1; i < nshift; i++)
        if (sigma[i] < sigma[0]) return -2;
    long V = vol(L);
    size_t nb = sizeof(double) * 24 * (size_t)V;
    double *Ainv = NULL;
    if (A) {
        Ainv = (double *)malloc(sizeof(double) * 288 * (size_t)V);
        if (orc_clover_invert(Ainv, A, L, 0)) { free(Ainv); return -1; }
    }
    double *t1 = calloc(1, nb), *t2 = calloc(1, nb), *g = calloc(1, nb), *mp = calloc(1, nb);
    double *r = calloc(1, nb), *q = calloc(1, nb), *p = calloc(1, nb * nshift);
    op_t op = {L, U, A, Ainv, 4.0 + mass, V, t1, t2};
    double *zeta = malloc(sizeof(double) * nshift), *zeta_old = malloc(sizeof(double) * nshift);
    double *zeta_new = malloc(sizeof(double) * nshift);
    int *active = malloc(sizeof(int) * nshift);

    memset(x, 0, nb * nshift);
    for (long s = 0; s < V; s++)
        if (in_subset(s, L, 1)) {
            memcpy(r + s * 24, phi + s * 24, sizeof(double) * 24);
            for (int i = 0; i < nshift; i++) memcpy(p + i * 24 * V + s * 24, phi + s * 24, sizeof(double) * 24);
        }
    for (int i = 0; i < nshift; i++) { zeta[i] = zeta_old[i] = 1.0; active[i] = 1; conv_iter[i] = 0; }
    double alpha_old = 1.0, beta_old = 0.0;
    double rho0 = orc_norm2(r, L, 1), rho = rho0;
    int k = 0, status = 1;
    if (hist_cap > 0) hist[0] = 1.0;
    if (rho0 == 0.0) status = 0;
    while (status == 1 && k < maxit) {
        /* q = (Mhat^dag Mhat + sigma_0) p_0 */
        apply_Mhat(&op, mp, p);
        apply_Mhat_dag(&op, q, mp, g);
        orc_axpy(sigma[0], 0.0, p, q, L, 1);
        double pq[2];
        orc_inner(p, q, L, 1, pq);
        double alpha = rho / pq[0];
        /* shifted coefficients and solution updates */
        for (int i = 0; i < nshift; i++) {
            if (!active[i]) continue;
            double a_i = alpha;
            if (i == 0) zeta_new[i] = 1.0;
            else {
                double si = sigma[i] - sigma[0];
                zeta_new[i] = zeta[i] * zeta_old[i] * alpha_old /
                              (alpha * beta_old * (zeta_old[i] - zeta[i]) + zeta_old[i] * alpha_old * (1.0 + si * alpha));
                a_i = alpha * zeta_new[i] / zeta[i];
            }
            orc_axpy(a_i, 0.0, p + i * 24 * V, x + i * 24 * V, L, 1);
        }
        orc_axpy(-alpha, 0.0, q, r, L, 1);
        double rho_new = orc_norm2(r, L, 1);
        k++;
        if (k < hist_cap) hist[k] = sqrt(rho_new / rho0);
        double beta = rho_new / rho;
        for (int i = 0; i < nshift; i++) {
            if (!active[i]) continue;
            if (zeta_new[i] * zeta_new[i] * rho_new <= tol * tol * rho0) {  /* shift i converged */
                active[i] = 0;
                conv_iter[i] = k;
                continue;
            }
            double b_i = beta * (zeta_new[i] / zeta[i]) * (zeta_new[i] / zeta[i]);
            double *pi = p + i * 24 * V;
            for (long s = 0; s < V; s++)
                if (in_subset(s, L, 1))
                    for (int c = 0; c < 24; c++) pi[s * 24 + c] = zeta_new[i] * r[s * 24 + c] + b_i * pi[s * 24 + c];
            zeta_old[i] = zeta[i];
            zeta[i] = zeta_new[i];
        }
        if (!active[0]) status = 0;
        alpha_old = alpha;
        beta_old = beta;
        rho = rho_new;
    }
    for (int i = 0; i < nshift; i++)
        if (active[i]) conv_iter[i] = k;
    *iters = k;

    /* true residuals */
    for (int i = 0; i < nshift; i++) {
        double *xi = x + i * 24 * V;
        apply_Mhat(&op, mp, xi);
        apply_Mhat_dag(&op, q, mp, g);
        orc_axpy(sigma[i], 0.0, xi, q, L, 1);
        for (long s = 0; s < V; s++)
            if (in_subset(s, L, 1))
                for (int c = 0; c < 24; c++) q[s * 24 + c] = phi[s * 24 + c] - q[s * 24 + c];
        true_resid[i] = sqrt(orc_norm2(q, L, 1) / rho0);
    }
    free(t1); free(t2); free(g); free(mp); free(r); free(q); free(p);
    free(zeta); free(zeta_old); free(zeta_new); free(active); free(Ainv);
    return status;
}

/* ================= Table II test functions (section VI) ====================
 * Site-local products on n sites, host layouts: colour matrix [n][3][3][2], spin matrix
 * [n][4][4][2], fermion [n][4][3][2].  Plain definitions. */

/* lcm: out(x) = a(x) b(x), 3x3 complex */
void orc_lcm(double *out_, const double *a_, const double *b_, long n) {
    const cplx *a = (const cplx *)a_, *b = (const cplx *)b_;
    cplx *out = (cplx *)out_;
#pragma omp parallel for schedule(static)
    for (long s = 0; s < n; s++)
        for (int i = 0; i < 3; i++)
            for (int j = 0; j < 3; j++) {
                cplx acc = 0;
                for (int k = 0; k < 3; k++) acc += a[s * 9 + i * 3 + k] * b[s * 9 + k * 3 + j];
                out[s * 9 + i * 3 + j] = acc;
            }
}

/* upsi: out(x)_{spin,a} = sum_b u(x)_{a,b} psi(x)_{spin,b} */
void orc_upsi(double *out_, const double *u_, const double *psi_, long n) {
    const cplx *u = (const cplx *)u_, *psi = (const cplx *)psi_;
    cplx *out = (cplx *)out_;
#pragma omp parallel for schedule(static)
    for (long s = 0; s < n; s++)
        for (int sp = 0; sp < 4; sp++)
            for (int a = 0; a < 3; a++) {
                cplx acc = 0;
                for (int b = 0; b < 3; b++) acc += u[s * 9 + a * 3 + b] * psi[s * 12 + sp * 3 + b];
                out[s * 12 + sp * 3 + a] = acc;
            }
}

/* spmat: out(x) = a(x) b(x), 4x4 complex */
void orc_spmat(double *out_, const double *a_, const double *b_, long n) {
    const cplx *a = (const cplx *)a_, *b = (const cplx *)b_;
    cplx *out = (cplx *)out_;
#pragma omp parallel for schedule(static)
    for (long s = 0; s < n; s++)
        for (int i = 0; i < 4; i++)
            for (int j = 0; j < 4; j++) {
                cplx acc = 0;
                for (int k = 0; k < 4; k++) acc += a[s * 16 + i * 4 + k] * b[s * 16 + k * 4 + j];
                out[s * 16 + i * 4 + j] = acc;
            }
}

/* adj(u) * psi: out(x)_{spin,a} = sum_b conj(u(x)_{b,a}) psi(x)_{spin,b}  (Fig. 1) */
void orc_adj_upsi(double *out_, const double *u_, const double *psi_, long n) {
    const cplx *u = (const cplx *)u_, *psi = (const cplx *)psi_;
    cplx *out = (cplx *)out_;
#pragma omp parallel for schedule(static)
    for (long s = 0; s < n; s++)
        for (int sp = 0; sp < 4; sp++)
            for (int a = 0; a < 3; a++) {
                cplx acc = 0;
                for (int b = 0; b < 3; b++) acc += conj(u[s * 9 + b * 3 + a]) * psi[s * 12 + sp * 3 + b];
                out[s * 12 + sp * 3 + a] = acc;
            }
}

/* matvec: out(x) = u(x) psi1(x) + u(x) psi2(x) */
void orc_matvec(double *out, const double *u, const double *p1, const double *p2, long n) {
    double *t = (double *)malloc(sizeof(double) * 24 * (size_t)n);
    orc_upsi(out, u, p1, n);
    orc_upsi(t, u, p2, n);
    for (long k = 0; k < 24 * n; k++) out[k] += t[k];
    free(t);
}
