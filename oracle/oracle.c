/*
 * oracle/oracle.c -- plain, slow, fp64 CPU oracle for the ls1-mardyn hot path
 * (arXiv:1408.4599).  TEST INFRASTRUCTURE ONLY: it is loaded by tests/,
 * __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference leg,
 * and by nothing else.  It shares no code, header, table or constant with the
 * CUDA path (paper_1408_4599_b200/), and never reads anything that path wrote.
 *
 * Citation keys: "P:n" = /root/reference/PAPER.md line n; "A<k>" = reading k
 * of DESIGN.md §2 (the paper is silent or garbled there).
 *
 * What it computes (written out with no blocking or fusion):
 *   grid      n_k = floor(L_k/rc) cells per axis of edge >= rc and
 *             the fixed-point position lattice of reading A12.
 *   cells     cell_k = floor(u_k / E_k), u = fixed-point position (A12).
 *   forces    all unordered molecule pairs with COM distance < rc (A1),
 *             minimum image; for every site pair: LJ 12-6 (Eq. 1,
 *             P:70-74) truncated and shifted (A2), charge-charge with
 *             reaction field (A4), point dipoles and linear point
 *             quadrupoles (A5); forces, torques (A6), U, virial W.
 *             Three enumerations that must agree: brute force O(N^2)
 *             (the plain definition), the linked-cell Newton-3 half shell
 *             (Fig. 1) and a full 27-cell shell per molecule.
 *   integrate leapfrog Eqs. 2-3 and the Fincham quaternion
 *             leapfrog reading of Eqs. 4-5 (A7), A8 start, A9 T;
 *             NVT by velocity rescaling (reading A24).
 *   tail      isotropic mean-field LJ corrections of U and W beyond rc
 *             (reading A3: reported separately, not part of U_pot).
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

enum { OR_LJ = 0, OR_CHARGE = 1, OR_DIPOLE = 2, OR_QUADRUPOLE = 3 };

typedef struct {
    int32_t type;      /* OR_LJ, OR_CHARGE, OR_DIPOLE, OR_QUADRUPOLE            */
    int32_t pad;
    double r[3];       /* body-frame position relative to the COM              */
    double e[3];       /* body-frame unit axis (dipole / quadrupole)           */
    double m;          /* q, mu or Q                                           */
    double sigma, eps; /* LJ                                                   */
} or_site;

typedef struct {
    double mass;
    double I[3];       /* principal moments, body axes = principal axes       */
    int32_t site0, nsites;
} or_comp;

typedef struct {
    /* inputs */
    double L[3];       /* requested box                                        */
    double rc;
    double eps_rf;     /* reaction-field dielectric constant, INFINITY allowed */
    int32_t lj_shift;  /* 1 = truncated and shifted (LJTS)                     */
    int32_t n_comp;
    const or_comp* comp;
    const or_site* sites;
    const double* eta; /* n_comp*n_comp binary parameters, NULL = 1     */
    /* derived by or_setup (reading A12) */
    int32_t nc[3];     /* cells per axis                                       */
    int64_t E[3];      /* cell edge in quanta                                  */
    int64_t P[3];      /* period in quanta = nc*E                              */
    double s;          /* quantum (a power of two)                             */
    double box[3];     /* snapped box = P*s                                    */
} or_sys;

/* ------------------------------------------------------------------------ */
/* grid and fixed-point lattice (reading A12)                                */

int or_setup(or_sys* S)
{
    if (!(S->rc > 0)) return -1;
    for (int k = 0; k < 3; ++k) {
        S->nc[k] = (int32_t)floor(S->L[k] / S->rc);   /* edge = L/n >= rc */
        if (S->nc[k] < 2) return -1;
    }
    /* quantum s = 2^(ceil(log2(max edge)) - 22): a cell edge is <= 2^22 quanta   */
    for (int it = 0; it < 4; ++it) {
        double emax = 0;
        for (int k = 0; k < 3; ++k) emax = fmax(emax, S->L[k] / S->nc[k]);
        int ex = (int)ceil(log2(emax));
        S->s = ldexp(1.0, ex - 22);
        int again = 0;
        for (int k = 0; k < 3; ++k) {
            S->E[k] = llround(S->L[k] / (S->nc[k] * S->s));
            if ((double)S->E[k] * S->s < S->rc) { S->nc[k] -= 1; again = 1; }
            if (S->nc[k] < 2) return -1;
        }
        if (!again) break;
    }
    for (int k = 0; k < 3; ++k) {
        S->P[k] = S->E[k] * S->nc[k];
        S->box[k] = (double)S->P[k] * S->s;
    }
    return 0;
}

/* position -> fixed point u in [0, P) : u = rint(r/s) mod P                */
void or_quantize(const or_sys* S, int64_t n, const double* r, uint32_t* u)
{
    for (int64_t i = 0; i < n; ++i)
        for (int k = 0; k < 3; ++k) {
            int64_t v = (int64_t)rint(r[3 * i + k] / S->s);
            v %= S->P[k];
            if (v < 0) v += S->P[k];
            u[3 * i + k] = (uint32_t)v;
        }
}

/* cell of every molecule (x fastest) and the count per cell                 */
void or_cells(const or_sys* S, int64_t n, const uint32_t* u, int32_t* cell, int32_t* count)
{
    int64_t ncell = (int64_t)S->nc[0] * S->nc[1] * S->nc[2];
    for (int64_t c = 0; c < ncell; ++c) count[c] = 0;
    for (int64_t i = 0; i < n; ++i) {
        int64_t cx = u[3 * i + 0] / S->E[0];
        int64_t cy = u[3 * i + 1] / S->E[1];
        int64_t cz = u[3 * i + 2] / S->E[2];
        int64_t c = cx + S->nc[0] * (cy + S->nc[1] * cz);
        cell[i] = (int32_t)c;
        count[c] += 1;
    }
}

/* minimum-image COM separation r_j - r_i in quanta                  */
static void min_image(const or_sys* S, const uint32_t* ui, const uint32_t* uj, int64_t d[3])
{
    for (int k = 0; k < 3; ++k) {
        int64_t x = (int64_t)uj[k] - (int64_t)ui[k];
        if (2 * x > S->P[k]) x -= S->P[k];
        else if (2 * x < -S->P[k]) x += S->P[k];
        d[k] = x;
    }
}

/* ------------------------------------------------------------------------ */
/* rigid-body geometry                                                       */

/* body -> world rotation matrix of the unit quaternion q = (w,x,y,z)       */
static void quat_to_R(const double* q, double R[3][3])
{
    double w = q[0], x = q[1], y = q[2], z = q[3];
    R[0][0] = 1 - 2 * (y * y + z * z); R[0][1] = 2 * (x * y - w * z); R[0][2] = 2 * (x * z + w * y);
    R[1][0] = 2 * (x * y + w * z); R[1][1] = 1 - 2 * (x * x + z * z); R[1][2] = 2 * (y * z - w * x);
    R[2][0] = 2 * (x * z - w * y); R[2][1] = 2 * (y * z + w * x); R[2][2] = 1 - 2 * (x * x + y * y);
}

static void matvec(double R[3][3], const double* a, double* b)
{
    for (int k = 0; k < 3; ++k) b[k] = R[k][0] * a[0] + R[k][1] * a[1] + R[k][2] * a[2];
}

static void matTvec(double R[3][3], const double* a, double* b)
{
    for (int k = 0; k < 3; ++k) b[k] = R[0][k] * a[0] + R[1][k] * a[1] + R[2][k] * a[2];
}

static void cross(const double* a, const double* b, double* c)
{
    c[0] = a[1] * b[2] - a[2] * b[1];
    c[1] = a[2] * b[0] - a[0] * b[2];
    c[2] = a[0] * b[1] - a[1] * b[0];
}

static double dot(const double* a, const double* b) { return a[0] * b[0] + a[1] * b[1] + a[2] * b[2]; }

/* ------------------------------------------------------------------------ */
/* site-site interactions                                                    */

/* reaction-field constants (reading A4; Saager et al., bib of P:39)         */
static double krf_qq(const or_sys* S)
{
    double rc3 = S->rc * S->rc * S->rc;
    if (isinf(S->eps_rf)) return 1.0 / (2.0 * rc3);
    return (S->eps_rf - 1.0) / ((2.0 * S->eps_rf + 1.0) * rc3);
}
static double krf_mumu(const or_sys* S)
{
    double rc3 = S->rc * S->rc * S->rc;
    if (isinf(S->eps_rf)) return 1.0 / rc3;
    return 2.0 * (S->eps_rf - 1.0) / ((2.0 * S->eps_rf + 1.0) * rc3);
}

/*
 * One site pair.  rv = x_b - x_a (world), ea/eb world axes (polar sites).
 * Adds u to *U, the force on site b to fb (force on a is -fb), and the
 * site torques (about the site) to ta, tb.  eta = binary parameter.
 *
 * Polar kinds (reading A5, Gray & Gubbins normalisation Q = sum q z^2):
 * with c_a = e_a.rhat, c_b = e_b.rhat, c_ab = e_a.e_b
 *   q-mu  : u = -q mu c_b / r^2                 (dipole b)
 *   q-Q   : u =  q Q (3 c_b^2 - 1) / (2 r^3)
 *   mu-mu : u =  mu_a mu_b (c_ab - 3 c_a c_b) / r^3  - k_rf mu_a mu_b c_ab
 *   mu-Q  : u =  3 mu Q / (2 r^4) [c_a (5 c_b^2 - 1) - 2 c_b c_ab]
 *   Q-Q   : u =  3 Q_a Q_b / (4 r^5) [1 - 5c_a^2 - 5c_b^2 - 15 c_a^2 c_b^2
 *                                      + 2 (c_ab - 5 c_a c_b)^2]
 * Reversed order (polar a, lower-rank b): swap roles, c -> -c.
 * Force  f_b = -du/dr_vec, du/dr_vec = u_r rhat + u_ca (e_a - c_a rhat)/r
 *                                      + u_cb (e_b - c_b rhat)/r
 * Torque t_a = -e_a x (u_ca rhat + u_cab e_b), t_b = -e_b x (u_cb rhat + u_cab e_a).
 */
void or_site_pair(const or_sys* S, const or_site* a, const double* ea,
                  const or_site* b, const double* eb, double eta, const double* rv,
                  double* U, double* fb, double* ta, double* tb)
{
    double r2 = dot(rv, rv);
    double r = sqrt(r2);
    int A = a->type, B = b->type;
    if (A == OR_LJ || B == OR_LJ) {
        if (A != OR_LJ || B != OR_LJ) return;           /* LJ only with LJ */
        double sig = 0.5 * (a->sigma + b->sigma);       /* Lorentz          */
        double eps = eta * sqrt(a->eps * b->eps);       /* Berthelot * eta  */
        double sr2 = sig * sig / r2, sr6 = sr2 * sr2 * sr2, sr12 = sr6 * sr6;
        double u = 4.0 * eps * (sr12 - sr6);            /* Eq. 1      */
        if (S->lj_shift) {                              /* LJTS, A2   */
            double sc2 = sig * sig / (S->rc * S->rc), sc6 = sc2 * sc2 * sc2;
            u -= 4.0 * eps * (sc6 * sc6 - sc6);
        }
        double fr = 24.0 * eps * (2.0 * sr12 - sr6) / r2;
        *U += u;
        for (int k = 0; k < 3; ++k) fb[k] += fr * rv[k];
        return;
    }
    if (A == OR_CHARGE && B == OR_CHARGE) {             /* Coulomb + RF, A4 */
        double k = krf_qq(S);
        double c = 1.0 / S->rc + k * S->rc * S->rc;
        double qq = a->m * b->m;
        *U += qq * (1.0 / r + k * r2 - c);
        double fr = qq * (1.0 / (r2 * r) - 2.0 * k);
        for (int d = 0; d < 3; ++d) fb[d] += fr * rv[d];
        return;
    }
    /* polar kinds through the generic (u_r, u_ca, u_cb, u_cab) recipe */
    double rh[3] = {rv[0] / r, rv[1] / r, rv[2] / r};
    double zero[3] = {0, 0, 0};
    const double* EA = (A == OR_CHARGE) ? zero : ea;
    const double* EB = (B == OR_CHARGE) ? zero : eb;
    double ca = dot(EA, rh), cb = dot(EB, rh), cab = dot(EA, EB);
    double u = 0, ur = 0, uca = 0, ucb = 0, ucab = 0;
    double r3 = r2 * r, r4 = r2 * r2, r5 = r4 * r;
    if (A == OR_CHARGE && B == OR_DIPOLE) {
        double p = a->m * b->m;
        u = -p * cb / r2; ur = 2.0 * p * cb / r3; ucb = -p / r2;
    } else if (A == OR_DIPOLE && B == OR_CHARGE) {
        double p = a->m * b->m;
        u = p * ca / r2; ur = -2.0 * p * ca / r3; uca = p / r2;
    } else if (A == OR_CHARGE && B == OR_QUADRUPOLE) {
        double p = a->m * b->m;
        u = p * (3 * cb * cb - 1) / (2 * r3); ur = -3.0 * u / r; ucb = 3.0 * p * cb / r3;
    } else if (A == OR_QUADRUPOLE && B == OR_CHARGE) {
        double p = a->m * b->m;
        u = p * (3 * ca * ca - 1) / (2 * r3); ur = -3.0 * u / r; uca = 3.0 * p * ca / r3;
    } else if (A == OR_DIPOLE && B == OR_DIPOLE) {
        double p = a->m * b->m;
        u = p * (cab - 3 * ca * cb) / r3; ur = -3.0 * u / r;
        uca = -3.0 * p * cb / r3; ucb = -3.0 * p * ca / r3; ucab = p / r3;
        double k = krf_mumu(S);                          /* RF, A4   */
        u += -k * p * cab; ucab += -k * p;
    } else if (A == OR_DIPOLE && B == OR_QUADRUPOLE) {
        double p = 1.5 * a->m * b->m / r4;
        u = p * (ca * (5 * cb * cb - 1) - 2 * cb * cab); ur = -4.0 * u / r;
        uca = p * (5 * cb * cb - 1); ucb = p * (10 * ca * cb - 2 * cab); ucab = -2.0 * p * cb;
    } else if (A == OR_QUADRUPOLE && B == OR_DIPOLE) {
        double p = -1.5 * a->m * b->m / r4;
        u = p * (cb * (5 * ca * ca - 1) - 2 * ca * cab); ur = -4.0 * u / r;
        ucb = p * (5 * ca * ca - 1); uca = p * (10 * ca * cb - 2 * cab); ucab = -2.0 * p * ca;
    } else if (A == OR_QUADRUPOLE && B == OR_QUADRUPOLE) {
        double p = 0.75 * a->m * b->m / r5;
        double g = cab - 5 * ca * cb;
        u = p * (1 - 5 * ca * ca - 5 * cb * cb - 15 * ca * ca * cb * cb + 2 * g * g);
        ur = -5.0 * u / r;
        uca = p * (-10 * ca - 30 * ca * cb * cb - 20 * cb * g);
        ucb = p * (-10 * cb - 30 * ca * ca * cb - 20 * ca * g);
        ucab = p * 4 * g;
    }
    *U += u;
    for (int k = 0; k < 3; ++k) {
        double du = ur * rh[k] + (uca * (EA[k] - ca * rh[k]) + ucb * (EB[k] - cb * rh[k])) / r;
        fb[k] -= du;
    }
    if (A != OR_CHARGE) {
        double g[3], t[3];
        for (int k = 0; k < 3; ++k) g[k] = uca * rh[k] + ucab * EB[k];
        cross(EA, g, t);
        for (int k = 0; k < 3; ++k) ta[k] -= t[k];
    }
    if (B != OR_CHARGE) {
        double g[3], t[3];
        for (int k = 0; k < 3; ++k) g[k] = ucb * rh[k] + ucab * EA[k];
        cross(EB, g, t);
        for (int k = 0; k < 3; ++k) tb[k] -= t[k];
    }
}

/* ------------------------------------------------------------------------ */
/* molecule pairs                                                            */

typedef struct {
    const or_sys* S;
    int64_t n;
    const int32_t* comp;
    const uint32_t* u;
    double* sp;    /* world site offsets s_ia = R(q_i) d_a, [n][maxs][3]      */
    double* se;    /* world site axes    e_ia = R(q_i) e_a, [n][maxs][3]      */
    int maxs;
} or_state;

static int max_sites(const or_sys* S)
{
    int m = 0;
    for (int c = 0; c < S->n_comp; ++c) if (S->comp[c].nsites > m) m = S->comp[c].nsites;
    return m;
}

/* sites in the world frame: s_ia = R(q_i) d_a, e_ia = R(q_i) e_a */
static int state_init(or_state* X, const or_sys* S, int64_t n, const int32_t* comp,
                      const uint32_t* u, const double* q)
{
    X->S = S; X->n = n; X->comp = comp; X->u = u;
    X->maxs = max_sites(S);
    size_t sz = (size_t)n * X->maxs * 3;
    X->sp = (double*)malloc(sizeof(double) * (sz ? sz : 1));
    X->se = (double*)malloc(sizeof(double) * (sz ? sz : 1));
    if (!X->sp || !X->se) return -1;
    for (int64_t i = 0; i < n; ++i) {
        double R[3][3];
        quat_to_R(q + 4 * i, R);
        const or_comp* C = &S->comp[comp[i]];
        for (int a = 0; a < C->nsites; ++a) {
            const or_site* st = &S->sites[C->site0 + a];
            matvec(R, st->r, X->sp + ((size_t)i * X->maxs + a) * 3);
            matvec(R, st->e, X->se + ((size_t)i * X->maxs + a) * 3);
        }
    }
    return 0;
}

static void state_free(or_state* X) { free(X->sp); free(X->se); }

/*
 * Interaction of molecule j with molecule i given the COM separation
 * rij = r_j - r_i (world units).  Returns 1 if the pair is within the cutoff
 * (A1: COM distance decides, strict r < rc) and then adds to
 *   Fi (force on i), ti (torque on i about its COM), tj (torque on j),
 *   *U, and returns the molecular virial term -rij.F_i in *w.
 * The force on j is -Fi.
 */
static int mol_pair_r(const or_state* X, int64_t i, int64_t j, const double rij[3],
                      double* U, double* Fi, double* ti, double* tj, double* w)
{
    const or_sys* S = X->S;
    double r2 = dot(rij, rij);           /* exact when near rc (A12) */
    if (!(r2 < S->rc * S->rc)) return 0;
    const or_comp* Ci = &S->comp[X->comp[i]];
    const or_comp* Cj = &S->comp[X->comp[j]];
    double eta = S->eta ? S->eta[X->comp[i] * S->n_comp + X->comp[j]] : 1.0;
    double Fsum[3] = {0, 0, 0};
    for (int a = 0; a < Ci->nsites; ++a) {
        const or_site* sa = &S->sites[Ci->site0 + a];
        const double* pa = X->sp + ((size_t)i * X->maxs + a) * 3;
        const double* ea = X->se + ((size_t)i * X->maxs + a) * 3;
        for (int b = 0; b < Cj->nsites; ++b) {
            const or_site* sb = &S->sites[Cj->site0 + b];
            const double* pb = X->sp + ((size_t)j * X->maxs + b) * 3;
            const double* eb = X->se + ((size_t)j * X->maxs + b) * 3;
            double rv[3] = {rij[0] + pb[0] - pa[0], rij[1] + pb[1] - pa[1], rij[2] + pb[2] - pa[2]};
            double fb[3] = {0, 0, 0}, ta[3] = {0, 0, 0}, tb[3] = {0, 0, 0};
            or_site_pair(S, sa, ea, sb, eb, eta, rv, U, fb, ta, tb);
            /* force on site a is -fb; molecular torque = lever x force + site torque */
            double fa[3] = {-fb[0], -fb[1], -fb[2]}, c[3];
            cross(pa, fa, c);
            for (int k = 0; k < 3; ++k) { Fsum[k] += fa[k]; ti[k] += c[k] + ta[k]; }
            cross(pb, fb, c);
            for (int k = 0; k < 3; ++k) tj[k] += c[k] + tb[k];
        }
    }
    for (int k = 0; k < 3; ++k) Fi[k] += Fsum[k];
    *w = -dot(rij, Fsum);                /* molecular virial, A6 */
    return 1;
}

/* the same for a separation given in quanta (A12): rij = dq s, exact        */
static int mol_pair(const or_state* X, int64_t i, int64_t j, const int64_t dq[3],
                    double* U, double* Fi, double* ti, double* tj, double* w)
{
    const or_sys* S = X->S;
    double rij[3] = {dq[0] * S->s, dq[1] * S->s, dq[2] * S->s};   /* exact */
    return mol_pair_r(X, i, j, rij, U, Fi, ti, tj, w);
}

/* ------------------------------------------------------------------------ */
/* force evaluations                                                         */

typedef struct {
    double U, W;
    int64_t npairs;
} or_totals;

/* brute force over all unordered pairs i<j: the plain definition (A11)     */
int or_forces_brute(const or_sys* S, int64_t n, const int32_t* comp, const uint32_t* u,
                    const double* q, double* F, double* tau, or_totals* out)
{
    or_state X;
    if (state_init(&X, S, n, comp, u, q)) return -2;
    memset(F, 0, sizeof(double) * 3 * n);
    memset(tau, 0, sizeof(double) * 3 * n);
    double U = 0, W = 0;
    int64_t np = 0;
    for (int64_t i = 0; i < n; ++i)
        for (int64_t j = i + 1; j < n; ++j) {
            int64_t d[3];
            min_image(S, u + 3 * i, u + 3 * j, d);
            double Fi[3] = {0, 0, 0}, w = 0;
            if (mol_pair(&X, i, j, d, &U, Fi, tau + 3 * i, tau + 3 * j, &w)) {
                for (int k = 0; k < 3; ++k) { F[3 * i + k] += Fi[k]; F[3 * j + k] -= Fi[k]; }
                W += w;
                np += 1;
            }
        }
    state_free(&X);
    out->U = U; out->W = W; out->npairs = np;
    return 0;
}

/* cell lists: molecules of each cell in ascending index order              */
typedef struct {
    int64_t ncell;
    int64_t* start;   /* ncell + 1 */
    int64_t* list;
} or_cl;

static int cl_build(or_cl* C, const or_sys* S, int64_t n, const uint32_t* u)
{
    C->ncell = (int64_t)S->nc[0] * S->nc[1] * S->nc[2];
    C->start = (int64_t*)calloc(C->ncell + 1, sizeof(int64_t));
    C->list = (int64_t*)malloc(sizeof(int64_t) * (n ? n : 1));
    int32_t* cell = (int32_t*)malloc(sizeof(int32_t) * (n ? n : 1));
    int32_t* cnt = (int32_t*)malloc(sizeof(int32_t) * C->ncell);
    if (!C->start || !C->list || !cell || !cnt) return -1;
    or_cells(S, n, u, cell, cnt);
    for (int64_t c = 0; c < C->ncell; ++c) C->start[c + 1] = C->start[c] + cnt[c];
    for (int64_t c = 0; c < C->ncell; ++c) cnt[c] = 0;
    for (int64_t i = 0; i < n; ++i) C->list[C->start[cell[i]] + cnt[cell[i]]++] = i;
    free(cell); free(cnt);
    return 0;
}

static void cl_free(or_cl* C) { free(C->start); free(C->list); }

static int64_t cell_at(const or_sys* S, int cx, int cy, int cz)
{
    cx = (cx + S->nc[0]) % S->nc[0];
    cy = (cy + S->nc[1]) % S->nc[1];
    cz = (cz + S->nc[2]) % S->nc[2];
    return cx + (int64_t)S->nc[0] * (cy + (int64_t)S->nc[1] * cz);
}

/* linked cells, Newton-3 half shell: pairs inside a cell (i<j) plus the 13
 * "forward" neighbour cells (Fig. 1).  Needs >= 3 cells per
 * axis so that the 26 neighbours are distinct cells.                        */
int or_forces_cells(const or_sys* S, int64_t n, const int32_t* comp, const uint32_t* u,
                    const double* q, double* F, double* tau, or_totals* out)
{
    if (S->nc[0] < 3 || S->nc[1] < 3 || S->nc[2] < 3) return -1;
    or_state X;
    or_cl C;
    if (state_init(&X, S, n, comp, u, q) || cl_build(&C, S, n, u)) return -2;
    memset(F, 0, sizeof(double) * 3 * n);
    memset(tau, 0, sizeof(double) * 3 * n);
    double U = 0, W = 0;
    int64_t np = 0;
    for (int cz = 0; cz < S->nc[2]; ++cz)
        for (int cy = 0; cy < S->nc[1]; ++cy)
            for (int cx = 0; cx < S->nc[0]; ++cx) {
                int64_t c = cell_at(S, cx, cy, cz);
                for (int oz = -1; oz <= 1; ++oz)
                    for (int oy = -1; oy <= 1; ++oy)
                        for (int ox = -1; ox <= 1; ++ox) {
                            int fwd = oz > 0 || (oz == 0 && (oy > 0 || (oy == 0 && ox >= 0)));
                            if (!fwd) continue;
                            int self = (ox == 0 && oy == 0 && oz == 0);
                            int64_t c2 = cell_at(S, cx + ox, cy + oy, cz + oz);
                            for (int64_t a = C.start[c]; a < C.start[c + 1]; ++a)
                                for (int64_t b = self ? a + 1 : C.start[c2]; b < C.start[c2 + 1]; ++b) {
                                    int64_t i = C.list[a], j = C.list[b], d[3];
                                    min_image(S, u + 3 * i, u + 3 * j, d);
                                    double Fi[3] = {0, 0, 0}, w = 0;
                                    if (mol_pair(&X, i, j, d, &U, Fi, tau + 3 * i, tau + 3 * j, &w)) {
                                        for (int k = 0; k < 3; ++k) { F[3 * i + k] += Fi[k]; F[3 * j + k] -= Fi[k]; }
                                        W += w;
                                        np += 1;
                                    }
                                }
                        }
            }
    cl_free(&C);
    state_free(&X);
    out->U = U; out->W = W; out->npairs = np;
    return 0;
}

/* Full 27-cell shell per molecule, for the molecules listed in idx (all if
 * idx == NULL): F, tau of molecule i from every partner j.  Each molecule is
 * independent, so this is the "all cores" oracle (OpenMP over molecules);
 * per-molecule u_i, w_i are half the pair sums (each pair is seen twice).
 * Totals are summed afterwards in index order: deterministic for any
 * thread count.                                                              */
int or_forces_full(const or_sys* S, int64_t n, const int32_t* comp, const uint32_t* u,
                   const double* q, int64_t nsel, const int64_t* idx,
                   double* F, double* tau, double* ui, double* wi, int64_t* npi, int nthreads)
{
    if (S->nc[0] < 3 || S->nc[1] < 3 || S->nc[2] < 3) return -1;
    or_state X;
    or_cl C;
    if (state_init(&X, S, n, comp, u, q) || cl_build(&C, S, n, u)) return -2;
    int64_t m = idx ? nsel : n;
#ifdef _OPENMP
    if (nthreads > 0) omp_set_num_threads(nthreads);
#pragma omp parallel for schedule(dynamic, 256)
#endif
    for (int64_t t = 0; t < m; ++t) {
        int64_t i = idx ? idx[t] : t;
        double Fi[3] = {0, 0, 0}, ti[3] = {0, 0, 0}, U = 0, W = 0;
        int64_t np = 0;
        int cx = (int)(u[3 * i + 0] / S->E[0]);
        int cy = (int)(u[3 * i + 1] / S->E[1]);
        int cz = (int)(u[3 * i + 2] / S->E[2]);
        for (int oz = -1; oz <= 1; ++oz)
            for (int oy = -1; oy <= 1; ++oy)
                for (int ox = -1; ox <= 1; ++ox) {
                    int64_t c2 = cell_at(S, cx + ox, cy + oy, cz + oz);
                    for (int64_t b = C.start[c2]; b < C.start[c2 + 1]; ++b) {
                        int64_t j = C.list[b], d[3];
                        if (j == i) continue;
                        min_image(S, u + 3 * i, u + 3 * j, d);
                        double tj[3] = {0, 0, 0}, w = 0;
                        if (mol_pair(&X, i, j, d, &U, Fi, ti, tj, &w)) { W += w; np += 1; }
                    }
                }
        for (int k = 0; k < 3; ++k) { F[3 * t + k] = Fi[k]; tau[3 * t + k] = ti[k]; }
        if (ui) ui[t] = 0.5 * U;
        if (wi) wi[t] = 0.5 * W;
        if (npi) npi[t] = np;
    }
    cl_free(&C);
    state_free(&X);
    return 0;
}

/* ------------------------------------------------------------------------ */
/* integration (readings A7, A8, A9, A23)                         */

static void quat_mul(const double* a, const double* b, double* c)
{
    c[0] = a[0] * b[0] - a[1] * b[1] - a[2] * b[2] - a[3] * b[3];
    c[1] = a[0] * b[1] + a[1] * b[0] + a[2] * b[3] - a[3] * b[2];
    c[2] = a[0] * b[2] - a[1] * b[3] + a[2] * b[0] + a[3] * b[1];
    c[3] = a[0] * b[3] + a[1] * b[2] - a[2] * b[1] + a[3] * b[0];
}

static void quat_normalize(double* q)
{
    double n = sqrt(q[0] * q[0] + q[1] * q[1] + q[2] * q[2] + q[3] * q[3]);
    for (int k = 0; k < 4; ++k) q[k] /= n;
}

/* omega_body = I^-1 R^T(q) j  (zero about an axis with I_k = 0)             */
static void body_omega(const or_comp* C, const double* q, const double* j, double* wb)
{
    double R[3][3], jb[3];
    quat_to_R(q, R);
    matTvec(R, j, jb);
    for (int k = 0; k < 3; ++k) wb[k] = C->I[k] > 0 ? jb[k] / C->I[k] : 0.0;
}

static int rot_dof(const or_comp* C)
{
    int d = 0;
    for (int k = 0; k < 3; ++k) d += C->I[k] > 0;
    return d;
}

/* observables of one step (A23): U, W, KE_t, KE_r, T, n_pairs              */
typedef struct {
    double U, W, KEt, KEr, T;
    int64_t npairs;
} or_obs;

/*
 * Run nsteps leapfrog steps from (u, v, q, j).  half_step = 0: v, j are
 * on-step values at t0 and are first moved back half a step with F(t0),
 * tau(t0) (A8); 1: they already are v(t0-dt/2), j(t0-dt/2).
 * Step k: F, tau, U, W at t_k; KE at t_k (A9); record obs[k]; then
 *   v(t+dt/2) = v(t-dt/2) + dt F/m                                  Eq. 2
 *   r(t+dt)   = r(t) + dt v(t+dt/2), as u += rint(dt v / s) mod P  Eq. 3, A12
 *   Fincham rotation (A7):
 *     j(t)      = j(t-dt/2) + dt/2 tau
 *     w_b(t)    = I^-1 R^T(q(t)) j(t)
 *     q(t+dt/2) = q(t) + dt/2 * 1/2 q(t) (x) (0, w_b(t)), normalised
 *     j(t+dt/2) = j(t-dt/2) + dt tau                               Eq. 4
 *     w_b'      = I^-1 R^T(q(t+dt/2)) j(t+dt/2)
 *     q(t+dt)   = q(t) + dt * 1/2 q(t+dt/2) (x) (0, w_b'), normalised   Eq. 5
 * On return u, v, q, j hold r(t_n), v(t_n - dt/2), q(t_n), j(t_n - dt/2).
 * mode 0 = brute force, 1 = linked cells (half shell), 2 = full shell/OpenMP.
 */
int or_run_nvt(const or_sys* S, double dt, int64_t n, const int32_t* comp, uint32_t* u,
               double* v, double* q, double* j, int nsteps, int half_step, int mode,
               int nthreads, double T_target, int interval, or_obs* obs)
{
    double* F = (double*)malloc(sizeof(double) * 3 * (n ? n : 1));
    double* tau = (double*)malloc(sizeof(double) * 3 * (n ? n : 1));
    double* ui = (double*)malloc(sizeof(double) * (n ? n : 1));
    double* wi = (double*)malloc(sizeof(double) * (n ? n : 1));
    int64_t* npi = (int64_t*)malloc(sizeof(int64_t) * (n ? n : 1));
    if (!F || !tau || !ui || !wi || !npi) return -2;
    int64_t ndof = 3 * n;
    for (int64_t i = 0; i < n; ++i) ndof += rot_dof(&S->comp[comp[i]]);
    int rc = 0;
    for (int step = 0; step < nsteps; ++step) {
        or_totals tot = {0, 0, 0};
        if (mode == 0) rc = or_forces_brute(S, n, comp, u, q, F, tau, &tot);
        else if (mode == 1) rc = or_forces_cells(S, n, comp, u, q, F, tau, &tot);
        else {
            rc = or_forces_full(S, n, comp, u, q, 0, NULL, F, tau, ui, wi, npi, nthreads);
            for (int64_t i = 0; i < n; ++i) { tot.U += ui[i]; tot.W += wi[i]; tot.npairs += npi[i]; }
            tot.npairs /= 2;
        }
        if (rc) break;
        if (step == 0 && !half_step) {           /* A8: backward half kick */
            for (int64_t i = 0; i < n; ++i) {
                const or_comp* C = &S->comp[comp[i]];
                for (int k = 0; k < 3; ++k) {
                    v[3 * i + k] -= 0.5 * dt * F[3 * i + k] / C->mass;
                    j[3 * i + k] -= 0.5 * dt * tau[3 * i + k];
                }
            }
        }
        double KEt = 0, KEr = 0;
        for (int64_t i = 0; i < n; ++i) {
            const or_comp* C = &S->comp[comp[i]];
            double* vi = v + 3 * i;
            double* ji = j + 3 * i;
            double* qi = q + 4 * i;
            const double* Fi = F + 3 * i;
            const double* ti = tau + 3 * i;
            /* A9: KE_t(t) from v(t) = v(t-dt/2) + dt/2 F/m */
            double vt[3];
            for (int k = 0; k < 3; ++k) vt[k] = vi[k] + 0.5 * dt * Fi[k] / C->mass;
            KEt += 0.5 * C->mass * dot(vt, vt);
            /* Eqs. 2-3 */
            for (int k = 0; k < 3; ++k) {
                vi[k] += dt * Fi[k] / C->mass;
                int64_t x = (int64_t)u[3 * i + k] + (int64_t)rint(dt * vi[k] / S->s);
                x %= S->P[k];
                if (x < 0) x += S->P[k];
                u[3 * i + k] = (uint32_t)x;
            }
            if (rot_dof(C) == 0) continue;
            /* Fincham rotational leapfrog, A7 */
            double jt[3], wb[3], wq[4], dq[4], qh[4], jb[3];
            for (int k = 0; k < 3; ++k) jt[k] = ji[k] + 0.5 * dt * ti[k];
            body_omega(C, qi, jt, wb);
            {
                double R[3][3];
                quat_to_R(qi, R);
                matTvec(R, jt, jb);
                KEr += 0.5 * dot(jb, wb);
            }
            wq[0] = 0; wq[1] = wb[0]; wq[2] = wb[1]; wq[3] = wb[2];
            quat_mul(qi, wq, dq);
            for (int k = 0; k < 4; ++k) qh[k] = qi[k] + 0.5 * dt * 0.5 * dq[k];
            quat_normalize(qh);
            for (int k = 0; k < 3; ++k) ji[k] += dt * ti[k];
            body_omega(C, qh, ji, wb);
            wq[1] = wb[0]; wq[2] = wb[1]; wq[3] = wb[2];
            quat_mul(qh, wq, dq);
            for (int k = 0; k < 4; ++k) qi[k] += dt * 0.5 * dq[k];
            quat_normalize(qi);
        }
        obs[step].U = tot.U;
        obs[step].W = tot.W;
        obs[step].KEt = KEt;
        obs[step].KEr = KEr;
        obs[step].T = 2.0 * (KEt + KEr) / (double)ndof;
        obs[step].npairs = tot.npairs;
        /* NVT ("kept constant by velocity rescaling"; reading A24): after every
         * interval-th step the half-step velocities and angular momenta are scaled by
         * lambda = sqrt(T_target / T(t_k)) */
        if (T_target > 0 && interval > 0 && (step + 1) % interval == 0) {
            if (!(obs[step].T > 0)) { rc = -3; break; }
            const double lambda = sqrt(T_target / obs[step].T);
            for (int64_t i = 0; i < 3 * n; ++i) { v[i] *= lambda; j[i] *= lambda; }
        }
    }
    free(F); free(tau); free(ui); free(wi); free(npi);
    return rc;
}

int or_run(const or_sys* S, double dt, int64_t n, const int32_t* comp, uint32_t* u,
           double* v, double* q, double* j, int nsteps, int half_step, int mode,
           int nthreads, or_obs* obs)
{
    return or_run_nvt(S, dt, n, comp, u, v, q, j, nsteps, half_step, mode, nthreads, 0.0, 0, obs);
}

/* ------------------------------------------------------------------------ */
/* Unquantised reference run (pin of reading A12): the same    */
/* leapfrog + Fincham steps as or_run_nvt, but positions are plain doubles   */
/* r in [0, box) (no fixed-point lattice): r += dt v, wrapped mod box, and   */
/* the forces come from a brute-force full shell with the fp64 minimum image  */
/* d = r_j - r_i - box rint((r_j - r_i)/box) (A1 strict r < rc).      */
/* Used only to bound the effect of the position quantum s on U, W, T.       */
static int forces_cont(const or_sys* S, int64_t n, const int32_t* comp, const double* r, const double* q,
                       double* F, double* tau, double* ui, double* wi, int64_t* npi, int nthreads)
{
    or_state X;
    if (state_init(&X, S, n, comp, NULL, q)) return -2;
#ifdef _OPENMP
    if (nthreads > 0) omp_set_num_threads(nthreads);
#pragma omp parallel for schedule(dynamic, 64)
#endif
    for (int64_t i = 0; i < n; ++i) {
        double Fi[3] = {0, 0, 0}, ti[3] = {0, 0, 0}, U = 0, W = 0;
        int64_t np = 0;
        for (int64_t j = 0; j < n; ++j) {
            if (j == i) continue;
            double d[3];
            for (int k = 0; k < 3; ++k) {
                d[k] = r[3 * j + k] - r[3 * i + k];
                d[k] -= S->box[k] * rint(d[k] / S->box[k]);
            }
            double tj[3] = {0, 0, 0}, w = 0;
            if (mol_pair_r(&X, i, j, d, &U, Fi, ti, tj, &w)) { W += w; np += 1; }
        }
        for (int k = 0; k < 3; ++k) { F[3 * i + k] = Fi[k]; tau[3 * i + k] = ti[k]; }
        ui[i] = 0.5 * U; wi[i] = 0.5 * W; npi[i] = np;
    }
    state_free(&X);
    return 0;
}

int or_run_cont(const or_sys* S, double dt, int64_t n, const int32_t* comp, double* r,
                double* v, double* q, double* j, int nsteps, int half_step, int nthreads, or_obs* obs)
{
    double* F = (double*)malloc(sizeof(double) * 3 * (n ? n : 1));
    double* tau = (double*)malloc(sizeof(double) * 3 * (n ? n : 1));
    double* ui = (double*)malloc(sizeof(double) * (n ? n : 1));
    double* wi = (double*)malloc(sizeof(double) * (n ? n : 1));
    int64_t* npi = (int64_t*)malloc(sizeof(int64_t) * (n ? n : 1));
    if (!F || !tau || !ui || !wi || !npi) return -2;
    int64_t ndof = 3 * n;
    for (int64_t i = 0; i < n; ++i) ndof += rot_dof(&S->comp[comp[i]]);
    int rc = 0;
    for (int step = 0; step < nsteps; ++step) {
        rc = forces_cont(S, n, comp, r, q, F, tau, ui, wi, npi, nthreads);
        if (rc) break;
        double U = 0, W = 0;
        int64_t np = 0;
        for (int64_t i = 0; i < n; ++i) { U += ui[i]; W += wi[i]; np += npi[i]; }
        if (step == 0 && !half_step) {           /* A8: backward half kick */
            for (int64_t i = 0; i < n; ++i) {
                const or_comp* C = &S->comp[comp[i]];
                for (int k = 0; k < 3; ++k) {
                    v[3 * i + k] -= 0.5 * dt * F[3 * i + k] / C->mass;
                    j[3 * i + k] -= 0.5 * dt * tau[3 * i + k];
                }
            }
        }
        double KEt = 0, KEr = 0;
        for (int64_t i = 0; i < n; ++i) {
            const or_comp* C = &S->comp[comp[i]];
            double* vi = v + 3 * i;
            double* ji = j + 3 * i;
            double* qi = q + 4 * i;
            const double* Fi = F + 3 * i;
            const double* ti = tau + 3 * i;
            double vt[3];
            for (int k = 0; k < 3; ++k) vt[k] = vi[k] + 0.5 * dt * Fi[k] / C->mass;
            KEt += 0.5 * C->mass * dot(vt, vt);
            for (int k = 0; k < 3; ++k) {                 /* Eqs. 2-3, no lattice */
                vi[k] += dt * Fi[k] / C->mass;
                double x = r[3 * i + k] + dt * vi[k];
                x -= S->box[k] * floor(x / S->box[k]);
                r[3 * i + k] = x;
            }
            if (rot_dof(C) == 0) continue;
            double jt[3], wb[3], wq[4], dq[4], qh[4], jb[3];   /* A7, as in or_run_nvt */
            for (int k = 0; k < 3; ++k) jt[k] = ji[k] + 0.5 * dt * ti[k];
            body_omega(C, qi, jt, wb);
            {
                double R[3][3];
                quat_to_R(qi, R);
                matTvec(R, jt, jb);
                KEr += 0.5 * dot(jb, wb);
            }
            wq[0] = 0; wq[1] = wb[0]; wq[2] = wb[1]; wq[3] = wb[2];
            quat_mul(qi, wq, dq);
            for (int k = 0; k < 4; ++k) qh[k] = qi[k] + 0.5 * dt * 0.5 * dq[k];
            quat_normalize(qh);
            for (int k = 0; k < 3; ++k) ji[k] += dt * ti[k];
            body_omega(C, qh, ji, wb);
            wq[1] = wb[0]; wq[2] = wb[1]; wq[3] = wb[2];
            quat_mul(qh, wq, dq);
            for (int k = 0; k < 4; ++k) qi[k] += dt * 0.5 * dq[k];
            quat_normalize(qi);
        }
        obs[step].U = U;
        obs[step].W = W;
        obs[step].KEt = KEt;
        obs[step].KEr = KEr;
        obs[step].T = 2.0 * (KEt + KEr) / (double)ndof;
        obs[step].npairs = np / 2;
    }
    free(F); free(tau); free(ui); free(wi); free(npi);
    return rc;
}

/* ------------------------------------------------------------------------ */
/* isotropic LJ tail corrections ("isotropic cut-off corrections ... a  */
/* mean-field integral for the dispersive interaction"; reading A3): with     */
/* g(r) = 1 beyond rc, for every ordered pair of components and every LJ     */
/* site pair (a, b) with sigma, eps mixed as in the forces:           */
/*   U_lrc = (1/2) sum N_ci N_cj / V  int_rc^inf u_ab(r) 4 pi r^2 dr          */
/*   W_lrc = -(1/2) sum N_ci N_cj / V int_rc^inf r u_ab'(r) 4 pi r^2 dr        */
/* with u_ab the plain 12-6 potential (the shift of LJTS does not act beyond  */
/* rc).  The integrals in closed form:                                        */
/*   int_rc^inf u 4 pi r^2 dr    = 16 pi eps sig^3 [ (sig/rc)^9 / 9 - (sig/rc)^3 / 3 ] */
/*   int_rc^inf r u' 4 pi r^2 dr = 16 pi eps sig^3 [ -4/3 (sig/rc)^9 + 2 (sig/rc)^3 ] */
void or_lj_tail(const or_sys* S, const int64_t* counts, double volume, double* U, double* W)
{
    double u = 0.0, w = 0.0;
    for (int ci = 0; ci < S->n_comp; ++ci)
        for (int cj = 0; cj < S->n_comp; ++cj) {
            const double eta = S->eta ? S->eta[ci * S->n_comp + cj] : 1.0;
            const double nn = (double)counts[ci] * (double)counts[cj] / volume;
            const or_comp* A = &S->comp[ci];
            const or_comp* B = &S->comp[cj];
            for (int a = 0; a < A->nsites; ++a)
                for (int b = 0; b < B->nsites; ++b) {
                    const or_site* sa = &S->sites[A->site0 + a];
                    const or_site* sb = &S->sites[B->site0 + b];
                    if (sa->type != OR_LJ || sb->type != OR_LJ) continue;
                    const double sig = 0.5 * (sa->sigma + sb->sigma);
                    const double eps = eta * sqrt(sa->eps * sb->eps);
                    const double x3 = pow(sig / S->rc, 3.0), x9 = x3 * x3 * x3;
                    const double pre = 16.0 * 3.14159265358979323846 * eps * sig * sig * sig;
                    u += 0.5 * nn * pre * (x9 / 9.0 - x3 / 3.0);
                    w -= 0.5 * nn * pre * (-4.0 / 3.0 * x9 + 2.0 * x3);
                }
        }
    *U = u;
    *W = w;
}
