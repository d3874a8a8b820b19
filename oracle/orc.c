/*
 * orc.c -- plain, slow, obviously-correct complex128 CPU ORACLE for the RAS-PML hot path of
 * arXiv 2602.00735 ("Massively parallel Schwarz methods for the high frequency Helmholtz equation").
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
 * --impl reference legs may load this library.  The product (paper_2602_00735_b200/, libhelm) never
 * links, includes or calls it, and this file shares no code, header or table with the product.
 *
 * Citations: "P:n" = /root/reference/PAPER.md line n (section / equation named alongside).
 * Readings of ambiguous passages are the D-numbers of DESIGN.md section 3 (same IDs as SURVEY.md 8(c)).
 *
 * Everything is IEEE fp64 complex (C99 double complex).  No BLAS, no blocking, no reordering beyond the
 * textbook definition of each step.  OpenMP is used only to run independent subdomains concurrently.
 *
 * Pins (tests/test_oracle_*.py, -m "not gpu"): grid sizes printed in BASELINE.json; the interior
 * stencil closed form; PML closed forms / finite differences; A = A^T when sigma0 = 0; interior local
 * matrix = global matrix of the (int box + kappa PML) problem; band LU vs numpy.linalg.solve;
 * dense sum_j R~_j^T A_j^-1 R_j vs the apply; single subdomain => B^-1 = A^-1; Hankel far field;
 * FEM order 2.  Q1 / paper frame (tests/test_oracle_q1.py): the bilinear interior stencil closed form,
 * symmetry without PML, the g = 10 k t^3 profile closed forms / finite differences / local restarts, local rows =
 * global rows in the int box, Q1 FEM order 2, band LU vs zgesv, dense ramp-PoU RAS vs the apply, single subdomain
 * => exact inverse, unit mass of the smoothed delta, and the iteration counts printed in the paper's Tables 1 and 4
 * at k = 300 (tests/golden/paper_iterations.txt).  The right-hand side is pinned entrywise as b = M f_I with M the
 * consistent mass recovered from the assembly (tests/test_oracle_assembly.py).  Dedup mode (orc_factor_dedup, SURVEY
 * 8(d) memory fallback) is pinned by bitwise equality of its apply with the per-subdomain factorisation and by its
 * own bitwise member == representative assertion.  No function here is "parity unpinned".
 */
#include <complex.h>
#include <math.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

typedef double complex zc;

/* ------------------------------------------------------------------------------------------------
 * Problem description.  Omega_int = (0, nix*h) x (0, niy*h) ("hyper-rectangle"), surrounded by
 * ng PML cells per side (Omega = prod (a - kappa_g, b + kappa_g)).  The PML profile width
 * kappa (D3: the same kappa_g = 10 h profile for global and local layers) is separate from the
 * number of PML cells so that layers thicker than kappa_g use the linear continuation.
 * ----------------------------------------------------------------------------------------------*/
typedef struct {
    double k;       /* wavenumber (c = 1) */
    double sigma0;  /* PML strength in g (BASELINE.json configs[0]) */
    double h;       /* mesh size */
    int nix, niy;   /* cells of Omega_int per axis */
    int ng;         /* global PML cells per side */
    double kappa;   /* profile width kappa_g in length units */
    int px, py;     /* subdomains per axis (Cartesian covering) */
    int novlp;      /* overlap delta in cells, per side of every interior face (D8) */
    int npml;       /* local PML kappa in cells on every interior face */
    int local_bc;   /* 0: RAS-PML-Drch (u = 0 on dOmega_j); 1: RAS-PML-Imp */
    int pou;        /* 0: owner indicator chi_j = 1 on block j (D10); 1: linear ramps across overlaps */
    /* paper-faithful workload (D18-D22) */
    int elem;       /* 0: P1 on the SW->NE split (D1); 1: Q1 bilinear elements, 2x2 Gauss quadrature */
    int frame;      /* 0: BJ frame -- Omega_int = (0, nix h) x (0, niy h) inside ng PML cells per side;
                       1: paper frame -- Omega = (0, nix h) x (0, niy h) itself (ng = 0) and
                          Omega_int = Omega shrunk by kappa (= kappa_g = 3 lambda) on every side */
    double pml_c;   /* frame 1: g(t) = pml_c t^3 (g(x) = 10 k x^3) */
} orc_params;

typedef struct {
    /* per axis: node-index ranges (nodes 0..N on that axis) */
    int own_lo[2], own_hi[2];   /* owned nodes [own_lo, own_hi)  (D10) */
    int int_lo[2], int_hi[2];   /* int box nodes a_j, b_j */
    int full_lo[2], full_hi[2]; /* full box nodes */
    int has_lo[2], has_hi[2];   /* local PML on lower / upper face (kappa_{j,l/u} != 0) */
    int m[2];                   /* local free nodes per axis */
    int node0[2];               /* global index of the first local free node per axis */
    /* factor storage (band LU, O7) */
    zc *band;                   /* n x (2p+1), NULL until factored */
    int factored;
    int shared;                 /* dedup mode: band belongs to a class (orc_ctx.cls), not to this subdomain */
} orc_sub;

/* dedup mode (SURVEY 8(d) "memory fallback"): one factored representative per distinct A_j */
typedef struct {
    uint64_t hash;
    int mx, my;
    int rep;                    /* representative subdomain (lowest index) */
    int count;
    zc *raw;                    /* the representative's assembled band (verification only, freed after) */
    zc *band;                   /* its band LU factors, shared by every member */
} orc_class;

typedef struct {
    orc_params p;
    int N[2];        /* cells per axis incl. PML */
    int nf[2];       /* free nodes per axis = N - 1 */
    int64_t nfree;
    int nsub;
    int *split[2];   /* block starts s_0..s_P (cells == nodes) */
    orc_sub *sub;
    int ns;          /* slots per global row: 7 (P1) or 9 (Q1) */
    double lo_u[2], hi_u[2];   /* Omega_int per axis in cell units (node 0 at 0): where the global ramps start */
    zc *A7;          /* global matrix, ns slots per free row (see slot_of) */
    orc_class *cls;  /* dedup mode classes (NULL otherwise) */
    int ncls;
} orc_ctx;

/* ------------------------------------------------------------------------------------------------
 * PML scaling function (BASELINE.json configs[0]; P:37-43 properties):
 *   g(t) = sigma0 t^3 / (3 kappa^2)              0 <= t <= kappa
 *   g(t) = sigma0 kappa / 3 + sigma0 (t - kappa)  t > kappa      ("linear beyond", C^1 at kappa)
 * out[0..2] = g, g', g''.
 * ----------------------------------------------------------------------------------------------*/
void orc_gfun(double t, double kappa, double sigma0, double *out)
{
    if (t <= 0.0) { out[0] = out[1] = out[2] = 0.0; return; }
    if (t <= kappa) {
        out[0] = sigma0 * t * t * t / (3.0 * kappa * kappa);
        out[1] = sigma0 * t * t / (kappa * kappa);
        out[2] = 2.0 * sigma0 * t / (kappa * kappa);
    } else {
        out[0] = sigma0 * kappa / 3.0 + sigma0 * (t - kappa);
        out[1] = sigma0;
        out[2] = 0.0;
    }
}

/* gamma = 1 + i g'(t), gamma' = (+/-) i g''(t): upper ramps g_i(x) = g(x - b), lower ramps
 * g_i(x) = -g(a - x) so g_i'(x) = g'(a - x) and g_i''(x) = -g''(a - x)  (D4). */
static void ramp(double t, int upper, const orc_params *p, zc *gam, zc *dgam)
{
    double g[3];
    orc_gfun(t, p->kappa, p->sigma0, g);
    *gam = 1.0 + I * g[1];
    *dgam = upper ? I * g[2] : -I * g[2];
}

/* Global gamma along one axis at a position given in thirds of a cell: x = X3 * h / 3 in node units
 * (node 0 at X3 = 0).  Omega_int spans nodes [ng, ng + ni].  Depth is formed from integer offsets (D5). */
static void gamma_global(const orc_ctx *c, int axis, long X3, zc *gam, zc *dgam)
{
    const orc_params *p = &c->p;
    long lo = 3L * p->ng, hi = 3L * (p->ng + (axis == 0 ? p->nix : p->niy));
    double h3 = p->h / 3.0;
    if (X3 > hi) ramp((double)(X3 - hi) * h3, 1, p, gam, dgam);
    else if (X3 < lo) ramp((double)(lo - X3) * h3, 0, p, gam, dgam);
    else { *gam = 1.0; *dgam = 0.0; }
}

/* Local scaling g_j^i: upper ramp from b_j above the int box, lower ramp from a_j below it,
 * the global g_i inside.  Ramps exist only on faces that carry a local PML. */
static void gamma_local(const orc_ctx *c, const orc_sub *s, int axis, long X3, zc *gam, zc *dgam)
{
    long a = 3L * s->int_lo[axis], b = 3L * s->int_hi[axis];
    double h3 = c->p.h / 3.0;
    if (s->has_hi[axis] && X3 > b) ramp((double)(X3 - b) * h3, 1, &c->p, gam, dgam);
    else if (s->has_lo[axis] && X3 < a) ramp((double)(a - X3) * h3, 0, &c->p, gam, dgam);
    else gamma_global(c, axis, X3, gam, dgam);
}

/* exported for the PML pins: sub < 0 -> global */
void orc_gamma(const orc_ctx *c, int sub, int axis, long X3, zc *gam, zc *dgam)
{
    if (sub < 0) gamma_global(c, axis, X3, gam, dgam);
    else gamma_local(c, &c->sub[sub], axis, X3, gam, dgam);
}

/* ------------------------------------------------------------------------------------------------
 * Q1 path (elem = 1): PML coefficients at arbitrary points x = (ci + xi) h of cell ci (xi in [0,1]).
 * Depth below / above a ramp start r (cell units) is formed as (r - ci) - xi resp. (ci - r) + xi, then
 * scaled by h, so identical relative positions give identical bits whenever r is a node (D5 carried over).
 * Profile: frame 0 -> the BJ profile (orc_gfun); frame 1 -> the paper's g(t) = pml_c t^3, with
 * g' = 3 pml_c t^2 and g'' = 6 pml_c t.  Signs of gamma' as in D4.
 * ----------------------------------------------------------------------------------------------*/
static void ramp_q(double t, int upper, const orc_params *p, zc *gam, zc *dgam)
{
    double g1, g2;
    if (p->frame == 1) {
        g1 = 3.0 * p->pml_c * t * t;
        g2 = 6.0 * p->pml_c * t;
    } else {
        double g[3];
        orc_gfun(t, p->kappa, p->sigma0, g);
        g1 = g[1];
        g2 = g[2];
    }
    *gam = 1.0 + I * g1;
    *dgam = upper ? I * g2 : -I * g2;
}

static void gamma_global_q(const orc_ctx *c, int axis, int ci, double xi, zc *gam, zc *dgam)
{
    double up = ((double)ci - c->hi_u[axis]) + xi, dn = (c->lo_u[axis] - (double)ci) - xi;
    if (up > 0.0) ramp_q(up * c->p.h, 1, &c->p, gam, dgam);
    else if (dn > 0.0) ramp_q(dn * c->p.h, 0, &c->p, gam, dgam);
    else { *gam = 1.0; *dgam = 0.0; }
}

/* local scaling g_j^i at a Q1 quadrature point */
static void gamma_local_q(const orc_ctx *c, const orc_sub *s, int axis, int ci, double xi, zc *gam, zc *dgam)
{
    double up = (double)(ci - s->int_hi[axis]) + xi, dn = (double)(s->int_lo[axis] - ci) - xi;
    if (s->has_hi[axis] && up > 0.0) ramp_q(up * c->p.h, 1, &c->p, gam, dgam);
    else if (s->has_lo[axis] && dn > 0.0) ramp_q(dn * c->p.h, 0, &c->p, gam, dgam);
    else gamma_global_q(c, axis, ci, xi, gam, dgam);
}

/* exported for the PML pins (Q1 path): sub < 0 -> global */
void orc_gamma_q(const orc_ctx *c, int sub, int axis, int ci, double xi, zc *gam, zc *dgam)
{
    if (sub < 0) gamma_global_q(c, axis, ci, xi, gam, dgam);
    else gamma_local_q(c, &c->sub[sub], axis, ci, xi, gam, dgam);
}

/* 2-point Gauss-Legendre abscissae on [0, 1]; weights 1/2 each */
static double gauss_xi(int q) { return q == 0 ? 0.5 - 0.5 / sqrt(3.0) : 0.5 + 0.5 / sqrt(3.0); }

/* ------------------------------------------------------------------------------------------------
 * Q1 element matrix of eq. (weak) on a square cell of side h, bilinear basis
 *   phi_a(x, y) = N_{ax}(xi) N_{ay}(eta),  N_0 = 1 - xi, N_1 = xi,  a = ax + 2 ay  (vertex (ci+ax, cj+ay)),
 * integrated with the 2 x 2 Gauss rule (weight h^2/4 per point; exact for the mass and for constant D):
 *   A_e[a][b] = sum_q h^2/4 [ D11 dx phi_a dx phi_b + D22 dy phi_a dy phi_b - (beta . grad phi_b) phi_a
 *                             - k^2 phi_a phi_b ]   (row = test phi_a, column = trial phi_b; bilinear, D6),
 * D11 = gamma_x^-2, D22 = gamma_y^-2, beta_i = gamma_i' / gamma_i^3 at the quadrature point.
 * gx[q], dgx[q]: gamma_x, gamma_x' at xi = gauss_xi(q); gy, dgy likewise in y.
 * ----------------------------------------------------------------------------------------------*/
static void element_matrix_q1(const orc_params *p, const zc gx[2], const zc dgx[2], const zc gy[2], const zc dgy[2],
                              zc Ae[4][4])
{
    double h = p->h, w = 0.25 * h * h;
    for (int a = 0; a < 4; a++)
        for (int b = 0; b < 4; b++) Ae[a][b] = 0;
    for (int qx = 0; qx < 2; qx++)
        for (int qy = 0; qy < 2; qy++) {
            double xi = gauss_xi(qx), eta = gauss_xi(qy);
            double Nx[2] = { 1.0 - xi, xi }, Ny[2] = { 1.0 - eta, eta }, dN[2] = { -1.0 / h, 1.0 / h };
            zc D11 = 1.0 / (gx[qx] * gx[qx]), D22 = 1.0 / (gy[qy] * gy[qy]);
            zc b1 = dgx[qx] / (gx[qx] * gx[qx] * gx[qx]), b2 = dgy[qy] / (gy[qy] * gy[qy] * gy[qy]);
            for (int a = 0; a < 4; a++) {
                int ax = a & 1, ay = a >> 1;
                double pa = Nx[ax] * Ny[ay], pax = dN[ax] * Ny[ay], pay = Nx[ax] * dN[ay];
                for (int b = 0; b < 4; b++) {
                    int bx = b & 1, by = b >> 1;
                    double pb = Nx[bx] * Ny[by], pbx = dN[bx] * Ny[by], pby = Nx[bx] * dN[by];
                    Ae[a][b] += w * (D11 * pax * pbx + D22 * pay * pby - (b1 * pbx + b2 * pby) * pa
                                     - p->k * p->k * pa * pb);
                }
            }
        }
}

/* ------------------------------------------------------------------------------------------------
 * P1 element matrix (weak form eq. (weak)):
 *   a(u,v) = int D grad u . grad v - (beta . grad u) v - k^2 u v,
 *   D = diag(gamma_x^-2, gamma_y^-2), beta = (gamma_x'/gamma_x^3, gamma_y'/gamma_y^3),
 * with D, beta frozen at the triangle centroid (BASELINE.json configs[0]; D5).  Bilinear, no
 * conjugation (D6).  Row = test function phi_p, column = trial phi_q:
 *   A_T[p][q] = |T| (D11 dx phi_p dx phi_q + D22 dy phi_p dy phi_q) - beta . grad phi_q * |T|/3
 *               - k^2 |T| (1 + delta_pq) / 12.
 * Cell (i,j) is split on its SW->NE diagonal (D1):
 *   T_lo = {(i,j),(i+1,j),(i+1,j+1)}  centroid (i+2/3, j+1/3)  h*grad: (-1,0) (1,-1) (0,1)
 *   T_up = {(i,j),(i+1,j+1),(i,j+1)}  centroid (i+1/3, j+2/3)  h*grad: (0,-1) (1,0) (-1,1)
 * ----------------------------------------------------------------------------------------------*/
static const int TRI_V[2][3][2] = { { {0, 0}, {1, 0}, {1, 1} }, { {0, 0}, {1, 1}, {0, 1} } };
static const double TRI_G[2][3][2] = { { {-1, 0}, {1, -1}, {0, 1} }, { {0, -1}, {1, 0}, {-1, 1} } };
static const int TRI_C3[2][2] = { {2, 1}, {1, 2} }; /* centroid offset in thirds (x, y) */

static void element_matrix(const orc_params *p, zc gx, zc dgx, zc gy, zc dgy, int tri, zc Ae[3][3])
{
    double h = p->h, area = 0.5 * h * h;
    zc D11 = 1.0 / (gx * gx), D22 = 1.0 / (gy * gy);
    zc b1 = dgx / (gx * gx * gx), b2 = dgy / (gy * gy * gy);
    for (int a = 0; a < 3; a++)
        for (int q = 0; q < 3; q++) {
            double dxa = TRI_G[tri][a][0] / h, dya = TRI_G[tri][a][1] / h;
            double dxq = TRI_G[tri][q][0] / h, dyq = TRI_G[tri][q][1] / h;
            zc stiff = area * (D11 * dxa * dxq + D22 * dya * dyq);
            zc conv = (b1 * dxq + b2 * dyq) * (area / 3.0);
            double mass = p->k * p->k * area * (a == q ? 2.0 : 1.0) / 12.0;
            Ae[a][q] = stiff - conv - mass;
        }
}

/* global free-row slot of neighbour (dx,dy); 7-point pattern of the SW->NE split (D1) */
static int slot_of(int dx, int dy)
{
    if (dx == 0 && dy == 0) return 0;
    if (dx == 1 && dy == 0) return 1;   /* E  */
    if (dx == -1 && dy == 0) return 2;  /* W  */
    if (dx == 0 && dy == 1) return 3;   /* N  */
    if (dx == 0 && dy == -1) return 4;  /* S  */
    if (dx == 1 && dy == 1) return 5;   /* NE */
    if (dx == -1 && dy == -1) return 6; /* SW */
    if (dx == -1 && dy == 1) return 7;  /* NW (Q1 only) */
    if (dx == 1 && dy == -1) return 8;  /* SE (Q1 only) */
    fprintf(stderr, "orc: neighbour (%d,%d) outside the 9-point pattern\n", dx, dy);
    abort();
}

/* ------------------------------------------------------------------------------------------------
 * Decomposition (D8, D10).  Cells 0..N-1 of each axis are cut into P blocks of floor/ceil
 * size, larger blocks first.  Int box = block extended by delta cells on every side not on dOmega;
 * full box = int box extended by kappa cells on the same sides.  Local free nodes = nodes strictly
 * inside the full box (Dirichlet on dOmega_j, RAS-PML-Drch; D9).
 * Owner of node i: the block p with s_p <= i < s_{p+1}.
 * ----------------------------------------------------------------------------------------------*/
orc_ctx *orc_create(const orc_params *p, char *err, int errlen)
{
    orc_ctx *c = calloc(1, sizeof(orc_ctx));
    c->p = *p;
    c->N[0] = p->nix + 2 * p->ng;
    c->N[1] = p->niy + 2 * p->ng;
    c->nf[0] = c->N[0] - 1;
    c->nf[1] = c->N[1] - 1;
    c->nfree = (int64_t)c->nf[0] * c->nf[1];
    int P[2] = { p->px, p->py };
    c->nsub = P[0] * P[1];
    int w = p->novlp + p->npml;
    if (P[0] < 1 || P[1] < 1 || c->N[0] < 2 || c->N[1] < 2) {
        snprintf(err, errlen, "empty grid or subdomain count");
        free(c); return NULL;
    }
    if (p->elem != 0 && p->elem != 1) { snprintf(err, errlen, "elem must be 0 (P1) or 1 (Q1)"); free(c); return NULL; }
    if (p->frame == 1 && (p->elem != 1 || p->ng != 0)) {
        snprintf(err, errlen, "the paper frame is Q1 with ng = 0"); free(c); return NULL;
    }
    c->ns = p->elem == 1 ? 9 : 7;
    for (int ax = 0; ax < 2; ax++) {
        if (p->frame == 1) {     /* Omega_int = (kappa_g, L - kappa_g) in cell units */
            c->lo_u[ax] = p->kappa / p->h;
            c->hi_u[ax] = (double)c->N[ax] - p->kappa / p->h;
        } else {                 /* Omega_int = nodes [ng, ng + ni] */
            c->lo_u[ax] = (double)p->ng;
            c->hi_u[ax] = (double)(p->ng + (ax == 0 ? p->nix : p->niy));
        }
    }
    c->split[0] = malloc(sizeof(int) * (P[0] + 1));
    c->split[1] = malloc(sizeof(int) * (P[1] + 1));
    for (int ax = 0; ax < 2; ax++) {
        int q = c->N[ax] / P[ax], r = c->N[ax] % P[ax];
        c->split[ax][0] = 0;
        for (int b = 0; b < P[ax]; b++) c->split[ax][b + 1] = c->split[ax][b] + q + (b < r ? 1 : 0);
        for (int b = 0; b < P[ax]; b++) {
            int sz = c->split[ax][b + 1] - c->split[ax][b];
            if ((P[ax] > 1 && sz < w) || sz < 2 || (p->pou == 1 && P[ax] > 1 && sz < 2 * p->novlp)) {
                snprintf(err, errlen, "block %d on axis %d has %d cells (< delta+kappa = %d, < 2, or < 2 delta for "
                         "ramps)", b, ax, sz, w);
                free(c->split[0]); free(c->split[1]); free(c); return NULL;
            }
        }
    }
    c->sub = calloc(c->nsub, sizeof(orc_sub));
    for (int jy = 0; jy < P[1]; jy++)
        for (int jx = 0; jx < P[0]; jx++) {
            orc_sub *s = &c->sub[jx + P[0] * jy];
            int jj[2] = { jx, jy };
            for (int ax = 0; ax < 2; ax++) {
                int b = jj[ax];
                s->own_lo[ax] = c->split[ax][b];
                s->own_hi[ax] = c->split[ax][b + 1];
                s->has_lo[ax] = b > 0;
                s->has_hi[ax] = b < P[ax] - 1;
                s->int_lo[ax] = s->own_lo[ax] - (s->has_lo[ax] ? p->novlp : 0);
                s->int_hi[ax] = s->own_hi[ax] + (s->has_hi[ax] ? p->novlp : 0);
                s->full_lo[ax] = s->int_lo[ax] - (s->has_lo[ax] ? p->npml : 0);
                s->full_hi[ax] = s->int_hi[ax] + (s->has_hi[ax] ? p->npml : 0);
                /* local free nodes: strictly inside the full box (Dirichlet on dOmega_j), plus the
                   nodes on faces that carry the impedance condition (RAS-PML-Imp) */
                int imp = p->local_bc == 1;
                s->node0[ax] = s->full_lo[ax] + ((imp && s->has_lo[ax]) ? 0 : 1);
                int last = s->full_hi[ax] - ((imp && s->has_hi[ax]) ? 0 : 1);
                s->m[ax] = last - s->node0[ax] + 1;
                /* every local free node must be a global free node: an impedance face on dOmega (a block
                   narrower than delta + kappa + 1 next to the boundary) would put node 0 or N into Omega_j */
                if (s->full_lo[ax] < 0 || s->full_hi[ax] > c->N[ax] || s->node0[ax] < 1 || last > c->N[ax] - 1) {
                    snprintf(err, errlen, "full box of subdomain (%d,%d) leaves Omega (or puts an impedance face on dOmega)", jx, jy);
                    free(c->sub); free(c->split[0]); free(c->split[1]); free(c); return NULL;
                }
            }
        }
    return c;
}

void orc_release(orc_ctx *c);

void orc_destroy(orc_ctx *c)
{
    if (!c) return;
    orc_release(c);
    free(c->sub);
    free(c->split[0]);
    free(c->split[1]);
    free(c->A7);
    free(c);
}

/* dims: N[0], N[1], nf[0], nf[1], nsub, px, py */
void orc_dims(const orc_ctx *c, int *out)
{
    out[0] = c->N[0]; out[1] = c->N[1]; out[2] = c->nf[0]; out[3] = c->nf[1];
    out[4] = c->nsub; out[5] = c->p.px; out[6] = c->p.py;
}

/* subdomain j: own_lo/hi, int_lo/hi, full_lo/hi, has_lo/hi, m, node0 per axis -> 20 ints (x then y) */
void orc_subdomain(const orc_ctx *c, int j, int *out)
{
    const orc_sub *s = &c->sub[j];
    for (int ax = 0; ax < 2; ax++) {
        int *o = out + 10 * ax;
        o[0] = s->own_lo[ax]; o[1] = s->own_hi[ax]; o[2] = s->int_lo[ax]; o[3] = s->int_hi[ax];
        o[4] = s->full_lo[ax]; o[5] = s->full_hi[ax]; o[6] = s->has_lo[ax]; o[7] = s->has_hi[ax];
        o[8] = s->m[ax]; o[9] = s->node0[ax];
    }
}

/* ------------------------------------------------------------------------------------------------
 * Global assembly (eq. (weak) on V_h subset H^1_0(Omega)): element loop over all
 * N x N cells with the global coefficients; rows/columns of Dirichlet nodes dropped.
 * Free node (i,j), 1 <= i,j <= N-1, has index (i-1) + nf (j-1).
 * ----------------------------------------------------------------------------------------------*/
static void scatter_global(orc_ctx *c, int ci, int cj, int nv, const int (*V)[2], const zc *Ae /* nv x nv */)
{
    for (int a = 0; a < nv; a++) {
        int pi = ci + V[a][0], pj = cj + V[a][1];
        if (pi < 1 || pi > c->nf[0] || pj < 1 || pj > c->nf[1]) continue;
        int64_t row = (pi - 1) + (int64_t)c->nf[0] * (pj - 1);
        for (int q = 0; q < nv; q++) {
            int qi = ci + V[q][0], qj = cj + V[q][1];
            if (qi < 1 || qi > c->nf[0] || qj < 1 || qj > c->nf[1]) continue;
            c->A7[row * c->ns + slot_of(qi - pi, qj - pj)] += Ae[a * nv + q];
        }
    }
}

static const int Q1_V[4][2] = { {0, 0}, {1, 0}, {0, 1}, {1, 1} };   /* a = ax + 2 ay */

static void assemble_global(orc_ctx *c)
{
    if (c->A7) return;
    c->A7 = calloc((size_t)c->nfree * c->ns, sizeof(zc));
    for (int cj = 0; cj < c->N[1]; cj++)
        for (int ci = 0; ci < c->N[0]; ci++) {
            if (c->p.elem == 1) {
                zc gx[2], dgx[2], gy[2], dgy[2], Ae[4][4];
                for (int q = 0; q < 2; q++) {
                    gamma_global_q(c, 0, ci, gauss_xi(q), &gx[q], &dgx[q]);
                    gamma_global_q(c, 1, cj, gauss_xi(q), &gy[q], &dgy[q]);
                }
                element_matrix_q1(&c->p, gx, dgx, gy, dgy, Ae);
                scatter_global(c, ci, cj, 4, Q1_V, &Ae[0][0]);
                continue;
            }
            for (int tri = 0; tri < 2; tri++) {
                zc gx, dgx, gy, dgy, Ae[3][3];
                gamma_global(c, 0, 3L * ci + TRI_C3[tri][0], &gx, &dgx);
                gamma_global(c, 1, 3L * cj + TRI_C3[tri][1], &gy, &dgy);
                element_matrix(&c->p, gx, dgx, gy, dgy, tri, Ae);
                scatter_global(c, ci, cj, 3, TRI_V[tri], &Ae[0][0]);
            }
        }
}

/* ns slots per free row: 0 centre, 1 E, 2 W, 3 N, 4 S, 5 NE, 6 SW [, 7 NW, 8 SE for Q1] (row-major [nfree][ns]) */
void orc_global_stencil(orc_ctx *c, zc *out)
{
    assemble_global(c);
    memcpy(out, c->A7, sizeof(zc) * c->ns * (size_t)c->nfree);
}

static const int SDX[9] = { 0, 1, -1, 0, 0, 1, -1, -1, 1 }, SDY[9] = { 0, 0, 0, 1, -1, 1, -1, 1, -1 };

static zc matvec_row(const orc_ctx *c, const zc *x, int64_t row)
{
    int nfx = c->nf[0], nfy = c->nf[1];
    int i = (int)(row % nfx) + 1, j = (int)(row / nfx) + 1;
    zc acc = 0;
    for (int s = 0; s < c->ns; s++) {
        int qi = i + SDX[s], qj = j + SDY[s];
        if (qi < 1 || qi > nfx || qj < 1 || qj > nfy) continue;
        acc += c->A7[row * c->ns + s] * x[(qi - 1) + (int64_t)nfx * (qj - 1)];
    }
    return acc;
}

/* y = A x (S: matvec; eq. (weak)) */
void orc_matvec(orc_ctx *c, const zc *x, zc *y)
{
    assemble_global(c);
#pragma omp parallel for schedule(static)
    for (int64_t row = 0; row < c->nfree; row++) y[row] = matvec_row(c, x, row);
}

/* y[rows[r]] = (A x)[rows[r]] for a sample of rows (full-size parity on sampled outputs) */
void orc_matvec_rows(orc_ctx *c, const zc *x, const int64_t *rows, int nrows, zc *y)
{
    assemble_global(c);
    for (int r = 0; r < nrows; r++) y[r] = matvec_row(c, x, rows[r]);
}

/* ------------------------------------------------------------------------------------------------
 * Right-hand side (D14): f(x) = sum_s a_s (2 pi sigma^2)^-1 exp(-|x - x_s|^2 / (2 sigma^2)), nodal
 * interpolation at the free nodes, b = M_ff f_I with the consistent P1 (or Q1) mass matrix
 * (int_T phi_p phi_q = |T| (1 + delta_pq) / 12), assembled element by element.
 * Node (i,j) sits at ((i - ng) h, (j - ng) h): Omega_int's corner is the origin in the BJ frame, Omega's
 * corner in the paper frame (ng = 0; the smoothed delta of P:217-218 is one unit-mass Gaussian).
 * ----------------------------------------------------------------------------------------------*/
void orc_rhs(orc_ctx *c, int nsrc, const double *xy, const zc *amp, double sigma, zc *b)
{
    int nfx = c->nf[0], nfy = c->nf[1];
    double h = c->p.h, area = 0.5 * h * h;
    zc *f = calloc((size_t)c->nfree, sizeof(zc));
#pragma omp parallel for schedule(static)
    for (int j = 1; j <= nfy; j++)
        for (int i = 1; i <= nfx; i++) {
            double x = (i - c->p.ng) * h, y = (j - c->p.ng) * h;
            zc acc = 0;
            for (int s = 0; s < nsrc; s++) {
                double dx = x - xy[2 * s], dy = y - xy[2 * s + 1];
                acc += amp[s] * exp(-(dx * dx + dy * dy) / (2.0 * sigma * sigma)) / (2.0 * M_PI * sigma * sigma);
            }
            f[(i - 1) + (int64_t)nfx * (j - 1)] = acc;
        }
    memset(b, 0, sizeof(zc) * (size_t)c->nfree);
    for (int cj = 0; cj < c->N[1]; cj++)
        for (int ci = 0; ci < c->N[0]; ci++) {
            /* element mass: P1 |T| (1 + delta_pq) / 12 per triangle; Q1 the tensor product of the 1D P1 mass
               (h/6)[[2,1],[1,2]] (exact, = the 2 x 2 Gauss rule) */
            int nt = c->p.elem == 1 ? 1 : 2, nv = c->p.elem == 1 ? 4 : 3;
            for (int tri = 0; tri < nt; tri++)
                for (int a = 0; a < nv; a++) {
                    const int *va = c->p.elem == 1 ? Q1_V[a] : TRI_V[tri][a];
                    int pi = ci + va[0], pj = cj + va[1];
                    if (pi < 1 || pi > nfx || pj < 1 || pj > nfy) continue;
                    for (int q = 0; q < nv; q++) {
                        const int *vq = c->p.elem == 1 ? Q1_V[q] : TRI_V[tri][q];
                        int qi = ci + vq[0], qj = cj + vq[1];
                        if (qi < 1 || qi > nfx || qj < 1 || qj > nfy) continue;
                        double mq = c->p.elem == 1
                            ? (h / 6.0) * (va[0] == vq[0] ? 2.0 : 1.0) * (h / 6.0) * (va[1] == vq[1] ? 2.0 : 1.0)
                            : area * (a == q ? 2.0 : 1.0) / 12.0;
                        b[(pi - 1) + (int64_t)nfx * (pj - 1)] += mq * f[(qi - 1) + (int64_t)nfx * (qj - 1)];
                    }
                }
        }
    free(f);
}

/* ------------------------------------------------------------------------------------------------
 * Local operator A_j (a_j = a restricted to H^1_0(Omega_j) with the local scaling g_j),
 * assembled element by element over the cells of the full box into band storage.
 * The local free nodes are the global nodes node0 .. node0 + m - 1 per axis (node0 = full_lo + 1 for a
 * Dirichlet face; = full_lo when the face carries the impedance condition of P:185-195); global node
 * (gi, gj) has local index (gi - node0x) + mx (gj - node0y); half-bandwidth p = mx + 1 (D1).
 * band[r*(2p+1) + (col - r + p)].
 * RAS-PML-Imp (eq. impedance): on every face of Omega_j that is not on dOmega the condition
 * d_nu u - i k u = 0 is imposed as a natural boundary condition, i.e. a_j gains -i k int_face u v; with P1
 * on an edge of length h: -i k (h/6) [[2,1],[1,2]] (no PML metric).
 * ----------------------------------------------------------------------------------------------*/
static int local_index(const orc_sub *s, int gi, int gj, int64_t *idx)
{
    int lx = gi - s->node0[0], ly = gj - s->node0[1];
    if (lx < 0 || lx >= s->m[0] || ly < 0 || ly >= s->m[1]) return 0;
    *idx = lx + (int64_t)s->m[0] * ly;
    return 1;
}

static void assemble_local(const orc_ctx *c, int j, zc *band)
{
    const orc_sub *s = &c->sub[j];
    int mx = s->m[0], my = s->m[1], p = mx + 1, bw = 2 * p + 1;
    int64_t n = (int64_t)mx * my;
    memset(band, 0, sizeof(zc) * (size_t)n * bw);
    for (int cj = s->full_lo[1]; cj < s->full_hi[1]; cj++)
        for (int ci = s->full_lo[0]; ci < s->full_hi[0]; ci++) {
            if (c->p.elem == 1) {
                zc gx[2], dgx[2], gy[2], dgy[2], Ae[4][4];
                for (int q = 0; q < 2; q++) {
                    gamma_local_q(c, s, 0, ci, gauss_xi(q), &gx[q], &dgx[q]);
                    gamma_local_q(c, s, 1, cj, gauss_xi(q), &gy[q], &dgy[q]);
                }
                element_matrix_q1(&c->p, gx, dgx, gy, dgy, Ae);
                for (int a = 0; a < 4; a++) {
                    int64_t r, col;
                    if (!local_index(s, ci + Q1_V[a][0], cj + Q1_V[a][1], &r)) continue;
                    for (int q = 0; q < 4; q++) {
                        if (!local_index(s, ci + Q1_V[q][0], cj + Q1_V[q][1], &col)) continue;
                        band[r * bw + (col - r + p)] += Ae[a][q];
                    }
                }
                continue;
            }
            for (int tri = 0; tri < 2; tri++) {
                zc gx, dgx, gy, dgy, Ae[3][3];
                gamma_local(c, s, 0, 3L * ci + TRI_C3[tri][0], &gx, &dgx);
                gamma_local(c, s, 1, 3L * cj + TRI_C3[tri][1], &gy, &dgy);
                element_matrix(&c->p, gx, dgx, gy, dgy, tri, Ae);
                for (int a = 0; a < 3; a++) {
                    int64_t r, col;
                    if (!local_index(s, ci + TRI_V[tri][a][0], cj + TRI_V[tri][a][1], &r)) continue;
                    for (int q = 0; q < 3; q++) {
                        if (!local_index(s, ci + TRI_V[tri][q][0], cj + TRI_V[tri][q][1], &col)) continue;
                        band[r * bw + (col - r + p)] += Ae[a][q];
                    }
                }
            }
        }
    if (c->p.local_bc != 1) return;
    /* impedance faces: x = full_lo / full_hi (edges along y) and y = full_lo / full_hi (edges along x) */
    for (int ax = 0; ax < 2; ax++)
        for (int side = 0; side < 2; side++) {
            if (!(side ? s->has_hi[ax] : s->has_lo[ax])) continue;
            int f = side ? s->full_hi[ax] : s->full_lo[ax];
            int o = 1 - ax;
            for (int e = s->full_lo[o]; e < s->full_hi[o]; e++) {   /* edge between nodes e and e+1 */
                int pts[2][2];
                for (int q = 0; q < 2; q++) {
                    pts[q][ax] = f;
                    pts[q][o] = e + q;
                }
                for (int a = 0; a < 2; a++)
                    for (int q = 0; q < 2; q++) {
                        int64_t r, col;
                        if (!local_index(s, pts[a][0], pts[a][1], &r)) continue;
                        if (!local_index(s, pts[q][0], pts[q][1], &col)) continue;
                        band[r * bw + (col - r + p)] += -I * c->p.k * (c->p.h / 6.0) * (a == q ? 2.0 : 1.0);
                    }
            }
        }
}

/* export the local band (n x (2p+1)) for pins; returns n */
int64_t orc_local_band(const orc_ctx *c, int j, zc *band)
{
    assemble_local(c, j, band);
    return (int64_t)c->sub[j].m[0] * c->sub[j].m[1];
}

/* ------------------------------------------------------------------------------------------------
 * Naive banded LU without pivoting (D12; exact local solves), in place on band storage.
 *   for kk: u = a[kk][kk]; if u == 0 -> zero pivot at row kk
 *           for i in kk+1..kk+p: l = a[i][kk]/u; a[i][kk] = l; a[i][kk+1..kk+p] -= l a[kk][kk+1..kk+p]
 * Returns -1 on success, else the zero-pivot row.
 * ----------------------------------------------------------------------------------------------*/
int64_t orc_band_lu(int64_t n, int p, zc *a)
{
    int bw = 2 * p + 1;
#define AB(r, col) a[(r) * bw + ((col) - (r) + p)]
    for (int64_t kk = 0; kk < n; kk++) {
        zc u = AB(kk, kk);
        if (u == 0) return kk;
        int64_t iend = kk + p < n - 1 ? kk + p : n - 1;
        for (int64_t i = kk + 1; i <= iend; i++) {
            zc l = AB(i, kk) / u;
            AB(i, kk) = l;
            if (l == 0) continue;
            for (int64_t col = kk + 1; col <= iend; col++) AB(i, col) -= l * AB(kk, col);
        }
    }
    return -1;
}

/* forward (unit L) then backward (U) substitution, x in/out */
void orc_band_solve(int64_t n, int p, const zc *a, zc *x)
{
    int bw = 2 * p + 1;
    for (int64_t i = 0; i < n; i++) {
        zc acc = x[i];
        for (int64_t col = (i - p > 0 ? i - p : 0); col < i; col++) acc -= AB(i, col) * x[col];
        x[i] = acc;
    }
    for (int64_t i = n - 1; i >= 0; i--) {
        zc acc = x[i];
        int64_t cend = i + p < n - 1 ? i + p : n - 1;
        for (int64_t col = i + 1; col <= cend; col++) acc -= AB(i, col) * x[col];
        x[i] = acc / AB(i, i);
    }
#undef AB
}

/* Factor the listed subdomains (list == NULL -> all).  Returns 0, or -(1 + j) with *zero_row set on
 * a zero pivot in subdomain j. */
int orc_factor(orc_ctx *c, const int *list, int nlist, int64_t *zero_row)
{
    int cnt = list ? nlist : c->nsub;
    int bad = -1;
    int64_t badrow = -1;
#pragma omp parallel for schedule(dynamic, 1)
    for (int t = 0; t < cnt; t++) {
        int j = list ? list[t] : t;
        orc_sub *s = &c->sub[j];
        if (s->factored) continue;
        int mx = s->m[0], p = mx + 1;
        int64_t n = (int64_t)mx * s->m[1];
        zc *band = malloc(sizeof(zc) * (size_t)n * (2 * p + 1));
        assemble_local(c, j, band);
        int64_t zr = orc_band_lu(n, p, band);
        if (zr >= 0) {
#pragma omp critical
            { if (bad < 0) { bad = j; badrow = zr; } }
            free(band);
            continue;
        }
        s->band = band;
        s->factored = 1;
    }
    if (bad >= 0) { if (zero_row) *zero_row = badrow; return -(1 + bad); }
    return 0;
}

/* drop factors (bench / memory control) */
void orc_release(orc_ctx *c)
{
    for (int j = 0; j < c->nsub; j++) {
        if (!c->sub[j].shared) free(c->sub[j].band);
        c->sub[j].band = NULL; c->sub[j].factored = 0; c->sub[j].shared = 0;
    }
    for (int q = 0; q < c->ncls; q++) { free(c->cls[q].band); free(c->cls[q].raw); }
    free(c->cls);
    c->cls = NULL;
    c->ncls = 0;
}

/* ------------------------------------------------------------------------------------------------
 * Dedup mode (SURVEY 8(d) "memory fallback"; exact, oracle only).  Identical matrices have identical
 * factors, so instead of storing one band LU per subdomain (86 GB at c3) the oracle
 *   1. assembles every A_j (assemble_local, unchanged) and hashes its bytes (FNV-1a over 64-bit words,
 *      together with m_x, m_y);
 *   2. groups equal (hash, m_x, m_y) into classes, the lowest subdomain index being the representative;
 *   3. factors each representative once (orc_band_lu, unchanged);
 *   4. ASSERTS that every member's assembled band is bitwise equal to its representative's (memcmp): a
 *      hash collision or a non-bitwise-equal pair fails loudly instead of sharing the wrong factors.
 * The apply is unchanged (orc_band_solve per subdomain, on the shared factors).
 * Returns 0 and *ncls; -(1 + j) with *zero_row on a zero pivot of representative j; or -(1 + nsub + j)
 * when member j differs from its class representative.  Must be called on an unfactored context.
 * ----------------------------------------------------------------------------------------------*/
static uint64_t band_hash(const zc *band, size_t nz, int mx, int my)
{
    const uint64_t *w = (const uint64_t *)band;
    uint64_t h = 1469598103934665603ULL;
    h = (h ^ (uint64_t)mx) * 1099511628211ULL;
    h = (h ^ (uint64_t)my) * 1099511628211ULL;
    for (size_t i = 0; i < 2 * nz; i++) h = (h ^ w[i]) * 1099511628211ULL;
    return h;
}

int orc_factor_dedup(orc_ctx *c, int64_t *zero_row, int *ncls_out)
{
    int ns = c->nsub;
    uint64_t *hash = malloc(sizeof(uint64_t) * ns);
    int *cls_of = malloc(sizeof(int) * ns);
    orc_release(c);
    /* 1. hash every assembled A_j */
#pragma omp parallel
    {
        zc *buf = NULL;
        size_t cap = 0;
#pragma omp for schedule(dynamic, 1)
        for (int j = 0; j < ns; j++) {
            orc_sub *s = &c->sub[j];
            int mx = s->m[0], my = s->m[1];
            size_t nz = (size_t)mx * my * (2 * (mx + 1) + 1);
            if (nz > cap) { free(buf); buf = malloc(sizeof(zc) * nz); cap = nz; }
            assemble_local(c, j, buf);
            hash[j] = band_hash(buf, nz, mx, my);
        }
        free(buf);
    }
    /* 2. classes in subdomain order (representative = first member) */
    c->cls = calloc(ns, sizeof(orc_class));
    c->ncls = 0;
    for (int j = 0; j < ns; j++) {
        int q;
        for (q = 0; q < c->ncls; q++)
            if (c->cls[q].hash == hash[j] && c->cls[q].mx == c->sub[j].m[0] && c->cls[q].my == c->sub[j].m[1]) break;
        if (q == c->ncls) {
            c->cls[q].hash = hash[j]; c->cls[q].mx = c->sub[j].m[0]; c->cls[q].my = c->sub[j].m[1];
            c->cls[q].rep = j;
            c->ncls++;
        }
        c->cls[q].count++;
        cls_of[j] = q;
    }
    /* 3. factor each representative once */
    int bad = -1;
    int64_t badrow = -1;
#pragma omp parallel for schedule(dynamic, 1)
    for (int q = 0; q < c->ncls; q++) {
        orc_class *k = &c->cls[q];
        int p = k->mx + 1;
        int64_t n = (int64_t)k->mx * k->my;
        size_t nz = (size_t)n * (2 * p + 1);
        k->raw = malloc(sizeof(zc) * nz);
        k->band = malloc(sizeof(zc) * nz);
        assemble_local(c, k->rep, k->raw);
        memcpy(k->band, k->raw, sizeof(zc) * nz);
        int64_t zr = orc_band_lu(n, p, k->band);
        if (zr >= 0) {
#pragma omp critical
            { if (bad < 0 || k->rep < bad) { bad = k->rep; badrow = zr; } }
        }
    }
    /* 4. every member must equal its representative bitwise */
    int differ = -1;
    if (bad < 0) {
#pragma omp parallel
        {
            zc *buf = NULL;
            size_t cap = 0;
#pragma omp for schedule(dynamic, 1)
            for (int j = 0; j < ns; j++) {
                orc_class *k = &c->cls[cls_of[j]];
                if (k->rep == j) continue;
                size_t nz = (size_t)k->mx * k->my * (2 * (k->mx + 1) + 1);
                if (nz > cap) { free(buf); buf = malloc(sizeof(zc) * nz); cap = nz; }
                assemble_local(c, j, buf);
                if (memcmp(buf, k->raw, sizeof(zc) * nz) != 0) {
#pragma omp critical
                    { if (differ < 0 || j < differ) differ = j; }
                }
            }
            free(buf);
        }
    }
    for (int q = 0; q < c->ncls; q++) { free(c->cls[q].raw); c->cls[q].raw = NULL; }
    if (bad < 0 && differ < 0)
        for (int j = 0; j < ns; j++) {
            c->sub[j].band = c->cls[cls_of[j]].band;
            c->sub[j].shared = 1;
            c->sub[j].factored = 1;
        }
    free(hash);
    free(cls_of);
    if (ncls_out) *ncls_out = c->ncls;
    if (bad >= 0) { if (zero_row) *zero_row = badrow; orc_release(c); return -(1 + bad); }
    if (differ >= 0) { orc_release(c); return -(1 + ns + differ); }
    return 0;
}

/* class of subdomain j in dedup mode (-1 if not in dedup mode): out[0] = class, out[1] = representative,
 * out[2] = class size */
void orc_dedup_class(const orc_ctx *c, int j, int *out)
{
    out[0] = out[1] = out[2] = -1;
    if (!c->cls || !c->sub[j].shared) return;
    for (int q = 0; q < c->ncls; q++)
        if (c->cls[q].band == c->sub[j].band) { out[0] = q; out[1] = c->cls[q].rep; out[2] = c->cls[q].count; return; }
}

/* ------------------------------------------------------------------------------------------------
 * RAS-PML preconditioner: z = sum_j R~_j^T A_j^-1 R_j v, with
 *   R_j    = restriction to all local free nodes of Omega_j (D11),
 *   R~_j^T = extension by the 0/1 owner indicator chi_j = 1 on block j (D10).
 * Only the listed subdomains are applied (list == NULL -> all); z is written at their owned nodes.
 * Returns 0, or -1 if a listed subdomain is not factored.
 * ----------------------------------------------------------------------------------------------*/
/* ------------------------------------------------------------------------------------------------
 * Partition of unity chi_j.  pou = 0: the owner indicator (D10).  pou = 1: the paper's
 * experiments, "tensor products of the 1D PoU functions which vary linearly across the overlap
 * regions": along an axis, block b = cells [s_b, s_{b+1}) with int box [s_b - delta, s_{b+1} + delta]
 * on sides with a neighbour; chi rises linearly from 0 at s_b - delta to 1 at s_b + delta, falls from 1 at
 * s_{b+1} - delta to 0 at s_{b+1} + delta, and is 1 up to dOmega on sides without a neighbour.  The two
 * ramps of an overlap of width 2 delta sum to 1.  Evaluated at node x (integer).
 * ----------------------------------------------------------------------------------------------*/
double orc_chi1(const orc_ctx *c, int ax, int b, int x)
{
    int P = ax ? c->p.py : c->p.px, d = c->p.novlp;
    int s0 = c->split[ax][b], s1 = c->split[ax][b + 1];
    int lo = b > 0, hi = b < P - 1;
    if (c->p.pou != 1 || d == 0) return (x >= s0 && x < s1) ? 1.0 : 0.0;   /* owner indicator */
    if (lo && x <= s0 - d) return 0.0;
    if (hi && x >= s1 + d) return 0.0;
    if (lo && x < s0 + d) return (double)(x - (s0 - d)) / (2.0 * d);
    if (hi && x > s1 - d) return (double)(s1 + d - x) / (2.0 * d);
    return 1.0;
}

int orc_apply(orc_ctx *c, const zc *v, zc *z, const int *list, int nlist)
{
    int cnt = list ? nlist : c->nsub;
    int nfx = c->nf[0];
    int missing = 0;
    if (c->p.pou == 1) {
        /* z += sum_j chi_j R_j^T A_j^-1 R_j v: local solves in parallel, accumulation in subdomain order */
        zc **sol = calloc(cnt, sizeof(zc *));
#pragma omp parallel for schedule(dynamic, 1)
        for (int t = 0; t < cnt; t++) {
            int j = list ? list[t] : t;
            orc_sub *s = &c->sub[j];
            if (!s->factored) { missing = 1; continue; }
            int mx = s->m[0], my = s->m[1];
            int64_t n = (int64_t)mx * my;
            zc *x = malloc(sizeof(zc) * (size_t)n);
            for (int ly = 0; ly < my; ly++)
                for (int lx = 0; lx < mx; lx++)
                    x[lx + (int64_t)mx * ly] = v[(s->node0[0] + lx - 1) + (int64_t)nfx * (s->node0[1] + ly - 1)];
            orc_band_solve(n, mx + 1, s->band, x);
            sol[t] = x;
        }
        if (!list) memset(z, 0, sizeof(zc) * (size_t)c->nfree);
        for (int t = 0; t < cnt && !missing; t++) {
            int j = list ? list[t] : t;
            orc_sub *s = &c->sub[j];
            int bx = j % c->p.px, by = j / c->p.px;
            for (int gj = s->int_lo[1]; gj <= s->int_hi[1]; gj++)
                for (int gi = s->int_lo[0]; gi <= s->int_hi[0]; gi++) {
                    if (gi < 1 || gi > c->nf[0] || gj < 1 || gj > c->nf[1]) continue;
                    double w = orc_chi1(c, 0, bx, gi) * orc_chi1(c, 1, by, gj);
                    if (w == 0.0) continue;
                    int64_t r;
                    local_index(s, gi, gj, &r);
                    z[(gi - 1) + (int64_t)nfx * (gj - 1)] += w * sol[t][r];
                }
        }
        for (int t = 0; t < cnt; t++) free(sol[t]);
        free(sol);
        return missing ? -1 : 0;
    }
#pragma omp parallel for schedule(dynamic, 1)
    for (int t = 0; t < cnt; t++) {
        int j = list ? list[t] : t;
        orc_sub *s = &c->sub[j];
        if (!s->factored) { missing = 1; continue; }
        int mx = s->m[0], my = s->m[1];
        int64_t n = (int64_t)mx * my;
        zc *x = malloc(sizeof(zc) * (size_t)n);
        for (int ly = 0; ly < my; ly++)
            for (int lx = 0; lx < mx; lx++) {
                int gi = s->node0[0] + lx, gj = s->node0[1] + ly;
                x[lx + (int64_t)mx * ly] = v[(gi - 1) + (int64_t)nfx * (gj - 1)];
            }
        orc_band_solve(n, mx + 1, s->band, x);
        for (int gj = s->own_lo[1]; gj < s->own_hi[1]; gj++)
            for (int gi = s->own_lo[0]; gi < s->own_hi[0]; gi++) {
                if (gi < 1 || gi > c->nf[0] || gj < 1 || gj > c->nf[1]) continue; /* Dirichlet node */
                int64_t r;
                local_index(s, gi, gj, &r);
                z[(gi - 1) + (int64_t)nfx * (gj - 1)] = x[r];
            }
        free(x);
    }
    return missing ? -1 : 0;
}
