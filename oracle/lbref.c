/*
 * lbref.c — CPU oracle for the D2Q37 time step of arXiv 1703.00186.
 *
 * TEST INFRASTRUCTURE ONLY (see lbref.h).  Written from PAPER.md and the
 * readings of DESIGN.md §3; follows the algorithm step by step in the paper's
 * order (pbc -> propagate -> bc -> collide) with no blocking,
 * fusion or reordering.  Build: gcc -O2 -ffp-contract=off [-fopenmp].
 * OpenMP (optional) only splits the outer ix loop of propagate / collide;
 * every site's arithmetic is unchanged by it.
 */
#include "lbref.h"
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

#define Q LBREF_Q
#define HX LBREF_HALO
#define HY LBREF_HALO
#define D 2.0 /* space dimensions, Eq. 2 */

/* App. A: scale factor a with T0 = 1/a^2 (reading G3). */
static const double A_SCALE = 1.19697977039307435897239;

/* App. A: weights per velocity shell |c|^2 (reading G4). */
static double shell_weight(int c2)
{
    switch (c2) {
    case 0:  return 0.23315066913235250228650;
    case 1:  return 0.10730609154221900241246;
    case 2:  return 0.05766785988879488203006;
    case 4:  return 0.01420821615845075026469;
    case 5:  return 0.00535304900051377523273;
    case 8:  return 0.00101193759267357547541;
    case 9:  return 0.00024530102775771734547;
    case 10: return 0.00028341425299419821740;
    default: return 0.0;
    }
}

/* Readings G1, G2: the set {c in Z^2 : |c|^2 <= 10}, labelled with cx from
 * +3 down to -3 and cy ascending within each cx.  This reproduces the two
 * offsets printed at P:452-453 (l=0 -> (3,-1), l=1 -> (3,0)). */
void lbref_velocities(int c[Q][2])
{
    int l = 0;
    for (int cx = 3; cx >= -3; --cx)
        for (int cy = -3; cy <= 3; ++cy)
            if (cx * cx + cy * cy <= 10) {
                c[l][0] = cx;
                c[l][1] = cy;
                ++l;
            }
}

void lbref_weights(double w[Q])
{
    int c[Q][2];
    lbref_velocities(c);
    for (int l = 0; l < Q; ++l) w[l] = shell_weight(c[l][0] * c[l][0] + c[l][1] * c[l][1]);
}

double lbref_scale_a(void) { return A_SCALE; }
double lbref_t0(void) { return 1.0 / (A_SCALE * A_SCALE); }

static int find_label(int cx, int cy)
{
    int c[Q][2];
    lbref_velocities(c);
    for (int l = 0; l < Q; ++l)
        if (c[l][0] == cx && c[l][1] == cy) return l;
    return -1;
}

int lbref_refl(int l)
{
    int c[Q][2];
    lbref_velocities(c);
    return find_label(c[l][0], -c[l][1]);
}

int lbref_opp(int l)
{
    int c[Q][2];
    lbref_velocities(c);
    return find_label(-c[l][0], -c[l][1]);
}

/* Eq. 2, written literally:
 *   rho = sum_l f_l,  rho u = sum_l c_l f_l,  D rho T = sum_l |c_l - u|^2 f_l. */
void lbref_macro(const double f[Q], double out[4])
{
    int c[Q][2];
    lbref_velocities(c);
    double rho = 0.0, jx = 0.0, jy = 0.0;
    for (int l = 0; l < Q; ++l) {
        rho += f[l];
        jx += c[l][0] * f[l];
        jy += c[l][1] * f[l];
    }
    double ux = jx / rho, uy = jy / rho;
    double s = 0.0;
    for (int l = 0; l < Q; ++l) {
        double dx = c[l][0] - ux, dy = c[l][1] - uy;
        s += (dx * dx + dy * dy) * f[l];
    }
    out[0] = rho;
    out[1] = ux;
    out[2] = uy;
    out[3] = s / (D * rho);
}

/* App. B (reading G5): 4th-order Hermite expansion of the Maxwellian in the
 * normalised variables xi = a c, uh = a u, theta = a^2 T, t = theta - 1. */
void lbref_feq(double rho, double ux, double uy, double T, double out[Q])
{
    int c[Q][2];
    double w[Q];
    lbref_velocities(c);
    lbref_weights(w);
    const double a = A_SCALE;
    const double uhx = a * ux, uhy = a * uy;
    const double theta = a * a * T;
    const double t = theta - 1.0;
    const double u2 = uhx * uhx + uhy * uhy;
    for (int l = 0; l < Q; ++l) {
        const double xix = a * c[l][0], xiy = a * c[l][1];
        const double cu = xix * uhx + xiy * uhy;
        const double x2 = xix * xix + xiy * xiy;
        const double cu2 = cu * cu;
        const double o1 = cu;
        const double o2 = 0.5 * (cu2 - u2 + t * (x2 - D));
        const double o3 = (cu / 6.0) * (cu2 - 3.0 * u2 + 3.0 * t * (x2 - D - 2.0));
        const double o4 = (1.0 / 24.0) *
            (cu2 * cu2 - 6.0 * cu2 * u2 + 3.0 * u2 * u2
             + 6.0 * t * (cu2 * (x2 - D - 4.0) + u2 * (D + 2.0 - x2))
             + 3.0 * t * t * (x2 * x2 - 2.0 * (D + 2.0) * x2 + D * (D + 2.0)));
        out[l] = w[l] * rho * (1.0 + o1 + o2 + o3 + o4);
    }
}

/* Reading G16 / G25: the canonical expression tree of DESIGN.md §3,
 * evaluated on the host, left-to-right as parenthesised. */
void lbref_kwall(double t_wall, double K[Q])
{
    int c[Q][2];
    double w[Q];
    lbref_velocities(c);
    lbref_weights(w);
    const double a2 = A_SCALE * A_SCALE;
    const double t = a2 * t_wall - 1.0;
    for (int l = 0; l < Q; ++l) {
        const double x2 = a2 * (double)(c[l][0] * c[l][0] + c[l][1] * c[l][1]);
        K[l] = w[l] * ((1.0 + (0.5 * t) * (x2 - 2.0)) + ((0.125 * t) * t) * ((x2 * x2 - 8.0 * x2) + 8.0));
    }
}

/* Eq. 1 collision part: f <- f - (dt/tau)(f - f_eq), with f_eq
 * evaluated from the moments (Eq. 2) of the post-propagate, post-bc f at the
 * site (reading G24). */
void lbref_collide_site(double f[Q], double omega)
{
    double m[4], feq[Q];
    lbref_macro(f, m);
    lbref_feq(m[0], m[1], m[2], m[3], feq);
    for (int l = 0; l < Q; ++l) f[l] = f[l] - omega * (f[l] - feq[l]);
}

/* Tensor Hermite polynomial H^(n)_{i1..in}(xi), n <= 4, in D = 2 (reading G6):
 *   H0 = 1, H1_i = xi_i, H2_ij = xi_i xi_j - d_ij,
 *   H3_ijk = xi_i xi_j xi_k - (xi_i d_jk + xi_j d_ik + xi_k d_ij),
 *   H4_ijkl = xi_i xi_j xi_k xi_l - (xi_i xi_j d_kl + xi_i xi_k d_jl + xi_i xi_l d_jk
 *             + xi_j xi_k d_il + xi_j xi_l d_ik + xi_k xi_l d_ij)
 *             + (d_ij d_kl + d_ik d_jl + d_il d_jk). */
static double kd(int i, int j) { return i == j ? 1.0 : 0.0; }

static double hermite(int n, const int* t, const double* xi)
{
    switch (n) {
    case 0: return 1.0;
    case 1: return xi[t[0]];
    case 2: return xi[t[0]] * xi[t[1]] - kd(t[0], t[1]);
    case 3: {
        const int i = t[0], j = t[1], k = t[2];
        return xi[i] * xi[j] * xi[k] - (xi[i] * kd(j, k) + xi[j] * kd(i, k) + xi[k] * kd(i, j));
    }
    default: {
        const int i = t[0], j = t[1], k = t[2], l = t[3];
        return xi[i] * xi[j] * xi[k] * xi[l]
             - (xi[i] * xi[j] * kd(k, l) + xi[i] * xi[k] * kd(j, l) + xi[i] * xi[l] * kd(j, k)
                + xi[j] * xi[k] * kd(i, l) + xi[j] * xi[l] * kd(i, k) + xi[k] * xi[l] * kd(i, j))
             + (kd(i, j) * kd(k, l) + kd(i, k) * kd(j, l) + kd(i, l) * kd(j, k));
    }
    }
}

/* Hermite projection ("systematic projection onto a basis of
 * Hermite polynomials"; reading G6): a^(n) = sum_l f_l H^(n)(xi_l) for every
 * index tuple, then out_l = w_l sum_{n=0}^{4} (1/n!) sum_tuples a^(n) H^(n)(xi_l),
 * the full tensor contraction over all 2^n index tuples. */
void lbref_project(const double f[Q], double out[Q])
{
    int c[Q][2];
    double w[Q];
    lbref_velocities(c);
    lbref_weights(w);
    double xi[Q][2];
    for (int l = 0; l < Q; ++l) {
        xi[l][0] = A_SCALE * c[l][0];
        xi[l][1] = A_SCALE * c[l][1];
        out[l] = 0.0;
    }
    double fact = 1.0;
    for (int n = 0; n <= 4; ++n) {
        if (n > 0) fact *= n;
        const int ntup = 1 << n;
        for (int m = 0; m < ntup; ++m) {
            int t[4];
            for (int b = 0; b < n; ++b) t[b] = (m >> b) & 1;
            double a = 0.0;
            for (int l = 0; l < Q; ++l) a += f[l] * hermite(n, t, xi[l]);
            for (int l = 0; l < Q; ++l) out[l] += w[l] * (a / fact) * hermite(n, t, xi[l]);
        }
    }
}

/* Regularised collide: relax in the Hermite space of
 * orders <= 4 and drop the rest: f <- f_eq + (1 - omega)(P f - f_eq). */
void lbref_collide_site_reg(double f[Q], double omega)
{
    double m[4], feq[Q], pf[Q];
    lbref_macro(f, m);
    lbref_feq(m[0], m[1], m[2], m[3], feq);
    lbref_project(f, pf);
    for (int l = 0; l < Q; ++l) f[l] = feq[l] + (1.0 - omega) * (pf[l] - feq[l]);
}

/* Body force (reading G7b; NEXT 2): the shifted-equilibrium scheme of the
 * D2Q37 thermal model of the paper's reference [JFM]: with
 * tau = 1/omega, f_eq is evaluated at u + tau g and at
 * T + tau (1 - tau) |g|^2 / D, so that one collision adds exactly rho g to the
 * momentum and rho (u.g + |g|^2/2) to the energy of the site. */
void lbref_collide_site_force(double f[Q], double omega, double gx, double gy, int collision)
{
    const double tau = 1.0 / omega;
    double m[4], feq[Q];
    lbref_macro(f, m);
    const double ux = m[1] + tau * gx, uy = m[2] + tau * gy;
    const double T = m[3] + tau * (1.0 - tau) * (gx * gx + gy * gy) / D;
    lbref_feq(m[0], ux, uy, T, feq);
    if (collision == LBREF_REGULARIZED) {
        double pf[Q];
        lbref_project(f, pf);
        for (int l = 0; l < Q; ++l) f[l] = feq[l] + (1.0 - omega) * (pf[l] - feq[l]);
    } else {
        for (int l = 0; l < Q; ++l) f[l] = f[l] - omega * (f[l] - feq[l]);
    }
}

/* ------------------------------------------------------------------------ */

struct lbref {
    int lx, ly, nx, ny, bc_y, collision;
    double omega, t_bottom, t_top, gx, gy;
    double *a, *b;            /* canonical [Q][NX][NY] */
    int c[Q][2];
    int refl[Q];
    double k_bottom[Q], k_top[Q];
};

#define IDX(s, l, ix, iy) (((size_t)(l) * (s)->nx + (size_t)(ix)) * (s)->ny + (size_t)(iy))

lbref* lbref_init(int lx, int ly, double tau, double dt,
                  double t_bottom, double t_top, int bc_y, int collision)
{
    if (lx < 3 || ly < 3) return NULL;
    if (bc_y != LBREF_PERIODIC && ly < 6) return NULL;
    if (bc_y < 0 || bc_y > 2) return NULL;
    if (collision != LBREF_BGK && collision != LBREF_REGULARIZED) return NULL;
    if (!(tau > 0.0) || !(dt > 0.0)) return NULL;
    double om = dt / tau;
    if (!(om > 0.0 && om <= 2.0)) return NULL;
    if (bc_y == LBREF_WALL_THERMAL && !(t_bottom > 0.0 && t_top > 0.0)) return NULL;
    lbref* s = (lbref*)calloc(1, sizeof(lbref));
    if (!s) return NULL;
    s->lx = lx;
    s->ly = ly;
    s->nx = lx + 2 * HX;
    s->ny = ly + 2 * HY;
    s->bc_y = bc_y;
    s->collision = collision;
    s->omega = om;
    s->t_bottom = t_bottom;
    s->t_top = t_top;
    size_t n = (size_t)Q * s->nx * s->ny;
    s->a = (double*)calloc(n, sizeof(double)); /* zero-filled (G10) */
    s->b = (double*)calloc(n, sizeof(double));
    if (!s->a || !s->b) {
        lbref_free(s);
        return NULL;
    }
    lbref_velocities(s->c);
    for (int l = 0; l < Q; ++l) s->refl[l] = lbref_refl(l);
    lbref_kwall(t_bottom, s->k_bottom);
    lbref_kwall(t_top, s->k_top);
    return s;
}

void lbref_free(lbref* s)
{
    if (!s) return;
    free(s->a);
    free(s->b);
    free(s);
}

void lbref_set_gravity(lbref* s, double gx, double gy)
{
    s->gx = gx;
    s->gy = gy;
}

int lbref_nx(const lbref* s) { return s->nx; }
int lbref_ny(const lbref* s) { return s->ny; }
double* lbref_buffer(lbref* s, int which) { return which == LBREF_B ? s->b : s->a; }

void lbref_set_state(lbref* s, const double* phys)
{
    for (int l = 0; l < Q; ++l)
        for (int x = 0; x < s->lx; ++x)
            for (int y = 0; y < s->ly; ++y)
                s->a[IDX(s, l, x + HX, y + HY)] = phys[((size_t)l * s->lx + x) * s->ly + y];
}

void lbref_get_state(const lbref* s, int which, double* phys)
{
    const double* f = which == LBREF_B ? s->b : s->a;
    for (int l = 0; l < Q; ++l)
        for (int x = 0; x < s->lx; ++x)
            for (int y = 0; y < s->ly; ++y)
                phys[((size_t)l * s->lx + x) * s->ly + y] = f[IDX(s, l, x + HX, y + HY)];
}

void lbref_init_macro(lbref* s, const double* rho, const double* ux,
                      const double* uy, const double* T)
{
    double feq[Q];
    for (int x = 0; x < s->lx; ++x)
        for (int y = 0; y < s->ly; ++y) {
            size_t m = (size_t)x * s->ly + y;
            lbref_feq(rho[m], ux[m], uy[m], T[m], feq);
            for (int l = 0; l < Q; ++l) s->a[IDX(s, l, x + HX, y + HY)] = feq[l];
        }
}

/* O4: periodic-X halo columns, full columns including
 * the y-halo (G12); N=1 is a local wrap (G13).  PERIODIC-Y additionally wraps
 * the y-halo rows (test configuration only). */
void lbref_pbc(lbref* s)
{
    for (int l = 0; l < Q; ++l)
        for (int iy = 0; iy < s->ny; ++iy) {
            for (int ix = 0; ix < HX; ++ix)
                s->a[IDX(s, l, ix, iy)] = s->a[IDX(s, l, ix + s->lx, iy)];
            for (int ix = s->lx + HX; ix < s->lx + 2 * HX; ++ix)
                s->a[IDX(s, l, ix, iy)] = s->a[IDX(s, l, ix - s->lx, iy)];
        }
    if (s->bc_y == LBREF_PERIODIC)
        for (int l = 0; l < Q; ++l)
            for (int ix = 0; ix < s->nx; ++ix) {
                for (int iy = 0; iy < HY; ++iy)
                    s->a[IDX(s, l, ix, iy)] = s->a[IDX(s, l, ix, iy + s->ly)];
                for (int iy = s->ly + HY; iy < s->ly + 2 * HY; ++iy)
                    s->a[IDX(s, l, ix, iy)] = s->a[IDX(s, l, ix, iy - s->ly)];
            }
}

/* O5: pull gather B[l,x] = A[l, x - c_l]. */
void lbref_propagate(lbref* s)
{
    int ix;
#pragma omp parallel for schedule(static)
    for (ix = HX; ix < HX + s->lx; ++ix)
        for (int l = 0; l < Q; ++l)
            for (int iy = HY; iy < HY + s->ly; ++iy)
                s->b[IDX(s, l, ix, iy)] = s->a[IDX(s, l, ix - s->c[l][0], iy - s->c[l][1])];
}

/* O6 (reading G9): walls at y = Hy - 1/2 and
 * y = Hy + Ly - 1/2.  (i) specular mirror of populations whose pull source
 * lies beyond the wall; (ii) WALL_THERMAL: f_l <- rho K_wall,l with rho the
 * sequential sum l = 0..36 (G14). */
static void bc_band(lbref* s, int iy0, int iy1, const double* K)
{
    const int ylo = HY, yhi = HY + s->ly;
    for (int ix = HX; ix < HX + s->lx; ++ix)
        for (int iy = iy0; iy < iy1; ++iy) {
            for (int l = 0; l < Q; ++l) {
                int ys = iy - s->c[l][1];
                int ystar;
                if (ys < ylo)
                    ystar = 2 * ylo - 1 - ys;
                else if (ys >= yhi)
                    ystar = 2 * yhi - 1 - ys;
                else
                    continue;
                s->b[IDX(s, l, ix, iy)] = s->a[IDX(s, s->refl[l], ix - s->c[l][0], ystar)];
            }
            if (s->bc_y == LBREF_WALL_THERMAL) {
                double rho = s->b[IDX(s, 0, ix, iy)];
                for (int l = 1; l < Q; ++l) rho = rho + s->b[IDX(s, l, ix, iy)];
                for (int l = 0; l < Q; ++l) s->b[IDX(s, l, ix, iy)] = rho * K[l];
            }
        }
}

void lbref_bc(lbref* s)
{
    if (s->bc_y == LBREF_PERIODIC) return;
    bc_band(s, HY, HY + 3, s->k_bottom);                 /* bottom wall */
    bc_band(s, HY + s->ly - 3, HY + s->ly, s->k_top);     /* top wall    */
}

/* O7: per site, in place on B. */
void lbref_collide(lbref* s)
{
    int ix;
#pragma omp parallel for schedule(static)
    for (ix = HX; ix < HX + s->lx; ++ix)
        for (int iy = HY; iy < HY + s->ly; ++iy) {
            double f[Q];
            for (int l = 0; l < Q; ++l) f[l] = s->b[IDX(s, l, ix, iy)];
            if (s->gx != 0.0 || s->gy != 0.0)
                lbref_collide_site_force(f, s->omega, s->gx, s->gy, s->collision);
            else if (s->collision == LBREF_REGULARIZED)
                lbref_collide_site_reg(f, s->omega);
            else
                lbref_collide_site(f, s->omega);
            for (int l = 0; l < Q; ++l) s->b[IDX(s, l, ix, iy)] = f[l];
        }
}

void lbref_swap(lbref* s)
{
    double* t = s->a;
    s->a = s->b;
    s->b = t;
}

/* A10: pbc -> propagate -> bc -> collide, then swap (G11). */
void lbref_step(lbref* s, int nsteps)
{
    for (int k = 0; k < nsteps; ++k) {
        lbref_pbc(s);
        lbref_propagate(s);
        lbref_bc(s);
        lbref_collide(s);
        lbref_swap(s);
    }
}

void lbref_invariants(const lbref* s, int which, double out[4])
{
    const double* f = which == LBREF_B ? s->b : s->a;
    double m = 0.0, jx = 0.0, jy = 0.0, e = 0.0;
    for (int l = 0; l < Q; ++l) {
        const double c2 = (double)(s->c[l][0] * s->c[l][0] + s->c[l][1] * s->c[l][1]);
        for (int ix = HX; ix < HX + s->lx; ++ix)
            for (int iy = HY; iy < HY + s->ly; ++iy) {
                const double v = f[IDX(s, l, ix, iy)];
                m += v;
                jx += s->c[l][0] * v;
                jy += s->c[l][1] * v;
                e += 0.5 * c2 * v;
            }
    }
    out[0] = m;
    out[1] = jx;
    out[2] = jy;
    out[3] = e;
}

/* Timing harness only (bench.py cpu_baseline): thread count of the OpenMP
 * loops over ix; the per-site arithmetic does not depend on it. */
void lbref_set_threads(int n)
{
#ifdef _OPENMP
    if (n > 0) omp_set_num_threads(n);
#else
    (void)n;
#endif
}

int lbref_threads(void)
{
#ifdef _OPENMP
    return omp_get_max_threads();
#else
    return 1;
#endif
}
