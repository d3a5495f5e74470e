/*
 * lbref — plain, slow, obviously-correct CPU oracle for the D2Q37 thermal
 * Lattice Boltzmann time step of arXiv 1703.00186 (Calore et al., "Performance
 * and Portability of Accelerated Lattice Boltzmann Applications with OpenACC").
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and the
 * cpu_baseline / --impl reference legs of bench.py may load this library.  It
 * shares no code, header, table or constant generator with the CUDA library
 * under paper_1703_00186_b200/ and includes nothing from it.
 *
 * Citations: "P:a-b" = /root/reference/PAPER.md lines a-b; readings G1..G25
 * are listed in DESIGN.md §3 (taken from SURVEY.md §8c).
 *
 * Layout (canonical, "site_i=(ix*NY)+iy", "nxt[NX*NY+site_i]"):
 *   offset(l, ix, iy) = l*NX*NY + ix*NY + iy,  NX = Lx+6, NY = Ly+6,
 *   physical sites ix in [3, 3+Lx), iy in [3, 3+Ly).
 * All floating point is IEEE binary64; the library is built with
 * -O2 -ffp-contract=off (no FMA contraction, no fast-math) (G15).
 */
#ifndef LBREF_H_INCLUDED
#define LBREF_H_INCLUDED
#include <stdint.h>
#ifdef __cplusplus
extern "C" {
#endif

#define LBREF_Q 37
#define LBREF_HALO 3

enum { LBREF_WALL_THERMAL = 0, LBREF_WALL_ADIABATIC = 1, LBREF_PERIODIC = 2 };
enum { LBREF_A = 0, LBREF_B = 1 };

typedef struct lbref lbref;

/* ---- constants and per-site pure functions (for pins) ------------------ */
void   lbref_velocities(int c[LBREF_Q][2]);   /* App. A / G1, G2 label order  */
void   lbref_weights(double w[LBREF_Q]);      /* App. A / G4                  */
double lbref_scale_a(void);                   /* a; T0 = 1/a^2 (G3)           */
double lbref_t0(void);
int    lbref_refl(int l);                     /* label of (cx, -cy)           */
int    lbref_opp(int l);                      /* label of (-cx, -cy)          */
/* Eq. 2: out = {rho, ux, uy, T}; T from D*rho*T = sum |c-u|^2 f */
void   lbref_macro(const double f[LBREF_Q], double out[4]);
/* App. B 4th-order Hermite equilibrium (G5) in lattice units rho, u, T       */
void   lbref_feq(double rho, double ux, double uy, double T, double out[LBREF_Q]);
/* Wall constants K_wall,l(T_wall) with the canonical expression tree (G16)   */
void   lbref_kwall(double t_wall, double K[LBREF_Q]);
/* Eq. 1 collide of one site in place, omega = dt/tau (O7)                   */
void   lbref_collide_site(double f[LBREF_Q], double omega);
/* Hermite projection onto orders <= 4 (reading G6):
 * out_l = w_l sum_{n<=4} (1/n!) a^(n) : H^(n)(xi_l),  a^(n) = sum_l f_l H^(n)(xi_l)  */
void   lbref_project(const double f[LBREF_Q], double out[LBREF_Q]);
/* Regularised collide in place: f <- f_eq + (1 - omega)(P f - f_eq)          */
void   lbref_collide_site_reg(double f[LBREF_Q], double omega);
/* Collide with a body force g (reading G7b: shifted equilibrium,
 * dt = 1, tau = 1/omega): f_eq is evaluated at u + tau g and
 * T + tau (1 - tau) |g|^2 / D.  collision = LBREF_BGK or LBREF_REGULARIZED.  */
void   lbref_collide_site_force(double f[LBREF_Q], double omega, double gx, double gy,
                                int collision);

/* ---- lattice stepper --------------------------------------------------- */
enum { LBREF_BGK = 0, LBREF_REGULARIZED = 1 };
/* Returns NULL on invalid parameters (Lx<3, Ly<6, dt/tau not in (0,2], T<=0) */
lbref* lbref_init(int lx, int ly, double tau, double dt,
                  double t_bottom, double t_top, int bc_y, int collision);
void   lbref_free(lbref*);
/* body force per unit mass (lattice units), default 0 (reading G7b)          */
void   lbref_set_gravity(lbref*, double gx, double gy);
int    lbref_nx(const lbref*);
int    lbref_ny(const lbref*);
double* lbref_buffer(lbref*, int which);       /* canonical [37][NX][NY]     */
/* physical state in/out, layout [37][Lx][Ly] (iy fastest)                   */
void   lbref_set_state(lbref*, const double* phys);
void   lbref_get_state(const lbref*, int which, double* phys);
/* A := f_eq(rho,u,T) on physical sites; macro fields are [Lx][Ly]           */
void   lbref_init_macro(lbref*, const double* rho, const double* ux,
                        const double* uy, const double* T);
void   lbref_pbc(lbref*);        /* O4 on A                                  */
void   lbref_propagate(lbref*);  /* O5 A -> B (raw pull)                     */
void   lbref_bc(lbref*);         /* O6 on B, reading A                       */
void   lbref_collide(lbref*);    /* O7 in place on B                         */
void   lbref_swap(lbref*);       /* O8                                       */
void   lbref_step(lbref*, int nsteps);
/* O9: {sum rho, sum jx, sum jy, sum 0.5|c|^2 f} over physical sites        */
void   lbref_invariants(const lbref*, int which, double out[4]);
int    lbref_threads(void);      /* OpenMP threads the stepper uses          */
void   lbref_set_threads(int n); /* timing only: OpenMP threads (n > 0)      */

#ifdef __cplusplus
}
#endif
#endif
