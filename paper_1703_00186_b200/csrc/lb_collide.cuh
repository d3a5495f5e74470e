// lb_collide.cuh — thermal wall repopulation and regularised collide (device).
//
// Included by every translation unit that runs a full site update (lb_kernels.cu,
// lb_tb.cu).  The __constant__ tables are `static`: each TU owns its copy and
// uploads it itself (upload_kwall / upload_ginv in each TU), so the library
// needs no relocatable device code.
#pragma once
#include "lb_device.cuh"

namespace lbd {
// Wall constants K_wall,l for the bottom (0) and top (1) wall; computed on
// the host with the canonical expression tree (G16) and uploaded by lb_init.
static __constant__ double c_kwall[2][Q];

// Thermal wall repopulation (G9 ii): rho = ((f0 + f1) + f2) + ... + f36
// sequentially, then f_l = rho * K_l — the expression tree of DESIGN.md §3.
__device__ __forceinline__ void thermal_wall(double (&f)[Q], int wall) {
  double rho = f[0];
#pragma unroll
  for (int l = 1; l < Q; ++l) rho = dadd(rho, f[l]);
#pragma unroll
  for (int l = 0; l < Q; ++l) f[l] = dmul(rho, c_kwall[wall][l]);
}

// ---- regularised collide (DESIGN.md §3 reading G6)
// Packed block-diagonal inverse of the Gram matrix G_ab = sum_l w_l c^(alpha_a+alpha_b)
// over the 15 monomials c^alpha, |alpha| <= 4 (lb_device.cuh MP/MQ), host-computed.
static __constant__ double c_ginv[NGINV];

LB_HD constexpr double ipow(int c, int p) {
  double r = 1.0;
  for (int i = 0; i < p; ++i) r *= c;
  return r;
}

// f <- f_eq + (1 - omega)(P f - f_eq), P the projection onto span{w_l p(c_l):
// deg p <= 4} (= Hermite orders <= 4, the quadrature being exact to degree 9).
// Evaluated in the monomial basis: both P f and f_eq lie in that space, so the
// result is w_l sum_a gamma_a c_l^alpha_a with gamma = G^-1 M', where
// M'_a = (1 - omega) M_a(f) + omega rho m_p(ux, T) m_q(uy, T): the raw moments
// of f blended with the Maxwellian moments that f_eq reproduces exactly
// (m_k(u, T) = E[(u + sqrt(T) Z)^k], lattice units).
// hook(moments): rho, j = (M_10, M_01), e = M_20 + M_02 and u, T of the
// pre-collision f (monitors and failure detection, lb_tb.cu).
template <class Hook = NoHook>
__device__ __forceinline__ void collide_site_reg(double (&f)[Q], const Relax& r, const Hook& hook = Hook{}) {
  const double omega = r.omega, one_m_omega = r.one_m_omega;
  // 1. column sums T[cx+3][q] = sum_{l: cx_l = cx} cy_l^q f_l
  double T[7][5];
  {
    bool first[7] = {true, true, true, true, true, true, true};
#pragma unroll
    for (int l = 0; l < Q; ++l) {
      const int k = CX(l) + 3;
      const double cy = (double)CY(l);
      if (first[k]) {
        T[k][0] = f[l];
#pragma unroll
        for (int q = 1; q < 5; ++q) T[k][q] = CY(l) == 0 ? 0.0 : dmul(ipow(CY(l), q), f[l]);
        first[k] = false;
      } else {
        T[k][0] = dadd(T[k][0], f[l]);
        if (CY(l) != 0) {
          T[k][1] = dfma(cy, f[l], T[k][1]);
#pragma unroll
          for (int q = 2; q < 5; ++q) T[k][q] = dfma(ipow(CY(l), q), f[l], T[k][q]);
        }
      }
    }
  }
  // 2. raw moments M_a = sum_l cx^p cy^q f_l via the +-cx symmetric sums
  double E[4][5], O[4][5];
#pragma unroll
  for (int c = 1; c <= 3; ++c)
#pragma unroll
    for (int q = 0; q < 5; ++q) {
      E[c][q] = dadd(T[3 + c][q], T[3 - c][q]);
      O[c][q] = dsub(T[3 + c][q], T[3 - c][q]);
    }
  double M[NMOM];
#pragma unroll
  for (int a = 0; a < NMOM; ++a) {
    const int p = MP(a), q = MQ(a);
    if (p % 2 == 0) {
      double s = p == 0 ? dadd(T[3][q], E[1][q]) : E[1][q];
      s = dfma(ipow(2, p), E[2][q], s);
      M[a] = dfma(ipow(3, p), E[3][q], s);
    } else {
      double s = dfma(ipow(2, p), O[2][q], O[1][q]);
      M[a] = dfma(ipow(3, p), O[3][q], s);
    }
  }
  // 3. macroscopic fields (Eq. 2): rho, u, T = (e/rho - |u|^2)/2
  const double rho = M[0];
  const double inv = __drcp_rn(rho);
  const double ux0 = dmul(M[6], inv), uy0 = dmul(M[9], inv);
  const double Tm0 = dmul(0.5, dsub(dmul(dadd(M[1], M[2]), inv), dfma(ux0, ux0, dmul(uy0, uy0))));
  {
    Macro mo;
    mo.rho = rho;
    mo.jx = M[6];
    mo.jy = M[9];
    mo.e = dadd(M[1], M[2]);
    mo.ux = ux0;
    mo.uy = uy0;
    mo.T = Tm0;
    hook(mo);
  }
  // equilibrium arguments with the body-force shift (G7b)
  const double ux = dadd(ux0, r.tgx), uy = dadd(uy0, r.tgy), Tm = dadd(Tm0, r.dT);
  // 4. Maxwellian moments per axis
  double mx[5], my[5];
  {
    const double ux2 = dmul(ux, ux), uy2 = dmul(uy, uy), T3 = dmul(3.0, Tm);
    mx[0] = 1.0; mx[1] = ux; mx[2] = dadd(ux2, Tm); mx[3] = dmul(ux, dadd(ux2, T3));
    mx[4] = dfma(ux2, dfma(6.0, Tm, ux2), dmul(T3, Tm));
    my[0] = 1.0; my[1] = uy; my[2] = dadd(uy2, Tm); my[3] = dmul(uy, dadd(uy2, T3));
    my[4] = dfma(uy2, dfma(6.0, Tm, uy2), dmul(T3, Tm));
  }
  // 5. blended moments
  const double orho = dmul(omega, rho);
  double Mp[NMOM];
#pragma unroll
  for (int a = 0; a < NMOM; ++a) {
    const int p = MP(a), q = MQ(a);
    const double meq = (p == 0 && q == 0) ? 1.0 : (p == 0 ? my[q] : (q == 0 ? mx[p] : dmul(mx[p], my[q])));
    Mp[a] = dfma(orho, meq, dmul(one_m_omega, M[a]));
  }
  // 6. gamma = G^-1 M' block by block
  double gam[5][5];  // gam[p][q]
#pragma unroll
  for (int gb = 0; gb < 4; ++gb) {
    const int first = GBLK_FIRST(gb), n = GBLK_SIZE(gb), off = GBLK_OFF(gb);
#pragma unroll
    for (int i = 0; i < n; ++i) {
      double s = dmul(c_ginv[off + i * n], Mp[first]);
#pragma unroll
      for (int j = 1; j < n; ++j) s = dfma(c_ginv[off + i * n + j], Mp[first + j], s);
      gam[MP(first + i)][MQ(first + i)] = s;
    }
  }
  // 7. U_q(cx) = sum_p gam[p][q] cx^p, by +-cx parity
  double U[7][5];
#pragma unroll
  for (int q = 0; q < 5; ++q) {
    U[3][q] = gam[0][q];
#pragma unroll
    for (int c = 1; c <= 3; ++c) {
      double ue = gam[0][q], uo = 0.0;
      bool has_odd = false;
#pragma unroll
      for (int p = 1; p <= 4 - q; ++p) {
        if (p % 2 == 0) ue = dfma(ipow(c, p), gam[p][q], ue);
        else if (!has_odd) { uo = dmul(ipow(c, p), gam[p][q]); has_odd = true; }
        else uo = dfma(ipow(c, p), gam[p][q], uo);
      }
      U[3 + c][q] = has_odd ? dadd(ue, uo) : ue;
      U[3 - c][q] = has_odd ? dsub(ue, uo) : ue;
    }
  }
  // 8. f_l = w_l sum_q U_q(cx_l) cy_l^q, by +-cy pairs (l, refl(l))
#pragma unroll
  for (int l = 0; l < Q; ++l) {
    if (CY(l) < 0) continue;
    const int k = CX(l) + 3;
    const double w = SHELL_W(shell_of(l));
    if (CY(l) == 0) {
      f[l] = dmul(w, U[k][0]);
    } else {
      const double cy = (double)CY(l), cy2 = (double)(CY(l) * CY(l));
      const double ev = dfma(cy2, dfma(cy2, U[k][4], U[k][2]), U[k][0]);
      const double od = dmul(cy, dfma(cy2, U[k][3], U[k][1]));
      f[l] = dmul(w, dadd(ev, od));
      f[refl(l)] = dmul(w, dsub(ev, od));
    }
  }
}

}  // namespace lbd
