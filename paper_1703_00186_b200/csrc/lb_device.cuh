// lb_device.cuh — D2Q37 constants and per-site device math for sm_100a.
//
// Product code (shares nothing with oracle/).  The velocity table is the
// label order of DESIGN.md reading G2 (cx from +3 down to -3, cy ascending;
// l=0 -> (3,-1), l=1 -> (3,0)).  Weights and the scale factor a are
// App. A of DESIGN.md (reading G3/G4).  Every per-population quantity is a
// compile-time constant, so with the loops unrolled each one is an immediate
// or constant-bank operand (the paper's CUDA lesson).
#pragma once
#include <cstdint>

namespace lbd {

constexpr int Q = 37;
constexpr int H = 3;

#if defined(__CUDACC__)
#define LB_HD __host__ __device__
#else
#define LB_HD
#endif

// Velocity table c_l = (CX(l), CY(l)), label order G2.
LB_HD constexpr int CX(int l) {
  constexpr int t[Q] = {3, 3, 3, 2, 2, 2, 2, 2, 1, 1, 1, 1, 1, 1, 1, 0, 0, 0, 0,
                        0, 0, 0, -1, -1, -1, -1, -1, -1, -1, -2, -2, -2, -2, -2, -3, -3, -3};
  return t[l];
}
LB_HD constexpr int CY(int l) {
  constexpr int t[Q] = {-1, 0, 1, -2, -1, 0, 1, 2, -3, -2, -1, 0, 1, 2, 3, -3, -2, -1, 0,
                        1, 2, 3, -3, -2, -1, 0, 1, 2, 3, -2, -1, 0, 1, 2, -1, 0, 1};
  return t[l];
}

LB_HD constexpr int c2(int l) { return CX(l) * CX(l) + CY(l) * CY(l); }

// shells |c|^2 in {0,1,2,4,5,8,9,10} -> shell id 0..7
constexpr int NSHELL = 8;
LB_HD constexpr int SHELL_C2(int s) {
  constexpr int t[NSHELL] = {0, 1, 2, 4, 5, 8, 9, 10};
  return t[s];
}
LB_HD constexpr int shell_of(int l) {
  return c2(l) == 0 ? 0 : c2(l) == 1 ? 1 : c2(l) == 2 ? 2 : c2(l) == 4 ? 3
       : c2(l) == 5 ? 4 : c2(l) == 8 ? 5 : c2(l) == 9 ? 6 : 7;
}
LB_HD constexpr int refl(int l) {  // label of (cx, -cy): reverse within a cx group
  int k = 0;
  for (int m = 0; m < Q; ++m)
    if (CX(m) == CX(l) && CY(m) == -CY(l)) k = m;
  return k;
}
LB_HD constexpr int opp(int l) { return Q - 1 - l; }  // label of (-cx, -cy)

// App. A: shell weights and scale a (T0 = 1/a^2).
LB_HD constexpr double SHELL_W(int s) {
  constexpr double t[NSHELL] = {
      0.23315066913235250228650, 0.10730609154221900241246, 0.05766785988879488203006,
      0.01420821615845075026469, 0.00535304900051377523273, 0.00101193759267357547541,
      0.00024530102775771734547, 0.00028341425299419821740};
  return t[s];
}
constexpr double A_SCALE = 1.19697977039307435897239;
constexpr double A2 = A_SCALE * A_SCALE;

// ---- regularised collide: moment index map ---------------------------------
// The 15 monomials cx^p cy^q with p + q <= 4, grouped by the parity of (p, q):
// the Gram matrix G_ab = sum_l w_l c^(alpha_a + alpha_b) is block-diagonal in
// these groups (odd lattice moments vanish by symmetry).
constexpr int NMOM = 15;
LB_HD constexpr int MP(int k) {
  constexpr int t[NMOM] = {0, 2, 0, 4, 2, 0, /*OE*/ 1, 3, 1, /*EO*/ 0, 0, 2, /*OO*/ 1, 3, 1};
  return t[k];
}
LB_HD constexpr int MQ(int k) {
  constexpr int t[NMOM] = {0, 0, 2, 0, 2, 4, /*OE*/ 0, 0, 2, /*EO*/ 1, 3, 1, /*OO*/ 1, 1, 3};
  return t[k];
}
// block [first, first + size) of group g: EE (6), OE (3), EO (3), OO (3)
LB_HD constexpr int GBLK_FIRST(int g) { return g == 0 ? 0 : 3 + 3 * g; }
LB_HD constexpr int GBLK_SIZE(int g) { return g == 0 ? 6 : 3; }
// offset of block g inside the packed inverse (36 + 9 + 9 + 9 = 63 doubles)
LB_HD constexpr int GBLK_OFF(int g) { return g == 0 ? 0 : 36 + 9 * (g - 1); }
constexpr int NGINV = 63;

// ---- compile-time self checks of the table ---------------------------------
constexpr bool table_ok() {
  int sx = 0, sy = 0, s2 = 0;
  for (int l = 0; l < Q; ++l) {
    sx += CX(l);
    sy += CY(l);
    s2 += c2(l);
    if (c2(l) > 10) return false;
    if (CX(opp(l)) != -CX(l) || CY(opp(l)) != -CY(l)) return false;
    if (CX(refl(l)) != CX(l) || CY(refl(l)) != -CY(l)) return false;
    for (int m = 0; m < l; ++m)
      if (CX(m) == CX(l) && CY(m) == CY(l)) return false;
    if (l > 0 && (CX(l) > CX(l - 1) || (CX(l) == CX(l - 1) && CY(l) <= CY(l - 1)))) return false;
  }
  return sx == 0 && sy == 0 && s2 == 216;
}
static_assert(table_ok(), "D2Q37 velocity table");
static_assert(CX(0) == 3 && CY(0) == -1 && CX(1) == 3 && CY(1) == 0, "P:452-453 offsets");
static_assert(CX(18) == 0 && CY(18) == 0, "rest population");

#ifdef __CUDACC__

// ---- collide (Eq. 1 with the App. B equilibrium) ----------------------------
//
// Explicit _rn intrinsics everywhere, so every kernel that inlines this
// function performs the identical operation sequence (split == fused,
// bulk+border == whole, bit for bit) whatever the surrounding code.
//
// Moments (Eq. 2): rho = sum f, j = sum c f, e = sum |c|^2 f, formed from the
// column sums S_k = sum_{cx=k} f and row sums R_k = sum_{cy=k} f.
// T = (e/rho - |u|^2)/D with D = 2 (G8).  Normalised: Ux = a^2 ux (so that
// xi.uh = cx Ux + cy Uy), u2 = a^2 |u|^2, t = a^2 T - 1.
// Equilibrium per shell (x2 = a^2 |c|^2) as a quartic in cu = xi.uh:
//   P(cu) = A0 + A1 cu + A2 cu^2 + cu^3/6 + cu^4/24,
//   A1 = 1 - u2/2 + t (x2-4)/2,   A2 = 1/2 - u2/4 + t (x2-6)/4,
//   A0 = 1 - u2/2 + u2^2/8 + t [ (x2-2)/2 + u2 (4-x2)/4 ] + t^2 (x2^2-8x2+8)/8,
// which is App. B regrouped; f_eq = w rho P.  Populations l and opp(l) have
// cu of opposite sign, so P(+-cu) = E(cu^2) +- cu O(cu^2) is evaluated once per
// pair.  Relaxation: f <- (1-omega) f + (omega rho w) P.

struct Macro {
  double rho, ux, uy, T;
  double jx, jy, e;  // the raw sums: j = sum c f, e = sum |c|^2 f
};

// Relaxation parameters of one launch: omega = dt/tau, 1 - omega, and the
// body-force shift of the equilibrium (reading G7b): u_eq = u + (tgx, tgy)
// with (tgx, tgy) = g/omega, T_eq = T + dT with dT = (1/omega)(1 - 1/omega)|g|^2/D.
// With g = 0 the shifts are exact zeros and the arithmetic is unchanged.
struct Relax {
  double omega, one_m_omega, tgx, tgy, dT;
};

__device__ __forceinline__ double dadd(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ double dsub(double a, double b) { return __dsub_rn(a, b); }
__device__ __forceinline__ double dmul(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ double dfma(double a, double b, double c) { return __fma_rn(a, b, c); }

__device__ __forceinline__ Macro moments(const double (&f)[Q]) {
  // column sums S[cx+3]
  double S[7];
#pragma unroll
  for (int k = 0; k < 7; ++k) S[k] = 0.0;
  {
    bool first[7] = {true, true, true, true, true, true, true};
#pragma unroll
    for (int l = 0; l < Q; ++l) {
      const int k = CX(l) + 3;
      if (first[k]) { S[k] = f[l]; first[k] = false; }
      else S[k] = dadd(S[k], f[l]);
    }
  }
  double R[7];
  {
    bool first[7] = {true, true, true, true, true, true, true};
#pragma unroll
    for (int l = 0; l < Q; ++l) {
      const int k = CY(l) + 3;
      if (first[k]) { R[k] = f[l]; first[k] = false; }
      else R[k] = dadd(R[k], f[l]);
    }
  }
  const double rho = dadd(dadd(dadd(S[0], S[6]), dadd(S[1], S[5])), dadd(dadd(S[2], S[4]), S[3]));
  const double jx = dfma(3.0, dsub(S[6], S[0]), dfma(2.0, dsub(S[5], S[1]), dsub(S[4], S[2])));
  const double jy = dfma(3.0, dsub(R[6], R[0]), dfma(2.0, dsub(R[5], R[1]), dsub(R[4], R[2])));
  const double ex = dfma(9.0, dadd(S[6], S[0]), dfma(4.0, dadd(S[5], S[1]), dadd(S[4], S[2])));
  const double ey = dfma(9.0, dadd(R[6], R[0]), dfma(4.0, dadd(R[5], R[1]), dadd(R[4], R[2])));
  const double e = dadd(ex, ey);
  const double inv = __drcp_rn(rho);
  Macro m;
  m.rho = rho;
  m.jx = jx;
  m.jy = jy;
  m.e = e;
  m.ux = dmul(jx, inv);
  m.uy = dmul(jy, inv);
  const double uu = dfma(m.ux, m.ux, dmul(m.uy, m.uy));
  m.T = dmul(0.5, dsub(dmul(e, inv), uu));
  return m;
}

// Shell coefficients of the quartic.
struct Shell {
  double A0, A1, A2;
};

#ifdef LB_CONST_BANK
// (variant build, tools/build_tb_variant.py ... LB_CONST_BANK=1) the per-shell
// constants as constant-bank operands instead of 64-bit immediates (2 UMOV each)
struct ShellK {
  double k0, k1, k2, ka, kb, w;
};
constexpr ShellK shell_k(int s) {
  const double x2 = A2 * (double)SHELL_C2(s);
  return ShellK{0.5 * (x2 - 2.0), 0.25 * (4.0 - x2), 0.125 * ((x2 * x2 - 8.0 * x2) + 8.0), 0.5 * (x2 - 4.0),
                0.25 * (x2 - 6.0), SHELL_W(s)};
}
static __constant__ ShellK c_shk[NSHELL] = {shell_k(0), shell_k(1), shell_k(2), shell_k(3),
                                            shell_k(4), shell_k(5), shell_k(6), shell_k(7)};
#define LB_SHK(s, f, expr) c_shk[s].f
#else
#define LB_SHK(s, f, expr) (expr)
#endif

__device__ __forceinline__ void shell_coeffs(double u2, double t, Shell (&sh)[NSHELL]) {
  const double tt = dmul(t, t);
  const double b1 = dfma(-0.5, u2, 1.0);                  // 1 - u2/2
  const double b0 = dfma(dmul(0.125, u2), u2, b1);        // 1 - u2/2 + u2^2/8
  const double b2 = dfma(-0.25, u2, 0.5);                 // 1/2 - u2/4
#pragma unroll
  for (int s = 0; s < NSHELL; ++s) {
    const double x2 = A2 * (double)SHELL_C2(s);
    const double k0 = LB_SHK(s, k0, 0.5 * (x2 - 2.0));
    const double k1 = LB_SHK(s, k1, 0.25 * (4.0 - x2));
    const double k2 = LB_SHK(s, k2, 0.125 * ((x2 * x2 - 8.0 * x2) + 8.0));
    const double ka = LB_SHK(s, ka, 0.5 * (x2 - 4.0));
    const double kb = LB_SHK(s, kb, 0.25 * (x2 - 6.0));
    sh[s].A0 = dfma(t, dfma(u2, k1, k0), dfma(tt, k2, b0));
    sh[s].A1 = dfma(t, ka, b1);
    sh[s].A2 = dfma(t, kb, b2);
  }
}

__device__ __forceinline__ double cu_of(int l, double Ux, double Uy) {
  if (CX(l) == 0) return dmul((double)CY(l), Uy);
  if (CY(l) == 0) return dmul((double)CX(l), Ux);
  return dfma((double)CX(l), Ux, dmul((double)CY(l), Uy));
}

// A collision hook sees the moments of the pre-collision f as soon as they are
// formed (monitors, lb_tb.cu); the default does nothing.
struct NoHook {
  __device__ __forceinline__ void operator()(const Macro&) const {}
};

// f <- f - omega (f - f_eq(moments of f)), in registers; hook(moments).
template <class Hook = NoHook>
__device__ __forceinline__ void collide_site(double (&f)[Q], const Relax& r, const Hook& hook = Hook{}) {
  const double omega = r.omega, one_m_omega = r.one_m_omega;
  const Macro m = moments(f);
  hook(m);
  const double ux = dadd(m.ux, r.tgx), uy = dadd(m.uy, r.tgy), Te = dadd(m.T, r.dT);
  const double Ux = dmul(A2, ux), Uy = dmul(A2, uy);
  const double u2 = dmul(A2, dfma(ux, ux, dmul(uy, uy)));
  const double t = dfma(A2, Te, -1.0);
  Shell sh[NSHELL];
  shell_coeffs(u2, t, sh);
  const double orho = dmul(omega, m.rho);
  double g[NSHELL];
#pragma unroll
  for (int s = 0; s < NSHELL; ++s) g[s] = dmul(orho, LB_SHK(s, w, SHELL_W(s)));
  constexpr double C3 = 1.0 / 6.0, C4 = 1.0 / 24.0;
#pragma unroll
  for (int l = 0; l < Q / 2; ++l) {
    const int s = shell_of(l);
    const double cu = cu_of(l, Ux, Uy);
    const double q = dmul(cu, cu);
    const double E = dfma(q, dfma(q, C4, sh[s].A2), sh[s].A0);
    const double O = dmul(cu, dfma(q, C3, sh[s].A1));
    const double pp = dadd(E, O), pm = dsub(E, O);
    f[l] = dfma(g[s], pp, dmul(one_m_omega, f[l]));
    f[opp(l)] = dfma(g[s], pm, dmul(one_m_omega, f[opp(l)]));
  }
  f[Q / 2] = dfma(g[0], sh[0].A0, dmul(one_m_omega, f[Q / 2]));
}

// f_eq(rho, u, T) for initialisation (same quartic).
__device__ __forceinline__ void feq_site(double rho, double ux, double uy, double T, double (&f)[Q]) {
  const double Ux = dmul(A2, ux), Uy = dmul(A2, uy);
  const double u2 = dmul(A2, dfma(ux, ux, dmul(uy, uy)));
  const double t = dfma(A2, T, -1.0);
  Shell sh[NSHELL];
  shell_coeffs(u2, t, sh);
  double g[NSHELL];
#pragma unroll
  for (int s = 0; s < NSHELL; ++s) g[s] = dmul(rho, SHELL_W(s));
  constexpr double C3 = 1.0 / 6.0, C4 = 1.0 / 24.0;
#pragma unroll
  for (int l = 0; l < Q / 2; ++l) {
    const int s = shell_of(l);
    const double cu = cu_of(l, Ux, Uy);
    const double q = dmul(cu, cu);
    const double E = dfma(q, dfma(q, C4, sh[s].A2), sh[s].A0);
    const double O = dmul(cu, dfma(q, C3, sh[s].A1));
    f[l] = dmul(g[s], dadd(E, O));
    f[opp(l)] = dmul(g[s], dsub(E, O));
  }
  f[Q / 2] = dmul(g[0], sh[0].A0);
}

#endif  // __CUDACC__

}  // namespace lbd
