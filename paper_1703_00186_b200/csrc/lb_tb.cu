// lb_tb.cu — two time steps per pass over HBM (temporal blocking of the fused
// pull step, §8a5 extended; DESIGN.md §8 "k_step2_tb").
//
// The fused step (k_step_fused) moves 592 B/site per step and runs at the HBM
// copy roof, with the FP64 pipe ~25 % busy.  This kernel computes steps n+1 AND
// n+2 from state n in one pass, keeping the intermediate state n+1 in shared
// memory, so HBM sees ~296·(1 + overlap) B read + 296 B written per site per
// TWO steps.  The per-site arithmetic is the very same device code as the fused
// kernel (gather order, thermal_wall, collide_site / collide_site_reg), so the
// result is bit-identical to two k_step_fused launches.
//
// Tiling.  A CTA owns a strip of HT rows [ya, ya+HT) and sweeps a range of
// output columns [xs, xs + W) in x.  Iteration t of a sweep:
//   * TMA: for every column group g (the populations of one cx_g, consecutive
//     labels), the window of state n that phase 1 of iteration t + PF pulls
//     them from — column c1(t + PF) - cx_g (wrapped periodically: N = 1 needs
//     no halo), rows [ya - 6, ya + HT + 6) (the union over cy of the rows
//     [ya - 3 - cy, ya + HT + 3 - cy); ya even, so the box starts on 16 bytes,
//     the TMA alignment rule of tools/tma_probe.cu), RB = HT + 12 rows.  The
//     TMA coordinates perform the whole x-pull (propagate), so the state-n
//     ring is just NB = PF + 1 = 2 buffers.  7 loads per column, one per
//     issuing lane.  The phase-1 warps refill the buffer they just gathered
//     from (named barrier 2 among them, then their lanes issue the loads of
//     iteration t + NB), so a load has ~2 iterations in flight (EARLY);
//   * phase 1 (warps [0, NW1)): state n+1 at column c1 = xs - 3 + t for the
//     R1 = HT + 6 rows [ya - 3, ya + HT + 3) (the ±3-row apron step n+2 pulls
//     from), written to the state-(n+1) ring;
//   * phase 2 (warps [NW1, NW1 + NW2)): state n+2 at column c2 = c1 - 4 for the
//     HT rows of the strip, gathered from the state-(n+1) ring, stored to B
//     (and, for the 3+3 border columns, into B's halo: the next step's wrap).
// Both phases of an iteration are independent (phase 2 lags by one column more
// than the ±3 reach), so ONE __syncthreads per iteration orders everything
// (BGK).  The regularised kernel (LB_TB_DECOUPLE) hands the state-(n+1) ring
// between the phases with mbarriers instead: phase 2 of iteration t waits
// until phase 1 wrote iteration t-1 and releases its slots right after its
// gather; phase 1 of iteration t waits for that release of iteration t-1, so
// either phase can run up to one iteration ahead of the other.
//
// State-(n+1) ring.  Population l of column c1 is pulled by phase 2 at column
// c1 + cx_l, cx_l + 4 iterations later: cx_l + 5 slots of R1 rows (185 slots
// over the 37 populations).  HT = 104, PF = 1: 69 KB (state n) + 163 KB
// (state n+1) of shared memory, 214 sites per iteration, 8 warps.
//
// Walls (G9) are data: the mirrored populations are copied into ring rows
// beyond each wall ("virtual rows"), so the plain gather is exact for every row
// and all warps run ONE code path per phase.  Periodic-Y geometry is not
// supported here (the 1-step kernel serves it).
//
// Work split: the strips × lx column-units are cut into gridDim.x contiguous
// ranges (one CTA per SM, persistent); a range crossing a strip boundary is two
// sweeps (strip_ya: the layout).
#include <cuda.h>
#include <cudaTypedefs.h>

#include "lb_collide.cuh"
#include "lb_device.cuh"
#include "lb_internal.h"

#ifndef LB_TB_LEAD  // lead-in weight of a sweep in the work split (0: none)
#define LB_TB_LEAD 7
#endif
#ifndef LB_TB_STCS
#define LB_TB_STCS 0
#endif
// bit 0: BGK, bit 1: regularised — the time-aligned work split can be used
// (see the kernel; the host's default, with wall / tail weights 21 / 17
// x1/16: BGK +7.6 %, regularised +3.4 % at 1920x2048)
#ifndef LB_TB_ALIGN
#define LB_TB_ALIGN 3
#endif
// clusters of 2 CTAs sweeping adjacent strips in lockstep (see the kernel;
// variant builds only: -3 %, the per-iteration cluster barrier costs more than
// the 208-row store runs gain)
#ifndef LB_TB_PAIR
#define LB_TB_PAIR 0
#endif
// phase-2 warp rotation (see the kernel; 0 = warp NW1 + k handles row block k).
// Measured neutral (rotations 0 / 1 / 2 at the tuned weights: 17.85K / 17.79K /
// 17.83K, then 17.65K / 17.81K / 17.77K): the wall strips' extra cost is not
// scheduler contention.  Variant builds only.
// phase 2 stores only the rows its strip owns (see phase2_update; variant
// builds only): measured -0.8 % (18.27K vs 18.42K MLUPS, 3 alternating reps) —
// the 32 overlap rows no longer stored twice, but the top strip's first owned
// row starts mid-line, so both strips write partial 128-byte lines
#ifndef LB_TB_STORE_OWNED
#define LB_TB_STORE_OWNED 0
#endif
#ifndef LB_TB_P2ROT
#define LB_TB_P2ROT 0
#endif
#ifndef LB_TB_CLOCK  // variant builds only: per-CTA start/end times (tools/tb_clock.py)
#define LB_TB_CLOCK 0
#endif
#if LB_TB_CLOCK
__device__ unsigned long long g_tb_clock[1024 * 4];
#endif

namespace lbk {
using namespace lbd;

namespace {

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

#ifndef LB_TB_WAR_FENCE  // proxy fence between the phase-1 gather and the TMA refill of its buffer
#define LB_TB_WAR_FENCE 1
#endif
// (Measured and rejected: with SKEW in every kernel, phase 2 gathers the
// populations with cx >= -2 one iteration early, so cx + 4 slots suffice (151
// instead of 185) and HT = 114 fits (18 strips at ly = 2048 instead of 20):
// 15.2K MLUPS against 16.4-16.5K — the taller iterations cost more than the
// 10 % fewer of them save.)
LB_HD constexpr int L1(int l) { return CX(l) + 5; }

// Literal tables (a constexpr loop evaluated in device code is NOT folded by
// cicc: it materialises the velocity table on the stack, and inside this
// kernel's loops it made the compile time explode).  CXSUM(l) = sum_{m<l} cx_m;
// REFL(l) = refl(l).  Both are checked against lb_device.cuh by static_assert.
LB_HD constexpr int CXSUM(int l) {
  constexpr int t[Q + 1] = {0,  3,  6,  9,  11, 13, 15, 17, 19, 20, 21, 22, 23, 24, 25, 26, 26, 26, 26,
                            26, 26, 26, 26, 25, 24, 23, 22, 21, 20, 19, 17, 15, 13, 11, 9,  6,  3,  0};
  return t[l];
}
LB_HD constexpr int REFL(int l) {
  constexpr int t[Q] = {2,  1,  0,  7,  6,  5,  4,  3,  14, 13, 12, 11, 10, 9,  8,  21, 20, 19, 18,
                        17, 16, 15, 28, 27, 26, 25, 24, 23, 22, 33, 32, 31, 30, 29, 36, 35, 34};
  return t[l];
}
constexpr bool tables_ok() {
  int s = 0;
  for (int l = 0; l < Q; ++l) {
    if (CXSUM(l) != s || REFL(l) != refl(l)) return false;
    s += CX(l);
  }
  return CXSUM(Q) == s;
}
static_assert(tables_ok(), "CXSUM / REFL tables");

// state-(n+1) ring slots of the populations before l
LB_HD constexpr int SLOTS1_BEFORE(int l) {
  return CXSUM(l) + 5 * l;
}
constexpr bool slots_ok() {
  int s = 0;
  for (int l = 0; l < Q; ++l) {
    if (SLOTS1_BEFORE(l) != s) return false;
    s += L1(l);
  }
  return SLOTS1_BEFORE(Q) == s;
}
static_assert(slots_ok(), "ring slot offsets");

// Column groups.  The labels run cx = +3 .. -3 with cy ascending (App. A), so
// the populations of one cx are consecutive labels: group g = 3 - cx holds
// GN(g) populations from label GFIRST(g).  Phase 1 pulls every population of
// group g from the same state-n column c1 - cx, and the union of their row
// windows is [ya - 6, ya + HT + 6), so ONE TMA box {HT + 12 rows, GN(g)
// populations, 1 column} loads the whole group: 7 TMA loads per column
// instead of 37.  Box heights of 3, 5 and 7 populations need 3 tensor maps
// (class GCLS(g)).
constexpr int NG = 7;
LB_HD constexpr int GFIRST(int g) {
  constexpr int t[NG + 1] = {0, 3, 8, 15, 22, 29, 34, 37};
  return t[g];
}
LB_HD constexpr int GN(int g) { return GFIRST(g + 1) - GFIRST(g); }
LB_HD constexpr int GCLS(int g) { return GN(g) == 3 ? 0 : (GN(g) == 5 ? 1 : 2); }
LB_HD constexpr int GOF(int l) { return 3 - CX(l); }  // group of population l
constexpr int CLS_N[3] = {3, 5, 7};
constexpr bool groups_ok() {
  for (int l = 0; l < Q; ++l)
    if (l < GFIRST(GOF(l)) || l >= GFIRST(GOF(l) + 1)) return false;
  for (int g = 0; g < NG; ++g)
    if (CLS_N[GCLS(g)] != GN(g)) return false;
  return true;
}
static_assert(groups_ok(), "column groups of the label order");
// shared-memory offset (doubles) of group g in a state-n buffer: each group's
// slab starts on a 128-byte boundary (TMA destination alignment)
LB_HD constexpr int GOFF(int g, int RB) {
  int o = 0;
  for (int h = 0; h < g; ++h) o += (GN(h) * RB + 15) / 16 * 16;
  return o;
}
// offset of population l's window (row ya - 6) in a state-n buffer
LB_HD constexpr int POFF(int l, int RB) { return GOFF(GOF(l), RB) + (l - GFIRST(GOF(l))) * RB; }

// ---- TMEM-resident state-(n+1) ring (LB_TB_TMEM) ----------------------------
// Phase 1 writes state n+1 of its rows to a shared-memory staging buffer, two
// populations of equal cy per 16-byte row ("pairs": each cy group in label
// order, i.e. cx descending, paired off, 22 pairs); one thread then copies
// every pair into the ring in tensor memory with tcgen05.cp .128x128b from a
// descriptor whose start is shifted by 3 - cy rows, so TMEM lane p receives
// staging row p + 3 - cy — exactly the value phase 2 pulls for strip row p.
// Phase 2 (lane quarter = its warp) reads its own lane with tcgen05.ld, so the
// ±3-row pull costs no shared-memory traffic.  Pair j keeps TP_LT(j) =
// cx_A + 5 slots of 4 columns (its first population has the larger cx): 440
// of the 512 columns.  tools/tmem_probe.cu checks the shifted copy.
constexpr int NPAIR = 22;
LB_HD constexpr int TP_A(int j) {
  constexpr int t[NPAIR] = {8, 22, 3, 16, 29, 0, 10, 24, 34, 1, 11, 25, 35, 2, 12, 26, 36, 7, 20, 33, 14, 28};
  return t[j];
}
LB_HD constexpr int TP_B(int j) {  // -1: a single population
  constexpr int t[NPAIR] = {15, -1, 9, 23, -1, 4, 17, 30, -1, 5, 18, 31, -1, 6, 19, 32, -1, 13, 27, -1, 21, -1};
  return t[j];
}
LB_HD constexpr int TP_CY(int j) {
  constexpr int t[NPAIR] = {-3, -3, -2, -2, -2, -1, -1, -1, -1, 0, 0, 0, 0, 1, 1, 1, 1, 2, 2, 2, 3, 3};
  return t[j];
}
LB_HD constexpr int TP_LT(int j) {
  constexpr int t[NPAIR] = {6, 4, 7, 5, 3, 8, 6, 4, 2, 8, 6, 4, 2, 8, 6, 4, 2, 7, 5, 3, 6, 4};
  return t[j];
}
LB_HD constexpr int TP_COL(int j) {  // first TMEM column of pair j's slots
  constexpr int t[NPAIR + 1] = {0,   24,  40,  68,  88,  100, 132, 156, 172, 180, 212, 236,
                                252, 260, 292, 316, 332, 340, 368, 388, 400, 424, 440};
  return t[j];
}
LB_HD constexpr int POP_PAIR(int l) {
  constexpr int t[Q] = {5, 9,  13, 2,  5,  9,  13, 17, 0, 2,  6,  10, 14, 17, 20, 0,  3,  6, 10,
                        14, 18, 20, 1, 3, 7, 11, 15, 18, 21, 4, 7, 11, 15, 19, 8, 12, 16};
  return t[l];
}
LB_HD constexpr int POP_HALF(int l) {
  constexpr int t[Q] = {0, 0, 0, 0, 1, 1, 1, 0, 0, 1, 0, 0, 0, 1, 0, 1, 0, 1, 1,
                        1, 0, 1, 0, 1, 0, 0, 0, 1, 0, 0, 1, 1, 1, 0, 0, 0, 0};
  return t[l];
}
constexpr bool tmem_tables_ok() {
  int col = 0, seen = 0;
  for (int j = 0; j < NPAIR; ++j) {
    const int a = TP_A(j), b = TP_B(j);
    if (TP_COL(j) != col || CY(a) != TP_CY(j) || TP_LT(j) != CX(a) + 5) return false;
    if (POP_PAIR(a) != j || POP_HALF(a) != 0) return false;
    ++seen;
    if (b >= 0) {
      if (CY(b) != TP_CY(j) || CX(b) >= CX(a) || POP_PAIR(b) != j || POP_HALF(b) != 1) return false;
      ++seen;
    }
    col += 4 * TP_LT(j);
  }
  return seen == Q && TP_COL(NPAIR) == col && col <= 512;
}
static_assert(tmem_tables_ok(), "TMEM ring pair tables");

#ifndef LB_TB_TMEM
#define LB_TB_TMEM 0
#endif

template <int HT_, int PF_>
struct TbCfg {
  static constexpr int HT = HT_;
  static constexpr int PF = PF_;
  static constexpr int RB = HT + 12;                // TMA box rows of a group window [ya - 6, ya + HT + 6)
  static constexpr int BUFD = GOFF(NG, RB);         // doubles per state-n buffer (7 group slabs)
  static constexpr int R1 = HT + 6;
  static constexpr int NW1 = (R1 + 31) / 32;        // phase-1 warps
  static constexpr int NW2 = (HT + 31) / 32;        // phase-2 warps
  static constexpr int NW = NW1 + NW2;
  static constexpr int NT = 32 * NW;
  static constexpr int NB = PF + 1;                 // state-n buffers per population = mbarriers
  static constexpr int S0_DBL = NB * BUFD;
  // the state-(n+1) ring in shared memory, or (LB_TB_TMEM) two staging buffers
  // of NPAIR pair regions of R1 rows x 16 bytes (+ 24 rows: the shifted copy
  // of the last pair reads up to row 6 + 127)
  static constexpr int STG_DBL = NPAIR * R1 * 2 + 48;
  static constexpr int S1_DBL = LB_TB_TMEM ? 2 * STG_DBL : SLOTS1_BEFORE(Q) * R1;
  // mbarriers: NB TMA buffers + (LB_TB_DECOUPLE) 2 full + 2 empty ring barriers
  // + (LB_TB_TMEM) 2 copy-complete barriers; then the TMEM base address
  static constexpr size_t SMEM = (size_t)(S0_DBL + S1_DBL) * sizeof(double) + (NB + 6) * sizeof(uint64_t) + 16;
  static_assert(RB % 2 == 0 && RB <= 256, "TMA box rows");
  static_assert(SMEM <= 232448, "shared memory per CTA");
  static_assert(NW <= 8, "two warps per scheduler at most (64 KB register file per scheduler)");
};

__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t parity) {
  asm volatile(
      "{\n"
      " .reg .pred p;\n"
      "WAIT_%=:\n"
      " mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      " @!p bra WAIT_%=;\n"
      "}\n" ::"r"(bar),
      "r"(parity)
      : "memory");
}

// An opaque copy of a loop-invariant value: keeps the compiler from hoisting
// the 37 per-population store addresses out of the sweep loop (37 live 64-bit
// registers on top of the 37 populations).
__device__ __forceinline__ int opaque(int v) {
  int r;
  asm volatile("mov.b32 %0, %1;" : "=r"(r) : "r"(v));
  return r;
}

// periodic wrap of an internal column index into the physical range [3, 3+lx)
__device__ __forceinline__ int wrap_col(int j, int lx) {
  int x = j - H;
  if (x < 0) x += lx;
  else if (x >= lx) x -= lx;
  return H + x;
}

// Walls as data (reading G9 i): a pull source row sy < 0 of population l reads
// population refl(l) at row -1 - sy, a source row sy >= ly reads refl(l) at
// 2 ly - 1 - sy.  Both rings hold those mirrored values in their rows beyond
// the wall ("virtual rows"), so the plain gather is exact for every row and all
// warps run ONE code path per phase (no mirror variant: fewer instructions, a
// smaller instruction footprint, and wall strips cost what interior strips cost).
//
// Strip layout.  Strip s covers rows [ya, ya + HT) (ya even: TMA box starts
// are 16-byte aligned).  A strip whose phase-1 rows [ya - 3, ya + HT + 3) reach
// a wall band (3 rows) must contain that wall, because the mirror sources of
// the band rows lie only in the windows of a strip that does.  So: strips from
// the bottom at s·HT; the top strip moved down to end on the wall; the strip
// below it moved down (if needed) to end >= 6 rows below the wall.  Heights
// HT < ly < HT + 6 admit no such layout (tb_layout_ok; lb_step then uses
// the one-step kernel).
LB_HD inline int strip_ya(int s, int nstrips, int ly, int HT) {
  if (s == nstrips - 1) return ((ly - HT + 1) & ~1) > 0 ? ((ly - HT + 1) & ~1) : 0;
  if (s == nstrips - 2) {
    const int lim = (ly - 6 - HT) & ~1;
    return s * HT < lim ? s * HT : lim;
  }
  return s * HT;
}

// State-n virtual rows.  Buffer b (just arrived): population l's window comes
// from the same column as refl(l)'s (same cx, same group), so the virtual rows
// are copies within buffer b — 26 per wall (cy_l > 0: rows -1..-cy_l at the
// bottom; cy_l < 0: rows ly..ly+|cy_l|-1 at the top), one per lane.  Offsets
// relative to s0 + b·BUFD - ya (bottom) or s0 + b·BUFD - ya + ly (top); the
// strip layout keeps every copy inside the window [ya - 6, ya + HT + 6): a
// bottom strip has ya = 0, a top strip ends on the wall (strip_ya).
constexpr int NVROW = 26;
struct VRowTab {
  int2 bot[32], top[32];  // (dst, src) offsets; entries >= NVROW unused
};
template <int RB>
constexpr VRowTab make_vrows() {
  VRowTab t{};
  int nb = 0, nt = 0;
  for (int l = 0; l < Q; ++l) {
    const int c = CY(l), m = REFL(l);
    for (int q = 1; q <= c; ++q)  // row -q <- refl row q - 1
      t.bot[nb++] = int2{POFF(l, RB) + 6 - q, POFF(m, RB) + 6 + q - 1};
    for (int q = 0; q < -c; ++q)  // row ly + q <- refl row ly - 1 - q
      t.top[nt++] = int2{POFF(l, RB) + 6 + q, POFF(m, RB) + 6 - 1 - q};
  }
  return t;
}
constexpr bool vrows_ok() {
  int nb = 0, nt = 0;
  for (int l = 0; l < Q; ++l) {
    nb += CY(l) > 0 ? CY(l) : 0;
    nt += CY(l) < 0 ? -CY(l) : 0;
  }
  return nb == NVROW && nt == NVROW;
}

// Monitors (lb_monitor): per-thread running sums of the invariants of the
// sites a CTA owns after the collision: rho, j_x, j_y, E = 1/2 sum |c|^2 f and
// min rho (a NaN density counts as -inf so the minimum flags it).  They are
// formed from the moments the collision computes anyway — rho, j, e = sum
// |c|^2 f of the pre-collision site — which the collision conserves exactly in
// arithmetic, plus the body-force increments of reading G7b (j += rho omega tg,
// E += omega (j . tg + rho (|tg|^2 / 2 + dT)), zero without gravity): a few
// FP64 operations per site instead of a second pass over the 37 values (the
// two-step kernel is FP64-latency-bound).  They equal the sums over the stored
// state up to rounding (tests: <= 1e-13 of the mass).
//
// Failure detection: the minimum takes -inf when this collision's own output
// cannot be finite — rho NaN, or u or T NaN / infinite (f_eq and the relaxed
// values are then NaN; 0 * inf = NaN below) — so a blow-up created by the
// collision that produces the stored state is flagged by the same launch
// (k_monitor_reduce* -> the context's non-physical flag -> LB_ENONPHYS at lb_sync).
__device__ __forceinline__ double checked_rho(const Macro& m) {
  const double chk = __fma_rn(0.0, __dadd_rn(__dadd_rn(m.ux, m.uy), m.T), m.rho);
  return chk != chk ? -INFINITY : m.rho;
}

#ifndef LB_TB_MON_BRANCHLESS  // monitors accumulated without branches inside the collision (see below)
#define LB_TB_MON_BRANCHLESS 1
#endif
// Branch-free form (LB_TB_MON_BRANCHLESS): the owned-site test and the body
// force enter as factors, so the hook adds no branch in the middle of the
// collision (a branch there ends the basic block the compiler schedules the
// relaxation in).  w = 1 for an owned site, 0 otherwise; without a body force
// the increments are exact zeros, so the sums equal the branched form's
// (w m.rho + a is exact for w in {0, 1}).
__device__ __forceinline__ void acc_invariants_w(const Macro& m, const Relax& r, double w, double (&a)[5]) {
  const double djx = __dmul_rn(r.omega, __dmul_rn(m.rho, r.tgx));
  const double djy = __dmul_rn(r.omega, __dmul_rn(m.rho, r.tgy));
  const double tg2 = __fma_rn(r.tgx, r.tgx, __dmul_rn(r.tgy, r.tgy));
  const double dE = __dmul_rn(r.omega, __fma_rn(m.jx, r.tgx, __fma_rn(m.jy, r.tgy,
                                                    __dmul_rn(m.rho, __fma_rn(0.5, tg2, r.dT)))));
  a[0] = __fma_rn(w, m.rho, a[0]);
  a[1] = __fma_rn(w, __dadd_rn(m.jx, djx), a[1]);
  a[2] = __fma_rn(w, __dadd_rn(m.jy, djy), a[2]);
  a[3] = __fma_rn(w, __fma_rn(0.5, m.e, dE), a[3]);
  a[4] = fmin(a[4], w != 0.0 ? checked_rho(m) : INFINITY);
}

__device__ __forceinline__ void acc_invariants(const Macro& m, const Relax& r, double (&a)[5]) {
  if (r.tgx == 0.0 && r.tgy == 0.0 && r.dT == 0.0) {
    // no body force (uniform branch): the increments below are exact zeros
    a[0] = __dadd_rn(a[0], m.rho);
    a[1] = __dadd_rn(a[1], m.jx);
    a[2] = __dadd_rn(a[2], m.jy);
    a[3] = __dadd_rn(a[3], __dmul_rn(0.5, m.e));
    a[4] = fmin(a[4], checked_rho(m));
    return;
  }
  const double djx = __dmul_rn(r.omega, __dmul_rn(m.rho, r.tgx));
  const double djy = __dmul_rn(r.omega, __dmul_rn(m.rho, r.tgy));
  const double tg2 = __fma_rn(r.tgx, r.tgx, __dmul_rn(r.tgy, r.tgy));
  const double dE = __dmul_rn(r.omega, __fma_rn(m.jx, r.tgx, __fma_rn(m.jy, r.tgy,
                                                    __dmul_rn(m.rho, __fma_rn(0.5, tg2, r.dT)))));
  a[0] = __dadd_rn(a[0], m.rho);
  a[1] = __dadd_rn(a[1], __dadd_rn(m.jx, djx));
  a[2] = __dadd_rn(a[2], __dadd_rn(m.jy, djy));
  a[3] = __dadd_rn(a[3], __fma_rn(0.5, m.e, dE));
  a[4] = fmin(a[4], checked_rho(m));
}

#ifndef LB_TB_FAKE
#define LB_TB_FAKE 0
#endif
// LB_TB_NOLOAD (variant builds only, timing experiments): no state-n loads and
// no waits for them — the compute + stores of the kernel alone (results are
// then meaningless)
#ifndef LB_TB_NOLOAD
#define LB_TB_NOLOAD 0
#endif
// The collision of both phases.  LB_TB_FAKE (variant builds only, timing
// experiments): a one-multiply stand-in, to time the kernel's data-movement
// skeleton without the FP64 work (results are then meaningless).
template <int COLL, class Hook>
__device__ __forceinline__ void tb_collide(double (&f)[Q], const Relax& r, const Hook& hook) {
#if LB_TB_FAKE
#pragma unroll
  for (int l = 0; l < Q; ++l) f[l] = __dmul_rn(f[l], r.one_m_omega);
#else
  if (COLL == COLL_REGULARIZED) collide_site_reg(f, r, hook);
  else collide_site(f, r, hook);
#endif
}

// Phase 1 site update: state n+1 at row y = ya - 3 + i from state-n buffer b
// (the pulled values), result into the state-(n+1) ring slot of iteration t;
// the rows next to a wall also write the virtual rows their values mirror into.
// row y = ya - 3 + i of population l pulls row y - cy_l: window index i + 3 - cy_l
template <int BUFD, int RB>
__device__ __forceinline__ void phase1_gather(const double* s0, int b, int i, double (&f)[Q]) {
  const int io = opaque(i);  // not hoistable: no per-population address registers
  const double* sb = s0 + b * BUFD + io;
#pragma unroll
  for (int l = 0; l < Q; ++l) f[l] = sb[POFF(l, RB) + 3 - CY(l)];
}

template <int COLL, bool MON>
__device__ __forceinline__ void phase1_collide(double (&f)[Q], int y, int ly, bool thermal, const Relax& r, bool own,
                                               double (&acc)[5]) {
  if (thermal && (y < 3 || y >= ly - 3)) thermal_wall(f, y < 3 ? 0 : 1);
  // monitors: accumulated as soon as the collision has formed the moments
  auto hook = [&](const Macro& m) {
    if (MON && LB_TB_MON_BRANCHLESS) acc_invariants_w(m, r, own ? 1.0 : 0.0, acc);
    else if (MON && own) acc_invariants(m, r, acc);
  };
  tb_collide<COLL>(f, r, hook);
}

// state n+1 of row y into the ring slot of iteration t (+ the virtual rows it mirrors into)
// (Measured and rejected: slots of HT rows instead of R1 = HT + 6 — phase 1
// stores row i at i - 3 + cy_l when in range, phase 2 reads its own row — which
// frees the shared memory for HT = 108 (19 strips instead of 20 at ly = 2048):
// 16.30K MLUPS, and 16.33K at HT = 104, against 16.55K for this layout; the
// per-population store predicates cost more than the 5 % fewer iterations save.)
template <int R1>
__device__ __forceinline__ void phase1_store(const double (&f)[Q], double* s1, int t, int i, int y, int ly) {
  const int io = opaque(i);
  const bool wall = y < 3 || y >= ly - 3;
#pragma unroll
  for (int l = 0; l < Q; ++l) s1[(SLOTS1_BEFORE(l) + (t % L1(l))) * R1 + io] = f[l];
  if (wall) {
    // virtual row of refl(l): -1 - y (bottom) or 2 ly - 1 - y (top); ring row
    // index = absolute row - (ya - 3), and i = y - (ya - 3)
    const int vi = y < 3 ? i - 2 * y - 1 : i + 2 * (ly - 1 - y) + 1;
    if (vi >= 0 && vi < R1) {
#pragma unroll
      for (int l = 0; l < Q; ++l) s1[(SLOTS1_BEFORE(REFL(l)) + (t % L1(l))) * R1 + vi] = f[l];
    }
  }
}

template <int COLL, int R1, bool MON>
__device__ __forceinline__ void phase1_update(double (&f)[Q], double* s1, int t, int i, int y, int ly,
                                              bool thermal, const Relax& r, bool own, double (&acc)[5]) {
  phase1_collide<COLL, MON>(f, y, ly, thermal, r, own, acc);
  phase1_store<R1>(f, s1, t, i, y, ly);
}

// Phase 2 site update: state n+2 at row y = ya + i, column c2, from the
// state-(n+1) ring, stored to B (+ B's halo for the 3+3 border columns).
template <int COLL, int BUFD, int RB, int R1, bool MON>
__device__ __forceinline__ void phase1(const double* s0, double* s1, int b, int t, int i, int y, int ly,
                                       bool thermal, const Relax& r, bool own, double (&acc)[5]) {
  double f[Q];
  phase1_gather<BUFD, RB>(s0, b, i, f);
  phase1_update<COLL, R1, MON>(f, s1, t, i, y, ly, thermal, r, own, acc);
}

template <int R1>
__device__ __forceinline__ void phase2_gather(const double* s1, int t, int i, double (&f)[Q]) {
  const int io = opaque(i);
#pragma unroll
  for (int l = 0; l < Q; ++l) f[l] = s1[((t - 4 - CX(l)) % L1(l)) * R1 + SLOTS1_BEFORE(l) * R1 + io + 3 - CY(l)];
}

// SKEW: phase 2's gather split in two — the 34 populations of items <= t - 2
// (cx >= -2) at the end of iteration t - 1, the 3 of item t - 1 (cx = -3)
// at the start of iteration t (phase1_store / phase2_gather slot rules)
template <int R1, bool NEWEST>
__device__ __forceinline__ void phase2_gather_part(const double* s1, int t, int i, double (&f)[Q]) {
  const int io = opaque(i);
#pragma unroll
  for (int l = 0; l < Q; ++l)
    if ((CX(l) == -3) == NEWEST)
      f[l] = s1[((t - 4 - CX(l)) % L1(l)) * R1 + SLOTS1_BEFORE(l) * R1 + io + 3 - CY(l)];
}

template <int COLL, bool MON>
__device__ __forceinline__ void phase2_update(double (&f)[Q], double* __restrict__ B, const Geo& g, int y, int c2,
                                              bool thermal, const Relax& r, bool own, double (&acc)[5],
                                              bool wrap) {
  const int ly = g.ly;
  if (thermal && (y < 3 || y >= ly - 3)) thermal_wall(f, y < 3 ? 0 : 1);
  auto hook = [&](const Macro& m) {
    if (MON && LB_TB_MON_BRANCHLESS) acc_invariants_w(m, r, own ? 1.0 : 0.0, acc);
    else if (MON && own) acc_invariants(m, r, acc);
  };
  tb_collide<COLL>(f, r, hook);
  // LB_TB_STORE_OWNED: only the rows this strip owns are stored — the top
  // strip, moved down to end on the wall, overlaps the strip below by
  // (nstrips HT - ly) rows (32 at ly = 2048), whose identical values that strip
  // stores already
  if (LB_TB_STORE_OWNED && !own) return;
  // 64-bit stride: one IMAD.WIDE per store instead of IMAD + LEA + LEA.HI.X
  const int64_t nyp = opaque(g.nyp);
  double* p = B + (int64_t)c2 * g.cs + g.y0 + y;
#pragma unroll
  for (int l = 0; l < Q; ++l) {
#if LB_TB_STCS  // variant: streaming (evict-first) stores of state n+2
    __stcs(p + l * nyp, f[l]);
#else
    p[l * nyp] = f[l];
#endif
  }
  // N = 1 wrap of the next step: border columns also go to the halo
  if (wrap && c2 < 2 * H) {
    double* q = p + (int64_t)g.lx * g.cs;
#pragma unroll
    for (int l = 0; l < Q; ++l) q[l * nyp] = f[l];
  }
  if (wrap && c2 >= g.lx) {
    double* q = p - (int64_t)g.lx * g.cs;
#pragma unroll
    for (int l = 0; l < Q; ++l) q[l * nyp] = f[l];
  }
}

template <int COLL, int R1, bool MON>
__device__ __forceinline__ void phase2(const double* s1, double* __restrict__ B, const Geo& g, int t, int i,
                                       int y, int c2, bool thermal, const Relax& r, bool own, double (&acc)[5],
                                       bool wrap) {
  double f[Q];
  phase2_gather<R1>(s1, t, i, f);
  phase2_update<COLL, MON>(f, B, g, y, c2, thermal, r, own, acc, wrap);
}

// ---- TMEM ring helpers (LB_TB_TMEM) ------------------------------------------
// state n+1 of phase-1 row i (strip-relative, i = y - ya + 3) into staging row
// i of every pair (16-byte stores; single populations 8 bytes), and the
// mirrored values of the wall rows into the rows beyond the wall
// (phase1_store's virtual rows, same rule)
template <int R1>
__device__ __forceinline__ void stage_store(const double (&f)[Q], double* stg, int i, int y, int ly) {
  const int io = opaque(i);
#pragma unroll
  for (int j = 0; j < NPAIR; ++j) {
    double* q = stg + 2 * (j * R1 + io);
    if (TP_B(j) >= 0) *reinterpret_cast<double2*>(q) = make_double2(f[TP_A(j)], f[TP_B(j)]);
    else q[0] = f[TP_A(j)];
  }
  if (y < 3 || y >= ly - 3) {
    const int vi = y < 3 ? i - 2 * y - 1 : i + 2 * (ly - 1 - y) + 1;
    if (vi >= 0 && vi < R1) {
#pragma unroll
      for (int l = 0; l < Q; ++l) stg[2 * (POP_PAIR(REFL(l)) * R1 + vi) + POP_HALF(REFL(l))] = f[l];
    }
  }
}

// SM100 shared-memory matrix descriptor, K-major, no swizzle (rows of 16 B,
// 8-row core matrices 128 B apart; version 1), start address saddr
__device__ __forceinline__ uint64_t stage_desc(uint32_t saddr) {
  return (uint64_t)((saddr >> 4) & 0x3FFF) | ((uint64_t)(16 >> 4) << 16) | ((uint64_t)(128 >> 4) << 32) |
         ((uint64_t)1 << 46);
}

// one thread: copy staging buffer stg (phase-1 item of local iteration t)
// into every pair's ring slot t % TP_LT, shifted by 3 - cy rows, then commit
// the copies to the mbarrier cp_bar
template <int R1>
__device__ __forceinline__ void stage_copy(const double* stg, uint32_t tbase, int t, uint32_t cp_bar) {
  const uint32_t s0 = smem_u32(stg);
#pragma unroll
  for (int j = 0; j < NPAIR; ++j) {
    const uint64_t d = stage_desc(s0 + 16u * (uint32_t)(j * R1 + 3 - TP_CY(j)));
    const uint32_t dst = tbase + (uint32_t)(TP_COL(j) + 4 * (t % TP_LT(j)));
    asm volatile("tcgen05.cp.cta_group::1.128x128b [%0], %1;" ::"r"(dst), "l"(d) : "memory");
  }
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(cp_bar)
               : "memory");
}

// phase 2 (lane quarter q = warp % 4, lane = strip row 32 q + lane): the 37
// populations of state n+1 it pulls, from its own TMEM lane.  Population l
// comes from the item of iteration t - 4 - cx_l; only the three with cx = -3
// (labels 34..36) need the newest item t - 1, so their loads follow
// wait_newest() (the copies of item t - 1 complete) and the other 34 are in
// flight meanwhile.
template <class Wait>
__device__ __forceinline__ void tmem_gather(uint32_t tlane, int t, double (&f)[Q], const Wait& wait_newest) {
  uint32_t lo[Q], hi[Q];
  auto ld = [&](int l) {
    const int j = POP_PAIR(l);
    const uint32_t a = tlane + (uint32_t)(TP_COL(j) + 4 * ((t - 4 - CX(l)) % TP_LT(j)) + 2 * POP_HALF(l));
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x2.b32 {%0, %1}, [%2];" : "=r"(lo[l]), "=r"(hi[l]) : "r"(a));
  };
#pragma unroll
  for (int l = 0; l < Q; ++l)
    if (CX(l) != -3) ld(l);
  wait_newest();
#pragma unroll
  for (int l = 0; l < Q; ++l)
    if (CX(l) == -3) ld(l);
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
  for (int l = 0; l < Q; ++l) {
    // the registers are written asynchronously: tie every use to the wait
    asm volatile("" : "+r"(lo[l]), "+r"(hi[l]));
    f[l] = __hiloint2double((int)hi[l], (int)lo[l]);
  }
}

#ifndef LB_TB_HT
#define LB_TB_HT 104
#define LB_TB_PF 1
#endif
#ifndef LB_TB_EARLY
#define LB_TB_EARLY 1
#endif
// bit 0: BGK, bit 1: regularised collide (default: regularised only — the
// decoupled hand-over measured +7 % there, -1 % to +1 % with BGK)
#ifndef LB_TB_DECOUPLE
#define LB_TB_DECOUPLE 2
#endif
// bit 0: BGK, bit 1: regularised — the kernels NOT decoupled with mbarriers
// hand the ring over with two hardware named barriers (producer bar.arrive,
// consumer bar.sync) instead of one CTA barrier per iteration
#ifndef LB_TB_NBAR
#define LB_TB_NBAR 0
#endif
// bit 0: BGK, bit 1: regularised (default: BGK; +0.8 %, 16.50K vs 16.36K on one box;
// the regularised kernel keeps its decoupled hand-over: 15.57K vs 12.42K) — SKEW: the two phases are offset within an
// iteration so that one collides while the other moves data: phase 2 gathers
// the older 34 populations of its next column at the end of an iteration and
// only the 3 newest after the barrier, then collides at once, while phase 1
// gathers; phase 2's populations stay in registers across the iteration
// barrier (in the registers phase 1 gathers into).
#ifndef LB_TB_SKEW
#define LB_TB_SKEW 1
#endif
constexpr int TB_HT = LB_TB_HT;
constexpr int TB_PF = LB_TB_PF;
using Cfg = TbCfg<TB_HT, TB_PF>;
static_assert(vrows_ok(), "virtual-row copy count");
__constant__ VRowTab c_vrows = make_vrows<Cfg::RB>();
static_assert(GOFF(NG, Cfg::RB) == Cfg::BUFD, "group slabs");

// per-group TMA parameters of the issuing threads: (box class, first label,
// slab offset in a state-n buffer, cx)
__constant__ int4 c_tb_grp[NG] = {
#define LBTB_G(g) {GCLS(g), GFIRST(g), GOFF(g, Cfg::RB), 3 - g}
    LBTB_G(0), LBTB_G(1), LBTB_G(2), LBTB_G(3), LBTB_G(4), LBTB_G(5), LBTB_G(6)};
#undef LBTB_G

// Kernel tensor maps (all __grid_constant__): the state-n group windows of the
// source buffer per box class (3 / 5 / 7 populations), the same for the N > 1
// staging of the left / right neighbour's edge columns.
struct alignas(64) TbKMaps {
  CUtensorMap src[3], stL[3], stR[3];
};

// Warps [0, NW1): phase 1; [NW1, NW1 + NW2): phase 2.
// MON: monitors — each CTA reduces the invariants of the sites it owns (rows
// of its strips not covered by a lower strip, its output columns) for state
// n+1 into mon[blockIdx] and for state n+2 into mon[gridDim + blockIdx]
// (5 doubles each; fixed-order reductions, deterministic).
__device__ __forceinline__ unsigned long long ld_acquire_sys_u64(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}

// Thread 0 waits until the neighbour counters that are non-null reach *my_done
// (watchdog: *status = 1 after timeout_ns, then proceed; LB_EPEER at the next sync).
__device__ __forceinline__ void peer_wait(const unsigned long long* a, const unsigned long long* b,
                                          const unsigned long long* my_done, unsigned int* status,
                                          unsigned long long timeout_ns) {
  unsigned long long t0;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
  const unsigned long long want = *my_done;
  while ((a && ld_acquire_sys_u64(a) < want) || (b && ld_acquire_sys_u64(b) < want)) {
    __nanosleep(128);
    unsigned long long t1;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t1));
    if (timeout_ns && t1 - t0 > timeout_ns) {
      atomicExch(status, 1u);
      break;
    }
  }
}

template <int COLL, int HT, int PF, bool MON>
__global__ void __launch_bounds__(TbCfg<HT, PF>::NT, 1)
    k_step2_tb(const __grid_constant__ TbKMaps km, double* __restrict__ B, Geo g, Relax r, int nstrips,
               int l2_dist, int thermal, int wall_w16, double* __restrict__ mon, int peers,
               const double* __restrict__ Asrc, TbPeer pp, int inpull) {
  using C = TbCfg<HT, PF>;
  constexpr int RB = C::RB, BUFD = C::BUFD, R1 = C::R1, NB = C::NB;
  // EARLY (LB_TB_EARLY, or PF = 0): the phase-1 warps refill the buffer they
  // just gathered from with the windows of iteration t + NB (a named barrier
  // among them, then their lanes issue), so a load has ~NB iterations in
  // flight instead of PF
  constexpr bool EARLY = PF == 0 || LB_TB_EARLY;
  // DECOUPLE (LB_TB_DECOUPLE): no CTA barrier per iteration; the state-(n+1)
  // ring is handed between the phases with mbarriers, alternating between two
  // per direction (item I = the CTA's iteration count): full[I & 1] — the
  // phase-1 warps wrote item I; empty[I & 1] — the phase-2 warps finished
  // gathering in iteration I (the slots phase 1 overwrites at I + 1).  A phase
  // can run up to one iteration ahead of the other.
  constexpr bool DECOUPLE = !LB_TB_TMEM && ((LB_TB_DECOUPLE >> (COLL == COLL_REGULARIZED ? 1 : 0)) & 1);
  static_assert(!DECOUPLE || EARLY, "decoupled phases need the phase-1 warps to issue the loads");
  // NBAR: named barriers F(t) = 3 + (t & 1), "phase 1 wrote iteration t"
  // (phase 1 arrives, phase 2 syncs before its gather of t + 1), and
  // E(t) = 5 + (t & 1), "phase 2 gathered iteration t" (phase 2 arrives,
  // phase 1 syncs before its ring stores of t + 1, which overwrite the slots
  // phase 2 read in t).  Each phase can run up to one iteration ahead; the
  // two ids per direction keep a barrier's next arrival behind the
  // completion of its previous generation (hardware barriers count
  // arrivals: a second arrival of the same side would complete it alone).
  // Arrivals (t = 0 .. niter - 2) and syncs (t = 1 .. niter - 1) pair up
  // within a sweep, so no generation is left open across sweeps.
  constexpr bool NBAR = !DECOUPLE && ((LB_TB_NBAR >> (COLL == COLL_REGULARIZED ? 1 : 0)) & 1);
  static_assert(!NBAR || EARLY, "named-barrier hand-over needs the phase-1 warps to issue the loads");
  // TMEM (LB_TB_TMEM): the state-(n+1) ring in tensor memory (see NPAIR);
  // one CTA-wide barrier per iteration orders the staging, copies and reads
  constexpr bool TMEM = LB_TB_TMEM;
  constexpr bool SKEW = EARLY && !DECOUPLE && !NBAR && !TMEM &&
                        ((LB_TB_SKEW >> (COLL == COLL_REGULARIZED ? 1 : 0)) & 1);
  static_assert(!TMEM || (EARLY && !DECOUPLE && !NBAR), "TMEM ring: CTA barrier per iteration, early refill");
  static_assert(!TMEM || C::NW2 == 4, "TMEM ring: one phase-2 warp per TMEM lane quarter");
  // programmatic dependent launch (host option): the next launch may start
  // its CTAs (on SMs this launch frees) and run its prologue; it waits at
  // griddepcontrol.wait below for this grid's completion and memory
  asm volatile("griddepcontrol.launch_dependents;");
  extern __shared__ __align__(128) double sm[];
  double* s0 = sm;
  double* s1 = sm + C::S0_DBL;  // the ring, or (TMEM) the two staging buffers
  uint64_t* bars = reinterpret_cast<uint64_t*>(sm + C::S0_DBL + C::S1_DBL);
  uint32_t* tbase_smem = reinterpret_cast<uint32_t*>(bars + NB + 6);
  const int tid = threadIdx.x;
  const int warp = tid >> 5;
  const int lx = g.lx, ly = g.ly;

  if (TMEM && warp == 0) {  // the whole 512-column tensor memory (one CTA per SM)
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(tbase_smem)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (tid == 0) {
    for (int i = 0; i < NB; ++i) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(bars + i)));
    for (int i = 0; i < 2; ++i) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bars + NB + i)), "r"(32 * C::NW1));
      asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bars + NB + 2 + i)), "r"(32 * C::NW2));
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(bars + NB + 4 + i)));  // TMEM copies
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (TMEM) asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (TMEM) asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tbase = TMEM ? *tbase_smem : 0u;
  const uint32_t bar_cp = smem_u32(bars + NB + 4);  // TMEM: copies of phase-1 item k done: bar_cp + 8 (k & 1)
  // TMEM: this phase-2 warp's lane quarter
  const uint32_t tlane = tbase + ((uint32_t)(32 * (warp & 3)) << 16);
  // phase-2 warp w handles the strip rows of block (w - NW1 + P2ROT) mod NW2
  // (variant builds; P2ROT = 0 by default): rotation would place the warps
  // holding the wall band rows of the two phases
  // (the thermal repopulation and the virtual-row copies) sit on different
  // schedulers (warp w issues on scheduler w mod 4: unrotated, phase 1's
  // rows [ya-3, ya+29) and phase 2's [ya, ya+32) both land on scheduler 0 at
  // the bottom wall, and on scheduler 3 at the top wall).  TMEM: a warp reads
  // only its own lane quarter, so no rotation.
  constexpr int P2ROT = TMEM ? 0 : LB_TB_P2ROT;
  const int p2row = 32 * ((warp - C::NW1 + P2ROT) % C::NW2) + (tid & 31);

  // Weighted split: a column of a wall strip costs wall_w16 / 16 of an interior
  // one (thermal repopulation and mirror copies on its wall warps), so the CTAs
  // that sweep wall strips get proportionally fewer columns.  unit_at(T): the
  // first (strip, column) unit whose weighted start is >= T.
  // A sweep costs its W columns plus a lead-in of TB_LEAD iterations (phase 1
  // starts 6 columns early, phase 2 lags 1 more), and a range that crosses a
  // strip start pays a second lead-in: so every strip but the first is
  // preceded by TB_LEAD columns of weight, which the range holding that strip
  // start absorbs (unit_at maps T inside it to the strip start).
  constexpr int TB_LEAD = LB_TB_LEAD;
  // wall_w16 packs the wall-strip weight (low 16 bits) and the tail weight
  // (high 16 bits) of the aligned split, both x16
  const int tail_w16 = wall_w16 >> 16;
  wall_w16 &= 0xffff;
  auto strip_w = [&](int s) { return (nstrips > 1 && (s == 0 || s == nstrips - 1)) ? wall_w16 : 16; };
  // LB_TB_PAIR (variant, launched as clusters of 2 CTAs): the two CTAs of a
  // cluster sweep two vertically adjacent strips (a "virtual strip") over the
  // same columns in lockstep (a cluster barrier per iteration), so their
  // state-n+2 stores form 208-row runs; the split below then works on virtual
  // strips (pairs, weighted by the heavier strip) and cluster indices.
  const bool paired = LB_TB_PAIR && nstrips % 2 == 0 && gridDim.x % 2 == 0;
  const int CL = paired ? 2 : 1;
  const int nv = nstrips / CL, ng = (int)gridDim.x / CL, gid = (int)blockIdx.x / CL, rank = (int)blockIdx.x % CL;
  auto vw = [&](int v) { return CL == 1 ? strip_w(v) : std::max(strip_w(2 * v), strip_w(2 * v + 1)); };
  auto unit_at = [&](int64_t T) -> int64_t {
    int64_t acc = 0;
    for (int s = 0; s < nv; ++s) {
      const int w = vw(s);
      if (s > 0) {
        acc += (int64_t)TB_LEAD * w;
        if (T < acc) return (int64_t)s * lx;
      }
      const int64_t sw = (int64_t)lx * w;
      if (T < acc + sw) return (int64_t)s * lx + (T - acc + w - 1) / w;
      acc += sw;
    }
    return (int64_t)nv * lx;
  };
  int64_t wtot = 0;
  for (int s = 0; s < nv; ++s) wtot += (int64_t)(lx + (s > 0 ? TB_LEAD : 0)) * vw(s);
  // units u: (virtual strip, column) = v lx + x
  int64_t u = unit_at(wtot * gid / ng);
  int64_t u_end = unit_at(wtot * (gid + 1) / ng);
  // LB_TB_ALIGN / LB_TB_PAIR: time-aligned split.  R = ng / nv work units
  // (CTAs or clusters) per virtual strip sweep the same column ranges
  // [r c_v, (r + 1) c_v) of every virtual strip at the same time (main region
  // [0, R c_v), c_v shorter on the heavier wall strips), so the units of one
  // range write (and read) whole population columns together; the
  // E = ng - R nv remaining units share the columns [R c_v, lx) of every
  // virtual strip (tail region) by the weighted split above.
  constexpr bool ALIGN = (LB_TB_ALIGN >> (COLL == COLL_REGULARIZED ? 1 : 0)) & 1;
  const int R_al = ((ALIGN && tail_w16 >= 16) || paired) && nv > 1 ? ng / nv : 0;  // tail_w16 < 16: contiguous split
  const int E_al = ng - R_al * nv;
  const bool aligned = R_al >= 1 && E_al >= 1;
  const bool tail = aligned && gid >= R_al * nv;
  // weighted work per main unit: the E tail units work at tail_w16 / 16 of
  // the main units' rate, so a main unit takes W f / (E + f M) (f = tail
  // factor, M = R nv main units) instead of the average W / (E + M)
  int64_t t16 = 0;
  for (int s = 0; s < nv; ++s) t16 += (int64_t)lx * vw(s);
  t16 += (int64_t)16 * TB_LEAD * (ng + nv);
  if (aligned) {
    const int64_t f = tail_w16 >= 16 ? tail_w16 : 16;
    t16 = t16 * f / (16 * (int64_t)E_al + f * R_al * nv);
  }
  // main-region columns per unit: two values (interior weight 16, the wall
  // strips' weight), computed once — a 64-bit division per strip inside the
  // tail loops below cost the tail CTAs ~15 us before their first load
  // (two scalars, not an indexed array: that would live in local memory)
  auto cols_for = [&](int w) -> int {
    const int c = (int)std::max<int64_t>(1, t16 / w - TB_LEAD);
    return (int64_t)c * R_al >= lx ? (lx + R_al - 1) / R_al : c;
  };
  const int cm_int = aligned ? cols_for(16) : 0, cm_wall = aligned ? cols_for(vw(0)) : 0;
  auto main_cols = [&](int s) -> int { return vw(s) == 16 ? cm_int : cm_wall; };
  auto tail_lo = [&](int s) -> int { return tail ? std::min(lx, R_al * main_cols(s)) : 0; };
  if (aligned && !tail) {
    const int s = gid % nv, r = gid / nv, c = main_cols(s);
    u = (int64_t)s * lx + std::min(lx, r * c);
    u_end = (int64_t)s * lx + std::min(lx, (r + 1) * c);
  } else if (tail) {
    // the tail sequence: virtual strip s contributes its columns [tail_lo(s), lx)
    auto tail_at = [&](int64_t T) -> int64_t {
      int64_t acc = 0;
      bool first = true;
      for (int s = 0; s < nv; ++s) {
        const int lo = tail_lo(s), w = vw(s);
        if (lo >= lx) continue;
        if (!first) {
          acc += (int64_t)TB_LEAD * w;
          if (T < acc) return (int64_t)s * lx + lo;
        }
        first = false;
        const int64_t sw = (int64_t)(lx - lo) * w;
        if (T < acc + sw) return (int64_t)s * lx + lo + (T - acc + w - 1) / w;
        acc += sw;
      }
      return (int64_t)nv * lx;
    };
    int64_t wt = 0;
    bool first = true;
    for (int s = 0; s < nv; ++s)
      if (tail_lo(s) < lx) {
        wt += (int64_t)(lx - tail_lo(s) + (first ? 0 : TB_LEAD)) * vw(s);
        first = false;
      }
    const int e = gid - R_al * nv;
    u = tail_at(wt * e / E_al);
    u_end = tail_at(wt * (e + 1) / E_al);
  }
#if LB_TB_CLOCK
  unsigned long long clk0;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(clk0));
  int nsweeps = 0;
#endif
  uint32_t kglob = 0;  // load iterations of this CTA over all its sweeps (barrier phase)
  uint32_t iglob = 0;  // DECOUPLE: iterations of this CTA over all its sweeps (ring items)
  const uint32_t bar_full = smem_u32(bars + NB), bar_empty = smem_u32(bars + NB + 2);
  double acc[5] = {0.0, 0.0, 0.0, 0.0, INFINITY};  // MON: this thread's state (n+1 or n+2)
  bool cl_armed = false;  // PAIR: a cluster-barrier arrival is pending
  // everything above touched only kernel parameters and shared memory: from
  // here on global memory (the previous launch's output, the buffer it read)
  asm volatile("griddepcontrol.wait;" ::: "memory");

  while (u < u_end) {
    const int vstrip = (int)(u / lx);
    const int x0 = (int)(u % lx);
    if (x0 < tail_lo(vstrip)) {  // (tail units) the main region of this strip is not theirs
      u = (int64_t)vstrip * lx + tail_lo(vstrip);
      continue;
    }
    const int strip = vstrip * CL + rank;
    const int x1 = (int)std::min<int64_t>(lx, x0 + (u_end - u));
    u += x1 - x0;
    const int xs = H + x0, W = x1 - x0;  // output columns [xs, xs + W)
#if LB_TB_CLOCK
    nsweeps += 1;
#endif
    // strip rows [ya, ya + HT) (strip_ya); the top strip may reach one row
    // past the wall, which is simply not computed
    const int ya = strip_ya(strip, nstrips, ly, HT);
    const int nload = W + 6;          // phase-1 iterations (columns c1 = xs - 3 + t)
    const int niter = W + 7;          // + the phase-2 lag
    const int rbase = g.y0 + ya;      // internal row of ya
    // MON: rows this strip owns (not covered by the strip below)
    const int own_lo = strip == 0 ? 0 : std::max(ya, strip_ya(strip - 1, nstrips, ly, HT) + HT);
    const int own_hi = std::min(ya + HT, ly);
    // do phase-1 rows [ya - 3, ya + HT + 3) pull across a wall (CTA-uniform)?
    const bool vbottom = ya - 3 < 3;
    const bool vtop = ya + HT + 3 > ly - 3;

    // N > 1, exchange inside the kernel: this sweep reads state-n columns
    // [x0 - 6, x1 + 6) and writes [x0, x1).  Within 6 columns of the left
    // edge it reads the left neighbour's last columns (final once its previous
    // launch completed) and overwrites columns that neighbour's previous
    // launch read: wait for its counter, then the TMA loads those columns
    // straight from its current buffer.  Same on the right.  Interior sweeps
    // never wait.
    if (inpull) {
      const bool needL = x0 < 6, needR = x1 > lx - 6;
      if (needL || needR) {  // CTA-uniform
        if (tid == 0) peer_wait(needL ? pp.waitL : nullptr, needR ? pp.waitR : nullptr, pp.my_done, pp.status,
                                pp.timeout_ns);
        __syncthreads();
        // the neighbours' generic-proxy stores (other kernels), read next by this CTA's TMA
        asm volatile("fence.proxy.async.global;" ::: "memory");
      }
    }

    // TMA of the state-n window of column group g that phase 1 of iteration k
    // pulls (column c1(k) - cx_g, rows [ya - 6, ya + HT + 6)); one thread per
    // group; the thread of g = 0 also posts the expected bytes (complete_tx may
    // precede it: the phase cannot complete before that single arrival)
    auto issue_one = [&](int k, int gq) {
      if (LB_TB_NOLOAD) return;
      const uint32_t kb = kglob + (uint32_t)k;
      const uint32_t bar = smem_u32(bars + kb % NB);
      const int buf = (int)(kb % NB);
      const int c1 = xs - 3 + k;
      if (gq == 0) {
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar),
                     "r"((uint32_t)(Q * RB * sizeof(double))));
      }
      const int4 gp = c_tb_grp[gq];  // (box class, first label, slab offset, cx)
      const int cls = gp.x;
      const double* dst = s0 + buf * BUFD + gp.z;
      // source column: N = 1 periodic wrap; N > 1 the staging buffers beyond
      // the slab (left: internal -3..2, right: lx+3..lx+8)
      // (in-kernel exchange: the neighbours' buffers, whose internal column
      // lx + j resp. j - lx is our column j; staged: the staging buffers)
      const int j = c1 - gp.w;
      const CUtensorMap* m = &km.src[cls];
      int col = j;
      if (!peers) col = wrap_col(j, lx);
      else if (j < H) { m = &km.stL[cls]; col = inpull ? j + lx : j + H; }
      else if (j >= lx + H) { m = &km.stR[cls]; col = inpull ? j - lx : j - lx - H; }
      asm volatile(
          "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes"
          " [%0], [%1, {%2, %3, %4}], [%5];" ::"r"(smem_u32(dst)),
          "l"(m), "r"(rbase - 6), "r"(gp.y), "r"(col), "r"(bar)
          : "memory");
    };
    // lanes [0, GPW) of warp w issue groups GPW w + lane (EARLY: the phase-1
    // warps only — they refill their single buffer right after gathering from
    // it.  Measured and rejected: the phase-2 warps refilling it after an
    // mbarrier hand-over from phase 1, 11.2K / 15.2K MLUPS with the refill
    // after / before their collision, against 16.0-16.3K)
    constexpr int NWI = EARLY ? C::NW1 : (C::NW < NG ? C::NW : NG);
    constexpr int GPW = (NG + NWI - 1) / NWI;
    const int my_grp = GPW * warp + (tid & 31);
    const bool issuer = warp < NWI && (tid & 31) < GPW && my_grp < NG;

    if (issuer)
      for (int k = 0; k < (EARLY ? NB : PF) && k < nload; ++k) issue_one(k, my_grp);

    // SKEW: phase 2's next-column populations are carried across the
    // iteration barrier in fk; phase 1 gathers into the same registers (it
    // overwrites all of them before any use), so the carried values add no
    // register pressure to its path
    double fk[Q];
    for (int t = 0; t < niter; ++t) {
      const uint32_t I = iglob + (uint32_t)t;
      if (!DECOUPLE && !NBAR) __syncthreads();  // every read of iteration t-1 is done: the buffers refilled below are free
      if (LB_TB_PAIR && paired) {
        // lockstep with the other CTA of the cluster: wait for its arrival of
        // the previous iteration (latency hidden behind one iteration), arrive
        if (cl_armed) asm volatile("barrier.cluster.wait.aligned;" ::: "memory");
        asm volatile("barrier.cluster.arrive.relaxed.aligned;" ::: "memory");
        cl_armed = true;
      }
      if (TMEM) {
        // phase 1 staged item t - 1 and phase 2 finished reading the ring
        // slots of iteration t - 1 (tcgen05.wait::ld + fence before the
        // barrier): copy the staging into the ring; a phase-2 lane issues
        // (that phase waits for phase 1 at the barrier anyway)
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        if (tid == 32 * C::NW1 && t >= 1 && t - 1 < nload) {
          const uint32_t k = kglob + (uint32_t)(t - 1);
          stage_copy<R1>(s1 + (k & 1) * C::STG_DBL, tbase, t - 1, bar_cp + 8 * (k & 1));
        }
      }
      if (l2_dist > 0 && t + l2_dist < nload) {
        // L2 prefetch (LSU, not the TMA queue) of the newest column the loads
        // of iteration t + l2_dist touch: rows [ya - 6, ya + HT + 6) of all 37
        // planes, 8 lines of 128 B each; N > 1: slab columns only.  Off by
        // default (slower at every distance: 14.5K at 1 down to 11.4K at 6,
        // against 16.5K; a TMA prefetch of the whole window,
        // cp.async.bulk.prefetch.tensor, was slower still).  With it on the
        // refills hit L2 — the stress that exposed the gather / refill
        // write-after-read fixed by LB_TB_WAR_FENCE below.
        const int j = xs + t + l2_dist;  // c1(t + l2_dist) + 3
        if (!peers || j < lx + H) {
          const double* col = Asrc + (int64_t)(peers ? j : wrap_col(j, lx)) * g.cs + (rbase - 6);
          for (int q = tid; q < Q * 8; q += C::NT)
            asm volatile("prefetch.global.L2 [%0];" ::"l"(col + (int64_t)(q >> 3) * g.nyp + (q & 7) * 16));
        }
      }
      if (!EARLY && issuer && t + PF < nload) issue_one(t + PF, my_grp);
      if (warp < C::NW1) {
        // DECOUPLE: the slots written below were last read by phase 2 in I - 1
        if (DECOUPLE && t > 0) mbar_wait(bar_empty + 8 * ((I - 1) & 1), ((I - 1) >> 1) & 1);
        if (t < nload) {
          // phase 1: state n+1 at column c1 = xs - 3 + t, rows [ya-3, ya+HT+3)
          const uint32_t kb = kglob + (uint32_t)t;
          const int buf = (int)(kb % NB);
          if (!LB_TB_NOLOAD) mbar_wait(smem_u32(bars + buf), (kb / NB) & 1);
          // wall strips: warp 0 fills the virtual rows (one copy per lane),
          // then the phase-1 warps meet at named barrier 1 before reading
          if (vbottom || vtop) {
            const int lane = tid & 31;
            if (warp == 0 && lane < NVROW) {
              double* sb = s0 + buf * BUFD - ya;
              if (vbottom) {
                const int2 e = c_vrows.bot[lane];
                sb[e.x] = sb[e.y];
              }
              if (vtop) {
                const int2 e = c_vrows.top[lane];
                sb[ly + e.x] = sb[ly + e.y];
              }
              // generic-proxy writes to a buffer the TMA (async proxy) refills later
              asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            }
            asm volatile("bar.sync 1, %0;" ::"r"(32 * C::NW1) : "memory");
          }
          const int i = tid;
          const int y = ya - 3 + i;
          const bool valid = i < R1 && y >= 0 && y < ly;
          const bool own = t >= 3 && t < W + 3 && y >= own_lo && y < own_hi;
          if (EARLY) {
            // gather, then (all phase-1 warps done reading) refill the buffer
            // with iteration t + NB's windows while the collisions run
            double fl[Q];
            double(&f)[Q] = SKEW ? fk : fl;
            phase1_gather<BUFD, RB>(s0, buf, valid ? i : 0, f);
            // the TMA refill below (async proxy) overwrites what these loads
            // (generic proxy) read, and a load may still be in flight at the
            // barrier: order them (write-after-read across proxies).  Without
            // it, a refill that hits L2 (fast) could land under a pending load.
            if (LB_TB_WAR_FENCE) asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            asm volatile("bar.sync 2, %0;" ::"r"(32 * C::NW1) : "memory");
            if (issuer && t + NB < nload) issue_one(t + NB, my_grp);
            if (TMEM) {
              if (valid) {
                phase1_collide<COLL, MON>(f, y, ly, thermal, r, own, acc);
                // staging buffer kb & 1 was last read by the copies of item kb - 2
                if (kb >= 2) mbar_wait(bar_cp + 8 * (kb & 1), ((kb - 2) >> 1) & 1);
                stage_store<R1>(f, s1 + (kb & 1) * C::STG_DBL, i, y, ly);
                // generic-proxy stores, read next by tcgen05.cp (async proxy)
                asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
              }
            } else if (NBAR) {
              if (valid) phase1_collide<COLL, MON>(f, y, ly, thermal, r, own, acc);
              if (t > 0) asm volatile("bar.sync %0, %1;" ::"r"(5 + ((t - 1) & 1)), "r"(C::NT) : "memory");
              if (valid) phase1_store<R1>(f, s1, t, i, y, ly);
            } else if (valid) {
              phase1_update<COLL, R1, MON>(f, s1, t, i, y, ly, thermal, r, own, acc);
            }
          } else if (valid) {
            phase1<COLL, BUFD, RB, R1, MON>(s0, s1, buf, t, i, y, ly, thermal, r, own, acc);
          }
        }
        else if (NBAR && t > 0)  // t >= nload: no stores, but the hand-over protocol continues
          asm volatile("bar.sync %0, %1;" ::"r"(5 + ((t - 1) & 1)), "r"(C::NT) : "memory");
        if (DECOUPLE)  // item I written (every phase-1 thread arrives: release of its ring stores)
          asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(bar_full + 8 * (I & 1)) : "memory");
        if (NBAR && t + 1 < niter) asm volatile("bar.arrive %0, %1;" ::"r"(3 + (t & 1)), "r"(C::NT) : "memory");
      } else if (NBAR) {
        // phase 2 (named-barrier hand-over): wait until phase 1 wrote t - 1, gather, release
        if (t > 0) asm volatile("bar.sync %0, %1;" ::"r"(3 + ((t - 1) & 1)), "r"(C::NT) : "memory");
        const int i = p2row;
        const int y = ya + i;
        const bool valid = t >= 7 && i < HT && y < ly;
        double f[Q];
        if (t >= 7) phase2_gather<R1>(s1, t, valid ? i : 0, f);
        if (t + 1 < niter) asm volatile("bar.arrive %0, %1;" ::"r"(5 + (t & 1)), "r"(C::NT) : "memory");
        if (valid)
          phase2_update<COLL, MON>(f, B, g, y, xs - 7 + t, thermal, r, y >= own_lo && y < own_hi, acc, !peers);
      } else if (DECOUPLE) {
        // phase 2 (decoupled): wait for item I - 1, gather, release the slots
        if (t > 0) mbar_wait(bar_full + 8 * ((I - 1) & 1), ((I - 1) >> 1) & 1);
        const int i = p2row;
        const int y = ya + i;
        const bool valid = t >= 7 && i < HT && y < ly;
        double f[Q];
        if (t >= 7) phase2_gather<R1>(s1, t, valid ? i : 0, f);
        asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(bar_empty + 8 * (I & 1)) : "memory");
        if (valid)
          phase2_update<COLL, MON>(f, B, g, y, xs - 7 + t, thermal, r, y >= own_lo && y < own_hi, acc, !peers);
      } else if (SKEW) {
        // phase 2, offset against phase 1: collide right after the barrier
        // (only the 3 newest populations still to load), then gather the
        // next column's older populations after the stores
        const int i = p2row;
        const int y = ya + i;
        const bool valid = i < HT && y < ly;
        if (t >= 7) {
          phase2_gather_part<R1, true>(s1, t, valid ? i : 0, fk);
          if (valid)
            phase2_update<COLL, MON>(fk, B, g, y, xs - 7 + t, thermal, r, y >= own_lo && y < own_hi, acc, !peers);
        }
        if (t + 1 >= 7 && t + 1 < niter) phase2_gather_part<R1, false>(s1, t + 1, valid ? i : 0, fk);
      } else if (TMEM) {
        // phase 2 from the TMEM ring: wait for the copies of the newest item
        // it pulls (t - 1: the populations with cx = -3), read its own lane
        if (t >= 7) {
          const uint32_t k = kglob + (uint32_t)(t - 1);
          double f[Q];
          tmem_gather(tlane, t, f, [&] {
            mbar_wait(bar_cp + 8 * (k & 1), (k >> 1) & 1);
            asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
          });
          const int i = p2row;
          const int y = ya + i;
          if (i < HT && y < ly)
            phase2_update<COLL, MON>(f, B, g, y, xs - 7 + t, thermal, r, y >= own_lo && y < own_hi, acc, !peers);
        }
        asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
      } else if (t >= 7) {
        // phase 2: state n+2 at column c2 = xs - 7 + t, rows [ya, ya+HT)
        const int i = p2row;
        const int y = ya + i;
        if (i < HT && y < ly)
          phase2<COLL, R1, MON>(s1, B, g, t, i, y, xs - 7 + t, thermal, r, y >= own_lo && y < own_hi, acc,
                                !peers);
      }
    }
    if (DECOUPLE) {
      // wait for the last item's hand-over too, so every barrier phase is
      // observed before the next sweep re-arms it
      const uint32_t last = iglob + (uint32_t)niter - 1;
      mbar_wait((warp < C::NW1 ? bar_empty : bar_full) + 8 * (last & 1), (last >> 1) & 1);
    }
    kglob += (uint32_t)nload;
    iglob += (uint32_t)niter;
    __syncthreads();  // the next sweep refills every ring
  }
  if (LB_TB_PAIR && cl_armed) asm volatile("barrier.cluster.wait.aligned;" ::: "memory");
  if (TMEM) {  // every copy completed (phase 2 waited for the last one of each sweep)
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tbase));
  }
  if (inpull) {
    // publish this launch (the neighbours may now read our new state and
    // overwrite the columns we read): the last CTA to finish, after every
    // CTA's stores, raises this rank's counter (system-scope release)
    __syncthreads();
    if (tid == 0) {
      __threadfence_system();
      if (atomicAdd(pp.ctas_done, 1u) == gridDim.x - 1) {
        __threadfence_system();
        *pp.ctas_done = 0u;  // for the next launch (stream order)
        const unsigned long long v = *pp.my_done + 1;
        asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(pp.my_done), "l"(v) : "memory");
      }
    }
  }
#if LB_TB_CLOCK
  if (tid == 0 && blockIdx.x < 1024) {
    unsigned long long clk1;
    unsigned int smid;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(clk1));
    asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
    g_tb_clock[4 * blockIdx.x + 0] = clk0;
    g_tb_clock[4 * blockIdx.x + 1] = clk1;
    g_tb_clock[4 * blockIdx.x + 2] = smid;
    g_tb_clock[4 * blockIdx.x + 3] = ((unsigned long long)nsweeps << 32) | (unsigned)iglob;
  }
#endif
  if (MON) {
    // warp xor-tree, then the warps of each phase in order (deterministic)
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
#pragma unroll
      for (int k = 0; k < 4; ++k) acc[k] = __dadd_rn(acc[k], __shfl_xor_sync(0xffffffffu, acc[k], o));
      acc[4] = fmin(acc[4], __shfl_xor_sync(0xffffffffu, acc[4], o));
    }
    double* red = s1;  // the rings are free now
    if ((tid & 31) == 0)
#pragma unroll
      for (int k = 0; k < 5; ++k) red[warp * 5 + k] = acc[k];
    __syncthreads();
    if (tid < 2) {
      const int w0 = tid == 0 ? 0 : C::NW1, w1 = tid == 0 ? C::NW1 : C::NW;
      double v[5];
#pragma unroll
      for (int k = 0; k < 5; ++k) v[k] = red[w0 * 5 + k];
      for (int w = w0 + 1; w < w1; ++w) {
#pragma unroll
        for (int k = 0; k < 4; ++k) v[k] = __dadd_rn(v[k], red[w * 5 + k]);
        v[4] = fmin(v[4], red[w * 5 + 4]);
      }
      double* slot = mon + ((int64_t)(tid == 0 ? 0 : gridDim.x) + blockIdx.x) * 5;
#pragma unroll
      for (int k = 0; k < 5; ++k) slot[k] = v[k];
    }
  }
}

// TMA maps of one buffer: group windows (box {HT + 12, 3 | 5 | 7, 1}).
CUtensorMapL2promotion promo_enum(int promo) {
  return promo == 256 ? CU_TENSOR_MAP_L2_PROMOTION_L2_256B
         : promo == 128 ? CU_TENSOR_MAP_L2_PROMOTION_L2_128B
         : promo == 64  ? CU_TENSOR_MAP_L2_PROMOTION_L2_64B
                        : CU_TENSOR_MAP_L2_PROMOTION_NONE;
}

bool encode(CUtensorMap* m, double* base, const Geo& g, int box_rows, int box_pops, int promo) {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  if (!fn) {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
      return false;
    fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  }
  const cuuint64_t dims[3] = {(cuuint64_t)g.nyp, (cuuint64_t)Q, (cuuint64_t)g.nx};
  const cuuint64_t strides[2] = {(cuuint64_t)g.nyp * sizeof(double), (cuuint64_t)g.cs * sizeof(double)};
  const cuuint32_t box[3] = {(cuuint32_t)box_rows, (cuuint32_t)box_pops, 1};
  const cuuint32_t estr[3] = {1, 1, 1};
  return fn(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, base, dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
            CU_TENSOR_MAP_SWIZZLE_NONE, promo_enum(promo),
            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}



template <int COLL, bool MON>
cudaError_t launch_tb(const Geo& g, const TbMaps* t, int src_buf, double* B, const Relax& r, int grid,
                      int l2_dist, int thermal, int wall_w16, double* mon, int peers, const TbPeer* pull,
                      cudaStream_t s, bool pdl) {
  auto kern = k_step2_tb<COLL, TB_HT, TB_PF, MON>;
  static unsigned long long done_mask = 0;  // opt-in smem is a per-device attribute
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  if (dev >= 64 || !(done_mask >> dev & 1ull)) {
    e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)Cfg::SMEM);
    if (e != cudaSuccess) return e;
    if (dev < 64) done_mask |= 1ull << dev;
  }
  const bool inpull = peers && pull;
  if (peers && !(inpull ? t->direct : t->staged)) return cudaErrorInvalidValue;
  TbKMaps km;
  for (int c = 0; c < 3; ++c) {
    km.src[c] = t->load[src_buf][c];
    km.stL[c] = !peers ? t->load[src_buf][c] : inpull ? t->nb[0][src_buf][c] : t->st[0][c];
    km.stR[c] = !peers ? t->load[src_buf][c] : inpull ? t->nb[1][src_buf][c] : t->st[1][c];
  }
  const TbPeer pp = inpull ? *pull : TbPeer{};
#if LB_TB_PAIR
  if (tb_grid(g, grid) >= 2) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((unsigned)(tb_grid(g, grid) & ~1));
    cfg.blockDim = dim3(Cfg::NT);
    cfg.dynamicSmemBytes = Cfg::SMEM;
    cfg.stream = s;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = 2;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    const double* asrc = t->bufs[src_buf];
    const int nstr = (g.ly + TB_HT - 1) / TB_HT, ip = inpull ? 1 : 0;
    return cudaLaunchKernelEx(&cfg, kern, km, B, g, r, nstr, l2_dist, thermal, wall_w16, mon, peers, asrc, pp, ip);
  }
#endif
  if (pdl) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((unsigned)tb_grid(g, grid));
    cfg.blockDim = dim3(Cfg::NT);
    cfg.dynamicSmemBytes = Cfg::SMEM;
    cfg.stream = s;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    const double* asrc = t->bufs[src_buf];
    const int nstr = (g.ly + TB_HT - 1) / TB_HT, ip = inpull ? 1 : 0;
    return cudaLaunchKernelEx(&cfg, kern, km, B, g, r, nstr, l2_dist, thermal, wall_w16, mon, peers, asrc, pp, ip);
  }
  kern<<<tb_grid(g, grid), Cfg::NT, Cfg::SMEM, s>>>(km, B, g, r, (g.ly + TB_HT - 1) / TB_HT, l2_dist, thermal,
                                                    wall_w16, mon, peers, t->bufs[src_buf], pp,
                                                    inpull ? 1 : 0);
  return cudaGetLastError();
}

}  // namespace

bool tb_layout_ok(int ly) { return ly <= TB_HT || ly >= TB_HT + 6; }

int tb_strip_height() { return TB_HT; }

int tb_grid(const Geo& g, int grid) {
  const int64_t U = (int64_t)((g.ly + TB_HT - 1) / TB_HT) * g.lx;
  return (int)std::min<int64_t>(grid, U);
}

bool encode_buffers(TbMaps* t, const Geo& g) {
  for (int k = 0; k < 2; ++k)
  {
    for (int c = 0; c < 3; ++c)
      if (!encode(&t->load[k][c], t->bufs[k], g, Cfg::RB, CLS_N[c], t->promo)) return false;
  }
  return true;
}

TbMaps* tb_create(const Geo& g, double* buf0, double* buf1, int promo) {
  if (g.y0 % 2 || g.nyp % 2 || g.lx < 2 * H) return nullptr;
  auto* t = new TbMaps();
  t->promo = promo;
  t->bufs[0] = buf0;
  t->bufs[1] = buf1;
  if (!encode_buffers(t, g)) {
    delete t;
    return nullptr;
  }
  return t;
}

bool tb_set_promotion(TbMaps* t, const Geo& g, int promo) {
  t->promo = promo;
  if (!encode_buffers(t, g)) return false;
  if (t->direct && !tb_attach_peers(t, g, t->nbuf[0], t->nbuf[1])) return false;
  return !t->staged || tb_attach_staging(t, g, t->stage);
}

void tb_destroy(TbMaps* t) { delete t; }

cudaError_t tb_upload_constants(const double* k_bottom, const double* k_top, const double* ginv, cudaStream_t s) {
  cudaError_t e = cudaMemcpyToSymbolAsync(c_kwall, k_bottom, sizeof(double) * Q, 0, cudaMemcpyHostToDevice, s);
  if (e == cudaSuccess)
    e = cudaMemcpyToSymbolAsync(c_kwall, k_top, sizeof(double) * Q, sizeof(double) * Q, cudaMemcpyHostToDevice, s);
  if (e == cudaSuccess)
    e = cudaMemcpyToSymbolAsync(c_ginv, ginv, sizeof(double) * NGINV, 0, cudaMemcpyHostToDevice, s);
  if (e != cudaSuccess) return e;
  return cudaStreamSynchronize(s);
}

cudaError_t launch_step2_tb(const Geo& g, const TbMaps* t, int src_buf, double* B, int bc, int coll,
                            const Relax& r, int grid, int l2_dist, int wall_w16, double* mon, int peers,
                            const TbPeer* pull, cudaStream_t s, bool pdl) {
  if (bc != BC_THERMAL && bc != BC_ADIABATIC) return cudaErrorNotSupported;
  const int th = bc == BC_THERMAL;
  if (mon)
    return coll == COLL_REGULARIZED
               ? launch_tb<COLL_REGULARIZED, true>(g, t, src_buf, B, r, grid, l2_dist, th, wall_w16, mon, peers, pull, s, pdl)
               : launch_tb<COLL_BGK, true>(g, t, src_buf, B, r, grid, l2_dist, th, wall_w16, mon, peers, pull, s, pdl);
  return coll == COLL_REGULARIZED
             ? launch_tb<COLL_REGULARIZED, false>(g, t, src_buf, B, r, grid, l2_dist, th, wall_w16, mon, peers, pull, s, pdl)
             : launch_tb<COLL_BGK, false>(g, t, src_buf, B, r, grid, l2_dist, th, wall_w16, mon, peers, pull, s, pdl);
}

// ---- N > 1: staging of the neighbours' edge columns (peer memory -> local)
namespace {

// One thread waits until both neighbours completed as many launches as this
// rank (their current buffer then holds the same state as ours, and they are
// done reading our previous one); the copy kernel behind it on the stream then
// stages the left neighbour's internal columns [lx-3, lx+3) and the right
// one's [3, 9).  The wait is a one-block kernel of its own so that a waiting
// rank holds one SM slot, not a grid of spinning blocks (ranks sharing one GPU
// in tests would otherwise starve the neighbour they wait for).
__global__ void k_tb_wait(const unsigned long long* waitL, const unsigned long long* waitR,
                          const unsigned long long* my_done, unsigned int* status, unsigned long long timeout_ns) {
  if (threadIdx.x == 0) peer_wait(waitL, waitR, my_done, status, timeout_ns);
}

__global__ void __launch_bounds__(256) k_tb_pull(double2* __restrict__ stage, const double2* L, const double2* R,
                                                 int64_t lx, int64_t cs2) {
  const int64_t n = 6 * cs2;  // double2 per side
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < 2 * n; i += (int64_t)gridDim.x * blockDim.x)
    stage[i] = i < n ? __ldcg(L + (lx - 3) * cs2 + i) : __ldcg(R + 3 * cs2 + (i - n));
}

}  // namespace

bool tb_attach_staging(TbMaps* t, const Geo& g, double* stage) {
  Geo g6 = g;
  g6.nx = 6;  // 6 columns per side
  for (int c = 0; c < 3; ++c)
    if (!encode(&t->st[0][c], stage, g6, Cfg::RB, CLS_N[c], t->promo) ||
        !encode(&t->st[1][c], stage + 6 * g.cs, g6, Cfg::RB, CLS_N[c], t->promo))
      return false;
  t->stage = stage;
  t->staged = true;
  return true;
}

bool tb_attach_peers(TbMaps* t, const Geo& g, double* const left[2], double* const right[2]) {
  for (int k = 0; k < 2; ++k)
    for (int c = 0; c < 3; ++c)
      if (!encode(&t->nb[0][k][c], left[k], g, Cfg::RB, CLS_N[c], t->promo) ||
          !encode(&t->nb[1][k][c], right[k], g, Cfg::RB, CLS_N[c], t->promo))
        return t->direct = false;
  t->nbuf[0][0] = left[0];
  t->nbuf[0][1] = left[1];
  t->nbuf[1][0] = right[0];
  t->nbuf[1][1] = right[1];
  return t->direct = true;
}

cudaError_t launch_tb_pull(const Geo& g, double* stage, const double* left_A, const double* right_A,
                           const unsigned long long* waitL, const unsigned long long* waitR,
                           const unsigned long long* my_done, unsigned int* status, unsigned long long timeout_ns,
                           cudaStream_t s) {
  const int64_t cs2 = g.cs / 2;
  const int blocks = (int)std::min<int64_t>((12 * cs2 + 255) / 256, 148 * 4);
  k_tb_wait<<<1, 32, 0, s>>>(waitL, waitR, my_done, status, timeout_ns);
  k_tb_pull<<<blocks, 256, 0, s>>>(reinterpret_cast<double2*>(stage), reinterpret_cast<const double2*>(left_A),
                                   reinterpret_cast<const double2*>(right_A), g.lx, cs2);
  return cudaGetLastError();
}

}  // namespace lbk

#if LB_TB_CLOCK
extern "C" int lb_debug_tb_clock(unsigned long long* host, int n) {
  return (int)cudaMemcpyFromSymbol(host, g_tb_clock, sizeof(unsigned long long) * 4 * (n < 1024 ? n : 1024));
}
#endif
