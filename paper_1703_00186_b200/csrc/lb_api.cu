// lb_api.cu — the C ABI of include/lb.h: context, validation, the step
// scheduler (split / fused, bulk || exchange then borders), NCCL ring
// exchange, state I/O, invariants and per-kernel instrumentation.
#include "../../include/lb.h"
#include "lb_device.cuh"
#include "lb_internal.h"

#include <cuda_runtime.h>
#include <nccl.h>

#include <algorithm>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <new>
#include <string>
#include <vector>

using lbk::Cols;
using lbk::Geo;

namespace {

thread_local char g_err[512] = "";

int fail(int code, const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  std::vsnprintf(g_err, sizeof(g_err), fmt, ap);
  va_end(ap);
  return code;
}

#define CU(call)                                                              \
  do {                                                                        \
    cudaError_t e_ = (call);                                                  \
    if (e_ != cudaSuccess)                                                    \
      return fail(LB_ECUDA, "CUDA error %s at line %d", cudaGetErrorString(e_), __LINE__); \
  } while (0)

#define NC(call)                                                              \
  do {                                                                        \
    ncclResult_t r_ = (call);                                                 \
    if (r_ != ncclSuccess)                                                    \
      return fail(LB_ENCCL, "NCCL error %s at line %d", ncclGetErrorString(r_), __LINE__); \
  } while (0)

constexpr int Y0 = 16;  // internal row of physical row 0: 128-byte aligned

// Host copy of the velocity / weight tables, from the device header's
// constexpr arrays (one source of truth inside the library).
double host_weight(int l) { return lbd::SHELL_W(lbd::shell_of(l)); }

// K_wall,l(T_wall), App. B with the canonical expression tree of DESIGN.md
// §3 (reading G16/G25), evaluated on the host (compiled -ffp-contract=off).
void kwall(double t_wall, double* K) {
  const double a = lbd::A_SCALE;
  const double a2 = a * a;
  const double t = a2 * t_wall - 1.0;
  for (int l = 0; l < lbd::Q; ++l) {
    const double x2 = a2 * (double)(lbd::CX(l) * lbd::CX(l) + lbd::CY(l) * lbd::CY(l));
    K[l] = host_weight(l) * ((1.0 + (0.5 * t) * (x2 - 2.0)) + ((0.125 * t) * t) * ((x2 * x2 - 8.0 * x2) + 8.0));
  }
}

// Packed block inverse of the Gram matrix G_ab = sum_l w_l c_l^(alpha_a + alpha_b)
// of the 15 monomials |alpha| <= 4 (regularised collide, lb_kernels.cu).
// Each parity block is inverted by Gauss-Jordan with partial pivoting in long
// double.  Returns false if a block is singular.
bool gram_inverse(double* out) {
  for (int g = 0; g < 4; ++g) {
    const int first = lbd::GBLK_FIRST(g), n = lbd::GBLK_SIZE(g), off = lbd::GBLK_OFF(g);
    long double a[6][12];
    for (int i = 0; i < n; ++i)
      for (int j = 0; j < n; ++j) {
        long double s = 0.0L;
        const int p = lbd::MP(first + i) + lbd::MP(first + j), q = lbd::MQ(first + i) + lbd::MQ(first + j);
        for (int l = 0; l < lbd::Q; ++l) {
          long double t = host_weight(l);
          for (int k = 0; k < p; ++k) t *= lbd::CX(l);
          for (int k = 0; k < q; ++k) t *= lbd::CY(l);
          s += t;
        }
        a[i][j] = s;
        a[i][n + j] = (i == j) ? 1.0L : 0.0L;
      }
    for (int col = 0; col < n; ++col) {
      int piv = col;
      for (int r = col + 1; r < n; ++r)
        if (fabsl(a[r][col]) > fabsl(a[piv][col])) piv = r;
      if (fabsl(a[piv][col]) < 1e-30L) return false;
      for (int k = 0; k < 2 * n; ++k) std::swap(a[col][k], a[piv][k]);
      const long double d = a[col][col];
      for (int k = 0; k < 2 * n; ++k) a[col][k] /= d;
      for (int r = 0; r < n; ++r)
        if (r != col) {
          const long double m = a[r][col];
          for (int k = 0; k < 2 * n; ++k) a[r][k] -= m * a[col][k];
        }
    }
    for (int i = 0; i < n; ++i)
      for (int j = 0; j < n; ++j) out[off + i * n + j] = (double)a[i][n + j];
  }
  return true;
}

struct ProfEntry {
  int kernel;
  cudaEvent_t e0, e1;
  int64_t units;
};

}  // namespace

struct lb_ctx {
  lb_params p{};
  lb_layout L{};
  lb_xplan X{};
  Geo g{};
  int rank = 0, nranks = 1, left = 0, right = 0;
  double *A = nullptr, *B = nullptr;
  cudaStream_t s = nullptr;       // compute stream (caller's)
  cudaStream_t s_comm = nullptr;  // high-priority exchange stream
  cudaEvent_t ev_ready = nullptr, ev_comm = nullptr;
  ncclComm_t comm = nullptr;
  double* d_part = nullptr;   // invariants partials (+16 result doubles)
  double* h_pin = nullptr;    // pinned 8 doubles for results
  int phase = 0;              // 0 = step boundary, 1 = after propagate, 2 = after bc
  bool halo_fresh = false;    // A's x-halo columns are current (wrap or peer stores)
  int par = 0;                // A == caller's f_a if 0, f_b if 1 (toggles on swap)
  bool peers_on = false;      // peer-store exchange (lb_set_peers)
  lb_peers peers{};
  uint64_t peer_step = 0;     // steps completed since lb_set_peers
  bool mon_on = false;        // fused monitors (lb_monitor)
  bool mon_valid = false;     // d_mon describes the current A
  double* d_mon = nullptr;    // monitor_slots x 5 partials, then MON_REDUCE_MAX_BLOCKS x 5 (reduce scratch)
  unsigned int* d_ticket = nullptr;        // k_monitor_reduce arrival counter (kept zero)
  unsigned int* d_status = nullptr;        // peer watchdog flag (device)
  unsigned int* d_nonphys = nullptr;       // sticky: an invariants reduction saw NaN or rho <= 0 (device)
  unsigned long long peer_timeout_ns = 20000000000ull;
  lbk::TmaMaps* tma = nullptr;  // tensor maps of f_a / f_b (TMA propagate)
  int prop_impl = 0;            // LB_OPT_PROPAGATE_IMPL (1 = TMA when available)
  int fused_impl = 0;           // LB_OPT_FUSED_IMPL (1 = TMA-staged windows)
  bool graph_on = false;        // LB_OPT_CUDA_GRAPH: lb_step replays 2-step graphs
  lbk::TbMaps* tb = nullptr;    // tensor maps of the two-step kernel (lb_tb.cu)
  int tb_on = 0;                // LB_OPT_TEMPORAL: two steps per pass where possible
  int tb_grid = 0;              // LB_OPT_TB_GRID: CTAs of the two-step kernel (0 = SM count)
  int tb_l2 = 0;                // LB_OPT_TB_L2_PREFETCH: L2 prefetch distance in columns
  int tb_promo = 64;            // LB_OPT_TB_L2_PROMOTION: L2 promotion of its TMA loads (bytes)
  int tb_wall_w16 = 0;          // LB_OPT_TB_WALL_WEIGHT: wall-strip column cost x16 (work split; 0 = per collision)
  int tb_tail_w16 = 0;          // LB_OPT_TB_TAIL_WEIGHT: tail-region column cost x16 (aligned split; 0 = default)
  int tb_pdl = 1;               // LB_OPT_TB_PDL: programmatic dependent launch of the two-step kernel
  int tb_edge_pull = 1;         // LB_OPT_TB_EDGE_PULL: N > 1 two-step exchange inside the kernel (1) or k_tb_pull first (0)
  double* d_stage = nullptr;    // N > 1 two-step: the neighbours' 6 edge columns (2 x 6 x cs doubles)
  unsigned int* d_ctas = nullptr;  // N > 1 two-step, in-kernel exchange: finished-CTA count (kept zero)
  double* d_mon_tb = nullptr;   // two-step monitors: 2 x cap x 5 per-CTA partials, then reduce scratch
  int mon_tb_cap = 0;           // CTAs d_mon_tb holds partials for
  int mon_tb_G = 0;             // CTAs of the last two-step launch
  bool mon_tb = false;          // mon_valid refers to d_mon_tb (state n+1 and n+2 of the last launch)
  int sm_count = 148;
  cudaGraphExec_t gexec[2] = {nullptr, nullptr};  // keyed by the parity at graph start
  int gkey[2] = {-1, -1};       // configuration each graph was captured for
  int64_t glaunch[2] = {0, 0};  // kernel launches inside each graph
  double omega = 1.0;
  lbd::Relax relax{};
  int64_t launches = 0;
  // instrumentation
  bool prof = false;
  std::vector<std::string> knames;
  std::vector<ProfEntry> pending;
  std::vector<cudaEvent_t> evpool;
  std::vector<double> kms;
  std::vector<int64_t> kcount, kunits;
};

extern "C" {
static void graph_reset(lb_ctx* c);
}

namespace {

int kernel_id(lb_ctx* c, const char* name) {
  for (size_t i = 0; i < c->knames.size(); ++i)
    if (c->knames[i] == name) return (int)i;
  c->knames.emplace_back(name);
  c->kms.push_back(0.0);
  c->kcount.push_back(0);
  c->kunits.push_back(0);
  return (int)c->knames.size() - 1;
}

cudaEvent_t get_event(lb_ctx* c) {
  if (!c->evpool.empty()) {
    cudaEvent_t e = c->evpool.back();
    c->evpool.pop_back();
    return e;
  }
  cudaEvent_t e = nullptr;
  cudaEventCreate(&e);
  return e;
}

int harvest(lb_ctx* c) {
  for (auto& pe : c->pending) {
    CU(cudaEventSynchronize(pe.e1));
    float ms = 0.f;
    CU(cudaEventElapsedTime(&ms, pe.e0, pe.e1));
    c->kms[pe.kernel] += ms;
    c->kcount[pe.kernel] += 1;
    c->kunits[pe.kernel] += pe.units;
    c->evpool.push_back(pe.e0);
    c->evpool.push_back(pe.e1);
  }
  c->pending.clear();
  return LB_OK;
}

// Launch wrapper: counts launches and, when profiling, brackets the launch
// with events on the stream it is enqueued on.
template <class F>
int launch(lb_ctx* c, const char* name, cudaStream_t s, int64_t units, F&& f) {
  cudaEvent_t e0 = nullptr, e1 = nullptr;
  if (c->prof) {
    e0 = get_event(c);
    e1 = get_event(c);
    CU(cudaEventRecord(e0, s));
  }
  cudaError_t e = f();
  if (e != cudaSuccess) return fail(LB_ECUDA, "launch of %s failed: %s", name, cudaGetErrorString(e));
  c->launches++;
  if (c->prof) {
    CU(cudaEventRecord(e1, s));
    c->pending.push_back({kernel_id(c, name), e0, e1, units});
    if (c->pending.size() > 8192) return harvest(c);
  }
  return LB_OK;
}

#define TRY(x)                  \
  do {                          \
    int r_ = (x);               \
    if (r_ != LB_OK) return r_; \
  } while (0)

int validate(const lb_params* p, int rank, int nranks) {
  if (!p) return fail(LB_EINVAL, "params is NULL");
  if (nranks < 1 || rank < 0 || rank >= nranks) return fail(LB_EINVAL, "bad rank %d / nranks %d", rank, nranks);
  if (p->lx_total <= 0 || p->lx_total % nranks) return fail(LB_EINVAL, "lx_total %% nranks != 0");
  const int lx = p->lx_total / nranks;
  if (lx < (nranks == 1 ? 3 : 6)) return fail(LB_EINVAL, "per-rank lx = %d too small", lx);
  if (lx > 65535) return fail(LB_EINVAL, "per-rank lx = %d exceeds the 65535-column grid limit", lx);
  if (p->bc_y < 0 || p->bc_y > 2) return fail(LB_EINVAL, "bad bc_y");
  if (p->ly < (p->bc_y == LB_PERIODIC ? 3 : 6)) return fail(LB_EINVAL, "ly = %d too small", p->ly);
  if (p->mode < 0 || p->mode > 1) return fail(LB_EINVAL, "bad mode");
  if (p->collision < 0 || p->collision > 1) return fail(LB_EINVAL, "bad collision");
  if (!std::isfinite(p->gx) || !std::isfinite(p->gy)) return fail(LB_EINVAL, "gravity must be finite");
  if (!(p->tau > 0.0) || !(p->dt > 0.0)) return fail(LB_EINVAL, "tau and dt must be > 0");
  const double om = p->dt / p->tau;
  if (!(om > 0.0 && om <= 2.0)) return fail(LB_EINVAL, "dt/tau must be in (0, 2]");
  if (p->bc_y == LB_WALL_THERMAL && !(p->t_bottom > 0.0 && p->t_top > 0.0))
    return fail(LB_EINVAL, "wall temperatures must be > 0");
  const int64_t nyp = ((int64_t)Y0 + p->ly + 3 + 15) / 16 * 16;
  if (nyp * 37 * 3 > (int64_t)1 << 30) return fail(LB_EINVAL, "ly too large");
  return LB_OK;
}

void fill_layout(const lb_params* p, int rank, int nranks, lb_layout* L) {
  L->lx = p->lx_total / nranks;
  L->ly = p->ly;
  L->nx = L->lx + 2 * LB_HALO;
  L->y0 = Y0;
  L->nyp = (int)(((int64_t)Y0 + p->ly + 3 + 15) / 16 * 16);
  L->x0_global = rank * L->lx;
  L->col_stride = (int64_t)37 * L->nyp;
  L->elems = (int64_t)L->nx * L->col_stride;
  L->bytes = L->elems * 8;
  L->sites = (int64_t)L->lx * L->ly;
}

void fill_plan(const lb_layout& L, int rank, int nranks, lb_xplan* x) {
  x->left = (rank - 1 + nranks) % nranks;
  x->right = (rank + 1) % nranks;
  x->count = 3 * L.col_stride;
  x->recv_left_off = 0;
  x->recv_right_off = (int64_t)(L.lx + 3) * L.col_stride;
  x->send_right_off = (int64_t)L.lx * L.col_stride;
  x->send_left_off = (int64_t)3 * L.col_stride;
  x->bulk_x0 = LB_HALO + 3;
  x->bulk_x1 = std::max(LB_HALO + 3, LB_HALO + L.lx - 3);
  x->border_x0 = LB_HALO;
  x->border_x1 = LB_HALO + 3;
  x->border_x2 = LB_HALO + L.lx - 3;
  x->border_x3 = LB_HALO + L.lx;
}

Cols all_cols(const lb_ctx* c) { return Cols{LB_HALO, LB_HALO + c->g.lx, 0, 0}; }
Cols bulk_cols(const lb_ctx* c) { return Cols{c->X.bulk_x0, c->X.bulk_x1, 0, 0}; }
Cols border_cols(const lb_ctx* c) {
  return Cols{c->X.border_x0, c->X.border_x1, c->X.border_x2, c->X.border_x3};
}

// ---- exchange (§8a1) -------------------------------------------------------
// N = 1: local wrap kernel on stream s.  N > 1: grouped NCCL send/recv of the
// contiguous 3-column blocks on the ring.  For a pair of
// ranks the sends are posted (to right, to left) and the receives (from left,
// from right), so for N = 2 (left == right) the k-th send matches the k-th
// receive of the peer in the right halo.
int exchange_on(lb_ctx* c, cudaStream_t s) {
  const Geo& g = c->g;
  if (!c->comm) {
    if (c->nranks > 1) return fail(LB_ESTATE, "N > 1 without an NCCL communicator: use lb_set_peers");
    return launch(c, "k_pbc_wrap", s, 6LL * g.ly, [&] {
      return lbk::launch_pbc_wrap(g, c->A, c->p.bc_y, s);
    });
  }
  const lb_xplan& x = c->X;
  const size_t n = (size_t)x.count;
  NC(ncclGroupStart());
  NC(ncclRecv(c->A + x.recv_left_off, n, ncclDouble, x.left, c->comm, s));
  NC(ncclRecv(c->A + x.recv_right_off, n, ncclDouble, x.right, c->comm, s));
  NC(ncclSend(c->A + x.send_right_off, n, ncclDouble, x.right, c->comm, s));
  NC(ncclSend(c->A + x.send_left_off, n, ncclDouble, x.left, c->comm, s));
  NC(ncclGroupEnd());
  if (c->p.bc_y == LB_PERIODIC)
    TRY(launch(c, "k_ywrap", s, 0, [&] { return lbk::launch_ywrap(g, c->A, s); }));
  return LB_OK;
}

// part: "" (whole lattice), "_bulk" or "_border" (overlapped schedule) —
// instrumentation names only; all are launches of k_step_fused.
int fused(lb_ctx* c, Cols cols, const lbk::Halo& h = lbk::Halo(), const char* part = "") {
  static const char* names[2][3] = {{"k_step_fused", "k_step_fused_bulk", "k_step_fused_border"},
                                    {"k_step_fused_reg", "k_step_fused_reg_bulk", "k_step_fused_reg_border"}};
  const int pi = part[0] == 0 ? 0 : (part[1] == 'b' && part[2] == 'u' ? 1 : 2);
  return launch(c, names[c->p.collision ? 1 : 0][pi], c->s, (int64_t)cols.count() * c->g.ly, [&] {
    return lbk::launch_step_fused(c->g, c->A, c->B, c->p.bc_y, c->p.collision, c->relax, cols, h,
                                  c->mon_on ? c->d_mon : nullptr, c->s);
  });
}

void swap_ab(lb_ctx* c) {
  std::swap(c->A, c->B);
  c->par ^= 1;
}

// after a fused step: the monitor partials describe the new A iff monitors ran
void fused_step_done(lb_ctx* c) {
  c->mon_valid = c->mon_on;
  c->mon_tb = false;
}

// Peer mode (lb_set_peers): one fused kernel per step whose border blocks
// wait for both neighbours' previous step, pull their halo from this rank's A
// and store their results into the neighbours' next buffers; then a one-thread
// kernel publishes this rank's step counter.
int step_peer(lb_ctx* c) {
  const lb_peers& P = c->peers;
  if (!c->halo_fresh)
    TRY(launch(c, "k_peer_pull", c->s, 6LL * c->g.ly, [&] {
      lbk::Halo w;  // wait for the neighbours' previous launch (it may be a two-step one)
      w.waitL = reinterpret_cast<const unsigned long long*>(P.left_done);
      w.waitR = reinterpret_cast<const unsigned long long*>(P.right_done);
      w.my_done = reinterpret_cast<const unsigned long long*>(P.my_done);
      w.status = c->d_status;
      w.timeout_ns = c->peer_timeout_ns;
      return lbk::launch_peer_pull(c->g, c->A, P.left_buf[c->par], P.right_buf[c->par], w, c->s);
    }));
  lbk::Halo h;
  h.dstL = P.left_buf[c->par ^ 1];
  h.dstR = P.right_buf[c->par ^ 1];
  h.waitL = reinterpret_cast<const unsigned long long*>(P.left_done);
  h.waitR = reinterpret_cast<const unsigned long long*>(P.right_done);
  h.my_done = reinterpret_cast<const unsigned long long*>(P.my_done);
  h.status = c->d_status;
  h.timeout_ns = c->peer_timeout_ns;
  Cols cc = all_cols(c);
  cc.rev = c->par;  // alternate the column order: start on what the last step wrote (L2)
  TRY(fused(c, cc, h));
  c->peer_step += 1;
  TRY(launch(c, "k_signal", c->s, 0, [&] {
    return lbk::launch_signal(reinterpret_cast<unsigned long long*>(P.my_done), c->s);
  }));
  swap_ab(c);
  c->halo_fresh = true;
  fused_step_done(c);
  return LB_OK;
}

int step_once(lb_ctx* c) {
  if (c->p.mode == LB_MODE_SPLIT) {
    TRY(lb_exchange(c));
    TRY(lb_propagate(c));
    TRY(lb_bc(c));
    return lb_collide(c);
  }
  if (c->peers_on) return step_peer(c);
  // N = 1 without NCCL, walls: the fused kernel writes the next step's halo
  // columns itself (one launch per step); a separate wrap only when A's halo
  // is stale (after lb_set_state / lb_init_macro / a split step).
  if (c->nranks == 1 && !c->comm && c->p.bc_y != LB_PERIODIC) {
    if (!c->halo_fresh) TRY(exchange_on(c, c->s));
    lbk::Halo h;
    h.dstL = h.dstR = c->B;
    if (c->fused_impl == 1 && c->tma && !c->mon_on) {
      TRY(launch(c, c->p.collision ? "k_step_fused_reg_tma" : "k_step_fused_tma", c->s, c->L.sites, [&] {
        return lbk::launch_step_fused_tma(c->g, c->tma, c->par, c->A, c->B, c->p.bc_y, c->p.collision, c->relax,
                                          h, c->s);
      }));
    } else {
      Cols cc = all_cols(c);
      cc.rev = c->par;  // alternate the column order: start on what the last step wrote (L2)
      TRY(fused(c, cc, h));
    }
    swap_ab(c);
    c->halo_fresh = true;
    fused_step_done(c);
    return LB_OK;
  }
  // PERIODIC-Y: the y-halo wrap rewrites rows the bulk reads, so no overlap there
  const bool overlap = c->p.overlap && c->g.lx >= 6 && c->p.bc_y != LB_PERIODIC;
  c->halo_fresh = false;
  if (!overlap) {
    TRY(lb_exchange(c));
    TRY(fused(c, all_cols(c)));
  } else {
    // bulk || exchange, then borders.  A is read-only
    // during the step (G11), so the bulk and the exchange never race.
    CU(cudaEventRecord(c->ev_ready, c->s));
    CU(cudaStreamWaitEvent(c->s_comm, c->ev_ready, 0));
    TRY(exchange_on(c, c->s_comm));
    CU(cudaEventRecord(c->ev_comm, c->s_comm));
    TRY(fused(c, bulk_cols(c), lbk::Halo(), "_bulk"));
    CU(cudaStreamWaitEvent(c->s, c->ev_comm, 0));
    TRY(fused(c, border_cols(c), lbk::Halo(), "_border"));
  }
  swap_ab(c);
  fused_step_done(c);
  return LB_OK;
}

Geo make_geo(const lb_layout& L) {
  Geo g;
  g.lx = L.lx;
  g.ly = L.ly;
  g.nx = L.nx;
  g.nyp = L.nyp;
  g.y0 = L.y0;
  g.cs = L.col_stride;
  return g;
}

int check_boundary(lb_ctx* c, const char* what) {
  if (!c) return fail(LB_EINVAL, "ctx is NULL");
  if (c->phase != 0) return fail(LB_ESTATE, "%s is only allowed at a step boundary (phase %d)", what, c->phase);
  return LB_OK;
}

// Sticky non-physical flag (set by the invariants / monitor reductions on
// the device): LB_ENONPHYS once any reduction since the last state change saw
// a NaN or min rho <= 0.
int check_nonphys(lb_ctx* c) {
  unsigned int st = 0;
  CU(cudaMemcpy(&st, c->d_nonphys, sizeof(st), cudaMemcpyDeviceToHost));
  if (st) return fail(LB_ENONPHYS, "non-physical state: an invariants reduction saw NaN or rho <= 0");
  return LB_OK;
}

int reset_nonphys(lb_ctx* c) {
  CU(cudaMemsetAsync(c->d_nonphys, 0, sizeof(unsigned int), c->s));
  return LB_OK;
}

}  // namespace

// ============================================================================
extern "C" {

const char* lb_last_error(void) { return g_err; }

const char* lb_strerror(int s) {
  switch (s) {
    case LB_OK: return "ok";
    case LB_EINVAL: return "invalid argument";
    case LB_ESTATE: return "call out of order";
    case LB_ECUDA: return "CUDA error";
    case LB_ENCCL: return "NCCL error";
    case LB_ENONPHYS: return "non-physical state (NaN or rho <= 0)";
    case LB_ENOMEM: return "out of memory";
    case LB_EPEER: return "peer exchange timed out";
    default: return "unknown status";
  }
}

int lb_query_layout(const lb_params* p, int rank, int nranks, lb_layout* out) {
  TRY(validate(p, rank, nranks));
  if (!out) return fail(LB_EINVAL, "out is NULL");
  fill_layout(p, rank, nranks, out);
  return LB_OK;
}

int lb_exchange_plan(const lb_params* p, int rank, int nranks, lb_xplan* out) {
  TRY(validate(p, rank, nranks));
  if (!out) return fail(LB_EINVAL, "out is NULL");
  lb_layout L;
  fill_layout(p, rank, nranks, &L);
  fill_plan(L, rank, nranks, out);
  return LB_OK;
}

int lb_constants(int* c, double* w, double* a, double* t0) {
  for (int l = 0; l < lbd::Q; ++l) {
    if (c) {
      c[2 * l] = lbd::CX(l);
      c[2 * l + 1] = lbd::CY(l);
    }
    if (w) w[l] = host_weight(l);
  }
  if (a) *a = lbd::A_SCALE;
  if (t0) *t0 = 1.0 / (lbd::A_SCALE * lbd::A_SCALE);
  return LB_OK;
}

int lb_kwall(double t_wall, double* K) {
  if (!K) return fail(LB_EINVAL, "K is NULL");
  kwall(t_wall, K);
  return LB_OK;
}

int lb_nccl_unique_id(unsigned char* out) {
  if (!out) return fail(LB_EINVAL, "out is NULL");
  ncclUniqueId id;
  NC(ncclGetUniqueId(&id));
  static_assert(sizeof(id) == 128, "ncclUniqueId size");
  std::memcpy(out, &id, 128);
  return LB_OK;
}

int lb_init(const lb_params* p, const lb_dist* d, double* f_a, double* f_b, void* stream,
            lb_ctx** out) {
  if (!out) return fail(LB_EINVAL, "out is NULL");
  *out = nullptr;
  const int rank = d ? d->rank : 0, nranks = d ? d->nranks : 1;
  TRY(validate(p, rank, nranks));
  // overlap (§8a6) only where the bulk || exchange schedule exists:
  // an NCCL exchange (or, N > 1, the peer stores, which always overlap inside
  // the kernel), fused mode, walls in Y — anywhere else it would be a silent no-op
  if (p->overlap) {
    if (p->mode != LB_MODE_FUSED) return fail(LB_EINVAL, "overlap needs fused mode");
    if (p->bc_y == LB_PERIODIC) return fail(LB_EINVAL, "overlap needs walls in Y (periodic Y wraps rows the bulk reads)");
    if (nranks == 1 && !(d && d->nccl_id))
      return fail(LB_EINVAL, "overlap at N = 1 needs an NCCL communicator (the local wrap has no exchange to overlap)");
    if (p->lx_total / nranks < 6) return fail(LB_EINVAL, "overlap needs lx >= 6 (3+3 border columns)");
  }
  if (!f_a || !f_b || f_a == f_b) return fail(LB_EINVAL, "need two distinct device buffers");
  if (((uintptr_t)f_a | (uintptr_t)f_b) & 15) return fail(LB_EINVAL, "buffers must be 16-byte aligned");
  lb_ctx* c = new (std::nothrow) lb_ctx();
  if (!c) return fail(LB_ENOMEM, "host allocation failed");
  c->p = *p;
  fill_layout(p, rank, nranks, &c->L);
  c->g = make_geo(c->L);
  fill_plan(c->L, rank, nranks, &c->X);
  c->rank = rank;
  c->nranks = nranks;
  c->left = (rank - 1 + nranks) % nranks;
  c->right = (rank + 1) % nranks;
  c->A = f_a;
  c->B = f_b;
  c->s = (cudaStream_t)stream;
  c->omega = p->dt / p->tau;
  {
    // body force (reading G7b): u_eq = u + g/omega, T_eq = T + (1/omega)(1 - 1/omega)|g|^2/D
    const double it = 1.0 / c->omega;
    c->relax.omega = c->omega;
    c->relax.one_m_omega = 1.0 - c->omega;
    c->relax.tgx = it * p->gx;
    c->relax.tgy = it * p->gy;
    c->relax.dT = it * (1.0 - it) * (p->gx * p->gx + p->gy * p->gy) / 2.0;
  }
  auto bail = [&](int code) {
    lb_destroy(c);
    return code;
  };
  int lo = 0, hi = 0;
  if (cudaDeviceGetStreamPriorityRange(&lo, &hi) != cudaSuccess ||
      cudaStreamCreateWithPriority(&c->s_comm, cudaStreamNonBlocking, hi) != cudaSuccess ||
      cudaEventCreateWithFlags(&c->ev_ready, cudaEventDisableTiming) != cudaSuccess ||
      cudaEventCreateWithFlags(&c->ev_comm, cudaEventDisableTiming) != cudaSuccess)
    return bail(fail(LB_ECUDA, "stream/event creation failed"));
  const size_t npart = lbk::invariants_scratch(c->g) + 16;  // + result space (up to 2 x 5 doubles)
  if (cudaMalloc(&c->d_part, npart * sizeof(double)) != cudaSuccess)
    return bail(fail(LB_ENOMEM, "device scratch allocation failed"));
  if (cudaMallocHost(&c->h_pin, 16 * sizeof(double)) != cudaSuccess)
    return bail(fail(LB_ENOMEM, "pinned allocation failed"));
  if (cudaMalloc(&c->d_nonphys, sizeof(unsigned int)) != cudaSuccess ||
      cudaMemsetAsync(c->d_nonphys, 0, sizeof(unsigned int), c->s) != cudaSuccess)
    return bail(fail(LB_ENOMEM, "flag allocation failed"));
  if (cudaMemsetAsync(c->A, 0, c->L.bytes, c->s) != cudaSuccess ||
      cudaMemsetAsync(c->B, 0, c->L.bytes, c->s) != cudaSuccess)
    return bail(fail(LB_ECUDA, "zero-fill failed: %s", cudaGetErrorString(cudaGetLastError())));
  double kb[lbd::Q], kt[lbd::Q];
  kwall(p->t_bottom, kb);
  kwall(p->t_top, kt);
  if (lbk::upload_kwall(kb, kt, c->s) != cudaSuccess)
    return bail(fail(LB_ECUDA, "constant upload failed"));
  double ginv[lbd::NGINV];
  if (!gram_inverse(ginv)) return bail(fail(LB_EINVAL, "singular Gram matrix"));
  if (lbk::upload_ginv(ginv, c->s) != cudaSuccess || lbk::tb_upload_constants(kb, kt, ginv, c->s) != cudaSuccess)
    return bail(fail(LB_ECUDA, "constant upload failed"));
  {
    int dev = 0;
    if (cudaGetDevice(&dev) == cudaSuccess)
      cudaDeviceGetAttribute(&c->sm_count, cudaDevAttrMultiProcessorCount, dev);
  }
  // TMA-staged propagate is the default when the tensor maps encode (B200:
  // 6.62 vs 6.54 TB/s for the register gather); otherwise the gather
  c->tma = lbk::tma_create(c->g, c->A, c->B);
  c->prop_impl = c->tma ? 1 : 0;
  // Two steps per pass (lb_tb.cu) is the default where it applies (N = 1,
  // walls, fused mode; lb_step falls back to one fused step otherwise): it is
  // bit-identical to two fused steps and 1.35x faster at 1920x2048.
  // (N > 1: once lb_set_peers provides the neighbours' buffers for the staging)
  if (p->bc_y != LB_PERIODIC && p->mode == LB_MODE_FUSED) {
    c->tb = lbk::tb_create(c->g, c->A, c->B, c->tb_promo);
    c->tb_on = c->tb != nullptr;
  }
  if (d && d->nccl_id) {
    ncclUniqueId id;
    std::memcpy(&id, d->nccl_id, 128);
    ncclResult_t r = ncclCommInitRank(&c->comm, nranks, id, rank);
    if (r != ncclSuccess) return bail(fail(LB_ENCCL, "ncclCommInitRank: %s", ncclGetErrorString(r)));
  }
  if (cudaStreamSynchronize(c->s) != cudaSuccess)
    return bail(fail(LB_ECUDA, "init sync failed: %s", cudaGetErrorString(cudaGetLastError())));
  *out = c;
  return LB_OK;
}

void lb_destroy(lb_ctx* c) {
  if (!c) return;
  if (c->s) cudaStreamSynchronize(c->s);
  if (c->s_comm) cudaStreamSynchronize(c->s_comm);
  for (auto& pe : c->pending) {
    cudaEventDestroy(pe.e0);
    cudaEventDestroy(pe.e1);
  }
  for (auto e : c->evpool) cudaEventDestroy(e);
  if (c->comm) ncclCommDestroy(c->comm);
  if (c->ev_ready) cudaEventDestroy(c->ev_ready);
  if (c->ev_comm) cudaEventDestroy(c->ev_comm);
  if (c->s_comm) cudaStreamDestroy(c->s_comm);
  if (c->d_part) cudaFree(c->d_part);
  if (c->d_mon) cudaFree(c->d_mon);
  if (c->d_mon_tb) cudaFree(c->d_mon_tb);
  if (c->d_stage) cudaFree(c->d_stage);
  if (c->d_ctas) cudaFree(c->d_ctas);
  if (c->d_ticket) cudaFree(c->d_ticket);
  if (c->d_status) cudaFree(c->d_status);
  if (c->d_nonphys) cudaFree(c->d_nonphys);
  if (c->tma) lbk::tma_destroy(c->tma);
  if (c->tb) lbk::tb_destroy(c->tb);
  graph_reset(c);
  if (c->h_pin) cudaFreeHost(c->h_pin);
  delete c;
}

int lb_get_layout(const lb_ctx* c, lb_layout* out) {
  if (!c || !out) return fail(LB_EINVAL, "NULL argument");
  *out = c->L;
  return LB_OK;
}

int lb_set_stream(lb_ctx* c, void* stream) {
  if (!c) return fail(LB_EINVAL, "ctx is NULL");
  c->s = (cudaStream_t)stream;
  return LB_OK;
}

int lb_init_macro(lb_ctx* c, const double* rho, const double* ux, const double* uy,
                  const double* T, int on_device) {
  TRY(check_boundary(c, "lb_init_macro"));
  if (!rho || !ux || !uy || !T) return fail(LB_EINVAL, "NULL field");
  const int64_t n = c->L.sites;
  const double* src[4] = {rho, ux, uy, T};
  const double* dev[4];
  for (int k = 0; k < 4; ++k) {
    if (on_device) {
      dev[k] = src[k];
    } else {
      double* dst = c->B + k * n;  // B is scratch at a step boundary
      CU(cudaMemcpyAsync(dst, src[k], n * sizeof(double), cudaMemcpyHostToDevice, c->s));
      dev[k] = dst;
    }
  }
  c->halo_fresh = false;
  c->mon_valid = false;
  TRY(reset_nonphys(c));
  TRY(launch(c, "k_init_macro", c->s, n, [&] {
    return lbk::launch_init_macro(c->g, c->A, dev[0], dev[1], dev[2], dev[3], c->s);
  }));
  if (!on_device) CU(cudaMemsetAsync(c->B, 0, c->L.bytes, c->s));
  return LB_OK;
}

int lb_init_rt(lb_ctx* c, const double* eps, double t_ref, double amp, double width) {
  TRY(check_boundary(c, "lb_init_rt"));
  if (!eps) return fail(LB_EINVAL, "NULL eps");
  if (!(t_ref > 0.0) || !(width > 0.0) || !(std::fabs(amp) < 1.0))
    return fail(LB_EINVAL, "need t_ref > 0, width > 0, |amp| < 1 (T > 0)");
  const int lx_total = c->p.lx_total;
  CU(cudaMemcpyAsync(c->B, eps, lx_total * sizeof(double), cudaMemcpyDefault, c->s));
  c->halo_fresh = false;
  c->mon_valid = false;
  TRY(reset_nonphys(c));
  TRY(launch(c, "k_init_rt", c->s, c->L.sites, [&] {
    return lbk::launch_init_rt(c->g, c->A, c->B, lx_total, c->rank * c->g.lx, t_ref, amp, width, c->s);
  }));
  CU(cudaMemsetAsync(c->B, 0, c->L.bytes, c->s));
  return LB_OK;
}

int lb_set_state(lb_ctx* c, const double* canon, int on_device) {
  TRY(check_boundary(c, "lb_set_state"));
  if (!canon) return fail(LB_EINVAL, "NULL state");
  const int64_t n = (int64_t)37 * c->L.sites;
  const double* src = canon;
  if (!on_device) {
    CU(cudaMemcpyAsync(c->B, canon, n * sizeof(double), cudaMemcpyHostToDevice, c->s));
    src = c->B;
  }
  c->halo_fresh = false;
  c->mon_valid = false;
  TRY(reset_nonphys(c));
  TRY(launch(c, "k_canon_to_internal", c->s, c->L.sites, [&] {
    return lbk::launch_canon_to_internal(c->g, src, c->A, c->s);
  }));
  if (!on_device) CU(cudaMemsetAsync(c->B, 0, c->L.bytes, c->s));
  return LB_OK;
}

int lb_exchange(lb_ctx* c) {
  TRY(check_boundary(c, "lb_exchange"));
  if (!c->comm) {
    TRY(exchange_on(c, c->s));
    c->halo_fresh = true;
    return LB_OK;
  }
  CU(cudaEventRecord(c->ev_ready, c->s));
  CU(cudaStreamWaitEvent(c->s_comm, c->ev_ready, 0));
  TRY(exchange_on(c, c->s_comm));
  CU(cudaEventRecord(c->ev_comm, c->s_comm));
  CU(cudaStreamWaitEvent(c->s, c->ev_comm, 0));
  return LB_OK;
}

int lb_propagate(lb_ctx* c) {
  TRY(check_boundary(c, "lb_propagate"));
  if (c->prop_impl == 1)
    TRY(launch(c, "k_propagate_tma", c->s, c->L.sites, [&] {
      return lbk::launch_propagate_tma(c->g, c->tma, c->par, c->B, c->s);
    }));
  else
    TRY(launch(c, "k_propagate", c->s, c->L.sites, [&] {
      return lbk::launch_propagate(c->g, c->A, c->B, c->s);
    }));
  c->phase = 1;
  return LB_OK;
}

int lb_bc(lb_ctx* c) {
  if (!c) return fail(LB_EINVAL, "ctx is NULL");
  if (c->phase != 1) return fail(LB_ESTATE, "lb_bc must follow lb_propagate");
  if (c->p.bc_y != LB_PERIODIC)
    TRY(launch(c, "k_bc", c->s, 6LL * c->g.lx, [&] {
      return lbk::launch_bc(c->g, c->A, c->B, c->p.bc_y, c->s);
    }));
  c->phase = 2;
  return LB_OK;
}

int lb_collide(lb_ctx* c) {
  if (!c) return fail(LB_EINVAL, "ctx is NULL");
  if (c->phase != 2 && !(c->phase == 1 && c->p.bc_y == LB_PERIODIC))
    return fail(LB_ESTATE, "lb_collide must follow lb_bc");
  TRY(launch(c, c->p.collision ? "k_collide_reg" : "k_collide", c->s, c->L.sites, [&] {
    return lbk::launch_collide(c->g, c->B, c->relax, c->p.collision, c->s);
  }));
  swap_ab(c);
  c->phase = 0;
  c->halo_fresh = false;
  c->mon_valid = false;
  return LB_OK;
}

// CUDA-graph stepping (LB_OPT_CUDA_GRAPH): in the steady state of the fused
// N = 1 wrap path and of the peer path every step issues the same launches
// with the same parameters (the peer wait target is read on the device), and
// two steps return A/B to their places — so two steps are captured once per
// starting parity and replayed with one cudaGraphLaunch.
static int graph_config(const lb_ctx* c) {
  return c->fused_impl | (c->mon_on ? 2 : 0) | (c->peers_on ? 4 : 0);
}

static bool graphable(const lb_ctx* c) {
  return c->graph_on && !c->prof && c->s != nullptr && c->p.mode == LB_MODE_FUSED && c->halo_fresh &&
         (c->peers_on || (c->nranks == 1 && !c->comm && c->p.bc_y != LB_PERIODIC));
}

static void graph_reset(lb_ctx* c) {
  for (int k = 0; k < 2; ++k) {
    if (c->gexec[k]) cudaGraphExecDestroy(c->gexec[k]);
    c->gexec[k] = nullptr;
    c->gkey[k] = -1;
  }
}

static int graph_two_steps(lb_ctx* c) {
  const int par = c->par, key = graph_config(c);
  if (!c->gexec[par] || c->gkey[par] != key) {
    if (c->gexec[par]) cudaGraphExecDestroy(c->gexec[par]);
    c->gexec[par] = nullptr;
    const int64_t l0 = c->launches;
    CU(cudaStreamBeginCapture(c->s, cudaStreamCaptureModeThreadLocal));
    int r = step_once(c);
    if (r == LB_OK) r = step_once(c);
    cudaGraph_t graph = nullptr;
    const cudaError_t e = cudaStreamEndCapture(c->s, &graph);
    c->glaunch[par] = c->launches - l0;
    c->launches = l0;  // captured, not executed
    if (r != LB_OK) return r;
    if (e != cudaSuccess) return fail(LB_ECUDA, "graph capture failed: %s", cudaGetErrorString(e));
    const cudaError_t ei = cudaGraphInstantiate(&c->gexec[par], graph, 0);
    cudaGraphDestroy(graph);
    if (ei != cudaSuccess) return fail(LB_ECUDA, "graph instantiation failed: %s", cudaGetErrorString(ei));
    c->gkey[par] = key;
  } else {
    // host-side effects of two steps (the capture above performed them)
    swap_ab(c);
    swap_ab(c);
    fused_step_done(c);
  }
  CU(cudaGraphLaunch(c->gexec[par], c->s));
  c->launches += c->glaunch[par];
  return LB_OK;
}

// Two steps in one pass (lb_tb.cu): N = 1 without NCCL or peers, or N > 1 in
// peer mode (staged edge columns); walls, fused mode, with or without
// monitors.  Bit-identical to two fused steps.
static bool tb_usable(const lb_ctx* c) {
  const bool alone = c->nranks == 1 && !c->comm && !c->peers_on;  // N = 1 periodic wrap
  const bool staged = c->peers_on && c->tb && c->tb->staged;       // N > 1 peer mode
  return c->tb_on && c->tb && (alone || staged) && c->p.mode == LB_MODE_FUSED && c->p.bc_y != LB_PERIODIC &&
         lbk::tb_layout_ok(c->g.ly);
}

// Cost of a wall-strip column relative to an interior one (x16) in the
// two-step kernel's work split: measured per-CTA times (tools/tb_clock.py,
// 1920x2048) give 1.17 (BGK) and 1.25 (regularised) per iteration, and a
// sweep of the BGK weight 17..21 peaks at 19.
// Both collides use the time-aligned split (LB_OPT_TB_TAIL_WEIGHT != 1),
// where a wall-strip column costs ~1.3x an interior one (per-CTA clocks, BGK:
// 1.92 vs 1.50 us per iteration) and weight sweeps (tools/gpu_job_r02_wt.sh,
// gpu_job_r02_wtreg.sh) peak at wall 21 / tail 17 (x1/16) for both; with the
// contiguous split 19 (BGK) and 20 (regularised) balance best.
static bool tb_aligned(const lb_ctx* c) { return c->tb_tail_w16 != 1; }
static int tb_wall_weight(const lb_ctx* c) {
  if (c->tb_wall_w16 > 0) return c->tb_wall_w16;
  return tb_aligned(c) ? 21 : c->p.collision == LB_COLLIDE_REGULARIZED ? 20 : 19;
}
// The kernel's split parameter: wall weight | tail weight << 16 (both x16;
// tail 0: the contiguous split).
// Default tail weight: 17 when each strip has several main-region CTAs
// (R >= 2: few tail CTAs, each sweeping several short unaligned segments —
// 1920x2048: R = 7, tail 17 beats 16 by 4 %), 16 when R = 1 (many tail CTAs
// on long segments — 8192x8192 and 4096x8192: R = 1, tail 16 beats 17 by
// 1.9 % / 1.1 %; tools/gpu_job_r02_wt_big.sh).
static int tb_split_weights(const lb_ctx* c, int G) {
  const int ns = (c->g.ly + lbk::tb_strip_height() - 1) / lbk::tb_strip_height();
  const int R = ns > 0 ? G / ns : 0;
  const int tail = !tb_aligned(c) ? 0 : c->tb_tail_w16 >= 16 ? c->tb_tail_w16 : R >= 2 ? 17 : 16;
  return tb_wall_weight(c) | (tail << 16);
}

static int step_tb(lb_ctx* c) {
  const int grid = c->tb_grid > 0 ? c->tb_grid : c->sm_count;
  const int G = lbk::tb_grid(c->g, grid);
  if (c->mon_on && c->mon_tb_cap < G) {  // per-CTA partials of both states + reduce scratch
    if (c->d_mon_tb) cudaFree(c->d_mon_tb);
    c->d_mon_tb = nullptr;
    c->mon_tb_cap = 0;
    if (cudaMalloc(&c->d_mon_tb, ((size_t)2 * G + lbk::MON_REDUCE_MAX_BLOCKS) * 5 * sizeof(double)) != cudaSuccess)
      return fail(LB_ENOMEM, "monitor allocation failed");
    c->mon_tb_cap = G;
  }
  double* mon = c->mon_on ? c->d_mon_tb : nullptr;
  const lb_peers& P = c->peers;
  const bool peers = c->peers_on;
  lbk::TbPeer pull;
  const bool inpull = peers && c->tb_edge_pull && c->tb->direct;
  if (inpull) {  // N > 1 default: only the edge CTAs wait; the kernel reads the neighbours' buffers and signals
    pull.waitL = reinterpret_cast<const unsigned long long*>(P.left_done);
    pull.waitR = reinterpret_cast<const unsigned long long*>(P.right_done);
    pull.my_done = reinterpret_cast<unsigned long long*>(P.my_done);
    pull.ctas_done = c->d_ctas;
    pull.status = c->d_status;
    pull.timeout_ns = c->peer_timeout_ns;
  } else if (peers) {  // LB_OPT_TB_EDGE_PULL = 0: wait for both neighbours, copy their 6 edge columns, then the kernel
    TRY(launch(c, "k_tb_pull", c->s, 12LL * c->g.ly, [&] {
      return lbk::launch_tb_pull(c->g, c->d_stage, P.left_buf[c->par], P.right_buf[c->par],
                                 reinterpret_cast<const unsigned long long*>(P.left_done),
                                 reinterpret_cast<const unsigned long long*>(P.right_done),
                                 reinterpret_cast<const unsigned long long*>(P.my_done), c->d_status,
                                 c->peer_timeout_ns, c->s);
    }));
    c->launches += 1;  // two kernels: k_tb_wait (one block) + the k_tb_pull copy
  }
  TRY(launch(c, c->p.collision ? "k_step2_tb_reg" : "k_step2_tb", c->s, 2 * c->L.sites, [&] {
    return lbk::launch_step2_tb(c->g, c->tb, c->par, c->B, c->p.bc_y, c->p.collision, c->relax, grid, c->tb_l2,
                                tb_split_weights(c, G), mon, peers ? 1 : 0, inpull ? &pull : nullptr, c->s,
                                c->tb_pdl != 0 && !peers);  // (peers: ranks sharing a GPU in tests must not
                                                            // park next-launch CTAs on SMs a neighbour needs)
  }));
  if (peers) {  // publish: this launch is complete (the neighbours may now read our new state)
    c->peer_step += 1;
    if (!inpull)  // (the in-kernel exchange publishes from the kernel's last CTA)
      TRY(launch(c, "k_signal", c->s, 0, [&] {
        return lbk::launch_signal(reinterpret_cast<unsigned long long*>(P.my_done), c->s);
      }));
  }
  swap_ab(c);  // B held state n + 2: it becomes A
  // N = 1: the kernel stored the border columns into B's halo; N > 1: halos
  // are not maintained by the two-step path (a following one-step pulls them)
  c->halo_fresh = !peers;
  fused_step_done(c);
  c->mon_tb = c->mon_on;
  c->mon_tb_G = G;
  return LB_OK;
}

int lb_step(lb_ctx* c, int nsteps) {
  TRY(check_boundary(c, "lb_step"));
  if (nsteps < 0) return fail(LB_EINVAL, "nsteps < 0");
  int k = 0;
  while (k < nsteps) {
    if (nsteps - k >= 2 && tb_usable(c)) {
      TRY(step_tb(c));
      k += 2;
    } else if (nsteps - k >= 2 && graphable(c)) {
      TRY(graph_two_steps(c));
      k += 2;
    } else {
      TRY(step_once(c));
      k += 1;
    }
  }
  return LB_OK;
}

// Peer-mode watchdog (step_peer): LB_EPEER if a border block gave up waiting.
static int check_peer_status(lb_ctx* c) {
  if (!c->d_status) return LB_OK;
  unsigned int st = 0;
  CU(cudaMemcpy(&st, c->d_status, sizeof(st), cudaMemcpyDeviceToHost));
  if (st) return fail(LB_EPEER, "peer exchange timed out: a neighbour did not complete its step");
  return LB_OK;
}

int lb_sync(lb_ctx* c) {
  if (!c) return fail(LB_EINVAL, "ctx is NULL");
  CU(cudaStreamSynchronize(c->s));
  CU(cudaStreamSynchronize(c->s_comm));
  TRY(check_peer_status(c));
  return check_nonphys(c);
}

int lb_gather(lb_ctx* c, double* host_out, int root) {
  TRY(check_boundary(c, "lb_gather"));
  if (root < 0 || root >= c->nranks) return fail(LB_EINVAL, "bad root %d", root);
  if (c->rank == root && !host_out) return fail(LB_EINVAL, "host_out is NULL on root");
  if (c->nranks > 1 && !c->comm) return fail(LB_ESTATE, "lb_gather at N > 1 needs an NCCL communicator");
  const Geo& g = c->g;
  const int64_t blk = (int64_t)g.lx * g.ly;  // one plane of one rank
  const size_t dpitch = (size_t)c->p.lx_total * g.ly * sizeof(double);
  TRY(launch(c, "k_internal_to_canon", c->s, c->L.sites, [&] {
    return lbk::launch_internal_to_canon(g, c->A, c->B, c->s);
  }));
  if (c->rank == root) {
    CU(cudaMemcpy2DAsync(host_out + (int64_t)c->rank * blk, dpitch, c->B, blk * sizeof(double),
                         blk * sizeof(double), 37, cudaMemcpyDeviceToHost, c->s));
    CU(cudaStreamSynchronize(c->s));
    for (int r = 0; r < c->nranks; ++r) {
      if (r == root) continue;
      NC(ncclRecv(c->B, (size_t)37 * blk, ncclDouble, r, c->comm, c->s));
      CU(cudaMemcpy2DAsync(host_out + (int64_t)r * blk, dpitch, c->B, blk * sizeof(double),
                           blk * sizeof(double), 37, cudaMemcpyDeviceToHost, c->s));
      CU(cudaStreamSynchronize(c->s));
    }
  } else {
    NC(ncclSend(c->B, (size_t)37 * blk, ncclDouble, root, c->comm, c->s));
  }
  CU(cudaMemsetAsync(c->B, 0, c->L.bytes, c->s));  // restore zero halo rows (G10)
  CU(cudaStreamSynchronize(c->s));
  return LB_OK;
}

int lb_peek_cols(lb_ctx* c, int which, int x0, int ncols, double* host_out) {
  if (!c || !host_out || (which != 0 && which != 1)) return fail(LB_EINVAL, "bad argument");
  const Geo& g = c->g;
  if (x0 < 0 || ncols < 1 || x0 + ncols > g.lx) return fail(LB_EINVAL, "column range out of bounds");
  std::vector<double> buf;
  try {
    buf.resize((size_t)ncols * g.cs);
  } catch (...) {
    return fail(LB_ENOMEM, "host staging allocation failed");
  }
  const double* src = (which ? c->B : c->A) + (int64_t)(x0 + 3) * g.cs;  // contiguous column block
  CU(cudaStreamSynchronize(c->s_comm));
  CU(cudaMemcpyAsync(buf.data(), src, buf.size() * sizeof(double), cudaMemcpyDeviceToHost, c->s));
  CU(cudaStreamSynchronize(c->s));
  for (int l = 0; l < 37; ++l)
    for (int x = 0; x < ncols; ++x)
      std::memcpy(host_out + ((int64_t)l * ncols + x) * g.ly,
                  buf.data() + (int64_t)x * g.cs + (int64_t)l * g.nyp + g.y0, sizeof(double) * g.ly);
  return LB_OK;
}

int lb_peek(lb_ctx* c, int which, double* host_out) {
  if (!c) return fail(LB_EINVAL, "ctx is NULL");
  return lb_peek_cols(c, which, 0, c->g.lx, host_out);
}

// Device address under which host_dst can be written by a kernel (pinned /
// registered host memory under UVA), else nullptr.
static double* host_mapped(double* host_dst) {
  cudaPointerAttributes a{};
  if (cudaPointerGetAttributes(&a, host_dst) != cudaSuccess) {
    cudaGetLastError();  // pageable memory on older runtimes: clear the sticky-free error
    return nullptr;
  }
  return a.type == cudaMemoryTypeHost ? static_cast<double*>(a.devicePointer) : nullptr;
}

// Enqueue the invariants of A (fused-monitor partials when valid, else a full
// pass), the cross-rank reduction, and their delivery to host_dst: written by
// the final reduction block itself when host_dst is pinned and there is no
// cross-rank step, else a 40-byte D2H copy.
static int invariants_enqueue(lb_ctx* c, double* host_dst) {
  double* res = c->d_part + lbk::invariants_scratch(c->g);
  double* mapped = c->comm ? nullptr : host_mapped(host_dst);
  double* out = mapped ? mapped : res;
  if (c->mon_valid && c->mon_tb) {  // state n+2 partials of the last two-step launch
    const int G = c->mon_tb_G;
    TRY(launch(c, "k_monitor_reduce", c->s, 0, [&] {
      return lbk::launch_monitor_reduce(c->d_mon_tb + (int64_t)G * 5, G, c->d_mon_tb + (int64_t)c->mon_tb_cap * 10,
                                        c->d_ticket, out, c->d_nonphys, c->s);
    }));
  } else if (c->mon_valid) {
    const int64_t nslots = (int64_t)lbk::monitor_slots(c->g);
    TRY(launch(c, "k_monitor_reduce", c->s, 0, [&] {
      return lbk::launch_monitor_reduce(c->d_mon, nslots, c->d_mon + nslots * 5, c->d_ticket, out, c->d_nonphys,
                                        c->s);
    }));
  } else {
    TRY(launch(c, "k_invariants", c->s, c->L.sites, [&] {
      return lbk::launch_invariants(c->g, c->A, c->d_part, out, c->d_nonphys, c->s);
    }));
  }
  if (mapped) return LB_OK;
  if (c->comm) {
    NC(ncclGroupStart());
    NC(ncclAllReduce(res, res, 4, ncclDouble, ncclSum, c->comm, c->s));
    NC(ncclAllReduce(res + 4, res + 4, 1, ncclDouble, ncclMin, c->comm, c->s));
    NC(ncclGroupEnd());
  }
  CU(cudaMemcpyAsync(host_dst, res, 5 * sizeof(double), cudaMemcpyDeviceToHost, c->s));
  return LB_OK;
}

int lb_invariants(lb_ctx* c, double* out) {
  TRY(check_boundary(c, "lb_invariants"));
  if (!out) return fail(LB_EINVAL, "out is NULL");
  TRY(invariants_enqueue(c, c->h_pin));
  CU(cudaStreamSynchronize(c->s));
  TRY(check_peer_status(c));
  std::memcpy(out, c->h_pin, 5 * sizeof(double));
  for (int k = 0; k < 5; ++k)
    if (std::isnan(out[k])) return fail(LB_ENONPHYS, "NaN in invariants");
  if (!(out[4] > 0.0)) return fail(LB_ENONPHYS, "site density <= 0 or NaN");
  return LB_OK;
}

int lb_invariants_async(lb_ctx* c, double* host_out) {
  TRY(check_boundary(c, "lb_invariants_async"));
  if (!host_out) return fail(LB_EINVAL, "host_out is NULL");
  return invariants_enqueue(c, host_out);
}

int lb_invariants_pair_async(lb_ctx* c, double* host_out) {
  TRY(check_boundary(c, "lb_invariants_pair_async"));
  if (!host_out) return fail(LB_EINVAL, "host_out is NULL");
  if (!(c->mon_valid && c->mon_tb))
    return fail(LB_ESTATE, "no two-step launch with monitors since the last state change");
  double* mapped = host_mapped(host_out);
  double* res = c->d_part + lbk::invariants_scratch(c->g);  // 2 x 5 doubles of device result space
  const int G = c->mon_tb_G;
  TRY(launch(c, "k_monitor_reduce_pair", c->s, 0, [&] {
    return lbk::launch_monitor_reduce_pair(c->d_mon_tb, G, mapped ? mapped : res, c->d_nonphys, c->s,
                                           c->tb_pdl != 0 && !c->peers_on);
  }));
  if (!mapped) CU(cudaMemcpyAsync(host_out, res, 10 * sizeof(double), cudaMemcpyDeviceToHost, c->s));
  return LB_OK;
}

int lb_set_peers(lb_ctx* c, const lb_peers* p) {
  if (!c || !p) return fail(LB_EINVAL, "NULL argument");
  if (c->phase != 0) return fail(LB_ESTATE, "lb_set_peers only at a step boundary");
  if (c->p.mode != LB_MODE_FUSED || c->p.bc_y == LB_PERIODIC)
    return fail(LB_EINVAL, "peer exchange needs fused mode and walls in Y");
  if (c->g.lx < 6 && c->nranks > 1) return fail(LB_EINVAL, "peer exchange needs lx >= 6");
  for (int k = 0; k < 2; ++k)
    if (!p->left_buf[k] || !p->right_buf[k]) return fail(LB_EINVAL, "NULL peer buffer");
  if (!p->left_done || !p->right_done || !p->my_done) return fail(LB_EINVAL, "NULL step counter");
  // memory of a neighbour on another GPU (CUDA-IPC mapping): make sure this
  // device may access it directly (P2P over NVLink); same-device: nothing to do
  int dev = 0;
  CU(cudaGetDevice(&dev));
  const void* ptrs[6] = {p->left_buf[0], p->left_buf[1], p->right_buf[0], p->right_buf[1], p->left_done,
                         p->right_done};
  for (const void* q : ptrs) {
    cudaPointerAttributes a;
    CU(cudaPointerGetAttributes(&a, q));
    if (a.type != cudaMemoryTypeDevice) return fail(LB_EINVAL, "peer pointer is not device memory");
    if (a.device != dev) {
      int can = 0;
      CU(cudaDeviceCanAccessPeer(&can, dev, a.device));
      if (!can) return fail(LB_EINVAL, "device %d cannot access peer device %d", dev, a.device);
      cudaError_t e = cudaDeviceEnablePeerAccess(a.device, 0);
      if (e == cudaErrorPeerAccessAlreadyEnabled) (void)cudaGetLastError();
      else if (e != cudaSuccess) return fail(LB_ECUDA, "peer access to device %d: %s", a.device, cudaGetErrorString(e));
    }
  }
  if (!c->d_status && cudaMalloc(&c->d_status, sizeof(unsigned int)) != cudaSuccess)
    return fail(LB_ENOMEM, "status allocation failed");
  CU(cudaMemsetAsync(c->d_status, 0, sizeof(unsigned int), c->s));
  if (const char* e = std::getenv("LB_PEER_TIMEOUT_MS")) c->peer_timeout_ns = 1000000ull * std::strtoull(e, nullptr, 10);
  // two-step kernel at N > 1: tensor maps of the neighbours' buffers (the
  // in-kernel exchange), and staging for the neighbours' edge columns (the
  // k_tb_pull path: LB_OPT_TB_EDGE_PULL = 0, or maps the driver refuses)
  if (c->tb) {
    if (!c->tb->staged) {
      if (!c->d_stage && cudaMalloc(&c->d_stage, (size_t)12 * c->g.cs * sizeof(double)) != cudaSuccess)
        return fail(LB_ENOMEM, "staging allocation failed");
      if (!lbk::tb_attach_staging(c->tb, c->g, c->d_stage)) return fail(LB_ECUDA, "staging tensor maps failed");
    }
    lbk::tb_attach_peers(c->tb, c->g, p->left_buf, p->right_buf);  // false: the kernel falls back to k_tb_pull
    if (!c->d_ctas && cudaMalloc(&c->d_ctas, sizeof(unsigned int)) != cudaSuccess)
      return fail(LB_ENOMEM, "CTA counter allocation failed");
    CU(cudaMemsetAsync(c->d_ctas, 0, sizeof(unsigned int), c->s));
  }
  c->peers = *p;
  c->peers_on = true;
  c->peer_step = 0;
  c->halo_fresh = false;
  CU(cudaMemsetAsync(p->my_done, 0, sizeof(uint64_t), c->s));
  CU(cudaStreamSynchronize(c->s));
  return LB_OK;
}

int lb_set_option(lb_ctx* c, int option, int value) {
  if (!c) return fail(LB_EINVAL, "ctx is NULL");
  switch (option) {
    case LB_OPT_PROPAGATE_IMPL:
      if (value != 0 && value != 1) return fail(LB_EINVAL, "propagate impl must be 0 (LDG) or 1 (TMA)");
      if (value == 1 && !c->tma) {
        c->tma = lbk::tma_create(c->g, c->par ? c->B : c->A, c->par ? c->A : c->B);
        if (!c->tma) return fail(LB_ECUDA, "TMA tensor-map encoding unavailable");
      }
      c->prop_impl = value;
      return LB_OK;
    case LB_OPT_CUDA_GRAPH:
      if (value && !c->s) return fail(LB_EINVAL, "CUDA graphs need a non-default context stream");
      c->graph_on = value != 0;
      if (!c->graph_on) graph_reset(c);
      return LB_OK;
    case LB_OPT_TEMPORAL:
      if (value != 0 && value != 1) return fail(LB_EINVAL, "temporal blocking must be 0 or 1");
      if (value == 1 && !c->tb) {
        c->tb = lbk::tb_create(c->g, c->par ? c->B : c->A, c->par ? c->A : c->B, c->tb_promo);
        if (!c->tb) return fail(LB_ECUDA, "two-step kernel unavailable (tensor maps or lx < 6)");
      }
      c->tb_on = value;
      return LB_OK;
    case LB_OPT_TB_GRID:
      if (value < 0) return fail(LB_EINVAL, "grid must be >= 0");
      c->tb_grid = value;
      return LB_OK;
    case LB_OPT_TB_L2_PREFETCH:
      if (value < 0 || value > 64) return fail(LB_EINVAL, "L2 prefetch distance must be in [0, 64]");
      c->tb_l2 = value;
      return LB_OK;
    case LB_OPT_TB_L2_PROMOTION:
      if (value != 0 && value != 64 && value != 128 && value != 256)
        return fail(LB_EINVAL, "L2 promotion must be 0, 64, 128 or 256");
      c->tb_promo = value;
      if (c->tb && !lbk::tb_set_promotion(c->tb, c->g, value)) return fail(LB_ECUDA, "tensor-map re-encoding failed");
      return LB_OK;
    case LB_OPT_TB_WALL_WEIGHT:
      if (value < 0 || value > 256) return fail(LB_EINVAL, "wall weight (x16) must be in [0 (auto), 256]");
      c->tb_wall_w16 = value;
      return LB_OK;
    case LB_OPT_TB_EDGE_PULL:
      if (value != 0 && value != 1) return fail(LB_EINVAL, "edge pull must be 0 (k_tb_pull) or 1 (in-kernel)");
      c->tb_edge_pull = value;
      return LB_OK;
    case LB_OPT_TB_PDL:
      if (value != 0 && value != 1) return fail(LB_EINVAL, "PDL must be 0 or 1");
      c->tb_pdl = value;
      return LB_OK;
    case LB_OPT_TB_TAIL_WEIGHT:
      if (value != 0 && value != 1 && (value < 16 || value > 64))
        return fail(LB_EINVAL, "tail weight (x16) must be 0 (auto), 1 (contiguous split) or in [16, 64]");
      c->tb_tail_w16 = value;
      return LB_OK;
    case LB_OPT_FUSED_IMPL:
      if (value != 0 && value != 1) return fail(LB_EINVAL, "fused impl must be 0 (gather) or 1 (TMA)");
      if (value == 1 && !c->tma) return fail(LB_ECUDA, "TMA tensor-map encoding unavailable");
      c->fused_impl = value;
      return LB_OK;
    default:
      return fail(LB_EINVAL, "unknown option %d", option);
  }
}

int lb_monitor(lb_ctx* c, int enable) {
  if (!c) return fail(LB_EINVAL, "ctx is NULL");
  if (enable && !c->d_mon) {
    const size_t n = (lbk::monitor_slots(c->g) + lbk::MON_REDUCE_MAX_BLOCKS) * 5;
    if (cudaMalloc(&c->d_mon, n * sizeof(double)) != cudaSuccess ||
        cudaMalloc(&c->d_ticket, sizeof(unsigned int)) != cudaSuccess)
      return fail(LB_ENOMEM, "monitor allocation failed");
    CU(cudaMemsetAsync(c->d_ticket, 0, sizeof(unsigned int), c->s));
  }
  c->mon_on = enable != 0;
  c->mon_valid = false;
  return LB_OK;
}

int lb_profile_enable(lb_ctx* c, int enable) {
  if (!c) return fail(LB_EINVAL, "ctx is NULL");
  c->prof = enable != 0;
  return LB_OK;
}

int lb_profile_reset(lb_ctx* c) {
  if (!c) return fail(LB_EINVAL, "ctx is NULL");
  TRY(harvest(c));
  std::fill(c->kms.begin(), c->kms.end(), 0.0);
  std::fill(c->kcount.begin(), c->kcount.end(), 0);
  std::fill(c->kunits.begin(), c->kunits.end(), 0);
  return LB_OK;
}

int lb_profile_read(lb_ctx* c, lb_kprof* out, int max, int* n) {
  if (!c) return fail(LB_EINVAL, "ctx is NULL");
  TRY(harvest(c));
  const int k = (int)c->knames.size();
  if (n) *n = k;
  for (int i = 0; i < k && i < max && out; ++i) {
    std::memset(out[i].name, 0, sizeof(out[i].name));
    std::strncpy(out[i].name, c->knames[i].c_str(), sizeof(out[i].name) - 1);
    out[i].launches = c->kcount[i];
    out[i].total_ms = c->kms[i];
    out[i].units = c->kunits[i];
  }
  return LB_OK;
}

int64_t lb_launch_count(const lb_ctx* c) { return c ? c->launches : -1; }

int lb_tb_strip_height(void) { return lbk::tb_strip_height(); }

}  // extern "C"
