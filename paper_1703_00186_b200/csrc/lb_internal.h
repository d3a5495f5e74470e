// lb_internal.h — host-side declarations shared by lb_kernels.cu and lb_api.cu.
#pragma once
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdint>

#include "lb_device.cuh"

namespace lbk {

// Geometry of one rank's internal buffers (see include/lb.h "internal").
struct Geo {
  int lx, ly;      // physical extents
  int nx;          // lx + 6
  int nyp;         // padded rows per population column
  int y0;          // internal row of physical row 0
  int64_t cs;      // column stride = 37 * nyp
};

enum BcKind { BC_THERMAL = 0, BC_ADIABATIC = 1, BC_PERIODIC = 2 };
enum CollKind { COLL_BGK = 0, COLL_REGULARIZED = 1 };

// Column ranges are in internal column indices (physical columns are
// [3, 3+lx)).  A launch covers [xa0, xa1) U [xb0, xb1).
// rev != 0: blocks take the columns in reverse order (alternated step by step,
// so a step starts on the columns the previous step wrote last: those are
// still in the 126 MB L2 and are read from there instead of HBM).
struct Cols {
  int xa0, xa1, xb0, xb1;
  int rev = 0;
  int count() const { return (xa1 - xa0) + (xb1 - xb0); }
};

cudaError_t upload_kwall(const double* k_bottom, const double* k_top, cudaStream_t s);
// packed block inverse of the regularised-collide Gram matrix (lbd::NGINV doubles)
cudaError_t upload_ginv(const double* ginv, cudaStream_t s);

// N=1 periodic wrap of the x-halo columns (and y-halo rows when periodic).
cudaError_t launch_pbc_wrap(const Geo& g, double* A, int bc, cudaStream_t s);
// y-halo wrap only (periodic bc, N>1 after the x exchange)
cudaError_t launch_ywrap(const Geo& g, double* A, cudaStream_t s);
cudaError_t launch_propagate(const Geo& g, const double* A, double* B, cudaStream_t s);
cudaError_t launch_bc(const Geo& g, const double* A, double* B, int bc, cudaStream_t s);
cudaError_t launch_collide(const Geo& g, double* B, const lbd::Relax& r, int coll, cudaStream_t s);
// Where the border columns' results also go (the next step's halos) and, in
// peer mode, which step counters the border blocks wait on (lb_kernels.cu).
struct Halo {
  double* dstL = nullptr;   // ix in [3,6)      -> column ix + lx of dstL
  double* dstR = nullptr;   // ix in [lx, lx+3) -> column ix - lx of dstR
  const unsigned long long* waitL = nullptr;
  const unsigned long long* waitR = nullptr;
  // this rank's own counter = steps it has completed; the border blocks wait
  // until both neighbours' counters reach it (read on device: the launch
  // parameters are the same every step, so steps can be replayed from a graph)
  const unsigned long long* my_done = nullptr;
  unsigned int* status = nullptr;      // set to 1 if a wait timed out (watchdog)
  unsigned long long timeout_ns = 0;   // 0: wait forever
};
// mon != nullptr: fused monitors, monitor_slots(g) x 5 doubles of per-block partials
cudaError_t launch_step_fused(const Geo& g, const double* A, double* B, int bc, int coll,
                              const lbd::Relax& r, Cols cols, const Halo& h, double* mon, cudaStream_t s);
size_t monitor_slots(const Geo& g);
// Sum of the slots into out[5] (device or host-mapped pointer) in one launch;
// part: MON_REDUCE_MAX_BLOCKS x 5 doubles of scratch, ticket: a zeroed counter
// (left zeroed).  Deterministic: fixed block ranges, partials summed in order.
// flag (may be null): set to 1 if a result has a NaN sum or min rho <= 0.
constexpr int MON_REDUCE_MAX_BLOCKS = 148;
cudaError_t launch_monitor_reduce(const double* mon, int64_t nslots, double* part, unsigned int* ticket,
                                  double* out, unsigned int* flag, cudaStream_t s);
// Two slot sets (nslots each, consecutive) reduced by one block into out[10].
cudaError_t launch_monitor_reduce_pair(const double* mon, int64_t nslots, double* out, unsigned int* flag,
                                       cudaStream_t s, bool pdl = false);
// TMA-staged kernels (lb_tma.cu): tensor maps of both buffers, built once.
// Buffer k viewed as {nyp rows, 37 populations, nx columns}, box {256, 1, 1}.
struct TmaMaps {
  CUtensorMap load[2];
};
TmaMaps* tma_create(const Geo& g, double* buf0, double* buf1);
void tma_destroy(TmaMaps* t);
cudaError_t launch_propagate_tma(const Geo& g, const TmaMaps* t, int src_buf, double* B, cudaStream_t s);
// Fused step with TMA-staged windows (N = 1 local wrap path; walls only)
cudaError_t launch_step_fused_tma(const Geo& g, const TmaMaps* t, int src_buf, const double* A, double* B,
                                  int bc, int coll, const lbd::Relax& r, const Halo& h, cudaStream_t s);
// Two steps per pass (lb_tb.cu, temporal blocking): N = 1, walls only.  The
// state-n windows are loaded by TMA straight from the physical columns
// (periodic wrap in the coordinates), so A's halo is not read; B's halo is
// written (the next step's wrap).
struct TbMaps {
  CUtensorMap load[2][3];  // column-group windows, box {HT + 12, 3 | 5 | 7, 1}, per buffer
  CUtensorMap st[2][3];    // N > 1: staging of the left / right neighbour's 6 edge columns
  CUtensorMap nb[2][2][3]; // N > 1: the left (0) / right (1) neighbour's buffer k, read directly (tb_attach_peers)
  bool direct = false;     // nb[] encoded
  double* nbuf[2][2] = {{nullptr, nullptr}, {nullptr, nullptr}};  // the buffers nb[] describes
  bool staged = false;  // st[] encoded (tb_attach_staging)
  int promo = 0;        // L2 promotion of every map: 0 / 64 / 128 / 256 bytes (LB_OPT_TB_L2_PROMOTION)
  double* bufs[2] = {nullptr, nullptr};
  double* stage = nullptr;
};
TbMaps* tb_create(const Geo& g, double* buf0, double* buf1, int promo);
// re-encode every map of t with another L2 promotion (0 / 64 / 128 / 256)
bool tb_set_promotion(TbMaps* t, const Geo& g, int promo);
// N > 1 (peer mode): stage = 2 x 6 x g.cs doubles — [0, 6 cs) the left
// neighbour's last 6 physical columns (our internal columns -3..2), [6 cs,
// 12 cs) the right neighbour's first 6 (our internal lx+3..lx+8)
bool tb_attach_staging(TbMaps* t, const Geo& g, double* stage);
// N > 1 (peer mode): tensor maps of the neighbours' two buffers (same layout
// as ours: equal slabs), so the kernel's edge CTAs load the columns beyond the
// slab straight from the neighbours' current buffer; false if the driver
// cannot encode them (peer mapping), the caller then stages (k_tb_pull)
bool tb_attach_peers(TbMaps* t, const Geo& g, double* const left[2], double* const right[2]);
// Fill the staging buffer from the neighbours' current buffers (peer memory)
// once both have completed as many launches as this rank (*waitL/R >= *my_done;
// watchdog: *status = 1 after timeout_ns, 0 = wait forever).
cudaError_t launch_tb_pull(const Geo& g, double* stage, const double* left_A, const double* right_A,
                           const unsigned long long* waitL, const unsigned long long* waitR,
                           const unsigned long long* my_done, unsigned int* status, unsigned long long timeout_ns,
                           cudaStream_t s);
// false for the few heights with no valid strip layout (HT < ly < HT + 6)
bool tb_layout_ok(int ly);
int tb_strip_height();  // HT of the compiled two-step kernel
void tb_destroy(TbMaps* t);
// lb_tb.cu's own copies of the wall constants and the Gram inverse
cudaError_t tb_upload_constants(const double* k_bottom, const double* k_top, const double* ginv, cudaStream_t s);
// N > 1, in-kernel edge pulls (the default of peer mode): only the CTAs whose
// sweep reads or writes within 6 columns of a slab edge wait (thread 0,
// ld.acquire.sys, watchdog) until that neighbour completed as many launches as
// this rank, then copy the rows of the neighbour's 6 edge columns their strip
// needs into the staging buffer themselves; every other CTA starts at once,
// so the exchange overlaps the interior sweeps (§8a6).
// N > 1, exchange inside the two-step kernel: the edge CTAs wait for the
// neighbours' launch counters (watchdog: status, timeout_ns) and load the
// columns beyond the slab from the neighbours' current buffers (TbMaps::nb);
// the last CTA to finish publishes this rank's counter (my_done += 1) —
// ctas_done counts finished CTAs and is reset by that last CTA.
struct TbPeer {
  const unsigned long long* waitL = nullptr;
  const unsigned long long* waitR = nullptr;
  unsigned long long* my_done = nullptr;
  unsigned int* ctas_done = nullptr;
  unsigned int* status = nullptr;
  unsigned long long timeout_ns = 0;
};
// grid: CTAs (one per SM); l2_dist: L2 prefetch distance in columns (0 = off; LSU prefetch);
// wall_w16: cost of a wall-strip column in 1/16 of an interior one (work split);
// mon != nullptr: monitors, 2 x tb_grid(g, grid) x 5 doubles of per-CTA
// partials (state n+1, then state n+2)
// peers != 0: columns beyond the slab come from the staging buffer (N > 1) and
// B's halo is not written; else the N = 1 periodic wrap.
// pull != nullptr (peers only): in-kernel edge pulls instead of a preceding launch_tb_pull.
// pdl: launch with programmatic dependent launch (the kernel's prologue may
// overlap the previous kernel's last CTAs; griddepcontrol.wait before any
// global-memory access).
cudaError_t launch_step2_tb(const Geo& g, const TbMaps* t, int src_buf, double* B, int bc, int coll,
                            const lbd::Relax& r, int grid, int l2_dist, int wall_w16, double* mon, int peers,
                            const TbPeer* pull, cudaStream_t s, bool pdl = false);
// CTAs a two-step launch with `grid` requested actually uses
int tb_grid(const Geo& g, int grid);
// this rank's counter += 1 (system-scope release), after the step kernel
cudaError_t launch_signal(unsigned long long* done, cudaStream_t s);
// wait.waitL != nullptr: first wait (watchdog) for both neighbours' counters
// to reach *wait.my_done (the pull after a two-step launch)
cudaError_t launch_peer_pull(const Geo& g, double* A, const double* left_A, const double* right_A,
                             const Halo& wait, cudaStream_t s);
cudaError_t launch_init_macro(const Geo& g, double* A, const double* rho, const double* ux,
                              const double* uy, const double* T, cudaStream_t s);
cudaError_t launch_init_rt(const Geo& g, double* A, const double* eps, int lx_total, int x0, double t_ref,
                           double amp, double width, cudaStream_t s);
cudaError_t launch_canon_to_internal(const Geo& g, const double* canon, double* A, cudaStream_t s);
cudaError_t launch_internal_to_canon(const Geo& g, const double* A, double* canon, cudaStream_t s);
// partials: scratch of at least invariants_scratch(g) doubles; out: 5 doubles on device
size_t invariants_scratch(const Geo& g);
cudaError_t launch_invariants(const Geo& g, const double* A, double* partials, double* out,
                              unsigned int* flag, cudaStream_t s);

}  // namespace lbk
