/*
 * lb.h — C ABI of the B200-native D2Q37 thermal Lattice Boltzmann hot path
 * (arXiv 1703.00186, Calore et al., CCPE 28:3485).  Library: liblb_d2q37.so
 * (paper_1703_00186_b200/), hand-written sm_100a CUDA kernels.
 *
 * Citations "P:a-b" are lines of the paper text; "G<n>" are the
 * readings of the paper listed in DESIGN.md §3; "§8x" are rows of SURVEY.md §8.
 *
 * ---------------------------------------------------------------------------
 * What one time step computes (Eq. 1 at P:183-187):
 *   pbc       periodic-X halo columns (3 per side, all 37 populations)   §8a1
 *   propagate B[l, x] = A[l, x - c_l]  (pull; populations hop <= 3 sites) §8a2
 *   bc        top/bottom walls: specular mirror + thermal repopulation   §8a3
 *   collide   f <- f - (dt/tau)(f - f_eq(rho, u, T)), moments of Eq. 2   §8a4
 *   swap      A <-> B                                                    §8a7
 * fused mode does propagate+bc+collide in one pull pass A -> B (§8a5) and is
 * bit-identical to split mode.  With N ranks the lattice is split into X
 * slabs on a ring; the halo exchange runs on a communication
 * stream overlapped with the bulk columns (§8a6).
 *
 * ---------------------------------------------------------------------------
 * Layouts.
 *   canonical (host side of lb_set_state / lb_gather / lb_init_macro):
 *     populations  [37][Lx][Ly]  doubles, iy fastest, physical sites only
 *                  (the SoA order of P:493-496 with halos stripped);
 *     macro fields [Lx][Ly]      doubles.
 *     Population labels follow G2: l = 0..36 enumerates c = (cx, cy) with cx
 *     from +3 down to -3 and cy ascending; l = 0 is (3,-1), l = 1 is (3,0)
 *     (P:452-453), l = 18 is the rest population.
 *   internal (device buffers f_a, f_b; "column-blocked SoA"):
 *     element (ix, l, r) at  (ix * 37 + l) * nyp + r,
 *     ix in [0, Lx+6): columns, physical columns are [3, 3+Lx);
 *     r in [0, nyp): rows, physical row y (0-based) is r = y0 + y, the
 *     y-halo rows are [y0-3, y0) and [y0+Ly, y0+Ly+3).  y0 and nyp are
 *     multiples of 16 doubles (128 B), so every physical column starts on a
 *     128-byte boundary.  Each column holds the 37 population rows of one
 *     lattice column contiguously, so a rank's 3 halo / border columns are one
 *     contiguous block of 3*37*nyp doubles (no packing for the exchange).
 *
 * Ownership.  The caller allocates f_a and f_b (lb_layout.elems doubles each,
 * 16-byte aligned device memory, e.g. torch tensors) and keeps them alive
 * until lb_destroy returns; the library borrows them.  The context owns its
 * streams, events, NCCL communicator and small scratch; lb_destroy frees them.
 *
 * Errors.  Every call returns an int status (LB_OK = 0).  No exception crosses
 * the ABI.  Calls other than lb_gather, lb_invariants, lb_sync and
 * lb_profile_read only enqueue work on the context's stream; an error of an
 * asynchronous kernel surfaces at the next synchronising call as LB_ECUDA.
 * lb_last_error() gives a human-readable message for the calling thread.
 *
 * Threading.  One context per process and GPU; a context is not thread-safe.
 */
#ifndef LB_D2Q37_H
#define LB_D2Q37_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define LB_Q 37    /* populations per site                      */
#define LB_HALO 3  /* halo width Hx = Hy = 3        */

/* status codes (SPEC S:469 exit-code classes: rejected = 2, blow-up = 3) */
enum lb_status {
  LB_OK = 0,
  LB_EINVAL = 1,     /* invalid argument or parameter set                   */
  LB_ESTATE = 2,     /* call out of order (e.g. lb_gather mid-step)         */
  LB_ECUDA = 3,      /* CUDA runtime / kernel error                          */
  LB_ENCCL = 4,      /* NCCL error                                           */
  LB_ENONPHYS = 5,   /* NaN or rho <= 0 detected by lb_invariants, or (sticky
                        device flag) by any invariants / monitor reduction
                        since the last state change, reported by lb_sync     */
  LB_ENOMEM = 6,     /* host or device allocation failed                     */
  LB_EPEER = 7       /* peer exchange watchdog: a neighbour never signalled  */
};

enum lb_bc_y {
  LB_WALL_THERMAL = 0,   /* mirror + thermal repopulation at T_bottom/T_top (G9) */
  LB_WALL_ADIABATIC = 1, /* mirror only                                          */
  LB_PERIODIC = 2        /* no bc; y-halo rows wrapped by pbc (test geometry)    */
};

enum lb_collision {
  LB_COLLIDE_BGK = 0,         /* Eq. 1 BGK relaxation to f_eq (App. B)          */
  LB_COLLIDE_REGULARIZED = 1  /* Hermite-projected (orders <= 4):
                                 f <- f_eq + (1 - dt/tau)(P f - f_eq) (NEXT 1)   */
};

enum lb_mode {
  LB_MODE_FUSED = 0,     /* one pull kernel: propagate+bc+collide, A -> B     */
  LB_MODE_SPLIT = 1      /* propagate, bc, collide as separate kernels        */
};

typedef struct lb_params {
  int lx_total;          /* global physical columns (X, decomposed)           */
  int ly;                /* physical rows (Y, never decomposed)               */
  double tau;            /* relaxation time (Eq. 1)                           */
  double dt;             /* time step (Eq. 1); 0 < dt/tau <= 2                */
  double t_bottom;       /* wall temperature at y = -1/2  (lattice units)     */
  double t_top;          /* wall temperature at y = Ly - 1/2                  */
  int bc_y;              /* enum lb_bc_y                                       */
  int mode;              /* enum lb_mode                                       */
  int overlap;           /* 1: exchange || bulk, then borders.
                            lb_init returns LB_EINVAL where the schedule cannot
                            run: split mode, bc_y = PERIODIC, lx < 6, or N = 1
                            without an NCCL id (the local wrap has no exchange).
                            The peer-store exchange (lb_set_peers) always
                            overlaps inside the kernel, whatever this flag.   */
  int collision;         /* enum lb_collision                                 */
  double gx, gy;         /* body force: velocity increment per step (NEXT 2,
                            shifted equilibrium u + tau g, T + tau(1-tau)|g|^2/D;
                            DESIGN.md reading G7b); 0 = unforced Eq. 1         */
} lb_params;

typedef struct lb_dist {
  int rank;              /* this process' slab, 0..nranks-1                    */
  int nranks;            /* ring size N; lx_total % N == 0                     */
  const unsigned char* nccl_id; /* 128-byte ncclUniqueId from rank 0.  N > 1 without
                            it: only the peer-store exchange (lb_set_peers) is
                            available.  At N == 1, NULL selects the local wrap kernel;
                            non-NULL runs the exchange through NCCL as a 1-rank ring
                            (self send/recv) — the N > 1 transport on one GPU. */
} lb_dist;

typedef struct lb_layout {
  int lx;                /* physical columns of this rank = lx_total / N       */
  int ly;                /* physical rows                                      */
  int nx;                /* lx + 6 columns (3 halo columns per side)          */
  int nyp;               /* padded rows per population column (mult. of 16)   */
  int y0;                /* internal row of physical row 0 (multiple of 16)   */
  int x0_global;         /* global index of this rank's first physical column */
  int64_t col_stride;    /* 37 * nyp doubles between consecutive columns       */
  int64_t elems;         /* doubles per buffer = nx * col_stride               */
  int64_t bytes;         /* elems * 8                                          */
  int64_t sites;         /* lx * ly physical sites of this rank                */
} lb_layout;

/* The ring exchange of one rank (§8a1, §8e), as lb_exchange / lb_step issue
 * it: offsets are element offsets into the rank's A buffer (internal layout),
 * each message is `count` contiguous doubles (3 full columns).  The four
 * transfers are posted in this order inside one NCCL group: receive the left
 * halo from `left`, receive the right halo from `right`, send the right border
 * to `right`, send the left border to `left` — so for N = 2 (left == right)
 * the k-th send of a rank matches the k-th receive of its peer.  Bulk and
 * border column ranges (internal column indices) are those of the overlapped
 * schedule: the bulk reads no halo column. */
typedef struct lb_xplan {
  int left, right;              /* ring neighbours                 */
  int64_t count;                /* doubles per message = 3 * 37 * nyp          */
  int64_t recv_left_off;        /* columns [0, 3): left halo                   */
  int64_t recv_right_off;       /* columns [lx+3, lx+6): right halo            */
  int64_t send_right_off;       /* columns [lx, lx+3): -> right's left halo    */
  int64_t send_left_off;        /* columns [3, 6): -> left's right halo        */
  int bulk_x0, bulk_x1;         /* bulk columns [bulk_x0, bulk_x1)             */
  int border_x0, border_x1, border_x2, border_x3; /* [x0,x1) U [x2,x3)        */
} lb_xplan;

/* Peer-store exchange ("exchange fused into the kernel"):
 * device pointers, valid in this process (CUDA IPC mappings of the
 * neighbours' buffers over NVLink, or plain pointers for contexts of one
 * process), of the two neighbours' population buffers (their f_a, f_b in
 * lb_init order) and of three 8-byte step counters in device memory. */
typedef struct lb_peers {
  double* left_buf[2];         /* left neighbour's f_a, f_b                    */
  double* right_buf[2];        /* right neighbour's f_a, f_b                   */
  const uint64_t* left_done;   /* left neighbour's step counter                */
  const uint64_t* right_done;  /* right neighbour's step counter               */
  uint64_t* my_done;           /* this rank's counter (read by both neighbours) */
} lb_peers;

typedef struct lb_ctx lb_ctx;

/* Per-kernel timing record (see lb_profile_enable). */
typedef struct lb_kprof {
  char name[32];         /* kernel name, e.g. "k_step_fused"                   */
  int64_t launches;      /* launches timed since the last reset               */
  double total_ms;       /* summed CUDA-event time of those launches          */
  int64_t units;         /* lattice sites those launches processed            */
} lb_kprof;

/* ---- host-only queries (no GPU needed) ---------------------------------- */

/* Validate p for (rank, nranks) and fill *out.  Rules: lx_total % nranks == 0;
 * per-rank lx >= 3 (N = 1) or >= 6 (N > 1, so the 3+3 border columns are
 * disjoint); ly >= 6 for walls (>= 3 periodic); 0 < dt/tau <= 2; wall
 * temperatures > 0; enums in range.  Returns LB_EINVAL otherwise. */
int lb_query_layout(const lb_params* p, int rank, int nranks, lb_layout* out);

/* The D2Q37 constants the library uses (host copies; DESIGN.md App. A):
 * c[37][2] lattice velocities (label order G2), w[37] weights, *a the scale
 * factor, *t0 = 1/a^2 the reference temperature (G3).  Any pointer may be NULL. */
int lb_constants(int* c, double* w, double* a, double* t0);

/* Wall constants K_wall,l(T_wall) (App. B, canonical expression tree G16)
 * exactly as uploaded by lb_init: K[37]. */
int lb_kwall(double t_wall, double* K);

/* Fill *out with the exchange plan of (rank, nranks) for p (host only). */
int lb_exchange_plan(const lb_params* p, int rank, int nranks, lb_xplan* out);

/* ncclGetUniqueId into out[128] (rank 0 calls it; broadcast it to the others). */
int lb_nccl_unique_id(unsigned char* out);

/* Message for the last failing call on this thread (static storage). */
const char* lb_last_error(void);
const char* lb_strerror(int status);

/* ---- context ------------------------------------------------------------ */

/* Create a context on the current CUDA device.  f_a, f_b: caller-owned
 * device buffers of lb_layout.elems doubles (16-byte aligned).  stream: the
 * cudaStream_t all compute work is enqueued on (NULL = legacy default
 * stream).  Zero-fills both buffers (so halo rows are deterministic, G10),
 * uploads K_wall for t_bottom / t_top, and for nranks > 1 creates the NCCL
 * communicator from d->nccl_id plus a high-priority communication stream.
 * Synchronising. */
int lb_init(const lb_params* p, const lb_dist* d, double* f_a, double* f_b,
            void* stream, lb_ctx** out);
void lb_destroy(lb_ctx* ctx);
int lb_get_layout(const lb_ctx* ctx, lb_layout* out);
int lb_set_stream(lb_ctx* ctx, void* stream);

/* A := f_eq(rho, u, T) (App. B) on this rank's physical sites.  rho, ux, uy,
 * T: [Lx][Ly] doubles (this rank's columns), in host memory if on_device == 0
 * (pageable or pinned), else device memory.  Uses B as staging and re-zeroes
 * it.  Only at a step boundary (LB_ESTATE otherwise). */
int lb_init_macro(lb_ctx* ctx, const double* rho, const double* ux,
                  const double* uy, const double* T, int on_device);

/* A := f_eq of the isobaric Rayleigh-Taylor state of DESIGN.md §4 (the
 * benchmark workload), evaluated on the device for this
 * rank's columns: interface y_i(x) = (Ly-1)/2 + max(1, Ly/64) cos(2 pi x /
 * Lx_tot) + eps[x] (x global), T = t_ref (1 + amp tanh((y_i - y)/width)),
 * rho = t_ref / T, u = 0.  eps: lx_total doubles, host or device memory (the
 * caller draws them; lbgen draws U(-1/4, 1/4) from PCG64).  Equals
 * lb_init_macro on the host-evaluated fields up to the last-ulp differences
 * of device cos/tanh.  Needs t_ref > 0, width > 0, |amp| < 1 (LB_EINVAL).
 * Uses B as staging and re-zeroes it.  Only at a step boundary. */
int lb_init_rt(lb_ctx* ctx, const double* eps, double t_ref, double amp, double width);

/* A := populations given in canonical local layout [37][Lx][Ly] (host memory
 * if on_device == 0, else device).  Only at a step boundary. */
int lb_set_state(lb_ctx* ctx, const double* canon, int on_device);

/* ---- the hot path (§8b): each call enqueues on the context stream ------- */

int lb_exchange(lb_ctx* ctx);   /* pbc on A (§8a1): wrap (N=1) or NCCL ring   */
int lb_propagate(lb_ctx* ctx);  /* raw pull A -> B (§8a2); entries pulled from
                                   the y-halo stay zero until lb_bc            */
int lb_bc(lb_ctx* ctx);         /* walls on B reading A (§8a3); no-op if PERIODIC */
int lb_collide(lb_ctx* ctx);    /* in place on B (§8a4), THEN swaps A <-> B, so
                                   exchange, propagate, bc, collide == lb_step(1) */
int lb_step(lb_ctx* ctx, int nsteps); /* nsteps full steps in p->mode, with the
                                   overlapped schedule when p->overlap         */

/* Switch lb_step to the peer-store exchange: each step is ONE fused kernel
 * whose 3+3 border-column blocks (i) wait until both neighbours' counters
 * reach this rank's step index (their previous step is complete, so this
 * rank's halo is current and theirs may be overwritten), (ii) compute, and
 * (iii) also store their results into the neighbours' next buffers (left
 * border -> left neighbour's right halo, right border -> right neighbour's
 * left halo); bulk blocks never wait.  A one-thread kernel then publishes this
 * rank's counter (st.release.sys).  Fused mode and walls only; per-rank
 * lx >= 6.  Zeroes *my_done and synchronises.  Collective in effect: every
 * rank calls it, then all ranks barrier before the next lb_step; the first
 * step after it (or after lb_set_state / lb_init_macro, which must likewise be
 * followed by a barrier) fills the halos by reading the neighbours' A.
 * Watchdog: a border block that waits longer than 20 s (env
 * LB_PEER_TIMEOUT_MS overrides) gives up, flags the context and proceeds, so
 * a dead neighbour cannot hang the GPU; lb_sync / lb_invariants then return
 * LB_EPEER and the state is invalid. */
int lb_set_peers(lb_ctx* ctx, const lb_peers* peers);

/* ---- results ------------------------------------------------------------ */

/* Collective over the ring.  Physical state A in canonical GLOBAL layout
 * [37][lx_total][Ly] written to host_out on rank `root` (other ranks may pass
 * NULL).  Uses B as device staging; only at a step boundary.  Synchronising.
 * N > 1 needs the NCCL communicator (LB_ESTATE otherwise; use lb_peek). */
int lb_gather(lb_ctx* ctx, double* host_out, int root);

/* Debug view: this rank's physical sites of buffer which (0 = A, 1 = B) in
 * canonical local layout [37][Lx][Ly], converted on the host; allowed mid-step
 * (e.g. between lb_propagate and lb_bc).  Synchronising. */
int lb_peek(lb_ctx* ctx, int which, double* host_out);
/* Same for this rank's physical columns [x0, x0+ncols) only: host_out is
 * [37][ncols][Ly] (one contiguous D2H of the column block; used for sampled
 * checks of lattices too large to gather). */
int lb_peek_cols(lb_ctx* ctx, int which, int x0, int ncols, double* host_out);

/* Collective (local sums if the context has no NCCL communicator).
 * out[0..3] = global sum over physical sites of rho, j_x, j_y
 * and E = 1/2 sum_l |c_l|^2 f_l, out[4] = global minimum site density.
 * Deterministic for a fixed N (fixed-order block partials).  Returns
 * LB_ENONPHYS if any value is NaN or min rho <= 0.  Synchronising. */
int lb_invariants(lb_ctx* ctx, double* out);

/* Non-blocking variant: enqueues the same reduction (collective) and an async
 * copy of the 5 values into host_out (page-locked memory for true asynchrony),
 * valid after the next lb_sync.  The check runs on the device: a result with a
 * NaN sum or min rho <= 0 sets the context's sticky non-physical flag, and the
 * next lb_sync returns LB_ENONPHYS ("numerical blow-up").
 * With monitors on (lb_monitor) the minimum also turns -inf when a collision's
 * own u or T is NaN / infinite, so a blow-up is caught by the launch whose
 * collision created it. */
int lb_invariants_async(lb_ctx* ctx, double* host_out);

/* Both states of the last two-step launch (LB_OPT_TEMPORAL) with monitors on:
 * enqueues host_out[0..4] = the invariants (as lb_invariants) of state n+1 and
 * host_out[5..9] = those of state n+2, reduced from per-CTA partials the
 * two-step kernel wrote (so a two-step lb_step(2) still yields one result per
 * time step).  host_out: 10 doubles, page-locked for true asynchrony; valid
 * after the next lb_sync.  LB_ESTATE if the last step was not such a launch.
 * Non-physical results set the sticky flag lb_sync reports (as above).  Not
 * collective: at N > 1 the values are this rank's slab (sum them over ranks,
 * e.g. after the run; lb_invariants is the collective form). */
int lb_invariants_pair_async(lb_ctx* ctx, double* host_out);

/* Waits for the context's streams.  LB_EPEER if a peer wait timed out;
 * LB_ENONPHYS if any invariants / monitor reduction since the last
 * lb_set_state / lb_init_macro / lb_init_rt saw NaN or rho <= 0 (the flag
 * stays set until the state is replaced). */
int lb_sync(lb_ctx* ctx);

/* Options.  LB_OPT_PROPAGATE_IMPL (lb_propagate, split mode): 1 = TMA-staged
 * (cp.async.bulk.tensor 3-D loads of the +-3-row windows into shared memory,
 * 16-byte vector stores; the default when the tensor maps can be encoded),
 * 0 = register gather with coalesced 8-byte loads, all 37 in flight per
 * thread.  Both are bit-identical; bench.py reports both. */
/* LB_OPT_FUSED_IMPL (lb_step, fused mode, N = 1 with walls, monitors off):
 * 0 = register gather (default), 1 = TMA-staged windows in shared memory. */
/* LB_OPT_CUDA_GRAPH (value 1): lb_step replays CUDA graphs of two steps in the
 * steady state of the fused N = 1 path and of the peer path (bit-identical;
 * fewer host launches, matters for small lattices).  Needs a non-default
 * context stream; ignored while profiling. */
/* LB_OPT_TEMPORAL (value 1, the default for N = 1 with walls in fused mode;
 * 0 disables): lb_step advances two steps per pass over HBM where it can
 * (N = 1 without NCCL or peers, or N > 1 in peer mode; walls, fused mode;
 * monitors on or off):
 * one launch of the two-step kernel computes states n+1 and n+2, keeping n+1
 * in shared memory (temporal blocking).  Bit-identical to two
 * fused steps; an odd remainder takes one fused step.  LB_OPT_TB_GRID: CTAs of
 * that kernel (0 = one per SM), LB_OPT_TB_L2_PREFETCH: L2 prefetch distance in
 * columns (0 = off, the default, <= 64; per-line prefetch of the newest column).  LB_OPT_TB_WALL_WEIGHT: cost of a column of a
 * wall strip relative to an interior one, x16 (work split; 0 = the default: 21 with the
 * time-aligned split, with the contiguous one 19 for BGK and 20 for the regularised collide).
 * LB_OPT_TB_L2_PROMOTION: L2 promotion of that kernel's TMA window loads in
 * bytes (0 = none, 64 = default, 128, 256); results do not depend on it.
 * LB_OPT_TB_EDGE_PULL (N > 1, peer mode): 1 (default) = the exchange runs
 * inside the two-step kernel — only the CTAs whose sweep reads or writes
 * within 6 columns of a slab edge wait for that neighbour's launch counter and
 * stage their strip's rows of its 6 edge columns, so the interior sweeps
 * overlap the exchange (§8a6); 0 = a separate k_tb_pull launch
 * (wait for both neighbours, stage whole columns) before the kernel.  Both
 * give the same bits.
 * LB_OPT_TB_TAIL_WEIGHT: the two-step kernel splits its work
 * time-aligned (every strip's main region cut into the same column ranges, the
 * CTAs left over share the remaining columns of every strip: the tail); the
 * cost of a tail column relative to a main-region one, x16 (0 = the default,
 * measured: 17 when every strip has >= 2 main-region CTAs, else 16; 16..64),
 * or 1 = the contiguous split instead (strip-major column ranges).  Work split only: results do not depend on it.
 * LB_OPT_TB_PDL (1 = default, 0 = off): the two-step kernel is launched with
 * programmatic dependent launch, so its CTAs start (and compute their work
 * split) on the SMs the previous launch's CTAs free; each waits for the
 * previous grid's completion before touching global memory.  Same results.
 * Not used with peers (N > 1): ranks sharing one GPU (tests) would park CTAs
 * of their next launch on SMs a waiting neighbour needs. */
enum lb_option {
  LB_OPT_PROPAGATE_IMPL = 0,
  LB_OPT_FUSED_IMPL = 1,
  LB_OPT_CUDA_GRAPH = 2,
  LB_OPT_TEMPORAL = 3,
  LB_OPT_TB_GRID = 4,
  LB_OPT_TB_L2_PREFETCH = 5,
  LB_OPT_TB_WALL_WEIGHT = 6,
  LB_OPT_TB_L2_PROMOTION = 7,
  LB_OPT_TB_EDGE_PULL = 8,
  LB_OPT_TB_TAIL_WEIGHT = 9,
  LB_OPT_TB_PDL = 10
};
int lb_set_option(lb_ctx* ctx, int option, int value);

/* Fused monitors.  enable != 0: every fused step also reduces, per block, the
 * invariants of the state it writes (rho, j, E sums and min rho of its sites)
 * into a small per-block array, and lb_invariants after such a step sums
 * those partials (one tiny kernel) instead of re-reading the lattice (296
 * B/site).  Values agree with the full pass to rounding (different summation
 * tree).  Allocates lx*ceil(ly/128)*40 B on first enable.  The two-step
 * kernel (LB_OPT_TEMPORAL) reduces both of its states per CTA from the
 * moments its collisions form (rho, j, sum |c|^2 f of each site before the
 * collision, which the collision conserves, plus the body-force increments of
 * reading G7b): equal to the sums over the stored states up to rounding;
 * lb_invariants_pair_async returns both. */
int lb_monitor(lb_ctx* ctx, int enable);

/* ---- instrumentation ----------------------------------------------------- */

/* enable != 0: bracket every kernel launch with CUDA events on the stream it
 * is launched on and accumulate per-kernel time (lb_profile_read, which
 * synchronises).  Costs two event records per launch.  Disabled by default. */
int lb_profile_enable(lb_ctx* ctx, int enable);
int lb_profile_reset(lb_ctx* ctx);
/* Fills up to max records; *n receives the number of distinct kernels. */
int lb_profile_read(lb_ctx* ctx, lb_kprof* out, int max, int* n);
/* Number of kernel launches the library issued since lb_init (all streams). */
int64_t lb_launch_count(const lb_ctx* ctx);
/* Strip height HT of the two-step kernel this library was built with (rows a
 * CTA computes per sweep).  lb_step uses that kernel for
 * ly <= HT or ly >= HT + 6 (other heights admit no strip layout that keeps
 * each wall band inside a wall strip) and the one-step kernel otherwise.
 * No context, no GPU needed. */
int lb_tb_strip_height(void);

#ifdef __cplusplus
}
#endif
#endif /* LB_D2Q37_H */
