// lb_kernels.cu — sm_100a kernels of the D2Q37 hot path.
//
// Memory layout: column-blocked SoA, element (ix, l, r) at (ix*37 + l)*nyp + r
// (include/lb.h).  Thread mapping for every per-site kernel: one thread per
// lattice site, a warp covers 32 consecutive rows of one column, so every
// population access of a warp is one contiguous 256-byte run (coalesced; the
// +-3 row shift of the pull makes it straddle one extra 32-byte sector, which
// the neighbouring warp uses — DRAM traffic stays at 1x).
//
// None of these kernels is a dense contraction, so there is no tensor-core
// path (SURVEY.md §2 "Hardware"); propagate / fused are HBM-bound, collide's
// FP64 work sits on the FP64 pipe with all constants as immediates or
// constant-bank operands.
#include "lb_device.cuh"
#include "lb_internal.h"
#include "lb_collide.cuh"


namespace lbk {
using namespace lbd;

constexpr int TPB = 128;  // threads per block of the per-site kernels

cudaError_t upload_ginv(const double* ginv, cudaStream_t s) {
  cudaError_t e = cudaMemcpyToSymbolAsync(c_ginv, ginv, sizeof(double) * NGINV, 0,
                                          cudaMemcpyHostToDevice, s);
  if (e != cudaSuccess) return e;
  return cudaStreamSynchronize(s);
}

cudaError_t upload_kwall(const double* k_bottom, const double* k_top, cudaStream_t s) {
  cudaError_t e = cudaMemcpyToSymbolAsync(c_kwall, k_bottom, sizeof(double) * Q, 0,
                                          cudaMemcpyHostToDevice, s);
  if (e != cudaSuccess) return e;
  e = cudaMemcpyToSymbolAsync(c_kwall, k_top, sizeof(double) * Q, sizeof(double) * Q,
                              cudaMemcpyHostToDevice, s);
  if (e != cudaSuccess) return e;
  return cudaStreamSynchronize(s);
}

// ---------------------------------------------------------------- pbc (§8a1)
// N=1 wrap: halo columns [0,3) <- [lx, lx+3), [lx+3, lx+6) <- [3, 6),
// full columns including the y-halo rows (G12).  Column blocks are contiguous,
// so this is two 16-byte-vectorised block copies.
__global__ void __launch_bounds__(256) k_pbc_wrap(double2* __restrict__ A, int64_t lx, int64_t cs2) {
  const int64_t n = 3 * cs2;  // double2 per side
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < 2 * n;
       i += (int64_t)gridDim.x * blockDim.x) {
    if (i < n)
      A[i] = A[lx * cs2 + i];                       // left halo <- rightmost physical
    else
      A[(lx + 3) * cs2 + (i - n)] = A[3 * cs2 + (i - n)];  // right halo <- leftmost physical
  }
}

// Periodic-Y wrap of the y-halo rows of every column (test geometry only).
__global__ void k_ywrap(double* __restrict__ A, Geo g) {
  const int64_t ncl = (int64_t)g.nx * Q;  // (column, population) pairs
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < ncl * 6;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t cl = i / 6;
    const int j = (int)(i % 6);
    double* col = A + cl * g.nyp + g.y0;
    if (j < 3)
      col[j - 3] = col[g.ly + j - 3];      // rows -3..-1 <- ly-3..ly-1
    else
      col[g.ly + (j - 3)] = col[j - 3];    // rows ly..ly+2 <- 0..2
  }
}

cudaError_t launch_pbc_wrap(const Geo& g, double* A, int bc, cudaStream_t s) {
  const int64_t cs2 = g.cs / 2;
  int blocks = (int)std::min<int64_t>((6 * cs2 + 255) / 256, 148 * 8);
  k_pbc_wrap<<<blocks, 256, 0, s>>>(reinterpret_cast<double2*>(A), g.lx, cs2);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess || bc != BC_PERIODIC) return e;
  return launch_ywrap(g, A, s);
}

cudaError_t launch_ywrap(const Geo& g, double* A, cudaStream_t s) {
  const int64_t n = (int64_t)g.nx * Q * 6;
  int blocks = (int)std::min<int64_t>((n + 255) / 256, 148 * 8);
  k_ywrap<<<blocks, 256, 0, s>>>(A, g);
  return cudaGetLastError();
}

// ---------------------------------------------------------------- gather
// Pull of the 37 populations of site (ix, y) from A (Eq. 1):
// f_l = A[ix - cx_l, l, y - cy_l].  With MIRROR, a source row beyond a wall
// (walls at y = -1/2 and y = ly - 1/2) is replaced by the specular image
// (G9 i): population refl(l) at row -1 - sy (bottom) or 2 ly - 1 - sy (top).
template <bool MIRROR>
__device__ __forceinline__ void gather(const double* __restrict__ A, const Geo& g, int ix, int y,
                                       double (&f)[Q]) {
  const int64_t b = (int64_t)ix * g.cs + g.y0 + y;
#pragma unroll
  for (int l = 0; l < Q; ++l) {
    int plane = l;
    int dy = -CY(l);
    if (MIRROR) {
      const int sy = y - CY(l);
      if (sy < 0) { plane = refl(l); dy = (-1 - sy) - y; }
      else if (sy >= g.ly) { plane = refl(l); dy = (2 * g.ly - 1 - sy) - y; }
    }
    const int64_t off = (int64_t)plane * g.nyp - (int64_t)CX(l) * g.cs + dy;
    f[l] = __ldg(A + b + off);
  }
}

// Same pull without MIRROR, with the 37 loads as ordered volatile coherent
// ld.global: ptxas may not sink them below the possibly-aliasing stores (it
// does with .nc), so all 37 loads are in flight before the first store (pure
// copy kernel: maximum memory-level parallelism per thread).
__device__ __forceinline__ void gather_ordered(const double* __restrict__ A, const Geo& g, int ix,
                                               int y, double (&f)[Q]) {
  const double* b = A + (int64_t)ix * g.cs + g.y0 + y;
#pragma unroll
  for (int l = 0; l < Q; ++l) {
    const double* p = b + ((int64_t)l * g.nyp - (int64_t)CX(l) * g.cs - CY(l));
    asm volatile("ld.global.f64 %0, [%1];" : "=d"(f[l]) : "l"(p));
  }
}

__device__ __forceinline__ void store_site(double* __restrict__ B, const Geo& g, int ix, int y,
                                           const double (&f)[Q]) {
  double* p = B + (int64_t)ix * g.cs + g.y0 + y;
#pragma unroll
  for (int l = 0; l < Q; ++l) p[(int64_t)l * g.nyp] = f[l];
}

// ---------------------------------------------------------------- propagate (§8a2)
// Raw pull over all physical sites; entries pulled from the y-halo rows read
// whatever those rows hold (zeros under walls, G10; wrapped rows if periodic).
__global__ void __launch_bounds__(TPB) k_propagate(const double* __restrict__ A,
                                                   double* __restrict__ B, Geo g) {
  const int y = blockIdx.x * TPB + threadIdx.x;
  const int ix = H + blockIdx.y;
  if (y >= g.ly) return;
  double f[Q];
  // all 37 loads in flight before the first store (the compiler would
  // otherwise pair load/store and keep only a few loads outstanding)
  gather_ordered(A, g, ix, y, f);
  asm volatile("" ::: "memory");
  store_site(B, g, ix, y, f);
}

cudaError_t launch_propagate(const Geo& g, const double* A, double* B, cudaStream_t s) {
  dim3 grid((g.ly + TPB - 1) / TPB, g.lx);
  k_propagate<<<grid, TPB, 0, s>>>(A, B, g);
  return cudaGetLastError();
}

// ---------------------------------------------------------------- bc (§8a3)
// One thread per wall-band site (3 rows per wall: both walls in
// one launch, they touch disjoint rows).  (i) mirror: for every population
// whose pull source lies beyond the wall, B <- A[refl, ix - cx, image row];
// (ii) thermal: rho = sequential sum, B_l <- rho K_l.
template <int BC>
__global__ void __launch_bounds__(TPB) k_bc(const double* __restrict__ A, double* __restrict__ B,
                                            Geo g) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= g.lx * 6) return;
  const int ix = H + t / 6;
  const int j = t % 6;
  const int y = j < 3 ? j : g.ly - 6 + j;
  double* p = B + (int64_t)ix * g.cs + g.y0 + y;
  // all 37 values of the site in registers (mirrored ones from A, the rest as
  // propagated into B), so no load waits on a store to the same address
  double f[Q];
#pragma unroll
  for (int l = 0; l < Q; ++l) {
    const int sy = y - CY(l);
    int ys = -1;
    if (sy < 0) ys = -1 - sy;
    else if (sy >= g.ly) ys = 2 * g.ly - 1 - sy;
    f[l] = ys >= 0 ? __ldg(A + (int64_t)(ix - CX(l)) * g.cs + (int64_t)refl(l) * g.nyp + g.y0 + ys)
                   : p[(int64_t)l * g.nyp];
  }
  if (BC == BC_THERMAL) thermal_wall(f, j < 3 ? 0 : 1);
#pragma unroll
  for (int l = 0; l < Q; ++l) p[(int64_t)l * g.nyp] = f[l];
}

cudaError_t launch_bc(const Geo& g, const double* A, double* B, int bc, cudaStream_t s) {
  if (bc == BC_PERIODIC) return cudaSuccess;
  const int n = g.lx * 6;
  constexpr int BC_TPB = 32;  // few, latency-bound threads: spread them over many SMs
  const int blocks = (n + BC_TPB - 1) / BC_TPB;
  if (bc == BC_THERMAL)
    k_bc<BC_THERMAL><<<blocks, BC_TPB, 0, s>>>(A, B, g);
  else
    k_bc<BC_ADIABATIC><<<blocks, BC_TPB, 0, s>>>(A, B, g);
  return cudaGetLastError();
}

// ---------------------------------------------------------------- collide (§8a4)
template <int COLL>
__device__ __forceinline__ void collide_any(double (&f)[Q], const Relax& r) {
  if (COLL == COLL_REGULARIZED)
    collide_site_reg(f, r);
  else
    collide_site(f, r);
}

template <int COLL>
__global__ void __launch_bounds__(TPB) k_collide(double* __restrict__ B, Geo g, Relax r) {
  const int y = blockIdx.x * TPB + threadIdx.x;
  const int ix = H + blockIdx.y;
  if (y >= g.ly) return;
  double* p = B + (int64_t)ix * g.cs + g.y0 + y;
  double f[Q];
#pragma unroll
  for (int l = 0; l < Q; ++l) f[l] = p[(int64_t)l * g.nyp];
  collide_any<COLL>(f, r);
#pragma unroll
  for (int l = 0; l < Q; ++l) p[(int64_t)l * g.nyp] = f[l];
}

cudaError_t launch_collide(const Geo& g, double* B, const Relax& r, int coll, cudaStream_t s) {
  dim3 grid((g.ly + TPB - 1) / TPB, g.lx);
  if (coll == COLL_REGULARIZED)
    k_collide<COLL_REGULARIZED><<<grid, TPB, 0, s>>>(B, g, r);
  else
    k_collide<COLL_BGK><<<grid, TPB, 0, s>>>(B, g, r);
  return cudaGetLastError();
}

// ---------------------------------------------------------------- fused pull step (§8a5)
// gather (+mirror) -> thermal wall -> collide -> store, A -> B in one pass:
// 296 B read + 296 B written per site.  Warps whose 32 rows are all at least
// 3 rows from both walls take the mirror-free gather (warp-uniform branch).
//
// Halo h — the exchange of the NEXT step done by the producing kernel: the
// blocks of the 3+3 border columns also store their result into the halo
// columns of a destination buffer: ix in [3,6) -> column ix + lx of h.dstL
// (the LEFT neighbour's next buffer: its right halo), ix in [lx, lx+3) ->
// column ix - lx of h.dstR (the RIGHT neighbour's left halo).  N = 1 wrap:
// dstL = dstR = own B.  Peer mode (N > 1, include/lb.h lb_set_peers): dstL /
// dstR are the neighbours' buffers mapped into this process (NVLink P2P
// stores), and before touching any halo the border blocks wait until both
// neighbours have completed the previous step (h.waitL/R >= *h.my_done): that
// both makes this rank's halo current and the neighbour's halo free to
// overwrite.  Bulk blocks never wait, so the exchange overlaps the bulk inside
// one grid (P:585-613 without a communication stream).
__device__ __forceinline__ unsigned long long ld_acquire_sys(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}

__device__ __forceinline__ unsigned long long globaltimer_ns() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

template <bool MIRROR>
__device__ __forceinline__ void gather_cg(const double* A, const Geo& g, int ix, int y, double (&f)[Q]) {
  // like gather<MIRROR> but with L2-coherent loads (halo data written by a
  // peer during this kernel's lifetime must not go through the .nc path)
  const int64_t b = (int64_t)ix * g.cs + g.y0 + y;
#pragma unroll
  for (int l = 0; l < Q; ++l) {
    int plane = l;
    int dy = -CY(l);
    if (MIRROR) {
      const int sy = y - CY(l);
      if (sy < 0) { plane = refl(l); dy = (-1 - sy) - y; }
      else if (sy >= g.ly) { plane = refl(l); dy = (2 * g.ly - 1 - sy) - y; }
    }
    const int64_t off = (int64_t)plane * g.nyp - (int64_t)CX(l) * g.cs + dy;
    f[l] = __ldcg(A + b + off);
  }
}

// Per-site contributions to the invariants: rho, j_x, j_y, E = 1/2 sum |c|^2 f.
__device__ __forceinline__ void site_invariants(const double (&f)[Q], double (&v)[4]) {
  double rho = 0.0, jx = 0.0, jy = 0.0, e = 0.0;
#pragma unroll
  for (int l = 0; l < Q; ++l) {
    rho = __dadd_rn(rho, f[l]);
    jx = __fma_rn((double)CX(l), f[l], jx);
    jy = __fma_rn((double)CY(l), f[l], jy);
    e = __fma_rn(0.5 * (double)c2(l), f[l], e);
  }
  v[0] = rho;
  v[1] = jx;
  v[2] = jy;
  v[3] = e;
}

// Fixed-order (deterministic) reduction of 4 sums + 1 min over a TPB block;
// the result is valid in thread 0.
__device__ __forceinline__ void block_sum4_min1(double (&v)[5]) {
  __shared__ double sm[TPB / 32][5];
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
#pragma unroll
    for (int k = 0; k < 4; ++k) v[k] = __dadd_rn(v[k], __shfl_xor_sync(0xffffffffu, v[k], o));
    v[4] = fmin(v[4], __shfl_xor_sync(0xffffffffu, v[4], o));
  }
  const int w = threadIdx.x >> 5;
  if ((threadIdx.x & 31) == 0)
#pragma unroll
    for (int k = 0; k < 5; ++k) sm[w][k] = v[k];
  __syncthreads();
  if (threadIdx.x == 0) {
#pragma unroll
    for (int k = 0; k < 5; ++k) v[k] = sm[0][k];
#pragma unroll
    for (int ww = 1; ww < TPB / 32; ++ww) {
#pragma unroll
      for (int k = 0; k < 4; ++k) v[k] = __dadd_rn(v[k], sm[ww][k]);
      v[4] = fmin(v[4], sm[ww][4]);
    }
  }
}

// MON: fused monitors — each block also reduces the invariants of the state it
// writes (post-collision rho, j, E and min rho of its 128 sites) into its slot
// mon[(ix - 3) * nblk_y + blockIdx.x][5]; lb_invariants then only sums slots.
template <int BC, int COLL, bool MON>
__global__ void __launch_bounds__(TPB, BC == BC_PERIODIC ? 3 : 4) k_step_fused(const double* __restrict__ A,
                                                    double* __restrict__ B, Geo g, Cols cols,
                                                    Relax r, Halo h, double* __restrict__ mon) {
  const int y = blockIdx.x * TPB + threadIdx.x;
  const int na = cols.xa1 - cols.xa0;
  const int by = cols.rev ? (int)gridDim.y - 1 - (int)blockIdx.y : (int)blockIdx.y;
  const int ix = by < na ? cols.xa0 + by : cols.xb0 + (by - na);
  const bool border = ix < 2 * H || ix >= g.lx;
  const bool peer_wait = h.waitL != nullptr && border;
  if (peer_wait) {  // block-uniform
    if (threadIdx.x == 0) {
      // watchdog: a neighbour that never signals (dead rank) must not hang the
      // GPU — after timeout_ns the block flags *status and proceeds (the step
      // result is then invalid; the host reports LB_EPEER at the next sync)
      const unsigned long long t0 = globaltimer_ns();
      const unsigned long long want = *h.my_done;  // steps this rank has completed
      while (ld_acquire_sys(h.waitL) < want || ld_acquire_sys(h.waitR) < want) {
        __nanosleep(128);
        if (h.timeout_ns && globaltimer_ns() - t0 > h.timeout_ns) {
          atomicExch(h.status, 1u);
          break;
        }
      }
    }
    __syncthreads();
  }
  const bool valid = y < g.ly;
  if (!MON && !valid) return;
  double f[Q];
  if (valid) {
    if (BC == BC_PERIODIC) {
      gather<false>(A, g, ix, y, f);
    } else {
      const int wy0 = blockIdx.x * TPB + (threadIdx.x & ~31);
      const bool interior = (wy0 >= 3) && (wy0 + 32 <= g.ly - 3);
      if (peer_wait) {
        if (interior) gather_cg<false>(A, g, ix, y, f);
        else gather_cg<true>(A, g, ix, y, f);
      } else if (interior) {
        gather<false>(A, g, ix, y, f);
      } else {
        gather<true>(A, g, ix, y, f);
      }
      if (!interior && BC == BC_THERMAL && (y < 3 || y >= g.ly - 3)) thermal_wall(f, y < 3 ? 0 : 1);
    }
    collide_any<COLL>(f, r);
    store_site(B, g, ix, y, f);
    if (h.dstL != nullptr && ix < 2 * H) store_site(h.dstL, g, ix + g.lx, y, f);
    if (h.dstR != nullptr && ix >= g.lx) store_site(h.dstR, g, ix - g.lx, y, f);
  }
  if (MON) {
    double v[5] = {0.0, 0.0, 0.0, 0.0, INFINITY};
    if (valid) {
      double s[4];
      site_invariants(f, s);
#pragma unroll
      for (int k = 0; k < 4; ++k) v[k] = s[k];
      v[4] = (s[0] != s[0]) ? -INFINITY : s[0];
    }
    block_sum4_min1(v);
    if (threadIdx.x == 0) {
      double* slot = mon + ((int64_t)(ix - H) * gridDim.x + blockIdx.x) * 5;
#pragma unroll
      for (int k = 0; k < 5; ++k) slot[k] = v[k];
    }
  }
  if (peer_wait) __threadfence_system();  // remote halo stores performed before the step signal
}

template <int COLL, bool MON>
void launch_fused_bc(const Geo& g, const double* A, double* B, int bc, const Relax& r, Cols cols,
                     const Halo& h, double* mon, dim3 grid, cudaStream_t s) {
  switch (bc) {
    case BC_THERMAL: k_step_fused<BC_THERMAL, COLL, MON><<<grid, TPB, 0, s>>>(A, B, g, cols, r, h, mon); break;
    case BC_ADIABATIC: k_step_fused<BC_ADIABATIC, COLL, MON><<<grid, TPB, 0, s>>>(A, B, g, cols, r, h, mon); break;
    default: k_step_fused<BC_PERIODIC, COLL, MON><<<grid, TPB, 0, s>>>(A, B, g, cols, r, h, mon); break;
  }
}

size_t monitor_slots(const Geo& g) { return (size_t)g.lx * ((g.ly + TPB - 1) / TPB); }

cudaError_t launch_step_fused(const Geo& g, const double* A, double* B, int bc, int coll,
                              const Relax& r, Cols cols, const Halo& h, double* mon, cudaStream_t s) {
  const int n = cols.count();
  if (n <= 0) return cudaSuccess;
  dim3 grid((g.ly + TPB - 1) / TPB, n);
  if (coll == COLL_REGULARIZED) {
    if (mon) launch_fused_bc<COLL_REGULARIZED, true>(g, A, B, bc, r, cols, h, mon, grid, s);
    else launch_fused_bc<COLL_REGULARIZED, false>(g, A, B, bc, r, cols, h, mon, grid, s);
  } else {
    if (mon) launch_fused_bc<COLL_BGK, true>(g, A, B, bc, r, cols, h, mon, grid, s);
    else launch_fused_bc<COLL_BGK, false>(g, A, B, bc, r, cols, h, mon, grid, s);
  }
  return cudaGetLastError();
}

// Step signal of peer mode: this rank's counter += 1 (only this rank writes
// it; system-scope release), after the fused kernel (stream order) and its
// border blocks' system fences.
__global__ void k_signal(unsigned long long* done) {
  __threadfence_system();
  const unsigned long long v = *done + 1;
  asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(done), "l"(v) : "memory");
}

cudaError_t launch_signal(unsigned long long* done, cudaStream_t s) {
  k_signal<<<1, 1, 0, s>>>(done);
  return cudaGetLastError();
}

// Initial halo fill of peer mode: A[0,3) <- left's A[lx, lx+3), A[lx+3, lx+6)
// <- right's A[3, 6) (full columns; the caller guarantees the neighbours'
// states are set and that no step is in flight).
__global__ void k_peer_pull(double2* __restrict__ A, const double2* L, const double2* R, int64_t lx,
                            int64_t cs2, Halo h) {
  // h.waitL != nullptr: first wait until both neighbours completed as many
  // launches as this rank (a pull right after a two-step launch: they may
  // still be writing the state we read), with the watchdog of the step kernel
  if (h.waitL) {
    if (threadIdx.x == 0) {
      const unsigned long long t0 = globaltimer_ns();
      const unsigned long long want = *h.my_done;
      while (ld_acquire_sys(h.waitL) < want || ld_acquire_sys(h.waitR) < want) {
        __nanosleep(128);
        if (h.timeout_ns && globaltimer_ns() - t0 > h.timeout_ns) {
          atomicExch(h.status, 1u);
          break;
        }
      }
    }
    __syncthreads();
  }
  const int64_t n = 3 * cs2;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < 2 * n;
       i += (int64_t)gridDim.x * blockDim.x) {
    if (i < n)
      A[i] = __ldcg(L + lx * cs2 + i);
    else
      A[(lx + 3) * cs2 + (i - n)] = __ldcg(R + 3 * cs2 + (i - n));
  }
}

cudaError_t launch_peer_pull(const Geo& g, double* A, const double* left_A, const double* right_A,
                             const Halo& wait, cudaStream_t s) {
  const int64_t cs2 = g.cs / 2;
  int blocks = (int)std::min<int64_t>((6 * cs2 + 255) / 256, 148 * 8);
  k_peer_pull<<<blocks, 256, 0, s>>>(reinterpret_cast<double2*>(A), reinterpret_cast<const double2*>(left_A),
                                     reinterpret_cast<const double2*>(right_A), g.lx, cs2, wait);
  return cudaGetLastError();
}

// ---------------------------------------------------------------- init / layout
// A := f_eq(rho, u, T) on physical sites; macro fields are [lx][ly].
__global__ void __launch_bounds__(TPB) k_init_macro(double* __restrict__ A, Geo g,
                                                    const double* __restrict__ rho,
                                                    const double* __restrict__ ux,
                                                    const double* __restrict__ uy,
                                                    const double* __restrict__ T) {
  const int y = blockIdx.x * TPB + threadIdx.x;
  const int x = blockIdx.y;
  if (y >= g.ly) return;
  const int64_t m = (int64_t)x * g.ly + y;
  double f[Q];
  feq_site(rho[m], ux[m], uy[m], T[m], f);
  store_site(A, g, H + x, y, f);
}

cudaError_t launch_init_macro(const Geo& g, double* A, const double* rho, const double* ux,
                              const double* uy, const double* T, cudaStream_t s) {
  dim3 grid((g.ly + TPB - 1) / TPB, g.lx);
  k_init_macro<<<grid, TPB, 0, s>>>(A, g, rho, ux, uy, T);
  return cudaGetLastError();
}

// Rayleigh-Taylor initial state on the device (lb_init_rt): the recipe of
// DESIGN.md §4 evaluated per site, then A := f_eq.  eps: the lx_total column
// jitters (device), x0: this rank's first global column.
__global__ void __launch_bounds__(TPB) k_init_rt(double* __restrict__ A, Geo g,
                                                 const double* __restrict__ eps, int lx_total, int x0,
                                                 double t_ref, double amp, double width) {
  const int y = blockIdx.x * TPB + threadIdx.x;
  const int x = blockIdx.y;
  if (y >= g.ly) return;
  const int xg = x0 + x;
  const double ampl = fmax(1.0, g.ly / 64.0);
  const double yi = (g.ly - 1) / 2.0 + ampl * cos(2.0 * M_PI * (double)xg / (double)lx_total) + eps[xg];
  const double T = t_ref * (1.0 + amp * tanh((yi - (double)y) / width));
  double f[Q];
  feq_site(t_ref / T, 0.0, 0.0, T, f);
  store_site(A, g, H + x, y, f);
}

cudaError_t launch_init_rt(const Geo& g, double* A, const double* eps, int lx_total, int x0, double t_ref,
                           double amp, double width, cudaStream_t s) {
  dim3 grid((g.ly + TPB - 1) / TPB, g.lx);
  k_init_rt<<<grid, TPB, 0, s>>>(A, g, eps, lx_total, x0, t_ref, amp, width);
  return cudaGetLastError();
}

// canonical [37][lx][ly] <-> internal physical sites
__global__ void k_canon_to_internal(const double* __restrict__ C, double* __restrict__ A, Geo g) {
  const int y = blockIdx.x * blockDim.x + threadIdx.x;
  const int x = blockIdx.y;
  const int l = blockIdx.z;
  if (y >= g.ly) return;
  A[(int64_t)(H + x) * g.cs + (int64_t)l * g.nyp + g.y0 + y] = C[((int64_t)l * g.lx + x) * g.ly + y];
}

__global__ void k_internal_to_canon(const double* __restrict__ A, double* __restrict__ C, Geo g) {
  const int y = blockIdx.x * blockDim.x + threadIdx.x;
  const int x = blockIdx.y;
  const int l = blockIdx.z;
  if (y >= g.ly) return;
  C[((int64_t)l * g.lx + x) * g.ly + y] = A[(int64_t)(H + x) * g.cs + (int64_t)l * g.nyp + g.y0 + y];
}

cudaError_t launch_canon_to_internal(const Geo& g, const double* canon, double* A, cudaStream_t s) {
  dim3 grid((g.ly + 255) / 256, g.lx, Q);
  k_canon_to_internal<<<grid, 256, 0, s>>>(canon, A, g);
  return cudaGetLastError();
}

cudaError_t launch_internal_to_canon(const Geo& g, const double* A, double* canon, cudaStream_t s) {
  dim3 grid((g.ly + 255) / 256, g.lx, Q);
  k_internal_to_canon<<<grid, 256, 0, s>>>(A, canon, g);
  return cudaGetLastError();
}

// ---------------------------------------------------------------- invariants
// Deterministic two-pass reduction: block partials (fixed tree) then one
// block sums the partials in a fixed order.  Per site: rho, jx, jy,
// E = 1/2 sum |c|^2 f, and min rho.
constexpr int RED_TPB = 256;

// Failure detection ("numerical blow-up"): a final
// invariants result with a NaN sum or min rho <= 0 (NaN densities arrive as
// -inf) sets the context's sticky device flag, which lb_sync reports as
// LB_ENONPHYS — so the asynchronous monitored path needs no host-side check.
__device__ __forceinline__ void flag_nonphysical(const double (&v)[5], unsigned int* flag) {
  const bool bad = v[0] != v[0] || v[1] != v[1] || v[2] != v[2] || v[3] != v[3] || !(v[4] > 0.0);
  if (bad && flag) atomicOr(flag, 1u);
}

__device__ __forceinline__ void block_reduce5(double (&v)[5], double* sm) {
  const int t = threadIdx.x;
#pragma unroll
  for (int k = 0; k < 5; ++k) sm[k * RED_TPB + t] = v[k];
  __syncthreads();
  for (int w = RED_TPB / 2; w > 0; w >>= 1) {
    if (t < w) {
#pragma unroll
      for (int k = 0; k < 4; ++k) sm[k * RED_TPB + t] = sm[k * RED_TPB + t] + sm[k * RED_TPB + t + w];
      sm[4 * RED_TPB + t] = fmin(sm[4 * RED_TPB + t], sm[4 * RED_TPB + t + w]);
    }
    __syncthreads();
  }
#pragma unroll
  for (int k = 0; k < 5; ++k) v[k] = sm[k * RED_TPB];
}

__global__ void __launch_bounds__(RED_TPB) k_invariants_partial(const double* __restrict__ A, Geo g,
                                                                double* __restrict__ part) {
  __shared__ double sm[5 * RED_TPB];
  const int ix = H + blockIdx.x;
  double v[5] = {0.0, 0.0, 0.0, 0.0, INFINITY};
  for (int y = threadIdx.x; y < g.ly; y += RED_TPB) {
    const double* p = A + (int64_t)ix * g.cs + g.y0 + y;
    double rho = 0.0, jx = 0.0, jy = 0.0, e = 0.0;
#pragma unroll
    for (int l = 0; l < Q; ++l) {
      const double f = p[(int64_t)l * g.nyp];
      rho = __dadd_rn(rho, f);
      jx = __fma_rn((double)CX(l), f, jx);
      jy = __fma_rn((double)CY(l), f, jy);
      e = __fma_rn(0.5 * (double)c2(l), f, e);
    }
    v[0] += rho;
    v[1] += jx;
    v[2] += jy;
    v[3] += e;
    // NaN propagates through fmin only if both are NaN; flag NaN as -inf
    v[4] = (rho != rho) ? -INFINITY : fmin(v[4], rho);
  }
  block_reduce5(v, sm);
  if (threadIdx.x == 0)
#pragma unroll
    for (int k = 0; k < 5; ++k) part[(int64_t)blockIdx.x * 5 + k] = v[k];
}

__global__ void __launch_bounds__(RED_TPB) k_invariants_final(const double* __restrict__ part,
                                                              int nb, double* __restrict__ out,
                                                              unsigned int* flag) {
  __shared__ double sm[5 * RED_TPB];
  double v[5] = {0.0, 0.0, 0.0, 0.0, INFINITY};
  for (int b = threadIdx.x; b < nb; b += RED_TPB) {
#pragma unroll
    for (int k = 0; k < 4; ++k) v[k] += part[(int64_t)b * 5 + k];
    const double m = part[(int64_t)b * 5 + 4];
    v[4] = (m != m || m == -INFINITY) ? -INFINITY : fmin(v[4], m);
  }
  block_reduce5(v, sm);
  if (threadIdx.x == 0) {
#pragma unroll
    for (int k = 0; k < 5; ++k) out[k] = v[k];
    flag_nonphysical(v, flag);
  }
}

size_t invariants_scratch(const Geo& g) { return (size_t)g.lx * 5; }

cudaError_t launch_invariants(const Geo& g, const double* A, double* partials, double* out,
                              unsigned int* flag, cudaStream_t s) {
  k_invariants_partial<<<g.lx, RED_TPB, 0, s>>>(A, g, partials);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  k_invariants_final<<<1, RED_TPB, 0, s>>>(partials, g.lx, out, flag);
  return cudaGetLastError();
}

// Sum of the fused-monitor slots in ONE launch: block b reduces the fixed slot
// range [b*chunk, (b+1)*chunk) (one slot per thread at 1920x2048), writes its
// partial, and the last block to arrive (ticket) sums the partials in block
// order — so the result is deterministic and no single block walks all slots
// (a one-block pass over 30k slots cost 56 us per step).
__global__ void __launch_bounds__(RED_TPB) k_monitor_reduce(const double* __restrict__ mon, int nslots,
                                                            double* part, unsigned int* ticket,
                                                            double* out, unsigned int* flag) {
  __shared__ double sm[5 * RED_TPB];
  __shared__ bool last;
  const int t = threadIdx.x;
  const int chunk = (nslots + (int)gridDim.x - 1) / (int)gridDim.x;
  const int lo = (int)blockIdx.x * chunk, hi = min(lo + chunk, nslots);
  double v[5] = {0.0, 0.0, 0.0, 0.0, INFINITY};
  for (int b = lo + t; b < hi; b += RED_TPB) {
#pragma unroll
    for (int k = 0; k < 4; ++k) v[k] += mon[(int64_t)b * 5 + k];
    const double m = mon[(int64_t)b * 5 + 4];
    v[4] = (m != m || m == -INFINITY) ? -INFINITY : fmin(v[4], m);
  }
  block_reduce5(v, sm);
  if (t == 0) {
#pragma unroll
    for (int k = 0; k < 5; ++k) part[(int64_t)blockIdx.x * 5 + k] = v[k];
    __threadfence();
    last = atomicAdd(ticket, 1u) == gridDim.x - 1;
  }
  __syncthreads();
  if (!last) return;
  __threadfence();
  double w[5] = {0.0, 0.0, 0.0, 0.0, INFINITY};
  for (int b = t; b < (int)gridDim.x; b += RED_TPB) {
#pragma unroll
    for (int k = 0; k < 4; ++k) w[k] += __ldcg(part + (int64_t)b * 5 + k);
    const double m = __ldcg(part + (int64_t)b * 5 + 4);
    w[4] = (m != m || m == -INFINITY) ? -INFINITY : fmin(w[4], m);
  }
  __syncthreads();  // sm reused
  block_reduce5(w, sm);
  if (t == 0) {
#pragma unroll
    for (int k = 0; k < 5; ++k) out[k] = w[k];
    flag_nonphysical(w, flag);
    *ticket = 0u;  // ready for the next launch (stream-ordered)
  }
}

// Both states of a two-step launch in ONE single-block launch (nslots per
// set, set 1 at mon + 5 nslots): out[0..4] = set 0, out[5..9] = set 1.
// Launched with programmatic dependent launch after the two-step kernel
// (pdl): it may start while that kernel drains and waits for it before
// reading the partials; the next two-step launch may start during it.
__global__ void __launch_bounds__(RED_TPB) k_monitor_reduce_pair(const double* __restrict__ mon, int nslots,
                                                                 double* out, unsigned int* flag) {
  asm volatile("griddepcontrol.launch_dependents;");
  asm volatile("griddepcontrol.wait;" ::: "memory");
  __shared__ double sm[5 * RED_TPB];
  const int t = threadIdx.x;
  for (int set = 0; set < 2; ++set) {
    const double* m0 = mon + (int64_t)set * nslots * 5;
    double v[5] = {0.0, 0.0, 0.0, 0.0, INFINITY};
    for (int b = t; b < nslots; b += RED_TPB) {
#pragma unroll
      for (int k = 0; k < 4; ++k) v[k] += m0[(int64_t)b * 5 + k];
      const double m = m0[(int64_t)b * 5 + 4];
      v[4] = (m != m || m == -INFINITY) ? -INFINITY : fmin(v[4], m);
    }
    block_reduce5(v, sm);
    if (t == 0) {
#pragma unroll
      for (int k = 0; k < 5; ++k) out[set * 5 + k] = v[k];
      flag_nonphysical(v, flag);
    }
    __syncthreads();  // sm reused
  }
}

cudaError_t launch_monitor_reduce_pair(const double* mon, int64_t nslots, double* out, unsigned int* flag,
                                       cudaStream_t s, bool pdl) {
  if (pdl) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(1);
    cfg.blockDim = dim3(RED_TPB);
    cfg.stream = s;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, k_monitor_reduce_pair, mon, (int)nslots, out, flag);
  }
  k_monitor_reduce_pair<<<1, RED_TPB, 0, s>>>(mon, (int)nslots, out, flag);
  return cudaGetLastError();
}

static int monitor_reduce_blocks(int64_t nslots) {
  const int64_t b = (nslots + RED_TPB - 1) / RED_TPB;
  return (int)(b < 1 ? 1 : (b > MON_REDUCE_MAX_BLOCKS ? MON_REDUCE_MAX_BLOCKS : b));
}

cudaError_t launch_monitor_reduce(const double* mon, int64_t nslots, double* part, unsigned int* ticket,
                                  double* out, unsigned int* flag, cudaStream_t s) {
  k_monitor_reduce<<<monitor_reduce_blocks(nslots), RED_TPB, 0, s>>>(mon, (int)nslots, part, ticket, out, flag);
  return cudaGetLastError();
}

// ---------------------------------------------------------------- fused step, TMA-staged
// Same step as k_step_fused, but the 37 +-3-row windows of a 254-row tile are
// brought into shared memory by TMA (one elected thread, one mbarrier; box
// starts rounded down to 16 bytes, see lb_tma.cu) and each thread reads its
// site's populations from smem.  Wall-band sites replace the populations whose
// pull source lies beyond the wall with the specular image read from global
// memory (the image rows can fall outside the loaded windows).
constexpr int FT_TILE = 254;
constexpr int FT_ROW = 256;
constexpr int FT_THREADS = 256;
constexpr size_t FT_SMEM = (size_t)Q * FT_ROW * sizeof(double) + 16;

__device__ __forceinline__ uint32_t smem_addr(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

template <int BC, int COLL>
__global__ void __launch_bounds__(FT_THREADS, 2) k_step_fused_tma(const __grid_constant__ CUtensorMap src,
                                                                  const double* __restrict__ A,
                                                                  double* __restrict__ B, Geo g, Relax r,
                                                                  Halo h) {
  extern __shared__ __align__(1024) double sm[];
  uint64_t* bar = reinterpret_cast<uint64_t*>(sm + Q * FT_ROW);
  const uint32_t b = smem_addr(bar);
  const int ix = H + (int)blockIdx.y;
  const int t = threadIdx.x;
  const int y = (int)blockIdx.x * FT_TILE + t;  // physical row of this thread
  const int r0 = g.y0 + (int)blockIdx.x * FT_TILE;
  if (t == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(b));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (t == 0) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(b),
                 "r"((uint32_t)(Q * (FT_TILE + 2) * sizeof(double))));
#pragma unroll
    for (int l = 0; l < Q; ++l) {
      const int base = r0 - CY(l) - (CY(l) & 1);
      asm volatile(
          "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes"
          " [%0], [%1, {%2, %3, %4}], [%5];" ::"r"(smem_addr(sm + l * FT_ROW)),
          "l"(&src), "r"(base), "r"(l), "r"(ix - CX(l)), "r"(b)
          : "memory");
    }
  }
  asm volatile(
      "{\n"
      " .reg .pred p;\n"
      "WAIT_%=:\n"
      " mbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n"
      " @!p bra WAIT_%=;\n"
      "}\n" ::"r"(b)
      : "memory");
  if (t >= FT_TILE || y >= g.ly) return;
  double f[Q];
#pragma unroll
  for (int l = 0; l < Q; ++l) f[l] = sm[l * FT_ROW + t + (CY(l) & 1)];
  if (y < 3 || y >= g.ly - 3) {
    const int64_t colbase = (int64_t)g.y0;
#pragma unroll
    for (int l = 0; l < Q; ++l) {
      const int sy = y - CY(l);
      int ys = -1;
      if (sy < 0) ys = -1 - sy;
      else if (sy >= g.ly) ys = 2 * g.ly - 1 - sy;
      if (ys >= 0) f[l] = __ldg(A + (int64_t)(ix - CX(l)) * g.cs + (int64_t)refl(l) * g.nyp + colbase + ys);
    }
    if (BC == BC_THERMAL) thermal_wall(f, y < 3 ? 0 : 1);
  }
  collide_any<COLL>(f, r);
  store_site(B, g, ix, y, f);
  if (h.dstL != nullptr && ix < 2 * H) store_site(h.dstL, g, ix + g.lx, y, f);
  if (h.dstR != nullptr && ix >= g.lx) store_site(h.dstR, g, ix - g.lx, y, f);
}

template <int BC, int COLL>
cudaError_t launch_ft(const Geo& g, const TmaMaps* t, int src_buf, const double* A, double* B, const Relax& r,
                      const Halo& h, cudaStream_t s) {
  // opt-in shared memory is a per-device function attribute: set it once per device
  static unsigned long long done_mask = 0;
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  if (dev >= 64 || !(done_mask >> dev & 1ull)) {
    e = cudaFuncSetAttribute(k_step_fused_tma<BC, COLL>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)FT_SMEM);
    if (e != cudaSuccess) return e;
    if (dev < 64) done_mask |= 1ull << dev;
  }
  dim3 grid((g.ly + FT_TILE - 1) / FT_TILE, g.lx);
  k_step_fused_tma<BC, COLL><<<grid, FT_THREADS, FT_SMEM, s>>>(t->load[src_buf], A, B, g, r, h);
  return cudaGetLastError();
}

cudaError_t launch_step_fused_tma(const Geo& g, const TmaMaps* t, int src_buf, const double* A, double* B,
                                  int bc, int coll, const Relax& r, const Halo& h, cudaStream_t s) {
  if (bc == BC_THERMAL)
    return coll == COLL_REGULARIZED ? launch_ft<BC_THERMAL, COLL_REGULARIZED>(g, t, src_buf, A, B, r, h, s)
                                    : launch_ft<BC_THERMAL, COLL_BGK>(g, t, src_buf, A, B, r, h, s);
  return coll == COLL_REGULARIZED ? launch_ft<BC_ADIABATIC, COLL_REGULARIZED>(g, t, src_buf, A, B, r, h, s)
                                  : launch_ft<BC_ADIABATIC, COLL_BGK>(g, t, src_buf, A, B, r, h, s);
}

}  // namespace lbk
