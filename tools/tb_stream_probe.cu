// tb_stream_probe.cu — the data movement of the two-step kernel alone
// (development tool, not on the product path; DESIGN.md §8 "where the
// two-step kernel stands").
//
// k_step2_tb's memory half: per CTA (one per SM) a sweep over columns of one
// 104-row strip; per column 7 TMA group boxes {116 rows, 3/5/7 populations,
// 1 column} of state n into a ring of state-n buffers, and 37 x 104 rows of
// state n+2 written back.  This probe keeps exactly that traffic (same layout,
// strip layout, boxes, work split) and drops everything else — no gathers, no
// state-(n+1) ring, no collision — so that the number of buffers in flight
// (NBUF 1..6, up to 206 KB per SM) and the store path can be varied freely:
//   store 0: 4 warps copy the 104 output rows of each population from the
//            buffer to global memory with 8-byte stores (the kernel's STG path)
//   store 1: one thread per population issues a 832-byte bulk copy
//            shared -> global (cp.async.bulk, no register round trip)
//   store 2: no stores (reads alone);  store 3: stores only, no loads
// and the loads as (load 0) the kernel's 7 TMA group boxes per column, (1) one
// 1-D bulk copy per population window, (2) 16-byte cp.async (LDGSTS) by the
// consumer threads, which refill the buffer they just used (PROBE_LOAD=n: one mode)
// plus a plain double2 copy of the same 1.19 GB state (the copy roof on the
// same box).  Reports requested bytes / time; ncu gives the DRAM bytes.
//
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo --expt-relaxed-constexpr -o tools/tb_stream_probe tools/tb_stream_probe.cu -lcuda
// ./tools/tb_stream_probe [lx ly reps]   (prints one JSON line per configuration)
#include <cuda.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <vector>

#define CK(x)                                                                                  \
  do {                                                                                         \
    cudaError_t e_ = (x);                                                                      \
    if (e_ != cudaSuccess) {                                                                   \
      fprintf(stderr, "%s:%d %s: %s\n", __FILE__, __LINE__, #x, cudaGetErrorString(e_));      \
      exit(1);                                                                                 \
    }                                                                                          \
  } while (0)

#ifndef PROBE_HT  // strip height (HT = 244: 256-row boxes, 2 buffers at most)
#define PROBE_HT 104
#endif
constexpr int Q = 37, HT = PROBE_HT, RB = HT + 12, H = 3, Y0 = 16, NG = 7;
constexpr int NCONS = (HT + 31) / 32 * 32;  // consumer threads (one per output row)
__host__ __device__ constexpr int gfirst(int g) { return g == 0 ? 0 : g == 1 ? 3 : g == 2 ? 8 : g == 3 ? 15 : g == 4 ? 22 : g == 5 ? 29 : g == 6 ? 34 : 37; }
__host__ __device__ constexpr int gn(int g) { return g == 0 || g == 6 ? 3 : (g == 1 || g == 5 ? 5 : 7); }
__host__ __device__ constexpr int gcls(int g) { return gn(g) == 3 ? 0 : (gn(g) == 5 ? 1 : 2); }
__host__ __device__ constexpr int goff(int g) {  // 128-byte aligned group slabs, as in lb_tb.cu
  int o = 0;
  for (int h = 0; h < g; ++h) o += (gn(h) * RB + 15) / 16 * 16;
  return o;
}
constexpr int BUFD = goff(NG);  // doubles per state-n buffer
constexpr int MAXBUF = HT > 200 ? 2 : 6;

struct Maps {
  CUtensorMap m[12], m2[3];  // m[3 (depth - 1) + class]: boxes of depth 1-4 columns  // 3-D {rows, 37, columns} and 2-D {rows, 37 columns} maps
};

__device__ __forceinline__ uint32_t s32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t par) {
  asm volatile(
      "{\n .reg .pred p;\nW_%=:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n @!p bra W_%=;\n}\n" ::"r"(
          bar),
      "r"(par)
      : "memory");
}
__host__ __device__ inline int strip_ya(int s, int ns, int ly) {  // lb_tb.cu's strip layout
  if (s == ns - 1) return ((ly - HT + 1) & ~1) > 0 ? ((ly - HT + 1) & ~1) : 0;
  if (s == ns - 2) {
    const int lim = (ly - 6 - HT) & ~1;
    return s * HT < lim ? s * HT : lim;
  }
  return s * HT;
}

// warps [0, NCONS / 32): consumers (stores), the last warp: producer (7 issuing lanes)
__global__ void __launch_bounds__(NCONS + 32, 1)
    k_probe(const __grid_constant__ Maps mp, const double* __restrict__ A, double* __restrict__ B, int lx, int ly,
            int nyp, int ns, int nbuf, int store, int aligned, int load, int tma_mask) {
  extern __shared__ __align__(128) double sm[];
  uint64_t* full = reinterpret_cast<uint64_t*>(sm + MAXBUF * BUFD);
  uint64_t* empty = full + MAXBUF;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int64_t cs = (int64_t)Q * nyp;
  if (tid == 0) {
    for (int i = 0; i < nbuf; ++i) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(s32(full + i)), "r"(load == 2 ? NCONS : load == 3 ? NCONS + 1 : 1));
      asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(s32(empty + i)), "r"(store == 1 ? 1 : NCONS));
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  const int64_t U = (int64_t)ns * lx;
  int64_t u = U * blockIdx.x / gridDim.x;
  int64_t ue = U * (blockIdx.x + 1) / gridDim.x;
  if (aligned) {  // CTA k: strip k % ns, column range k / ns of gridDim.x / ns equal ranges
    const int R = gridDim.x / ns, s = blockIdx.x % ns, r = blockIdx.x / ns;
    u = (int64_t)s * lx + (int64_t)lx * r / R;
    ue = (int64_t)s * lx + (int64_t)lx * (r + 1) / R;
  }
  uint32_t k = 0;  // buffer uses of this CTA
  while (u < ue) {
    const int s = (int)(u / lx), x0 = (int)(u % lx);
    const int x1 = (int)std::min<int64_t>(lx, x0 + (ue - u));
    u += x1 - x0;
    const int ya = strip_ya(s, ns, ly), xs = H + x0, W = x1 - x0;
    const int nit = W + 6;  // load columns c1 = xs - 3 + t (the kernel's phase-1 iterations)
    // load 2: the consumer threads refill the buffer they just used with 16-byte
    // cp.async (LDGSTS): warp w takes the populations l = w mod 4, 58 chunks each
    auto ldgsts = [&](int t) {
      const uint32_t kb = k + t, b = kb % nbuf;
      int colg[NG];
#pragma unroll
      for (int g = 0; g < NG; ++g) {
        int c = xs - 3 + t - (3 - g);
        if (c < H) c += lx;
        else if (c >= lx + H) c -= lx;
        colg[g] = c;
      }
      const uint32_t sb = s32(sm + b * BUFD);
#pragma unroll
      for (int l = 0; l < Q; ++l) {
        if ((l & 3) != warp) continue;
        int g = 0;
#pragma unroll
        for (int h = 1; h < NG; ++h) g += l >= gfirst(h) ? 1 : 0;
        if (load == 3 && ((tma_mask >> g) & 1)) continue;
        const double* src = A + ((int64_t)colg[g] * Q + l) * nyp + Y0 + ya - 6;
        const uint32_t dst = sb + 8u * (uint32_t)(goff(g) + (l - gfirst(g)) * RB);
        asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(dst + 16u * lane), "l"(src + 2 * lane) : "memory");
        if (lane < RB / 2 - 32)
          asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(dst + 16u * (32 + lane)), "l"(src + 2 * (32 + lane))
                       : "memory");
      }
      asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];" ::"r"(s32(full + b)) : "memory");
    };
    if ((load == 2 || load == 3) && warp < NCONS / 32) {
      asm volatile("bar.sync 1, %0;" ::"r"(NCONS) : "memory");  // the previous sweep's reads are done
      for (int t = 0; t < nbuf && t < nit; ++t) ldgsts(t);
    }
    if (warp == NCONS / 32) {
      if (load != 2 && lane < NG && (load != 3 || ((tma_mask >> lane) & 1) || lane == 0))
        for (int t = 0; t < nit; ++t) {
          const uint32_t kb = k + t, b = kb % nbuf;
          if (kb >= (uint32_t)nbuf) mbar_wait(s32(empty + b), ((kb / nbuf) - 1) & 1);
          if (store == 3) {
            if (lane == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(s32(full + b)) : "memory");
            continue;
          }
          if (lane == 0) {
            uint32_t npop = Q;
            if (load == 3) {
              npop = 0;
              for (int g = 0; g < NG; ++g) npop += ((tma_mask >> g) & 1) ? gn(g) : 0;
            }
            asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(s32(full + b)),
                         "r"(npop * RB * 8u));
          }
          if (load == 3 && !((tma_mask >> lane) & 1)) continue;
          if (load == 1) {  // one 1-D bulk copy per population window (928 contiguous bytes)
            for (int l = lane; l < Q; l += NG) {
              int g = 0;
#pragma unroll
              for (int h = 1; h < NG; ++h) g += l >= gfirst(h) ? 1 : 0;
              int col = xs - 3 + t - (3 - g);
              if (col < H) col += lx;
              else if (col >= lx + H) col -= lx;
              asm volatile(
                  "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                      s32(sm + b * BUFD + goff(g) + (l - gfirst(g)) * RB)),
                  "l"(A + ((int64_t)col * Q + l) * nyp + Y0 + ya - 6), "r"((uint32_t)(RB * 8)), "r"(s32(full + b))
                  : "memory");
            }
            continue;
          }
          int col = xs - 3 + t - (3 - lane) - H;  // group g = lane has cx = 3 - g
          col = ((col % lx) + lx) % lx + H;
          if (load == 4)  // the same box through a 2-D map: planes col * 37 + l have the uniform stride nyp
            asm volatile(
                "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], "
                "[%4];" ::"r"(s32(sm + b * BUFD + goff(lane))),
                "l"(&mp.m2[gcls(lane)]), "r"(Y0 + ya - 6), "r"(col * Q + gfirst(lane)), "r"(s32(full + b))
                : "memory");
          else
            asm volatile(
                "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, "
                "%4}], [%5];" ::"r"(s32(sm + b * BUFD + goff(lane))),
                "l"(&mp.m[gcls(lane)]), "r"(Y0 + ya - 6), "r"(gfirst(lane)), "r"(col), "r"(s32(full + b))
                : "memory");
        }
    } else {
      for (int t = 0; t < nit; ++t) {
        const uint32_t kb = k + t, b = kb % nbuf;
        mbar_wait(s32(full + b), (kb / nbuf) & 1);
        const int c2 = xs - 3 + t - 3;  // an output column (W of them per sweep)
        const bool out = t >= 6;
        const double* buf = sm + b * BUFD;
        if (store == 0 || store == 3) {
          if (out && tid < HT && ya + tid < ly) {
            double* p = B + (int64_t)c2 * cs + Y0 + ya + tid;
#pragma unroll
            for (int g = 0; g < NG; ++g)
#pragma unroll
              for (int j = 0; j < gn(g); ++j) p[(int64_t)(gfirst(g) + j) * nyp] = buf[goff(g) + j * RB + 6 + tid];
          }
          if (load == 2 || load == 3) {
            asm volatile("bar.sync 1, %0;" ::"r"(NCONS) : "memory");
            if (load == 3) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(s32(empty + b)) : "memory");
            if (t + nbuf < nit) ldgsts(t + nbuf);
          } else
            asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(s32(empty + b)) : "memory");
        } else if (store == 1) {
          if (warp == 0) {
            if (out)
              for (int l = lane; l < Q; l += 32) {
                int g = 0;
                while (l >= gfirst(g + 1)) ++g;
                const int rows = ly - ya < HT ? ly - ya : HT;
                asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(
                                 B + (int64_t)c2 * cs + (int64_t)l * nyp + Y0 + ya),
                             "r"(s32(buf + goff(g) + (l - gfirst(g)) * RB + 6)), "r"((uint32_t)(rows * 8))
                             : "memory");
              }
            asm volatile("cp.async.bulk.commit_group;" ::: "memory");
            asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
            __syncwarp();
            if (lane == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(s32(empty + b)) : "memory");
          }
        } else {  // store == 2: reads only
          if (load == 2 || load == 3) {
            asm volatile("bar.sync 1, %0;" ::"r"(NCONS) : "memory");
            if (load == 3) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(s32(empty + b)) : "memory");
            if (t + nbuf < nit) ldgsts(t + nbuf);
          } else
            asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(s32(empty + b)) : "memory");
        }
      }
    }
    k += nit;
  }
  if (store == 1 && warp == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

// Boxes of DEPTH consecutive columns: one TMA box per group loads the windows of
// DEPTH iterations at once ({116 rows, n populations, DEPTH columns}), DEPTH
// output columns stored per iteration — tests whether the TMA cost is per box
// (fewer, bigger boxes help) or per row (they do not).
__host__ __device__ constexpr int goffd(int g, int depth) {
  int o = 0;
  for (int h = 0; h < g; ++h) o += (depth * gn(h) * RB + 15) / 16 * 16;
  return o;
}
template <int DEPTH>
__global__ void __launch_bounds__(NCONS + 32, 1)
    k_probe_deep(const __grid_constant__ Maps mp, double* __restrict__ B, int lx, int ly, int nyp, int ns, int nbuf,
                 int store) {
  extern __shared__ __align__(128) double sm[];
  constexpr int BD = goffd(NG, DEPTH);
  uint64_t* full = reinterpret_cast<uint64_t*>(sm + MAXBUF * BUFD);
  uint64_t* empty = full + MAXBUF;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int64_t cs = (int64_t)Q * nyp;
  if (tid == 0) {
    for (int i = 0; i < nbuf; ++i) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(s32(full + i)));
      asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(s32(empty + i)), "r"(NCONS));
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  const int64_t U = (int64_t)ns * lx;
  int64_t u = U * blockIdx.x / gridDim.x;
  const int64_t ue = U * (blockIdx.x + 1) / gridDim.x;
  uint32_t k = 0;
  while (u < ue) {
    const int s = (int)(u / lx), x0 = (int)(u % lx);
    const int x1 = (int)std::min<int64_t>(lx, x0 + (ue - u));
    u += x1 - x0;
    const int ya = strip_ya(s, ns, ly), xs = H + x0, W = x1 - x0;
    const int nit = (W + 6 + DEPTH - 1) / DEPTH;  // iterations of DEPTH load columns
    if (warp == NCONS / 32) {
      if (lane < NG)
        for (int t = 0; t < nit; ++t) {
          const uint32_t kb = k + t, b = kb % nbuf;
          if (kb >= (uint32_t)nbuf) mbar_wait(s32(empty + b), ((kb / nbuf) - 1) & 1);
          if (lane == 0)
            asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(s32(full + b)),
                         "r"((uint32_t)(DEPTH * Q * RB * 8)));
          int col = xs - 3 + DEPTH * t - (3 - lane);  // first of DEPTH columns (no wrap: interior only)
          if (col < H) col += lx;
          if (col + DEPTH > lx + H) col = lx + H - DEPTH;  // (clamped at the right edge: bytes, not values, matter)
          asm volatile(
              "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, "
              "%4}], [%5];" ::"r"(s32(sm + b * BD + goffd(lane, DEPTH))),
              "l"(&mp.m[3 * (DEPTH - 1) + gcls(lane)]), "r"(Y0 + ya - 6), "r"(gfirst(lane)), "r"(col),
              "r"(s32(full + b))
              : "memory");
        }
    } else {
      for (int t = 0; t < nit; ++t) {
        const uint32_t kb = k + t, b = kb % nbuf;
        mbar_wait(s32(full + b), (kb / nbuf) & 1);
        const double* buf = sm + b * BD;
        if (store == 0 && tid < HT && ya + tid < ly)
#pragma unroll
          for (int j = 0; j < DEPTH; ++j) {
            const int c2 = xs - 6 + DEPTH * t + j;
            if (c2 < xs || c2 >= xs + W) continue;
            double* p = B + (int64_t)c2 * cs + Y0 + ya + tid;
#pragma unroll
            for (int g = 0; g < NG; ++g)
#pragma unroll
              for (int i = 0; i < gn(g); ++i)
                p[(int64_t)(gfirst(g) + i) * nyp] = buf[goffd(g, DEPTH) + (j * gn(g) + i) * RB + 6 + tid];
          }
        asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(s32(empty + b)) : "memory");
      }
    }
    k += nit;
  }
}

// Stores alone, the kernel's pattern (37 x 104-row runs per output column of a
// strip), issued by NW warps per CTA: 4 = the kernel (one row per thread, 37
// stores), 8 / 16 = the populations split between 2 / 4 warp groups.
template <int NW>
__global__ void __launch_bounds__(NW * 32, 1) k_store_only(double* __restrict__ B, int lx, int ly, int nyp, int ns) {
  constexpr int GROUPS = NW / 4;
  const int tid = threadIdx.x, row = tid & 127, grp = tid >> 7;
  const int64_t cs = (int64_t)Q * nyp;
  const int64_t U = (int64_t)ns * lx;
  int64_t u = U * blockIdx.x / gridDim.x;
  const int64_t ue = U * (blockIdx.x + 1) / gridDim.x;
  const double v = 1.0 + tid;
  while (u < ue) {
    const int s = (int)(u / lx), x0 = (int)(u % lx);
    const int x1 = (int)std::min<int64_t>(lx, x0 + (ue - u));
    u += x1 - x0;
    const int ya = strip_ya(s, ns, ly);
    if (row < HT && ya + row < ly)
      for (int c = x0; c < x1; ++c) {
        double* p = B + (int64_t)(H + c) * cs + Y0 + ya + row;
#pragma unroll
        for (int l = 0; l < Q; ++l)
          if (l % GROUPS == grp) p[(int64_t)l * nyp] = v;
      }
  }
}

__global__ void k_copy(const double2* __restrict__ a, double2* __restrict__ b, int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    b[i] = a[i];
}

int main(int argc, char** argv) {
  const int lx = argc > 1 ? atoi(argv[1]) : 1920, ly = argc > 2 ? atoi(argv[2]) : 2048;
  const int reps = argc > 3 ? atoi(argv[3]) : 20;
  const int nyp = (Y0 + ly + 3 + 15) / 16 * 16;
  const int64_t cols = lx + 2 * H, n = cols * Q * (int64_t)nyp;
  double *A, *B;
  CK(cudaMalloc(&A, n * 8));
  CK(cudaMalloc(&B, n * 8));
  CK(cudaMemset(A, 0, n * 8));
  CK(cudaMemset(B, 0, n * 8));
  Maps mp;
  for (int c = 0; c < 3; ++c) {
    cuuint64_t dims[3] = {(cuuint64_t)nyp, (cuuint64_t)Q, (cuuint64_t)cols};
    cuuint64_t str[2] = {(cuuint64_t)nyp * 8, (cuuint64_t)Q * nyp * 8};
    for (int d = 2; d <= 4; ++d) {
      cuuint32_t boxd[3] = {RB, (cuuint32_t)(3 + 2 * c), (cuuint32_t)d}, esd[3] = {1, 1, 1};
      if (cuTensorMapEncodeTiled(&mp.m[3 * (d - 1) + c], CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, A, dims, str, boxd, esd,
                                 CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                                 CU_TENSOR_MAP_L2_PROMOTION_L2_64B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
        return 1;
    }
    cuuint32_t box[3] = {RB, (cuuint32_t)(3 + 2 * c), 1}, es[3] = {1, 1, 1};
    CUresult r = cuTensorMapEncodeTiled(&mp.m[c], CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, A, dims, str, box, es,
                                        CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                                        CU_TENSOR_MAP_L2_PROMOTION_L2_64B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    cuuint64_t dims2[2] = {(cuuint64_t)nyp, (cuuint64_t)Q * cols};
    cuuint64_t str2[1] = {(cuuint64_t)nyp * 8};
    cuuint32_t box2[2] = {RB, (cuuint32_t)(3 + 2 * c)}, es2[2] = {1, 1};
    if (r == CUDA_SUCCESS)
      r = cuTensorMapEncodeTiled(&mp.m2[c], CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, A, dims2, str2, box2, es2,
                                 CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                                 CU_TENSOR_MAP_L2_PROMOTION_L2_64B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) {
      fprintf(stderr, "tensor map %d: %d\n", c, (int)r);
      return 1;
    }
  }
  int nsm;
  CK(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0));
  const int ns = (ly + HT - 1) / HT;  // strips (ly >= HT + 6)
  const size_t smem = (size_t)MAXBUF * BUFD * 8 + 2 * MAXBUF * 8;
  CK(cudaFuncSetAttribute(k_probe, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  cudaEvent_t e0, e1;
  CK(cudaEventCreate(&e0));
  CK(cudaEventCreate(&e1));
  const double sites = (double)lx * ly;
  auto timeit = [&](auto&& launch) {
    for (int i = 0; i < 3; ++i) launch();
    CK(cudaDeviceSynchronize());
    std::vector<float> ts;
    for (int i = 0; i < reps; ++i) {
      CK(cudaEventRecord(e0));
      launch();
      CK(cudaEventRecord(e1));
      CK(cudaEventSynchronize(e1));
      float ms;
      CK(cudaEventElapsedTime(&ms, e0, e1));
      ts.push_back(ms);
    }
    CK(cudaGetLastError());
    std::sort(ts.begin(), ts.end());
    return (double)ts[ts.size() / 2];
  };
  // requested bytes of one launch: loads Q * RB * 8 per load column, stores Q * rows * 8 per output column
  auto req = [&](int grid, int aligned, double& ld_bytes, double& st_bytes) {
    ld_bytes = st_bytes = 0;
    for (int b = 0; b < grid; ++b) {
      const int64_t U = (int64_t)ns * lx;
      int64_t u = U * b / grid, ue = U * (b + 1) / grid;
      if (aligned) {
        const int R = grid / ns, s = b % ns, r = b / ns;
        u = (int64_t)s * lx + (int64_t)lx * r / R;
        ue = (int64_t)s * lx + (int64_t)lx * (r + 1) / R;
      }
      while (u < ue) {
        const int s = (int)(u / lx), x0 = (int)(u % lx);
        const int x1 = (int)std::min<int64_t>(lx, x0 + (ue - u));
        u += x1 - x0;
        ld_bytes += (double)(x1 - x0 + 6) * Q * RB * 8;
        st_bytes += (double)(x1 - x0) * Q * std::min(HT, ly - strip_ya(s, ns, ly)) * 8;
      }
    }
  };
  if (getenv("PROBE_STORES")) {
    double ld_bytes, st_bytes;
    req(nsm, 0, ld_bytes, st_bytes);
    auto run = [&](auto kern, int nw, int grid) {
      const double ms = timeit([&] { kern<<<grid, nw * 32>>>(B, lx, ly, nyp, ns); });
      printf("{\"probe\": \"stores only\", \"warps_per_cta\": %d, \"ctas\": %d, \"ms\": %.4f, \"gbs\": %.1f}\n", nw,
             grid, ms, st_bytes / ms * 1e-6);
    };
    run(k_store_only<4>, 4, nsm);
    run(k_store_only<8>, 8, nsm);
    run(k_store_only<16>, 16, nsm);
    run(k_store_only<4>, 4, 4 * nsm);
    return 0;
  }
  const double ms_copy = timeit([&] { k_copy<<<nsm * 8, 512>>>((const double2*)A, (double2*)B, n / 2); });
  printf("{\"probe\": \"double2 copy\", \"ms\": %.4f, \"gbs\": %.1f}\n", ms_copy, 2.0 * n * 8 / ms_copy * 1e-6);
  const char* sname[4] = {"stg", "bulk", "loads only", "stores only"};
  const char* lname[5] = {"tma group boxes", "1-D bulk per population", "ldgsts 16 B", "tma + ldgsts", "tma group boxes, 2-D map"};
  const int tma_mask = getenv("PROBE_TMA_MASK") ? atoi(getenv("PROBE_TMA_MASK")) : 0x6b;
  const int only_load = getenv("PROBE_LOAD") ? atoi(getenv("PROBE_LOAD")) : -1;
  const int nb_list[3] = {1, 2, 4};
  for (int load = 0; load < 5; ++load)
    for (int aligned = 0; aligned < 2; ++aligned)
      for (int store = 0; store < 4; ++store)
        for (int nbuf : nb_list) {
          if (nbuf > MAXBUF || (only_load >= 0 && load != only_load)) continue;
          if (store == 3 && (nbuf != 2 || load)) continue;
          if (store == 1 && (nbuf == 1 || (load && load != 4))) continue;
          if (load && load != 4 && aligned) continue;
          const int grid = aligned ? nsm / ns * ns : nsm;
          double ld_bytes, st_bytes;
          req(grid, aligned, ld_bytes, st_bytes);
          const double ms = timeit([&] {
            k_probe<<<grid, NCONS + 32, smem>>>(mp, A, B, lx, ly, nyp, ns, nbuf, store, aligned, load, tma_mask);
          });
          const double bytes = (store != 3 ? ld_bytes : 0) + (store != 2 ? st_bytes : 0);
          printf("{\"probe\": \"tb pattern\", \"ht\": %d, \"load\": \"%s\", \"split\": \"%s\", \"ctas\": %d, "
                 "\"store\": \"%s\", \"nbuf\": %d, \"kb_in_flight_max\": %.1f, \"ms\": %.4f, \"requested_gbs\": %.1f, "
                 "\"load_gb\": %.3f, \"store_gb\": %.3f, \"mlups_if_kernel\": %.0f}\n",
                 HT, lname[load], aligned ? "aligned strips" : "kernel", grid, sname[store], nbuf,
                 nbuf * Q * RB * 8 / 1024.0, ms, bytes / ms * 1e-6, ld_bytes * 1e-9, st_bytes * 1e-9,
                 2 * sites / ms * 1e-3);
        }
  if (getenv("PROBE_DEEP")) {
    auto run_deep = [&](auto kern, int depth) {
      CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
      const int maxb = (int)((MAXBUF * BUFD) / goffd(NG, depth));
      for (int store = 0; store < 3; store += 2)
        for (int nbuf = 1; nbuf <= std::min(maxb, 4); ++nbuf) {
          double ld_bytes, st_bytes;
          req(nsm, 0, ld_bytes, st_bytes);
          const double ms = timeit([&] { kern<<<nsm, NCONS + 32, smem>>>(mp, B, lx, ly, nyp, ns, nbuf, store); });
          const double bytes = ld_bytes + (store == 0 ? st_bytes : 0);
          printf("{\"probe\": \"deep boxes\", \"depth\": %d, \"store\": \"%s\", \"nbuf\": %d, \"kb_in_flight_max\": %.1f, "
                 "\"ms\": %.4f, \"requested_gbs\": %.1f, \"mlups_if_kernel\": %.0f}\n",
                 depth, store == 0 ? "stg" : "loads only", nbuf, nbuf * depth * Q * RB * 8 / 1024.0, ms,
                 bytes / ms * 1e-6, 2 * sites / ms * 1e-3);
        }
    };
    run_deep(k_probe_deep<1>, 1);
    run_deep(k_probe_deep<2>, 2);
    run_deep(k_probe_deep<4>, 4);
    return 0;
  }
  return 0;
}
