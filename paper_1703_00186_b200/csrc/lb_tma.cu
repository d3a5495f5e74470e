// lb_tma.cu — TMA-staged variant of propagate (§8a2): the ±3-row neighbour
// window of every population is staged in shared memory by the Tensor Memory
// Accelerator, then written back with 16-byte vector stores.
//
// One CTA = one lattice column ix and a tile of TILE rows starting at the
// internal row r0 (even).  One elected thread issues 37 cp.async.bulk.tensor
// 3-D loads on one mbarrier: box {TILE+2 rows, 1 population, 1 column} from
// source column ix - cx_l, population l, starting at row b_l = r0 - cy_l - d_l
// with d_l = cy_l & 1.  (TMA tile boxes must start on a 16-byte boundary of the
// innermost dimension — measured on B200 with tools/tma_probe.cu: an 8-byte
// offset faults — so an odd row shift is absorbed by loading one extra row and
// reading smem at offset d_l.)  After the barrier, each thread takes 2
// consecutive rows and, for every population, reads smem[l][2p + d_l .. + 1]
// and issues one st.global.v2.f64 (16-byte aligned: r0, nyp and y0 are even).
// Rows at or beyond the last physical row are not stored (y-halo rows keep
// their zeros, G10).
#include <cuda.h>
#include <cudaTypedefs.h>

#include "lb_device.cuh"
#include "lb_internal.h"

namespace lbk {
using namespace lbd;

constexpr int TMA_TILE = 254;             // rows per CTA tile (box = TILE + 2 <= 256, the TMA limit)
constexpr int TMA_BOX = TMA_TILE + 2;     // rows per TMA box (odd-shift slack)
constexpr int TMA_ROW = 256;               // smem row pitch: 128-byte aligned boxes
constexpr int TMA_THREADS = 128;
constexpr size_t TMA_SMEM = (size_t)Q * TMA_ROW * sizeof(double) + 16;

namespace {

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}

__global__ void __launch_bounds__(TMA_THREADS) k_propagate_tma(const __grid_constant__ CUtensorMap src,
                                                               double* __restrict__ B, Geo g) {
  // dynamic smem only: [37][TMA_ROW] doubles, then the mbarrier
  extern __shared__ __align__(1024) double sm[];
  uint64_t* bar = reinterpret_cast<uint64_t*>(sm + Q * TMA_ROW);
  const uint32_t b = smem_u32(bar);
  const int ix = H + (int)blockIdx.y;
  const int r0 = g.y0 + (int)blockIdx.x * TMA_TILE;
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(b));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(b),
                 "r"((uint32_t)(Q * TMA_BOX * sizeof(double))));
#pragma unroll
    for (int l = 0; l < Q; ++l) {
      const int base = r0 - CY(l) - (CY(l) & 1);
      asm volatile(
          "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes"
          " [%0], [%1, {%2, %3, %4}], [%5];" ::"r"(smem_u32(sm + l * TMA_ROW)),
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
  const int rend = g.y0 + g.ly;  // first row NOT to store
  double* col = B + (int64_t)ix * g.cs;
  for (int p = threadIdx.x; p < TMA_TILE / 2; p += TMA_THREADS) {
    const int r = r0 + 2 * p;
    if (r >= rend) break;
#pragma unroll
    for (int l = 0; l < Q; ++l) {
      const double* s = sm + l * TMA_ROW + 2 * p + (CY(l) & 1);
      double* d = col + (int64_t)l * g.nyp + r;
      if (r + 1 < rend) {
        const double2 v = make_double2(s[0], s[1]);
        asm volatile("st.global.v2.f64 [%0], {%1, %2};" ::"l"(d), "d"(v.x), "d"(v.y) : "memory");
      } else {
        d[0] = s[0];
      }
    }
  }
}

PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  if (!fn) {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  }
  return fn;
}

bool encode(CUtensorMap* m, double* base, const Geo& g) {
  auto fn = encode_fn();
  if (!fn) return false;
  const cuuint64_t dims[3] = {(cuuint64_t)g.nyp, (cuuint64_t)Q, (cuuint64_t)g.nx};
  const cuuint64_t strides[2] = {(cuuint64_t)g.nyp * sizeof(double), (cuuint64_t)g.cs * sizeof(double)};
  const cuuint32_t box[3] = {(cuuint32_t)TMA_BOX, 1, 1};
  const cuuint32_t estr[3] = {1, 1, 1};
  return fn(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, base, dims, strides, box, estr,
            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

}  // namespace

TmaMaps* tma_create(const Geo& g, double* buf0, double* buf1) {
  if (g.y0 % 2 || g.nyp % 2) return nullptr;
  auto* t = new TmaMaps();
  if (!encode(&t->load[0], buf0, g) || !encode(&t->load[1], buf1, g)) {
    delete t;
    return nullptr;
  }
  return t;
}

void tma_destroy(TmaMaps* t) { delete t; }

cudaError_t launch_propagate_tma(const Geo& g, const TmaMaps* t, int src_buf, double* B, cudaStream_t s) {
  // opt-in shared memory is a per-device function attribute: set it once per device
  static unsigned long long done_mask = 0;
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  if (dev >= 64 || !(done_mask >> dev & 1ull)) {
    e = cudaFuncSetAttribute(k_propagate_tma, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)TMA_SMEM);
    if (e != cudaSuccess) return e;
    if (dev < 64) done_mask |= 1ull << dev;
  }
  dim3 grid((g.ly + TMA_TILE - 1) / TMA_TILE, g.lx);
  k_propagate_tma<<<grid, TMA_THREADS, TMA_SMEM, s>>>(t->load[src_buf], B, g);
  return cudaGetLastError();
}

}  // namespace lbk
