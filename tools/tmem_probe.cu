// tmem_probe.cu — does tcgen05.cp (shared -> tensor memory) with a row-shifted
// no-swizzle descriptor deliver shared-memory row k + s to TMEM lane k, and can
// the four lane quarters read it back with tcgen05.ld?  (tools only; the
// mechanism a TMEM-resident state-(n+1) ring of the two-step kernel needs)
//
// nvcc -gencode arch=compute_100a,code=sm_100a -O2 -o tools/tmem_probe tools/tmem_probe.cu && tools/tmem_probe
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

constexpr int NP = 22;    // column pairs (16 B per row each)
constexpr int NR = 134;   // staging rows per pair (reads run up to row 6 + 127)
constexpr int NCOL = 512; // TMEM columns allocated

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

// SM100 shared-memory matrix descriptor, K-major, no swizzle: rows of 16 B,
// 8-row core matrices SBO bytes apart (cute/arch/mma_sm100_desc.hpp layout)
__device__ __forceinline__ uint64_t desc_noswizzle(uint32_t saddr, uint32_t sbo_bytes) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFF);
  d |= (uint64_t)((16u >> 4) & 0x3FFF) << 16;         // leading byte offset (unused: one 16-B column)
  d |= (uint64_t)((sbo_bytes >> 4) & 0x3FFF) << 32;   // stride byte offset
  d |= (uint64_t)1 << 46;                              // version 1 (Blackwell)
  return d;                                            // base offset 0, lbo mode 0, layout SWIZZLE_NONE
}

__global__ void __launch_bounds__(256, 1) k_probe(double* out, int* shift_out) {
  __shared__ __align__(128) double stg[NP * NR * 2];
  __shared__ uint32_t tbase;
  __shared__ __align__(8) uint64_t bar;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&tbase)),
                 "r"(NCOL));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (tid == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  for (int i = tid; i < NP * NR; i += 256) {
    const int j = i / NR, r = i % NR;
    stg[2 * i] = j * 1000.0 + r;
    stg[2 * i + 1] = -(j * 1000.0 + r) - 0.5;
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // generic writes -> tcgen05.cp (async proxy)
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tb = tbase;
  if (tid == 0) {
    for (int j = 0; j < NP; ++j) {
      const int s = j % 7;  // row shift 0..6
      const uint64_t d = desc_noswizzle(smem_u32(stg + (size_t)j * NR * 2 + 2 * s), 128);
      asm volatile("tcgen05.cp.cta_group::1.128x128b [%0], %1;" ::"r"(tb + 4 * j), "l"(d));
    }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
        smem_u32(&bar)));
  }
  if (warp >= 4) {
    asm volatile(
        "{\n .reg .pred p;\n W: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n @!p bra W;\n}\n" ::"r"(
            smem_u32(&bar))
        : "memory");
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const int q = warp & 3;
    for (int j = 0; j < NP; ++j)
      for (int h = 0; h < 2; ++h) {
        uint32_t a, b;
        asm volatile("tcgen05.ld.sync.aligned.32x32b.x2.b32 {%0, %1}, [%2];"
                     : "=r"(a), "=r"(b)
                     : "r"(tb + ((uint32_t)(32 * q) << 16) + 4 * j + 2 * h));
        asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
        out[((size_t)j * 128 + 32 * q + lane) * 2 + h] = __hiloint2double((int)b, (int)a);
      }
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tb), "r"(NCOL));
  if (tid == 0) *shift_out = 1;
}

int main() {
  double* d_out;
  int* d_flag;
  cudaMalloc(&d_out, sizeof(double) * NP * 128 * 2);
  cudaMalloc(&d_flag, sizeof(int));
  cudaMemset(d_out, 0, sizeof(double) * NP * 128 * 2);
  k_probe<<<1, 256>>>(d_out, d_flag);
  cudaError_t e = cudaDeviceSynchronize();
  if (e != cudaSuccess) {
    printf("{\"ok\": false, \"error\": \"%s\"}\n", cudaGetErrorString(e));
    return 1;
  }
  static double h[NP * 128 * 2];
  cudaMemcpy(h, d_out, sizeof(h), cudaMemcpyDeviceToHost);
  int bad = 0, first_j = -1, first_k = -1;
  double got = 0, want = 0;
  for (int j = 0; j < NP; ++j)
    for (int k = 0; k < 128; ++k)
      for (int hh = 0; hh < 2; ++hh) {
        const int s = j % 7;
        const double w = hh == 0 ? j * 1000.0 + (k + s) : -(j * 1000.0 + (k + s)) - 0.5;
        const double g = h[((size_t)j * 128 + k) * 2 + hh];
        if (g != w) {
          if (!bad) first_j = j, first_k = k, got = g, want = w;
          ++bad;
        }
      }
  printf("{\"ok\": %s, \"mismatches\": %d, \"first\": [%d, %d, %.1f, %.1f]}\n", bad ? "false" : "true", bad, first_j,
         first_k, got, want);
  return bad != 0;
}
