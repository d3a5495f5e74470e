// FP64 DFMA peak and HBM copy microbenchmark (SURVEY.md §8d "FP64 peak microbenchmark").
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o fp64_peak fp64_peak.cu
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>
#define CK(x) do{cudaError_t e=(x); if(e!=cudaSuccess){printf("CUDA %s @%d\n",cudaGetErrorString(e),__LINE__); return 1;}}while(0)

template<int CH>
__global__ void dfma_chains(double* out, int iters, double y) {
  double x[CH];
#pragma unroll
  for (int c = 0; c < CH; ++c) x[c] = threadIdx.x * 1e-9 + c;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int c = 0; c < CH; ++c) x[c] = fma(x[c], y, x[c]);
  }
  double s = 0;
#pragma unroll
  for (int c = 0; c < CH; ++c) s += x[c];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

__global__ void copy_v2(const double2* __restrict__ a, double2* __restrict__ b, size_t n) {
  size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x;
  size_t st = (size_t)gridDim.x * blockDim.x;
  for (; i < n; i += st) b[i] = a[i];
}

int main(int argc, char** argv) {
  const int reps = argc > 1 ? atoi(argv[1]) : 5;   // timed DFMA launches (best one reported)
  int sms; CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  int clk; CK(cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0));
  int l2; CK(cudaDeviceGetAttribute(&l2, cudaDevAttrL2CacheSize, 0));
  const int CH = 8, TPB = 256; int blocks = sms * 8; int iters = 1 << 16;
  double* out; CK(cudaMalloc(&out, sizeof(double) * blocks * TPB));
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  dfma_chains<CH><<<blocks, TPB>>>(out, 1000, 1.0000001);
  CK(cudaDeviceSynchronize());
  float best = 1e30f;
  for (int r = 0; r < reps; ++r) {
    cudaEventRecord(e0); dfma_chains<CH><<<blocks, TPB>>>(out, iters, 1.0000001); cudaEventRecord(e1);
    CK(cudaEventSynchronize(e1)); float ms; cudaEventElapsedTime(&ms, e0, e1); if (ms < best) best = ms;
  }
  double flops = 2.0 * CH * (double)iters * blocks * TPB;
  printf("{\"sms\": %d, \"clock_khz_attr\": %d, \"l2_bytes\": %d, \"fp64_tflops\": %.3f, \"fp64_ms\": %.3f",
         sms, clk, l2, flops / best / 1e9, best);
  size_t n = (size_t)1 << 27; // 2 GiB per buffer in double2 → 128M double2 = 2 GiB
  double2 *a, *b; CK(cudaMalloc(&a, n * 16)); CK(cudaMalloc(&b, n * 16));
  cudaMemset(a, 0, n * 16); cudaMemset(b, 0, n * 16);
  best = 1e30f;
  for (int r = 0; r < 10; ++r) {
    cudaEventRecord(e0); copy_v2<<<sms * 16, 512>>>(a, b, n); cudaEventRecord(e1);
    CK(cudaEventSynchronize(e1)); float ms; cudaEventElapsedTime(&ms, e0, e1); if (ms < best) best = ms;
  }
  printf(", \"copy_gbs\": %.1f}\n", 2.0 * n * 16 / best / 1e6);
  return 0;
}
