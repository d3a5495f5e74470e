// Probe of a single TMA tensor load on sm_100a (development tool).
// nvcc -gencode arch=compute_100a,code=sm_100a -O2 -o tma_probe tma_probe.cu -lcuda
// ./tma_probe <dtype 0=f64 1=u64 2=f32> <box elems> [global]
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdint>
#include <cstdio>
#include <cstdlib>

__device__ __forceinline__ uint32_t s32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__global__ void probe(const __grid_constant__ CUtensorMap pm, const CUtensorMap* gm, int use_global,
                      unsigned bytes, int c0, unsigned char* out) {
  extern __shared__ __align__(1024) unsigned char sm[];
  uint64_t* bar = reinterpret_cast<uint64_t*>(sm + 4096);
  const uint32_t b = s32(bar);
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(b));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    const void* desc = use_global ? (const void*)gm : (const void*)&pm;
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(b), "r"(bytes));
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(
            s32(sm)),
        "l"(desc), "r"(c0), "r"(1), "r"(b)
        : "memory");
    // bounded wait (a probe must never hang the box)
    uint32_t done = 0;
    for (int it = 0; it < (1 << 22) && !done; ++it)
      asm volatile(
          "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0;\n selp.u32 %0, 1, 0, p;\n}\n"
          : "=r"(done)
          : "r"(b)
          : "memory");
    for (unsigned i = 0; i < bytes; ++i) out[i] = done ? sm[i] : 0;
  }
}

int main(int argc, char** argv) {
  const int dt = argc > 1 ? atoi(argv[1]) : 0;
  const unsigned box0 = argc > 2 ? atoi(argv[2]) : 256;
  const int use_global = argc > 3 && atoi(argv[3]) == 1;
  const int c0 = argc > 4 ? atoi(argv[4]) : 5;
  const int cluster = argc > 5 && atoi(argv[5]) == 1;
  const unsigned es = dt == 2 ? 4 : 8;
  const int rowbytes = 8192, rows = 32;
  unsigned char* buf;
  cudaMalloc(&buf, rowbytes * rows);
  unsigned char* h = new unsigned char[rowbytes * rows];
  for (int i = 0; i < rowbytes * rows; ++i) h[i] = (unsigned char)(i * 7 + 3);
  cudaMemcpy(buf, h, rowbytes * rows, cudaMemcpyHostToDevice);
  unsigned char* out;
  cudaMalloc(&out, 4096);
  CUtensorMap m;
  cuuint64_t dims[2] = {(cuuint64_t)(rowbytes / es), (cuuint64_t)rows};
  cuuint64_t strides[1] = {(cuuint64_t)rowbytes};
  cuuint32_t box[2] = {box0, 1}, estr[2] = {1, 1};
  CUtensorMapDataType t = dt == 0 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT64
                        : dt == 1 ? CU_TENSOR_MAP_DATA_TYPE_UINT64 : CU_TENSOR_MAP_DATA_TYPE_FLOAT32;
  CUresult r = cuTensorMapEncodeTiled(&m, t, 2, buf, dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                                      CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_NONE,
                                      CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  CUtensorMap* gm;
  cudaMalloc(&gm, sizeof(m));
  cudaMemcpy(gm, &m, sizeof(m), cudaMemcpyHostToDevice);
  cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, 4096 + 64);
  const unsigned bytes = box0 * es;
  if (cluster) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(1);
    cfg.blockDim = dim3(32);
    cfg.dynamicSmemBytes = 4096 + 64;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = 1;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    cudaLaunchKernelEx(&cfg, probe, m, (const CUtensorMap*)gm, use_global, bytes, c0, out);
  } else {
    probe<<<1, 32, 4096 + 64>>>(m, gm, use_global, bytes, c0, out);
  }
  cudaError_t e = cudaDeviceSynchronize();
  unsigned char o[4096] = {0};
  cudaMemcpy(o, out, bytes, cudaMemcpyDeviceToHost);
  int ok = e == cudaSuccess;
  for (unsigned i = 0; ok && i < bytes; ++i) ok = o[i] == h[rowbytes + c0 * es + i];
  printf("dtype %d box %u c0 %d cluster %d %s: encode %d, %s, data %s\n", dt, box0, c0, cluster,
         use_global ? "global" : "param", (int)r,
         cudaGetErrorString(e), ok ? "OK" : "WRONG");
  return !ok;
}
