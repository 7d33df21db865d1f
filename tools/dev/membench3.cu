// Development microbenchmark: write 93.6 MB in the r2c output pattern
// (544 bins x 128-B line per 16-plane group, lines `groups*128` bytes apart)
// with (a) STG from all warps, (b) TMA tensor stores from a smem tile,
// (c) TMA 1-D bulk stores of a contiguous 69.6 KB block (blocked layout).
#include <cstdio>
#include <cuda.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>

__device__ __forceinline__ unsigned smem_u32(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }

__global__ void __launch_bounds__(512, 1) stg_k(float2* out, int bins, int groups) {
  // thread: plane jl = t % 16, row u = t / 16 (32 rows) -> 17 v each (544 = 32 x 17)
  for (int g = blockIdx.x; g < groups; g += gridDim.x) {
    const int jl = threadIdx.x & 15, u = threadIdx.x >> 4;
    float2* o = out + ((long long)(u * 17) * groups + g) * 16 + jl;
#pragma unroll
    for (int v = 0; v < 17; ++v) o[(long long)v * groups * 16] = make_float2(1.f, 2.f);
  }
}

__global__ void __launch_bounds__(512, 1) tma_k(const __grid_constant__ CUtensorMap tm, int bins, int groups) {
  extern __shared__ __align__(128) unsigned char sm[];
  float2* st = reinterpret_cast<float2*>(sm);  // 2 buffers of bins x 16 float2
  int it = 0;
  for (int g = blockIdx.x; g < groups; g += gridDim.x, ++it) {
    float2* b = st + (it & 1) * bins * 16;
    if (threadIdx.x == 0) asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
    __syncthreads();
    for (int i = threadIdx.x; i < bins * 16; i += blockDim.x) b[i] = make_float2(1.f, 2.f);
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    __syncthreads();
    if (threadIdx.x == 0) {
      for (int k = 0; k < 4; ++k)
        asm volatile("cp.async.bulk.tensor.3d.global.shared::cta.bulk_group [%0, {%1, %2, %3}], [%4];" ::"l"(&tm),
                     "r"(0), "r"(g), "r"(k * (bins / 4)), "r"(smem_u32(b + k * (bins / 4) * 16))
                     : "memory");
      asm volatile("cp.async.bulk.commit_group;" ::: "memory");
    }
  }
  if (threadIdx.x == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

__global__ void __launch_bounds__(512, 1) bulk_k(float2* out, int bins, int groups) {
  extern __shared__ __align__(128) unsigned char sm[];
  float2* st = reinterpret_cast<float2*>(sm);
  int it = 0;
  for (int g = blockIdx.x; g < groups; g += gridDim.x, ++it) {
    float2* b = st + (it & 1) * bins * 16;
    if (threadIdx.x == 0) asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
    __syncthreads();
    for (int i = threadIdx.x; i < bins * 16; i += blockDim.x) b[i] = make_float2(1.f, 2.f);
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    __syncthreads();
    if (threadIdx.x == 0) {
      asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(out + (long long)g * bins * 16),
                   "r"(smem_u32(b)), "r"(bins * 16 * 8)
                   : "memory");
      asm volatile("cp.async.bulk.commit_group;" ::: "memory");
    }
  }
  if (threadIdx.x == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

int main() {
  const int bins = 544, groups = 1344;
  const size_t n = (size_t)bins * groups * 16;
  float2* out;
  cudaMalloc(&out, n * 8);
  float* flush;
  cudaMalloc(&flush, 512u << 20);
  void* fn = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
  auto enc = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
  CUtensorMap tm;
  cuuint64_t dims[3] = {32, (cuuint64_t)groups, (cuuint64_t)bins};
  cuuint64_t strides[2] = {128, (cuuint64_t)groups * 128};
  cuuint32_t box[3] = {32, 1, (cuuint32_t)(bins / 4)}, es[3] = {1, 1, 1};
  CUresult r = enc(&tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, out, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                   CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r) printf("encode %d\n", (int)r);
  const int smem = 2 * bins * 16 * 8;
  cudaFuncSetAttribute(tma_k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaFuncSetAttribute(bulk_k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  auto timeit = [&](const char* name, auto&& f) {
    float best = 1e9;
    for (int rr = 0; rr < 6; ++rr) {
      cudaMemsetAsync(flush, rr, 512u << 20);
      cudaEventRecord(e0);
      f();
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      if (rr && ms < best) best = ms;
    }
    printf("%-28s %8.2f us %7.0f GB/s\n", name, best * 1e3, n * 8 / (best * 1e-3) / 1e9);
  };
  timeit("STG 512thr x1/SM", [&] { stg_k<<<148, 512>>>(out, bins, groups); });
  timeit("STG 512thr x2/SM", [&] { stg_k<<<296, 512>>>(out, bins, groups); });
  timeit("TMA tensor store", [&] { tma_k<<<148, 512, smem>>>(tm, bins, groups); });
  timeit("TMA bulk store (blocked)", [&] { bulk_k<<<148, 512, smem>>>(out, bins, groups); });
  printf("%s\n", cudaGetErrorString(cudaDeviceSynchronize()));
}
