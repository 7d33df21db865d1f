// Kernel-to-kernel hand-off cost on B200: a chain of persistent 148-CTA
// kernels (big smem, PDL-launched), each CTA doing ~2 us of work, handing
// off either by griddepcontrol.wait (grid completion + flush) or by a
// device counter the next kernel's CTAs spin on (release/acquire).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/dev/handoff_bench tools/dev/handoff_bench.cu
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>

__device__ __forceinline__ unsigned long long gns() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

template <bool COUNTER>
__global__ void k_step(const float* in, float* out, int n, unsigned* ctr, unsigned target_prev, int work_ns) {
  if (COUNTER) {
    if (threadIdx.x == 0) {
      unsigned v;
      do {
        asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(ctr) : "memory");
      } while (v < target_prev);
    }
    __syncthreads();
  } else {
    asm volatile("griddepcontrol.wait;" ::: "memory");
  }
  asm volatile("griddepcontrol.launch_dependents;");
  // read the previous step's output, write ours (a real data dependence)
  float acc = 0.f;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) acc += in[i];
  const unsigned long long t0 = gns();
  while (gns() - t0 < (unsigned long long)work_ns) {
  }
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) out[i] = acc * 0.5f + i;
  if (COUNTER) {
    __syncthreads();
    if (threadIdx.x == 0) {
      __threadfence();
      atomicAdd(ctr, 1u);
    }
  }
}

template <bool COUNTER>
float run(float* a, float* b, int n, unsigned* ctr, int steps, int work_ns) {
  cudaMemset(ctr, 0, 4);
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = 148;
  cfg.blockDim = 512;
  cfg.dynamicSmemBytes = 200 * 1024;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaDeviceSynchronize();
  cudaEventRecord(e0);
  for (int s = 0; s < steps; ++s) {
    float* src = (s & 1) ? b : a;
    float* dst = (s & 1) ? a : b;
    cudaLaunchKernelEx(&cfg, k_step<COUNTER>, (const float*)src, dst, n, ctr, (unsigned)(148 * s), work_ns);
  }
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  return ms * 1e3f / steps;
}

int main() {
  const int n = 148 * 512 * 4;
  float *a, *b;
  unsigned* ctr;
  cudaMalloc(&a, n * 4);
  cudaMalloc(&b, n * 4);
  cudaMalloc(&ctr, 4);
  cudaMemset(a, 0, n * 4);
  cudaFuncSetAttribute(k_step<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  cudaFuncSetAttribute(k_step<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  for (int w : {0, 2000, 10000}) {
    run<false>(a, b, n, ctr, 50, w);
    run<true>(a, b, n, ctr, 50, w);
    const float g = run<false>(a, b, n, ctr, 400, w), c = run<true>(a, b, n, ctr, 400, w);
    printf("work %5d ns: griddepcontrol.wait %.2f us/step, counter %.2f us/step\n", w, g, c);
  }
  printf("status %s\n", cudaGetErrorString(cudaDeviceSynchronize()));
  return 0;
}
