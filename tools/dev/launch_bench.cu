// Fixed cost of a persistent, big-smem kernel launch on B200: back-to-back
// launches of near-empty kernels with the transform kernels' shape (608
// threads, ~220 KB dynamic smem, 148 CTAs), with and without programmatic
// dependent launch, against a small-CTA baseline.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/dev/launch_bench tools/dev/launch_bench.cu
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>

__global__ void k_empty(int* p) {
  extern __shared__ char smem[];
  asm volatile("griddepcontrol.wait;" ::: "memory");
  asm volatile("griddepcontrol.launch_dependents;");
  (void)smem;
  if (threadIdx.x == 0 && p) p[blockIdx.x] += 1;
}

// touch ~64 KB per CTA from HBM: one load round trip
__global__ void k_load(const float4* in, float4* out, int n4) {
  asm volatile("griddepcontrol.wait;" ::: "memory");
  asm volatile("griddepcontrol.launch_dependents;");
  float4 acc = make_float4(0, 0, 0, 0);
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n4; i += gridDim.x * blockDim.x) {
    float4 v = in[i];
    acc.x += v.x; acc.y += v.y; acc.z += v.z; acc.w += v.w;
  }
  if (acc.x == 12345.f) out[0] = acc;
}

template <typename F>
float time_it(F f, int reps) {
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  for (int i = 0; i < 20; ++i) f();
  cudaEventRecord(a);
  for (int i = 0; i < reps; ++i) f();
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms;
  cudaEventElapsedTime(&ms, a, b);
  return ms * 1e3f / reps;
}

template <typename... A>
void launch(void (*k)(A...), int grid, int threads, int smem, bool pdl, A... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = threads;
  cfg.dynamicSmemBytes = smem;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = pdl ? 1 : 0;
  cudaError_t e = cudaLaunchKernelEx(&cfg, k, args...);
  if (e != cudaSuccess) {
    printf("launch failed: %s\n", cudaGetErrorString(e));
    fflush(stdout);
    exit(1);
  }
}

int main() {
  int* p = nullptr;
  if (cudaMalloc(&p, 4096 * sizeof(int)) != cudaSuccess) { printf("malloc failed\n"); return 1; }
  cudaMemset(p, 0, 4096 * sizeof(int));
  cudaFuncSetAttribute(k_empty, cudaFuncAttributeMaxDynamicSharedMemorySize, 225 * 1024);
  const int n4 = 148 * 64 * 1024 / 16;
  float4 *in, *out;
  cudaMalloc(&in, n4 * 16);
  cudaMalloc(&out, 16);
  cudaMemset(in, 0, n4 * 16);
  struct C { int grid, threads, smem; };
  const C cs[] = {{148, 128, 0}, {148, 608, 0}, {148, 608, 220 * 1024}, {148, 1024, 220 * 1024}, {48, 608, 220 * 1024}};
  for (const C& c : cs)
    for (int pdl = 0; pdl < 2; ++pdl)
    {
      const float us = time_it([&] { launch(k_empty, c.grid, c.threads, c.smem, pdl == 1, p); }, 2000);
      printf("empty grid %3d threads %4d smem %6d pdl %d: %.2f us/launch\n", c.grid, c.threads, c.smem, pdl, us);
      fflush(stdout);
    }
  // alternate small-smem and big-smem kernels (carveout changes between them)
  for (int pdl = 0; pdl < 2; ++pdl)
    printf("alternating 0 / 220 KB smem, pdl %d: %.2f us/launch\n", pdl, time_it([&] {
             launch(k_empty, 148, 256, 0, pdl == 1, p);
             launch(k_empty, 148, 608, 220 * 1024, pdl == 1, p);
           }, 1000) / 2);
  for (int pdl = 0; pdl < 2; ++pdl)
    printf("load 9.7 MB (64 KB/CTA), 148 x 608, pdl %d: %.2f us/launch\n", pdl,
           time_it([&] { launch(k_load, 148, 608, 0, pdl == 1, (const float4*)in, out, n4); }, 1000));
  cudaError_t e = cudaDeviceSynchronize();
  printf("status %s\n", cudaGetErrorString(e));
  return 0;
}
