// pure write bandwidth: contiguous vs 128-B segments at a large stride
#include <cstdio>
#include <cuda_runtime.h>
__global__ void wcontig(float2* out, size_t n) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x)
    out[i] = make_float2(1.f, 2.f);
}
// line l = (t, g): t in [0,bins), g in [0,groups): address (t*groups + g)*16 float2; each warp writes 2 lines
__global__ void wscatter(float2* out, int bins, int groups) {
  const int lane = threadIdx.x & 15;
  long long nlines = (long long)bins * groups;
  for (long long L = (blockIdx.x * (long long)blockDim.x + threadIdx.x) / 16; L < nlines; L += (long long)gridDim.x * blockDim.x / 16) {
    // consecutive L -> same group g, consecutive t (the r2c per-thread order)
    const long long g = L / bins, t = L % bins;
    out[(t * groups + g) * 16 + lane] = make_float2(1.f, 2.f);
  }
}
int main() {
  const int bins = 544, groups = 1344;
  size_t n = (size_t)bins * groups * 16;
  float2* out; cudaMalloc(&out, n * 8);
  float* flush; cudaMalloc(&flush, 512u << 20);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  auto timeit = [&](const char* name, auto&& f) {
    float best = 1e9;
    for (int r = 0; r < 6; ++r) { cudaMemsetAsync(flush, r, 512u << 20); cudaEventRecord(e0); f(); cudaEventRecord(e1); cudaEventSynchronize(e1);
      float ms; cudaEventElapsedTime(&ms, e0, e1); if (r && ms < best) best = ms; }
    printf("%-24s %8.2f us %7.0f GB/s\n", name, best * 1e3, n * 8 / (best * 1e-3) / 1e9);
  };
  for (int per : {4, 8, 16}) {
    char nm[64];
    snprintf(nm, 64, "contig %d blk/SM", per); timeit(nm, [&] { wcontig<<<148 * per, 256>>>(out, n); });
    snprintf(nm, 64, "scatter %d blk/SM", per); timeit(nm, [&] { wscatter<<<148 * per, 256>>>(out, bins, groups); });
  }
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
}
