// Access-pattern microbenchmark (development tool, not product code):
// how fast can B200 HBM absorb the transform kernels' traffic patterns?
//   copy      : contiguous float4 copy (reference)
//   scatter_w : each CTA writes 544 bins x 128 B, bins `stride` bytes apart
//               (K1 r2c output pattern), reads its input contiguously
//   gather_r  : K4 c2r input pattern (128-B segments, strided), contiguous writes
//   blocked_w : same bytes, but each CTA writes one contiguous 70 KB block
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o membench membench.cu
#include <cstdio>
#include <cuda_runtime.h>

__global__ void copy_k(const float4* __restrict__ a, float4* __restrict__ b, size_t n) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x)
    b[i] = a[i];
}

// group g (=CTA work item) reads in_bytes contiguous, writes bins x 128 B.
template <bool BLOCKED>
__global__ void scatter_w(const float4* __restrict__ in, float4* __restrict__ out, int groups,
                          int bins, int rows_per_bin /* groups sharing a bin row */, int in_f4) {
  for (int g = blockIdx.x; g < groups; g += gridDim.x) {
    const float4* src = in + (size_t)g * in_f4;
    float4 acc = make_float4(0, 0, 0, 0);
    for (int i = threadIdx.x; i < in_f4; i += blockDim.x) {
      float4 v = src[i];
      acc.x += v.x; acc.y += v.y; acc.z += v.z; acc.w += v.w;
    }
    // 8 float4 per 128-B segment; thread -> (bin, part)
    for (int e = threadIdx.x; e < bins * 8; e += blockDim.x) {
      const int t = e >> 3, part = e & 7;
      size_t idx;
      if (BLOCKED) idx = ((size_t)g * bins + t) * 8 + part;
      else idx = ((size_t)t * rows_per_bin + g) * 8 + part;
      out[idx] = acc;
    }
  }
}

template <bool BLOCKED>
__global__ void gather_r(const float4* __restrict__ in, float4* __restrict__ out, int groups, int bins,
                         int rows_per_bin, int out_f4) {
  for (int g = blockIdx.x; g < groups; g += gridDim.x) {
    float4 acc = make_float4(0, 0, 0, 0);
    for (int e = threadIdx.x; e < bins * 8; e += blockDim.x) {
      const int t = e >> 3, part = e & 7;
      size_t idx;
      if (BLOCKED) idx = ((size_t)g * bins + t) * 8 + part;
      else idx = ((size_t)t * rows_per_bin + g) * 8 + part;
      float4 v = in[idx];
      acc.x += v.x; acc.y += v.y; acc.z += v.z; acc.w += v.w;
    }
    float4* dst = out + (size_t)g * out_f4;
    for (int i = threadIdx.x; i < out_f4; i += blockDim.x) dst[i] = acc;
  }
}

int main() {
  const int bins = 544, groups = 768;  // paper point x: 128 rows x 6 K-groups
  const int in_f4 = 16 * 1024 / 4;      // 16 planes x 32x32 floats = 64 KB
  const int out_f4 = 16 * 676 / 4;      // c2r output: 16 planes of 26x26
  const size_t spec_f4 = (size_t)groups * bins * 8;
  float4 *a, *b, *spec;
  cudaMalloc(&a, (size_t)groups * in_f4 * 16);
  cudaMalloc(&b, (size_t)groups * in_f4 * 16);
  cudaMalloc(&spec, spec_f4 * 16);
  cudaMemset(a, 0, (size_t)groups * in_f4 * 16);
  cudaMemset(spec, 0, spec_f4 * 16);
  float* flush;
  cudaMalloc(&flush, 512u << 20);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  auto timeit = [&](const char* name, double bytes, auto&& launch) {
    float best = 1e9;
    for (int rep = 0; rep < 6; ++rep) {
      cudaMemsetAsync(flush, rep, 512u << 20);
      cudaEventRecord(e0);
      launch();
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      if (rep > 0 && ms < best) best = ms;
    }
    printf("%-28s %8.2f us  %7.0f GB/s\n", name, best * 1e3, bytes / (best * 1e-3) / 1e9);
  };
  const int sms = 148;
  const double inB = (double)groups * in_f4 * 16, specB = (double)spec_f4 * 16;
  timeit("copy 50MB", 2 * inB, [&] { copy_k<<<sms * 8, 256>>>(a, b, (size_t)groups * in_f4); });
  for (int ctas : {1, 2, 4}) {
    char nm[64];
    snprintf(nm, 64, "scatter_w x%d/SM", ctas);
    timeit(nm, inB + specB, [&] { scatter_w<false><<<sms * ctas, 256>>>(a, spec, groups, bins, groups, in_f4); });
    snprintf(nm, 64, "blocked_w x%d/SM", ctas);
    timeit(nm, inB + specB, [&] { scatter_w<true><<<sms * ctas, 256>>>(a, spec, groups, bins, groups, in_f4); });
    snprintf(nm, 64, "gather_r x%d/SM", ctas);
    timeit(nm, specB + (double)groups * out_f4 * 16,
           [&] { gather_r<false><<<sms * ctas, 256>>>(spec, b, groups, bins, groups, out_f4); });
    snprintf(nm, 64, "blocked_r x%d/SM", ctas);
    timeit(nm, specB + (double)groups * out_f4 * 16,
           [&] { gather_r<true><<<sms * ctas, 256>>>(spec, b, groups, bins, groups, out_f4); });
  }
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
