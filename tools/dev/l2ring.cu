// Does B200's L2 keep a repeatedly rewritten buffer out of HBM?  (The
// premise of a bin-blocked, L2-resident producer / consumer ring, DESIGN.md
// section 7 item 5.)  Each pass: a writer kernel overwrites a ring of R MB,
// a reader kernel reads it back.  Run under
//   ncu --metrics dram__bytes_write.sum,dram__bytes_read.sum,gpu__time_duration.sum ./l2ring R
// and compare per-kernel DRAM bytes with R.  A third argument repeats the
// ring inside each launch (steady-state L2 bandwidth without launch gaps).  Build:
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/dev/l2ring tools/dev/l2ring.cu
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>

__global__ void writer(float4* ring, long long n4, float v, int reps) {
  for (int r = 0; r < reps; ++r, v += 1.f)
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n4; i += (long long)gridDim.x * blockDim.x)
    ring[i] = make_float4(v, v + 1.f, v + 2.f, v + 3.f);
}
__global__ void reader(const float4* ring, long long n4, float* out, int reps) {
  float acc = 0.f;
  for (int r = 0; r < reps; ++r)
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n4; i += (long long)gridDim.x * blockDim.x) {
    const float4 v = ring[i];
    acc += v.x + v.y + v.z + v.w;
  }
  if (acc == 12345.f) out[0] = acc;
}

int main(int argc, char** argv) {
  const long long mb = argc > 1 ? atoll(argv[1]) : 32;
  const int passes = argc > 2 ? atoi(argv[2]) : 8;
  const int reps = argc > 3 ? atoi(argv[3]) : 1;  // ring rewrites / re-reads inside one launch
  const long long n4 = mb * (1 << 20) / 16;
  float4* ring;
  float* out;
  cudaMalloc(&ring, n4 * 16);
  cudaMalloc(&out, 4);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  for (int p = 0; p < passes; ++p) {
    cudaEventRecord(e0);
    writer<<<148 * 8, 256>>>(ring, n4, (float)p, reps);
    reader<<<148 * 8, 256>>>(ring, n4, out, reps);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    printf("ring %lld MB pass %d: write+read %.1f us (%.2f TB/s of ring traffic)\n", mb, p, ms * 1e3,
           2.0 * reps * mb * (1 << 20) / (ms * 1e-3) / 1e12);
  }
  cudaDeviceSynchronize();
  return 0;
}
