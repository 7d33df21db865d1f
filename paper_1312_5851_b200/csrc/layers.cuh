// Layer-stack elementwise stages around the convolution hot path (the
// reference's training-step driver, layers.hpp:34-109 and :393-407):
//   relu forward / backward, 2x2 stride-2 max pooling forward (with the
//   winning flat index per window) / backward, and fit_to (top-left pad or
//   crop of every plane).
// All are single-pass HBM-bound kernels: grid-stride loops over output
// elements, 16-B vector accesses where the layout allows.
#pragma once
#include <cstdint>

namespace fcb {

// layers.hpp:88-97: y = max(x, 0)
__global__ void relu_fwd_kernel(const float4* __restrict__ x, float4* __restrict__ y, long long n4) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n4;
       i += (long long)gridDim.x * blockDim.x) {
    const float4 v = x[i];
    y[i] = make_float4(v.x > 0.f ? v.x : 0.f, v.y > 0.f ? v.y : 0.f, v.z > 0.f ? v.z : 0.f,
                       v.w > 0.f ? v.w : 0.f);
  }
}

// layers.hpp:99-109: gx = x > 0 ? gy : 0
__global__ void relu_bwd_kernel(const float4* __restrict__ gy, const float4* __restrict__ x,
                                float4* __restrict__ gx, long long n4) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n4;
       i += (long long)gridDim.x * blockDim.x) {
    const float4 v = x[i], g = gy[i];
    gx[i] = make_float4(v.x > 0.f ? g.x : 0.f, v.y > 0.f ? g.y : 0.f, v.z > 0.f ? g.z : 0.f,
                        v.w > 0.f ? g.w : 0.f);
  }
}

// Scalar tails (n not a multiple of 4).
__global__ void relu_fwd_tail(const float* x, float* y, long long b, long long n) {
  const long long i = b + threadIdx.x;
  if (i < n) y[i] = x[i] > 0.f ? x[i] : 0.f;
}
__global__ void relu_bwd_tail(const float* gy, const float* x, float* gx, long long b, long long n) {
  const long long i = b + threadIdx.x;
  if (i < n) gx[i] = x[i] > 0.f ? gy[i] : 0.f;
}

// layers.hpp:34-66: 2x2 windows, stride 2; ties go to the earliest element in
// row-major order; argmax = flat index of the winner inside its input plane.
__global__ void maxpool_fwd_kernel(const float* __restrict__ x, float* __restrict__ y,
                                   uint32_t* __restrict__ arg, long long planes, int rows, int cols) {
  const int orow = rows / 2, ocol = cols / 2;
  const long long total = planes * orow * ocol;
  for (long long o = blockIdx.x * (long long)blockDim.x + threadIdx.x; o < total;
       o += (long long)gridDim.x * blockDim.x) {
    const long long pl = o / (orow * ocol);
    const int rem = (int)(o - pl * orow * ocol);
    const int i = rem / ocol, j = rem - i * ocol;
    const float* in = x + pl * rows * cols;
    int best = 2 * i * cols + 2 * j;
    float bv = in[best];
#pragma unroll
    for (int di = 0; di < 2; ++di)
#pragma unroll
      for (int dj = 0; dj < 2; ++dj) {
        const int q = (2 * i + di) * cols + 2 * j + dj;
        const float v = in[q];
        if (v > bv) {
          bv = v;
          best = q;
        }
      }
    y[o] = bv;
    arg[o] = (uint32_t)best;
  }
}

// layers.hpp:68-83: the windows tile the plane, so every input element is
// written exactly once: the window's gradient where it won, zero elsewhere.
__global__ void maxpool_bwd_kernel(const float* __restrict__ gy, const uint32_t* __restrict__ arg,
                                   float* __restrict__ gx, long long planes, int rows, int cols) {
  const int orow = rows / 2, ocol = cols / 2;
  const long long total = planes * orow * ocol;
  for (long long o = blockIdx.x * (long long)blockDim.x + threadIdx.x; o < total;
       o += (long long)gridDim.x * blockDim.x) {
    const long long pl = o / (orow * ocol);
    const int rem = (int)(o - pl * orow * ocol);
    const int i = rem / ocol, j = rem - i * ocol;
    float* out = gx + pl * rows * cols;
    const float g = gy[o];
    const int win = (int)arg[o];
#pragma unroll
    for (int di = 0; di < 2; ++di)
#pragma unroll
      for (int dj = 0; dj < 2; ++dj) {
        const int q = (2 * i + di) * cols + 2 * j + dj;
        out[q] = (q == win) ? g : 0.f;
      }
  }
}

// layers.hpp:393-407: every plane padded (zeros) or cropped at the top-left
// to size x size.
__global__ void fit_to_kernel(const float* __restrict__ x, float* __restrict__ y, long long planes,
                              int rows, int cols, int size) {
  const long long total = planes * size * size;
  for (long long o = blockIdx.x * (long long)blockDim.x + threadIdx.x; o < total;
       o += (long long)gridDim.x * blockDim.x) {
    const long long pl = o / ((long long)size * size);
    const int rem = (int)(o - pl * size * size);
    const int i = rem / size, j = rem - i * size;
    y[o] = (i < rows && j < cols) ? x[pl * rows * cols + (long long)i * cols + j] : 0.f;
  }
}

}  // namespace fcb
