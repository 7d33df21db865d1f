// Layer-stack elementwise stages around the convolution hot path (the
// reference's training-step driver, layers.hpp:34-109 and :393-407):
//   relu forward / backward, 2x2 stride-2 max pooling forward (with the
//   winning flat index per window) / backward, and fit_to (top-left pad or
//   crop of every plane).
// All are single-pass HBM-bound kernels: relu as grid-stride float4 loops,
// pooling and fit_to as plane-walking blocks (below).
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

// Pooling and fit_to: blocks walk whole planes (grid-stride over planes),
// the block's threads tile a plane's output rows -- thread (i0, j) with
// j = t % C, i0 = t / C handles rows i0, i0 + 256 / C, ... -- so the index
// arithmetic is one 32-bit division per thread, not a 64-bit div / mod per
// element (round 1's flat loops spent ~1.3 ms of an AlexNet-128 iteration on
// fit_to's index math; one block per (plane, row) or a warp per row were
// slower still, §4 of DESIGN.md).
struct PlaneTiler {
  int j, i0, rpi;  // column, first row, rows per pass (0: thread idle when C <= 256)
  __device__ PlaneTiler(int C) {
    const int t = threadIdx.x, nt = blockDim.x;
    if (C <= nt) {
      rpi = nt / C;
      j = t % C;
      i0 = t / C;
      if (i0 >= rpi) rpi = 0;
    } else {  // wide rows: every thread walks columns j, j + nt, ... of each row
      rpi = 1;
      j = t;
      i0 = 0;
    }
  }
};

// layers.hpp:34-66: 2x2 windows, stride 2; ties go to the earliest element in
// row-major order; argmax = flat index of the winner inside its input plane.
__global__ void maxpool_fwd_kernel(const float* __restrict__ x, float* __restrict__ y,
                                   uint32_t* __restrict__ arg, long long planes, int rows, int cols) {
  const int orow = rows / 2, ocol = cols / 2;
  const PlaneTiler tl(ocol);
  if (!tl.rpi) return;
  for (long long pl = blockIdx.x; pl < planes; pl += gridDim.x) {
    const float* in = x + pl * rows * cols;
    float* yo = y + pl * orow * ocol;
    uint32_t* ao = arg + pl * orow * ocol;
    for (int i = tl.i0; i < orow; i += tl.rpi)
      for (int j = tl.j; j < ocol; j += blockDim.x) {
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
        yo[i * ocol + j] = bv;
        ao[i * ocol + j] = (uint32_t)best;
      }
  }
}

// layers.hpp:68-83: the windows tile the plane, so every input element is
// written exactly once: the window's gradient where it won, zero elsewhere.
// ypool != nullptr: the following relu backward fused in (gradient kept
// only where the pooled value, the winner's relu output, is > 0)
__global__ void maxpool_bwd_kernel(const float* __restrict__ gy, const uint32_t* __restrict__ arg,
                                   float* __restrict__ gx, long long planes, int rows, int cols,
                                   const float* __restrict__ ypool = nullptr) {
  const int orow = rows / 2, ocol = cols / 2;
  const PlaneTiler tl(ocol);
  if (!tl.rpi) return;
  for (long long pl = blockIdx.x; pl < planes; pl += gridDim.x) {
    float* out = gx + pl * rows * cols;
    const float* g0 = gy + pl * orow * ocol;
    const float* y0 = ypool ? ypool + pl * orow * ocol : nullptr;
    const uint32_t* a0 = arg + pl * orow * ocol;
    for (int i = tl.i0; i < orow; i += tl.rpi)
      for (int j = tl.j; j < ocol; j += blockDim.x) {
        const float g = (!y0 || y0[i * ocol + j] > 0.f) ? g0[i * ocol + j] : 0.f;
        const int win = (int)a0[i * ocol + j];
#pragma unroll
        for (int di = 0; di < 2; ++di) {
          const int q = (2 * i + di) * cols + 2 * j;
          *reinterpret_cast<float2*>(out + q) = make_float2(q == win ? g : 0.f, q + 1 == win ? g : 0.f);
        }
      }
  }
}

// layers.hpp:393-407: every plane padded (zeros) or cropped at the top-left
// to size x size.
__global__ void fit_to_kernel(const float* __restrict__ x, float* __restrict__ y, long long planes,
                              int rows, int cols, int size) {
  const PlaneTiler tl(size);
  if (!tl.rpi) return;
  for (long long pl = blockIdx.x; pl < planes; pl += gridDim.x) {
    const float* in = x + pl * rows * cols;
    float* o = y + pl * size * size;
    for (int i = tl.i0; i < size; i += tl.rpi)
      for (int j = tl.j; j < size; j += blockDim.x)
        o[i * size + j] = (i < rows && j < cols) ? in[i * cols + j] : 0.f;
  }
}

}  // namespace fcb
