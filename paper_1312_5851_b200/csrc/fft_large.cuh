// K1 / K4 for FFT size m = 128 (image edges 65..128, e.g. the first layer of
// BASELINE configs[4], n = 128).  Replaces the same reference functions as
// the m <= 64 kernels (detail::r2c_plane / c2r_plane + the bin-major
// scatter / gather glue, fft.hpp:160-203, conv_fft.hpp:242-304).
//
// A 128 x 65 half spectrum (66.5 KB per plane) does not fit the one-pass
// shared-memory design of fft_tma.cuh with enough planes per CTA to write
// whole lines, so each direction runs as two passes through an
// L2-sized scratch (the host walks the planes in chunks of operand rows
// whose scratch fits ~48 MB, so the intermediate never leaves L2):
//
//   r2c  K1a  column pass  (plane, u class c, column x):
//             X[4k + c][x] = FFT32_k( w128^(c y') * sum_q x[y' + 32q][x] (-i)^(cq) )
//             (radix-4 decimation in frequency: a 32-point register FFT per
//             thread yields the rows u = c mod 4), rows u <= 64 -> scratch
//             S[plane][u][x]
//        K1b  row pass  (16 planes, one u): the 16 scratch rows staged in
//             smem, per (plane, v class h) the same decimation over x, the
//             [v][16 planes] tile written as full 128-B lines of the
//             bin-major operand F[t][r][2*kpad] (K padding as zeros),
//             optional conjugate, max-magnitude word for the fp16x3 GEMM
//   c2r  K4a  row pass  (16 planes, one u): inverse over v of the product
//             rows (group-major or bin-major, as the GEMM wrote them), only
//             the cropped columns -> scratch Z[plane][u][x']
//        K4b  column pass  (plane, column x', y class c): Hermitian
//             extension Z[128 - u] = conj(Z[u]), inverse over u by the same
//             decimation, real part * scale -> output rows y = c mod 4
//             (lanes = consecutive columns: 128-B stores), optional accumulate
#pragma once
#include "fft_planes.cuh"

namespace fcb {

constexpr int kL = 128;          // FFT size of this path
constexpr int kLRows = kL / 2 + 1;  // half-spectrum rows u in [0, 64]

// a * (-i)^E (forward) or a * (+i)^E (inverse), E in [0, 4)
template <bool INV, int E>
__device__ __forceinline__ float2 rot_i(float2 a) {
  if constexpr (E == 0) return a;
  else if constexpr (E == 2) return make_float2(-a.x, -a.y);
  else if constexpr ((E == 1) != INV) return make_float2(a.y, -a.x);  // * (-i)
  else return make_float2(-a.y, a.x);                                  // * (+i)
}

// z[n] *= w128^(+-C n), n < 32
template <bool INV, int C>
__device__ __forceinline__ void class_twiddle(float2 (&z)[32]) {
  static_for<1, 32>([&](auto N) {
    constexpr int n = decltype(N)::value;
    if constexpr ((C * n) % kL != 0) z[n] = cmul(z[n], tw128c<INV, (C * n) % kL>());
  });
}

// ---------------------------------------------------------------- r2c K1a
template <int C>
__device__ __forceinline__ void r2c128_col_class(const R2CParams& p, const float* col, float2* o, int src) {
  float2 z[32];
  static_for<0, 32>([&](auto Y) {
    constexpr int y0 = decltype(Y)::value;
    float2 acc = make_float2(0.f, 0.f);
    static_for<0, 4>([&](auto Q) {
      constexpr int q = decltype(Q)::value;
      const int y = y0 + 32 * q;
      if (y < src) acc = cadd(acc, rot_i<false, (C * q) & 3>(make_float2(__ldg(col + (long long)y * src), 0.f)));
    });
    z[y0] = acc;
  });
  class_twiddle<false, C>(z);
  fft_reg<32, false>(z);
  static_for<0, 17>([&](auto K) {
    constexpr int u = 4 * decltype(K)::value + C;
    if constexpr (u < kLRows) o[(long long)u * src] = z[decltype(K)::value];
  });
}

// grid = (rows * J, 4 classes), block = 128 (one thread per column)
__global__ void __launch_bounds__(128) r2c128_cols_kernel(const R2CParams p, int r0, float2* scr) {
  pdl_wait();
  pdl_trigger();
  const int ql = blockIdx.x;
  const int r = r0 + ql / p.J, j = ql % p.J;
  const int x = threadIdx.x, src = p.src;
  if (x >= src) return;
  const float* col = p.in + (long long)r * p.in_sr + (long long)j * p.in_sj + x;
  float2* o = scr + (long long)ql * kLRows * src + x;
  switch (blockIdx.y) {
    case 0: r2c128_col_class<0>(p, col, o, src); break;
    case 1: r2c128_col_class<1>(p, col, o, src); break;
    case 2: r2c128_col_class<2>(p, col, o, src); break;
    default: r2c128_col_class<3>(p, col, o, src); break;
  }
}

// ---------------------------------------------------------------- r2c K1b
template <int H>
__device__ __forceinline__ void r2c128_row_class(const float2* row, float2 (&z)[32], int src) {
  static_for<0, 32>([&](auto X) {
    constexpr int x0 = decltype(X)::value;
    float2 acc = make_float2(0.f, 0.f);
    static_for<0, 4>([&](auto Q) {
      constexpr int q = decltype(Q)::value;
      if (x0 + 32 * q < src) acc = cadd(acc, rot_i<false, (H * q) & 3>(row[x0 + 32 * q]));
    });
    z[x0] = acc;
  });
  class_twiddle<false, H>(z);
  fft_reg<32, false>(z);
}

constexpr int kLRowPad = kL + 1;  // odd float2 stride of the staged rows

// grid = (rows, kpad / 16, 65), block = 64 = (plane jl, v class h)
__global__ void __launch_bounds__(64) r2c128_rows_kernel(const R2CParams p, int r0, const float2* scr) {
  __shared__ float2 rows_s[16 * kLRowPad];
  __shared__ __align__(16) float2 tile[kL * 16];  // [v][plane]
  pdl_wait();
  pdl_trigger();
  const int rl = blockIdx.x, r = r0 + rl;
  const int j0 = blockIdx.y * 16, u = blockIdx.z;
  const int jv = max(0, min(16, p.J - j0));
  const int src = p.src;
  for (int i = threadIdx.x; i < 16 * src; i += 64) {
    const int jl = i / src, x = i - jl * src;
    rows_s[jl * kLRowPad + x] =
        jl < jv ? scr[((long long)(rl * p.J + j0 + jl) * kLRows + u) * src + x] : make_float2(0.f, 0.f);
  }
  __syncthreads();
  const int jl = threadIdx.x & 15, h = threadIdx.x >> 4;
  float2 z[32];
  const float2* row = rows_s + jl * kLRowPad;
  switch (h) {
    case 0: r2c128_row_class<0>(row, z, src); break;
    case 1: r2c128_row_class<1>(row, z, src); break;
    case 2: r2c128_row_class<2>(row, z, src); break;
    default: r2c128_row_class<3>(row, z, src); break;
  }
  const float csign = p.conj ? -1.f : 1.f;
  uint32_t amx = 0;
#pragma unroll
  for (int k = 0; k < 32; ++k) {
    const float2 v = jl < jv ? make_float2(z[k].x, csign * z[k].y) : make_float2(0.f, 0.f);
    tile[(4 * k + h) * 16 + jl] = v;
    amx = max(amx, max(__float_as_uint(v.x) & 0x7fffffffu, __float_as_uint(v.y) & 0x7fffffffu));
  }
  __syncthreads();
  // 128 bins x 16 planes: one 128-B line per bin
  const long long bstride = (long long)p.R * p.kpad;  // float2 per bin
  float2* out = reinterpret_cast<float2*>(p.out) + (long long)u * kL * bstride + (long long)r * p.kpad + j0;
  for (int i = threadIdx.x; i < kL * 8; i += 64) {
    const int v = i >> 3, part = i & 7;
    *reinterpret_cast<float4*>(out + v * bstride + 2 * part) = *reinterpret_cast<const float4*>(tile + v * 16 + 2 * part);
  }
  if (p.amax) {
    amx = __reduce_max_sync(0xffffffffu, amx);
    if ((threadIdx.x & 31) == 0) atomicMax(p.amax, ((unsigned long long)p.epoch << 32) | amx);
  }
}

// ---------------------------------------------------------------- c2r K4a
template <int H>
__device__ __forceinline__ void c2r128_row_class(const float2* tile, int jl, float2 (&z)[32]) {
  static_for<0, 32>([&](auto V) {
    constexpr int v0 = decltype(V)::value;
    float2 acc = make_float2(0.f, 0.f);
    static_for<0, 4>([&](auto Q) {
      constexpr int q = decltype(Q)::value;
      acc = cadd(acc, rot_i<true, (H * q) & 3>(tile[(v0 + 32 * q) * 17 + jl]));
    });
    z[v0] = acc;
  });
  class_twiddle<true, H>(z);
  fft_reg<32, true>(z);
}

// grid = (rows, ceil(J / 16), 65), block = 64 = (plane jl, x' class h)
__global__ void __launch_bounds__(64) c2r128_rows_kernel(const C2RParams p, int r0, float2* scr) {
  __shared__ float2 tile[kL * 17];  // [v][plane], odd stride
  __shared__ float2 outb[16 * kLRowPad];
  pdl_wait();
  pdl_trigger();
  const int rl = blockIdx.x, r = r0 + rl;
  const int jg = blockIdx.y, j0 = jg * 16, u = blockIdx.z;
  const int jv = min(16, p.J - j0);
  const int crop = p.crop;
  const float2* in = reinterpret_cast<const float2*>(p.in);
  if (p.gm) {  // P[r][J/16][t][16]: the 128 bins x 16 planes of row u are contiguous
    const int ngj = (p.J + 15) >> 4;
    const float2* b = in + (((long long)r * ngj + jg) * (kL * kLRows) + (long long)u * kL) * 16;
    for (int i = threadIdx.x; i < kL * 16; i += 64) tile[(i >> 4) * 17 + (i & 15)] = __ldg(b + i);
  } else {  // P[t][r][ld]
    const long long bstride = (long long)p.R * p.ld;
    for (int i = threadIdx.x; i < kL * 16; i += 64) {
      const int v = i >> 4, jl = i & 15;
      tile[v * 17 + jl] = jl < jv ? __ldg(in + ((long long)u * kL + v) * bstride + (long long)r * p.ld + j0 + jl)
                                  : make_float2(0.f, 0.f);
    }
  }
  __syncthreads();
  const int jl = threadIdx.x & 15, h = threadIdx.x >> 4;
  float2 z[32];
  switch (h) {
    case 0: c2r128_row_class<0>(tile, jl, z); break;
    case 1: c2r128_row_class<1>(tile, jl, z); break;
    case 2: c2r128_row_class<2>(tile, jl, z); break;
    default: c2r128_row_class<3>(tile, jl, z); break;
  }
#pragma unroll
  for (int k = 0; k < 32; ++k)
    if (4 * k + h < crop) outb[jl * kLRowPad + 4 * k + h] = z[k];
  __syncthreads();
  for (int i = threadIdx.x; i < jv * crop; i += 64) {
    const int l = i / crop, x = i - l * crop;
    scr[((long long)(rl * p.J + j0 + l) * kLRows + u) * crop + x] = outb[l * kLRowPad + x];
  }
}

// ---------------------------------------------------------------- c2r K4b
template <int C>
__device__ __forceinline__ void c2r128_col_class(const C2RParams& p, const float2* col, float* o, int crop) {
  float2 z[32];
  static_for<0, 32>([&](auto U) {
    constexpr int u0 = decltype(U)::value;
    float2 acc = make_float2(0.f, 0.f);
    static_for<0, 4>([&](auto Q) {
      constexpr int q = decltype(Q)::value;
      constexpr int u = u0 + 32 * q;
      const float2 v = u < kLRows ? __ldg(col + (long long)u * crop) : cconj(__ldg(col + (long long)(kL - u) * crop));
      acc = cadd(acc, rot_i<true, (C * q) & 3>(v));
    });
    z[u0] = acc;
  });
  class_twiddle<true, C>(z);
  fft_reg<32, true>(z);
  const float scale = p.scale;
#pragma unroll
  for (int k = 0; k < 32; ++k) {
    const int y = 4 * k + C;
    if (y < crop) {
      float* d = o + (long long)y * crop;
      *d = p.accum ? *d + scale * z[k].x : scale * z[k].x;
    }
  }
}

// grid = (rows * J, ceil(crop / 32)), block = 128 = (column lane, y class)
__global__ void __launch_bounds__(128) c2r128_cols_kernel(const C2RParams p, int r0, const float2* scr) {
  pdl_wait();
  pdl_trigger();
  const int ql = blockIdx.x;
  const int r = r0 + ql / p.J, j = ql % p.J;
  const int crop = p.crop;
  const int x = blockIdx.y * 32 + (threadIdx.x & 31);
  if (x >= crop) return;
  const float2* col = scr + (long long)ql * kLRows * crop + x;
  float* o = p.out + (long long)r * p.out_sr + (long long)j * p.out_sj + x;
  switch (threadIdx.x >> 5) {
    case 0: c2r128_col_class<0>(p, col, o, crop); break;
    case 1: c2r128_col_class<1>(p, col, o, crop); break;
    case 2: c2r128_col_class<2>(p, col, o, crop); break;
    default: c2r128_col_class<3>(p, col, o, crop); break;
  }
}

}  // namespace fcb
