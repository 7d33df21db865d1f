// K1 / K4 for FFT size m = 128 (image edges 65..128, e.g. the first layer of
// BASELINE configs[4], n = 128).  Replaces the same reference functions as
// the m <= 64 kernels (detail::r2c_plane / c2r_plane + the bin-major
// scatter / gather glue, fft.hpp:160-203, conv_fft.hpp:242-304).
//
// A 128 x 65 half spectrum (66.5 KB per plane) does not fit the one-pass
// shared-memory design of fft_tma.cuh with enough planes per CTA to write
// whole lines, so each direction runs as two passes through an HBM scratch
// sized for the whole operator (the host walks operand rows in chunks only
// above a 1 GB cap):
//
//   r2c  K1a  column pass  (plane, column pair p = (2p, 2p + 1), u class c):
//             Z[4k + c][p] = FFT32_k( w128^(c y') * sum_q z[y' + 32q] (-i)^(cq) ),
//             z[y] = x[y][2p] + i x[y][2p + 1] (two real columns per complex
//             FFT; radix-4 decimation in frequency: a 32-point register FFT
//             per thread yields the rows u = c mod 4), all 128 rows u of the
//             packed Z -> scratch S[plane][u][p]; planes streamed by bulk
//             copies through a 2-stage smem ring (persistent CTAs)
//        K1b  row pass  (16 planes, one u): the pairs separated on load,
//             A[u] = (Z[u] + conj Z[-u]) / 2, B[u] = (Z[u] - conj Z[-u]) / 2i,
//             staged in smem, per (plane, v class h) the same decimation
//             over x, the [v][16 planes] tile written as full 128-B lines of
//             the bin-major operand F[t][r][2*kpad] (K padding as zeros),
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

// Runtime-class forms of rot_i / class_twiddle (FCB_LARGE_RT, default on):
// the four decimation classes then share one instruction stream instead of
// four unrolled copies -- each class's 32-point FFT is ~1.4k instructions,
// and four of them in one kernel made instruction fetch ("no_instructions")
// the top ncu stall of K1a / K4b.  Twiddles from a constant-memory table
// (the class is warp-uniform: broadcast reads); same values as tw128c, so
// the results are bit-identical.
#ifndef FCB_LARGE_RT
#define FCB_LARGE_RT 1
#endif
struct Tw128Tab {
  float re[128], im[128];
};
__host__ __device__ constexpr Tw128Tab make_tw128_tab() {
  Tw128Tab t{};
  for (int k = 0; k < 128; ++k) {
    t.re[k] = tw128_re(k);
    t.im[k] = tw128_im(k);
  }
  return t;
}
__constant__ Tw128Tab c_tw128 = make_tw128_tab();

template <bool INV>
__device__ __forceinline__ float2 rot_i_rt(float2 a, int e) {  // a * (-+i)^e
  float2 r = a;
  if (e & 1) r = INV ? make_float2(-a.y, a.x) : make_float2(a.y, -a.x);
  if (e & 2) r = make_float2(-r.x, -r.y);
  return r;
}
template <bool INV>
__device__ __forceinline__ void class_twiddle_rt(float2 (&z)[32], int c) {
  if (c == 0) return;
  static_for<1, 32>([&](auto N) {
    constexpr int n = decltype(N)::value;
    const int k = (c * n) & (kL - 1);
    const float im = c_tw128.im[k];
    z[n] = cmul(z[n], make_float2(c_tw128.re[k], INV ? -im : im));
  });
}

// ---------------------------------------------------------------- r2c K1a
// Two real columns per complex FFT: the column pair (2p, 2p + 1) is
// transformed as a + i b; K1b separates A[u] = (Z[u] + conj(Z[-u])) / 2 and
// B[u] = (Z[u] - conj(Z[-u])) / 2i when it reads the scratch, so K1a keeps
// all 128 rows u of the packed Z (half the column-pass work of a transform
// per column).
template <int C>
__device__ __forceinline__ void r2c128_colpair_class(const float2* col, int cs, float2* o, int src, long long np) {
  // q-outer accumulation keeps one input live at a time (z + 1 load)
  float2 z[32];
  static_for<0, 32>([&](auto Y) {
    constexpr int y0 = decltype(Y)::value;
    z[y0] = y0 < src ? col[y0 * cs] : make_float2(0.f, 0.f);
  });
  static_for<1, 4>([&](auto Q) {
    constexpr int q = decltype(Q)::value;
    if (32 * q < src)
      static_for<0, 32>([&](auto Y) {
        constexpr int y0 = decltype(Y)::value;
        const int y = y0 + 32 * q;
        if (y < src) z[y0] = cadd(z[y0], rot_i<false, (C * q) & 3>(col[(y0 + 32 * q) * cs]));
      });
  });
  class_twiddle<false, C>(z);
  fft_reg<32, false>(z);
  static_for<0, 32>([&](auto K) {
    constexpr int u = 4 * decltype(K)::value + C;
    o[(long long)u * np] = z[decltype(K)::value];
  });
}

__device__ __forceinline__ void r2c128_colpair_rt(const float2* col, int cs, float2* o, int src, long long np,
                                                  int c) {
  float2 z[32];
  static_for<0, 32>([&](auto Y) {
    constexpr int y0 = decltype(Y)::value;
    z[y0] = y0 < src ? col[y0 * cs] : make_float2(0.f, 0.f);
  });
  static_for<1, 4>([&](auto Q) {
    constexpr int q = decltype(Q)::value;
    if (32 * q < src)
      static_for<0, 32>([&](auto Y) {
        constexpr int y0 = decltype(Y)::value;
        if (y0 + 32 * q < src) z[y0] = cadd(z[y0], rot_i_rt<false>(col[(y0 + 32 * q) * cs], c * q));
      });
  });
  class_twiddle_rt<false>(z, c);
  fft_reg<32, false>(z);
  static_for<0, 32>([&](auto K) { o[(long long)(4 * decltype(K)::value + c) * np] = z[decltype(K)::value]; });
}
// np: the scratch u stride (float2)
__device__ __forceinline__ void r2c128_colpair(const float2* col, int cs, float2* o, int src, long long np, int c) {
#if FCB_LARGE_RT
  r2c128_colpair_rt(col, cs, o, src, np, c);
#else
  switch (c) {
    case 0: r2c128_colpair_class<0>(col, cs, o, src, np); break;
    case 1: r2c128_colpair_class<1>(col, cs, o, src, np); break;
    case 2: r2c128_colpair_class<2>(col, cs, o, src, np); break;
    default: r2c128_colpair_class<3>(col, cs, o, src, np); break;
  }
#endif
}

// K1a -> K1b scratch layout: S[plane][u][np] (default), or with
// FCB_LARGE_GLAYOUT=1 grouped, S[row][16-plane group][u][plane][npad]
// (npad = column pairs rounded up to even), so the 16 planes of one u row
// that a K1b CTA reads are one contiguous block -- measured slower (alex1
// bprop 0.89 -> 0.98 ms): K1a's per-plane writes then scatter over 1 MB
// instead of one 60 KB plane.
#ifndef FCB_LARGE_GLAYOUT
#define FCB_LARGE_GLAYOUT 0
#endif
__host__ __device__ inline int large_npad(int np) { return FCB_LARGE_GLAYOUT ? (np + 1) & ~1 : np; }
// scratch of plane (row rl, column j): base pointer (u = 0) and u stride
__device__ __forceinline__ float2* large_scr_plane(float2* scr, int rl, int j, int J, int np, long long& ustride) {
#if FCB_LARGE_GLAYOUT
  const int npad = large_npad(np), ngj = (J + 15) >> 4;
  ustride = 16LL * npad;
  return scr + (((long long)(rl * ngj + (j >> 4)) * kL) * 16 + (j & 15)) * npad;
#else
  ustride = np;
  return scr + (long long)(rl * J + j) * kL * np;
#endif
}

constexpr int kLColPad = kL + 1;  // odd float2 stride of a staged column pair

// grid = rows * J (one plane per CTA), block = 256 = (column pair p, class
// c): the plane is staged pair-interleaved in smem ([p][y] float2 = (x[y][2p],
// x[y][2p + 1]), odd stride: conflict-free 4-B stores and 8-B reads) with
// coalesced loads; thread (p, c) runs class c of pair p and writes rows
// u = c mod 4 of the packed scratch Z[plane][u][p].
// dynamic smem = ceil(src / 2) * 129 float2.
__global__ void __launch_bounds__(256, 2) r2c128_cols_kernel(const R2CParams p, int r0, float2* scr) {
  extern __shared__ float2 pair_s[];
  pdl_wait();
  pdl_trigger();
  const int ql = blockIdx.x;
  const int r = r0 + ql / p.J, j = ql % p.J;
  const int src = p.src, np = (src + 1) >> 1;
  const float* in = p.in + (long long)r * p.in_sr + (long long)j * p.in_sj;
  {
    const int x = threadIdx.x & 127, g = threadIdx.x >> 7;
    float* ps = reinterpret_cast<float*>(pair_s) + (x >> 1) * (2 * kLColPad) + (x & 1);
    if (x < 2 * np) {  // row y of the plane: lanes = consecutive columns (coalesced)
#pragma unroll 8
      for (int y = g; y < src; y += 2) ps[2 * y] = x < src ? __ldg(in + y * src + x) : 0.f;
    }
  }
  __syncthreads();
  const int pp = threadIdx.x & 63, c = threadIdx.x >> 6;
  if (pp >= np) return;
  long long us;
  float2* o = large_scr_plane(scr, ql / p.J, j, p.J, np, us) + pp;
  r2c128_colpair(pair_s + pp * kLColPad, 1, o, src, us, c);
}

// K1a with the planes streamed by 1-D bulk copies (TMA) through a 2-stage
// ring: a persistent CTA computes plane i from one stage while plane i + 1
// lands in the other, so the loads no longer serialise with the FFTs.
// Needs src even and 16-B aligned contiguous planes (host checks); the
// stage holds the plane row-major ([y][x], 8-B column-pair reads,
// conflict-free).  dynamic smem = 16 + 2 * round_up(src * src * 4, 16).
__global__ void __launch_bounds__(256, 2) r2c128_cols_bulk_kernel(const R2CParams p, int r0, int nplanes,
                                                                 float2* scr) {
  extern __shared__ __align__(16) unsigned char lsm[];
  uint64_t* bar = reinterpret_cast<uint64_t*>(lsm);
  const int src = p.src, np = src >> 1;
  const uint32_t pbytes = (uint32_t)(src * src * 4);
  const uint32_t sbytes = (pbytes + 15u) & ~15u;
  auto plane_in = [&](int ql) {
    const int r = r0 + ql / p.J, j = ql % p.J;
    return p.in + (long long)r * p.in_sr + (long long)j * p.in_sj;
  };
  const int G = gridDim.x;
  if (threadIdx.x == 0) {
    mbar_init(bar, 1);
    mbar_init(bar + 1, 1);
    fence_barrier_init();
  }
  __syncthreads();
  pdl_wait();
  pdl_trigger();
  const uint64_t pol = l2_policy_evict_first();
  if (threadIdx.x == 0)
    for (int s = 0; s < 2; ++s) {
      const int ql = blockIdx.x + s * G;
      if (ql < nplanes) {
        mbar_arrive_expect_tx(bar + s, pbytes);
        bulk_load(lsm + 16 + s * sbytes, plane_in(ql), pbytes, bar + s, pol);
      }
    }
  const int pp = threadIdx.x & 63, c = threadIdx.x >> 6;
  int it = 0;
  for (int ql = blockIdx.x; ql < nplanes; ql += G, ++it) {
    const int s = it & 1;
    mbar_wait(bar + s, (it >> 1) & 1);
    const float2* stage = reinterpret_cast<const float2*>(lsm + 16 + s * sbytes);
    if (pp < np) {
      long long us;
      float2* o = large_scr_plane(scr, ql / p.J, ql % p.J, p.J, np, us) + pp;
      r2c128_colpair(stage + pp, np, o, src, us, c);
    }
    __syncthreads();  // stage s read by every thread
    if (threadIdx.x == 0 && ql + 2 * G < nplanes) {
      fence_proxy_async_smem();
      mbar_arrive_expect_tx(bar + s, pbytes);
      bulk_load(lsm + 16 + s * sbytes, plane_in(ql + 2 * G), pbytes, bar + s, pol);
    }
  }
}

// ---------------------------------------------------------------- r2c K1b
template <int H>
__device__ __forceinline__ void r2c128_row_class(const float2* row, float2 (&z)[32], int src) {
  // 16-B pair reads: the staged row is zero-filled up to the even edge, so
  // x0 < src (x0 even) makes the pair (x0, x0 + 1) safe to read whole
  const float4* row4 = reinterpret_cast<const float4*>(row);
  static_for<0, 16>([&](auto X2) {
    constexpr int x0 = 2 * decltype(X2)::value;
    const float4 v = x0 < src ? row4[x0 / 2] : make_float4(0.f, 0.f, 0.f, 0.f);
    z[x0] = make_float2(v.x, v.y);
    z[x0 + 1] = make_float2(v.z, v.w);
  });
  static_for<1, 4>([&](auto Q) {
    constexpr int q = decltype(Q)::value;
    if (32 * q < src)
      static_for<0, 16>([&](auto X2) {
        constexpr int x0 = 2 * decltype(X2)::value;
        if (x0 + 32 * q < src) {
          const float4 v = row4[(x0 + 32 * q) / 2];
          z[x0] = cadd(z[x0], rot_i<false, (H * q) & 3>(make_float2(v.x, v.y)));
          z[x0 + 1] = cadd(z[x0 + 1], rot_i<false, (H * q) & 3>(make_float2(v.z, v.w)));
        }
      });
  });
  class_twiddle<false, H>(z);
  fft_reg<32, false>(z);
}

__device__ __forceinline__ void r2c128_row(const float2* row, float2 (&z)[32], int src, int h) {
#if FCB_LARGE_RT
  const float4* row4 = reinterpret_cast<const float4*>(row);
  static_for<0, 16>([&](auto X2) {
    constexpr int x0 = 2 * decltype(X2)::value;
    const float4 v = x0 < src ? row4[x0 / 2] : make_float4(0.f, 0.f, 0.f, 0.f);
    z[x0] = make_float2(v.x, v.y);
    z[x0 + 1] = make_float2(v.z, v.w);
  });
  static_for<1, 4>([&](auto Q) {
    constexpr int q = decltype(Q)::value;
    if (32 * q < src)
      static_for<0, 16>([&](auto X2) {
        constexpr int x0 = 2 * decltype(X2)::value;
        if (x0 + 32 * q < src) {
          const float4 v = row4[(x0 + 32 * q) / 2];
          z[x0] = cadd(z[x0], rot_i_rt<false>(make_float2(v.x, v.y), h * q));
          z[x0 + 1] = cadd(z[x0 + 1], rot_i_rt<false>(make_float2(v.z, v.w), h * q));
        }
      });
  });
  class_twiddle_rt<false>(z, h);
  fft_reg<32, false>(z);
#else
  switch (h) {
    case 0: r2c128_row_class<0>(row, z, src); break;
    case 1: r2c128_row_class<1>(row, z, src); break;
    case 2: r2c128_row_class<2>(row, z, src); break;
    default: r2c128_row_class<3>(row, z, src); break;
  }
#endif
}

constexpr int kLRowPad = kL + 1;                 // odd float2 stride of K4a's output rows
// K1b's staged rows: even float2 stride so column pairs are 16-B reads
// (quarter-warp lanes jl at 4 jl banks: conflict-free)
constexpr int kLRowPadF = kL + 2;
constexpr int kLRowBuf = 16 * kLRowPadF;         // float2 per staged u row (>= 128 x 16 tile)
constexpr int kLUPerCta = 2;                     // u rows per K1b / K4a CTA
constexpr int kLUPairs = (kLRows + kLUPerCta - 1) / kLUPerCta;
// K1b / K4a grid order: u pairs fastest (FCB_LARGE_UFAST, default on), so
// CTAs resident together read adjacent scratch / product rows of the same
// planes; else sample rows fastest.
#ifndef FCB_LARGE_UFAST
#define FCB_LARGE_UFAST 1
#endif
__device__ __forceinline__ int large_bu() { return FCB_LARGE_UFAST ? blockIdx.x : blockIdx.z; }
__device__ __forceinline__ int large_br() { return FCB_LARGE_UFAST ? blockIdx.z : blockIdx.x; }
__host__ inline dim3 large_row_grid(int rows, int groups) {
  return FCB_LARGE_UFAST ? dim3(kLUPairs, groups, rows) : dim3(rows, groups, kLUPairs);
}

// grid = large_row_grid(ceil(rows / rpc), kpad / 16 or 1), block = 128 =
// (u row, slot jl, v class h).  The 16 staged scratch rows of a u row are
// overwritten by its [v][slot] output tile once every thread holds its FFT.
// A slot is one plane of the operand row: with kpad >= 16 the CTA's 16 slots
// are planes j0 .. j0 + 15 of row r; with a narrow kpad of 4 / 8 (a
// first-layer f = 3) they are rpc = 16 / kpad consecutive rows x kpad planes
// -- the same 16 consecutive complex of every bin row of F[t][R][kpad], so
// the output is still one full 128-B line per bin (the first cut left 12 of
// 16 slots idle and wrote 32-B pieces).  Rows >= r1 (the chunk end) are
// neither read nor written.
template <bool NARROW>
__global__ void __launch_bounds__(128, 6) r2c128_rows_kernel(const R2CParams p, int r0, int r1, const float2* scr) {
  __shared__ __align__(16) float2 buf[kLUPerCta * kLRowBuf];
  pdl_wait();
  pdl_trigger();
  const int kp = p.kpad;
  constexpr bool narrow = NARROW;  // the launcher's choice: kpad < 16
  const int rpc = narrow ? 16 / kp : 1;
  const int rl0 = large_br() * rpc;  // first row of the CTA (relative to r0)
  const int j0 = narrow ? 0 : blockIdx.y * 16;
  const int nrows = min(rpc, r1 - (r0 + rl0));  // rows of this CTA inside the chunk
  // slot jl -> (row rl0 + sub, plane j)
  auto slot_row = [&](int jl) { return narrow ? jl / kp : 0; };
  auto slot_j = [&](int jl) { return narrow ? jl % kp : j0 + jl; };
  auto slot_ok = [&](int jl) { return slot_row(jl) < nrows && slot_j(jl) < p.J; };
  const int src = p.src;
  const int ul = threadIdx.x >> 6, u = large_bu() * kLUPerCta + ul;
  const int t = threadIdx.x & 63;
  float2* rows_s = buf + ul * kLRowBuf;
  const int np = (src + 1) >> 1;
  if (u < kLRows && t < np) {  // separate the packed column pairs (K1a): A = (Z[u] + conj Z[-u]) / 2,
    float2 za[16], zb[16];     //                                          B = (Z[u] - conj Z[-u]) / 2i
    if constexpr (!narrow) {  // 16 planes of one row: one base pointer, plane stride js
      long long us;
      const float2* zp = large_scr_plane(const_cast<float2*>(scr), rl0, j0, p.J, np, us) + t;
#if FCB_LARGE_GLAYOUT
      const long long js = large_npad(np);
#else
      const long long js = (long long)kL * np;
#endif
      const long long ou = (long long)u * us, onu = (long long)((kL - u) & (kL - 1)) * us;
      const int jv = max(0, min(16, p.J - j0));
#pragma unroll
      for (int jl = 0; jl < 16; ++jl)  // all 32 loads in flight before the first use
        if (jl < jv) {
          za[jl] = zp[jl * js + ou];
          zb[jl] = zp[jl * js + onu];
        }
    } else {
#pragma unroll
      for (int jl = 0; jl < 16; ++jl)
        if (slot_ok(jl)) {
          long long us;
          const float2* zp =
              large_scr_plane(const_cast<float2*>(scr), rl0 + slot_row(jl), slot_j(jl), p.J, np, us) + t;
          za[jl] = zp[(long long)u * us];
          zb[jl] = zp[(long long)((kL - u) & (kL - 1)) * us];
        }
    }
#pragma unroll
    for (int jl = 0; jl < 16; ++jl)
      if (slot_ok(jl)) {  // pair (2t, 2t + 1); a column at x = src (odd src) is zero
        const bool two = 2 * t + 1 < src;
        *reinterpret_cast<float4*>(rows_s + jl * kLRowPadF + 2 * t) =
            make_float4(0.5f * (za[jl].x + zb[jl].x), 0.5f * (za[jl].y - zb[jl].y),
                        two ? 0.5f * (za[jl].y + zb[jl].y) : 0.f, two ? 0.5f * (zb[jl].x - za[jl].x) : 0.f);
      }
  }
  __syncthreads();
  // FFT phase: warp = class h (warp-uniform), lanes = (u row, slot)
  const int h = threadIdx.x >> 5, cul = (threadIdx.x >> 4) & 1, jl = threadIdx.x & 15;
  const int cu = large_bu() * kLUPerCta + cul;
  float2 z[32];
  const bool act = cu < kLRows && slot_ok(jl);
  if (act) {
    r2c128_row(buf + cul * kLRowBuf + jl * kLRowPadF, z, src, h);
  }
  __syncthreads();  // rows read: reuse as the tile
  float2* tile = buf + cul * kLRowBuf;  // [v][16]
  const float csign = p.conj ? -1.f : 1.f;
  uint32_t amx = 0;
  if (cu < kLRows) {
#pragma unroll
    for (int k = 0; k < 32; ++k) {
      const float2 v = act ? make_float2(z[k].x, csign * z[k].y) : make_float2(0.f, 0.f);
      tile[(4 * k + h) * 16 + jl] = v;
      amx = max(amx, max(__float_as_uint(v.x) & 0x7fffffffu, __float_as_uint(v.y) & 0x7fffffffu));
    }
  }
  __syncthreads();
  // 128 bins x 16 slots per u row: one 128-B line per bin (fewer bytes only
  // where the chunk ends inside the CTA's rows, or kpad < 16 on one row)
  const long long bstride = (long long)p.R * kp;  // float2 per bin
  if (u < kLRows) {
    const float2* tile = rows_s;
    float2* out = reinterpret_cast<float2*>(p.out) + (long long)u * kL * bstride + (long long)(r0 + rl0) * kp + j0;
    const int width = narrow ? nrows * kp : min(16, kp - j0);  // complex per bin (even)
    if (width == 16) {
#pragma unroll 8
      for (int i = t; i < kL * 8; i += 64) {
        const int v = i >> 3, part = i & 7;
        *reinterpret_cast<float4*>(out + v * bstride + 2 * part) =
            *reinterpret_cast<const float4*>(tile + v * 16 + 2 * part);
      }
    } else {
      const int hp = width >> 1;  // float4 parts per bin
      for (int i = t; i < kL * hp; i += 64) {
        const int v = i / hp, part = i - v * hp;
        *reinterpret_cast<float4*>(out + v * bstride + 2 * part) =
            *reinterpret_cast<const float4*>(tile + v * 16 + 2 * part);
      }
    }
  }
  if (p.amax) {  // each row's maximum: reduce over the lanes of the same row
    if constexpr (narrow) {
      for (int m = 1; m < kp; m <<= 1) amx = max(amx, __shfl_xor_sync(0xffffffffu, amx, m));
      amx = max(amx, __shfl_xor_sync(0xffffffffu, amx, 16));  // both u rows
      if ((jl % kp) == 0 && cul == 0 && slot_row(jl) < nrows)
        atomicMax(p.amax + r0 + rl0 + slot_row(jl), ((unsigned long long)p.epoch << 32) | amx);
    } else {
      amx = __reduce_max_sync(0xffffffffu, amx);
      if ((threadIdx.x & 31) == 0) atomicMax(p.amax + r0 + rl0, ((unsigned long long)p.epoch << 32) | amx);
    }
  }
}

// ---------------------------------------------------------------- c2r K4a
template <int H, int TS>  // TS = tile stride per bin (float2)
__device__ __forceinline__ void c2r128_row_class(const float2* tile, int jl, float2 (&z)[32]) {
  static_for<0, 32>([&](auto V) { z[decltype(V)::value] = tile[decltype(V)::value * TS + jl]; });
  static_for<1, 4>([&](auto Q) {
    constexpr int q = decltype(Q)::value;
    static_for<0, 32>([&](auto V) {
      constexpr int v0 = decltype(V)::value;
      z[v0] = cadd(z[v0], rot_i<true, (H * q) & 3>(tile[(v0 + 32 * q) * TS + jl]));
    });
  });
  class_twiddle<true, H>(z);
  fft_reg<32, true>(z);
}

template <int TS>
__device__ __forceinline__ void c2r128_row(const float2* tile, int jl, float2 (&z)[32], int h) {
#if FCB_LARGE_RT
  static_for<0, 32>([&](auto V) { z[decltype(V)::value] = tile[decltype(V)::value * TS + jl]; });
  static_for<1, 4>([&](auto Q) {
    constexpr int q = decltype(Q)::value;
    static_for<0, 32>([&](auto V) {
      constexpr int v0 = decltype(V)::value;
      z[v0] = cadd(z[v0], rot_i_rt<true>(tile[(v0 + 32 * q) * TS + jl], h * q));
    });
  });
  class_twiddle_rt<true>(z, h);
  fft_reg<32, true>(z);
#else
  switch (h) {
    case 0: c2r128_row_class<0, TS>(tile, jl, z); break;
    case 1: c2r128_row_class<1, TS>(tile, jl, z); break;
    case 2: c2r128_row_class<2, TS>(tile, jl, z); break;
    default: c2r128_row_class<3, TS>(tile, jl, z); break;
  }
#endif
}

constexpr int kLTile = kL * 17;  // [v][16 planes] with an odd stride (>= kLRowBuf)
static_assert(kLTile >= 16 * kLRowPad, "K4a reuses the input tile for the output rows");

// grid = (rows, ceil(J / 16), ceil(65 / 2)), block = 128 = (u row, plane jl,
// x' class h).  The input tile of a u row is overwritten by its cropped
// output rows once every thread holds its FFT.
__global__ void __launch_bounds__(128, 6) c2r128_rows_kernel(const C2RParams p, int r0, float2* scr) {
  __shared__ __align__(128) float2 buf[kLUPerCta * kLTile];
  __shared__ uint64_t bar;
  // group-major product: each u row's 128 bins x 16 planes are one
  // contiguous 16 KB block -> one bulk copy per row, tile stride 16
  const bool bulk = p.gm && ((uintptr_t)p.in & 15u) == 0;
  if (bulk && threadIdx.x == 0) {
    mbar_init(&bar, 1);
    fence_barrier_init();
  }
  __syncthreads();
  pdl_wait();
  pdl_trigger();
  const int rl = large_br(), r = r0 + rl;
  const int jg = blockIdx.y, j0 = jg * 16;
  const int jv = min(16, p.J - j0);
  const int crop = p.crop;
  const int ul = threadIdx.x >> 6, u = large_bu() * kLUPerCta + ul;
  const int t = threadIdx.x & 63;
  float2* tile = buf + ul * kLTile;
  const float2* in = reinterpret_cast<const float2*>(p.in);
  if (bulk) {
    if (threadIdx.x == 0) {
      const int ngj = (p.J + 15) >> 4, u0 = large_bu() * kLUPerCta;
      const int nr = min(kLUPerCta, kLRows - u0);
      const uint64_t pol = l2_policy_evict_first();
      mbar_arrive_expect_tx(&bar, (uint32_t)nr * kL * 16 * 8);
      for (int i = 0; i < nr; ++i)
        bulk_load(buf + i * kLTile, in + (((long long)r * ngj + jg) * (kL * kLRows) + (long long)(u0 + i) * kL) * 16,
                  kL * 16 * 8, &bar, pol);
    }
    mbar_wait(&bar, 0);
  } else if (u < kLRows) {
    if (p.gm) {  // P[r][J/16][t][16]: the 128 bins x 16 planes of row u are contiguous
      const int ngj = (p.J + 15) >> 4;
      const float4* b = reinterpret_cast<const float4*>(
          in + (((long long)r * ngj + jg) * (kL * kLRows) + (long long)u * kL) * 16);
#pragma unroll 8
      for (int i = t; i < kL * 8; i += 64) {
        const float4 v = __ldg(b + i);
        const int bin = i >> 3, jl = (i & 7) * 2;
        tile[bin * 17 + jl] = make_float2(v.x, v.y);
        tile[bin * 17 + jl + 1] = make_float2(v.z, v.w);
      }
    } else {  // P[t][r][ld]
      const long long bstride = (long long)p.R * p.ld;
#pragma unroll 8
      for (int i = t; i < kL * 16; i += 64) {
        const int v = i >> 4, jl = i & 15;
        tile[v * 17 + jl] = jl < jv ? __ldg(in + ((long long)u * kL + v) * bstride + (long long)r * p.ld + j0 + jl)
                                    : make_float2(0.f, 0.f);
      }
    }
  }
  __syncthreads();
  {  // FFT phase: warp = class h (warp-uniform switch), lanes = (u row, plane)
    const int h = threadIdx.x >> 5, cul = (threadIdx.x >> 4) & 1, jl = threadIdx.x & 15;
    const bool act = large_bu() * kLUPerCta + cul < kLRows && jl < jv;
    float2* ctile = buf + cul * kLTile;
    float2 z[32];
    if (act) {
      if (bulk) c2r128_row<16>(ctile, jl, z, h);
      else c2r128_row<17>(ctile, jl, z, h);
    }
    __syncthreads();  // tile read: reuse it for the output rows [plane][x']
    if (act) {
#pragma unroll
      for (int k = 0; k < 32; ++k)
        if (4 * k + h < crop) ctile[jl * kLRowPad + 4 * k + h] = z[k];
    }
  }
  float2* outb = tile;
  __syncthreads();
  if (u < kLRows)
    for (int l = 0; l < jv; ++l) {
      float2* row = scr + ((long long)(rl * p.J + j0 + l) * kLRows + u) * crop;
#pragma unroll
      for (int x = t; x < kL; x += 64)
        if (x < crop) row[x] = outb[l * kLRowPad + x];
    }
}

// ---------------------------------------------------------------- c2r K4b
template <int C>
__device__ __forceinline__ void c2r128_col_class(const C2RParams& p, const float2* col, int cs, float* o, int crop) {
  float2 z[32];
  static_for<0, 32>([&](auto U) { z[decltype(U)::value] = col[decltype(U)::value * cs]; });
  static_for<1, 4>([&](auto Q) {
    constexpr int q = decltype(Q)::value;
    static_for<0, 32>([&](auto U) {
      constexpr int u0 = decltype(U)::value;
      constexpr int u = u0 + 32 * q;
      const float2 v = u < kLRows ? col[u * cs] : cconj(col[(kL - u) * cs]);
      z[u0] = cadd(z[u0], rot_i<true, (C * q) & 3>(v));
    });
  });
  class_twiddle<true, C>(z);
  fft_reg<32, true>(z);
  const float scale = p.scale;
  const bool accum = p.accum;
  const long long step = 4LL * crop;
  float* d = o + (long long)C * crop;  // walks rows y = 4k + C
  if (accum) {  // branch outside the stores: no speculative loads of *d
    static_for<0, 32>([&](auto K) {
      constexpr int k = decltype(K)::value;
      if (4 * k + C < crop) *d += scale * z[k].x;
      d += step;
    });
  } else {
    static_for<0, 32>([&](auto K) {
      constexpr int k = decltype(K)::value;
      if (4 * k + C < crop) *d = c2r_out(scale * z[k].x, p.relu);
      d += step;
    });
  }
}

__device__ __forceinline__ void c2r128_col_rt(const C2RParams& p, const float2* col, int cs, float* o, int crop,
                                              int c) {
  float2 z[32];
  static_for<0, 32>([&](auto U) { z[decltype(U)::value] = col[decltype(U)::value * cs]; });
  static_for<1, 4>([&](auto Q) {
    constexpr int q = decltype(Q)::value;
    static_for<0, 32>([&](auto U) {
      constexpr int u0 = decltype(U)::value;
      constexpr int u = u0 + 32 * q;
      const float2 v = u < kLRows ? col[u * cs] : cconj(col[(kL - u) * cs]);
      z[u0] = cadd(z[u0], rot_i_rt<true>(v, c * q));
    });
  });
  class_twiddle_rt<true>(z, c);
  fft_reg<32, true>(z);
  const float scale = p.scale;
  const long long step = 4LL * crop;
  float* d = o + (long long)c * crop;  // walks rows y = 4k + c
  if (p.accum) {  // branch outside the stores: no speculative loads of *d
    static_for<0, 32>([&](auto K) {
      if (4 * decltype(K)::value + c < crop) *d += scale * z[decltype(K)::value].x;
      d += step;
    });
  } else {
    static_for<0, 32>([&](auto K) {
      if (4 * decltype(K)::value + c < crop) *d = c2r_out(scale * z[decltype(K)::value].x, p.relu);
      d += step;
    });
  }
}
// thread (x', g) runs classes g and g + 2.  K4b keeps the unrolled class
// copies (FCB_LARGE_RT_K4B=0): with runtime twiddles it turned issue-bound
// (ncu issue 81 %, 295 -> 325 us at alex1) -- its two classes per thread
// already halve the instruction footprint.
#ifndef FCB_LARGE_RT_K4B
#define FCB_LARGE_RT_K4B 0
#endif
__device__ __forceinline__ void c2r128_col_pair(const C2RParams& p, const float2* col, int cs, float* o, int crop,
                                                int g) {
#if FCB_LARGE_RT_K4B
#pragma unroll 1
  for (int c = g; c < 4; c += 2) {
    c2r128_col_rt(p, col, cs, o, crop, c);
    __syncwarp();
  }
#else
  // __syncwarp between the classes keeps their register live ranges apart
  if (g == 0) {
    c2r128_col_class<0>(p, col, cs, o, crop);
    __syncwarp();
    c2r128_col_class<2>(p, col, cs, o, crop);
  } else {
    c2r128_col_class<1>(p, col, cs, o, crop);
    __syncwarp();
    c2r128_col_class<3>(p, col, cs, o, crop);
  }
#endif
}

// grid = rows * J (one plane per CTA), block = 256 = (column x', class
// pair): the plane's 65 x crop scratch rows are staged transposed in smem
// ([x'][u], stride 65: conflict-free 64-bit accesses per half-warp) with
// coalesced loads; thread (x', g) runs classes g and g + 2.
// dynamic smem = crop * 65 float2.
__global__ void __launch_bounds__(256, 2) c2r128_cols_kernel(const C2RParams p, int r0, const float2* scr) {
  extern __shared__ float2 zs[];
  pdl_wait();
  pdl_trigger();
  const int ql = blockIdx.x;
  const int r = r0 + ql / p.J, j = ql % p.J;
  const int crop = p.crop;
  const float2* src = scr + (long long)ql * kLRows * crop;
  const int x = threadIdx.x & 127, g = threadIdx.x >> 7;
  if (x < crop) {  // row u of the scratch plane: lanes = consecutive columns
#pragma unroll 8
    for (int u = g; u < kLRows; u += 2) zs[x * kLRows + u] = src[u * crop + x];
  }
  __syncthreads();
  if (x >= crop) return;
  float* o = p.out + (long long)r * p.out_sr + (long long)j * p.out_sj + x;
  c2r128_col_pair(p, zs + x * kLRows, 1, o, crop, g);
}


// K4b with the scratch plane fetched by one bulk copy (crop even: the
// [65][crop] plane is a 16-B multiple) into a flat smem plane; column x'
// reads stride crop (lanes = consecutive columns, conflict-free).  Same
// FFT and stores as c2r128_cols_kernel.  dynamic smem = 16 + 65 * crop * 8.
__global__ void __launch_bounds__(256, 2) c2r128_cols_flat_kernel(const C2RParams p, int r0, const float2* scr) {
  extern __shared__ __align__(16) unsigned char lsm[];
  uint64_t* bar = reinterpret_cast<uint64_t*>(lsm);
  const float2* zs = reinterpret_cast<const float2*>(lsm + 16);
  const int ql = blockIdx.x;
  const int r = r0 + ql / p.J, j = ql % p.J;
  const int crop = p.crop;
  if (threadIdx.x == 0) {
    mbar_init(bar, 1);
    fence_barrier_init();
  }
  __syncthreads();
  pdl_wait();
  pdl_trigger();
  if (threadIdx.x == 0) {
    const uint32_t bytes = (uint32_t)(kLRows * crop * 8);
    mbar_arrive_expect_tx(bar, bytes);
    bulk_load(lsm + 16, scr + (long long)ql * kLRows * crop, bytes, bar, l2_policy_evict_first());
  }
  const int x = threadIdx.x & 127, g = threadIdx.x >> 7;
  mbar_wait(bar, 0);
  if (x >= crop) return;
  float* o = p.out + (long long)r * p.out_sr + (long long)j * p.out_sj + x;
  c2r128_col_pair(p, zs + x, crop, o, crop, g);
}

}  // namespace fcb
