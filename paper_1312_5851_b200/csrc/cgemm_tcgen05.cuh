// K3: per-frequency-bin complex GEMM on tcgen05 tensor cores, fp32-accurate
// through a 3xTF32 split.  Replaces the three per-bin GEMM lambdas of the
// reference ConvWorkspace (conv_fft.hpp:90-107 fprop, :129-146 bprop,
// :171-189 accGrad).
//
// Per bin t:  D_t (M x Nc complex) = A_t (M x K complex) . op(B_t)^T
//   fprop   : A = X[b][f],   B = W[o][f],  D = Y[b][o]   = sum_f X conj(W)
//   bprop   : A = GY[b][o],  B = W[f][o],  D = GX[b][f]  = sum_o GY W
//   accGrad : A = GY[o][b],  B = X[f][b],  D = GW[o][f]  = sum_b conj(GY) X
//
// Complex arithmetic is embedded in one real GEMM: operand rows hold
// interleaved (re, im) pairs along K, so A is M x 2K real.  The B tile is
// expanded in shared memory into 2*Nc real rows -- Nc "re rows" then Nc
// "im rows" -- whose pair pattern encodes conjugation and the i factor:
//   fprop  : re (p, q)   im (-q, p)
//   bprop  : re (p, -q)  im (q, p)
//   accGrad: re (p, q)   im (q, -p)
// so D[:, 0:Nc] = Re, D[:, Nc:2Nc] = Im after a single MMA per K step.
//
// 3xTF32: every operand x is split as hi = tf32(x), lo = x - hi in smem
// (exact in fp32) and D += Ahi.Bhi + Ahi.Blo + Alo.Bhi, accumulated in
// fp32 TMEM.  This keeps fp32-level accuracy (plain TF32 misses the 1e-4
// bar, SURVEY.md section 7 hard part 4).
//
// Pipeline (one CTA per SM, persistent over tiles (t, m-tile, n-tile)):
//   warp 0      TMA producer: raw fp32 A (128 x 32) and B (Nc x 32) tiles
//               per K chunk of 16 complex, 128-B swizzle, OOB zero fill.
//   warps 4-11  converters: split hi/lo in place, expand B re/im rows,
//               fence.proxy.async, arrive.
//   warp 1      MMA issuer (one thread): 4 K-steps x 3 UMMA (M=128,
//               N=2Nc, K=8) per chunk into a double-buffered TMEM
//               accumulator; tcgen05.commit frees smem / signals epilogue.
//   warps 12-15 epilogue: tcgen05.ld -> (re, im) float2 stores into the
//               bin-major product spectrum P[t][n][2*M_valid] (lanes =
//               consecutive M rows -> coalesced 256-B stores).
//   warp 2      TMEM allocator.
#pragma once
#include <cuda.h>

#include <cstdint>

#include "ptx.cuh"

namespace fcb {

enum GemmMode : int { kModeFprop = 0, kModeBprop = 1, kModeAccGrad = 2 };

struct GemmParams {
  float* out;     // P[t][n][2*m_valid]
  int bins;
  int m_valid;    // A rows (M)
  int n_valid;    // complex output columns (N)
  int k_chunks;   // kpad / 16
  int m_tiles, n_tiles;
  int nc;         // complex columns per N tile (multiple of 8, <= 128)
  int stages;
  int mode;
  int dbg;  // experiment bits (0 in production): 1 skip conversion, 2 hi.hi only,
            // 4 raw A as hi (relies on tf32 truncation), lo = x - trunc(x)
};

constexpr int kGemmThreads = 512;
constexpr int kConvThreads = 256;  // warps 4..11
constexpr int kTileM = 128;
constexpr int kChunkBytesA = kTileM * 128;  // 128 rows x 128 B (32 fp32)

__host__ __device__ inline int gemm_stage_bytes(int nc) {
  return 2 * kChunkBytesA + 2 * (2 * nc * 128);
}

__global__ void __launch_bounds__(kGemmThreads, 1)
    cgemm_bins_tcgen05(const __grid_constant__ CUtensorMap tmA,
                       const __grid_constant__ CUtensorMap tmB, const GemmParams p) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  // 1024-B alignment for the swizzle atoms.
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~uintptr_t(1023));
  const int nc = p.nc;
  const int S = p.stages;
  const int bBytes = 2 * nc * 128;  // expanded B (re rows + im rows)
  const int stageBytes = gemm_stage_bytes(nc);
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + S * stageBytes);
  uint64_t* full = bars;            // TMA -> converters
  uint64_t* conv = bars + S;        // converters -> MMA
  uint64_t* empty = bars + 2 * S;   // MMA -> TMA
  uint64_t* tfull = bars + 3 * S;   // MMA -> epilogue [2]
  uint64_t* tempty = bars + 3 * S + 2;  // epilogue -> MMA [2]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 3 * S + 4);

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const uint32_t tmem_cols = (4 * nc <= 32) ? 32 : (4 * nc <= 64) ? 64 : (4 * nc <= 128) ? 128
                             : (4 * nc <= 256) ? 256 : 512;

  if (threadIdx.x == 0) {
    for (int s = 0; s < S; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&conv[s], kConvThreads);
      mbar_init(&empty[s], 1);
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(&tfull[a], 1);
      mbar_init(&tempty[a], 128);
    }
    fence_barrier_init();
  }
  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&tmA);
    tma_prefetch_desc(&tmB);
  }
  if (warp == 2) tmem_alloc(tmem_slot, tmem_cols);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  const int tiles_per_bin = p.m_tiles * p.n_tiles;
  const int total_tiles = p.bins * tiles_per_bin;
  const int kc_n = p.k_chunks;

  if (warp == 0) {
    // ------------------------------------------------ TMA producer
    if (lane == 0) {
      int s = 0;
      uint32_t ph = 0;
      const uint32_t tx = kChunkBytesA + nc * 128;
      for (int tile = blockIdx.x; tile < total_tiles; tile += gridDim.x) {
        const int t = tile / tiles_per_bin;
        const int rem = tile - t * tiles_per_bin;
        const int mt = rem / p.n_tiles, nt = rem - mt * p.n_tiles;
        for (int kc = 0; kc < kc_n; ++kc) {
          mbar_wait(&empty[s], ph ^ 1);
          uint8_t* st = smem + s * stageBytes;
          mbar_arrive_expect_tx(&full[s], tx);
          tma_load_3d(st, &tmA, &full[s], kc * 32, mt * kTileM, t);
          tma_load_3d(st + 2 * kChunkBytesA, &tmB, &full[s], kc * 32, nt * nc, t);
          if (++s == S) { s = 0; ph ^= 1; }
        }
      }
    }
  } else if (warp == 1) {
    // ------------------------------------------------ MMA issuer
    const uint32_t idesc = umma_idesc_tf32(kTileM, 2 * nc);
    int s = 0;
    uint32_t ph = 0;
    int local = 0;
    for (int tile = blockIdx.x; tile < total_tiles; tile += gridDim.x, ++local) {
      const int a = local & 1;
      const uint32_t aph = (local >> 1) & 1;
      mbar_wait(&tempty[a], aph ^ 1);
      tc_fence_after();
      const uint32_t d_tmem = tmem_base + a * (2 * nc);
      for (int kc = 0; kc < kc_n; ++kc) {
        mbar_wait(&conv[s], ph);
        tc_fence_after();
        if (lane == 0) {
          const uint32_t st = smem_u32(smem + s * stageBytes);
          const uint32_t a_hi = st, a_lo = st + kChunkBytesA;
          const uint32_t b_hi = st + 2 * kChunkBytesA, b_lo = b_hi + bBytes;
#pragma unroll
          for (int kk = 0; kk < 4; ++kk) {
            const uint32_t off = kk * 32;
            const uint64_t dah = umma_desc_sw128(a_hi + off);
            const uint64_t dal = umma_desc_sw128(a_lo + off);
            const uint64_t dbh = umma_desc_sw128(b_hi + off);
            const uint64_t dbl = umma_desc_sw128(b_lo + off);
            umma_tf32(d_tmem, dah, dbh, idesc, (kc | kk) ? 1u : 0u);
            if (!(p.dbg & 2)) {
              umma_tf32(d_tmem, dah, dbl, idesc, 1u);
              umma_tf32(d_tmem, dal, dbh, idesc, 1u);
            }
          }
          umma_commit(&empty[s]);
          if (kc == kc_n - 1) umma_commit(&tfull[a]);
        }
        __syncwarp();
        if (++s == S) { s = 0; ph ^= 1; }
      }
    }
  } else if (warp >= 4 && warp < 12) {
    // ------------------------------------------------ converters
    const int ct = threadIdx.x - 128;  // 0..255
    float s1 = 1.f, s2 = 1.f, s3 = 1.f;  // re=(p, s1 q)  im=(s2 q, s3 p)
    // fprop: re (p,q) im (-q,p); bprop: re (p,-q) im (q,p); accGrad: re (p,q) im (q,-p)
    bool swap_im = true;
    if (p.mode == kModeFprop) { s1 = 1.f; s2 = -1.f; s3 = 1.f; }
    else if (p.mode == kModeBprop) { s1 = -1.f; s2 = 1.f; s3 = 1.f; }
    else { s1 = 1.f; s2 = 1.f; s3 = -1.f; }
    (void)swap_im;
    int s = 0;
    uint32_t ph = 0;
    for (int tile = blockIdx.x; tile < total_tiles; tile += gridDim.x) {
      for (int kc = 0; kc < kc_n; ++kc) {
        mbar_wait(&full[s], ph);
        if (p.dbg & 1) {
          fence_proxy_async_smem();
          mbar_arrive(&conv[s]);
          if (++s == S) { s = 0; ph ^= 1; }
          continue;
        }
        uint8_t* st = smem + s * stageBytes;
        float4* ahi = reinterpret_cast<float4*>(st);
        float4* alo = reinterpret_cast<float4*>(st + kChunkBytesA);
        if (p.dbg & 4) {
#pragma unroll 4
          for (int i = ct; i < kChunkBytesA / 16; i += kConvThreads) {
            const float4 v = ahi[i];
            float4 l;
            l.x = v.x - __uint_as_float(__float_as_uint(v.x) & 0xFFFFE000u);
            l.y = v.y - __uint_as_float(__float_as_uint(v.y) & 0xFFFFE000u);
            l.z = v.z - __uint_as_float(__float_as_uint(v.z) & 0xFFFFE000u);
            l.w = v.w - __uint_as_float(__float_as_uint(v.w) & 0xFFFFE000u);
            alo[i] = l;
          }
        } else {
#pragma unroll 4
          for (int i = ct; i < kChunkBytesA / 16; i += kConvThreads) {
            const float4 v = ahi[i];
            float4 h, l;
            h.x = tf32_round(v.x); l.x = v.x - h.x;
            h.y = tf32_round(v.y); l.y = v.y - h.y;
            h.z = tf32_round(v.z); l.z = v.z - h.z;
            h.w = tf32_round(v.w); l.w = v.w - h.w;
            ahi[i] = h;
            alo[i] = l;
          }
        }
        float4* bre_hi = reinterpret_cast<float4*>(st + 2 * kChunkBytesA);
        float4* bim_hi = reinterpret_cast<float4*>(st + 2 * kChunkBytesA + nc * 128);
        float4* bre_lo = reinterpret_cast<float4*>(st + 2 * kChunkBytesA + bBytes);
        float4* bim_lo = reinterpret_cast<float4*>(st + 2 * kChunkBytesA + bBytes + nc * 128);
        const int nb = nc * 8;  // float4 per raw B tile
#pragma unroll 2
        for (int i = ct; i < nb; i += kConvThreads) {
          const float4 v = bre_hi[i];  // (p0, q0, p1, q1)
          const float4 re = make_float4(v.x, s1 * v.y, v.z, s1 * v.w);
          const float4 im = make_float4(s2 * v.y, s3 * v.x, s2 * v.w, s3 * v.z);
          float4 h, l;
          h.x = tf32_round(re.x); l.x = re.x - h.x;
          h.y = tf32_round(re.y); l.y = re.y - h.y;
          h.z = tf32_round(re.z); l.z = re.z - h.z;
          h.w = tf32_round(re.w); l.w = re.w - h.w;
          bre_hi[i] = h;
          bre_lo[i] = l;
          h.x = tf32_round(im.x); l.x = im.x - h.x;
          h.y = tf32_round(im.y); l.y = im.y - h.y;
          h.z = tf32_round(im.z); l.z = im.z - h.z;
          h.w = tf32_round(im.w); l.w = im.w - h.w;
          bim_hi[i] = h;
          bim_lo[i] = l;
        }
        fence_proxy_async_smem();
        mbar_arrive(&conv[s]);
        if (++s == S) { s = 0; ph ^= 1; }
      }
    }
  } else if (warp >= 12) {
    // ------------------------------------------------ epilogue
    const int q = warp & 3;  // TMEM lane quadrant accessible to this warp
    const int row = q * 32 + lane;
    int local = 0;
    for (int tile = blockIdx.x; tile < total_tiles; tile += gridDim.x, ++local) {
      const int t = tile / tiles_per_bin;
      const int rem = tile - t * tiles_per_bin;
      const int mt = rem / p.n_tiles, nt = rem - mt * p.n_tiles;
      const int a = local & 1;
      const uint32_t aph = (local >> 1) & 1;
      mbar_wait(&tfull[a], aph);
      tc_fence_after();
      const int m = mt * kTileM + row;
      const bool mok = m < p.m_valid;
      const uint32_t tbase = tmem_base + ((uint32_t)(q * 32) << 16) + a * (2 * nc);
      float2* out = reinterpret_cast<float2*>(p.out) + (long long)t * p.n_valid * p.m_valid + m;
      for (int nb = 0; nb < nc; nb += 16) {
        float re[16], im[16];
        tmem_ld_32x32b_x16(tbase + nb, re);
        tmem_ld_32x32b_x16(tbase + nc + nb, im);
        tmem_ld_wait();
        const int n0 = nt * nc + nb;
#pragma unroll
        for (int i = 0; i < 16; ++i) {
          const int n = n0 + i;
          if (mok && nb + i < nc && n < p.n_valid)
            out[(long long)n * p.m_valid] = make_float2(re[i], im[i]);
        }
      }
      tc_fence_before();
      mbar_arrive(&tempty[a]);
    }
  }

  __syncthreads();
  if (warp == 2) {
    tc_fence_after();
    tmem_dealloc(tmem_base, tmem_cols);
  }
}

}  // namespace fcb
