// K3: per-frequency-bin complex GEMM on tcgen05 tensor cores, fp32-accurate
// through a 3xTF32 split.  Replaces the three per-bin GEMM lambdas of the
// reference ConvWorkspace (conv_fft.hpp:90-107 fprop, :129-146 bprop,
// :171-189 accGrad).
//
// Per bin t:  D_t (M x Nc complex) = A_t (M x K complex) . op(B_t)^T
//   fprop   : A = X[b][f],   B = W[o][f],        D = Y[b][o]  = sum_f X conj(W)
//   bprop   : A = GY[b][o],  B = conj(W)[f][o],  D = GX[b][f] = sum_o GY W
//             (K1 stores the conjugate spectrum for this operand)
//   accGrad : A = GY[o][b],  B = X[f][b],        D = GW[o][f] = sum_b conj(GY) X
//             (computed as -conj of the fprop form: the epilogue negates Im)
// so all three share one product: D = A . conj(B)^T.
//
// Complex arithmetic is embedded in one real GEMM.  Operand rows hold
// interleaved (re, im) pairs along K, so A is M x 2K real.  In shared memory
// the B tile becomes 2*Nc real rows: the Nc raw rows (p, q) give Re(D), and
// Nc derived rows (-q, p) give Im(D).  One MMA per K step (N = 2*Nc) thus
// writes [Re | Im] into TMEM.
//
// 3xTF32: x = hi + lo with hi = x truncated to tf32 (the tensor core's own
// fp32 -> tf32 conversion, so raw fp32 is the hi operand) and lo = x - hi
// (exact).  D += Ahi.Bhi + Ahi.Blo + Alo.Bhi in fp32 TMEM keeps fp32-level
// accuracy (plain TF32 misses the 1e-4 bar, SURVEY.md section 7 part 4).
//
// The A operand (128 rows) lives in TMEM: the A converters read the TMA'd
// raw chunk row-per-thread and tcgen05.st both hi and lo into a TMEM
// staging buffer, so the MMAs read A from TMEM (".kind::tf32 [d], [a], b")
// and only B needs hi/lo copies in shared memory.
//
// Pipeline (one CTA per SM, persistent over tiles (t, m-tile, n-tile)):
//   warp 0      TMA: raw fp32 A (128 x 32) and B (Nc x 32) per K chunk of
//               16 complex into a ring of raw stages; 128-B swizzle; OOB
//               rows/cols zero-filled
//   warps 4-7   A converters (thread = row): raw stage -> regs -> TMEM hi/lo
//   warps 8-11  B converters: raw stage -> one of two converted-B buffers
//               (re = raw, im rows, lo rows, lo-im rows), fence.proxy.async
//   warp 1      MMA issuer (one thread): 4 K-steps x 3 UMMA (M=128,
//               N=2Nc, K=8) per chunk, double-buffered TMEM accumulator
//   warps 12-19 epilogue: tcgen05.ld -> float2 (re, im) stores into the
//               product spectrum P[t][n][m] (lanes = consecutive m rows);
//               two warps per TMEM lane quadrant split the 16-column blocks
//               (a tile's 98 KB of stores from 4 warps took longer than its
//               MMAs and stalled the accumulator double buffer)
//   warp 2      TMEM allocator
// Both converter groups release a raw stage as soon as they have read it,
// so the TMA runs up to RS chunks ahead of the MMAs (the first cut held each
// stage until its MMAs retired, which capped the loads in flight at ~2
// chunks and left the tensor pipe ~50% idle at the paper point).
#pragma once
#include <cuda.h>

#include <cstdint>

#include "ptx.cuh"

namespace fcb {

struct GemmParams {
  float* out;     // product spectrum, complex element (t, n, m) at
                  // t*s_t + (m/gm)*s_mg + n*s_n + m%gm (see OutLayout)
  int bins;
  int m_valid;    // A rows (M)
  int n_valid;    // complex output columns (N)
  int k_chunks;   // kpad / 16
  int m_tiles, n_tiles;
  int nc;         // complex columns per N tile (multiple of 16, <= 96)
  int stages;
  float im_sign;  // +1 (fprop, bprop) or -1 (accGrad)
  long long s_t, s_mg, s_n;  // output strides in complex elements
  int gm_log2;                // log2 of the m-group size gm
  // per operand row, the max-magnitude words written by K1 (R2CParams::amax;
  // low 32 bits = float bits): the fp16x3 scale and the auto selection
  const unsigned long long* amax_a;
  const unsigned long long* amax_b;
  int rows_a, rows_b;
  // 0: run; 1: run only if every operand row is within kF16SafeBinades of
  // its operand's maximum (fp16x3 is exact enough); 2: run only if not
  // (the 3xTF32 fallback of the same launch pair)
  int select;
  int* path;  // optional: the kernel that runs writes 1 (fp16x3) or 0 (3xTF32)
  unsigned long long* tspan = nullptr;  // live span slot (ptx.cuh)
};

// fp16x3 keeps ~2^-20 row-relative accuracy for rows within 2^18 of the
// operand maximum (global power-of-two scale, fp16 subnormal floor 2^-38).
constexpr int kF16SafeBinades = 18;

constexpr int kGemmThreads = 640;
constexpr int kTileM = 128;
constexpr int kChunkBytesA = kTileM * 128;  // 128 rows x 128 B (32 fp32)
constexpr int kMaxNc = 96;                  // TMEM: 2 x 2*96 accumulator + 2 x 64 A columns
constexpr int kBConvF16 = 192;              // fp16 B converters: warps 2, 3, 8-11

// FCB_GEMM_TRACE: per-chunk clock64 timeline of CTA 0, printed at exit
// (development builds only).
#ifdef FCB_GEMM_TRACE
__device__ long long g_gemm_trace[6][64];
__device__ unsigned long long g_cta_time[3][160];  // globaltimer: launch, work start, end
__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
#ifndef FCB_GEMM_TRACE_G0
#define FCB_GEMM_TRACE_G0 0  // first traced chunk (a steady-state window: > 0)
#endif
#define GTRACE(ev, idx)                                                                 \
  do {                                                                                  \
    const int i_ = (int)(idx) - ((ev) == 5 ? 0 : FCB_GEMM_TRACE_G0);                    \
    if (blockIdx.x == 0 && i_ >= 0 && i_ < 64) g_gemm_trace[ev][i_] = clock64();        \
  } while (0)
#else
#define GTRACE(ev, idx) \
  do {                  \
  } while (0)
#endif

// Tile order.  One tile per bin (P, the narrow first layers; RANGES, a
// template flag so the loops keep a constant stride): contiguous bin ranges
// per CTA (P step 265 -> 260 us: each CTA's product and operand pieces are
// adjacent).  Several tiles per bin (W): round-robin, bins
// outermost -- the tiles of one bin share its operand rows in L2 (contiguous
// ranges measured 1.67 -> 1.72 ms at W, S = 16).
template <bool RANGES>
__device__ __forceinline__ void decode_tile(int tile, const GemmParams& p, int& t, int& mt, int& nt) {
  if (RANGES) {  // one tile per bin
    t = tile;
    mt = nt = 0;
    return;
  }
  const int tpb = p.m_tiles * p.n_tiles;
  t = tile / tpb;
  const int rem = tile - t * tpb;
  mt = rem / p.n_tiles;
  nt = rem - mt * p.n_tiles;
}

// One raw stage holds one K chunk (tf32 mode) or two (fp16 mode: a 128-B
// fp16 row covers 32 complex).
__host__ __device__ inline int gemm_raw_stage_bytes(int nc, bool f16 = false) {
  return (f16 ? 2 : 1) * (kChunkBytesA + nc * 128);  // raw A | raw B (x2: A0 A1 B0 B1)
}

// fp16 operand scaling: max|x| < 2^e  ->  x * 2^(14 - e) < 2^14, inside the
// fp16 range with headroom; 0 / non-finite maxima keep scale 1.
__device__ __forceinline__ int amax_exp(unsigned long long w) {
  const float a = __uint_as_float((uint32_t)w);
  if (!(a > 0.f) || !isfinite(a)) return 14;
  int e;
  frexpf(a, &e);
  return max(-100, min(e, 120));
}

// x -> hi + mid: hi = x rounded to an 11-bit significand in fp32 (exact in
// fp16 for the scaled range), mid = x - hi (exact, |mid| <= 2^-11 |x|), so
// hi + rn16(mid) = x to ~2^-22 relative.
struct Split {
  float hi, mid;
};
__device__ __forceinline__ Split split11(float x) {
  const float h = __uint_as_float((__float_as_uint(x) + 0x1000u) & 0xffffe000u);
  return {h, x - h};
}
// fp16x2 with `lo` in the low half (= the even K element)
__device__ __forceinline__ uint32_t pack_f16x2(float lo, float hi) {
  const __half2 h = __floats2half2_rn(lo, hi);
  return *reinterpret_cast<const uint32_t*>(&h);
}
__device__ __forceinline__ void split_f16x2(float x0, float x1, uint32_t& hi, uint32_t& mid) {
  const Split a = split11(x0), b = split11(x1);
  hi = pack_f16x2(a.hi, b.hi);
  mid = pack_f16x2(a.mid, b.mid);
}
__host__ __device__ inline int gemm_bbuf_bytes(int nc) {
  return 4 * nc * 128;  // B re (= raw) | B im | B lo re | B lo im
}

// F16 = false: 3xTF32 (hi = raw fp32, lo = x - tf32(x)); true: 3xFP16 on
// per-operand power-of-two scaled values, kind::f16 MMAs (twice the K per
// instruction), hi.hi + hi.mid + mid.hi.
template <bool F16, bool RANGES>
__global__ void __launch_bounds__(kGemmThreads, 1)
    cgemm_bins_tcgen05(const __grid_constant__ CUtensorMap tmA,
                       const __grid_constant__ CUtensorMap tmB, const GemmParams p) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
#ifdef FCB_GEMM_TRACE
  if (threadIdx.x == 0 && blockIdx.x < 160) g_cta_time[0][blockIdx.x] = gtimer();
#endif
  // 1024-B alignment for the swizzle atoms, derived from the __shared__
  // pointer so the converters' accesses compile to LDS/STS.
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  const int nc = p.nc;
  const int RS = p.stages;  // raw stages
  const int rowsB = nc * 128;  // bytes of nc rows
  const int rawBytes = gemm_raw_stage_bytes(nc, F16);
  const int offB = (F16 ? 2 : 1) * kChunkBytesA;  // raw B within a stage
  uint8_t* bbuf0 = smem + RS * rawBytes;  // 2 converted-B buffers
  const int bbufBytes = gemm_bbuf_bytes(nc);
  uint64_t* bars = reinterpret_cast<uint64_t*>(bbuf0 + 2 * bbufBytes);
  uint64_t* rfull = bars;               // TMA -> converters          [RS]
  uint64_t* rempty = bars + RS;         // converters -> TMA          [RS]
  uint64_t* aready = bars + 2 * RS;     // A converters -> MMA        [2]
  uint64_t* bready = aready + 2;        // B converters -> MMA        [2]
  uint64_t* atfree = bready + 2;        // MMA -> A converters (TMEM) [2]
  uint64_t* bfree = atfree + 2;         // MMA -> B converters (smem) [2]
  uint64_t* tfull = bfree + 2;          // MMA -> epilogue            [2]
  uint64_t* tempty = tfull + 2;         // epilogue -> MMA            [2]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  constexpr uint32_t kTmemCols = 512;
  const uint32_t a_col0 = 4 * nc;  // A staging: 2 buffers x (32 hi + 32 lo) columns

  if (threadIdx.x == 0) {
    for (int s = 0; s < RS; ++s) {
      mbar_init(&rfull[s], 1);
      mbar_init(&rempty[s], F16 ? 128 + kBConvF16 : 256);  // every A and B converter thread
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(&aready[a], 128);
      mbar_init(&bready[a], F16 ? kBConvF16 : 128);
      mbar_init(&atfree[a], 1);
      mbar_init(&bfree[a], 1);
      mbar_init(&tfull[a], 1);
      mbar_init(&tempty[a], 256);
    }
    fence_barrier_init();
  }
  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&tmA);
    tma_prefetch_desc(&tmB);
  }
  if (warp == 2) tmem_alloc(tmem_slot, kTmemCols);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  pdl_wait();  // prologue above overlaps the previous kernel's tail
  pdl_trigger();
#ifdef FCB_GEMM_TRACE
  if (threadIdx.x == 0 && blockIdx.x < 160) g_cta_time[1][blockIdx.x] = gtimer();
#endif

  const int tiles_per_bin = p.m_tiles * p.n_tiles;
  const int total_tiles = p.bins * tiles_per_bin;
  // RANGES (the launcher's choice: one tile per bin): contiguous tile ranges
  const int per = (total_tiles + gridDim.x - 1) / gridDim.x;
  const int tile_b = RANGES ? blockIdx.x * per : blockIdx.x;
  const int tile_e = RANGES ? min(total_tiles, tile_b + per) : total_tiles;
  const int tile_s = RANGES ? 1 : gridDim.x;
  // pipeline steps per tile: K chunks (tf32) or chunk pairs (fp16)
  const int kc_n = F16 ? (p.k_chunks + 1) >> 1 : p.k_chunks;
  int ea = 14, eb = 14;  // fp16 operand scale exponents
  if (F16 || p.select != 0) {
    // operand maxima and smallest non-zero row maxima (float bits order as
    // the values): the fp16 scales and the fp16x3 / 3xTF32 choice
    uint32_t* dec = tmem_slot + 4;  // max A, min A, max B, min B (inside the 256-B barrier tail)
    if (threadIdx.x < 4) dec[threadIdx.x] = (threadIdx.x & 1) ? 0xffffffffu : 0u;
    __syncthreads();
    uint32_t v[4] = {0u, 0xffffffffu, 0u, 0xffffffffu};
    for (int r = threadIdx.x; r < p.rows_a; r += blockDim.x) {
      const uint32_t b = (uint32_t)p.amax_a[r];
      if (b) { v[0] = max(v[0], b); v[1] = min(v[1], b); }
    }
    for (int r = threadIdx.x; r < p.rows_b; r += blockDim.x) {
      const uint32_t b = (uint32_t)p.amax_b[r];
      if (b) { v[2] = max(v[2], b); v[3] = min(v[3], b); }
    }
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const uint32_t w = (i & 1) ? __reduce_min_sync(0xffffffffu, v[i]) : __reduce_max_sync(0xffffffffu, v[i]);
      if (lane == 0) {
        if (i & 1) atomicMin(&dec[i], w);
        else atomicMax(&dec[i], w);
      }
    }
    __syncthreads();
    ea = amax_exp(dec[0]);
    eb = amax_exp(dec[2]);
    auto spread = [](uint32_t mx, uint32_t mn) {  // binades between max and min row maxima
      return mn == 0xffffffffu ? 0 : (int)((mx >> 23) & 0xffu) - (int)((mn >> 23) & 0xffu);
    };
    const bool safe = spread(dec[0], dec[1]) <= kF16SafeBinades && spread(dec[2], dec[3]) <= kF16SafeBinades;
    if (p.select != 0 && (p.select == 1) != safe) {  // the other kernel of the pair runs
      __syncthreads();
      if (warp == 2) {
        tc_fence_after();
        tmem_dealloc(tmem_base, kTmemCols);
      }
      return;
    }
  }
  if (p.path && blockIdx.x == 0 && threadIdx.x == 0) *p.path = F16 ? 1 : 0;
  span_begin(p.tspan);  // the kernel of an auto pair that runs

  if (warp == 0) {
    // ------------------------------------------------ TMA producer
    if (lane == 0) {
      int s = 0;
      uint32_t ph = 0;
      int gi = 0;
      (void)gi;
      // operand spectra are read by the tiles of one bin at about the same
      // time, then never again: evict them first, so the product the c2r
      // reads next stays in L2 (FCB_GEMM_EVF=0: default policy)
#ifndef FCB_GEMM_EVF
#define FCB_GEMM_EVF 1
#endif
      // (only an operand no other tile re-reads: A when one N tile covers the
      // bin, B when one M tile does -- W re-reads A three times)
      const uint64_t pol_first = l2_policy_evict_first(), pol_norm = l2_policy_evict_normal();
      const uint64_t pol_a = (FCB_GEMM_EVF && p.n_tiles == 1) ? pol_first : pol_norm;
      const uint64_t pol_b = (FCB_GEMM_EVF && p.m_tiles == 1) ? pol_first : pol_norm;
      for (int tile = tile_b; tile < tile_e; tile += tile_s) {
        int t, mt, nt;
        decode_tile<RANGES>(tile, p, t, mt, nt);
        for (int kc = 0; kc < kc_n; ++kc) {
          mbar_wait(&rempty[s], ph ^ 1);
          GTRACE(0, gi);
          ++gi;
          uint8_t* st = smem + s * rawBytes;
          if constexpr (!F16) {
            mbar_arrive_expect_tx(&rfull[s], kChunkBytesA + rowsB);
#ifdef FCB_GEMM_LAYOUT_EXP
            tma_load_3d_hint(st, &tmA, &rfull[s], 0, kc * p.m_valid + mt * kTileM, t, pol_a);
            tma_load_3d_hint(st + offB, &tmB, &rfull[s], 0, kc * p.n_valid + nt * nc, t, pol_b);
#else
            tma_load_3d_hint(st, &tmA, &rfull[s], kc * 32, mt * kTileM, t, pol_a);
            tma_load_3d_hint(st + offB, &tmB, &rfull[s], kc * 32, nt * nc, t, pol_b);
#endif
          } else {  // chunks 2kc, 2kc+1 (the second absent at odd k_chunks: converters zero it)
            const bool two = 2 * kc + 1 < p.k_chunks;
            mbar_arrive_expect_tx(&rfull[s], (two ? 2 : 1) * (kChunkBytesA + rowsB));
            tma_load_3d_hint(st, &tmA, &rfull[s], kc * 64, mt * kTileM, t, pol_a);
            tma_load_3d_hint(st + offB, &tmB, &rfull[s], kc * 64, nt * nc, t, pol_b);
            if (two) {
              tma_load_3d_hint(st + kChunkBytesA, &tmA, &rfull[s], kc * 64 + 32, mt * kTileM, t, pol_a);
              tma_load_3d_hint(st + offB + rowsB, &tmB, &rfull[s], kc * 64 + 32, nt * nc, t, pol_b);
            }
          }
          if (++s == RS) { s = 0; ph ^= 1; }
        }
      }
    }
  } else if (warp == 1) {
    // ------------------------------------------------ MMA issuer
    const uint32_t idesc = F16 ? umma_idesc_f16(kTileM, 2 * nc) : umma_idesc_tf32(kTileM, 2 * nc);
    uint32_t g = 0;  // global chunk counter (TMEM A buffer / B buffer = g & 1)
    int local = 0;
    for (int tile = tile_b; tile < tile_e; tile += tile_s, ++local) {
      const int a = local & 1;
      mbar_wait(&tempty[a], ((local >> 1) & 1) ^ 1);
      tc_fence_after();
      const uint32_t d_tmem = tmem_base + a * (2 * nc);
      for (int kc = 0; kc < kc_n; ++kc, ++g) {
        const int b = g & 1;
        mbar_wait(&aready[b], (g >> 1) & 1);
        mbar_wait(&bready[b], (g >> 1) & 1);
        tc_fence_after();
        if (lane == 0) GTRACE(4, g);
        if (lane == 0) {
          const uint32_t a_hi = tmem_base + a_col0 + b * 64;
          const uint32_t a_lo = a_hi + 32;
          const uint32_t b_hi = smem_u32(bbuf0 + b * bbufBytes);
          const uint32_t b_lo = b_hi + 2 * rowsB;
#pragma unroll
          for (int kk = 0; kk < 4; ++kk) {
            const uint64_t dbh = umma_desc_sw128(b_hi + kk * 32);
            const uint64_t dbl = umma_desc_sw128(b_lo + kk * 32);
            if constexpr (F16) {  // K = 16 fp16 = 8 TMEM columns / 32 B per step
              umma_f16_ts(d_tmem, a_hi + kk * 8, dbh, idesc, (kc | kk) ? 1u : 0u);
              umma_f16_ts(d_tmem, a_hi + kk * 8, dbl, idesc, 1u);
              umma_f16_ts(d_tmem, a_lo + kk * 8, dbh, idesc, 1u);
            } else {
              umma_tf32_ts(d_tmem, a_hi + kk * 8, dbh, idesc, (kc | kk) ? 1u : 0u);
              umma_tf32_ts(d_tmem, a_hi + kk * 8, dbl, idesc, 1u);
              umma_tf32_ts(d_tmem, a_lo + kk * 8, dbh, idesc, 1u);
            }
          }
          umma_commit(&atfree[b]);
          umma_commit(&bfree[b]);
          if (kc == kc_n - 1) umma_commit(&tfull[a]);
        }
        __syncwarp();
      }
    }
  } else if (warp >= 4 && warp < 8) {
    // ------------------------------------------------ A converters: raw -> TMEM hi/lo
    const int q = warp & 3;        // TMEM lane quadrant of this warp
    const int m = q * 32 + lane;   // A row
    const uint32_t lane_off = (uint32_t)(q * 32) << 16;
    int s = 0;
    uint32_t ph = 0;
    uint32_t g = 0;
    for (int tile = tile_b; tile < tile_e; tile += tile_s) {
      for (int kc = 0; kc < kc_n; ++kc, ++g) {
        mbar_wait(&rfull[s], ph);
        if (threadIdx.x == 128) GTRACE(1, g);
        const uint8_t* arow = smem + s * rawBytes + (m >> 3) * 1024 + (m & 7) * 128;
        if constexpr (F16) {
          // TMEM column 16c + j holds the scaled pair (K 32c + 2j, 32c + 2j + 1);
          // hi in columns 0-31 of the staging buffer, mid in 32-63
          const float sc = ldexpf(1.f, 14 - ea);
          const bool two = 2 * kc + 1 < p.k_chunks;
          mbar_wait(&atfree[g & 1], ((g >> 1) & 1) ^ 1);  // MMAs of step g-2 done with it
          tc_fence_after();
          const uint32_t ta = tmem_base + lane_off + a_col0 + (g & 1) * 64;
#pragma unroll
          for (int c = 0; c < 2; ++c) {
            uint32_t hi[16], mid[16];
#pragma unroll
            for (int j = 0; j < 8; ++j) {
              float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
              if (c == 0 || two)
                v = *reinterpret_cast<const float4*>(arow + c * kChunkBytesA + ((j ^ (m & 7)) << 4));
              split_f16x2(v.x * sc, v.y * sc, hi[2 * j], mid[2 * j]);
              split_f16x2(v.z * sc, v.w * sc, hi[2 * j + 1], mid[2 * j + 1]);
            }
            if (c == 1) mbar_arrive(&rempty[s]);
            tmem_st_32x32b_x16(ta + 16 * c, hi);
            tmem_st_32x32b_x16(ta + 32 + 16 * c, mid);
          }
          tmem_st_wait();
          tc_fence_before();
          mbar_arrive(&aready[g & 1]);
        } else {
          float x[32], lo[32];
#pragma unroll
          for (int c = 0; c < 8; ++c) {  // 16-B chunk c of the row sits at c ^ (m & 7)
            const float4 v = *reinterpret_cast<const float4*>(arow + ((c ^ (m & 7)) << 4));
            x[4 * c + 0] = v.x;
            x[4 * c + 1] = v.y;
            x[4 * c + 2] = v.z;
            x[4 * c + 3] = v.w;
          }
          mbar_arrive(&rempty[s]);  // raw A read: the TMA may refill the stage
#pragma unroll
          for (int i = 0; i < 32; ++i) lo[i] = tf32_lo(x[i]);
          mbar_wait(&atfree[g & 1], ((g >> 1) & 1) ^ 1);  // MMAs of chunk g-2 done with it
          tc_fence_after();
          const uint32_t ta = tmem_base + lane_off + a_col0 + (g & 1) * 64;
          tmem_st_32x32b_x32(ta, x);
          tmem_st_32x32b_x32(ta + 32, lo);
          tmem_st_wait();
          tc_fence_before();
          mbar_arrive(&aready[g & 1]);
        }
        if (threadIdx.x == 128) GTRACE(2, g);
        if (++s == RS) { s = 0; ph ^= 1; }
      }
    }
  } else if ((warp >= 8 && warp < 12) || (F16 && (warp == 2 || warp == 3))) {
    // ------------------------------------------------ B converters: raw -> re, im, lo, lo-im
    const int ct = threadIdx.x - 256;  // 0..127
    const int nb = nc * 8;             // float4 per raw B tile
    int s = 0;
    uint32_t ph = 0;
    uint32_t g = 0;
    for (int tile = tile_b; tile < tile_e; tile += tile_s) {
      for (int kc = 0; kc < kc_n; ++kc, ++g) {
        mbar_wait(&rfull[s], ph);
        const float4* braw = reinterpret_cast<const float4*>(smem + s * rawBytes + offB);
        if constexpr (F16) {
          // Six warps; warp task = (chunk c, 8-row block b, row half hv).
          // Raw float4 (row n, logical slot j) = K 32c + 4j .. +3 -> fp16
          // bytes 64c + 8j of row n: SW128 slot q = 4c + j/2 stored at
          // q ^ (n % 8), half j % 2.  8-B stores go out per half-warp; a half
          // takes rows r and r + 4, which fill opposite bank halves.
          const int bw = warp >= 8 ? warp - 6 : warp - 2;  // 0..5
          const int hv = bw & 1, b0 = bw >> 1;             // blocks b0, b0+3, b0+6, b0+9
          const int r7 = 2 * hv + (((lane >> 3) & 1) << 2) + (lane >> 4);  // n % 8
          const int j = (lane & 7) ^ r7;
          const int rawoff = r7 * 8 + (lane & 7);  // float4 index within a block
          const int off0 = r7 * 128 + (((j >> 1) ^ r7) << 4) + (j & 1) * 8;
          const int off1 = r7 * 128 + (((4 + (j >> 1)) ^ r7) << 4) + (j & 1) * 8;
          const int nblk = nc >> 3;
          const float sc = ldexpf(1.f, 14 - eb);
          const bool two = 2 * kc + 1 < p.k_chunks;
          float4 v[8];
#pragma unroll
          for (int u = 0; u < 8; ++u) {
            const int c = u >> 2, b = b0 + 3 * (u & 3);
            v[u] = make_float4(0.f, 0.f, 0.f, 0.f);
            if (b < nblk && (c == 0 || two)) v[u] = braw[c * nb + b * 64 + rawoff];
          }
          mbar_arrive(&rempty[s]);
          mbar_wait(&bfree[g & 1], ((g >> 1) & 1) ^ 1);
          uint8_t* bb = bbuf0 + (g & 1) * bbufBytes;
#pragma unroll
          for (int u = 0; u < 8; ++u) {
            const int c = u >> 2, b = b0 + 3 * (u & 3);
            if (b < nblk) {
              const float4 w = v[u];  // (p0, q0, p1, q1)
              const Split p0 = split11(w.x * sc), q0 = split11(w.y * sc);
              const Split p1 = split11(w.z * sc), q1 = split11(w.w * sc);
              uint8_t* o = bb + b * 1024 + (c ? off1 : off0);
              // re rows (p, q); im rows (-q, p)
              *reinterpret_cast<uint2*>(o) = make_uint2(pack_f16x2(p0.hi, q0.hi), pack_f16x2(p1.hi, q1.hi));
              *reinterpret_cast<uint2*>(o + rowsB) =
                  make_uint2(pack_f16x2(-q0.hi, p0.hi), pack_f16x2(-q1.hi, p1.hi));
              *reinterpret_cast<uint2*>(o + 2 * rowsB) =
                  make_uint2(pack_f16x2(p0.mid, q0.mid), pack_f16x2(p1.mid, q1.mid));
              *reinterpret_cast<uint2*>(o + 3 * rowsB) =
                  make_uint2(pack_f16x2(-q0.mid, p0.mid), pack_f16x2(-q1.mid, p1.mid));
            }
          }
        } else {
          float4 v[6];  // nb / 128 <= 6 (nc <= 96)
#pragma unroll
          for (int k = 0; k < 6; ++k)
            if (ct + k * 128 < nb) v[k] = braw[ct + k * 128];
          mbar_arrive(&rempty[s]);
          mbar_wait(&bfree[g & 1], ((g >> 1) & 1) ^ 1);  // MMAs of chunk g-2 done with it
          uint8_t* bb = bbuf0 + (g & 1) * bbufBytes;
          float4* bre = reinterpret_cast<float4*>(bb);
          float4* bim = reinterpret_cast<float4*>(bb + rowsB);
          float4* blr = reinterpret_cast<float4*>(bb + 2 * rowsB);
          float4* bli = reinterpret_cast<float4*>(bb + 3 * rowsB);
#pragma unroll
          for (int k = 0; k < 6; ++k) {
            const int i = ct + k * 128;
            if (i < nb) {
              const float4 w = v[k];  // (p0, q0, p1, q1): re rows are the raw rows
              bre[i] = w;
              bim[i] = make_float4(-w.y, w.x, -w.w, w.z);
              const float4 l = make_float4(tf32_lo(w.x), tf32_lo(w.y), tf32_lo(w.z), tf32_lo(w.w));
              blr[i] = l;
              bli[i] = make_float4(-l.y, l.x, -l.w, l.z);
            }
          }
        }
        fence_proxy_async_smem();
        mbar_arrive(&bready[g & 1]);
        if (threadIdx.x == 256) GTRACE(3, g);
        if (++s == RS) { s = 0; ph ^= 1; }
      }
    }
  } else if (warp >= 12) {
    // ------------------------------------------------ epilogue
    const int q = warp & 3;              // TMEM lane quadrant
    const int half = (warp - 12) >> 2;   // which 16-column blocks
    const int row = q * 32 + lane;
    const float im_sign = p.im_sign;
    const float oscale = F16 ? ldexpf(1.f, ea - 14) * ldexpf(1.f, eb - 14) : 1.f;
    int local = 0;
    for (int tile = tile_b; tile < tile_e; tile += tile_s, ++local) {
      int t, mt, nt;
      decode_tile<RANGES>(tile, p, t, mt, nt);
      const int a = local & 1;
      mbar_wait(&tfull[a], (local >> 1) & 1);
      tc_fence_after();
      const int m = mt * kTileM + row;
      const bool mok = m < p.m_valid;
#if FCB_GEMM_EVL
      const uint64_t pol_out = l2_policy_evict_last();
#endif
      const uint32_t tbase = tmem_base + ((uint32_t)(q * 32) << 16) + a * (2 * nc);
      float2* out = reinterpret_cast<float2*>(p.out) + (long long)t * p.s_t + (m >> p.gm_log2) * p.s_mg +
                    (m & ((1 << p.gm_log2) - 1));
      for (int nb = half * 16; nb < nc; nb += 32) {
        float re[16], im[16];
        tmem_ld_32x32b_x16(tbase + nb, re);
        tmem_ld_32x32b_x16(tbase + nc + nb, im);
        tmem_ld_wait();
        const int n0 = nt * nc + nb;
#pragma unroll
        for (int i = 0; i < 16; ++i) {
          const int n = n0 + i;
          if (mok && n < p.n_valid) {
            const float2 v = F16 ? make_float2(re[i] * oscale, im_sign * oscale * im[i])
                                 : make_float2(re[i], im_sign * im[i]);
#if FCB_GEMM_EVL
            st_global_hint(out + (long long)n * p.s_n, v, pol_out);
#else
            out[(long long)n * p.s_n] = v;
#endif
          }
        }
      }
      tc_fence_before();
      mbar_arrive(&tempty[a]);
      if (threadIdx.x == 384) GTRACE(5, local);  // first epilogue warp
    }
  }

  __syncthreads();
  span_end(p.tspan);
  if (warp == 2) {
    tc_fence_after();
    tmem_dealloc(tmem_base, kTmemCols);
  }
#ifdef FCB_GEMM_TRACE
  if (threadIdx.x == 0 && blockIdx.x < 160) g_cta_time[2][blockIdx.x] = gtimer();
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    const long long t0 = g_gemm_trace[0][0];
    for (int i = 0; i < 30; ++i)
      printf("chunk %2d tma %7lld arawfull %7lld aready %7lld bready %7lld mma %7lld | tile %d epi_done %7lld\n", i,
             g_gemm_trace[0][i] - t0, g_gemm_trace[1][i] - t0, g_gemm_trace[2][i] - t0,
             g_gemm_trace[3][i] - t0, g_gemm_trace[4][i] - t0, i, g_gemm_trace[5][i] - t0);
  }
#endif
}

}  // namespace fcb
