// K1 (r2c) and K4 (c2r) plane transforms, TMA-fed (m in {4, 8, 16, 32, 64}).
//
// Same maths and frequency layout as fft_planes.cuh (see the header there;
// reference: detail::r2c_plane / c2r_plane, fft.hpp:160-203, and the
// bin-major glue of ConvWorkspace, conv_fft.hpp:242-304), re-pipelined for
// the memory system:
//
// * Plane groups (16 planes; 4 at m = 64) stream into a ring of S
//   shared-memory stages with bulk async copies (cp.async.bulk for the
//   real planes, cp.async.bulk.tensor for the product spectrum), counted by
//   transaction bytes on FULL[s].
// * Two consumer groups ping-pong over the CTA's groups.  Each runs both
//   1-D passes of its group: pass 1 reads the stage into registers, the
//   intermediate is written IN PLACE over the stage, pass 2 reads it back.
//   Once its pass-2 operands are in registers the group itself issues the
//   copy of the group S ahead into the freed stage (no producer warp).
// * Column work is packed densely over the src (or crop) non-zero columns
//   of the valid planes (r2c pass 1, c2r pass 2), so small kernels and
//   crops leave warps idle instead of running masked FFTs; full planes
//   (src == m) take a specialised path with constant offsets.
//
// Earlier cuts loaded planes straight into registers (one group's loads in
// flight per CTA; ncu: 27-41% DRAM) or split the passes over separate warp
// roles (the busier role had too few warps to hide FFT latency).
#pragma once
#include <cuda.h>

#include <cstdint>

#include "fft_planes.cuh"
#include "ptx.cuh"

namespace fcb {

__host__ __device__ constexpr int cmax_i(int a, int b) { return a > b ? a : b; }
__host__ __device__ constexpr int cmin_i(int a, int b) { return a < b ? a : b; }
__host__ __device__ constexpr int round_up_i(int a, int b) { return (a + b - 1) / b * b; }
__host__ __device__ constexpr int ceil32_i(int a) { return (a + 31) / 32 * 32; }

constexpr int kTmaSmemBudget = 220 * 1024;
// Development switch for bottleneck experiments (default 0 = real kernel):
// 1 skips the FFT arithmetic, 2 skips the HBM stores, 3 skips the HBM loads.
#ifndef FCB_XFORM_EXP
#define FCB_XFORM_EXP 0
#endif
constexpr int kConsumers = 2;

// FCB_XFORM_TRACE: per-group clock64 timeline of CTA 0 (development builds)
#ifdef FCB_XFORM_TRACE
__device__ long long g_xform_trace[6][64];
#define XTRACE(ev, idx)                                                     \
  do {                                                                      \
    if (blockIdx.x == 0 && (idx) < 64) g_xform_trace[ev][idx] = clock64();  \
  } while (0)
#else
#define XTRACE(ev, idx) \
  do {                  \
  } while (0)
#endif

// Output-tile stores the copy engine keeps in flight before it recycles the
// oldest stage (the refill lags by as many groups): one with a deep ring,
// none with three stages (measured: K1 at P 41 -> 39 us with one in flight;
// the 3-stage m = 64 kernels lose ~13% with one)
__host__ __device__ constexpr int stores_inflight(int stages) { return stages >= 6 ? 1 : 0; }

#ifndef FCB_R2C_G
#define FCB_R2C_G 8  // planes per K1 group at m = 32
#endif
#ifndef FCB_R2C_G_BIG
#define FCB_R2C_G_BIG 4  // planes per K1 group at m = 64
#endif
#ifndef FCB_C2R_G_BIG
#define FCB_C2R_G_BIG 4  // planes per K4 group at m = 64
#endif
#ifndef FCB_BIG_NPIPE
#define FCB_BIG_NPIPE 0  // 1: two pass pipelines at m = 64 when the stage count allows
#endif
#ifndef FCB_R2C_G_SMALL
#define FCB_R2C_G_SMALL 16  // planes per K1 group at m <= 16 (full 128-B lines; n=16 sweep step 122 -> 111 us vs 8)
#endif

// Independent pass-1/pass-2 pipelines: the largest of 4, 2, 1 that divides
// the stage count (each stage then belongs to one pipeline) and keeps the
// CTA within 1024 threads.
__host__ __device__ constexpr int npipe_for(int stages, int fixed, int per_pipe) {
  return (stages % 4 == 0 && fixed + 4 * per_pipe <= 1024) ? 4
         : (stages % 2 == 0 && fixed + 2 * per_pipe <= 1024) ? 2 : 1;
}

#ifndef FCB_C2R_G
#define FCB_C2R_G 16  // planes per K4 group at m <= 32
#endif

// smallest box count >= bins/256 that divides the bins (TMA box dims <= 256)
__host__ __device__ constexpr int nbox_for(int bins, int n = 0) {
  return n == 0 ? nbox_for(bins, (bins + 255) / 256) : (bins % n == 0 ? n : nbox_for(bins, n + 1));
}  // consumer groups per CTA (named barriers 1, 2)

// ---------------------------------------------------------------- K1: r2c
//
// Warp roles (stores never stall a compute warp: the measured bottleneck of
// the earlier cuts was warps issuing the 93.5 MB of scattered spectrum
// stores between FFTs):
//   warp 0         copy engine: bulk-loads plane groups into the stage ring
//                  and drains finished stages to HBM with TMA tensor stores
//   pass-1 warps   FULL[s] -> real column FFTs (dense (plane, column-pair)
//                  items) -> intermediate in place -> MID[s]
//   pass-2 warps   MID[s] -> complex row FFTs -> the spectrum rows written
//                  back into the same stage in the output tile layout
//                  [bin][plane] -> OUT[s]; the copy engine stores the tile
//                  and refills the stage once the store has read it
template <int M>
struct TR2C {
  static constexpr bool BIG = (M == 64);
  // planes (K indices) per group: 8 (64-B spectrum segments; a 16-plane
  // group made 72-KB stages, only 3 of which fit, too shallow to hide the
  // ~4.5k-cycle load latency under load), 4 at m = 64
  static constexpr int G = BIG ? FCB_R2C_G_BIG : (M <= 16 ? FCB_R2C_G_SMALL : FCB_R2C_G);
  static constexpr int PC = M / 2 + 1;
  static constexpr int CP = M + 1;        // intermediate row stride (float2)
  static constexpr int BINS = M * PC;
  // raw plane incl. 16-B alignment slack, in float2
  static constexpr int RAWF2 = (M * M * 4 + 16 + 7) / 8;
  static constexpr int PS0 = cmax_i(PC * CP, RAWF2 + 1);
  // Plane stride (float2).  m <= 32: odd, so the 16 planes a half-warp
  // reads in pass 2 hit distinct banks.  m = 64: 4 (mod 16), so the
  // (plane, u) pairs of a warp are spread over the banks.
  static constexpr int PS = BIG ? PS0 + ((4 - PS0 % 16) + 16) % 16 : (PS0 | 1);
  static constexpr int STAGE = round_up_i(cmax_i(G * PS * 8 + 8, BINS * G * 8), 128);
  static constexpr int S = cmin_i(8, kTmaSmemBudget / STAGE);
  static constexpr int P1 = BIG ? G * M : G * (M / 2);  // column (pair) items
  static constexpr int P2 = BIG ? G * PC * 2 : G * PC;  // row items
  static constexpr int P1W = ceil32_i(P1), P2W = ceil32_i(P2);
  // independent pass-1/pass-2 pipelines on alternating groups (an even
  // stage count keeps every stage in one parity class, so no mbarrier
  // phase is ever shared between the pipelines)
  static constexpr int NPIPE = (BIG && !FCB_BIG_NPIPE) ? 1 : npipe_for(S, 32, P1W + P2W);
  static constexpr int THREADS = 32 + NPIPE * (P1W + P2W);
  static constexpr int SMEM = S * STAGE + 3 * S * 8 + 128;
  // output tile stores: NBOX boxes of BT bins x G planes
  static constexpr int NBOX = nbox_for(BINS);
  static constexpr int BT = BINS / NBOX;
  static_assert(BT * NBOX == BINS && BT <= 256, "output box must tile the bins");
};

// byte offset of plane jl's raw copy inside a stage (16-B aligned, at or
// just after the plane's intermediate base jl * PS * 8)
__device__ __forceinline__ int r2c_raw_off(int jl, int ps) { return (jl * ps * 8 + 15) & ~15; }

struct GroupRef {
  const R2CParams* p;
  int which, r, j0;
};

template <int G>
__device__ __forceinline__ GroupRef r2c_group(const R2CPair& P, int ngA, int g) {
  const int which = g >= ngA;
  const R2CParams& p = P.op[which];
  const int gl = g - which * ngA, ngj = (p.kpad + G - 1) / G;
  const int r = gl / ngj;
  return {&p, which, r, (gl - r * ngj) * G};
}

// max(|Re|, |Im|) over N complex values (FMNMX with |.| operands; NaNs are
// skipped, they still propagate through the GEMM itself).
template <int N>
__device__ __forceinline__ float absmax_f(const float2 (&v)[N]) {
  float m = 0.f;
#pragma unroll
  for (int i = 0; i < N; ++i) m = fmaxf(m, fmaxf(fabsf(v[i].x), fabsf(v[i].y)));
  return m;
}

// Stores one spectrum row into the output tile (stride in float2).
template <int N>
__device__ __forceinline__ void tile_row(float2* o, int stride, const float2 (&w)[N], float csign) {
#pragma unroll
  for (int v = 0; v < N; ++v) o[v * stride] = make_float2(w[v].x, csign * w[v].y);
}

// grid = persistent (<= groups), block = THREADS, smem = SMEM.
// tmo[i]: 3-D fp32 map over operand i's spectrum F[t][R][2*kpad], box
// {2G floats, 1 row, BT bins}.
template <int M>
__global__ void __launch_bounds__(TR2C<M>::THREADS, 1)
    r2c_tma_kernel(const __grid_constant__ R2CPair P, const __grid_constant__ CUtensorMap tmo0,
                   const __grid_constant__ CUtensorMap tmo1) {
  using T = TR2C<M>;
  constexpr int G = T::G, PC = T::PC, CP = T::CP, PS = T::PS, S = T::S;
  extern __shared__ __align__(128) uint8_t smem[];
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + S * T::STAGE);  // loads landed
  uint64_t* mid = full + S;                                           // intermediate written
  uint64_t* outb = mid + S;                                           // output tile written
  const int ngA = P.op[0].R * ((P.op[0].kpad + G - 1) / G);
  const int ngroups = ngA + (P.n > 1 ? P.op[1].R * ((P.op[1].kpad + G - 1) / G) : 0);
  if (threadIdx.x == 0) {
    for (int s = 0; s < S; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&mid[s], T::P1W);
      mbar_init(&outb[s], T::P2W);
    }
    fence_barrier_init();
    tma_prefetch_desc(&tmo0);
    tma_prefetch_desc(&tmo1);
  }
  __syncthreads();
  pdl_wait();
  span_begin(P.tspan);
  pdl_trigger();

  if (threadIdx.x < 32) {
    // ------------------------------------------------ copy engine
    if (threadIdx.x == 0) {
      const uint64_t pol = l2_policy_evict_first();
      auto issue_load = [&](int i) {
        const int g = blockIdx.x + i * gridDim.x;
        if (g >= ngroups) return;
        XTRACE(0, i);
        const int s = i % S;
        const GroupRef q = r2c_group<G>(P, ngA, g);
        const R2CParams& p = *q.p;
        const int jv = FCB_XFORM_EXP == 3 ? 0 : min(G, p.J - q.j0);  // <= 0: pure K padding
        const uint32_t pb = (uint32_t)(p.src * p.src) * 4u;
        const float* base = p.in + (long long)q.r * p.in_sr + (long long)q.j0 * p.in_sj;
        uint32_t total = 0;
        for (int jl = 0; jl < jv; ++jl) {
          const uintptr_t a = reinterpret_cast<uintptr_t>(base + (long long)jl * p.in_sj);
          total += ((uint32_t)(a & 15) + pb + 15) & ~15u;
        }
        mbar_arrive_expect_tx(&full[s], total);
        uint8_t* st = smem + s * T::STAGE;
        for (int jl = 0; jl < jv; ++jl) {
          // the plane's enclosing 16-B aligned range (planes need not be aligned)
          const uintptr_t a = reinterpret_cast<uintptr_t>(base + (long long)jl * p.in_sj);
          const uint32_t sz = ((uint32_t)(a & 15) + pb + 15) & ~15u;
          bulk_load(st + r2c_raw_off(jl, PS), reinterpret_cast<const void*>(a & ~uintptr_t(15)), sz,
                    &full[s], pol);
        }
      };
#pragma unroll 1
      for (int i = 0; i < S; ++i) issue_load(i);
#pragma unroll 1
      for (int i = 0;; ++i) {
        const int g = blockIdx.x + i * gridDim.x;
        if (g >= ngroups) break;
        const int s = i % S;
        mbar_wait(&outb[s], (i / S) & 1);
        XTRACE(4, i);
        const GroupRef q = r2c_group<G>(P, ngA, g);
        const CUtensorMap* tm = q.which ? &tmo1 : &tmo0;
        const uint8_t* st = smem + s * T::STAGE;
        if (FCB_XFORM_EXP != 2)
          for (int k = 0; k < T::NBOX; ++k)
            tma_store_3d(tm, st + k * T::BT * G * 8, 2 * q.j0, q.r, k * T::BT);
        bulk_commit_group();
        constexpr int D = stores_inflight(S);
        if (i >= D) {  // the store of group i-D has read its tile: refill its stage
          bulk_wait_group_read<D>();
          XTRACE(5, i);
          issue_load(i - D + S);
        }
      }
      bulk_wait_group<0>();  // spectra written before the grid completes
    }
  } else if (threadIdx.x < 32 + T::NPIPE * T::P1W) {
    // ------------------------------------------------ pass 1: real column FFTs
    const int pipe = (threadIdx.x - 32) / T::P1W;
    const int t = threadIdx.x - 32 - pipe * T::P1W;
    const int bar = 1 + pipe;
#pragma unroll 1
    for (int i = pipe;; i += T::NPIPE) {
      const int g = blockIdx.x + i * gridDim.x;
      if (g >= ngroups) break;
      const int s = i % S;
      const GroupRef q = r2c_group<G>(P, ngA, g);
      const R2CParams& p = *q.p;
      const int src = p.src;
      const int jv = max(0, min(G, p.J - q.j0));
      uint8_t* st = smem + s * T::STAGE;
      mbar_wait(&full[s], (i / S) & 1);
      if (t == 0) XTRACE(1, i);
      // (plane, column[-pair]) items packed densely over the valid planes and
      // their src non-zero columns.  Each specialisation keeps its own
      // register arrays (a branch writing one array from two paths demotes
      // it to local memory).
      if constexpr (!T::BIG) {
        const int H = (src + 1) >> 1;  // column pairs (c, c + H): one complex FFT
        const bool act = t < jv * H;
        const int jl = act ? t / H : 0, c = t - jl * H;
        const bool hb = c + H < src;
        const float* pin = p.in + (long long)q.r * p.in_sr + (long long)(q.j0 + jl) * p.in_sj;
        const float* raw = reinterpret_cast<const float*>(st + r2c_raw_off(jl, PS)) +
                           ((reinterpret_cast<uintptr_t>(pin) & 15) >> 2) + c;
        float2* dst = reinterpret_cast<float2*>(st + jl * PS * 8) + c;
        // NZ: rows >= NZ are zero (src <= NZ): pruned column FFT
        auto pass1 = [&](auto full_tag, auto nz_tag) {
          constexpr bool FULL = decltype(full_tag)::value;
          constexpr int NZ = decltype(nz_tag)::value;
          float2 z[M];
#pragma unroll
          for (int row = 0; row < M; ++row) {
            if constexpr (FULL) {  // full plane: constant offsets, no predicates
              z[row].x = act ? raw[row * M] : 0.f;
              z[row].y = act ? raw[row * M + M / 2] : 0.f;
            } else {
              const bool ok = act && row < NZ && row < src;
              z[row].x = ok ? raw[0] : 0.f;
              z[row].y = (ok && hb) ? raw[H] : 0.f;
              raw += src;
            }
          }
          named_bar_sync(bar, T::P1W);  // every raw plane is read: overwrite in place
          if (act) {
            if (FCB_XFORM_EXP != 1) fft_reg_nz<M, NZ, false>(z);
            static_for<0, PC>([&](auto U) {
              constexpr int u = decltype(U)::value;
              const float2 zu = z[u];
              const float2 zc = cconj(z[(M - u) % M]);
              dst[u * CP] = make_float2(0.5f * (zu.x + zc.x), 0.5f * (zu.y + zc.y));
              if (FULL || hb) {
                const float2 d = csub(zu, zc);
                dst[u * CP + (FULL ? M / 2 : H)] = make_float2(0.5f * d.y, -0.5f * d.x);  // (zu - zc) / (2i)
              }
            });
          }
        };
        using FT = std::true_type;
        using FF = std::false_type;
        if (src == M) pass1(FT{}, std::integral_constant<int, M>{});
        else if (M >= 16 && src <= M / 4) pass1(FF{}, std::integral_constant<int, (M >= 16 ? M / 4 : M)>{});
        else pass1(FF{}, std::integral_constant<int, M>{});
      } else {
        // m = 64: one real column per thread (half-length complex FFT)
        const bool act = t < jv * src;
        const int jl = act ? t / src : 0, c = t - jl * src;
        const float* pin = p.in + (long long)q.r * p.in_sr + (long long)(q.j0 + jl) * p.in_sj;
        const float* raw = reinterpret_cast<const float*>(st + r2c_raw_off(jl, PS)) +
                           ((reinterpret_cast<uintptr_t>(pin) & 15) >> 2) + c;
        float2* dst = reinterpret_cast<float2*>(st + jl * PS * 8) + c;
        auto pass1 = [&](auto full_tag) {
          constexpr bool FULL = decltype(full_tag)::value;
          float2 z[M / 2];  // (even, odd) rows packed for the half-length FFT
#pragma unroll
          for (int i2 = 0; i2 < M / 2; ++i2) {
            if constexpr (FULL) {
              z[i2].x = act ? raw[(2 * i2) * M] : 0.f;
              z[i2].y = act ? raw[(2 * i2 + 1) * M] : 0.f;
            } else {
              z[i2].x = (act && 2 * i2 < src) ? raw[(2 * i2) * src] : 0.f;
              z[i2].y = (act && 2 * i2 + 1 < src) ? raw[(2 * i2 + 1) * src] : 0.f;
            }
          }
          named_bar_sync(bar, T::P1W);  // a plane spans two warps
          if (act) rfft_packed_emit<M>(z, [&](int u, float2 v) { dst[u * CP] = v; });
        };
        if (src == M) pass1(std::true_type{});
        else pass1(std::false_type{});
      }
      mbar_arrive(&mid[s]);
      if (t == 0) XTRACE(2, i);
    }
  } else {
    // ------------------------------------------------ pass 2: complex row FFTs -> output tile
    const int pipe = (threadIdx.x - 32 - T::NPIPE * T::P1W) / T::P2W;
    const int t = threadIdx.x - 32 - T::NPIPE * T::P1W - pipe * T::P2W;
    const int bar = 1 + T::NPIPE + pipe;
    const bool act = t < T::P2;
#pragma unroll 1
    for (int i = pipe;; i += T::NPIPE) {
      const int g = blockIdx.x + i * gridDim.x;
      if (g >= ngroups) break;
      const int s = i % S;
      const GroupRef q = r2c_group<G>(P, ngA, g);
      const R2CParams& p = *q.p;
      const int src = p.src;
      const int jv = max(0, min(G, p.J - q.j0));
      const float csign = p.conj ? -1.f : 1.f;
      float amx = 0.f;  // max |component| of this thread's outputs (the group's row)
      uint8_t* st = smem + s * T::STAGE;
      float2* tile = reinterpret_cast<float2*>(st);  // [bin][G planes]
      mbar_wait(&mid[s], (i / S) & 1);
      if constexpr (!T::BIG) {
        const int jl = t % G, u = t / G;
        const bool valid = act && jl < jv;
        const float2* row = reinterpret_cast<const float2*>(st + jl * PS * 8) + u * CP;
        auto pass2 = [&](auto full_tag, auto nz_tag) {
          constexpr bool FULL = decltype(full_tag)::value;
          constexpr int NZ = decltype(nz_tag)::value;  // columns >= NZ are zero
          float2 w[M];
#pragma unroll
          for (int cc = 0; cc < M; ++cc)
            w[cc] = (valid && cc < NZ && (FULL || cc < src)) ? row[cc] : make_float2(0.f, 0.f);
          named_bar_sync(bar, T::P2W);  // the intermediate is read: reuse the stage as the tile
          if (act) {  // invalid (K padding) planes store exact zeros
            if (FCB_XFORM_EXP != 1) fft_reg_nz<M, NZ, false>(w);
            tile_row<M>(tile + (u * M) * G + jl, G, w, csign);
            amx = fmaxf(amx, absmax_f<M>(w));
          }
        };
        using FT = std::true_type;
        using FF = std::false_type;
        if (src == M) pass2(FT{}, std::integral_constant<int, M>{});
        else if (M >= 16 && src <= M / 4) pass2(FF{}, std::integral_constant<int, (M >= 16 ? M / 4 : M)>{});
        else pass2(FF{}, std::integral_constant<int, M>{});
      } else {
        // (plane, u, half): one decimation-in-frequency stage splits the
        // 64-point row FFT into two 32-point halves, outputs v = 2k + h
        const int jl = t % G, h = (t / G) & 1, u = t / (2 * G);
        const bool valid = act && jl < jv;
        const float2* row = reinterpret_cast<const float2*>(st + jl * PS * 8) + u * CP;
        float2 z[32];
        static_for<0, 32>([&](auto Cc) {
          constexpr int cc = decltype(Cc)::value;
          const float2 a0 = (valid && cc < src) ? row[cc] : make_float2(0.f, 0.f);
          const float2 a1 = (valid && cc + 32 < src) ? row[cc + 32] : make_float2(0.f, 0.f);
          const float2 d = csub(a0, a1);
          if constexpr (cc == 0) z[cc] = h ? d : cadd(a0, a1);
          else z[cc] = h ? cmul(d, tw128c<false, cc * 2>()) : cadd(a0, a1);
        });
        named_bar_sync(bar, T::P2W);
        if (act) {
          if (FCB_XFORM_EXP != 1) fft_reg<32, false>(z);
          tile_row<32>(tile + (u * M + h) * G + jl, 2 * G, z, csign);
          amx = fmaxf(amx, absmax_f<32>(z));
        }
      }
      fence_proxy_async_smem();  // the tile is read by the TMA store (async proxy)
      mbar_arrive(&outb[s]);
      if (t == 0) XTRACE(3, i);
      if (p.amax) {  // row maximum; non-negative floats order like their bit patterns
        const uint32_t v = __reduce_max_sync(0xffffffffu, __float_as_uint(amx));
        if ((threadIdx.x & 31) == 0) atomicMax(p.amax + q.r, ((unsigned long long)p.epoch << 32) | v);
      }
    }
  }
  if (P.tspan) {  // uniform: the whole CTA is done
    __syncthreads();
    span_end(P.tspan);
  }
#ifdef FCB_XFORM_TRACE
  __syncthreads();
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    const long long t0 = g_xform_trace[0][0];
    for (int i = 0; i < 12; ++i)
      printf("grp %2d load %7lld full %7lld p1done %7lld p2done %7lld store %7lld refill %7lld\n", i,
             g_xform_trace[0][i] - t0, g_xform_trace[1][i] - t0, g_xform_trace[2][i] - t0,
             g_xform_trace[3][i] - t0, g_xform_trace[4][i] - t0, g_xform_trace[5][i] - t0);
  }
#endif
}

// ---------------------------------------------------------------- K4: c2r
//
// Warp roles, as for K1:
//   warp 0         copy engine: TMA tensor loads of the product spectrum
//                  (one box of m bins x G planes per u row) into the stage
//                  ring; refills a stage once pass 2 has read it
//   pass-1 warps   FULL[s] -> inverse row FFTs over v, cropped columns
//                  written in place -> MID[s]
//   pass-2 warps   MID[s] -> Hermitian column c2r (dense (plane,
//                  column-pair) items) -> the cropped planes written into
//                  the same stage -> OUT[s]; the copy engine bulk-stores them
//                  and refills the stage once the stores have read it.
//                  Planes that are not 16-B aligned (odd crops) are stored
//                  directly from registers instead (EMPTY[s] after the reads).
// K4 output-tile plane stride in floats: >= crop^2, a multiple of 4 (16-B
// aligned bulk-store sources) with an odd quotient.
__host__ __device__ constexpr int tile_plane_stride(int crop) {
  return ((crop * crop + 3) / 4 % 2 == 0) ? ((crop * crop + 3) / 4 + 1) * 4 : (crop * crop + 3) / 4 * 4;
}

// Stores jv staged planes (tile plane stride pst floats, pe floats each)
// to out + jl * out_sj with consecutive threads on consecutive floats of a
// plane; accum adds into the output.
__device__ __forceinline__ void c2r_store_tile(const float* tile, int pst, int jv, int pe, float* out,
                                               long long out_sj, int accum, int t, int nthreads) {
  // separate loops: with `v + (accum ? *d : 0)` the compiler may hoist the
  // load of *d (the store proves it valid), putting an HBM round trip in
  // front of every store (measured: accGrad's K4 pass 2 took 4-6k cycles)
  if (accum) {
    for (int e = t; e < jv * pe; e += nthreads) {
      const int jl = e / pe, rem = e - jl * pe;
      float* d = out + jl * out_sj + rem;
      *d += tile[jl * pst + rem];
    }
  } else {
    for (int e = t; e < jv * pe; e += nthreads) {
      const int jl = e / pe, rem = e - jl * pe;
      out[jl * out_sj + rem] = tile[jl * pst + rem];
    }
  }
}

template <int M>
struct TC2R {
  static constexpr bool BIG = (M == 64);
  static constexpr int G = BIG ? FCB_C2R_G_BIG : FCB_C2R_G;
  static constexpr int PC = M / 2 + 1;
  static constexpr int CP = M + 1;  // intermediate row stride (float2), >= crop
  static constexpr int PS = BIG ? PC * CP + ((4 - (PC * CP) % 16) + 16) % 16 : ((PC * CP) | 1);
  // raw u-row stride (float2): one TMA box of M bins x G planes per u row
  // (tensor-copy destinations must be 128-B aligned, so no bank padding)
  static constexpr int RS = M * G;
  static constexpr int RAW = PC * RS * 8;
  static constexpr int INTER = G * PS * 8;
  static constexpr int STAGE = round_up_i(cmax_i(RAW, INTER), 128);
  static constexpr int S = cmin_i(8, kTmaSmemBudget / STAGE);
  static constexpr int P1 = BIG ? G * PC * 2 : G * PC;  // (plane, u[, half]) row items
  static constexpr int P2 = BIG ? G * M : G * (M / 2);  // column (pair) items
  static constexpr int P1W = ceil32_i(P1), P2W = ceil32_i(P2);
  static constexpr int NPIPE = ((!BIG || FCB_BIG_NPIPE) && S % 2 == 0) ? 2 : 1;
  static constexpr int THREADS = 32 + NPIPE * (P1W + P2W);
  static constexpr int TW = S * STAGE + 4 * S * 8;  // inverse twiddle table e^(+2 pi i k / M), M float2
  static constexpr int SMEM = TW + M * 8 + 128;
  // small crops (weight gradients, crop <= M/4): pass 2 evaluates each
  // output as a direct Hermitian DFT over u, one thread per (plane, column),
  // instead of one FFT per column (pair) producing mostly discarded rows
  static constexpr uint32_t BOX_BYTES = 2 * G * 4 * M;  // one u row
  static_assert(G * tile_plane_stride(M) * 4 <= STAGE, "a staged output tile must fit a stage");
};

// tm: 3-D fp32 map over the product spectrum P[t][r][2*ld] with box
// {2G floats, 1 row, M bins}.  grid = persistent, groups g = r*ceil(J/G)+jg.
template <int M>
__global__ void __launch_bounds__(TC2R<M>::THREADS, 1)
    c2r_tma_kernel(const __grid_constant__ CUtensorMap tm, const C2RParams p) {
  using T = TC2R<M>;
  constexpr int G = T::G, PC = T::PC, CP = T::CP, PS = T::PS, RS = T::RS, S = T::S;
  extern __shared__ __align__(128) uint8_t smem[];
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + S * T::STAGE);
  uint64_t* mid = full + S;
  uint64_t* empty = mid + S;  // pass 2 read the stage (direct-store mode)
  uint64_t* outb = empty + S;  // pass 2 wrote the output tile (bulk mode)
  const int ngj = (p.J + G - 1) / G;
  const int ngroups = p.R * ngj;
  const int crop = p.crop;
  const bool dft2 = crop <= M / 4 && G * crop <= T::P2W;
  // output-tile plane stride (floats): 16-B aligned for the bulk stores and
  // an odd number of 16-B units, so the plane-fastest pass-2 lanes spread
  // over the banks (a 32 x 32 crop at stride 1024 put 16 planes on one bank)
  const int pst = tile_plane_stride(crop);
  if (threadIdx.x == 0) {
    for (int s = 0; s < S; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&mid[s], T::P1W);
      mbar_init(&empty[s], T::P2W);
      mbar_init(&outb[s], T::P2W);
    }
    fence_barrier_init();
    tma_prefetch_desc(&tm);
  }
  __syncthreads();
  pdl_wait();
  span_begin(p.tspan);
  pdl_trigger();

  if (threadIdx.x < 32) {
    // ------------------------------------------------ copy engine
    if (threadIdx.x == 0) {
      const uint64_t pol = l2_policy_evict_first();
      const uint32_t plane_bytes = (uint32_t)(crop * crop) * 4u;
      const uint32_t tile_stride = (uint32_t)pst * 4u;
      auto issue_load = [&](int i) {
        const int g = blockIdx.x + i * gridDim.x;
        if (g >= ngroups) return;
        const int s = i % S;
        const int r = g / ngj, j0 = (g - r * ngj) * G;
        XTRACE(0, i);
        mbar_arrive_expect_tx(&full[s], PC * T::BOX_BYTES);
        uint8_t* st = smem + s * T::STAGE;
        if (p.gm) {  // group-major product: the group is one contiguous block
          const int ngj_all = p.J_all ? (p.J_all + G - 1) / G : ngj;
          const float* src = p.in + (long long)(r * ngj_all + (p.jbase + j0) / G) * (PC * T::BOX_BYTES / 4);
          bulk_load(st, src, PC * T::BOX_BYTES, &full[s], pol);
        } else {
          for (int u = 0; u < PC; ++u)
            tma_load_3d_hint(st + u * RS * 8, &tm, &full[s], 2 * (p.jbase + j0), r, u * M, pol);
        }
      };
#pragma unroll 1
      for (int i = 0; i < S; ++i) issue_load(i);
#pragma unroll 1
      for (int i = 0;; ++i) {
        const int g = blockIdx.x + i * gridDim.x;
        if (g >= ngroups) break;
        const int s = i % S;
        if (p.bulk) {
          mbar_wait(&outb[s], (i / S) & 1);
          const int r = g / ngj, j0 = (g - r * ngj) * G;
          const int jv = min(G, p.J - j0);
          const uint8_t* tile = smem + s * T::STAGE;
          if (FCB_XFORM_EXP != 2)
            for (int jl = 0; jl < jv; ++jl)
              bulk_store(p.out + (long long)r * p.out_sr + (long long)(j0 + jl) * p.out_sj,
                         tile + jl * tile_stride, plane_bytes);
          bulk_commit_group();
          constexpr int D = stores_inflight(S);
          if (i >= D) {  // group i-D's stores have read their tile: refill its stage
            bulk_wait_group_read<D>();
            issue_load(i - D + S);
          }
        } else {
          mbar_wait(&empty[s], (i / S) & 1);
          issue_load(i + S);
        }
      }
      if (p.bulk) bulk_wait_group<0>();
    }
  } else if (threadIdx.x < 32 + T::NPIPE * T::P1W) {
    // ------------------------------------------------ pass 1: inverse row FFTs over v
    const int pipe = (threadIdx.x - 32) / T::P1W;
    const int t = threadIdx.x - 32 - pipe * T::P1W;
    const int bar = 1 + pipe;
    const bool act1 = t < T::P1;
#pragma unroll 1
    for (int i = pipe;; i += T::NPIPE) {
      const int g = blockIdx.x + i * gridDim.x;
      if (g >= ngroups) break;
      const int s = i % S;
      const int r = g / ngj, j0 = (g - r * ngj) * G;
      const int jv = min(G, p.J - j0);
      uint8_t* st = smem + s * T::STAGE;
      const float2* raw = reinterpret_cast<const float2*>(st);
      float2* inter = reinterpret_cast<float2*>(st);
      (void)r;
      mbar_wait(&full[s], (i / S) & 1);
      if (t == 0) XTRACE(1, i);
      if constexpr (!T::BIG) {
        const int jl = t % G, u = t / G;
        const float2* src = raw + u * RS + jl;
        float2 z[M];
#pragma unroll
        for (int v = 0; v < M; ++v) z[v] = act1 ? src[v * G] : make_float2(0.f, 0.f);
        named_bar_sync(bar, T::P1W);  // the whole stage is read: overwrite in place
        if (act1 && jl < jv) {
          if (FCB_XFORM_EXP != 1) fft_reg<M, true>(z);
          float2* dst = inter + jl * PS + u * CP;
#pragma unroll
          for (int c = 0; c < M; ++c)
            if (c < crop) dst[c] = z[c];
        }
      } else {
        const int jl = t % G, h = (t / G) & 1, u = t / (2 * G);
        const float2* src = raw + u * RS + jl;
        float2 z[32];
        static_for<0, 32>([&](auto Vv) {
          constexpr int v = decltype(Vv)::value;
          const float2 a0 = act1 ? src[v * G] : make_float2(0.f, 0.f);
          const float2 a1 = act1 ? src[(v + 32) * G] : make_float2(0.f, 0.f);
          const float2 d = csub(a0, a1);
          if constexpr (v == 0) z[v] = h ? d : cadd(a0, a1);
          else z[v] = h ? cmul(d, tw128c<true, v * 2>()) : cadd(a0, a1);
        });
        named_bar_sync(bar, T::P1W);
        if (act1 && jl < jv) {
          if (FCB_XFORM_EXP != 1) fft_reg<32, true>(z);
          float2* dst = inter + jl * PS + u * CP + h;
#pragma unroll
          for (int k = 0; k < 32; ++k)
            if (2 * k + h < crop) dst[2 * k] = z[k];
        }
      }
      mbar_arrive(&mid[s]);
      if (t == 0) XTRACE(2, i);
    }
  } else {
    // ------------------------------------------------ pass 2: Hermitian c2r over u -> HBM
    const int pipe = (threadIdx.x - 32 - T::NPIPE * T::P1W) / T::P2W;
    const int t = threadIdx.x - 32 - T::NPIPE * T::P1W - pipe * T::P2W;
    const float scale = p.scale;
#pragma unroll 1
    for (int i = pipe;; i += T::NPIPE) {
      const int g = blockIdx.x + i * gridDim.x;
      if (g >= ngroups) break;
      const int s = i % S;
      const int r = g / ngj, j0 = (g - r * ngj) * G;
      const int jv = min(G, p.J - j0);
      const float2* inter = reinterpret_cast<const float2*>(smem + s * T::STAGE);
      mbar_wait(&mid[s], (i / S) & 1);
      if (dft2) {
        // x[y] = Re Z[0] + (-1)^y Re Z[M/2] + 2 sum_{0<u<M/2} Re(Z[u] e^(2 pi i u y / M))
        // (the imaginary parts of Z[0] and Z[M/2] are dropped, as c2r does).
        // One thread per (plane, output column c), plane fastest (a half-warp
        // reads one column of G planes: distinct banks at the odd plane
        // stride): the column's M/2 + 1 values are loaded once and every row
        // y < crop <= M/4 is a direct Hermitian DFT with the twiddles
        // e^(2 pi i u y / M) as instruction immediates.  (Per-(plane, y, c)
        // items re-read the column and a twiddle table for each y: ~3
        // shared-memory wavefronts per term bounded accGrad's K4, ~3.5k
        // cycles per 16-plane group.)
        constexpr int YMAX = M / 4;
        const int jl = t % G, c = t / G;
        const bool act = jl < jv && c < crop;
        float res[YMAX];
        if (act) {
          const float2* col = inter + jl * PS + c;
          float2 z[M / 2 + 1];
          static_for<0, M / 2 + 1>([&](auto U) { z[decltype(U)::value] = col[decltype(U)::value * CP]; });
          static_for<0, YMAX>([&](auto Y) {
            constexpr int y = decltype(Y)::value;
            if (y < crop) {
              float acc = 0.f;
              static_for<1, M / 2>([&](auto U) {
                constexpr int u = decltype(U)::value;
                const float2 w = tw128c<true, (u * y * (128 / M)) % 128>();
                acc = fmaf(z[u].x, w.x, fmaf(-z[u].y, w.y, acc));
              });
              const float e = z[0].x + ((y & 1) ? -z[M / 2].x : z[M / 2].x);
              res[y] = c2r_out((e + 2.f * acc) * scale, p.relu);
            }
          });
        }
        named_bar_sync(1 + T::NPIPE + pipe, T::P2W);  // stage read: reuse it as the output tile
        float* tile = reinterpret_cast<float*>(smem + s * T::STAGE);
        if (act)
          static_for<0, YMAX>([&](auto Y) {
            constexpr int y = decltype(Y)::value;
            if (y < crop) tile[jl * pst + y * crop + c] = res[y];
          });
        if (p.bulk) {
          fence_proxy_async_smem();
          mbar_arrive(&outb[s]);
        } else {
          // coalesced stores of the jv cropped planes (each crop*crop floats
          // contiguous in HBM), accumulating when asked
          named_bar_sync(1 + T::NPIPE + pipe, T::P2W);
          c2r_store_tile(tile, pst, jv, crop * crop, p.out + (long long)r * p.out_sr + (long long)j0 * p.out_sj,
                         p.out_sj, p.accum, t, T::P2W);
          named_bar_sync(1 + T::NPIPE + pipe, T::P2W);  // every tile read: the stage may be refilled
          mbar_arrive(&empty[s]);
        }
        if (t == 0) XTRACE(4, i);
      } else if constexpr (!T::BIG) {
        // (plane, column-pair) items, columns (c, c + H) forming one complex
        // inverse FFT, with the plane fastest: a half-warp reads one column
        // of G planes (odd plane stride PS: distinct banks; the column-fastest
        // order had 2-3-way conflicts)
        const int H = (crop + 1) >> 1;
        const int jl = t % G, c = t / G;
        const bool act = jl < jv && c < H;
        const bool hb = c + H < crop;
        float2 zz[M];
        {
          const float2* col = inter + jl * PS + c;
          static_for<0, PC>([&](auto U) {
            constexpr int uu = decltype(U)::value;
            float2 a = act ? col[uu * CP] : make_float2(0.f, 0.f);
            float2 b = (act && hb) ? col[uu * CP + H] : make_float2(0.f, 0.f);
            if constexpr (uu == 0 || 2 * uu == M) {  // c2r ignores these imaginary parts
              a.y = 0.f;
              b.y = 0.f;
            }
            zz[uu] = make_float2(a.x - b.y, a.y + b.x);  // a + i b
            if constexpr (uu != 0 && 2 * uu != M) zz[M - uu] = make_float2(a.x + b.y, b.x - a.y);
          });
        }
        named_bar_sync(1 + T::NPIPE + pipe, T::P2W);  // stage read: reuse it as the output tile
        if (t == 0) XTRACE(3, i);
        if (act) {
          if (FCB_XFORM_EXP != 1) fft_reg<M, true>(zz);
          float* tile = reinterpret_cast<float*>(smem + s * T::STAGE) + jl * pst + c;
#pragma unroll
          for (int row = 0; row < M; ++row) {
            if (row < crop) {
              tile[0] = c2r_out(zz[row].x * scale, p.relu);
              if (hb) tile[H] = c2r_out(zz[row].y * scale, p.relu);
            }
            tile += crop;
          }
        }
        if (p.bulk) {
          fence_proxy_async_smem();  // the tile is read by the bulk store (async proxy)
          mbar_arrive(&outb[s]);
        } else {  // unaligned planes / accumulate: coalesced stores from the tile
          named_bar_sync(1 + T::NPIPE + pipe, T::P2W);
          if (FCB_XFORM_EXP != 2)
            c2r_store_tile(reinterpret_cast<const float*>(smem + s * T::STAGE), pst, jv, crop * crop,
                           p.out + (long long)r * p.out_sr + (long long)j0 * p.out_sj, p.out_sj, p.accum, t,
                           T::P2W);
          named_bar_sync(1 + T::NPIPE + pipe, T::P2W);  // every tile read: the stage may be refilled
          mbar_arrive(&empty[s]);
        }
        if (t == 0) XTRACE(4, i);
      } else {
        // one Hermitian column per thread: the half-length pre-twiddle is
        // formed straight from shared memory (X[k], X[H-k] pairs), so the
        // 33-entry column is never held whole in registers
        const bool act = t < jv * crop;
        const int jl = act ? t / crop : 0, c = t - jl * crop;
        constexpr int H = M / 2;
        float2 z[H];
        {
          const float2* col = inter + jl * PS + c;
          static_for<0, H>([&](auto K) {
            constexpr int k = decltype(K)::value;
            float2 xk = act ? col[k * CP] : make_float2(0.f, 0.f);
            float2 xc = cconj(act ? col[(H - k) * CP] : make_float2(0.f, 0.f));
            if constexpr (k == 0) {  // c2r ignores Im X[0] and Im X[H]
              xk.y = 0.f;
              xc.y = 0.f;
            }
            const float2 e = cadd(xk, xc);
            float2 o = csub(xk, xc);
            if constexpr (k != 0) o = cmul(o, tw128c<true, k * (128 / M)>());
            z[k] = make_float2(e.x - o.y, e.y + o.x);  // e + i*o
          });
        }
        if (p.bulk) {
          named_bar_sync(1 + T::NPIPE + pipe, T::P2W);
          if (act) {
            if (FCB_XFORM_EXP != 1) fft_reg<H, true>(z);
            float* tile = reinterpret_cast<float*>(smem + s * T::STAGE) + jl * pst + c;
#pragma unroll
            for (int i2 = 0; i2 < H; ++i2) {
              if (2 * i2 < crop) tile[(2 * i2) * crop] = c2r_out(z[i2].x * scale, p.relu);
              if (2 * i2 + 1 < crop) tile[(2 * i2 + 1) * crop] = c2r_out(z[i2].y * scale, p.relu);
            }
          }
          fence_proxy_async_smem();
          mbar_arrive(&outb[s]);
        } else {
          mbar_arrive(&empty[s]);
          if (act) {
            if (FCB_XFORM_EXP != 1) fft_reg<H, true>(z);
            float* dst = p.out + (long long)r * p.out_sr + (long long)(j0 + jl) * p.out_sj + c;
#pragma unroll
            for (int i2 = 0; i2 < H; ++i2) {
              float* d0 = dst + (2 * i2) * crop;
              float* d1 = d0 + crop;
              if (p.accum) {
                if (2 * i2 < crop) *d0 += z[i2].x * scale;
                if (2 * i2 + 1 < crop) *d1 += z[i2].y * scale;
              } else {
                if (2 * i2 < crop) *d0 = c2r_out(z[i2].x * scale, p.relu);
                if (2 * i2 + 1 < crop) *d1 = c2r_out(z[i2].y * scale, p.relu);
              }
            }
          }
        }
      }
    }
  }
  if (p.tspan) {
    __syncthreads();
    span_end(p.tspan);
  }
#ifdef FCB_XFORM_TRACE
  __syncthreads();
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    const long long t0 = g_xform_trace[0][0];
    for (int i = 0; i < 14; ++i)
      printf("c2r grp %2d load %7lld full %7lld p1done %7lld p2read %7lld p2done %7lld\n", i,
             g_xform_trace[0][i] - t0, g_xform_trace[1][i] - t0, g_xform_trace[2][i] - t0,
             g_xform_trace[3][i] - t0, g_xform_trace[4][i] - t0);
  }
#endif
}

}  // namespace fcb
