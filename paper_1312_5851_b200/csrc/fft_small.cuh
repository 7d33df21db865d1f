// K1 for operands whose planes are small against the FFT size (src <= m/4:
// the weight operand of fprop / bprop at every BASELINE config, e.g. 7 x 7
// kernels in 32 x 32 planes, 11 x 11 in 64 x 64), m in {32, 64}.
//
// Same maths and output layout as r2c_tma_kernel (fft_tma.cuh; reference
// detail::r2c_plane + transform_kernels, fft.hpp:160-179,
// conf_fft.hpp:263-281), re-blocked for what dominates such an operand: its
// spectrum writes (a 64 x 64 half spectrum of an 11 x 11 plane is 140x the
// plane).  r2c_tma_kernel keeps a group's whole output tile in a stage, so
// at m = 64 a group holds 4 planes and every bin leaves as a 32-B piece; here
// a group is 16 planes (one full 128-B line per bin) and the tile is built
// and stored a few u rows at a time:
//
//   pass 1  (plane, column c < src): real column FFT of src non-zero rows
//           (half-length complex FFT, zero-pruned) -> the m/2 + 1 rows u of
//           the intermediate [plane][u][c]   (src columns only: small)
//   pass 2  per chunk of u rows, (plane, u, quarter q): the row FFT over the
//           src non-zero columns by one radix-4 decimation-in-frequency step,
//           X[4k + q] = FFT_{m/4}( a[n] w_m^(q n) )[k]   (a[n] = 0 for n >= m/4)
//           -> the chunk's [u][v][16 planes] tile, drained by TMA tensor
//           stores (one M-bin box per u row) while the next chunk computes
//
// One persistent CTA per SM, 256 threads, double-buffered raw stages and
// output tiles.
#pragma once
#include <cuda.h>

#include <cstdint>

#include "fft_planes.cuh"
#include "ptx.cuh"

namespace fcb {

template <int M>
struct TSmall {
  static constexpr int G = 16;             // planes per group: one 128-B line per bin
  static constexpr int SRC = M / 4;        // largest plane edge
  static constexpr int H = M / 2, PC = M / 2 + 1;
  static constexpr int Q = M / 4;          // pass-2 FFT length (radix-4 DIF quarters)
  static constexpr int UC = 4;             // u rows per pass-2 chunk: 16 planes x 4 u x 4 quarters = 256
  static constexpr int NCHUNK = (PC + UC - 1) / UC;
  static constexpr int RAWP = (SRC * SRC * 4 + 16 + 15) / 16 * 16;  // plane slot (enclosing 16-B range)
  static constexpr int RAW = G * RAWP;                              // one raw stage (bytes)
  static constexpr int IS = SRC + 1;                                // intermediate row stride (float2)
  static constexpr int IPS = (PC * IS) | 1;                         // plane stride (odd: distinct banks)
  static constexpr int INTER = G * IPS * 8;
  static constexpr int TILE = UC * M * G * 8;                       // one output chunk (bytes)
  static constexpr int THREADS = 256;
  static constexpr int SMEM = 2 * RAW + INTER + 2 * TILE + 64;
  static_assert(G * SRC <= THREADS && G * UC * 4 == THREADS, "fft_small thread mapping");
};

// grid = persistent (<= groups), block = 256, smem = TSmall<M>::SMEM.
// tm: 3-D map over F[t][R][2 kpad] with box {32 floats, 1 row, M bins}.
template <int M>
__global__ void __launch_bounds__(256, 1)
    r2c_small_kernel(const __grid_constant__ R2CParams p, const __grid_constant__ CUtensorMap tm,
                     unsigned long long* tspan) {
  using T = TSmall<M>;
  constexpr int G = T::G, PC = T::PC, H = T::H, Q = T::Q, UC = T::UC;
  extern __shared__ __align__(128) uint8_t smem[];
  uint8_t* raw0 = smem;                                   // 2 raw stages
  float2* inter = reinterpret_cast<float2*>(smem + 2 * T::RAW);
  uint8_t* tile0 = smem + 2 * T::RAW + T::INTER;          // 2 output tiles (128-B aligned)
  uint64_t* full = reinterpret_cast<uint64_t*>(tile0 + 2 * T::TILE);
  const int ngj = (p.kpad + G - 1) / G;
  const int ngroups = p.R * ngj;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int src = p.src;
  if (tid == 0) {
    mbar_init(&full[0], 1);
    mbar_init(&full[1], 1);
    fence_barrier_init();
    tma_prefetch_desc(&tm);
  }
  __syncthreads();
  pdl_wait();
  span_begin(tspan);
  pdl_trigger();
  const uint64_t pol = l2_policy_evict_first();
  const float csign = p.conj ? -1.f : 1.f;
  const uint32_t pb = (uint32_t)(src * src) * 4u;
  auto issue = [&](int g, int s) {  // thread 0: the group's planes into raw stage s
    const int r = g / ngj, j0 = (g - r * ngj) * G;
    const int jv = max(0, min(G, p.J - j0));
    const float* base = p.in + (long long)r * p.in_sr + (long long)j0 * p.in_sj;
    uint32_t total = 0;
    for (int jl = 0; jl < jv; ++jl) {
      const uintptr_t a = reinterpret_cast<uintptr_t>(base + (long long)jl * p.in_sj);
      total += ((uint32_t)(a & 15) + pb + 15) & ~15u;
    }
    mbar_arrive_expect_tx(&full[s], total);
    for (int jl = 0; jl < jv; ++jl) {
      const uintptr_t a = reinterpret_cast<uintptr_t>(base + (long long)jl * p.in_sj);
      const uint32_t sz = ((uint32_t)(a & 15) + pb + 15) & ~15u;
      bulk_load(raw0 + s * T::RAW + jl * T::RAWP, reinterpret_cast<const void*>(a & ~uintptr_t(15)), sz, &full[s],
                pol);
    }
  };
  if (tid == 0 && (int)blockIdx.x < ngroups) issue(blockIdx.x, 0);
  int it = 0, nchunk_done = 0;
  for (int g = blockIdx.x; g < ngroups; g += gridDim.x, ++it) {
    const int s = it & 1;
    const int r = g / ngj, j0 = (g - r * ngj) * G;
    const int jv = max(0, min(G, p.J - j0));
    if (tid == 0 && g + (int)gridDim.x < ngroups) {
      fence_proxy_async_smem();  // stage s^1 was last read two groups ago
      issue(g + gridDim.x, s ^ 1);
    }
    mbar_wait(&full[s], (it >> 1) & 1);
    // ---- pass 1: (plane, column) items, column fastest (conflict-free reads)
    {
      const int c = tid % T::SRC, jl = tid / T::SRC;
      if (jl < jv && c < src) {
        const float* pin = p.in + (long long)r * p.in_sr + (long long)(j0 + jl) * p.in_sj;
        const float* col = reinterpret_cast<const float*>(raw0 + s * T::RAW + jl * T::RAWP) +
                           ((reinterpret_cast<uintptr_t>(pin) & 15) >> 2) + c;
        float2 z[H];  // (even, odd) rows packed: only the first SRC / 2 are non-zero
        static_for<0, H>([&](auto I) {
          constexpr int i = decltype(I)::value;
          if constexpr (2 * i < T::SRC) {
            z[i].x = 2 * i < src ? col[(2 * i) * src] : 0.f;
            z[i].y = 2 * i + 1 < src ? col[(2 * i + 1) * src] : 0.f;
          } else {
            z[i] = make_float2(0.f, 0.f);
          }
        });
        fft_reg_nz<H, T::SRC / 2, false>(z);
        float2* dst = inter + jl * T::IPS + c;
        static_for<0, H + 1>([&](auto K) {
          constexpr int k = decltype(K)::value;
          const float2 zk = z[k % H];
          const float2 zc = cconj(z[(H - k) % H]);
          const float2 e = make_float2(0.5f * (zk.x + zc.x), 0.5f * (zk.y + zc.y));
          const float2 d = csub(zk, zc);
          const float2 o = make_float2(0.5f * d.y, -0.5f * d.x);  // (zk - zc) / (2i)
          float2 wo;
          if constexpr (k == 0) wo = o;
          else if constexpr (k == H) wo = make_float2(-o.x, -o.y);
          else wo = cmul(o, tw128c<false, k * (128 / M)>());
          dst[k * T::IS] = cadd(e, wo);
        });
      }
    }
    __syncthreads();  // intermediate complete (and raw stage s read)
    // ---- pass 2 in chunks of UC u rows; warp = quarter q + u pair, lanes = (u, plane)
    float amx = 0.f;
    const int q = warp & 3, jl = lane & 15;
    for (int ch = 0; ch < T::NCHUNK; ++ch, ++nchunk_done) {
      const int b = nchunk_done & 1;
      float2* tile = reinterpret_cast<float2*>(tile0 + b * T::TILE);
      if (tid == 0) bulk_wait_group_read<1>();  // the stores that last read tile b are done with it
      __syncthreads();
      const int ul = (warp >> 2) * 2 + (lane >> 4), u = ch * UC + ul;
      if (u < PC) {
        const bool act = jl < jv;
        float2 y[Q];
        const float2* row = inter + jl * T::IPS + u * T::IS;
        // y[n] = a[n] w_m^(q n), a[n] = row[n] for n < src (columns >= src are zero)
        switch (q) {
#define FCB_SMALL_Q(QQ)                                                                     \
  case QQ:                                                                                  \
    static_for<0, Q>([&](auto N) {                                                          \
      constexpr int n = decltype(N)::value;                                                 \
      const float2 a = (act && n < src) ? row[n] : make_float2(0.f, 0.f);                   \
      if constexpr ((QQ * n) % M == 0) y[n] = a;                                            \
      else y[n] = cmul(a, tw128c<false, ((QQ * n) % M) * (128 / M)>());                     \
    });                                                                                     \
    break;
          FCB_SMALL_Q(0)
          FCB_SMALL_Q(1)
          FCB_SMALL_Q(2)
          FCB_SMALL_Q(3)
#undef FCB_SMALL_Q
        }
        fft_reg<Q, false>(y);
        float2* o = tile + (ul * M + q) * G + jl;  // bin v = 4k + q of row u
#pragma unroll
        for (int k = 0; k < Q; ++k) {
          const float2 v = make_float2(y[k].x, csign * y[k].y);
          o[4 * k * G] = v;
          amx = fmaxf(amx, fmaxf(fabsf(v.x), fabsf(v.y)));
        }
      }
      fence_proxy_async_smem();  // the tile is read by the TMA stores (async proxy)
      __syncthreads();
      if (tid == 0) {
        for (int l = 0; l < UC && ch * UC + l < PC; ++l)
          tma_store_3d(&tm, tile + l * M * G, 2 * j0, r, (ch * UC + l) * M);
        bulk_commit_group();
      }
    }
    if (p.amax) {  // row r's maximum over this group's planes
      const uint32_t v = __reduce_max_sync(0xffffffffu, __float_as_uint(amx));
      if (lane == 0) atomicMax(p.amax + r, ((unsigned long long)p.epoch << 32) | v);
    }
    __syncthreads();  // every thread is past pass 2: the next group may overwrite the intermediate
  }
  if (tid == 0) bulk_wait_group<0>();  // spectra written before the grid completes
  if (tspan) {
    __syncthreads();
    span_end(tspan);
  }
}

}  // namespace fcb
