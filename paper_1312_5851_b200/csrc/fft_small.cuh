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
#include "fft_tma.cuh"
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

namespace fcb {

// ---------------------------------------------------------------- K4, small crops
// The c2r of accGrad's weight gradients (crop <= m/4, e.g. 11 x 11 kernels
// in 64 x 64 planes) at m in {32, 64}, from the group-major product
// P[r][J/16][t][16] (the GEMM writes it so for this kernel): every 16-plane
// group's u row is one contiguous M x 128-B block, so the group streams in
// as UC-row chunks through a ring of stages (full-line bulk loads, loads in
// flight across groups), where c2r_tma_kernel at m = 64 holds 4-plane
// groups and reads 32-B pieces per bin.
//   pass 1  per chunk, (plane, u, half h): the inverse row FFT over v by one
//           radix-2 DIF step, x = 2k + h, only the x < crop outputs kept ->
//           the intermediate [plane][u][x] (crop columns: small)
//   pass 2  per group, (plane, column x): direct Hermitian DFTs over u for
//           every row y < crop, twiddles as immediates (as in c2r_tma_kernel)
//           -> staged tile -> coalesced stores (optionally accumulated)
template <int M>
struct TC2RSmall {
  static constexpr int G = 16;
  static constexpr int PC = M / 2 + 1, H = M / 2;
  static constexpr int UC = 8;                           // u rows per chunk
  static constexpr int NCH = (PC + UC - 1) / UC;
  static constexpr int STAGE = UC * M * G * 8;           // bytes
  static constexpr int NST = (M == 64) ? 2 : 4;          // stages
  static constexpr int CMAX = M / 4;                     // largest crop
  static constexpr int IS = CMAX + 1;                    // intermediate row stride (float2)
  static constexpr int IPS = (PC * IS) | 1;              // plane stride (odd)
  static constexpr int INTER = G * IPS * 8;
  static constexpr int PST = ((CMAX * CMAX + 3) / 4 % 2 == 0) ? ((CMAX * CMAX + 3) / 4 + 1) * 4
                                                             : (CMAX * CMAX + 3) / 4 * 4;
  static constexpr int TILE = G * PST * 4;
  static constexpr int NC = 256;                         // compute threads
  static constexpr int THREADS = 32 + NC;                // + the copy warp
  static constexpr int SMEM = NST * STAGE + INTER + TILE + 2 * NST * 8 + 64;
  static_assert(G * UC * 2 == NC && G * CMAX <= NC, "c2r_small thread mapping");
};

// grid = persistent (<= groups), block = THREADS, smem = SMEM.  p.gm must be
// set (group-major product); groups g = (row r, 16-column group jg).
template <int M>
__global__ void __launch_bounds__(TC2RSmall<M>::THREADS, 1) c2r_small_kernel(const __grid_constant__ C2RParams p) {
  using T = TC2RSmall<M>;
  constexpr int G = T::G, PC = T::PC, H = T::H, UC = T::UC, NST = T::NST;
  extern __shared__ __align__(128) uint8_t smem[];
  float2* inter = reinterpret_cast<float2*>(smem + NST * T::STAGE);
  float* tile = reinterpret_cast<float*>(smem + NST * T::STAGE + T::INTER);
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + NST * T::STAGE + T::INTER + T::TILE);
  uint64_t* empty = full + NST;
  const int ngj = (p.J + G - 1) / G;
  const int ngj_all = p.J_all ? (p.J_all + G - 1) / G : ngj;
  const int ngroups = p.R * ngj;
  const int crop = p.crop;
  constexpr long long BLOCK = (long long)M * PC * G;  // complex per group block
  if (threadIdx.x == 0) {
    for (int s = 0; s < NST; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], T::NC);
    }
    fence_barrier_init();
  }
  __syncthreads();
  pdl_wait();
  span_begin(p.tspan);
  pdl_trigger();
  if (threadIdx.x < 32) {
    // ------------------------------------------------ copy warp: u-row chunks into the ring
    if (threadIdx.x == 0) {
      const uint64_t pol = l2_policy_evict_first();
      int k = 0;
      for (int g = blockIdx.x; g < ngroups; g += gridDim.x) {
        const int r = g / ngj, jg = g - r * ngj;
        const float2* blk = reinterpret_cast<const float2*>(p.in) +
                            (long long)(r * ngj_all + p.jbase / G + jg) * BLOCK;
        for (int ch = 0; ch < T::NCH; ++ch, ++k) {
          const int s = k % NST;
          mbar_wait(&empty[s], ((k / NST) & 1) ^ 1);
          const int rows = min(UC, PC - ch * UC);
          const uint32_t bytes = (uint32_t)rows * M * G * 8;
          mbar_arrive_expect_tx(&full[s], bytes);
          bulk_load(smem + s * T::STAGE, blk + (long long)ch * UC * M * G, bytes, &full[s], pol);
        }
      }
    }
    return;  // the copy warp takes no part in the compute barriers below
  }
  const int t = threadIdx.x - 32;
  const float scale = p.scale;
  int k = 0;
  for (int g = blockIdx.x; g < ngroups; g += gridDim.x) {
    const int r = g / ngj, j0 = (g - r * ngj) * G;
    const int jv = min(G, p.J - j0);
    // ---- pass 1: (plane jl, u, half h): inverse row FFT over v, x = 2k' + h < crop kept
    for (int ch = 0; ch < T::NCH; ++ch, ++k) {
      const int s = k % NST;
      mbar_wait(&full[s], (k / NST) & 1);
      const int jl = t & 15, h = (t >> 4) & 1, ul = t >> 5, u = ch * UC + ul;
      const float2* row = reinterpret_cast<const float2*>(smem + s * T::STAGE) + ul * M * G + jl;
      float2 z[H];
      if (u < PC) {
        static_for<0, H>([&](auto Nn) {
          constexpr int n = decltype(Nn)::value;
          const float2 a0 = row[n * G], a1 = row[(n + H) * G];
          if constexpr (n == 0) {
            z[n] = h ? csub(a0, a1) : cadd(a0, a1);
          } else {
            const float2 d = csub(a0, a1);
            z[n] = h ? cmul(d, tw128c<true, n * (128 / M)>()) : cadd(a0, a1);
          }
        });
      }
      mbar_arrive(&empty[s]);  // the chunk is in registers: the ring slot may refill
      if (u < PC && jl < jv) {
        fft_reg<H, true>(z);
        float2* dst = inter + jl * T::IPS + u * T::IS + h;
#pragma unroll
        for (int kk = 0; kk < H; ++kk)
          if (2 * kk + h < crop) dst[2 * kk] = z[kk];
      }
    }
    named_bar_sync(1, T::NC);  // intermediate complete
    // ---- pass 2: (plane jl, column x), direct Hermitian DFTs over u
    {
      const int jl = t & 15, x = t >> 4;
      const bool act = jl < jv && x < crop;
      float res[T::CMAX];
      if (act) {
        const float2* col = inter + jl * T::IPS + x;
        float2 zz[H + 1];
        static_for<0, H + 1>([&](auto U) { zz[decltype(U)::value] = col[decltype(U)::value * T::IS]; });
        static_for<0, T::CMAX>([&](auto Y) {
          constexpr int y = decltype(Y)::value;
          if (y < crop) {
            float acc = 0.f;
            static_for<1, H>([&](auto U) {
              constexpr int u = decltype(U)::value;
              const float2 w = tw128c<true, (u * y * (128 / M)) % 128>();
              acc = fmaf(zz[u].x, w.x, fmaf(-zz[u].y, w.y, acc));
            });
            const float e = zz[0].x + ((y & 1) ? -zz[H].x : zz[H].x);
            res[y] = c2r_out((e + 2.f * acc) * scale, p.relu);
          }
        });
        static_for<0, T::CMAX>([&](auto Y) {
          constexpr int y = decltype(Y)::value;
          if (y < crop) tile[jl * T::PST + y * crop + x] = res[y];
        });
      }
    }
    named_bar_sync(1, T::NC);  // tile complete, intermediate read
    c2r_store_tile(tile, T::PST, jv, crop * crop, p.out + (long long)r * p.out_sr + (long long)j0 * p.out_sj,
                   p.out_sj, p.accum, t, T::NC);
    named_bar_sync(1, T::NC);  // tile read before the next group's pass 2 writes it
  }
  if (p.tspan) {  // thread 0 of the CTA is the copy thread (gone): compute thread 0 records
    named_bar_sync(1, T::NC);
    if (t == 0) atomicMax(p.tspan + kSpanEndOff, global_ns());
  }
}

}  // namespace fcb
