// FFT codelets and the frequency layout shared by the plane transforms, plus
// the simple one-pass-per-CTA K1/K4 kernels used for m in {1, 2} (the
// TMA-pipelined kernels for m >= 4 are in fft_tma.cuh).
//
// Replaces the reference's per-plane CPU transforms plus the strided
// bin-major scatter/gather glue:
//   detail::r2c_plane + transform_planes/transform_kernels
//     (/root/reference/proj/include/fftconv/fft.hpp:160-179,
//      conv_fft.hpp:242-281)
//   detail::c2r_plane + inverse_planes + the grad_weight gather
//     (fft.hpp:184-203, conv_fft.hpp:285-304, :192-203)
//
// Frequency layout (internal, not observable through the operator API):
// half spectrum over ROWS, u in [0, m/2], all columns v in [0, m); bin
// t = u*m + v.  A plane's real column pass (the rows of the plane are read
// with coalesced row loads, one lane per column) produces the u half, the
// complex row pass produces all v.  Spectra are stored as GEMM operands:
//   F[t][r][2*kpad]  (complex interleaved, fp32),
// where r is the operand row (M or N index of the per-bin GEMM) and j the
// K index.  One CTA owns 16 consecutive K indices (one 128-byte line per
// bin and row) so every store is a full line, and it writes zeros into the
// K padding so the tensor-core reduction over padded K is exact.
//
// Inverse: rows of the product spectrum are inverted over v first (only
// the cropped columns are produced), then each cropped column is a
// Hermitian length-m sequence over u, inverted by a packed c2r that drops
// the imaginary parts of the u = 0 and u = m/2 bins -- exactly the values
// the reference's c2r_plane discards when it takes .real().
#pragma once
#include <cstdint>
#include <type_traits>

#include "ptx.cuh"
#include "twiddles.cuh"

namespace fcb {

constexpr int kKChunk = 16;  // K padding granule: 16 complex = one 128-B line

__host__ __device__ constexpr int ilog2c(int n) { return n <= 1 ? 0 : 1 + ilog2c(n >> 1); }
__host__ __device__ constexpr int bitrev_c(int i, int bits) {
  int r = 0;
  for (int b = 0; b < bits; ++b)
    if (i & (1 << b)) r |= 1 << (bits - 1 - b);
  return r;
}

__device__ __forceinline__ float2 cadd(float2 a, float2 b) { return make_float2(a.x + b.x, a.y + b.y); }
__device__ __forceinline__ float2 csub(float2 a, float2 b) { return make_float2(a.x - b.x, a.y - b.y); }
__device__ __forceinline__ float2 cmul(float2 a, float2 b) {
  return make_float2(a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x);
}
__device__ __forceinline__ float2 cconj(float2 a) { return make_float2(a.x, -a.y); }

// exp(-+2 pi i K / 128), folded at compile time into instruction immediates.
template <bool INV, int K>
__device__ __forceinline__ float2 tw128c() {
  constexpr float re = tw128_re(K);
  constexpr float im = tw128_im(K);
  return make_float2(re, INV ? -im : im);
}

// Compile-time loop: f(std::integral_constant<int, i>) for i in [B, E), so
// every register-array index below is a constant expression and the arrays
// stay in registers.
template <int B, int E, typename F>
__device__ __forceinline__ void static_for(F&& f) {
  if constexpr (B < E) {
    f(std::integral_constant<int, B>{});
    static_for<B + 1, E>(f);
  }
}

template <int LEN, int J, bool INV>
__device__ __forceinline__ float2 twiddle_mul(float2 v) {
  if constexpr (J == 0) {
    return v;
  } else if constexpr (4 * J == LEN) {  // w = -i (forward) / +i (inverse)
    return INV ? make_float2(-v.y, v.x) : make_float2(v.y, -v.x);
  } else {
    return cmul(v, tw128c<INV, J * (128 / LEN)>());
  }
}

// In-register radix-2 DIT FFT of length N (N | 128), natural order in and
// out.  Forward is unnormalised; INV conjugates the twiddles (no scaling).
template <int N, bool INV>
__device__ __forceinline__ void fft_reg(float2 (&a)[N]) {
  if constexpr (N > 1) {
    constexpr int L = ilog2c(N);
    static_for<0, N>([&](auto I) {
      constexpr int i = decltype(I)::value;
      constexpr int r = bitrev_c(i, L);
      if constexpr (i < r) {
        const float2 t = a[i];
        a[i] = a[r];
        a[r] = t;
      }
    });
    static_for<1, L + 1>([&](auto S) {
      constexpr int len = 1 << decltype(S)::value;
      constexpr int half = len >> 1;
      static_for<0, N / len>([&](auto B) {
        constexpr int s = decltype(B)::value * len;
        static_for<0, half>([&](auto Jc) {
          constexpr int j = decltype(Jc)::value;
          const float2 u = a[s + j];
          const float2 v = twiddle_mul<len, j, INV>(a[s + j + half]);
          a[s + j] = cadd(u, v);
          a[s + j + half] = csub(u, v);
        });
      });
    });
  }
}

// N-point DFT (natural order in and out) of a sequence whose inputs at
// n >= NZ are zero: with k = q*R + r (R = N/NZ),
//   X[q*R + r] = FFT_NZ( x[n] * w_N^(n*r) )[q],
// i.e. R twiddled NZ-point FFTs -- the first log2(R) radix-2 stages would
// only ever add zeros.  Used for small kernels (e.g. 7x7 weights in 32x32
// planes: NZ = 8, ~1/3 fewer FP instructions than the full transform).
template <int N, int NZ, bool INV>
__device__ __forceinline__ void fft_reg_nz(float2 (&a)[N]) {
  static_assert(N % NZ == 0 && NZ >= 1, "fft_reg_nz");
  if constexpr (NZ == N) {
    fft_reg<N, INV>(a);
  } else {
    constexpr int R = N / NZ;
    float2 x[NZ];
    static_for<0, NZ>([&](auto I) { x[decltype(I)::value] = a[decltype(I)::value]; });
    static_for<0, R>([&](auto Rr) {
      constexpr int r = decltype(Rr)::value;
      float2 y[NZ];
      static_for<0, NZ>([&](auto I) {
        constexpr int n = decltype(I)::value;
        if constexpr ((n * r) % N == 0) y[n] = x[n];
        else y[n] = cmul(x[n], tw128c<INV, ((n * r) % N) * (128 / N)>());
      });
      fft_reg<NZ, INV>(y);
      static_for<0, NZ>([&](auto Q) { a[decltype(Q)::value * R + r] = y[decltype(Q)::value]; });
    });
  }
}

template <int N, typename Emit>
__device__ __forceinline__ void rfft_packed_emit(float2 (&z)[N / 2], Emit&& emit);

// Real-input forward DFT of length N (zero-padded column), emitting the
// N/2+1 non-redundant outputs X[k] through emit(k, X[k]).  N >= 4 uses the
// half-length complex FFT on (even, odd) pairs plus the split post-twiddle.
template <int N, typename Emit>
__device__ __forceinline__ void rfft_emit(const float (&x)[N], Emit&& emit) {
  if constexpr (N == 1) {
    emit(0, make_float2(x[0], 0.f));
  } else if constexpr (N == 2) {
    emit(0, make_float2(x[0] + x[1], 0.f));
    emit(1, make_float2(x[0] - x[1], 0.f));
  } else {
    constexpr int H = N / 2;
    float2 z[H];
    static_for<0, H>([&](auto I) {
      constexpr int i = decltype(I)::value;
      z[i] = make_float2(x[2 * i], x[2 * i + 1]);
    });
    rfft_packed_emit<N>(z, emit);
  }
}

// rfft_emit with the (even, odd) pairs already packed: z[i] = x[2i] + i x[2i+1]
// (saves holding the N reals and the N/2 complex values at once).
template <int N, typename Emit>
__device__ __forceinline__ void rfft_packed_emit(float2 (&z)[N / 2], Emit&& emit) {
  static_assert(N >= 4, "rfft_packed_emit");
  {
    constexpr int H = N / 2;
    fft_reg<H, false>(z);
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
      else wo = cmul(o, tw128c<false, k * (128 / N)>());
      emit(k, cadd(e, wo));
    });
  }
}

// Hermitian (c2r) inverse DFT of length N, unnormalised: input X[0..N/2]
// (imaginary parts of X[0] and X[N/2] are ignored), output x[0..N).
template <int N>
__device__ __forceinline__ void irfft_reg(float2 (&X)[N / 2 + 1], float (&x)[N]) {
  if constexpr (N == 1) {
    x[0] = X[0].x;
  } else if constexpr (N == 2) {
    x[0] = X[0].x + X[1].x;
    x[1] = X[0].x - X[1].x;
  } else {
    constexpr int H = N / 2;
    X[0].y = 0.f;
    X[H].y = 0.f;
    float2 z[H];
    static_for<0, H>([&](auto K) {
      constexpr int k = decltype(K)::value;
      const float2 xk = X[k];
      const float2 xc = cconj(X[H - k]);
      const float2 e = cadd(xk, xc);
      float2 o = csub(xk, xc);
      if constexpr (k != 0) o = cmul(o, tw128c<true, k * (128 / N)>());
      z[k] = make_float2(e.x - o.y, e.y + o.x);  // e + i*o
    });
    fft_reg<H, true>(z);
    static_for<0, H>([&](auto I) {
      constexpr int i = decltype(I)::value;
      x[2 * i] = z[i].x;
      x[2 * i + 1] = z[i].y;
    });
  }
}

// Threads per CTA: one pass-2 row item per thread (16 planes x (m/2+1)
// u-rows [x2 split halves for m = 64]) so no pass runs a lightly-filled
// second round.
#ifndef FCB_G_SMALL
#define FCB_G_SMALL 16
#endif
template <int M>
struct PlaneTraits {
  static constexpr int PC = M / 2 + 1;
  // Planes (K indices / spectrum columns) per CTA: 16 x 8 B = one 128-B
  // line per bin and operand row (8 -> 64-B half lines, twice the CTAs).
  static constexpr int G = (M == 64) ? 16 : FCB_G_SMALL;
  // r2c: u rows per CTA chunk; c2r / r2c row split for m = 64.
  static constexpr int UC = (M == 64) ? 11 : PC;
  static constexpr int SPLIT = (M == 64) ? 2 : 1;
  // Two real columns per complex FFT (m <= 32: registers allow it).
  static constexpr bool PAIR = (M >= 4 && M <= 32);
  // One pass-2 row item per thread: G planes x UC u-rows [x2 halves].
  static constexpr int THREADS = ((G * SPLIT * UC + 31) / 32) * 32 < 64 ? 64 : ((G * SPLIT * UC + 31) / 32) * 32;
#ifndef FCB_MINB32
#define FCB_MINB32 2
#endif
#ifndef FCB_MINB64
#define FCB_MINB64 2
#endif
  static constexpr int MIN_CTAS = (M == 64) ? FCB_MINB64 : (M == 32) ? (G == 8 ? 4 : FCB_MINB32) : 4;
};

// Hermitian inverse DFT emitting real outputs through emit(i, x_i) in
// order, without materialising the output array.
template <int N, typename Emit>
__device__ __forceinline__ void irfft_emit(float2 (&X)[N / 2 + 1], Emit&& emit) {
  static_assert(N >= 4, "irfft_emit");
  constexpr int H = N / 2;
  X[0].y = 0.f;
  X[H].y = 0.f;
  float2 z[H];
  static_for<0, H>([&](auto K) {
    constexpr int k = decltype(K)::value;
    const float2 xk = X[k];
    const float2 xc = cconj(X[H - k]);
    const float2 e = cadd(xk, xc);
    float2 o = csub(xk, xc);
    if constexpr (k != 0) o = cmul(o, tw128c<true, k * (128 / N)>());
    z[k] = make_float2(e.x - o.y, e.y + o.x);  // e + i*o
  });
  fft_reg<H, true>(z);
#pragma unroll
  for (int i = 0; i < H; ++i) {
    emit(2 * i, z[i].x);
    emit(2 * i + 1, z[i].y);
  }
}

// ---------------------------------------------------------------- K1: r2c
struct R2CParams {
  const float* in;  // real planes, plane (r, j) at in + r*in_sr + j*in_sj
  float* out;       // F[t][r][2*kpad]
  long long in_sr, in_sj;
  int R;     // operand rows
  int J;     // valid K count
  int kpad;  // padded K (multiple of 16)
  int src;   // source plane edge (square, src <= M): zero-padded implicitly
  int cpad;  // odd smem column stride >= src
  int conj;  // 1: store the conjugate spectrum
  // per operand row r: max |Re|, |Im| over the row's spectra (all K, all
  // bins) for the fp16 GEMM (TMA / m = 128 kernels only): amax[r] =
  // atomicMax of (epoch << 32 | float bits), so a newer epoch's maximum
  // supersedes the stale value without a reset.
  unsigned long long* amax = nullptr;
  unsigned epoch = 0;
};

// One launch transforms both operands of an operator (A groups first, then
// B groups) in the TMA kernels.
struct R2CPair {
  R2CParams op[2];
  int n;  // 1 or 2 operands
  unsigned long long* tspan = nullptr;  // live span slot (ptx.cuh span_begin / span_end)
};

// grid = (kpad/G, R, ceil((M/2+1)/UC)), block = PlaneTraits<M>::THREADS.
// smem = G * UC * cpad * sizeof(float2).
template <int M>
__global__ void __launch_bounds__(PlaneTraits<M>::THREADS, PlaneTraits<M>::MIN_CTAS) r2c_planes_kernel(const R2CParams p) {
  using Tr = PlaneTraits<M>;
  constexpr int PC = Tr::PC, UC = Tr::UC, SPLIT = Tr::SPLIT;
  constexpr int G = Tr::G;
  extern __shared__ float2 s1[];  // [G][UC][cpad]
  pdl_wait();
  pdl_trigger();
  const int r = blockIdx.y;
  const int j0 = blockIdx.x * G;
  const int u0 = blockIdx.z * UC;
  const int src = p.src, cpad = p.cpad;
  const int jvalid = min(G, p.J - j0);
  const float* inbase = p.in + (long long)r * p.in_sr + (long long)j0 * p.in_sj;

  // Pass 1: zero-padded real column FFTs over the plane rows; lanes walk
  // consecutive columns so every row load is coalesced.
  if constexpr (Tr::PAIR) {
    // two adjacent real columns (a, b) packed as a + i b in one complex FFT
    const int npair = (src + 1) >> 1;
    const int items1 = jvalid * npair;
    for (int item = threadIdx.x; item < items1; item += blockDim.x) {
      const int jl = item / npair, cp = item - jl * npair;
      const int c = 2 * cp;
      const float* col = inbase + (long long)jl * p.in_sj + c;
      const bool has_b = c + 1 < src;
      float2 z[M];
#pragma unroll
      for (int i = 0; i < M; ++i) {
        if (i < src) {
          z[i].x = __ldg(col + (long long)i * src);
          z[i].y = has_b ? __ldg(col + (long long)i * src + 1) : 0.f;
        } else {
          z[i] = make_float2(0.f, 0.f);
        }
      }
      fft_reg<M, false>(z);
      float2* dst = s1 + (jl * UC) * cpad + c;
      static_for<0, PC>([&](auto U) {
        constexpr int u = decltype(U)::value;
        const float2 zu = z[u];
        const float2 zc = cconj(z[(M - u) % M]);
        const float2 a = make_float2(0.5f * (zu.x + zc.x), 0.5f * (zu.y + zc.y));
        const float2 d = csub(zu, zc);
        const float2 b = make_float2(0.5f * d.y, -0.5f * d.x);  // (zu - zc) / (2i)
        const int ul = u - u0;
        if (ul >= 0 && ul < UC) {
          dst[ul * cpad] = a;
          if (has_b) dst[ul * cpad + 1] = b;
        }
      });
    }
  } else {
    const int items1 = jvalid * src;
    for (int item = threadIdx.x; item < items1; item += blockDim.x) {
      const int jl = item / src, c = item - jl * src;
      const float* col = inbase + (long long)jl * p.in_sj + c;
      float x[M];
#pragma unroll
      for (int i = 0; i < M; ++i) x[i] = (i < src) ? __ldg(col + (long long)i * src) : 0.f;
      float2* dst = s1 + (jl * UC) * cpad + c;
      rfft_emit<M>(x, [&](int u, float2 v) {
        const int ul = u - u0;
        if (ul >= 0 && ul < UC) dst[ul * cpad] = v;
      });
    }
  }
  __syncthreads();

  // Pass 2: one thread per (plane, u[, half]): complex row FFT over the
  // columns, written bin-major with 16 planes (128 B) per bin per row.
  const int urows = min(UC, PC - u0);
  const int items2 = G * SPLIT * urows;
  const long long bstride = (long long)p.R * p.kpad;  // float2 per bin
  float2* outbase = reinterpret_cast<float2*>(p.out) + (long long)r * p.kpad + j0;
  const float csign = p.conj ? -1.f : 1.f;
  for (int item = threadIdx.x; item < items2; item += blockDim.x) {
    const int jl = item % G;
    const int rest = item / G;
    const int h = rest % SPLIT;
    const int ul = rest / SPLIT;
    const int u = u0 + ul;
    float2* o = outbase + jl + (long long)(u * M + h) * bstride;
    constexpr int NS = M / SPLIT;
    if (jl >= jvalid) {  // K padding: exact zeros
#pragma unroll 4
      for (int i = 0; i < NS; ++i) o[(long long)(i * SPLIT) * bstride] = make_float2(0.f, 0.f);
      continue;
    }
    const float2* row = s1 + (jl * UC + ul) * cpad;
    float2 z[NS];
    if constexpr (SPLIT == 1) {
#pragma unroll
      for (int c = 0; c < M; ++c) z[c] = (c < src) ? row[c] : make_float2(0.f, 0.f);
    } else {
      static_assert(SPLIT == 2, "split");
      // decimation in frequency: outputs v = 2i + h
      static_for<0, NS>([&](auto Cc) {
        constexpr int c = decltype(Cc)::value;
        const float2 a = (c < src) ? row[c] : make_float2(0.f, 0.f);
        const float2 b = (c + NS < src) ? row[c + NS] : make_float2(0.f, 0.f);
        if (h == 0) {
          z[c] = cadd(a, b);
        } else {
          if constexpr (c == 0) z[c] = csub(a, b);
          else z[c] = cmul(csub(a, b), tw128c<false, c * (128 / M)>());
        }
      });
    }
    fft_reg<NS, false>(z);
#pragma unroll
    for (int i = 0; i < NS; ++i)
      o[(long long)(i * SPLIT) * bstride] = make_float2(z[i].x, csign * z[i].y);
  }
}

// ---------------------------------------------------------------- K4: c2r
struct C2RParams {
  const float* in;  // product spectrum P[t][r][2*J]
  float* out;       // real planes, plane (r, j) at out + r*out_sr + j*out_sj
  long long out_sr, out_sj;
  int R, J;     // spectrum rows, valid columns (== row length)
  int crop;     // output edge (top-left crop)
  int cc;       // output columns per CTA chunk
  int ccpad;    // odd smem stride >= cc
  float scale;  // 1 / m^2 (negated to fold a sign flip of the product)
  int ld;       // row stride of P in complex elements (>= J, even)
  int bulk;     // 1: output planes 16-B aligned -> staged + bulk-stored (K4 TMA kernel)
  int gm;       // 1: P is group-major P[r][J/16][t][16] (K4 TMA kernel, m <= 32)
  int accum;    // 1: add into the output (direct-store mode; chunked accGrad)
  // column window (K4 TMA kernel): columns [jbase, jbase + J) of a product
  // whose rows hold J_all columns; out points at column jbase's planes.
  // Lets accGrad's K4 run in f'-chunks (each chunk's gw rows all-reduced
  // while the next chunk transforms).  jbase is a multiple of the group size.
  int jbase = 0;
  int J_all = 0;  // 0: J
  unsigned long long* tspan = nullptr;  // live span slot (TMA K4 only)
  // 1: the stack's relu fused into the store, y = max(conv, 0) as
  // layers.hpp:88-97 writes it (x > 0 ? x : 0); never with accum
  int relu = 0;
};

// The output value of a K4 store: scaled, optionally through the fused relu.
__device__ __forceinline__ float c2r_out(float v, int relu) { return relu ? (v > 0.f ? v : 0.f) : v; }

// grid = (ceil(J/G), R, ceil(crop/cc)), block = PlaneTraits<M>::THREADS.
// smem = G * (M/2+1) * ccpad * sizeof(float2).
template <int M>
__global__ void __launch_bounds__(PlaneTraits<M>::THREADS, PlaneTraits<M>::MIN_CTAS) c2r_planes_kernel(const C2RParams p) {
  using Tr = PlaneTraits<M>;
  constexpr int PC = Tr::PC, SPLIT = Tr::SPLIT;
  constexpr int G = Tr::G;
  constexpr int NS = M / SPLIT;
  extern __shared__ float2 s1[];  // [G][PC][ccpad]
  pdl_wait();
  pdl_trigger();
  const int r = blockIdx.y;
  const int j0 = blockIdx.x * G;
  const int c0 = blockIdx.z * p.cc;
  const int ncols = min(p.cc, p.crop - c0);
  const int jvalid = min(G, p.J - j0);
  const int ccpad = p.ccpad;
  const long long bstride = (long long)p.R * p.ld;  // float2 per bin
  const float2* inbase = reinterpret_cast<const float2*>(p.in) + (long long)r * p.ld + j0;

  // Pass 1: per (plane, u[, half]) inverse row FFT over v, keep cropped
  // columns of this chunk.  Lanes = consecutive planes -> 128-B loads.
  const int items1 = G * SPLIT * PC;
  for (int item = threadIdx.x; item < items1; item += blockDim.x) {
    const int jl = item % G;
    const int rest = item / G;
    const int h = rest % SPLIT;
    const int u = rest / SPLIT;
    if (jl >= jvalid) continue;
    const float2* src = inbase + jl + (long long)(u * M) * bstride;
    float2 z[NS];
    if constexpr (SPLIT == 1) {
#pragma unroll
      for (int v = 0; v < M; ++v) z[v] = __ldg(src + (long long)v * bstride);
    } else {
      static_for<0, NS>([&](auto Vv) {
        constexpr int v = decltype(Vv)::value;
        const float2 a = __ldg(src + (long long)v * bstride);
        const float2 b = __ldg(src + (long long)(v + NS) * bstride);
        if (h == 0) {
          z[v] = cadd(a, b);
        } else {
          if constexpr (v == 0) z[v] = csub(a, b);
          else z[v] = cmul(csub(a, b), tw128c<true, v * (128 / M)>());
        }
      });
    }
    fft_reg<NS, true>(z);
    float2* dst = s1 + (jl * PC + u) * ccpad;
#pragma unroll
    for (int i = 0; i < NS; ++i) {
      const int c = i * SPLIT + h - c0;
      if (c >= 0 && c < ncols) dst[c] = z[i];
    }
  }
  __syncthreads();

  // Pass 2: Hermitian c2r over u per cropped column, write the cropped rows;
  // lanes = consecutive columns -> contiguous row segments.
  const float scale = p.scale;
  if constexpr (Tr::PAIR) {
    // two columns (a, b) at once: Z = Xa + i Xb over the full u range
    const int npair = (ncols + 1) >> 1;
    const int items2 = jvalid * npair;
    for (int item = threadIdx.x; item < items2; item += blockDim.x) {
      const int jl = item / npair, cp = item - jl * npair;
      const int cl = 2 * cp;
      const bool has_b = cl + 1 < ncols;
      const float2* colp = s1 + (jl * PC) * ccpad + cl;
      float2 z[M];
      static_for<0, PC>([&](auto U) {
        constexpr int u = decltype(U)::value;
        float2 a = colp[u * ccpad];
        float2 b = has_b ? colp[u * ccpad + 1] : make_float2(0.f, 0.f);
        if constexpr (u == 0 || 2 * u == M) {  // c2r ignores these imaginary parts
          a.y = 0.f;
          b.y = 0.f;
        }
        z[u] = make_float2(a.x - b.y, a.y + b.x);  // a + i b
        if constexpr (u != 0 && 2 * u != M) z[M - u] = make_float2(a.x + b.y, b.x - a.y);  // conj(a) + i conj(b)
      });
      fft_reg<M, true>(z);
      float* dst = p.out + (long long)r * p.out_sr + (long long)(j0 + jl) * p.out_sj + c0 + cl;
#pragma unroll
      for (int i = 0; i < M; ++i) {
        if (i < p.crop) {
          dst[(long long)i * p.crop] = c2r_out(z[i].x * scale, p.relu);
          if (has_b) dst[(long long)i * p.crop + 1] = c2r_out(z[i].y * scale, p.relu);
        }
      }
    }
  } else {
    const int items2 = jvalid * ncols;
    for (int item = threadIdx.x; item < items2; item += blockDim.x) {
      const int jl = item / ncols, cl = item - jl * ncols;
      const float2* colp = s1 + (jl * PC) * ccpad + cl;
      float2 X[PC];
#pragma unroll
      for (int u = 0; u < PC; ++u) X[u] = colp[u * ccpad];
      float x[M];
      irfft_reg<M>(X, x);
      float* dst = p.out + (long long)r * p.out_sr + (long long)(j0 + jl) * p.out_sj + c0 + cl;
#pragma unroll
      for (int i = 0; i < M; ++i)
        if (i < p.crop) dst[(long long)i * p.crop] = c2r_out(x[i] * scale, p.relu);
    }
  }
}

}  // namespace fcb
