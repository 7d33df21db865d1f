// K1 (r2c) and K4 (c2r) plane transforms for the FFT convolution path.
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
};

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
          dst[(long long)i * p.crop] = z[i].x * scale;
          if (has_b) dst[(long long)i * p.crop + 1] = z[i].y * scale;
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
        if (i < p.crop) dst[(long long)i * p.crop] = x[i] * scale;
    }
  }
}

// ======================================================================
// m in {4, 8, 16, 32}: warp-specialised persistent kernels.
//
// Each CTA loops over 16-plane groups.  Producer warps run pass 1 of group
// i+1 (global loads straight into registers, FFT, write the intermediate)
// while consumer warps run pass 2 of group i (read the intermediate, FFT,
// stream the result out), through a double-buffered shared-memory
// intermediate guarded by named barriers (FULL[b]: producers -> consumers,
// EMPTY[b]: consumers -> producers).  Loads of the next group therefore
// overlap the FFTs and stores of the current one instead of alternating
// within a CTA.
// ======================================================================
template <int M>
struct WsR2CTraits {
  static constexpr int G = 16;
  static constexpr int PC = M / 2 + 1;
  static constexpr int NPAIR = M / 2;
  static constexpr int P1_THREADS = ((G * NPAIR + 31) / 32) * 32;
  static constexpr int P2_THREADS = ((G * PC + 31) / 32) * 32;
  static constexpr int THREADS = P1_THREADS + P2_THREADS;
  static constexpr int CP = M + 1;  // intermediate row stride (float2), odd
  static constexpr int BUF = G * PC * CP;
  static constexpr int SMEM = 2 * BUF * 8;
};

enum : int { kBarFull0 = 1, kBarEmpty0 = 3 };  // named barrier ids (+buffer)

// One launch transforms both operands of an operator (A groups first, then
// B groups): the tail of one overlaps the other and a launch gap disappears.
struct R2CPair {
  R2CParams op[2];
  int n;  // 1 or 2 operands
};

// grid = persistent (<= groups), block = THREADS, smem = SMEM.
// Groups: g = r * (kpad/16) + jg.
template <int M>
__global__ void __launch_bounds__(WsR2CTraits<M>::THREADS, 1) r2c_ws_kernel(const R2CPair P) {
  using Tr = WsR2CTraits<M>;
  constexpr int G = Tr::G, PC = Tr::PC, NPAIR = Tr::NPAIR, CP = Tr::CP;
  constexpr int NT = Tr::THREADS;
  extern __shared__ __align__(16) float2 ws_s1[];  // [2][G][PC][CP]
  const int ngA = P.op[0].R * (P.op[0].kpad / G);
  const int ngroups = ngA + (P.n > 1 ? P.op[1].R * (P.op[1].kpad / G) : 0);
  pdl_wait();
  pdl_trigger();

  if (threadIdx.x < Tr::P1_THREADS) {
    // ---------------- producers: pass 1 (column pairs)
    const int item = threadIdx.x;
    const bool act = item < G * NPAIR;
    const int jl = item / NPAIR, cp = item - (item / NPAIR) * NPAIR;
    const int c = 2 * cp;
    int i = 0;
    for (int g = blockIdx.x; g < ngroups; g += gridDim.x, ++i) {
      const int b = i & 1;
      const int which = g >= ngA;
      const R2CParams& p = P.op[which];
      const int gl = g - which * ngA, ngj = p.kpad / G;
      const int r = gl / ngj, j0 = (gl - r * ngj) * G;
      const int src = p.src;
      float2 z[M];
      const bool ld = act && (j0 + jl) < p.J && c < src;
      const bool has_b = c + 1 < src;
      const float* col = p.in + (long long)r * p.in_sr + (long long)(j0 + jl) * p.in_sj + c;
#pragma unroll
      for (int row = 0; row < M; ++row) {
        z[row].x = (ld && row < src) ? __ldg(col + row * src) : 0.f;
        z[row].y = (ld && has_b && row < src) ? __ldg(col + row * src + 1) : 0.f;
      }
      fft_reg<M, false>(z);
      if (i >= 2) named_bar_sync(kBarEmpty0 + b, NT);
      if (act) {
        float2* dst = ws_s1 + b * Tr::BUF + (jl * PC) * CP + c;
        static_for<0, PC>([&](auto U) {
          constexpr int u = decltype(U)::value;
          const float2 zu = z[u];
          const float2 zc = cconj(z[(M - u) % M]);
          dst[u * CP] = make_float2(0.5f * (zu.x + zc.x), 0.5f * (zu.y + zc.y));
          const float2 d = csub(zu, zc);
          dst[u * CP + 1] = make_float2(0.5f * d.y, -0.5f * d.x);  // (zu - zc) / (2i)
        });
      }
      named_bar_arrive(kBarFull0 + b, NT);
    }
    // balance the consumers' final EMPTY arrivals
    for (int k = (i >= 2 ? i - 2 : 0); k < i; ++k) named_bar_sync(kBarEmpty0 + (k & 1), NT);
  } else {
    // ---------------- consumers: pass 2 (rows) + bin-major stores
    const int item = threadIdx.x - Tr::P1_THREADS;
    const bool act = item < G * PC;
    const int jl = item % G, u = item / G;
    int i = 0;
    for (int g = blockIdx.x; g < ngroups; g += gridDim.x, ++i) {
      const int b = i & 1;
      const int which = g >= ngA;
      const R2CParams& p = P.op[which];
      const int gl = g - which * ngA, ngj = p.kpad / G;
      const int r = gl / ngj, j0 = (gl - r * ngj) * G;
      const long long bstride = (long long)p.R * p.kpad;  // float2 per bin
      const float csign = p.conj ? -1.f : 1.f;
      named_bar_sync(kBarFull0 + b, NT);
      float2 w[M];
      if (act) {
        const float2* row = ws_s1 + b * Tr::BUF + (jl * PC + u) * CP;
#pragma unroll
        for (int cc = 0; cc < M; ++cc) w[cc] = row[cc];
      }
      named_bar_arrive(kBarEmpty0 + b, NT);
      if (act) {
        fft_reg<M, false>(w);
        float2* o = reinterpret_cast<float2*>(p.out) + (long long)r * p.kpad + j0 + jl +
                    (long long)(u * M) * bstride;
#pragma unroll
        for (int v = 0; v < M; ++v) {
          *o = make_float2(w[v].x, csign * w[v].y);
          o += bstride;
        }
      }
    }
  }
}

template <int M>
struct WsC2RTraits {
  static constexpr int G = 16;
  static constexpr int PC = M / 2 + 1;
  static constexpr int P1_THREADS = ((G * PC + 31) / 32) * 32;
  static constexpr int P2_THREADS = ((G * (M / 2) + 31) / 32) * 32;
  static constexpr int THREADS = P1_THREADS + P2_THREADS;
  static constexpr int CP = M + 1;  // odd
  static constexpr int BUF = G * PC * CP;
  static constexpr int SMEM = 2 * BUF * 8;
};

// grid = persistent, groups g = r * ceil(J/16) + jg.  crop <= M.
template <int M>
__global__ void __launch_bounds__(WsC2RTraits<M>::THREADS, 1) c2r_ws_kernel(const C2RParams p) {
  using Tr = WsC2RTraits<M>;
  constexpr int G = Tr::G, PC = Tr::PC, CP = Tr::CP;
  constexpr int NT = Tr::THREADS;
  extern __shared__ __align__(16) float2 ws_s1[];  // [2][G][PC][CP]
  pdl_wait();
  pdl_trigger();
  const int ngj = (p.J + G - 1) / G;
  const int ngroups = p.R * ngj;
  const int crop = p.crop;
  const long long bstride = (long long)p.R * p.ld;  // float2 per bin

  if (threadIdx.x < Tr::P1_THREADS) {
    // ---------------- producers: inverse row FFT over v (lanes = planes)
    const int item = threadIdx.x;
    const bool act = item < G * PC;
    const int jl = item % G, u = item / G;
    int i = 0;
    for (int g = blockIdx.x; g < ngroups; g += gridDim.x, ++i) {
      const int b = i & 1;
      const int r = g / ngj, j0 = (g - r * ngj) * G;
      const bool ld = act && (j0 + jl) < p.J;
      float2 z[M];
      const float2* srcp = reinterpret_cast<const float2*>(p.in) + (long long)r * p.ld + j0 + jl +
                           (long long)(u * M) * bstride;
#pragma unroll
      for (int v = 0; v < M; ++v) {
        z[v] = ld ? __ldg(srcp) : make_float2(0.f, 0.f);
        srcp += bstride;
      }
      fft_reg<M, true>(z);
      if (i >= 2) named_bar_sync(kBarEmpty0 + b, NT);
      if (act) {
        float2* dst = ws_s1 + b * Tr::BUF + (jl * PC + u) * CP;
#pragma unroll
        for (int cc = 0; cc < M; ++cc)
          if (cc < crop) dst[cc] = z[cc];
      }
      named_bar_arrive(kBarFull0 + b, NT);
    }
    for (int k = (i >= 2 ? i - 2 : 0); k < i; ++k) named_bar_sync(kBarEmpty0 + (k & 1), NT);
  } else {
    // ---------------- consumers: Hermitian c2r over u, two columns per FFT
    const int item = threadIdx.x - Tr::P1_THREADS;
    const int npair = (crop + 1) >> 1;
    const bool act = item < G * npair;
    const int jl = act ? item / npair : 0, cp = act ? item - (item / npair) * npair : 0;
    const int cl = 2 * cp;
    const bool has_b = cl + 1 < crop;
    const float scale = p.scale;
    int i = 0;
    for (int g = blockIdx.x; g < ngroups; g += gridDim.x, ++i) {
      const int b = i & 1;
      const int r = g / ngj, j0 = (g - r * ngj) * G;
      named_bar_sync(kBarFull0 + b, NT);
      float2 zz[M];
      if (act) {
        const float2* colp = ws_s1 + b * Tr::BUF + (jl * PC) * CP + cl;
        static_for<0, PC>([&](auto U) {
          constexpr int uu = decltype(U)::value;
          float2 a = colp[uu * CP];
          float2 bb = has_b ? colp[uu * CP + 1] : make_float2(0.f, 0.f);
          if constexpr (uu == 0 || 2 * uu == M) {  // c2r ignores these imaginary parts
            a.y = 0.f;
            bb.y = 0.f;
          }
          zz[uu] = make_float2(a.x - bb.y, a.y + bb.x);  // a + i b
          if constexpr (uu != 0 && 2 * uu != M) zz[M - uu] = make_float2(a.x + bb.y, bb.x - a.y);
        });
      }
      named_bar_arrive(kBarEmpty0 + b, NT);
      if (act && (j0 + jl) < p.J) {
        fft_reg<M, true>(zz);
        float* dst = p.out + (long long)r * p.out_sr + (long long)(j0 + jl) * p.out_sj + cl;
#pragma unroll
        for (int row = 0; row < M; ++row) {
          if (row < crop) {
            dst[0] = zz[row].x * scale;
            if (has_b) dst[1] = zz[row].y * scale;
            dst += crop;
          }
        }
      }
    }
  }
}

// ======================================================================
// m = 64: warp-specialised persistent kernels, 4 planes per group (a 64x33
// intermediate per plane; double-buffered that is 137 KB).  Pass-1 columns
// use the half-length real FFT; 64-point complex row FFTs are split into
// two 32-point halves by one decimation-in-frequency stage so a thread
// holds 32 complex values.
// ======================================================================
struct Ws64 {
  static constexpr int M = 64, G = 4, PC = 33, CP = 65;
  static constexpr int BUF = G * PC * CP;             // float2 per buffer
  static constexpr int SMEM = 2 * BUF * 8;
  static constexpr int COLS_THREADS = G * M;          // 256: one column per thread
  static constexpr int ROWS_THREADS = ((G * PC * 2 + 31) / 32) * 32;  // 264 -> 288
  static constexpr int THREADS = COLS_THREADS + ROWS_THREADS;
};

// grid = persistent, groups g = r * (kpad/4) + jg.
__global__ void __maxnreg__(96) r2c_ws64_kernel(const R2CPair P) {
  constexpr int M = 64, G = Ws64::G, PC = Ws64::PC, CP = Ws64::CP, NT = Ws64::THREADS;
  extern __shared__ __align__(16) float2 ws_s1[];  // [2][G][PC][CP]
  const int ngA = P.op[0].R * (P.op[0].kpad / G);
  const int ngroups = ngA + (P.n > 1 ? P.op[1].R * (P.op[1].kpad / G) : 0);
  pdl_wait();
  pdl_trigger();
  if (threadIdx.x < Ws64::COLS_THREADS) {
    // ---------------- producers: one real column per thread
    const int jl = threadIdx.x / M, c = threadIdx.x % M;
    int i = 0;
    for (int g = blockIdx.x; g < ngroups; g += gridDim.x, ++i) {
      const int b = i & 1;
      const int which = g >= ngA;
      const R2CParams& p = P.op[which];
      const int gl = g - which * ngA, ngj = p.kpad / G;
      const int r = gl / ngj, j0 = (gl - r * ngj) * G;
      const int src = p.src;
      const bool ld = (j0 + jl) < p.J && c < src;
      const float* col = p.in + (long long)r * p.in_sr + (long long)(j0 + jl) * p.in_sj + c;
      float x[M];
#pragma unroll
      for (int row = 0; row < M; ++row) x[row] = (ld && row < src) ? __ldg(col + row * src) : 0.f;
      if (i >= 2) named_bar_sync(kBarEmpty0 + b, NT);
      float2* dst = ws_s1 + b * Ws64::BUF + (jl * PC) * CP + c;
      rfft_emit<M>(x, [&](int u, float2 v) { dst[u * CP] = v; });
      named_bar_arrive(kBarFull0 + b, NT);
    }
    for (int k = (i >= 2 ? i - 2 : 0); k < i; ++k) named_bar_sync(kBarEmpty0 + (k & 1), NT);
  } else {
    // ---------------- consumers: (plane, u, half) -> 32-point FFT -> v = 2i + h
    const int item = threadIdx.x - Ws64::COLS_THREADS;
    const bool act = item < G * PC * 2;
    const int jl = item % G, h = (item / G) & 1, u = item / (2 * G);
    int i = 0;
    for (int g = blockIdx.x; g < ngroups; g += gridDim.x, ++i) {
      const int b = i & 1;
      const int which = g >= ngA;
      const R2CParams& p = P.op[which];
      const int gl = g - which * ngA, ngj = p.kpad / G;
      const int r = gl / ngj, j0 = (gl - r * ngj) * G;
      const long long bstride = (long long)p.R * p.kpad;  // float2 per bin
      const float csign = p.conj ? -1.f : 1.f;
      named_bar_sync(kBarFull0 + b, NT);
      float2 z[32];
      if (act) {
        const float2* row = ws_s1 + b * Ws64::BUF + (jl * PC + u) * CP;
        static_for<0, 32>([&](auto Cc) {
          constexpr int cc = decltype(Cc)::value;
          const float2 a0 = row[cc], a1 = row[cc + 32];
          if (h == 0) {
            z[cc] = cadd(a0, a1);
          } else {
            if constexpr (cc == 0) z[cc] = csub(a0, a1);
            else z[cc] = cmul(csub(a0, a1), tw128c<false, cc * 2>());
          }
        });
      }
      named_bar_arrive(kBarEmpty0 + b, NT);
      if (act) {
        fft_reg<32, false>(z);
        float2* o = reinterpret_cast<float2*>(p.out) + (long long)r * p.kpad + j0 + jl +
                    (long long)(u * M + h) * bstride;
        const long long st2 = 2 * bstride;
#pragma unroll
        for (int v = 0; v < 32; ++v) {
          *o = make_float2(z[v].x, csign * z[v].y);
          o += st2;
        }
      }
    }
  }
}

// grid = persistent, groups g = r * ceil(J/4) + jg.
__global__ void __maxnreg__(96) c2r_ws64_kernel(const C2RParams p) {
  constexpr int M = 64, G = Ws64::G, PC = Ws64::PC, CP = Ws64::CP, NT = Ws64::THREADS;
  extern __shared__ __align__(16) float2 ws_s1[];  // [2][G][PC][CP]
  pdl_wait();
  pdl_trigger();
  const int ngj = (p.J + G - 1) / G;
  const int ngroups = p.R * ngj;
  const int crop = p.crop;
  const long long bstride = (long long)p.R * p.ld;  // float2 per bin
  if (threadIdx.x >= Ws64::COLS_THREADS) {
    // ---------------- producers: (plane, u, half) inverse 64-point row FFT
    const int item = threadIdx.x - Ws64::COLS_THREADS;
    const bool act = item < G * PC * 2;
    const int jl = item % G, h = (item / G) & 1, u = item / (2 * G);
    int i = 0;
    for (int g = blockIdx.x; g < ngroups; g += gridDim.x, ++i) {
      const int b = i & 1;
      const int r = g / ngj, j0 = (g - r * ngj) * G;
      const bool ld = act && (j0 + jl) < p.J;
      const float2* srcp = reinterpret_cast<const float2*>(p.in) + (long long)r * p.ld + j0 + jl +
                           (long long)(u * M) * bstride;
      float2 z[32];
      static_for<0, 32>([&](auto Vv) {
        constexpr int v = decltype(Vv)::value;
        const float2 a0 = ld ? __ldg(srcp + v * bstride) : make_float2(0.f, 0.f);
        const float2 a1 = ld ? __ldg(srcp + (v + 32) * bstride) : make_float2(0.f, 0.f);
        if (h == 0) {
          z[v] = cadd(a0, a1);
        } else {
          if constexpr (v == 0) z[v] = csub(a0, a1);
          else z[v] = cmul(csub(a0, a1), tw128c<true, v * 2>());
        }
      });
      fft_reg<32, true>(z);
      if (i >= 2) named_bar_sync(kBarEmpty0 + b, NT);
      if (act) {
        float2* dst = ws_s1 + b * Ws64::BUF + (jl * PC + u) * CP;
#pragma unroll
        for (int k = 0; k < 32; ++k)
          if (2 * k + h < crop) dst[2 * k + h] = z[k];
      }
      named_bar_arrive(kBarFull0 + b, NT);
    }
    for (int k = (i >= 2 ? i - 2 : 0); k < i; ++k) named_bar_sync(kBarEmpty0 + (k & 1), NT);
  } else {
    // ---------------- consumers: one Hermitian column per thread
    const int jl = threadIdx.x / M, c = threadIdx.x % M;
    const bool act = c < crop;
    const float scale = p.scale;
    int i = 0;
    for (int g = blockIdx.x; g < ngroups; g += gridDim.x, ++i) {
      const int b = i & 1;
      const int r = g / ngj, j0 = (g - r * ngj) * G;
      named_bar_sync(kBarFull0 + b, NT);
      float2 X[PC];
      if (act) {
        const float2* colp = ws_s1 + b * Ws64::BUF + (jl * PC) * CP + c;
#pragma unroll
        for (int uu = 0; uu < PC; ++uu) X[uu] = colp[uu * CP];
      }
      named_bar_arrive(kBarEmpty0 + b, NT);
      if (act && (j0 + jl) < p.J) {
        float* dst = p.out + (long long)r * p.out_sr + (long long)(j0 + jl) * p.out_sj + c;
        irfft_emit<M>(X, [&](int row, float v) {
          if (row < crop) dst[row * crop] = v * scale;
        });
      }
    }
  }
}

}  // namespace fcb
