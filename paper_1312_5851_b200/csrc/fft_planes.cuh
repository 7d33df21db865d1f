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

#include "twiddles.cuh"

namespace fcb {

constexpr int kPlaneGroup = 16;  // planes (K indices) per CTA: 16 complex = 128 B

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

// exp(-+2 pi i k / 128) from the constant table (index folds to an immediate
// constant-bank operand once loops are unrolled).
template <bool INV>
__device__ __forceinline__ float2 tw128(int k) {
  float2 w = c_tw128[k & 127];
  if (INV) w.y = -w.y;
  return w;
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
    return cmul(v, tw128<INV>(J * (128 / LEN)));
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
      else wo = cmul(o, tw128<false>(k * (128 / N)));
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
      if constexpr (k != 0) o = cmul(o, tw128<true>(k * (128 / N)));
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
};

// grid = (kpad/16, R, ceil((M/2+1)/UC)), block = 256.
// smem = 16 * UC * cpad * sizeof(float2).
template <int M, int UC, int SPLIT>
__global__ void __launch_bounds__(256) r2c_planes_kernel(const R2CParams p) {
  constexpr int PC = M / 2 + 1;
  constexpr int G = kPlaneGroup;
  extern __shared__ float2 s1[];  // [G][UC][cpad]
  const int r = blockIdx.y;
  const int j0 = blockIdx.x * G;
  const int u0 = blockIdx.z * UC;
  const int src = p.src, cpad = p.cpad;
  const int jvalid = min(G, p.J - j0);

  // Pass 1: one thread per (plane, column): zero-padded real column FFT
  // over the rows (coalesced row loads across lanes), keep u in the chunk.
  const int items1 = jvalid * src;
  for (int item = threadIdx.x; item < items1; item += blockDim.x) {
    const int jl = item / src, c = item - jl * src;
    const float* col = p.in + (long long)r * p.in_sr + (long long)(j0 + jl) * p.in_sj + c;
    float x[M];
#pragma unroll
    for (int i = 0; i < M; ++i) x[i] = (i < src) ? __ldg(col + (long long)i * src) : 0.f;
    float2* dst = s1 + (jl * UC) * cpad + c;
    rfft_emit<M>(x, [&](int u, float2 v) {
      const int ul = u - u0;
      if (ul >= 0 && ul < UC) dst[ul * cpad] = v;
    });
  }
  __syncthreads();

  // Pass 2: one thread per (plane, u[, half]): complex row FFT over the
  // columns, written bin-major with 16 planes (128 B) per bin per row.
  const int urows = min(UC, PC - u0);
  const int items2 = G * SPLIT * urows;
  const long long rstride = (long long)p.R * p.kpad * 2;  // floats per bin
  float* outbase = p.out + ((long long)r * p.kpad + j0) * 2;
  for (int item = threadIdx.x; item < items2; item += blockDim.x) {
    const int jl = item % G;
    const int rest = item / G;
    const int h = rest % SPLIT;
    const int ul = rest / SPLIT;
    const int u = u0 + ul;
    float2* o = reinterpret_cast<float2*>(outbase + 2 * jl);
    if (jl >= jvalid) {
#pragma unroll 4
      for (int i = 0; i < M / SPLIT; ++i)
        o[(long long)(u * M + i * SPLIT + h) * (rstride / 2)] = make_float2(0.f, 0.f);
      continue;
    }
    const float2* row = s1 + (jl * UC + ul) * cpad;
    constexpr int NS = M / SPLIT;
    float2 z[NS];
    if constexpr (SPLIT == 1) {
#pragma unroll
      for (int c = 0; c < M; ++c) z[c] = (c < src) ? row[c] : make_float2(0.f, 0.f);
    } else {
      static_assert(SPLIT == 2, "split");
      // decimation in frequency: outputs v = 2i + h
#pragma unroll
      for (int c = 0; c < NS; ++c) {
        const float2 a = (c < src) ? row[c] : make_float2(0.f, 0.f);
        const float2 b = (c + NS < src) ? row[c + NS] : make_float2(0.f, 0.f);
        if (h == 0) z[c] = cadd(a, b);
        else z[c] = (c == 0) ? csub(a, b) : cmul(csub(a, b), tw128<false>(c * (128 / M)));
      }
    }
    fft_reg<NS, false>(z);
#pragma unroll
    for (int i = 0; i < NS; ++i) o[(long long)(u * M + i * SPLIT + h) * (rstride / 2)] = z[i];
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
  float scale;  // 1 / m^2
};

// grid = (ceil(J/16), R, ceil(crop/cc)), block = 256.
// smem = 16 * (M/2+1) * ccpad * sizeof(float2).
template <int M, int SPLIT>
__global__ void __launch_bounds__(256) c2r_planes_kernel(const C2RParams p) {
  constexpr int PC = M / 2 + 1;
  constexpr int G = kPlaneGroup;
  constexpr int NS = M / SPLIT;
  extern __shared__ float2 s1[];  // [G][PC][ccpad]
  const int r = blockIdx.y;
  const int j0 = blockIdx.x * G;
  const int c0 = blockIdx.z * p.cc;
  const int ncols = min(p.cc, p.crop - c0);
  const int jvalid = min(G, p.J - j0);
  const int ccpad = p.ccpad;
  const long long bstride = (long long)p.R * p.J;  // float2 per bin
  const float2* inbase = reinterpret_cast<const float2*>(p.in) + (long long)r * p.J + j0;

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
#pragma unroll
      for (int v = 0; v < NS; ++v) {
        const float2 a = __ldg(src + (long long)v * bstride);
        const float2 b = __ldg(src + (long long)(v + NS) * bstride);
        if (h == 0) z[v] = cadd(a, b);
        else z[v] = (v == 0) ? csub(a, b) : cmul(csub(a, b), tw128<true>(v * (128 / M)));
      }
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

  // Pass 2: per (plane, column) Hermitian c2r over u, write the cropped
  // rows; lanes = consecutive columns -> contiguous row segments.
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
      if (i < p.crop) dst[(long long)i * p.crop] = x[i] * p.scale;
  }
}

}  // namespace fcb
