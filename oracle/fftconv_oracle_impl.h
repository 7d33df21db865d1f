/*
 * TEST INFRASTRUCTURE ONLY -- never linked into the product path.
 *
 * Type-generic body of the CPU oracle (included twice by fftconv_oracle.c,
 * once with T=double and once with T=float).  It restates, loop for loop,
 * the reference FFT-convolution algorithm:
 *
 *   FftPlan<T>::FftPlan / transform   /root/reference/proj/include/fftconv/fft.hpp:27-75
 *   detail::r2c_plane                 fft.hpp:160-179
 *   detail::c2r_plane                 fft.hpp:184-203
 *   ConvWorkspace<T>::forward         conv_fft.hpp:74-113
 *   ConvWorkspace<T>::grad_input      conv_fft.hpp:115-152
 *   ConvWorkspace<T>::grad_weight     conv_fft.hpp:154-206
 *   transform_planes / kernels        conv_fft.hpp:242-281
 *   inverse_planes                    conv_fft.hpp:285-304
 *   forward/grad_input/grad_weight_direct  conv_direct.hpp:24-127
 *
 * Required macros: T (scalar type), SFX (name suffix, e.g. _f64).
 */

#define CAT_(a, b) a##b
#define CAT(a, b) CAT_(a, b)
#define FN(name) CAT(name, SFX)
#define CPX FN(orc_cpx)

typedef struct {
  T re, im;
} CPX;

static inline CPX FN(cmul)(CPX a, CPX b) {
  CPX r;
  r.re = a.re * b.re - a.im * b.im;
  r.im = a.re * b.im + a.im * b.re;
  return r;
}
static inline CPX FN(cconj)(CPX a) {
  a.im = -a.im;
  return a;
}

/* FftPlan<T>: twiddles exp(-2*pi*i*j/m) computed in double then cast to T
 * (fft.hpp:27-32); bit-reversal table (fft.hpp:33-41). */
typedef struct {
  size_t m;
  CPX *tw;
  size_t *rev;
} FN(orc_plan);

static int FN(plan_init)(FN(orc_plan) * p, size_t m) {
  if (!orc_is_pow2(m)) return ORC_PLAN_ERROR;
  p->m = m;
  p->tw = (CPX *)malloc(sizeof(CPX) * (m / 2 + 1));
  p->rev = (size_t *)malloc(sizeof(size_t) * m);
  for (size_t j = 0; j < m / 2; ++j) {
    const double a = -2.0 * ORC_PI * (double)j / (double)m;
    p->tw[j].re = (T)cos(a);
    p->tw[j].im = (T)sin(a);
  }
  size_t bits = 0;
  while (((size_t)1 << bits) < m) ++bits;
  for (size_t i = 0; i < m; ++i) {
    size_t r = 0;
    for (size_t b = 0; b < bits; ++b)
      if (i & ((size_t)1 << b)) r |= (size_t)1 << (bits - 1 - b);
    p->rev[i] = r;
  }
  return ORC_OK;
}

static void FN(plan_free)(FN(orc_plan) * p) {
  free(p->tw);
  free(p->rev);
}

/* In-place radix-2 DIT; the inverse conjugates the twiddles and scales by
 * 1/m (fft.hpp:51-75). */
static void FN(transform)(const FN(orc_plan) * p, CPX *d, int inverse) {
  const size_t m = p->m;
  if (m == 1) return;
  for (size_t i = 0; i < m; ++i)
    if (i < p->rev[i]) {
      CPX t = d[i];
      d[i] = d[p->rev[i]];
      d[p->rev[i]] = t;
    }
  for (size_t len = 2; len <= m; len <<= 1) {
    const size_t half = len >> 1, stride = m / len;
    for (size_t start = 0; start < m; start += len)
      for (size_t j = 0; j < half; ++j) {
        CPX w = p->tw[j * stride];
        if (inverse) w = FN(cconj)(w);
        const CPX a = d[start + j];
        const CPX b = FN(cmul)(d[start + j + half], w);
        d[start + j].re = a.re + b.re;
        d[start + j].im = a.im + b.im;
        d[start + j + half].re = a.re - b.re;
        d[start + j + half].im = a.im - b.im;
      }
  }
  if (inverse) {
    const T scale = (T)1 / (T)m;
    for (size_t i = 0; i < m; ++i) {
      d[i].re *= scale;
      d[i].im *= scale;
    }
  }
}

/* detail::r2c_plane (fft.hpp:160-179): row pass over the src_rows real rows
 * keeping columns 0..m/2, then a column pass over the m/2+1 packed columns. */
static void FN(r2c_plane)(const FN(orc_plan) * p, const T *src, size_t src_rows,
                          size_t src_cols, CPX *out, CPX *line) {
  const size_t m = p->m, pc = m / 2 + 1;
  memset(out, 0, sizeof(CPX) * m * pc);
  for (size_t i = 0; i < src_rows; ++i) {
    for (size_t j = 0; j < src_cols; ++j) {
      line[j].re = src[i * src_cols + j];
      line[j].im = 0;
    }
    for (size_t j = src_cols; j < m; ++j) line[j].re = line[j].im = 0;
    FN(transform)(p, line, 0);
    memcpy(out + i * pc, line, sizeof(CPX) * pc);
  }
  for (size_t v = 0; v < pc; ++v) {
    for (size_t u = 0; u < m; ++u) line[u] = out[u * pc + v];
    FN(transform)(p, line, 0);
    for (size_t u = 0; u < m; ++u) out[u * pc + v] = line[u];
  }
}

/* detail::c2r_plane (fft.hpp:184-203): inverse columns in place, then only
 * out_rows rows rebuilt to full width by Hermitian symmetry and inverted;
 * only out_cols real values are written (top-left crop). */
static void FN(c2r_plane)(const FN(orc_plan) * p, CPX *half, T *dst,
                          size_t out_rows, size_t out_cols, CPX *line) {
  const size_t m = p->m, pc = m / 2 + 1;
  for (size_t v = 0; v < pc; ++v) {
    for (size_t u = 0; u < m; ++u) line[u] = half[u * pc + v];
    FN(transform)(p, line, 1);
    for (size_t u = 0; u < m; ++u) half[u * pc + v] = line[u];
  }
  for (size_t i = 0; i < out_rows; ++i) {
    for (size_t v = 0; v < pc; ++v) line[v] = half[i * pc + v];
    for (size_t v = pc; v < m; ++v) line[v] = FN(cconj)(half[i * pc + (m - v)]);
    FN(transform)(p, line, 1);
    for (size_t j = 0; j < out_cols; ++j) dst[i * out_cols + j] = line[j].re;
  }
}

/* Public single-plane entry points (used by the K1/K4 unit parity tests). */
int FN(orc_r2c_plane)(const T *src, size_t src_rows, size_t src_cols, size_t m,
                      T *out_interleaved) {
  FN(orc_plan) p;
  int st = FN(plan_init)(&p, m);
  if (st) return st;
  CPX *line = (CPX *)malloc(sizeof(CPX) * m);
  FN(r2c_plane)(&p, src, src_rows, src_cols, (CPX *)out_interleaved, line);
  free(line);
  FN(plan_free)(&p);
  return ORC_OK;
}

int FN(orc_c2r_plane)(const T *half_in, size_t m, T *dst, size_t out_rows,
                      size_t out_cols) {
  FN(orc_plan) p;
  int st = FN(plan_init)(&p, m);
  if (st) return st;
  const size_t pc = m / 2 + 1;
  CPX *half = (CPX *)malloc(sizeof(CPX) * m * pc);
  CPX *line = (CPX *)malloc(sizeof(CPX) * m);
  memcpy(half, half_in, sizeof(CPX) * m * pc);
  FN(c2r_plane)(&p, half, dst, out_rows, out_cols, line);
  free(half);
  free(line);
  FN(plan_free)(&p);
  return ORC_OK;
}

int FN(orc_fft_1d)(T *data_interleaved, size_t m, int inverse) {
  FN(orc_plan) p;
  int st = FN(plan_init)(&p, m);
  if (st) return st;
  FN(transform)(&p, (CPX *)data_interleaved, inverse);
  FN(plan_free)(&p);
  return ORC_OK;
}

/* transform_planes (conv_fft.hpp:242-261): every plane of a [S][maps][r][r]
 * tensor -> bins_out[bin][map][b] (row index map*S + b, `planes` rows). */
static void FN(transform_planes)(const FN(orc_plan) * p, const T *t, size_t S,
                                 size_t maps, size_t rows, CPX *bins_out) {
  const size_t m = p->m, bins = m * (m / 2 + 1), planes = S * maps;
#pragma omp parallel
  {
    CPX *half = (CPX *)malloc(sizeof(CPX) * bins);
    CPX *line = (CPX *)malloc(sizeof(CPX) * m);
#pragma omp for schedule(static)
    for (long long idx = 0; idx < (long long)planes; ++idx) {
      const size_t b = (size_t)idx / maps, f = (size_t)idx % maps;
      FN(r2c_plane)(p, t + (b * maps + f) * rows * rows, rows, rows, half, line);
      CPX *col = bins_out + f * S + b;
      for (size_t bin = 0; bin < bins; ++bin) col[bin * planes] = half[bin];
    }
    free(half);
    free(line);
  }
}

/* transform_kernels (conv_fft.hpp:263-281): w_bins[bin][o][f]. */
static void FN(transform_kernels)(const FN(orc_plan) * p, const T *w, size_t fout,
                                  size_t fin, size_t k, CPX *w_bins) {
  const size_t m = p->m, bins = m * (m / 2 + 1), planes = fout * fin;
#pragma omp parallel
  {
    CPX *half = (CPX *)malloc(sizeof(CPX) * bins);
    CPX *line = (CPX *)malloc(sizeof(CPX) * m);
#pragma omp for schedule(static)
    for (long long idx = 0; idx < (long long)planes; ++idx) {
      FN(r2c_plane)(p, w + (size_t)idx * k * k, k, k, half, line);
      CPX *col = w_bins + idx;
      for (size_t bin = 0; bin < bins; ++bin) col[bin * planes] = half[bin];
    }
    free(half);
    free(line);
  }
}

/* inverse_planes (conv_fft.hpp:285-304): gather a plane's bins, c2r + crop. */
static void FN(inverse_planes)(const FN(orc_plan) * p, CPX *bins_in, T *out,
                               size_t S, size_t maps, size_t out_rows) {
  const size_t m = p->m, bins = m * (m / 2 + 1), planes = S * maps;
#pragma omp parallel
  {
    CPX *half = (CPX *)malloc(sizeof(CPX) * bins);
    CPX *line = (CPX *)malloc(sizeof(CPX) * m);
#pragma omp for schedule(static)
    for (long long idx = 0; idx < (long long)planes; ++idx) {
      const size_t b = (size_t)idx / maps, f = (size_t)idx % maps;
      const CPX *col = bins_in + f * S + b;
      for (size_t bin = 0; bin < bins; ++bin) half[bin] = col[bin * planes];
      FN(c2r_plane)(p, half, out + (b * maps + f) * out_rows * out_rows, out_rows,
                    out_rows, line);
    }
    free(half);
    free(line);
  }
}

/* ConvWorkspace<T>::forward (conv_fft.hpp:74-113).
 * per bin: Y[o][b] += conj(W[o][f]) * X[f][b]. */
int FN(orc_forward_fft)(const T *x, const T *w, T *y, size_t S, size_t fin,
                        size_t fout, size_t n, size_t k) {
  if (k > n) return ORC_SIZE_ERROR;
  const size_t no = n - k + 1, m = orc_next_pow2(n), bins = m * (m / 2 + 1);
  FN(orc_plan) p;
  int st = FN(plan_init)(&p, m);
  if (st) return st;
  CPX *xb = (CPX *)malloc(sizeof(CPX) * bins * fin * S);
  CPX *wb = (CPX *)malloc(sizeof(CPX) * bins * fout * fin);
  CPX *yb = (CPX *)calloc(bins * fout * S, sizeof(CPX));
  FN(transform_planes)(&p, x, S, fin, n, xb);
  FN(transform_kernels)(&p, w, fout, fin, k, wb);
#pragma omp parallel for schedule(static)
  for (long long t = 0; t < (long long)bins; ++t) {
    const CPX *xt = xb + t * fin * S;
    const CPX *wt = wb + t * fout * fin;
    CPX *yt = yb + t * fout * S;
    for (size_t o = 0; o < fout; ++o) {
      CPX *yrow = yt + o * S;
      for (size_t f = 0; f < fin; ++f) {
        const CPX c = FN(cconj)(wt[o * fin + f]);
        const CPX *xrow = xt + f * S;
        for (size_t b = 0; b < S; ++b) {
          const CPX pr = FN(cmul)(c, xrow[b]);
          yrow[b].re += pr.re;
          yrow[b].im += pr.im;
        }
      }
    }
  }
  FN(inverse_planes)(&p, yb, y, S, fout, no);
  free(xb);
  free(wb);
  free(yb);
  FN(plan_free)(&p);
  return ORC_OK;
}

/* ConvWorkspace<T>::grad_input (conv_fft.hpp:115-152).
 * per bin: X[f][b] += W[o][f] * Y[o][b]; n = n' + k - 1. */
int FN(orc_grad_input_fft)(const T *gy, const T *w, T *gx, size_t S, size_t fin,
                           size_t fout, size_t no, size_t k) {
  const size_t n = no + k - 1, m = orc_next_pow2(n), bins = m * (m / 2 + 1);
  FN(orc_plan) p;
  int st = FN(plan_init)(&p, m);
  if (st) return st;
  CPX *xb = (CPX *)calloc(bins * fin * S, sizeof(CPX));
  CPX *wb = (CPX *)malloc(sizeof(CPX) * bins * fout * fin);
  CPX *yb = (CPX *)malloc(sizeof(CPX) * bins * fout * S);
  FN(transform_planes)(&p, gy, S, fout, no, yb);
  FN(transform_kernels)(&p, w, fout, fin, k, wb);
#pragma omp parallel for schedule(static)
  for (long long t = 0; t < (long long)bins; ++t) {
    CPX *xt = xb + t * fin * S;
    const CPX *wt = wb + t * fout * fin;
    const CPX *yt = yb + t * fout * S;
    for (size_t o = 0; o < fout; ++o) {
      const CPX *yrow = yt + o * S;
      for (size_t f = 0; f < fin; ++f) {
        const CPX c = wt[o * fin + f];
        CPX *xrow = xt + f * S;
        for (size_t b = 0; b < S; ++b) {
          const CPX pr = FN(cmul)(c, yrow[b]);
          xrow[b].re += pr.re;
          xrow[b].im += pr.im;
        }
      }
    }
  }
  FN(inverse_planes)(&p, xb, gx, S, fin, n);
  free(xb);
  free(wb);
  free(yb);
  FN(plan_free)(&p);
  return ORC_OK;
}

/* ConvWorkspace<T>::grad_weight (conv_fft.hpp:154-206).
 * per bin: W[o][f] += sum_b conj(GY[o][b]) * X[f][b]; k = n - n' + 1. */
int FN(orc_grad_weight_fft)(const T *gy, const T *x, T *gw, size_t S, size_t fin,
                            size_t fout, size_t n, size_t no) {
  if (no > n) return ORC_SIZE_ERROR;
  const size_t k = n - no + 1, m = orc_next_pow2(n), bins = m * (m / 2 + 1);
  FN(orc_plan) p;
  int st = FN(plan_init)(&p, m);
  if (st) return st;
  CPX *xb = (CPX *)malloc(sizeof(CPX) * bins * fin * S);
  CPX *wb = (CPX *)calloc(bins * fout * fin, sizeof(CPX));
  CPX *yb = (CPX *)malloc(sizeof(CPX) * bins * fout * S);
  FN(transform_planes)(&p, x, S, fin, n, xb);
  FN(transform_planes)(&p, gy, S, fout, no, yb);
#pragma omp parallel for schedule(static)
  for (long long t = 0; t < (long long)bins; ++t) {
    const CPX *xt = xb + t * fin * S;
    CPX *wt = wb + t * fout * fin;
    const CPX *yt = yb + t * fout * S;
    for (size_t o = 0; o < fout; ++o) {
      const CPX *yrow = yt + o * S;
      for (size_t f = 0; f < fin; ++f) {
        const CPX *xrow = xt + f * S;
        CPX acc = {0, 0};
        for (size_t b = 0; b < S; ++b) {
          const CPX pr = FN(cmul)(FN(cconj)(yrow[b]), xrow[b]);
          acc.re += pr.re;
          acc.im += pr.im;
        }
        wt[o * fin + f].re += acc.re;
        wt[o * fin + f].im += acc.im;
      }
    }
  }
  const size_t planes = fout * fin;
#pragma omp parallel
  {
    CPX *half = (CPX *)malloc(sizeof(CPX) * bins);
    CPX *line = (CPX *)malloc(sizeof(CPX) * m);
#pragma omp for schedule(static)
    for (long long idx = 0; idx < (long long)planes; ++idx) {
      for (size_t t = 0; t < bins; ++t) half[t] = wb[t * planes + idx];
      FN(c2r_plane)(&p, half, gw + (size_t)idx * k * k, k, k, line);
    }
    free(half);
    free(line);
  }
  free(xb);
  free(wb);
  free(yb);
  FN(plan_free)(&p);
  return ORC_OK;
}

/* forward_direct (conv_direct.hpp:24-55): valid cross-correlation. */
int FN(orc_forward_direct)(const T *x, const T *w, T *y, size_t S, size_t fin,
                           size_t fout, size_t n, size_t k) {
  if (k > n) return ORC_SIZE_ERROR;
  const size_t no = n - k + 1;
#pragma omp parallel for schedule(static)
  for (long long idx = 0; idx < (long long)(S * fout); ++idx) {
    const size_t b = (size_t)idx / fout, o = (size_t)idx % fout;
    T *out = y + (b * fout + o) * no * no;
    memset(out, 0, sizeof(T) * no * no);
    for (size_t f = 0; f < fin; ++f) {
      const T *in = x + (b * fin + f) * n * n;
      const T *ker = w + (o * fin + f) * k * k;
      for (size_t i = 0; i < no; ++i)
        for (size_t j = 0; j < no; ++j) {
          T acc = out[i * no + j];
          for (size_t u = 0; u < k; ++u)
            for (size_t v = 0; v < k; ++v) acc += in[(i + u) * n + j + v] * ker[u * k + v];
          out[i * no + j] = acc;
        }
    }
  }
  return ORC_OK;
}

/* grad_input_direct (conv_direct.hpp:61-90): full convolution as a scatter. */
int FN(orc_grad_input_direct)(const T *gy, const T *w, T *gx, size_t S, size_t fin,
                              size_t fout, size_t no, size_t k) {
  const size_t n = no + k - 1;
#pragma omp parallel for schedule(static)
  for (long long idx = 0; idx < (long long)(S * fin); ++idx) {
    const size_t b = (size_t)idx / fin, f = (size_t)idx % fin;
    T *out = gx + (b * fin + f) * n * n;
    memset(out, 0, sizeof(T) * n * n);
    for (size_t o = 0; o < fout; ++o) {
      const T *grad = gy + (b * fout + o) * no * no;
      const T *ker = w + (o * fin + f) * k * k;
      for (size_t i = 0; i < no; ++i)
        for (size_t j = 0; j < no; ++j) {
          const T g = grad[i * no + j];
          for (size_t u = 0; u < k; ++u)
            for (size_t v = 0; v < k; ++v) out[(i + u) * n + j + v] += g * ker[u * k + v];
        }
    }
  }
  return ORC_OK;
}

/* grad_weight_direct (conv_direct.hpp:95-127). */
int FN(orc_grad_weight_direct)(const T *gy, const T *x, T *gw, size_t S, size_t fin,
                               size_t fout, size_t n, size_t no) {
  if (no > n) return ORC_SIZE_ERROR;
  const size_t k = n - no + 1;
#pragma omp parallel for schedule(static)
  for (long long idx = 0; idx < (long long)(fout * fin); ++idx) {
    const size_t o = (size_t)idx / fin, f = (size_t)idx % fin;
    T *out = gw + (size_t)idx * k * k;
    memset(out, 0, sizeof(T) * k * k);
    for (size_t b = 0; b < S; ++b) {
      const T *grad = gy + (b * fout + o) * no * no;
      const T *in = x + (b * fin + f) * n * n;
      for (size_t u = 0; u < k; ++u)
        for (size_t v = 0; v < k; ++v) {
          T acc = out[u * k + v];
          for (size_t i = 0; i < no; ++i)
            for (size_t j = 0; j < no; ++j) acc += grad[i * no + j] * in[(i + u) * n + j + v];
          out[u * k + v] = acc;
        }
    }
  }
  return ORC_OK;
}

/* Selected output planes of forward_direct -- lets the GPU tests check a
 * subset of a layer too large for the full oracle (e.g. the wide layer). */
int FN(orc_forward_direct_planes)(const T *x, const T *w, T *y_planes, size_t S,
                                  size_t fin, size_t fout, size_t n, size_t k,
                                  const long long *plane_ids, size_t nplanes) {
  if (k > n) return ORC_SIZE_ERROR;
  const size_t no = n - k + 1;
#pragma omp parallel for schedule(dynamic)
  for (long long q = 0; q < (long long)nplanes; ++q) {
    const size_t b = (size_t)plane_ids[q] / fout, o = (size_t)plane_ids[q] % fout;
    T *out = y_planes + (size_t)q * no * no;
    memset(out, 0, sizeof(T) * no * no);
    if (b >= S) continue;
    for (size_t f = 0; f < fin; ++f) {
      const T *in = x + (b * fin + f) * n * n;
      const T *ker = w + (o * fin + f) * k * k;
      for (size_t i = 0; i < no; ++i)
        for (size_t j = 0; j < no; ++j) {
          T acc = out[i * no + j];
          for (size_t u = 0; u < k; ++u)
            for (size_t v = 0; v < k; ++v) acc += in[(i + u) * n + j + v] * ker[u * k + v];
          out[i * no + j] = acc;
        }
    }
  }
  return ORC_OK;
}

int FN(orc_grad_input_direct_planes)(const T *gy, const T *w, T *gx_planes, size_t S,
                                     size_t fin, size_t fout, size_t no, size_t k,
                                     const long long *plane_ids, size_t nplanes) {
  const size_t n = no + k - 1;
#pragma omp parallel for schedule(dynamic)
  for (long long q = 0; q < (long long)nplanes; ++q) {
    const size_t b = (size_t)plane_ids[q] / fin, f = (size_t)plane_ids[q] % fin;
    T *out = gx_planes + (size_t)q * n * n;
    memset(out, 0, sizeof(T) * n * n);
    if (b >= S) continue;
    for (size_t o = 0; o < fout; ++o) {
      const T *grad = gy + (b * fout + o) * no * no;
      const T *ker = w + (o * fin + f) * k * k;
      for (size_t i = 0; i < no; ++i)
        for (size_t j = 0; j < no; ++j) {
          const T g = grad[i * no + j];
          for (size_t u = 0; u < k; ++u)
            for (size_t v = 0; v < k; ++v) out[(i + u) * n + j + v] += g * ker[u * k + v];
        }
    }
  }
  return ORC_OK;
}

int FN(orc_grad_weight_direct_planes)(const T *gy, const T *x, T *gw_planes, size_t S,
                                      size_t fin, size_t fout, size_t n, size_t no,
                                      const long long *plane_ids, size_t nplanes) {
  if (no > n) return ORC_SIZE_ERROR;
  const size_t k = n - no + 1;
#pragma omp parallel for schedule(dynamic)
  for (long long q = 0; q < (long long)nplanes; ++q) {
    const size_t o = (size_t)plane_ids[q] / fin, f = (size_t)plane_ids[q] % fin;
    T *out = gw_planes + (size_t)q * k * k;
    memset(out, 0, sizeof(T) * k * k);
    if (o >= fout) continue;
    for (size_t b = 0; b < S; ++b) {
      const T *grad = gy + (b * fout + o) * no * no;
      const T *in = x + (b * fin + f) * n * n;
      for (size_t u = 0; u < k; ++u)
        for (size_t v = 0; v < k; ++v) {
          T acc = out[u * k + v];
          for (size_t i = 0; i < no; ++i)
            for (size_t j = 0; j < no; ++j) acc += grad[i * no + j] * in[(i + u) * n + j + v];
          out[u * k + v] = acc;
        }
    }
  }
  return ORC_OK;
}

/* fill_uniform (rng.hpp:41-47): static_cast<T> of the double draw. */
void FN(orc_fill_uniform)(T *out, size_t count, uint64_t seed, uint64_t role,
                          uint64_t stream) {
  const uint64_t r = role | (stream << 8);
#pragma omp parallel for schedule(static)
  for (long long i = 0; i < (long long)count; ++i) out[i] = (T)orc_uniform_at(seed, r, (uint64_t)i);
}

#undef CPX
#undef FN
#undef CAT
#undef CAT_
