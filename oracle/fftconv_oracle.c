/*
 * fftconv CPU oracle -- TEST INFRASTRUCTURE ONLY.
 *
 * A plain-C restatement of the reference fftconv FFT-convolution path
 * (/root/reference/proj/include/fftconv/{fft,conv_fft,conv_direct,rng}.hpp).
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg may
 * load it, and only as the checker.  The B200 product path never links or
 * calls it: paper_1312_5851_b200 fails loudly when its CUDA library is
 * missing instead of falling back to anything here.
 *
 * Parity pinning: tests/test_oracle_golden.py checks this restatement
 * against golden vectors produced by the reference itself (compiled from its
 * own headers into oracle/_ref/, see oracle/Makefile and
 * tests/golden/make_golden.py) and against the reference's known-answer
 * tests (fft_test.cpp, conv_fft_test.cpp, conv_direct_test.cpp).
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define ORC_PI 3.14159265358979323846

enum {
  ORC_OK = 0,
  ORC_SIZE_ERROR = 1,
  ORC_SHAPE_ERROR = 2,
  ORC_CONFIG_ERROR = 3,
  ORC_CAPACITY_ERROR = 4,
  ORC_PLAN_ERROR = 5,
};

/* layer_config.hpp:11-17 */
static size_t orc_next_pow2(size_t n) {
  size_t m = 1;
  while (m < n) m <<= 1;
  return m;
}
static int orc_is_pow2(size_t n) { return n != 0 && (n & (n - 1)) == 0; }

/* rng.hpp:21-37: splitmix64 counter-based generator. */
uint64_t orc_splitmix64(uint64_t z) {
  z += 0x9e3779b97f4a7c15ULL;
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
  return z ^ (z >> 31);
}

double orc_uniform_at(uint64_t seed, uint64_t role, uint64_t index) {
  const uint64_t key = orc_splitmix64(seed ^ orc_splitmix64(role));
  const uint64_t h = orc_splitmix64(key ^ index);
  return 2.0 * ((double)(h >> 11) * 0x1.0p-53) - 1.0;
}

/* bench.hpp:164-183: random_verify_configs.  out[5*i..] = k, n, f, f', S. */
void orc_random_verify_configs(size_t count, uint64_t seed, uint64_t *out) {
  for (size_t i = 0; i < count; ++i) {
#define ORC_DRAW(salt, lo, hi)                                                    \
  ((lo) + (orc_splitmix64(seed ^ orc_splitmix64(i * 6364136223846793005ULL + (salt))) % \
           ((hi) - (lo) + 1)))
    const uint64_t image = ORC_DRAW(1, 2, 32);
    const uint64_t kernel = ORC_DRAW(2, 1, (image < 11 ? image : 11));
    const uint64_t in_maps = ORC_DRAW(3, 1, 8);
    const uint64_t out_maps = ORC_DRAW(4, 1, 8);
    const uint64_t batch = ORC_DRAW(5, 1, 4);
#undef ORC_DRAW
    out[5 * i + 0] = kernel;
    out[5 * i + 1] = image;
    out[5 * i + 2] = in_maps;
    out[5 * i + 3] = out_maps;
    out[5 * i + 4] = batch;
  }
}

size_t orc_next_pow2_export(size_t n) { return orc_next_pow2(n); }

#define T double
#define SFX _f64
#include "fftconv_oracle_impl.h"
#undef T
#undef SFX

#define T float
#define SFX _f32
#include "fftconv_oracle_impl.h"
#undef T
#undef SFX
