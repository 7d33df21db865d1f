// fftconv_b200: B200-native FFT convolution layer (fprop / bprop / accGrad)
// behind the reference ConvWorkspace operator interface.
//
// Host side of the C ABI declared in include/fftconv_b200.h.  Each operator
// is four launches on the caller's stream:
//   K1 r2c(operand A) -> K1 r2c(operand B) -> K3 per-bin complex GEMM
//   (tcgen05, 3xTF32) -> K4 c2r + crop.
// Reference call stacks this replaces: SURVEY.md section 3 (A)-(C);
// ConvWorkspace<T>::forward/grad_input/grad_weight at conv_fft.hpp:74-206.
#include <cuda.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>
#include <dlfcn.h>
#include <nccl.h>  // types only: libnccl is loaded at run time (nccl_api)

#include <algorithm>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <atomic>
#include <functional>
#include <map>
#include <mutex>
#include <unordered_map>
#include <stdexcept>
#include <string>
#include <vector>

#include "../../include/fftconv_b200.h"
#include "cgemm_tcgen05.cuh"
#include "fft_planes.cuh"
#include "fft_large.cuh"
#include "fft_tma.cuh"
#include "fft_small.cuh"
#include "layers.cuh"

namespace fcb {

// ------------------------------------------------------------ errors
struct Error : std::runtime_error {
  int code;
  Error(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};

static thread_local std::string g_last_error;

#define FCB_CUDA(call)                                                                     \
  do {                                                                                     \
    cudaError_t e_ = (call);                                                               \
    if (e_ != cudaSuccess)                                                                 \
      throw Error(FFTCONV_B200_CUDA_ERROR,                                                 \
                  std::string(#call) + ": " + cudaGetErrorString(e_));                     \
  } while (0)

// ------------------------------------------------------------ layer maths
static size_t next_pow2(size_t n) {
  size_t m = 1;
  while (m < n) m <<= 1;
  return m;
}
static size_t round_up(size_t v, size_t a) { return (v + a - 1) / a * a; }

// LayerConfig::validate (layer_config.hpp:32-39)
static void validate_cfg(const fftconv_b200_layer& c) {
  if (c.kernel == 0 || c.image == 0 || c.in_maps == 0 || c.out_maps == 0 || c.batch == 0)
    throw Error(FFTCONV_B200_CONFIG_ERROR, "layer config: all parameters must be >= 1");
  if (c.kernel > c.image)
    throw Error(FFTCONV_B200_CONFIG_ERROR, "layer config: kernel " + std::to_string(c.kernel) +
                                               " exceeds image " + std::to_string(c.image));
}

enum Pass { kFprop = 0, kBprop = 1, kAccGrad = 2 };

// Padded K (complex per operand row of a spectrum F[t][row][2 kpad]): the
// GEMM consumes K in chunks of 16 (one 128-B SW128 row), but a K below 16
// (a first layer's f = 3 input maps) is padded only to 4 or 8 -- the GEMM's
// TMA box reads past the row end and the copy engine zero-fills it, so the
// spectra carry 1.3x instead of 5.3x their bytes at f = 3.  The one-pass
// m <= 2 kernels write whole 16-plane lines and keep 16.
static size_t kpad_for(size_t K, size_t m) {
  if (m <= 2) return round_up(K, 16);
  return K <= 4 ? 4 : K <= 8 ? 8 : round_up(K, 16);
}

// Device bytes (floats) each pass needs in the three frequency buffers.
struct PassNeed {
  size_t a, b, d;
};
static PassNeed pass_need(Pass pass, size_t S, size_t f, size_t fo, size_t m) {
  const size_t bins = m * (m / 2 + 1);
  switch (pass) {
    case kFprop:  // D is [fo][S] or, swapped, [S][fo]
      return {bins * S * 2 * kpad_for(f, m), bins * fo * 2 * kpad_for(f, m),
              bins * 2 * std::max(fo * round_up(S, 16), S * round_up(fo, 16))};
    case kBprop:
      return {bins * S * 2 * kpad_for(fo, m), bins * f * 2 * kpad_for(fo, m),
              bins * 2 * std::max(f * round_up(S, 16), S * round_up(f, 16))};
    default:
      return {bins * fo * 2 * kpad_for(S, m), bins * f * 2 * kpad_for(S, m),
              bins * f * 2 * round_up(fo, 16)};
  }
}

// Product-spectrum layouts written by the GEMM epilogue:
//   kBinMajor   P[t][n][ld]         (ld >= M, even) -- m = 64 K4 and the
//                                    debug hook
//   kGroupMajor P[n][m/G][t][G]     every G-plane K4 group (G = the K4
//                                    group size) is one contiguous block
//                                    (one bulk load instead of bins
//                                    scattered rows)
enum OutLayout { kBinMajor = 0, kGroupMajor = 1 };

// ------------------------------------------------------------ driver API
static PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) ==
            cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  });
  if (!fn) throw Error(FFTCONV_B200_CUDA_ERROR, "cuTensorMapEncodeTiled unavailable");
  return fn;
}

// 3-D fp32 map over F[t][rows][2*kpad]; box {32 floats, box_rows, 1}, SW128.
static CUtensorMap make_operand_map(const float* base, size_t kpad, size_t rows, size_t bins,
                                    uint32_t box_rows) {
  CUtensorMap m;
#ifdef FCB_GEMM_LAYOUT_EXP  // timing experiment only: chunk-contiguous reads of the same bytes
  const cuuint64_t dims[3] = {32, rows * (kpad / 16), bins};
  const cuuint64_t strides[2] = {128, rows * 2 * kpad * sizeof(float)};
#else
  const cuuint64_t dims[3] = {2 * kpad, rows, bins};
  const cuuint64_t strides[2] = {2 * kpad * sizeof(float), rows * 2 * kpad * sizeof(float)};
#endif
  const cuuint32_t box[3] = {32, box_rows, 1};
  const cuuint32_t estr[3] = {1, 1, 1};
  CUresult r = encode_fn()(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, const_cast<float*>(base), dims,
                           strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                           CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                           CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS)
    throw Error(FFTCONV_B200_CUDA_ERROR, "cuTensorMapEncodeTiled failed: " + std::to_string(r));
  return m;
}

// ------------------------------------------------------------ launchers
struct DevInfo {
  int sms = 148;
  int max_smem_optin = 232448;
};
static DevInfo dev_info(int device) {
  DevInfo d;
  cudaDeviceGetAttribute(&d.sms, cudaDevAttrMultiProcessorCount, device);
  cudaDeviceGetAttribute(&d.max_smem_optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, device);
  return d;
}

// Every launch goes through cudaLaunchKernelEx with programmatic stream
// serialisation: a kernel's CTAs may start (prologue: smem carve-up, mbarrier
// init, TMEM alloc, descriptor prefetch) while the previous kernel on the
// stream drains; each kernel calls griddepcontrol.wait before touching
// global memory, so ordering is unchanged.
template <typename... KArgs, typename... Args>
static void launch_pdl(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem,
                       cudaStream_t st, Args&&... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  FCB_CUDA(cudaLaunchKernelEx(&cfg, kern, std::forward<Args>(args)...));
}

// Per-kernel host-side caches, keyed by (device, kernel address): the
// shared-memory opt-in is a per-device attribute, and several kernels share a
// signature, so a function-local static would be shared.
static std::mutex g_kcache_mu;
static std::map<std::pair<int, const void*>, int> g_smem_done;

// Opt a kernel into > 48 KB dynamic shared memory (once per device and size).
template <typename K>
static void smem_optin(K kern, int bytes) {
  if (bytes <= 48 * 1024) return;
  int dev = 0;
  FCB_CUDA(cudaGetDevice(&dev));
  std::lock_guard<std::mutex> lk(g_kcache_mu);
  int& done = g_smem_done[{dev, reinterpret_cast<const void*>(kern)}];
  if (bytes > done) {
    FCB_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes));
    done = bytes;
  }
}


// ---- K1 / K4 dispatch ----------------------------------------------------
// m in {4..64}: the TMA-pipelined kernels (fft_tma.cuh).  m in {1, 2} (tiny
// non-pow2-padded planes of the verification sweeps): the simple
// one-pass-per-CTA plane kernels (fft_planes.cuh).

static void size_unsupported(size_t m) {
  throw Error(FFTCONV_B200_SIZE_ERROR,
              "fft size " + std::to_string(m) + " not supported by the B200 kernels (max 128)");
}

template <int M>
static void launch_r2c_small(const R2CParams& p, cudaStream_t st) {
  using Tr = PlaneTraits<M>;
  auto kern = r2c_planes_kernel<M>;
  const size_t smem = (size_t)Tr::G * Tr::UC * p.cpad * sizeof(float2);
  smem_optin(kern, (int)smem);
  dim3 grid(p.kpad / Tr::G, p.R, (Tr::PC + Tr::UC - 1) / Tr::UC);
  launch_pdl(kern, grid, dim3(Tr::THREADS), smem, st, p);
}

template <int M>
static void launch_c2r_small(C2RParams p, cudaStream_t st) {
  using Tr = PlaneTraits<M>;
  p.cc = p.crop;
  p.ccpad = (p.cc % 2) ? p.cc : p.cc + 1;
  auto kern = c2r_planes_kernel<M>;
  const size_t smem = (size_t)Tr::G * Tr::PC * p.ccpad * sizeof(float2);
  smem_optin(kern, (int)smem);
  dim3 grid((p.J + Tr::G - 1) / Tr::G, p.R, 1);
  launch_pdl(kern, grid, dim3(Tr::THREADS), smem, st, p);
}

// 3-D fp32 map over a bin-major spectrum X[t][R][2*ld] (complex, ld even)
// with box {2g floats, 1 row, bt bins}: the transform kernels' tiles.
static CUtensorMap make_bin_map(const float* base, size_t ld, size_t R, size_t bins, uint32_t g,
                                uint32_t bt) {
  CUtensorMap t;
  const cuuint64_t dims[3] = {2 * ld, R, bins};
  const cuuint64_t strides[2] = {2 * ld * sizeof(float), R * 2 * ld * sizeof(float)};
  const cuuint32_t box[3] = {2 * g, 1, bt};
  const cuuint32_t estr[3] = {1, 1, 1};
  CUresult r = encode_fn()(&t, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, const_cast<float*>(base), dims,
                           strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                           CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
                           CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS)
    throw Error(FFTCONV_B200_CUDA_ERROR, "cuTensorMapEncodeTiled (spectrum) failed: " + std::to_string(r));
  return t;
}

template <int M>
static void launch_r2c_tma(const R2CPair& P, const DevInfo& di, cudaStream_t st) {
  using T = TR2C<M>;
  auto kern = r2c_tma_kernel<M>;
  smem_optin(kern, T::SMEM);
  int groups = 0;
  for (int i = 0; i < P.n; ++i) groups += P.op[i].R * ((P.op[i].kpad + T::G - 1) / T::G);
  const int grid = std::max(1, std::min(groups, di.sms));
  const size_t bins = (size_t)T::BINS;
  CUtensorMap tm[2];
  for (int i = 0; i < 2; ++i) {
    const R2CParams& p = P.op[i < P.n ? i : 0];
    tm[i] = make_bin_map(p.out, p.kpad, p.R, bins, T::G, T::BT);
  }
  launch_pdl(kern, dim3(grid), dim3(T::THREADS), T::SMEM, st, P, tm[0], tm[1]);
}

// Both forward transforms of an operator (one launch at m >= 4; operand A's
// groups first, then B's).  Returns the number of launches.
static int launch_r2c_both(size_t m, const R2CParams& a, const R2CParams& b, cudaStream_t st,
                           const DevInfo& di, unsigned long long* tspan = nullptr) {
  R2CPair P{{a, b}, 2};
  P.tspan = tspan;
  switch (m) {
    case 1: launch_r2c_small<1>(a, st); launch_r2c_small<1>(b, st); return 2;
    case 2: launch_r2c_small<2>(a, st); launch_r2c_small<2>(b, st); return 2;
    case 4: launch_r2c_tma<4>(P, di, st); return 1;
    case 8: launch_r2c_tma<8>(P, di, st); return 1;
    case 16: launch_r2c_tma<16>(P, di, st); return 1;
    case 32: launch_r2c_tma<32>(P, di, st); return 1;
    case 64: launch_r2c_tma<64>(P, di, st); return 1;
    default: size_unsupported(m);
  }
  return 0;
}

// K1 for an operand of small planes (src <= m/4, m in {32, 64}): 16-plane
// groups, full-line spectrum stores (fft_small.cuh).  FFTCONV_B200_SMALLSRC=0
// turns it off (A/B, tests).
static bool small_src_enabled() {
  const char* e = getenv("FFTCONV_B200_SMALLSRC");
  return !(e && atoi(e) == 0);
}
// m = 64 only: measured W 4.27 -> 3.87 ms and the n = 64 sweep point k = 7
// 1.045 -> 1.011 ms, but P (m = 32, where K1's 8-plane groups already store
// 64-B pieces) 265 -> 292 us.
// m = 32 only when FFTCONV_B200_SMALLSRC32_MIN (planes) is set and the
// operand has at least that many planes (tests force it): even AlexNet's
// 3 x 3 conv3-5 weights (98k-147k planes) ran slower through it (iteration
// 10.75 -> 11.70 ms; the extra launch and the 16-point row FFTs cost more
// than the full-line stores save at m = 32).
static size_t small_src32_min() {
  const char* e = getenv("FFTCONV_B200_SMALLSRC32_MIN");
  return (e && atoll(e) > 0) ? (size_t)atoll(e) : 0;
}
static bool small_src_ok(size_t m, const R2CParams& p) {
  if (!small_src_enabled() || p.src < 1 || (size_t)p.src * 4 > m) return false;
  if (m == 64) return true;
  const size_t mn = small_src32_min();
  return m == 32 && mn && (size_t)p.R * p.kpad >= mn;
}
template <int M>
static void launch_r2c_small_src(const R2CParams& p, const DevInfo& di, cudaStream_t st, unsigned long long* tspan) {
  using T = TSmall<M>;
  auto kern = r2c_small_kernel<M>;
  smem_optin(kern, T::SMEM);
  const int groups = p.R * ((p.kpad + T::G - 1) / T::G);
  const int grid = std::max(1, std::min(groups, di.sms));
  const CUtensorMap tm = make_bin_map(p.out, p.kpad, p.R, (size_t)M * (M / 2 + 1), T::G, M);
  launch_pdl(kern, dim3(grid), dim3(T::THREADS), T::SMEM, st, p, tm, tspan);
}
static void launch_r2c_small_any(size_t m, const R2CParams& p, const DevInfo& di, cudaStream_t st,
                                 unsigned long long* tspan) {
  if (m == 32) launch_r2c_small_src<32>(p, di, st, tspan);
  else launch_r2c_small_src<64>(p, di, st, tspan);
}

static void launch_r2c_one_span(size_t m, const R2CParams& p, cudaStream_t st, const DevInfo& di,
                                unsigned long long* tspan) {
  R2CPair P{{p, p}, 1};
  P.tspan = tspan;
  switch (m) {
    case 4: return launch_r2c_tma<4>(P, di, st);
    case 8: return launch_r2c_tma<8>(P, di, st);
    case 16: return launch_r2c_tma<16>(P, di, st);
    case 32: return launch_r2c_tma<32>(P, di, st);
    case 64: return launch_r2c_tma<64>(P, di, st);
    default: size_unsupported(m);
  }
}

static void launch_r2c_one(size_t m, const R2CParams& p, cudaStream_t st, const DevInfo& di) {
  const R2CPair P{{p, p}, 1};
  switch (m) {
    case 1: return launch_r2c_small<1>(p, st);
    case 2: return launch_r2c_small<2>(p, st);
    case 4: return launch_r2c_tma<4>(P, di, st);
    case 8: return launch_r2c_tma<8>(P, di, st);
    case 16: return launch_r2c_tma<16>(P, di, st);
    case 32: return launch_r2c_tma<32>(P, di, st);
    case 64: return launch_r2c_tma<64>(P, di, st);
    default: size_unsupported(m);
  }
}

// group-major products are laid out in K4-group-sized blocks
constexpr int kGroupPlanes = FCB_C2R_G;
static_assert((kGroupPlanes & (kGroupPlanes - 1)) == 0 && kGroupPlanes >= 2, "K4 group size");

// Layout the GEMM writes for K4 at fft size m (group-major where the TMA K4
// kernel groups 16 planes).
static OutLayout c2r_layout(size_t m) { return ((m >= 4 && m <= 32) || m == kL) ? kGroupMajor : kBinMajor; }

template <int M>
static void launch_c2r_tma(C2RParams p, const DevInfo& di, cudaStream_t st) {
  using T = TC2R<M>;
  // staged output tiles go out as 1-D bulk stores: planes must be 16-B aligned
  p.bulk = (!p.accum && (reinterpret_cast<uintptr_t>(p.out) & 15) == 0 && (p.out_sr % 4) == 0 &&
            (p.out_sj % 4) == 0 && ((size_t)p.crop * p.crop) % 4 == 0)
               ? 1
               : 0;
  auto kern = c2r_tma_kernel<M>;
  smem_optin(kern, T::SMEM);
  const size_t bins = (size_t)M * (M / 2 + 1);
  const CUtensorMap tm = make_bin_map(p.in, p.ld, p.R, bins, T::G, M);
  const int groups = p.R * ((p.J + T::G - 1) / T::G);
  const int grid = std::max(1, std::min(groups, di.sms));
  launch_pdl(kern, dim3(grid), dim3(T::THREADS), T::SMEM, st, tm, p);
}

// K4 for small crops (accGrad's weight gradients, crop <= m/4) from a
// group-major product (fft_small.cuh); m = 64 by default,
// FFTCONV_B200_SMALLCROP=0 off, =2 also at m = 32 (A/B).
static int small_crop_mode() {
  const char* e = getenv("FFTCONV_B200_SMALLCROP");
  return e ? atoi(e) : 1;
}
static bool small_crop_ok(size_t m, size_t crop) {
  const int mode = small_crop_mode();
  return crop * 4 <= m && crop >= 1 && ((m == 64 && mode >= 1) || (m == 32 && mode >= 2));
}
template <int M>
static void launch_c2r_small(const C2RParams& p, const DevInfo& di, cudaStream_t st) {
  using T = TC2RSmall<M>;
  auto kern = c2r_small_kernel<M>;
  smem_optin(kern, T::SMEM);
  const int groups = p.R * ((p.J + T::G - 1) / T::G);
  const int grid = std::max(1, std::min(groups, di.sms));
  launch_pdl(kern, dim3(grid), dim3(T::THREADS), T::SMEM, st, p);
}

static void launch_c2r(size_t m, const C2RParams& p, cudaStream_t st, const DevInfo& di) {
  if (p.gm && small_crop_ok(m, p.crop)) {
    if (m == 64) return launch_c2r_small<64>(p, di, st);
    if (m == 32) return launch_c2r_small<32>(p, di, st);
  }
  switch (m) {
    case 1: return launch_c2r_small<1>(p, st);
    case 2: return launch_c2r_small<2>(p, st);
    case 4: return launch_c2r_tma<4>(p, di, st);
    case 8: return launch_c2r_tma<8>(p, di, st);
    case 16: return launch_c2r_tma<16>(p, di, st);
    case 32: return launch_c2r_tma<32>(p, di, st);
    case 64: return launch_c2r_tma<64>(p, di, st);
    default: size_unsupported(m);
  }
}

// ---- m = 128: two passes per direction through an L2-sized scratch
// (fft_large.cuh).  Operand rows are walked in chunks whose scratch fits.
// The scratch holds a whole operator's intermediate planes when it fits
// under this cap (measured at alex1: one launch pair per operand, 3.73 ms per
// step, against 4.44 ms with 48 MB L2-sized chunks: the chunks' fill and
// drain cost more than the L2 residency of the intermediate saves).
constexpr size_t kLScratchBudget = (size_t)1 << 30;  // bytes

static size_t large_scratch_budget() {  // FFTCONV_B200_LSCRATCH_MB overrides (tests: force chunking)
  const char* e = getenv("FFTCONV_B200_LSCRATCH_MB");
  return (e && atoi(e) > 0) ? ((size_t)atoi(e) << 20) : kLScratchBudget;
}

// float2 elements: every plane of the largest role up to the budget, at
// least one operand row (maxJ planes)
static size_t large_scratch_elems(size_t maxJ, size_t planes) {
  const size_t per_plane = (size_t)kLRows * kL;  // >= K1a's 128 x 64 (grouped: rows of 16-plane groups)
  return std::max(round_up(maxJ, 16) * per_plane, std::min(large_scratch_budget() / sizeof(float2), planes * per_plane));
}

// per_plane = scratch float2 per plane (r2c: 128 rows x column pairs; c2r:
// 65 rows x crop)
static int large_rows_per_chunk(size_t J, size_t per_plane, size_t scratch_elems) {
  const size_t per_row = J * per_plane;
  const size_t cap = std::min(scratch_elems, large_scratch_budget() / sizeof(float2));
  // <= 65535: the row kernels put rows on gridDim.z
  return (int)std::min<size_t>(65535, std::max<size_t>(1, cap / std::max<size_t>(per_row, 1)));
}

// Persistent grid: as many CTAs as fit on all SMs at once (capped by the work).
template <typename K>
static int resident_grid(K kern, int threads, int smem, int work) {
  int dev = 0, sms = 148, per_sm = 1;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  FCB_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, threads, smem));
  return std::max(1, std::min(work, std::max(1, per_sm) * sms));
}

static bool aligned16(const void* p) { return ((uintptr_t)p & 15u) == 0; }

// K1a / K4b take the bulk-copy ring (fft_large.cuh) when the planes allow
// 16-B bulk copies; FFTCONV_B200_LBULK=0 forces the staged kernels (tests).
static bool large_bulk_enabled() {
  const char* e = getenv("FFTCONV_B200_LBULK");
  return !(e && atoi(e) == 0);
}

// Returns the number of launches.
static int launch_r2c_large(const R2CParams& p, float2* scr, size_t scr_n, cudaStream_t st) {
  const int np = (p.src + 1) / 2;  // column pairs (K1a packs two real columns per FFT)
  const int rpc = FCB_LARGE_GLAYOUT ? large_rows_per_chunk(round_up(p.J, 16), (size_t)kL * large_npad(np), scr_n)
                                    : large_rows_per_chunk(p.J, (size_t)kL * np, scr_n);
  int nl = 0;
  for (int r0 = 0; r0 < p.R; r0 += rpc) {
    const int rows = std::min(rpc, p.R - r0);
    const bool bulk = large_bulk_enabled() && p.src % 2 == 0 && (p.src * p.src) % 4 == 0 && aligned16(p.in) &&
                      p.in_sr % 4 == 0 && p.in_sj % 4 == 0;
    if (bulk) {
      const int smem = 16 + 2 * ((p.src * p.src * 4 + 15) & ~15);
      smem_optin(r2c128_cols_bulk_kernel, smem);
      const int planes = rows * p.J;
      launch_pdl(r2c128_cols_bulk_kernel, dim3(resident_grid(r2c128_cols_bulk_kernel, 256, smem, planes)), dim3(256),
                 smem, st, p, r0, planes, scr);
    } else {
      const int smem = np * kLColPad * (int)sizeof(float2);
      smem_optin(r2c128_cols_kernel, smem);
      launch_pdl(r2c128_cols_kernel, dim3(rows * p.J), dim3(256), smem, st, p, r0, scr);
    }
    const int rpc16 = p.kpad < 16 ? 16 / p.kpad : 1;  // narrow kpad: rows per K1b CTA
    launch_pdl(p.kpad < 16 ? r2c128_rows_kernel<true> : r2c128_rows_kernel<false>,
               large_row_grid((rows + rpc16 - 1) / rpc16, p.kpad < 16 ? 1 : p.kpad / 16), dim3(128), 0, st, p, r0,
               r0 + rows, (const float2*)scr);
    nl += 2;
  }
  return nl;
}

static int launch_c2r_large(const C2RParams& p, float2* scr, size_t scr_n, cudaStream_t st) {
  const int rpc = large_rows_per_chunk(p.J, (size_t)kLRows * p.crop, scr_n);
  int nl = 0;
  for (int r0 = 0; r0 < p.R; r0 += rpc) {
    const int rows = std::min(rpc, p.R - r0);
    launch_pdl(c2r128_rows_kernel, large_row_grid(rows, (p.J + 15) / 16), dim3(128), 0, st, p, r0, scr);
    const int smem = kLRows * p.crop * (int)sizeof(float2);
    if (large_bulk_enabled() && p.crop % 2 == 0) {
      smem_optin(c2r128_cols_flat_kernel, 16 + smem);
      launch_pdl(c2r128_cols_flat_kernel, dim3(rows * p.J), dim3(256), 16 + smem, st, p, r0, (const float2*)scr);
    } else {
      smem_optin(c2r128_cols_kernel, smem);
      launch_pdl(c2r128_cols_kernel, dim3(rows * p.J), dim3(256), smem, st, p, r0, (const float2*)scr);
    }
    nl += 2;
  }
  return nl;
}

struct GemmGeom {
  int nc, n_tiles, m_tiles, stages;
  size_t smem;
};
#ifndef FCB_F16_MAXNC
#define FCB_F16_MAXNC kMaxNc
#endif
#ifndef FCB_GEMM_MAXST
#define FCB_GEMM_MAXST 8
#endif
static GemmGeom gemm_geom(size_t M, size_t N, const DevInfo& di, bool f16) {
  GemmGeom g;
  const size_t n16 = round_up(N, 16);
  const size_t max_nc = f16 ? FCB_F16_MAXNC : kMaxNc;
  g.n_tiles = (int)((n16 + max_nc - 1) / max_nc);
  g.nc = (int)round_up((n16 + g.n_tiles - 1) / g.n_tiles, 16);
  g.m_tiles = (int)((M + kTileM - 1) / kTileM);
  // raw TMA stages (A + B chunks) fill what the two converted-B buffers leave
  const int sb = gemm_raw_stage_bytes(g.nc, f16);
  const int fixed = 2 * gemm_bbuf_bytes(g.nc);
  const int budget = di.max_smem_optin - 1024 - 256 - fixed;
  g.stages = std::min(f16 ? 4 : FCB_GEMM_MAXST, budget / sb);
  if (g.stages < 2) throw Error(FFTCONV_B200_CUDA_ERROR, "gemm tile does not fit shared memory");
  g.smem = (size_t)g.stages * sb + fixed + 1024 + 256;
  return g;
}

// D[t] = A[t] . conj(B[t])^T per bin; im_sign = -1 returns conj(D) (the
// accGrad orientation, conj(A) . B).  A: F[t][M][2*kpad], B: F[t][N][2*kpad].

// GEMM operand precision (fftconv_b200_set_gemm_kind, FFTCONV_B200_GEMM =
// tf32 | f16x3 | auto):
//   3xTF32  per-element fp32 range;
//   fp16x3  one power-of-two scale per operand, twice the tensor rate;
//   auto    (default) 3xTF32 where the GEMM's byte floor exceeds its 3xTF32
//           tensor floor (fp16x3 would not be faster), else the fp16x3 kernel
//           and a 3xTF32 fallback launched back to back: each reads K1's
//           per-row maxima and exactly one of them runs -- fp16x3 when every
//           operand row is within 2^18 of its operand's maximum.
// The process default (atomic: set from any thread); a workspace may
// override it (fftconv_b200_ws_set_gemm_kind).
static std::atomic<int> g_gemm_kind{[] {
  const char* e = getenv("FFTCONV_B200_GEMM");
  if (e && std::string(e) == "tf32") return FFTCONV_B200_GEMM_TF32X3;
  if (e && std::string(e) == "f16x3") return FFTCONV_B200_GEMM_F16X3;
  return FFTCONV_B200_GEMM_AUTO;
}()};

enum GemmRoute { kRouteTf32 = 0, kRouteF16 = 1, kRouteAuto = 2 };

// Which GEMM kernel(s) a product of M x N over K on `bins` bins needs, from
// a time model of the two kernels:
//   3xTF32  max(tensor, bytes);  fp16x3  max(tensor / 2, bytes) + 8 us
// (the auto pair's second launch, K1's per-row maxima, the heavier
// converters).  Per K chunk of 16 complex a tile issues 12 UMMAs (M = 128,
// N = 2 nc <= 192, K = 8), measured on the box at ~110 cycles each whatever
// nc (a GEMM trace of W at S = 16, nc = 16: 3xTF32 317 us, fp16x3 197 us;
// at P, nc = 96, ~105) -- so a small-N tile is tensor-bound long before its
// FLOPs say so.  Bytes at 6.5 TB/s (MEASURED_PEAKS.json), 148 SMs at
// 1.9 GHz; the tile shape follows gemm_swap / gemm_geom.  Near a tie at
// large N (AlexNet's conv2 at S = 128: fp16x3 measured faster, the model
// says even) round 1's FLOP / byte rule still picks fp16x3:
// MNK / (MK + NK + MN) > 274 TF/s / 6.55 TB/s ~= 42.
static GemmRoute gemm_route(int kind, size_t M, size_t N, size_t K, size_t bins) {
  if (kind == FFTCONV_B200_GEMM_TF32X3) return kRouteTf32;
  if (kind == FFTCONV_B200_GEMM_F16X3) return kRouteF16;
  if ((double)M * N * K > 42.0 * ((double)M * K + (double)N * K + (double)M * N)) return kRouteAuto;
  auto padded = [](size_t rows, size_t cols) { return ((rows + 127) / 128) * round_up(cols, 16); };
  if (padded(N, M) < padded(M, N)) std::swap(M, N);  // gemm_swap's orientation
  const size_t n16 = round_up(N, 16);
  const size_t n_tiles = (n16 + kMaxNc - 1) / kMaxNc;
  const size_t m_tiles = (M + kTileM - 1) / kTileM;
  const double umma = (double)bins * m_tiles * n_tiles * (round_up(K, 16) / 16) * 12.0;
  const double t_tensor = umma * 110.0 / (148.0 * 1.9e9);
  const double t_bytes = 8.0 * bins * ((double)M * K + (double)N * K + (double)M * N) / 6.5e12;
  const double t_tf32 = std::max(t_tensor, t_bytes), t_f16 = std::max(0.5 * t_tensor, t_bytes) + 8e-6;
  return t_f16 < t_tf32 ? kRouteAuto : kRouteTf32;
}

static void launch_gemm_kernel(const float* A, const float* B, float* out, size_t bins, size_t M, size_t N,
                               size_t kpad, float im_sign, OutLayout lay, size_t ldm, const DevInfo& di,
                               cudaStream_t st, bool f16, int select, const unsigned long long* amax_a,
                               const unsigned long long* amax_b, int* path, unsigned long long* tspan = nullptr);

// Returns the number of launches (2 for an auto pair).  amax_* (K1's per-row
// words, rows_* rows) are required for the fp16 routes; without them the
// GEMM runs 3xTF32.
static int launch_gemm(const float* A, const float* B, float* out, size_t bins, size_t M, size_t N,
                       size_t kpad, float im_sign, OutLayout lay, size_t ldm, const DevInfo& di,
                       cudaStream_t st, GemmRoute route = kRouteTf32,
                       const unsigned long long* amax_a = nullptr, const unsigned long long* amax_b = nullptr,
                       int* path = nullptr, unsigned long long* tspan = nullptr) {
  if (!amax_a || !amax_b) route = kRouteTf32;
  if (route == kRouteAuto) {
    launch_gemm_kernel(A, B, out, bins, M, N, kpad, im_sign, lay, ldm, di, st, true, 1, amax_a, amax_b, path, tspan);
    launch_gemm_kernel(A, B, out, bins, M, N, kpad, im_sign, lay, ldm, di, st, false, 2, amax_a, amax_b, path,
                       tspan);
    return 2;
  }
  launch_gemm_kernel(A, B, out, bins, M, N, kpad, im_sign, lay, ldm, di, st, route == kRouteF16, 0, amax_a,
                     amax_b, path, tspan);
  return 1;
}

static void launch_gemm_kernel(const float* A, const float* B, float* out, size_t bins, size_t M, size_t N,
                               size_t kpad, float im_sign, OutLayout lay, size_t ldm, const DevInfo& di,
                               cudaStream_t st, bool f16, int select, const unsigned long long* amax_a,
                               const unsigned long long* amax_b, int* path, unsigned long long* tspan) {
  const GemmGeom g = gemm_geom(M, N, di, f16);
  CUtensorMap ta = make_operand_map(A, kpad, M, bins, kTileM);
  CUtensorMap tb = make_operand_map(B, kpad, N, bins, (uint32_t)g.nc);
  GemmParams p;
  p.out = out;
  p.bins = (int)bins;
  p.m_valid = (int)M;
  p.n_valid = (int)N;
  p.k_chunks = (int)((kpad + 15) / 16);  // a K below 16: TMA zero-fills the chunk past the row
  p.m_tiles = g.m_tiles;
  p.n_tiles = g.n_tiles;
  p.nc = g.nc;
  p.stages = g.stages;
  p.im_sign = im_sign;
  p.amax_a = amax_a;
  p.amax_b = amax_b;
  p.rows_a = (int)M;
  p.rows_b = (int)N;
  p.select = select;
  p.path = path;
  p.tspan = tspan;
  p.gm_log2 = 4;
  if (lay == kBinMajor) {
    p.s_t = (long long)N * ldm;
    p.s_mg = 16;
    p.s_n = (long long)ldm;
  } else {
    const long long G = kGroupPlanes;
    p.gm_log2 = ilog2c(kGroupPlanes);
    p.s_t = G;
    p.s_mg = (long long)bins * G;
    p.s_n = (long long)((M + G - 1) / G) * (long long)bins * G;
  }
  const bool ranges = g.m_tiles * g.n_tiles == 1;
  auto kern = f16 ? (ranges ? cgemm_bins_tcgen05<true, true> : cgemm_bins_tcgen05<true, false>)
                  : (ranges ? cgemm_bins_tcgen05<false, true> : cgemm_bins_tcgen05<false, false>);
  smem_optin(kern, (int)g.smem);
  const long long tiles = (long long)bins * g.m_tiles * g.n_tiles;
  const int grid = (int)std::min<long long>(tiles, di.sms);
  launch_pdl(kern, dim3(grid), dim3(kGemmThreads), g.smem, st, ta, tb, p);
#ifdef FCB_GEMM_TRACE
  {  // per-CTA timeline (ns): launch -> work start -> end, relative to the earliest launch
    unsigned long long h[3][160];
    cudaStreamSynchronize(st);
    cudaMemcpyFromSymbol(h, g_cta_time, sizeof h);
    unsigned long long t0 = ~0ull;
    for (int i = 0; i < grid; ++i) t0 = std::min(t0, h[0][i]);
    std::vector<double> st_, en;
    for (int i = 0; i < grid; ++i) {
      st_.push_back((h[1][i] - t0) * 1e-3);
      en.push_back((h[2][i] - t0) * 1e-3);
    }
    std::vector<double> es = en;
    std::sort(es.begin(), es.end());
    printf("gemm %d CTAs: start max %.1f us; end min %.1f p50 %.1f p90 %.1f max %.1f us; tiles/CTA %.2f\n", grid,
           *std::max_element(st_.begin(), st_.end()), es.front(), es[es.size() / 2], es[es.size() * 9 / 10],
           es.back(), (double)tiles / grid);
    for (int i = 0; i < grid; i += 16) printf("  cta %3d start %.1f end %.1f\n", i, st_[i], en[i]);
  }
#endif
}

// Per-row max |component| of a bin-major operand F[t][rows][2*kp] into
// out[row] (epoch 0 words; debug hook helper).  grid = rows.
__global__ void absmax_rows_kernel(const float* v, long long bins, int rows, int kp2, unsigned long long* out) {
  const int r = blockIdx.x;
  float m = 0.f;
  for (long long i = threadIdx.x; i < bins * kp2; i += blockDim.x) {
    const long long t = i / kp2, k = i - t * kp2;
    m = fmaxf(m, fabsf(v[(t * rows + r) * kp2 + k]));
  }
  const uint32_t b = __reduce_max_sync(0xffffffffu, __float_as_uint(m));
  if ((threadIdx.x & 31) == 0) atomicMax(out + r, (unsigned long long)b);
}

// Negates every imaginary part of n complex values (debug hook helper).
__global__ void conj_inplace_kernel(float2* v, long long n) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x)
    v[i].y = -v[i].y;
}

// ---- packed-spectrum API (fft.hpp:105-152, :209-243) --------------------
// The kernels' half spectrum keeps rows u <= m/2 and every column v, planes
// as the K index: F[t][j] (t = u*m + v, row stride ld complex).  The
// reference packing keeps every row u and columns v <= m/2 per plane:
// spec[j][u][v].  Hermitian identity F[u][v] = conj(F[(m-u)%m][(m-v)%m]).

// F -> reference packing; one thread per output element, v fastest.
__global__ void spectrum_pack_ref_kernel(const float2* F, long long ld, int m, long long planes, float2* out) {
  const int pc = m / 2 + 1;
  const long long n = planes * m * pc;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
    const long long j = i / (m * pc);
    const int rem = (int)(i - j * m * pc), u = rem / pc, v = rem - u * pc;
    if (u <= m / 2) {
      out[i] = F[(long long)(u * m + v) * ld + j];
    } else {
      const float2 z = F[(long long)(((m - u) % m) * m + (m - v) % m) * ld + j];
      out[i] = make_float2(z.x, -z.y);
    }
  }
}

// reference packing -> F (ld complex per bin, planes >= J zero); one thread
// per F element, plane fastest.
__global__ void spectrum_unpack_ref_kernel(const float2* spec, int m, long long planes, long long ld, float2* F) {
  const int pc = m / 2 + 1;
  const long long n = (long long)pc * m * ld;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
    const long long t = i / ld, j = i - t * ld;
    const int u = (int)(t / m), v = (int)(t - (long long)u * m);
    float2 z = make_float2(0.f, 0.f);
    if (j < planes) {
      if (v <= m / 2) {
        z = spec[(j * m + u) * pc + v];
      } else {
        z = spec[(j * m + (m - u) % m) * pc + (m - v)];
        z.y = -z.y;
      }
    }
    F[i] = z;
  }
}

}  // namespace fcb

using namespace fcb;

// ------------------------------------------------------------ NCCL (run-time loaded)
// The product does not link NCCL: the sharded entry points dlopen
// libnccl.so.2 on first use (inside a torch process that is torch's own
// NCCL, already loaded under that soname), so single-GPU users never need it.
namespace fcb {
struct NcclApi {
  decltype(&ncclGetUniqueId) get_unique_id = nullptr;
  decltype(&ncclCommInitRank) comm_init_rank = nullptr;
  decltype(&ncclCommDestroy) comm_destroy = nullptr;
  decltype(&ncclAllReduce) all_reduce = nullptr;
  decltype(&ncclGetErrorString) error_string = nullptr;
  std::string why;
};

static const NcclApi& nccl_api() {
  static NcclApi api;
  static std::once_flag once;
  std::call_once(once, [] {
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
    if (!h) {
      const char* e = dlerror();
      api.why = e ? e : "dlopen failed";
      return;
    }
    api.get_unique_id = reinterpret_cast<decltype(api.get_unique_id)>(dlsym(h, "ncclGetUniqueId"));
    api.comm_init_rank = reinterpret_cast<decltype(api.comm_init_rank)>(dlsym(h, "ncclCommInitRank"));
    api.comm_destroy = reinterpret_cast<decltype(api.comm_destroy)>(dlsym(h, "ncclCommDestroy"));
    api.all_reduce = reinterpret_cast<decltype(api.all_reduce)>(dlsym(h, "ncclAllReduce"));
    api.error_string = reinterpret_cast<decltype(api.error_string)>(dlsym(h, "ncclGetErrorString"));
    if (!api.get_unique_id || !api.comm_init_rank || !api.comm_destroy || !api.all_reduce || !api.error_string)
      api.why = "libnccl.so.2 lacks an expected symbol";
  });
  if (!api.why.empty()) throw Error(FFTCONV_B200_NCCL_ERROR, "NCCL unavailable: " + api.why);
  return api;
}

#define FCB_NCCL(call)                                                                      \
  do {                                                                                      \
    ncclResult_t r_ = (call);                                                               \
    if (r_ != ncclSuccess)                                                                  \
      throw Error(FFTCONV_B200_NCCL_ERROR, std::string(#call) + ": " + nccl_api().error_string(r_)); \
  } while (0)
}  // namespace fcb

// ------------------------------------------------------------ workspace
constexpr int kMaxChunks = 16;

struct fftconv_b200_ws {
  int device = 0;
  DevInfo di;
  uint64_t cap_x = 0, cap_w = 0, cap_y = 0;
  size_t max_m = 1;
  // frequency-domain buffers (floats)
  // frequency-domain arena: [A | B | D], one allocation so a single L2
  // access-policy window can cover the spectra between K1 -> K3 -> K4
  float* freq = nullptr;
  float* bufA = nullptr;
  float* bufB = nullptr;
  float* bufD = nullptr;
  size_t nA = 0, nB = 0, nD = 0;
  // host-API device staging
  float* st_in0 = nullptr;
  float* st_in1 = nullptr;
  float* st_out = nullptr;
  size_t n_in0 = 0, n_in1 = 0, n_out = 0;
  cudaStream_t host_stream = nullptr;  // compute stream of the host-pointer entry points
  cudaStream_t h2d_stream = nullptr, d2h_stream = nullptr;
  cudaEvent_t pev[2][kMaxChunks + 1] = {};  // chunk pipeline: inputs landed / outputs ready
  bool pev_ready = false;
  uint64_t ctr[3] = {0, 0, 0};
  unsigned long long* amax = nullptr;  // K1 -> K3 per-row max-magnitude words: A rows | B rows
  size_t amax_rows = 0;                // rows per operand region
  int* gemm_path = nullptr;            // which GEMM kernel ran last (1 fp16x3, 0 3xTF32)
  float2* lscr = nullptr;              // m = 128 transform scratch (fft_large.cuh)
  size_t lscr_n = 0;
  unsigned epoch = 0;
  int gemm_kind = -1;                   // -1: the process default (g_gemm_kind)
  // Cross-stream ordering: the event recorded at the end of the last
  // operator and the stream it ran on.  An operator on another stream (the
  // host entry points' host_stream, or a different caller stream) waits on
  // it first, since every operator reuses the same spectra buffers.
  cudaEvent_t done_ev = nullptr;
  cudaStream_t last_st = nullptr;
  bool has_last = false;
  // sharded accGrad: the all-reduces run on comm_stream, each after the K4
  // chunk that wrote its rows (chunk_ev); comm_ev[0..2] time them (K4 end on
  // the compute stream, first all-reduce start, last all-reduce end)
  cudaStream_t comm_stream = nullptr;
  cudaEvent_t chunk_ev[kMaxChunks + 1] = {};
  cudaEvent_t comm_ev[3] = {};
  bool comm_ready = false;
  bool comm_timed = false;
  // live kernel spans (fftconv_b200_set_span_timing): per operator, K1 / K3 /
  // K4 start and end words (ptx.cuh kSpanSlots operators per batch)
  unsigned long long* spans = nullptr;
  int span_on = 0;
  int span_next = 0;
  unsigned long long* span_slot(int k) { return span_on ? spans + (size_t)(span_next % kSpanSlots) * 3 + k : nullptr; }
  std::string last_error;
  bool timing = false;
  cudaEvent_t ev[5] = {};
  bool ev_ready = false;
  int last_launches = 0;
};

namespace {

template <typename F>
int guarded(fftconv_b200_ws* ws, F&& f) {
  try {
    f();
    return FFTCONV_B200_OK;
  } catch (const Error& e) {
    g_last_error = e.what();
    if (ws) ws->last_error = e.what();
    return e.code;
  } catch (const std::exception& e) {
    g_last_error = e.what();
    if (ws) ws->last_error = e.what();
    return FFTCONV_B200_INVALID_ARGUMENT;
  }
}

struct DeviceGuard {
  int prev = -1;
  explicit DeviceGuard(int d) {
    cudaGetDevice(&prev);
    if (prev != d) cudaSetDevice(d);
  }
  ~DeviceGuard() {
    int cur = -1;
    cudaGetDevice(&cur);
    if (prev >= 0 && cur != prev) cudaSetDevice(prev);
  }
};

int ws_gemm_kind(const fftconv_b200_ws* ws) { return ws->gemm_kind >= 0 ? ws->gemm_kind : g_gemm_kind.load(); }

bool capturing(cudaStream_t st) {
  cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
  return cudaStreamIsCapturing(st, &cs) == cudaSuccess && cs != cudaStreamCaptureStatusNone;
}

// Orders an operator on `st` after the workspace's previous operator when that
// one ran on another stream (device- and host-path calls share
// bufA / bufB / bufD, amax and the scratch).  Not inside a stream capture: a
// captured graph's own dependencies order it.
void order_after_last(fftconv_b200_ws* ws, cudaStream_t st) {
  if (ws->has_last && ws->last_st != st && !capturing(st)) FCB_CUDA(cudaStreamWaitEvent(st, ws->done_ev, 0));
}

void mark_done(fftconv_b200_ws* ws, cudaStream_t st) {
  if (capturing(st)) return;
  FCB_CUDA(cudaEventRecord(ws->done_ev, st));
  ws->last_st = st;
  ws->has_last = true;
}

// K1's per-row max-magnitude words hold max(rows of A, rows of B) per operand
// region; a workspace reused for a layer with more operand rows than any
// registered config (the capacity check bounds bins x rows x maps, not rows)
// grows them.  cudaFree synchronises the device first.
void ensure_amax(fftconv_b200_ws* ws, size_t rows) {
  if (rows <= ws->amax_rows) return;
  if (ws->amax) cudaFree(ws->amax);
  ws->amax = nullptr;
  ws->amax_rows = 0;
  FCB_CUDA(cudaMalloc(&ws->amax, 2 * rows * sizeof(unsigned long long)));
  FCB_CUDA(cudaMemset(ws->amax, 0, 2 * rows * sizeof(unsigned long long)));
  ws->amax_rows = rows;
}

void grow(float*& p, size_t& have, size_t need) {
  if (need <= have) return;
  if (p) cudaFree(p);
  p = nullptr;
  have = 0;
  FCB_CUDA(cudaMalloc(&p, need * sizeof(float)));
  have = need;
}

// ConvWorkspace::prepare (conv_fft.hpp:211-222): validate -> capacity.
size_t prepare(fftconv_b200_ws* ws, const fftconv_b200_layer& c) {
  validate_cfg(c);
  const size_t m = next_pow2(c.image);
  const uint64_t bins = m * (m / 2 + 1);
  if (bins * c.batch * c.in_maps > ws->cap_x || bins * c.out_maps * c.in_maps > ws->cap_w ||
      bins * c.batch * c.out_maps > ws->cap_y)
    throw Error(FFTCONV_B200_CAPACITY_ERROR, "workspace too small for this layer");
  if (m > kL)
    throw Error(FFTCONV_B200_SIZE_ERROR,
                "fft size " + std::to_string(m) + " not supported by the B200 kernels (max 128)");
  return m;
}

void set_arena(fftconv_b200_ws* ws, size_t na, size_t nb, size_t nd) {
  na = round_up(std::max(na, ws->nA), 64);  // keep 256-B alignment of B and D
  nb = round_up(std::max(nb, ws->nB), 64);
  nd = round_up(std::max(nd, ws->nD), 64);
  if (ws->freq && na == ws->nA && nb == ws->nB && nd == ws->nD) return;
  if (ws->freq) cudaFree(ws->freq);
  ws->freq = nullptr;
  ws->nA = ws->nB = ws->nD = 0;
  FCB_CUDA(cudaMalloc(&ws->freq, (na + nb + nd) * sizeof(float)));
  ws->bufA = ws->freq;
  ws->bufB = ws->freq + na;
  ws->bufD = ws->bufB + nb;
  ws->nA = na;
  ws->nB = nb;
  ws->nD = nd;
}

void ensure_large_scratch(fftconv_b200_ws* ws, const fftconv_b200_layer& c, size_t m) {
  if (m != kL) return;
  const size_t need = large_scratch_elems(std::max({c.batch, c.in_maps, c.out_maps}),
                                         std::max({c.batch * c.in_maps, c.batch * c.out_maps, c.in_maps * c.out_maps}));
  if (need <= ws->lscr_n) return;
  if (ws->lscr) cudaFree(ws->lscr);
  ws->lscr = nullptr;
  ws->lscr_n = 0;
  FCB_CUDA(cudaMalloc(&ws->lscr, need * sizeof(float2)));
  ws->lscr_n = need;
}

void ensure_freq(fftconv_b200_ws* ws, Pass pass, const fftconv_b200_layer& c, size_t m) {
  const PassNeed need = pass_need(pass, c.batch, c.in_maps, c.out_maps, m);
  if (need.a > ws->nA || need.b > ws->nB || need.d > ws->nD) set_arena(ws, need.a, need.b, need.d);
  ensure_large_scratch(ws, c, m);
}

void record(fftconv_b200_ws* ws, int i, cudaStream_t st) {
  if (!ws->timing) return;
  if (!ws->ev_ready) {
    for (auto& e : ws->ev) FCB_CUDA(cudaEventCreate(&e));
    ws->ev_ready = true;
  }
  FCB_CUDA(cudaEventRecord(ws->ev[i], st));
}

void require_nonzero(size_t a, size_t b, size_t c, size_t d, const char* what) {
  if (!a || !b || !c || !d)
    throw Error(FFTCONV_B200_SIZE_ERROR, std::string(what) + ": all dimensions must be >= 1");
}

// GEMM orientation.  fprop / bprop put the minibatch on M, which the
// tcgen05 tile fixes at 128 rows; a small (e.g. minibatch-sharded) batch
// wastes most of every tile.  D = A.conj(B)^T equals conj(B.conj(A)^T)^T, so
// the operands can be swapped (maps on M, batch on N) with the epilogue
// conjugating, and K4 reads the transposed product (SURVEY.md section 7,
// hard part 3).  Chosen when it pads less work.
static bool gemm_swap(size_t M, size_t N) {
  auto padded = [](size_t rows, size_t cols) { return ((rows + 127) / 128) * round_up(cols, 16); };
  return padded(N, M) < padded(M, N);
}

// ---- the three operators (device pointers) ---------------------------

// Both forward transforms; when the GEMM route involves fp16x3 (and m >= 4,
// the TMA / m = 128 K1) they also record the operands' per-row
// max-magnitude words under a fresh epoch.  a.amax / b.amax stay null
// otherwise (the GEMM then runs 3xTF32).
int r2c_operands(fftconv_b200_ws* ws, size_t m, R2CParams& a, R2CParams& b, cudaStream_t st, GemmRoute route) {
  if (m >= 4 && route != kRouteTf32) {
    ensure_amax(ws, (size_t)std::max(a.R, b.R));
    a.amax = ws->amax;
    b.amax = ws->amax + ws->amax_rows;
    a.epoch = b.epoch = ++ws->epoch;
  }
  if (m == kL) return launch_r2c_large(a, ws->lscr, ws->lscr_n, st) + launch_r2c_large(b, ws->lscr, ws->lscr_n, st);
  const bool sa = small_src_ok(m, a), sb = small_src_ok(m, b);
  if (sa || sb) {  // the small-plane operand(s) through fft_small.cuh, the other through K1
    unsigned long long* ts = ws->span_slot(0);
    if (sa) launch_r2c_small_any(m, a, ws->di, st, ts);
    else launch_r2c_one_span(m, a, st, ws->di, ts);
    if (sb) launch_r2c_small_any(m, b, ws->di, st, ts);
    else launch_r2c_one_span(m, b, st, ws->di, ts);
    return 2;
  }
  return launch_r2c_both(m, a, b, st, ws->di, ws->span_slot(0));
}

// K4 for any supported m; returns the number of launches.
int c2r_run(fftconv_b200_ws* ws, size_t m, const C2RParams& c, cudaStream_t st) {
  if (m == kL) return launch_c2r_large(c, ws->lscr, ws->lscr_n, st);
  C2RParams cs = c;
  cs.tspan = ws->span_slot(2);
  launch_c2r(m, cs, st, ws->di);
  return 1;
}

// n_logical > xr: the input planes are the top-left xr x xr of the layer's
// n x n image, zero elsewhere (the layer stack's fit_to pad, layers.hpp:393-407,
// folded in: K1 zero-fills beyond the source edge anyway).
void run_forward(fftconv_b200_ws* ws, const float* x, size_t S, size_t f, size_t xr, size_t xc,
                 const float* w, size_t wo, size_t wi, size_t k, float* y, cudaStream_t st, bool relu = false,
                 size_t n_logical = 0) {
  require_nonzero(S, f, xr, xc, "Tensor4");
  require_nonzero(wo, wi, k, 1, "Weights4");
  if (xr != xc) throw Error(FFTCONV_B200_SIZE_ERROR, "forward_fft: planes must be square");
  if (wi != f) throw Error(FFTCONV_B200_SHAPE_ERROR, "forward_fft: weight in_maps != input maps");
  const size_t n = n_logical ? n_logical : xr;
  if (xr > n) throw Error(FFTCONV_B200_SIZE_ERROR, "forward_fft: input larger than the layer image");
  if (k > n) throw Error(FFTCONV_B200_SIZE_ERROR, "forward_fft: kernel larger than image");
  const size_t no = n - k + 1, fo = wo;
  const fftconv_b200_layer cfg{k, n, f, fo, S};
  const size_t m = prepare(ws, cfg);
  const size_t bins = m * (m / 2 + 1);
  ensure_freq(ws, kFprop, cfg, m);
  const size_t kp = kpad_for(f, m);

  record(ws, 0, st);
  R2CParams a{x, ws->bufA, (long long)(f * xr * xr), (long long)(xr * xr), (int)S, (int)f, (int)kp,
              (int)xr, (int)(xr | 1)};
  R2CParams b{w, ws->bufB, (long long)(f * k * k), (long long)(k * k), (int)fo, (int)f, (int)kp,
              (int)k, (int)(k | 1)};
  const GemmRoute route = gemm_route(ws_gemm_kind(ws), S, fo, f, bins);
  const int nl = r2c_operands(ws, m, a, b, st, route);
  record(ws, 1, st);  // both forward transforms
  record(ws, 2, st);
  C2RParams c{ws->bufD, y, (long long)(no * no), (long long)(fo * no * no), (int)fo, (int)S,
              (int)no, 0, 0, 1.0f / (float)(m * m), (int)round_up(S, 2)};
  int ng;
  if (!gemm_swap(S, fo)) {  // D[t][o][b]: planes (r = o, j = b)
    ng = launch_gemm(ws->bufA, ws->bufB, ws->bufD, bins, S, fo, kp, 1.0f, c2r_layout(m), round_up(S, 2),
                     ws->di, st, route, a.amax, b.amax, ws->gemm_path, ws->span_slot(1));
  } else {  // D^T[t][b][o]: planes (r = b, j = o)
    ng = launch_gemm(ws->bufB, ws->bufA, ws->bufD, bins, fo, S, kp, -1.0f, c2r_layout(m), round_up(fo, 2),
                     ws->di, st, route, b.amax, a.amax, ws->gemm_path, ws->span_slot(1));
    c = C2RParams{ws->bufD, y, (long long)(fo * no * no), (long long)(no * no), (int)S, (int)fo,
                  (int)no, 0, 0, 1.0f / (float)(m * m), (int)round_up(fo, 2)};
  }
  record(ws, 3, st);
  c.gm = c2r_layout(m) == kGroupMajor;
  c.relu = relu ? 1 : 0;
  const int nc = c2r_run(ws, m, c, st);
  record(ws, 4, st);
  ws->last_launches = nl + ng + nc;
  if (ws->span_on) ++ws->span_next;
  ws->ctr[0] += S * f + fo * f;
  ws->ctr[1] += S * fo;
  ws->ctr[2] += (uint64_t)bins * fo * f * S;
}

// gx_size < n: only the top-left gx_size x gx_size of every input-gradient
// plane is written (the stack's fit_to crop back to the pre-pad size folded
// into K4's crop).
void run_grad_input(fftconv_b200_ws* ws, const float* gy, size_t S, size_t fo, size_t gr,
                    size_t gc, const float* w, size_t wo, size_t wi, size_t k, float* gx,
                    cudaStream_t st, size_t gx_size = 0) {
  require_nonzero(S, fo, gr, gc, "Tensor4");
  require_nonzero(wo, wi, k, 1, "Weights4");
  if (gr != gc) throw Error(FFTCONV_B200_SIZE_ERROR, "grad_input_fft: planes must be square");
  if (wo != fo)
    throw Error(FFTCONV_B200_SHAPE_ERROR, "grad_input_fft: weight out_maps != gradient maps");
  const size_t no = gr, n = no + k - 1, f = wi;
  const fftconv_b200_layer cfg{k, n, f, fo, S};
  const size_t m = prepare(ws, cfg);
  const size_t bins = m * (m / 2 + 1);
  ensure_freq(ws, kBprop, cfg, m);
  const size_t kp = kpad_for(fo, m);

  record(ws, 0, st);
  R2CParams a{gy, ws->bufA, (long long)(fo * no * no), (long long)(no * no), (int)S, (int)fo,
              (int)kp, (int)no, (int)(no | 1)};
  R2CParams b{w, ws->bufB, (long long)(k * k), (long long)(f * k * k), (int)f, (int)fo, (int)kp,
              (int)k, (int)(k | 1), /*conj=*/1};  // GX = GY . W = GY . conj(conj W)
  const GemmRoute route = gemm_route(ws_gemm_kind(ws), S, f, fo, bins);
  const int nl = r2c_operands(ws, m, a, b, st, route);
  record(ws, 1, st);  // both forward transforms
  record(ws, 2, st);
  const size_t ge = gx_size ? gx_size : n;  // output plane edge
  if (ge > n) throw Error(FFTCONV_B200_SIZE_ERROR, "grad_input_fft: output larger than the layer image");
  C2RParams c{ws->bufD, gx, (long long)(ge * ge), (long long)(f * ge * ge), (int)f, (int)S, (int)ge,
              0, 0, 1.0f / (float)(m * m), (int)round_up(S, 2)};
  int ng;
  if (!gemm_swap(S, f)) {  // D[t][f][b]
    ng = launch_gemm(ws->bufA, ws->bufB, ws->bufD, bins, S, f, kp, 1.0f, c2r_layout(m), round_up(S, 2),
                     ws->di, st, route, a.amax, b.amax, ws->gemm_path, ws->span_slot(1));
  } else {  // D^T[t][b][f]
    ng = launch_gemm(ws->bufB, ws->bufA, ws->bufD, bins, f, S, kp, -1.0f, c2r_layout(m), round_up(f, 2),
                     ws->di, st, route, b.amax, a.amax, ws->gemm_path, ws->span_slot(1));
    c = C2RParams{ws->bufD, gx, (long long)(f * ge * ge), (long long)(ge * ge), (int)S, (int)f, (int)ge,
                  0, 0, 1.0f / (float)(m * m), (int)round_up(f, 2)};
  }
  record(ws, 3, st);
  c.gm = c2r_layout(m) == kGroupMajor;
  const int nc = c2r_run(ws, m, c, st);
  record(ws, 4, st);
  ws->last_launches = nl + ng + nc;
  if (ws->span_on) ++ws->span_next;
  ws->ctr[0] += S * fo + fo * f;
  ws->ctr[1] += S * f;
  ws->ctr[2] += (uint64_t)bins * fo * f * S;
}

// accGrad's K4 in f'-chunks: `done(o0, o1, st)` runs after the launch that
// wrote gw rows [o0, o1) (the sharded entry point all-reduces them there,
// overlapping the next chunk's transforms).
struct ChunkHook {
  int chunks = 1;
  std::function<void(size_t, size_t, cudaStream_t)> done;
};

void run_grad_weight(fftconv_b200_ws* ws, const float* gy, size_t Sg, size_t fo, size_t gr,
                     size_t gc, const float* x, size_t Sx, size_t f, size_t xr, size_t xc,
                     float* gw, cudaStream_t st, bool accum = false, const ChunkHook* hook = nullptr,
                     size_t n_logical = 0) {
  require_nonzero(Sg, fo, gr, gc, "Tensor4");
  require_nonzero(Sx, f, xr, xc, "Tensor4");
  if (gr != gc) throw Error(FFTCONV_B200_SIZE_ERROR, "grad_weight_fft: planes must be square");
  if (xr != xc) throw Error(FFTCONV_B200_SIZE_ERROR, "grad_weight_fft: planes must be square");
  if (Sg != Sx) throw Error(FFTCONV_B200_SHAPE_ERROR, "grad_weight_fft: batch mismatch");
  const size_t no = gr, n = n_logical ? n_logical : xr;  // n_logical: as run_forward
  if (xr > n) throw Error(FFTCONV_B200_SIZE_ERROR, "grad_weight_fft: input larger than the layer image");
  if (no > n) throw Error(FFTCONV_B200_SIZE_ERROR, "grad_weight_fft: gradient larger than input");
  const size_t k = n - no + 1, S = Sx;
  const fftconv_b200_layer cfg{k, n, f, fo, S};
  const size_t m = prepare(ws, cfg);
  const size_t bins = m * (m / 2 + 1);
  ensure_freq(ws, kAccGrad, cfg, m);
  const size_t kp = kpad_for(S, m);

  record(ws, 0, st);
  R2CParams a{gy, ws->bufA, (long long)(no * no), (long long)(fo * no * no), (int)fo, (int)S,
              (int)kp, (int)no, (int)(no | 1)};
  R2CParams b{x, ws->bufB, (long long)(xr * xr), (long long)(f * xr * xr), (int)f, (int)S, (int)kp,
              (int)xr, (int)(xr | 1)};
  const GemmRoute route = gemm_route(ws_gemm_kind(ws), fo, f, S, bins);
  const int nl = r2c_operands(ws, m, a, b, st, route);
  record(ws, 1, st);  // both forward transforms
  record(ws, 2, st);
  // small crops at m = 64 read a group-major product (the small-crop K4)
  const OutLayout lay = small_crop_ok(m, k) ? kGroupMajor : c2r_layout(m);
  const int ng = launch_gemm(ws->bufA, ws->bufB, ws->bufD, bins, fo, f, kp, -1.0f, lay, round_up(fo, 2),
                             ws->di, st, route, a.amax, b.amax, ws->gemm_path, ws->span_slot(1));
  record(ws, 3, st);
  C2RParams c{ws->bufD, gw, (long long)(k * k), (long long)(f * k * k), (int)f, (int)fo, (int)k,
              0, 0, 1.0f / (float)(m * m), (int)round_up(fo, 2)};
  c.gm = lay == kGroupMajor;
  c.accum = accum;
  int nc = 0;
  // chunked only where the TMA K4 runs (m in 4..64); chunk edges on 16-plane
  // group boundaries (the K4 group size at every such m divides 16)
  const int nchunk = (hook && m >= 4 && m <= 64) ? (int)std::max<size_t>(1, std::min<size_t>(hook->chunks, (fo + 15) / 16)) : 1;
  if (nchunk == 1) {
    nc = c2r_run(ws, m, c, st);
    if (hook && hook->done) hook->done(0, fo, st);
  } else {
    const size_t groups = (fo + 15) / 16;
    for (int ci = 0; ci < nchunk; ++ci) {
      const size_t o0 = std::min(fo, 16 * (groups * ci / nchunk)), o1 = std::min(fo, 16 * (groups * (ci + 1) / nchunk));
      if (o1 <= o0) continue;
      C2RParams cc = c;
      cc.jbase = (int)o0;
      cc.J = (int)(o1 - o0);
      cc.J_all = (int)fo;
      cc.out = gw + o0 * f * k * k;
      nc += c2r_run(ws, m, cc, st);
      if (hook->done) hook->done(o0, o1, st);
    }
  }
  record(ws, 4, st);
  ws->last_launches = nl + ng + nc;
  if (ws->span_on) ++ws->span_next;
  ws->ctr[0] += S * f + S * fo;
  ws->ctr[1] += fo * f;
  ws->ctr[2] += (uint64_t)bins * fo * f * S;
}


}  // namespace

// ------------------------------------------------------------ C ABI
extern "C" {

int fftconv_b200_ws_create(const fftconv_b200_layer* configs, size_t count, int device,
                           fftconv_b200_ws** out) {
  return guarded(nullptr, [&] {
    if (!out) throw Error(FFTCONV_B200_INVALID_ARGUMENT, "out is NULL");
    *out = nullptr;
    if (count == 0 || !configs)
      throw Error(FFTCONV_B200_CONFIG_ERROR, "workspace: at least one layer config required");
    auto* ws = new fftconv_b200_ws;
    try {
      ws->device = device;
      for (size_t i = 0; i < count; ++i) {
        const auto& c = configs[i];
        validate_cfg(c);
        const uint64_t m = next_pow2(c.image);
        const uint64_t bins = m * (m / 2 + 1);
        ws->cap_x = std::max<uint64_t>(ws->cap_x, bins * c.batch * c.in_maps);
        ws->cap_w = std::max<uint64_t>(ws->cap_w, bins * c.out_maps * c.in_maps);
        ws->cap_y = std::max<uint64_t>(ws->cap_y, bins * c.batch * c.out_maps);
        ws->max_m = std::max<size_t>(ws->max_m, m);
      }
      DeviceGuard g(device);
      ws->di = dev_info(device);
      FCB_CUDA(cudaStreamCreateWithFlags(&ws->host_stream, cudaStreamNonBlocking));
      for (size_t i = 0; i < count; ++i)  // operand rows are maps or samples
        ws->amax_rows = std::max({ws->amax_rows, (size_t)configs[i].batch, (size_t)configs[i].in_maps,
                                  (size_t)configs[i].out_maps});
      FCB_CUDA(cudaMalloc(&ws->amax, 2 * ws->amax_rows * sizeof(unsigned long long)));
      FCB_CUDA(cudaMemset(ws->amax, 0, 2 * ws->amax_rows * sizeof(unsigned long long)));
      FCB_CUDA(cudaMalloc(&ws->gemm_path, sizeof(int)));
      FCB_CUDA(cudaMemset(ws->gemm_path, 0xff, sizeof(int)));
      FCB_CUDA(cudaStreamCreateWithFlags(&ws->h2d_stream, cudaStreamNonBlocking));
      FCB_CUDA(cudaStreamCreateWithFlags(&ws->d2h_stream, cudaStreamNonBlocking));
      for (auto& row : ws->pev)
        for (auto& e : row) FCB_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
      ws->pev_ready = true;
      FCB_CUDA(cudaEventCreateWithFlags(&ws->done_ev, cudaEventDisableTiming));
      // Size the frequency buffers for every registered layer and pass up
      // front, so timed calls never allocate.
      size_t na = 0, nb = 0, nd = 0;
      for (size_t i = 0; i < count; ++i) {
        const auto& c = configs[i];
        const size_t m = next_pow2(c.image);
        for (Pass p : {kFprop, kBprop, kAccGrad}) {
          const PassNeed need = pass_need(p, c.batch, c.in_maps, c.out_maps, m);
          na = std::max(na, need.a);
          nb = std::max(nb, need.b);
          nd = std::max(nd, need.d);
        }
      }
      set_arena(ws, na, nb, nd);
      for (size_t i = 0; i < count; ++i) ensure_large_scratch(ws, configs[i], next_pow2(configs[i].image));
    } catch (...) {
      fftconv_b200_ws_destroy(ws);
      throw;
    }
    *out = ws;
  });
}

void fftconv_b200_ws_destroy(fftconv_b200_ws* ws) {
  if (!ws) return;
  {
    DeviceGuard g(ws->device);
    for (float* p : {ws->freq, ws->st_in0, ws->st_in1, ws->st_out})
      if (p) cudaFree(p);
    if (ws->amax) cudaFree(ws->amax);
    if (ws->gemm_path) cudaFree(ws->gemm_path);
    if (ws->lscr) cudaFree(ws->lscr);
    if (ws->host_stream) cudaStreamDestroy(ws->host_stream);
    if (ws->h2d_stream) cudaStreamDestroy(ws->h2d_stream);
    if (ws->d2h_stream) cudaStreamDestroy(ws->d2h_stream);
    if (ws->pev_ready)
      for (auto& row : ws->pev)
        for (auto& e : row) cudaEventDestroy(e);
    if (ws->ev_ready)
      for (auto& e : ws->ev) cudaEventDestroy(e);
    if (ws->done_ev) cudaEventDestroy(ws->done_ev);
    if (ws->spans) cudaFree(ws->spans);
    if (ws->comm_ready) {
      cudaStreamDestroy(ws->comm_stream);
      for (auto& e : ws->chunk_ev) cudaEventDestroy(e);
      for (auto& e : ws->comm_ev) cudaEventDestroy(e);
    }
  }
  delete ws;
}

int fftconv_b200_set_gemm_kind(int kind) {
  if (kind != FFTCONV_B200_GEMM_F16X3 && kind != FFTCONV_B200_GEMM_TF32X3 && kind != FFTCONV_B200_GEMM_AUTO)
    return -1;
  return g_gemm_kind.exchange(kind);
}

int fftconv_b200_ws_set_gemm_kind(fftconv_b200_ws* ws, int kind) {
  if (!ws) return -1;
  if (kind != -1 && kind != FFTCONV_B200_GEMM_F16X3 && kind != FFTCONV_B200_GEMM_TF32X3 &&
      kind != FFTCONV_B200_GEMM_AUTO)
    return -1;
  const int prev = ws->gemm_kind < 0 ? -1 : ws->gemm_kind;
  ws->gemm_kind = kind;
  return prev;
}

int fftconv_b200_last_gemm_path(fftconv_b200_ws* ws) {
  if (!ws) return -1;
  int v = -1;
  DeviceGuard g(ws->device);
  if (cudaDeviceSynchronize() != cudaSuccess) return -1;
  if (cudaMemcpy(&v, ws->gemm_path, sizeof v, cudaMemcpyDeviceToHost) != cudaSuccess) return -1;
  return v;
}

const char* fftconv_b200_last_error(const fftconv_b200_ws* ws) {
  return ws ? ws->last_error.c_str() : g_last_error.c_str();
}

int fftconv_b200_ws_info(const fftconv_b200_ws* ws, uint64_t out[6]) {
  if (!ws || !out) return FFTCONV_B200_INVALID_ARGUMENT;
  out[0] = ws->max_m;
  out[1] = ws->cap_x;
  out[2] = ws->cap_w;
  out[3] = ws->cap_y;
  out[4] = (ws->cap_x + ws->cap_w + ws->cap_y) * 8;  // sizeof(std::complex<float>)
  out[5] = (ws->nA + ws->nB + ws->nD + ws->n_in0 + ws->n_in1 + ws->n_out) * sizeof(float);
  return FFTCONV_B200_OK;
}

int fftconv_b200_counters(const fftconv_b200_ws* ws, uint64_t out[3]) {
  if (!ws || !out) return FFTCONV_B200_INVALID_ARGUMENT;
  for (int i = 0; i < 3; ++i) out[i] = ws->ctr[i];
  return FFTCONV_B200_OK;
}

int fftconv_b200_reset_counters(fftconv_b200_ws* ws) {
  if (!ws) return FFTCONV_B200_INVALID_ARGUMENT;
  ws->ctr[0] = ws->ctr[1] = ws->ctr[2] = 0;
  return FFTCONV_B200_OK;
}

int fftconv_b200_forward(fftconv_b200_ws* ws, const float* x, size_t S, size_t f, size_t x_rows,
                         size_t x_cols, const float* w, size_t w_out, size_t w_in, size_t k,
                         float* y, void* stream) {
  if (!ws) return FFTCONV_B200_INVALID_ARGUMENT;
  return guarded(ws, [&] {
    DeviceGuard g(ws->device);
    order_after_last(ws, (cudaStream_t)stream);
    run_forward(ws, x, S, f, x_rows, x_cols, w, w_out, w_in, k, y, (cudaStream_t)stream);
    mark_done(ws, (cudaStream_t)stream);
  });
}

int fftconv_b200_forward_relu(fftconv_b200_ws* ws, const float* x, size_t S, size_t f, size_t x_rows,
                              size_t x_cols, const float* w, size_t w_out, size_t w_in, size_t k,
                              float* y, void* stream) {
  if (!ws) return FFTCONV_B200_INVALID_ARGUMENT;
  return guarded(ws, [&] {
    DeviceGuard g(ws->device);
    order_after_last(ws, (cudaStream_t)stream);
    run_forward(ws, x, S, f, x_rows, x_cols, w, w_out, w_in, k, y, (cudaStream_t)stream, true);
    mark_done(ws, (cudaStream_t)stream);
  });
}

int fftconv_b200_forward_fit(fftconv_b200_ws* ws, const float* x, size_t S, size_t f, size_t x_rows,
                             size_t x_cols, size_t image, const float* w, size_t w_out, size_t w_in, size_t k,
                             float* y, unsigned flags, void* stream) {
  if (!ws) return FFTCONV_B200_INVALID_ARGUMENT;
  return guarded(ws, [&] {
    DeviceGuard g(ws->device);
    order_after_last(ws, (cudaStream_t)stream);
    run_forward(ws, x, S, f, x_rows, x_cols, w, w_out, w_in, k, y, (cudaStream_t)stream,
                (flags & FFTCONV_B200_FIT_RELU) != 0, image);
    mark_done(ws, (cudaStream_t)stream);
  });
}

int fftconv_b200_grad_input_fit(fftconv_b200_ws* ws, const float* gy, size_t S, size_t fo, size_t gy_rows,
                                size_t gy_cols, const float* w, size_t w_out, size_t w_in, size_t k, float* gx,
                                size_t gx_size, void* stream) {
  if (!ws) return FFTCONV_B200_INVALID_ARGUMENT;
  return guarded(ws, [&] {
    DeviceGuard g(ws->device);
    order_after_last(ws, (cudaStream_t)stream);
    run_grad_input(ws, gy, S, fo, gy_rows, gy_cols, w, w_out, w_in, k, gx, (cudaStream_t)stream, gx_size);
    mark_done(ws, (cudaStream_t)stream);
  });
}

int fftconv_b200_grad_weight_fit(fftconv_b200_ws* ws, const float* gy, size_t Sg, size_t fo, size_t gy_rows,
                                 size_t gy_cols, const float* x, size_t Sx, size_t f, size_t x_rows, size_t x_cols,
                                 size_t image, float* gw, void* stream) {
  if (!ws) return FFTCONV_B200_INVALID_ARGUMENT;
  return guarded(ws, [&] {
    DeviceGuard g(ws->device);
    order_after_last(ws, (cudaStream_t)stream);
    run_grad_weight(ws, gy, Sg, fo, gy_rows, gy_cols, x, Sx, f, x_rows, x_cols, gw, (cudaStream_t)stream, false,
                    nullptr, image);
    mark_done(ws, (cudaStream_t)stream);
  });
}

int fftconv_b200_grad_input(fftconv_b200_ws* ws, const float* gy, size_t S, size_t fo,
                            size_t gy_rows, size_t gy_cols, const float* w, size_t w_out,
                            size_t w_in, size_t k, float* gx, void* stream) {
  if (!ws) return FFTCONV_B200_INVALID_ARGUMENT;
  return guarded(ws, [&] {
    DeviceGuard g(ws->device);
    order_after_last(ws, (cudaStream_t)stream);
    run_grad_input(ws, gy, S, fo, gy_rows, gy_cols, w, w_out, w_in, k, gx, (cudaStream_t)stream);
    mark_done(ws, (cudaStream_t)stream);
  });
}

int fftconv_b200_grad_weight(fftconv_b200_ws* ws, const float* gy, size_t S_gy, size_t fo,
                             size_t gy_rows, size_t gy_cols, const float* x, size_t S_x,
                             size_t f, size_t x_rows, size_t x_cols, float* gw, void* stream) {
  if (!ws) return FFTCONV_B200_INVALID_ARGUMENT;
  return guarded(ws, [&] {
    DeviceGuard g(ws->device);
    order_after_last(ws, (cudaStream_t)stream);
    run_grad_weight(ws, gy, S_gy, fo, gy_rows, gy_cols, x, S_x, f, x_rows, x_cols, gw,
                    (cudaStream_t)stream);
    mark_done(ws, (cudaStream_t)stream);
  });
}

// ---- minibatch-sharded accGrad (NCCL over NVLink) ----------------------

int fftconv_b200_nccl_get_unique_id(void* id) {
  return guarded(nullptr, [&] {
    if (!id) throw Error(FFTCONV_B200_INVALID_ARGUMENT, "id is NULL");
    ncclUniqueId u;
    FCB_NCCL(nccl_api().get_unique_id(&u));
    std::memcpy(id, &u, sizeof u);
  });
}

int fftconv_b200_nccl_comm_create(const void* id, int nranks, int rank, int device, void** comm) {
  return guarded(nullptr, [&] {
    if (!id || !comm) throw Error(FFTCONV_B200_INVALID_ARGUMENT, "id / comm is NULL");
    if (nranks < 1 || rank < 0 || rank >= nranks) throw Error(FFTCONV_B200_INVALID_ARGUMENT, "bad nranks / rank");
    *comm = nullptr;
    ncclUniqueId u;
    std::memcpy(&u, id, sizeof u);
    DeviceGuard g(device);
    FCB_CUDA(cudaSetDevice(device));
    ncclComm_t c = nullptr;
    FCB_NCCL(nccl_api().comm_init_rank(&c, nranks, u, rank));
    *comm = c;
  });
}

int fftconv_b200_nccl_comm_destroy(void* comm) {
  return guarded(nullptr, [&] {
    if (comm) FCB_NCCL(nccl_api().comm_destroy(reinterpret_cast<ncclComm_t>(comm)));
  });
}

int fftconv_b200_grad_weight_sharded(fftconv_b200_ws* ws, const float* gy, size_t S_gy, size_t fo,
                                     size_t gy_rows, size_t gy_cols, const float* x, size_t S_x, size_t f,
                                     size_t x_rows, size_t x_cols, float* gw, void* comm, int chunks,
                                     unsigned flags, void* stream) {
  if (!ws) return FFTCONV_B200_INVALID_ARGUMENT;
  return guarded(ws, [&] {
    DeviceGuard g(ws->device);
    const cudaStream_t st = (cudaStream_t)stream;
    if (!comm) throw Error(FFTCONV_B200_INVALID_ARGUMENT, "grad_weight_sharded: comm is NULL");
    const NcclApi& api = nccl_api();
    if (!ws->comm_ready) {
      FCB_CUDA(cudaStreamCreateWithFlags(&ws->comm_stream, cudaStreamNonBlocking));
      for (auto& e : ws->chunk_ev) FCB_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
      for (auto& e : ws->comm_ev) FCB_CUDA(cudaEventCreate(&e));
      ws->comm_ready = true;
    }
    order_after_last(ws, st);
    int ci = 0;
    bool first = true;
    auto reduce_rows = [&](size_t o0, size_t o1, size_t per_row, cudaStream_t s_) {
      // the all-reduce of rows [o0, o1) waits for the launch that wrote them
      FCB_CUDA(cudaEventRecord(ws->chunk_ev[ci], s_));
      FCB_CUDA(cudaStreamWaitEvent(ws->comm_stream, ws->chunk_ev[ci], 0));
      if (first && ws->timing) FCB_CUDA(cudaEventRecord(ws->comm_ev[1], ws->comm_stream));
      first = false;
      FCB_NCCL(api.all_reduce(gw + o0 * per_row, gw + o0 * per_row, (o1 - o0) * per_row, ncclFloat32, ncclSum,
                              reinterpret_cast<ncclComm_t>(comm), ws->comm_stream));
      ci = std::min(ci + 1, kMaxChunks);
    };
    if (S_gy == 0 && S_x == 0) {
      // empty shard (world > S): contribute zeros so the peers' all-reduce completes
      require_nonzero(fo, gy_rows, gy_cols, 1, "Tensor4");
      require_nonzero(f, x_rows, x_cols, 1, "Tensor4");
      if (gy_rows > x_rows) throw Error(FFTCONV_B200_SIZE_ERROR, "grad_weight_fft: gradient larger than input");
      const size_t k = x_rows - gy_rows + 1;
      FCB_CUDA(cudaMemsetAsync(gw, 0, fo * f * k * k * sizeof(float), st));
      if (ws->timing) FCB_CUDA(cudaEventRecord(ws->comm_ev[0], st));
      reduce_rows(0, fo, f * k * k, st);
    } else {
      const size_t k = (gy_rows <= x_rows) ? x_rows - gy_rows + 1 : 1;
      ChunkHook hook;
      hook.chunks = std::max(1, std::min(chunks, kMaxChunks));
      hook.done = [&](size_t o0, size_t o1, cudaStream_t s_) { reduce_rows(o0, o1, f * k * k, s_); };
      run_grad_weight(ws, gy, S_gy, fo, gy_rows, gy_cols, x, S_x, f, x_rows, x_cols, gw, st, false, &hook);
      if (ws->timing) FCB_CUDA(cudaEventRecord(ws->comm_ev[0], st));  // K4 end
    }
    if (ws->timing) FCB_CUDA(cudaEventRecord(ws->comm_ev[2], ws->comm_stream));
    // the caller's stream resumes once every row is reduced -- now, or (ASYNC)
    // at fftconv_b200_comm_wait, so a training step's later layers overlap it
    FCB_CUDA(cudaEventRecord(ws->chunk_ev[kMaxChunks], ws->comm_stream));
    if (!(flags & FFTCONV_B200_SHARDED_ASYNC)) FCB_CUDA(cudaStreamWaitEvent(st, ws->chunk_ev[kMaxChunks], 0));
    ws->comm_timed = ws->timing;
    mark_done(ws, st);
  });
}

int fftconv_b200_comm_wait(fftconv_b200_ws* ws, void* stream) {
  if (!ws) return FFTCONV_B200_INVALID_ARGUMENT;
  return guarded(ws, [&] {
    if (!ws->comm_ready) return;
    DeviceGuard g(ws->device);
    FCB_CUDA(cudaStreamWaitEvent((cudaStream_t)stream, ws->chunk_ev[kMaxChunks], 0));
  });
}

int fftconv_b200_comm_ms(fftconv_b200_ws* ws, float out[2]) {
  if (!ws || !out) return FFTCONV_B200_INVALID_ARGUMENT;
  return guarded(ws, [&] {
    if (!ws->comm_timed) throw Error(FFTCONV_B200_INVALID_ARGUMENT, "no timed sharded call yet (enable stage timing)");
    DeviceGuard g(ws->device);
    FCB_CUDA(cudaEventSynchronize(ws->comm_ev[2]));
    float span = 0.f, exposed = 0.f;
    FCB_CUDA(cudaEventElapsedTime(&span, ws->comm_ev[1], ws->comm_ev[2]));
    FCB_CUDA(cudaEventElapsedTime(&exposed, ws->comm_ev[0], ws->comm_ev[2]));
    out[0] = span;
    out[1] = std::max(0.f, exposed);
  });
}

// ---- host-pointer entry points ---------------------------------------
// The drop-in for Tensor4/Weights4 storage: copy in, compute, copy out.
// Each call is pipelined over minibatch chunks (fprop/bprop are independent
// per sample; accGrad sums per-chunk gradients into the output): the H2D
// copies of chunk c+1 run on h2d_stream while chunk c computes on
// host_stream and chunk c-1 drains on d2h_stream, so a call costs about one
// PCIe transfer of its inputs instead of H2D + compute + D2H in series.

namespace {

// Chunks for a host call moving `bytes` of per-sample input, `mb` MB each:
// small enough that the exposed first H2D / last D2H stays short, large
// enough that each chunk's fixed work (the W-side transforms, one GEMM
// launch, accGrad's full-size K4) still hides under the next chunk's copy.
// Measured per-op optima at the paper point: fprop 12 MB, bprop 6 MB,
// accGrad 32 MB (its per-chunk K4 and GEMM do not shrink with the chunk).
// FFTCONV_B200_HOST_CHUNK_MB overrides all three (tuning).
int host_chunks(size_t S, size_t bytes, size_t m, size_t mb) {
  if (m < 4) return 1;  // the small-plane kernels do not accumulate
  static const size_t over = [] {
    const char* e = getenv("FFTCONV_B200_HOST_CHUNK_MB");
    return (size_t)((e && atoi(e) > 0) ? atoi(e) : 0);
  }();
  const size_t chunk = (over ? over : mb) << 20;
  const size_t c = (bytes + chunk - 1) / chunk;
  return (int)std::max<size_t>(1, std::min<size_t>({c, (size_t)kMaxChunks, S}));
}

std::pair<size_t, size_t> chunk_range(size_t S, int C, int c) {
  const size_t base = S / C, extra = S % C;
  const size_t b0 = c * base + std::min<size_t>(c, extra);
  return {b0, b0 + base + ((size_t)c < extra ? 1 : 0)};
}

void h2d(fftconv_b200_ws* ws, float* dst, const float* src, size_t n) {
  FCB_CUDA(cudaMemcpyAsync(dst, src, n * sizeof(float), cudaMemcpyHostToDevice, ws->h2d_stream));
}

}  // namespace

int fftconv_b200_forward_host(fftconv_b200_ws* ws, const float* x, size_t S, size_t f,
                              size_t x_rows, size_t x_cols, const float* w, size_t w_out,
                              size_t w_in, size_t k, float* y, unsigned threads) {
  (void)threads;
  if (!ws) return FFTCONV_B200_INVALID_ARGUMENT;
  return guarded(ws, [&] {
    DeviceGuard g(ws->device);
    // Shape checks first so errors never touch the device.
    require_nonzero(S, f, x_rows, x_cols, "Tensor4");
    require_nonzero(w_out, w_in, k, 1, "Weights4");
    if (!(x_rows == x_cols && w_in == f && k <= x_rows)) {  // raises the reference's error
      run_forward(ws, nullptr, S, f, x_rows, x_cols, nullptr, w_out, w_in, k, nullptr,
                  ws->host_stream);
      return;
    }
    const size_t n = x_rows, no = n - k + 1, fo = w_out;
    const size_t m = prepare(ws, fftconv_b200_layer{k, n, f, fo, S});
    const size_t px = f * n * n, py = fo * no * no, nw = fo * f * k * k;
    grow(ws->st_in0, ws->n_in0, S * px);
    grow(ws->st_in1, ws->n_in1, nw);
    grow(ws->st_out, ws->n_out, S * py);
    const int C = host_chunks(S, S * px * sizeof(float), m, 12);
    order_after_last(ws, ws->host_stream);
    uint64_t saved[3];
    std::memcpy(saved, ws->ctr, sizeof saved);
    h2d(ws, ws->st_in1, w, nw);
    for (int c = 0; c < C; ++c) {  // every copy queued first: the link never idles on host work
      const auto [b0, b1] = chunk_range(S, C, c);
      h2d(ws, ws->st_in0 + b0 * px, x + b0 * px, (b1 - b0) * px);
      FCB_CUDA(cudaEventRecord(ws->pev[0][c], ws->h2d_stream));
    }
    for (int c = 0; c < C; ++c) {
      const auto [b0, b1] = chunk_range(S, C, c);
      FCB_CUDA(cudaStreamWaitEvent(ws->host_stream, ws->pev[0][c], 0));
      run_forward(ws, ws->st_in0 + b0 * px, b1 - b0, f, n, n, ws->st_in1, fo, f, k,
                  ws->st_out + b0 * py, ws->host_stream);
      FCB_CUDA(cudaEventRecord(ws->pev[1][c], ws->host_stream));
      FCB_CUDA(cudaStreamWaitEvent(ws->d2h_stream, ws->pev[1][c], 0));
      FCB_CUDA(cudaMemcpyAsync(y + b0 * py, ws->st_out + b0 * py, (b1 - b0) * py * sizeof(float),
                               cudaMemcpyDeviceToHost, ws->d2h_stream));
    }
    FCB_CUDA(cudaStreamSynchronize(ws->d2h_stream));
    ws->has_last = false;  // everything this call enqueued has completed
    const uint64_t bins = m * (m / 2 + 1);  // one call = one reference forward
    ws->ctr[0] = saved[0] + S * f + fo * f;
    ws->ctr[1] = saved[1] + S * fo;
    ws->ctr[2] = saved[2] + bins * fo * f * S;
  });
}

int fftconv_b200_grad_input_host(fftconv_b200_ws* ws, const float* gy, size_t S, size_t fo,
                                 size_t gy_rows, size_t gy_cols, const float* w, size_t w_out,
                                 size_t w_in, size_t k, float* gx, unsigned threads) {
  (void)threads;
  if (!ws) return FFTCONV_B200_INVALID_ARGUMENT;
  return guarded(ws, [&] {
    DeviceGuard g(ws->device);
    require_nonzero(S, fo, gy_rows, gy_cols, "Tensor4");
    require_nonzero(w_out, w_in, k, 1, "Weights4");
    if (!(gy_rows == gy_cols && w_out == fo)) {
      run_grad_input(ws, nullptr, S, fo, gy_rows, gy_cols, nullptr, w_out, w_in, k, nullptr,
                     ws->host_stream);
      return;
    }
    const size_t no = gy_rows, n = no + k - 1, f = w_in;
    const size_t m = prepare(ws, fftconv_b200_layer{k, n, f, fo, S});
    const size_t pgy = fo * no * no, pgx = f * n * n, nw = fo * f * k * k;
    grow(ws->st_in0, ws->n_in0, S * pgy);
    grow(ws->st_in1, ws->n_in1, nw);
    grow(ws->st_out, ws->n_out, S * pgx);
    const int C = host_chunks(S, S * pgy * sizeof(float), m, 6);
    order_after_last(ws, ws->host_stream);
    uint64_t saved[3];
    std::memcpy(saved, ws->ctr, sizeof saved);
    h2d(ws, ws->st_in1, w, nw);
    for (int c = 0; c < C; ++c) {
      const auto [b0, b1] = chunk_range(S, C, c);
      h2d(ws, ws->st_in0 + b0 * pgy, gy + b0 * pgy, (b1 - b0) * pgy);
      FCB_CUDA(cudaEventRecord(ws->pev[0][c], ws->h2d_stream));
    }
    for (int c = 0; c < C; ++c) {
      const auto [b0, b1] = chunk_range(S, C, c);
      FCB_CUDA(cudaStreamWaitEvent(ws->host_stream, ws->pev[0][c], 0));
      run_grad_input(ws, ws->st_in0 + b0 * pgy, b1 - b0, fo, no, no, ws->st_in1, fo, f, k,
                     ws->st_out + b0 * pgx, ws->host_stream);
      FCB_CUDA(cudaEventRecord(ws->pev[1][c], ws->host_stream));
      FCB_CUDA(cudaStreamWaitEvent(ws->d2h_stream, ws->pev[1][c], 0));
      FCB_CUDA(cudaMemcpyAsync(gx + b0 * pgx, ws->st_out + b0 * pgx,
                               (b1 - b0) * pgx * sizeof(float), cudaMemcpyDeviceToHost,
                               ws->d2h_stream));
    }
    FCB_CUDA(cudaStreamSynchronize(ws->d2h_stream));
    ws->has_last = false;  // everything this call enqueued has completed
    const uint64_t bins = m * (m / 2 + 1);
    ws->ctr[0] = saved[0] + S * fo + fo * f;
    ws->ctr[1] = saved[1] + S * f;
    ws->ctr[2] = saved[2] + bins * fo * f * S;
  });
}

namespace {
// grad_weight on host buffers (chunked H2D / compute pipeline); with `comm`
// the finished gw is all-reduced over the ranks before the D2H (the
// minibatch-sharded host entry point; an empty shard contributes zeros).
void grad_weight_host_impl(fftconv_b200_ws* ws, const float* gy, size_t S_gy, size_t fo, size_t gy_rows,
                           size_t gy_cols, const float* x, size_t S_x, size_t f, size_t x_rows, size_t x_cols,
                           float* gw, void* comm) {
  DeviceGuard g(ws->device);
  const bool empty = comm && S_gy == 0 && S_x == 0;
  if (!empty) {
    require_nonzero(S_gy, fo, gy_rows, gy_cols, "Tensor4");
    require_nonzero(S_x, f, x_rows, x_cols, "Tensor4");
  } else {
    require_nonzero(fo, gy_rows, gy_cols, 1, "Tensor4");
    require_nonzero(f, x_rows, x_cols, 1, "Tensor4");
  }
  if (!(gy_rows == gy_cols && x_rows == x_cols && S_gy == S_x && gy_rows <= x_rows)) {
    run_grad_weight(ws, nullptr, S_gy, fo, gy_rows, gy_cols, nullptr, S_x, f, x_rows, x_cols, nullptr,
                    ws->host_stream);  // raises the reference's error
    return;
  }
  const size_t S = S_x, no = gy_rows, n = x_rows, k = n - no + 1;
  const size_t m = empty ? next_pow2(n) : prepare(ws, fftconv_b200_layer{k, n, f, fo, S});
  const size_t pgy = fo * no * no, px = f * n * n, ngw = fo * f * k * k;
  grow(ws->st_in0, ws->n_in0, std::max<size_t>(S, 1) * pgy);
  grow(ws->st_in1, ws->n_in1, std::max<size_t>(S, 1) * px);
  grow(ws->st_out, ws->n_out, ngw);
  order_after_last(ws, ws->host_stream);
  uint64_t saved[3];
  std::memcpy(saved, ws->ctr, sizeof saved);
  if (empty) {
    FCB_CUDA(cudaMemsetAsync(ws->st_out, 0, ngw * sizeof(float), ws->host_stream));
  } else {
    const int C = host_chunks(S, S * (pgy + px) * sizeof(float), m, 32);
    for (int c = 0; c < C; ++c) {
      const auto [b0, b1] = chunk_range(S, C, c);
      h2d(ws, ws->st_in0 + b0 * pgy, gy + b0 * pgy, (b1 - b0) * pgy);
      h2d(ws, ws->st_in1 + b0 * px, x + b0 * px, (b1 - b0) * px);
      FCB_CUDA(cudaEventRecord(ws->pev[0][c], ws->h2d_stream));
    }
    for (int c = 0; c < C; ++c) {
      const auto [b0, b1] = chunk_range(S, C, c);
      FCB_CUDA(cudaStreamWaitEvent(ws->host_stream, ws->pev[0][c], 0));
      // gw = sum over minibatch chunks (batch decomposability)
      run_grad_weight(ws, ws->st_in0 + b0 * pgy, b1 - b0, fo, no, no, ws->st_in1 + b0 * px, b1 - b0, f, n, n,
                      ws->st_out, ws->host_stream, /*accum=*/c > 0);
    }
  }
  if (comm)
    FCB_NCCL(nccl_api().all_reduce(ws->st_out, ws->st_out, ngw, ncclFloat32, ncclSum,
                                   reinterpret_cast<ncclComm_t>(comm), ws->host_stream));
  FCB_CUDA(cudaMemcpyAsync(gw, ws->st_out, ngw * sizeof(float), cudaMemcpyDeviceToHost, ws->host_stream));
  FCB_CUDA(cudaStreamSynchronize(ws->host_stream));
  ws->has_last = false;
  if (!empty) {
    const uint64_t bins = m * (m / 2 + 1);
    ws->ctr[0] = saved[0] + S * f + S * fo;
    ws->ctr[1] = saved[1] + fo * f;
    ws->ctr[2] = saved[2] + bins * fo * f * S;
  }
}
}  // namespace

int fftconv_b200_grad_weight_host(fftconv_b200_ws* ws, const float* gy, size_t S_gy, size_t fo,
                                  size_t gy_rows, size_t gy_cols, const float* x, size_t S_x,
                                  size_t f, size_t x_rows, size_t x_cols, float* gw,
                                  unsigned threads) {
  (void)threads;
  if (!ws) return FFTCONV_B200_INVALID_ARGUMENT;
  return guarded(ws, [&] {
    grad_weight_host_impl(ws, gy, S_gy, fo, gy_rows, gy_cols, x, S_x, f, x_rows, x_cols, gw, nullptr);
  });
}

int fftconv_b200_grad_weight_sharded_host(fftconv_b200_ws* ws, const float* gy, size_t S_gy, size_t fo,
                                          size_t gy_rows, size_t gy_cols, const float* x, size_t S_x, size_t f,
                                          size_t x_rows, size_t x_cols, float* gw, void* comm, unsigned threads) {
  (void)threads;
  if (!ws) return FFTCONV_B200_INVALID_ARGUMENT;
  return guarded(ws, [&] {
    if (!comm) throw Error(FFTCONV_B200_INVALID_ARGUMENT, "grad_weight_sharded_host: comm is NULL");
    grad_weight_host_impl(ws, gy, S_gy, fo, gy_rows, gy_cols, x, S_x, f, x_rows, x_cols, gw, comm);
  });
}

int fftconv_b200_set_stage_timing(fftconv_b200_ws* ws, int enable) {
  if (!ws) return FFTCONV_B200_INVALID_ARGUMENT;
  ws->timing = enable != 0;
  return FFTCONV_B200_OK;
}

int fftconv_b200_stage_ms(fftconv_b200_ws* ws, float out[4]) {
  if (!ws || !out) return FFTCONV_B200_INVALID_ARGUMENT;
  return guarded(ws, [&] {
    if (!ws->ev_ready) throw Error(FFTCONV_B200_INVALID_ARGUMENT, "stage timing not enabled");
    DeviceGuard g(ws->device);
    FCB_CUDA(cudaEventSynchronize(ws->ev[4]));
    for (int i = 0; i < 4; ++i) FCB_CUDA(cudaEventElapsedTime(&out[i], ws->ev[i], ws->ev[i + 1]));
  });
}

int fftconv_b200_set_span_timing(fftconv_b200_ws* ws, int enable) {
  if (!ws) return FFTCONV_B200_INVALID_ARGUMENT;
  return guarded(ws, [&] {
    DeviceGuard g(ws->device);
    ws->span_on = 0;
    if (!enable) return;
    const size_t words = 2 * 3 * (size_t)kSpanSlots;
    if (!ws->spans) FCB_CUDA(cudaMalloc(&ws->spans, words * sizeof(unsigned long long)));
    FCB_CUDA(cudaDeviceSynchronize());
    FCB_CUDA(cudaMemset(ws->spans, 0xff, words / 2 * sizeof(unsigned long long)));  // starts: +inf
    FCB_CUDA(cudaMemset(ws->spans + words / 2, 0, words / 2 * sizeof(unsigned long long)));
    ws->span_next = 0;
    ws->span_on = 1;
  });
}

int fftconv_b200_span_ms(fftconv_b200_ws* ws, float* out, int max_ops) {
  if (!ws || !out) return -FFTCONV_B200_INVALID_ARGUMENT;
  int n = -FFTCONV_B200_INVALID_ARGUMENT;
  const int code = guarded(ws, [&] {
    if (!ws->spans) throw Error(FFTCONV_B200_INVALID_ARGUMENT, "span timing never enabled");
    DeviceGuard g(ws->device);
    FCB_CUDA(cudaDeviceSynchronize());
    std::vector<unsigned long long> h(2 * 3 * (size_t)kSpanSlots);
    FCB_CUDA(cudaMemcpy(h.data(), ws->spans, h.size() * sizeof(unsigned long long), cudaMemcpyDeviceToHost));
    n = std::min({ws->span_next, kSpanSlots, max_ops});
    for (int i = 0; i < n; ++i)
      for (int k = 0; k < 3; ++k) {
        const unsigned long long b = h[(size_t)i * 3 + k], e = h[(size_t)kSpanEndOff + (size_t)i * 3 + k];
        out[i * 3 + k] = (b == ~0ull || e == 0 || e < b) ? -1.f : (float)((e - b) * 1e-6);
      }
  });
  return code == FFTCONV_B200_OK ? n : -code;
}

int fftconv_b200_last_launch_count(const fftconv_b200_ws* ws) {
  return ws ? ws->last_launches : -1;
}

// ---- packed-spectrum API ---------------------------------------------

namespace {
struct SpecScratch {
  size_t f_bytes, l_elems, total;
};
SpecScratch spectrum_scratch(size_t planes, size_t m) {
  const size_t bins = m * (m / 2 + 1), kp = round_up(std::max<size_t>(planes, 1), 16);
  SpecScratch s;
  s.f_bytes = round_up(bins * kp * sizeof(float2), 256);
  s.l_elems = (m == kL) ? large_scratch_elems(planes, planes) : 0;
  s.total = s.f_bytes + s.l_elems * sizeof(float2);
  return s;
}
void spectrum_checks(size_t planes, size_t m, const void* scratch, size_t scratch_bytes) {
  if (m == 0 || (m & (m - 1)))  // FftPlan (fft.hpp:23-26)
    throw Error(FFTCONV_B200_PLAN_ERROR, "fft plan: size " + std::to_string(m) + " is not a power of 2");
  if (m > kL) size_unsupported(m);
  if (planes == 0) throw Error(FFTCONV_B200_SIZE_ERROR, "HalfSpectrum: all dimensions must be >= 1");
  if (!scratch || scratch_bytes < spectrum_scratch(planes, m).total)
    throw Error(FFTCONV_B200_INVALID_ARGUMENT, "spectrum: scratch smaller than fftconv_b200_spectrum_scratch_bytes");
}
int ew_blocks(long long n) { return (int)std::max<long long>(1, std::min<long long>((n + 255) / 256, 148LL * 16)); }
}  // namespace

size_t fftconv_b200_spectrum_scratch_bytes(size_t planes, size_t m) {
  if (m == 0 || (m & (m - 1)) || m > kL) return 0;
  return spectrum_scratch(planes, m).total;
}

int fftconv_b200_fft_2d_real_batch(const float* planes, size_t P, size_t m, float* spec, void* scratch,
                                   size_t scratch_bytes, void* stream) {
  return guarded(nullptr, [&] {
    spectrum_checks(P, m, scratch, scratch_bytes);
    const SpecScratch ss = spectrum_scratch(P, m);
    const cudaStream_t st = (cudaStream_t)stream;
    int dev = 0;
    FCB_CUDA(cudaGetDevice(&dev));
    float* F = static_cast<float*>(scratch);
    const size_t kp = round_up(P, 16);
    // planes as the K index of one operand row: F[t][0][2 kp] (pad planes zero)
    R2CParams p{planes, F, 0, (long long)(m * m), 1, (int)P, (int)kp, (int)m, (int)(m | 1)};
    if (m == kL)
      launch_r2c_large(p, reinterpret_cast<float2*>(static_cast<char*>(scratch) + ss.f_bytes), ss.l_elems, st);
    else
      launch_r2c_one(m, p, st, dev_info(dev));
    const long long n = (long long)P * m * (m / 2 + 1);
    spectrum_pack_ref_kernel<<<ew_blocks(n), 256, 0, st>>>(reinterpret_cast<const float2*>(F), (long long)kp,
                                                           (int)m, (long long)P, reinterpret_cast<float2*>(spec));
    FCB_CUDA(cudaGetLastError());
  });
}

int fftconv_b200_ifft_2d_real_batch(const float* spec, size_t P, size_t m, float* planes, void* scratch,
                                    size_t scratch_bytes, void* stream) {
  return guarded(nullptr, [&] {
    spectrum_checks(P, m, scratch, scratch_bytes);
    const SpecScratch ss = spectrum_scratch(P, m);
    const cudaStream_t st = (cudaStream_t)stream;
    int dev = 0;
    FCB_CUDA(cudaGetDevice(&dev));
    float* F = static_cast<float*>(scratch);
    const size_t ld = round_up(P, 16);  // complex per bin (even, 16-B aligned rows for the TMA maps)
    const long long n = (long long)(m / 2 + 1) * m * ld;
    spectrum_unpack_ref_kernel<<<ew_blocks(n), 256, 0, st>>>(reinterpret_cast<const float2*>(spec), (int)m,
                                                             (long long)P, (long long)ld,
                                                             reinterpret_cast<float2*>(F));
    FCB_CUDA(cudaGetLastError());
    // bin-major product P[t][0][ld]: planes (0, j) -> planes + j m^2, full m x m, 1/m^2
    C2RParams c{F, planes, 0, (long long)(m * m), 1, (int)P, (int)m, 0, 0, 1.0f / (float)(m * m), (int)ld};
    if (m == kL)
      launch_c2r_large(c, reinterpret_cast<float2*>(static_cast<char*>(scratch) + ss.f_bytes), ss.l_elems, st);
    else
      launch_c2r(m, c, st, dev_info(dev));
  });
}

// ---- unit-level test hooks -------------------------------------------

int fftconv_b200_debug_r2c(const float* in, size_t planes, size_t src, size_t m, float* out,
                           void* stream) {
  return guarded(nullptr, [&] {
    if (next_pow2(src) > m || (m & (m - 1)))
      throw Error(FFTCONV_B200_PLAN_ERROR, "debug_r2c: bad m");
    // R = planes rows, J = 1: F[t][p][2*16]; copy out[p][t] with a strided 2-D memcpy.
    const size_t bins = m * (m / 2 + 1), kp = 16;
    float* F = nullptr;
    FCB_CUDA(cudaMalloc(&F, bins * planes * kp * 2 * sizeof(float)));
    R2CParams p{in, F, (long long)(src * src), 0, (int)planes, 1, (int)kp, (int)src,
                (int)(src | 1)};
    float2* scr = nullptr;
    if (m == kL) {
      FCB_CUDA(cudaMalloc(&scr, large_scratch_elems(planes, planes) * sizeof(float2)));
      launch_r2c_large(p, scr, large_scratch_elems(planes, planes), (cudaStream_t)stream);
    } else {
      launch_r2c_one(m, p, (cudaStream_t)stream, dev_info(0));
    }
    // F[(t*planes + p)*32 + 0..1] -> out[(p*bins + t)*2]
    for (size_t pl = 0; pl < planes; ++pl)
      FCB_CUDA(cudaMemcpy2DAsync(out + pl * bins * 2, 2 * sizeof(float), F + pl * kp * 2,
                                 planes * kp * 2 * sizeof(float), 2 * sizeof(float), bins,
                                 cudaMemcpyDeviceToDevice, (cudaStream_t)stream));
    FCB_CUDA(cudaStreamSynchronize((cudaStream_t)stream));
    cudaFree(F);
    if (scr) cudaFree(scr);
  });
}

int fftconv_b200_debug_c2r(const float* in, size_t planes, size_t m, size_t crop, float* out,
                           void* stream) {
  return guarded(nullptr, [&] {
    if ((m & (m - 1)) || crop > m) throw Error(FFTCONV_B200_PLAN_ERROR, "debug_c2r: bad m");
    // in[p][t] -> P[t][0][p] (R = 1, J = planes)
    const size_t bins = m * (m / 2 + 1), ld = round_up(planes, 2);
    float* P = nullptr;
    FCB_CUDA(cudaMalloc(&P, bins * ld * 2 * sizeof(float)));
    for (size_t pl = 0; pl < planes; ++pl)
      FCB_CUDA(cudaMemcpy2DAsync(P + pl * 2, ld * 2 * sizeof(float), in + pl * bins * 2,
                                 2 * sizeof(float), 2 * sizeof(float), bins,
                                 cudaMemcpyDeviceToDevice, (cudaStream_t)stream));
    C2RParams p{P, out, 0, (long long)(crop * crop), 1, (int)planes, (int)crop, 0, 0,
                1.0f / (float)(m * m), (int)round_up(planes, 2)};
    float2* scr = nullptr;
    if (m == kL) {
      FCB_CUDA(cudaMalloc(&scr, large_scratch_elems(planes, planes) * sizeof(float2)));
      launch_c2r_large(p, scr, large_scratch_elems(planes, planes), (cudaStream_t)stream);
    } else {
      launch_c2r(m, p, (cudaStream_t)stream, dev_info(0));
    }
    FCB_CUDA(cudaStreamSynchronize((cudaStream_t)stream));
    cudaFree(P);
    if (scr) cudaFree(scr);
  });
}

int fftconv_b200_debug_cgemm(const float* a, const float* b, float* out, size_t bins, size_t M,
                             size_t N, size_t K, int mode, void* stream) {
  return guarded(nullptr, [&] {
    if (mode < 0 || mode > 2) throw Error(FFTCONV_B200_INVALID_ARGUMENT, "mode");
    int dev = 0;
    FCB_CUDA(cudaGetDevice(&dev));
    const DevInfo di = dev_info(dev);
    const size_t kp = round_up(K, 16);
    float *A = nullptr, *B = nullptr;
    FCB_CUDA(cudaMalloc(&A, bins * M * kp * 2 * sizeof(float)));
    FCB_CUDA(cudaMalloc(&B, bins * N * kp * 2 * sizeof(float)));
    cudaStream_t st = (cudaStream_t)stream;
    FCB_CUDA(cudaMemsetAsync(A, 0, bins * M * kp * 2 * sizeof(float), st));
    FCB_CUDA(cudaMemsetAsync(B, 0, bins * N * kp * 2 * sizeof(float), st));
    FCB_CUDA(cudaMemcpy2DAsync(A, kp * 2 * sizeof(float), a, K * 2 * sizeof(float),
                               K * 2 * sizeof(float), bins * M, cudaMemcpyDeviceToDevice, st));
    FCB_CUDA(cudaMemcpy2DAsync(B, kp * 2 * sizeof(float), b, K * 2 * sizeof(float),
                               K * 2 * sizeof(float), bins * N, cudaMemcpyDeviceToDevice, st));
    if (mode == 1)  // A . B = A . conj(conj(B))
      conj_inplace_kernel<<<256, 256, 0, st>>>(reinterpret_cast<float2*>(B),
                                               (long long)(bins * N * kp));
    // per-row maxima for the fp16 routes; under "auto" this hook always
    // launches the fp16x3 / 3xTF32 pair, so the selection itself is tested
    unsigned long long* amax = nullptr;
    FCB_CUDA(cudaMalloc(&amax, (M + N) * sizeof(unsigned long long)));
    FCB_CUDA(cudaMemsetAsync(amax, 0, (M + N) * sizeof(unsigned long long), st));
    absmax_rows_kernel<<<(unsigned)M, 256, 0, st>>>(A, (long long)bins, (int)M, (int)(kp * 2), amax);
    absmax_rows_kernel<<<(unsigned)N, 256, 0, st>>>(B, (long long)bins, (int)N, (int)(kp * 2), amax + M);
    const int kind = g_gemm_kind.load();
    const GemmRoute route = kind == FFTCONV_B200_GEMM_TF32X3 ? kRouteTf32
                            : kind == FFTCONV_B200_GEMM_F16X3 ? kRouteF16
                                                              : kRouteAuto;
    launch_gemm(A, B, out, bins, M, N, kp, mode == 2 ? -1.0f : 1.0f, kBinMajor, M, di, st, route, amax, amax + M);
    FCB_CUDA(cudaStreamSynchronize(st));
    cudaFree(A);
    cudaFree(B);
    cudaFree(amax);
  });
}

// ---- layer-stack stages (layers.hpp) -----------------------------------

namespace {
int ew_grid(long long n) {
  return (int)std::max<long long>(1, std::min<long long>((n + 255) / 256, 148LL * 16));
}
// plane-walking layer kernels (layers.cuh): one 256-thread block per plane,
// at most 8 resident blocks per SM
int plane_grid(long long planes) { return (int)std::max<long long>(1, std::min<long long>(planes, 148LL * 8)); }
}  // namespace

int fftconv_b200_relu_forward(const float* x, float* y, size_t n, void* stream) {
  return guarded(nullptr, [&] {
    cudaStream_t st = (cudaStream_t)stream;
    const long long n4 = (long long)n / 4;
    if (n4) relu_fwd_kernel<<<ew_grid(n4), 256, 0, st>>>(reinterpret_cast<const float4*>(x),
                                                       reinterpret_cast<float4*>(y), n4);
    if (n % 4) relu_fwd_tail<<<1, 4, 0, st>>>(x, y, 4 * n4, (long long)n);
    FCB_CUDA(cudaGetLastError());
  });
}

int fftconv_b200_relu_backward(const float* gy, const float* x, float* gx, size_t n,
                               void* stream) {
  return guarded(nullptr, [&] {
    cudaStream_t st = (cudaStream_t)stream;
    const long long n4 = (long long)n / 4;
    if (n4)
      relu_bwd_kernel<<<ew_grid(n4), 256, 0, st>>>(reinterpret_cast<const float4*>(gy),
                                                  reinterpret_cast<const float4*>(x),
                                                  reinterpret_cast<float4*>(gx), n4);
    if (n % 4) relu_bwd_tail<<<1, 4, 0, st>>>(gy, x, gx, 4 * n4, (long long)n);
    FCB_CUDA(cudaGetLastError());
  });
}

int fftconv_b200_maxpool_forward(const float* x, size_t planes, size_t rows, size_t cols,
                                 float* y, uint32_t* argmax, void* stream) {
  return guarded(nullptr, [&] {
    if (rows % 2 || cols % 2)
      throw Error(FFTCONV_B200_SIZE_ERROR, "maxpool: rows and cols must be even");
    const long long total = (long long)planes * (rows / 2) * (cols / 2);
    if (total)
      maxpool_fwd_kernel<<<plane_grid((long long)planes), 256, 0, (cudaStream_t)stream>>>(
          x, y, argmax, (long long)planes, (int)rows, (int)cols);
    FCB_CUDA(cudaGetLastError());
  });
}

int fftconv_b200_maxpool_backward(const float* gy, const uint32_t* argmax, size_t planes,
                                  size_t rows, size_t cols, float* gx, void* stream) {
  return guarded(nullptr, [&] {
    if (rows % 2 || cols % 2)
      throw Error(FFTCONV_B200_SIZE_ERROR, "maxpool: rows and cols must be even");
    const long long total = (long long)planes * (rows / 2) * (cols / 2);
    if (total)
      maxpool_bwd_kernel<<<plane_grid((long long)planes), 256, 0, (cudaStream_t)stream>>>(
          gy, argmax, gx, (long long)planes, (int)rows, (int)cols);
    FCB_CUDA(cudaGetLastError());
  });
}

int fftconv_b200_maxpool_relu_backward(const float* gy, const uint32_t* argmax, const float* y, size_t planes,
                                       size_t rows, size_t cols, float* gx, void* stream) {
  return guarded(nullptr, [&] {
    if (rows % 2 || cols % 2)
      throw Error(FFTCONV_B200_SIZE_ERROR, "maxpool: rows and cols must be even");
    if (!y) throw Error(FFTCONV_B200_INVALID_ARGUMENT, "maxpool_relu_backward: pooled output required");
    const long long total = (long long)planes * (rows / 2) * (cols / 2);
    if (total)
      maxpool_bwd_kernel<<<plane_grid((long long)planes), 256, 0, (cudaStream_t)stream>>>(
          gy, argmax, gx, (long long)planes, (int)rows, (int)cols, y);
    FCB_CUDA(cudaGetLastError());
  });
}

int fftconv_b200_fit_to(const float* x, size_t planes, size_t rows, size_t cols, float* y,
                        size_t size, void* stream) {
  return guarded(nullptr, [&] {
    const long long total = (long long)planes * size * size;
    if (total)
      fit_to_kernel<<<plane_grid((long long)planes), 256, 0, (cudaStream_t)stream>>>(
          x, y, (long long)planes, (int)rows, (int)cols, (int)size);
    FCB_CUDA(cudaGetLastError());
  });
}

}  // extern "C"

