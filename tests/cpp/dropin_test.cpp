// Drop-in parity test: the reference's own ConvWorkspace test cases
// (/root/reference/proj/tests/conv_fft_test.cpp) re-instantiated on
// fftconv::b200::ConvWorkspace (fp32, B200 kernels), with the reference's
// fp64 direct convolution (conv_direct.hpp) as the oracle.
//
// Built by paper_1312_5851_b200/_build.py where the reference headers exist
// (this container); the binary ships to the GPU box and is run by
// tests/test_gpu_dropin.py.  Exit code 0 iff every check passed.
#include <cmath>
#include <cstdio>
#include <string>
#include <vector>

#include "fftconv/conv_direct.hpp"
#include "fftconv/rng.hpp"
#include "fftconv/tensor.hpp"
#include "fftconv_b200/conv_workspace.hpp"

using fftconv::LayerConfig;
using fftconv::Tensor4;
using fftconv::Weights4;
using WS = fftconv::b200::ConvWorkspace;

static int g_fail = 0, g_checks = 0;
#define CHECK(cond)                                                               \
  do {                                                                            \
    ++g_checks;                                                                   \
    if (!(cond)) {                                                                \
      ++g_fail;                                                                   \
      std::printf("FAIL %s:%d: %s\n", __FILE__, __LINE__, #cond);                \
    }                                                                             \
  } while (0)
#define CHECK_THROW(stmt, type)                                                   \
  do {                                                                            \
    ++g_checks;                                                                   \
    bool caught_ = false;                                                         \
    try {                                                                         \
      stmt;                                                                       \
    } catch (const type&) {                                                       \
      caught_ = true;                                                             \
    } catch (...) {                                                               \
    }                                                                             \
    if (!caught_) {                                                               \
      ++g_fail;                                                                   \
      std::printf("FAIL %s:%d: expected %s from %s\n", __FILE__, __LINE__, #type, #stmt); \
    }                                                                             \
  } while (0)

template <typename T>
Tensor4<T> random_tensor(std::size_t S, std::size_t f, std::size_t n, std::uint64_t seed,
                         fftconv::TensorRole role) {
  Tensor4<T> t(S, f, n, n);
  fftconv::fill_uniform(t.data(), seed, role);
  return t;
}

template <typename T>
Weights4<T> random_weights(std::size_t fp, std::size_t f, std::size_t k, std::uint64_t seed) {
  Weights4<T> w(fp, f, k);
  fftconv::fill_uniform(w.data(), seed, fftconv::TensorRole::weights);
  return w;
}

static Tensor4<double> to64(const Tensor4<float>& t) {
  Tensor4<double> o(t.batch(), t.maps(), t.rows(), t.cols());
  for (std::size_t i = 0; i < t.size(); ++i) o.data()[i] = t.data()[i];
  return o;
}
static Weights4<double> to64(const Weights4<float>& t) {
  Weights4<double> o(t.out_maps(), t.in_maps(), t.kernel());
  for (std::size_t i = 0; i < t.size(); ++i) o.data()[i] = t.data()[i];
  return o;
}
template <typename A, typename B>
static double rel(const A& got, const B& ref) {
  std::vector<double> g(got.data().begin(), got.data().end());
  return fftconv::max_rel_error<double>(g, ref.data());
}

static void expect_all_ops_match_direct(const LayerConfig& cfg, double tol, std::uint64_t seed) {
  auto x = random_tensor<float>(cfg.batch, cfg.in_maps, cfg.image, seed, fftconv::TensorRole::input);
  auto w = random_weights<float>(cfg.out_maps, cfg.in_maps, cfg.kernel, seed + 1);
  auto gy = random_tensor<float>(cfg.batch, cfg.out_maps, cfg.output_size(), seed + 2,
                                 fftconv::TensorRole::grad_output);
  WS ws({cfg});
  CHECK(rel(ws.forward(x, w), fftconv::forward_direct(to64(x), to64(w))) < tol);
  CHECK(rel(ws.grad_input(gy, w), fftconv::grad_input_direct(to64(gy), to64(w))) < tol);
  CHECK(rel(ws.grad_weight(gy, x), fftconv::grad_weight_direct(to64(gy), to64(x))) < tol);
}

int main() {
  // conv_fft_test.cpp:65-75 (f32 tolerance 1e-4)
  expect_all_ops_match_direct({3, 16, 4, 6, 2}, 1e-4, 21);
  expect_all_ops_match_direct({5, 16, 4, 4, 2}, 1e-4, 22);
  expect_all_ops_match_direct({7, 32, 3, 5, 1}, 1e-4, 23);
  expect_all_ops_match_direct({3, 8, 2, 2, 2}, 1e-4, 31);
  expect_all_ops_match_direct({8, 8, 1, 2, 1}, 1e-4, 32);
  expect_all_ops_match_direct({7, 32, 96, 96, 8}, 1e-4, 1234);

  {  // UnitKernelIsIdentity :77-85
    auto x = random_tensor<float>(2, 2, 6, 41, fftconv::TensorRole::input);
    Weights4<float> w(2, 2, 1);
    w.at(0, 0, 0, 0) = 1.0f;
    w.at(1, 1, 0, 0) = 1.0f;
    WS ws({{1, 6, 2, 2, 2}});
    CHECK(rel(ws.forward(x, w), to64(x)) < 1e-6);
  }
  {  // ZeroKernelGivesZeroOutput :87-93
    auto x = random_tensor<float>(1, 2, 5, 42, fftconv::TensorRole::input);
    Weights4<float> w(3, 2, 2);
    WS ws({{2, 5, 2, 3, 1}});
    auto y = ws.forward(x, w);
    for (float v : y.data()) CHECK(std::abs(v) < 1e-7f);
  }
  {  // CornerImpulseSelectsShiftedWindow :95-107
    const std::size_t n = 8, k = 3, u0 = 1, v0 = 2;
    auto x = random_tensor<float>(1, 1, n, 43, fftconv::TensorRole::input);
    Weights4<float> w(1, 1, k);
    w.at(0, 0, u0, v0) = 1.0f;
    WS ws({{k, n, 1, 1, 1}});
    auto y = ws.forward(x, w);
    for (std::size_t i = 0; i < n - k + 1; ++i)
      for (std::size_t j = 0; j < n - k + 1; ++j)
        CHECK(std::abs(y.at(0, 0, i, j) - x.at(0, 0, i + u0, j + v0)) < 1e-5);
  }
  {  // GradWeightImpulseExtractsInputWindow :109-119
    auto x = random_tensor<float>(1, 1, 6, 44, fftconv::TensorRole::input);
    Tensor4<float> gy(1, 1, 2, 2);
    gy.at(0, 0, 1, 1) = 1.0f;
    WS ws({{5, 6, 1, 1, 1}});
    auto gw = ws.grad_weight(gy, x);
    CHECK(gw.kernel() == 5u);
    for (std::size_t u = 0; u < 5; ++u)
      for (std::size_t v = 0; v < 5; ++v)
        CHECK(std::abs(gw.at(0, 0, u, v) - x.at(0, 0, u + 1, v + 1)) < 1e-5);
  }
  {  // CapacitiesForSingleConfig / PerRoleMaxima :142-161
    WS ws({{3, 8, 2, 5, 1}});
    CHECK(ws.max_fft_size() == 8u);
    CHECK(ws.capacity_x() == 40u * 1 * 2);
    CHECK(ws.capacity_w() == 40u * 5 * 2);
    CHECK(ws.capacity_y() == 40u * 1 * 5);
    CHECK(ws.frequency_bytes() == (80u + 400u + 200u) * 8u);
    WS ws2({{3, 8, 2, 5, 1}, {3, 8, 4, 1, 3}});
    CHECK(ws2.capacity_x() == 40u * 3 * 4);
    CHECK(ws2.capacity_w() == 40u * 5 * 2);
    CHECK(ws2.capacity_y() == 40u * 1 * 5);
  }
  // RejectsEmptyConfigList :163-165
  CHECK_THROW(WS(std::vector<LayerConfig>{}), fftconv::config_error);
  {  // RejectsLayerBeyondCapacity :167-174
    WS ws({{3, 8, 2, 2, 1}});
    auto w = random_weights<float>(2, 2, 3, 50);
    auto xb = random_tensor<float>(2, 2, 8, 51, fftconv::TensorRole::input);
    CHECK_THROW(ws.forward(xb, w), fftconv::capacity_error);
    auto xi = random_tensor<float>(1, 2, 9, 52, fftconv::TensorRole::input);
    CHECK_THROW(ws.forward(xi, w), fftconv::capacity_error);
  }
  {  // ShapeAndSizeErrors :176-189
    WS ws({{3, 8, 2, 2, 1}});
    auto x = random_tensor<float>(1, 2, 8, 53, fftconv::TensorRole::input);
    CHECK_THROW(ws.forward(x, Weights4<float>(2, 3, 3)), fftconv::shape_error);
    CHECK_THROW(ws.forward(x, Weights4<float>(2, 2, 9)), fftconv::size_error);
    Tensor4<float> rect(1, 2, 8, 6);
    CHECK_THROW(ws.forward(rect, Weights4<float>(2, 2, 3)), fftconv::size_error);
    auto gy = random_tensor<float>(1, 2, 6, 54, fftconv::TensorRole::grad_output);
    CHECK_THROW(ws.grad_input(gy, Weights4<float>(3, 2, 3)), fftconv::shape_error);
    Tensor4<float> gym(2, 2, 6, 6);
    CHECK_THROW(ws.grad_weight(gym, x), fftconv::shape_error);
  }
  {  // ReuseAcrossLayersIsBitStable :191-209
    const LayerConfig a{3, 6, 2, 3, 2}, b{5, 12, 3, 2, 1};
    WS ws({a, b});
    auto xa = random_tensor<float>(2, 2, 6, 60, fftconv::TensorRole::input);
    auto wa = random_weights<float>(3, 2, 3, 61);
    auto xb = random_tensor<float>(1, 3, 12, 62, fftconv::TensorRole::input);
    auto wb = random_weights<float>(2, 3, 5, 63);
    auto first = ws.forward(xa, wa);
    (void)ws.forward(xb, wb);
    auto again = ws.forward(xa, wa);
    for (std::size_t i = 0; i < first.size(); ++i) CHECK(first.data()[i] == again.data()[i]);
  }
  {  // CountersMatchPlanAndAreKernelInvariant :211-253
    const std::size_t n = 16, S = 2, f = 3, fp = 4;
    const std::uint64_t bins = 16 * 9;
    for (std::size_t k : {3u, 5u, 7u, 11u}) {
      WS ws({{k, n, f, fp, S}});
      auto x = random_tensor<float>(S, f, n, 70, fftconv::TensorRole::input);
      auto w = random_weights<float>(fp, f, k, 71);
      auto gy = random_tensor<float>(S, fp, n - k + 1, 72, fftconv::TensorRole::grad_output);
      (void)ws.forward(x, w);
      fftconv::OpCounters fwd = ws.counters();
      CHECK(fwd.forward_transforms == S * f + fp * f);
      CHECK(fwd.inverse_transforms == S * fp);
      CHECK(fwd.complex_macs == bins * fp * f * S);
      ws.reset_counters();
      (void)ws.grad_input(gy, w);
      fftconv::OpCounters gin = ws.counters();
      CHECK(gin.forward_transforms == S * fp + fp * f);
      CHECK(gin.inverse_transforms == S * f);
      ws.reset_counters();
      (void)ws.grad_weight(gy, x);
      fftconv::OpCounters gwc = ws.counters();
      CHECK(gwc.forward_transforms == S * f + S * fp);
      CHECK(gwc.inverse_transforms == fp * f);
      CHECK(gwc.complex_macs == bins * fp * f * S);
    }
  }
  {  // FreeFunctionWrappers :279-294
    const LayerConfig cfg{2, 5, 1, 2, 1};
    auto ws = fftconv::b200::workspace_for({cfg});
    auto x = random_tensor<float>(1, 1, 5, 90, fftconv::TensorRole::input);
    auto w = random_weights<float>(2, 1, 2, 91);
    auto gy = random_tensor<float>(1, 2, 4, 92, fftconv::TensorRole::grad_output);
    CHECK(rel(fftconv::b200::forward_fft(ws, x, w), fftconv::forward_direct(to64(x), to64(w))) < 1e-5);
    CHECK(rel(fftconv::b200::grad_input_fft(ws, gy, w),
              fftconv::grad_input_direct(to64(gy), to64(w))) < 1e-5);
    CHECK(rel(fftconv::b200::grad_weight_fft(ws, gy, x),
              fftconv::grad_weight_direct(to64(gy), to64(x))) < 1e-5);
  }
  std::printf("dropin_test: %d checks, %d failures\n", g_checks, g_fail);
  {  // grad_weight_sharded on a one-rank communicator: the shard is the whole
     // minibatch, so the summed gradient equals grad_weight bit for bit
     // (conv_direct_test.cpp:186-212 batch decomposability)
    const LayerConfig c{5, 16, 3, 4, 6};
    WS ws({c});
    auto x = random_tensor<float>(6, 3, 16, 80, fftconv::TensorRole::input);
    auto gy = random_tensor<float>(6, 4, 12, 81, fftconv::TensorRole::grad_output);
    void* comm = fftconv::b200::nccl_comm_create(fftconv::b200::nccl_unique_id(), 1, 0, 0);
    auto full = ws.grad_weight(gy, x);
    auto sh = ws.grad_weight_sharded(gy, x, comm);
    for (std::size_t i = 0; i < full.size(); ++i) CHECK(full.data()[i] == sh.data()[i]);
    fftconv::b200::nccl_comm_destroy(comm);
  }
  return g_fail == 0 ? 0 : 1;
}
