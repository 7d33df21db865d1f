// ctypes shim over the UNMODIFIED reference library -- TEST / BASELINE ONLY.
//
// Compiled by oracle/Makefile straight from the reference headers where they
// lie (/root/reference/proj/include, header-only C++20, no third-party deps)
// into oracle/_ref/libfftconv_ref.so.  Nothing of the reference is copied
// into this repository; this file only binds its public API with C linkage
// so Python tests can (a) generate golden vectors that pin the oracle and
// (b) time the reference CPU path as bench.py's cpu_baseline / --impl
// reference arm.
//
// Bound reference entry points:
//   fftconv::ConvWorkspace<T> ctor / forward / grad_input / grad_weight /
//     counters / capacities        conv_fft.hpp:43-206
//   fftconv::forward_direct / grad_input_direct / grad_weight_direct
//                                   conv_direct.hpp:24-127
//   fftconv::detail::r2c_plane / c2r_plane   fft.hpp:160-203
//   fftconv::fill_uniform, uniform_at        rng.hpp:32-47
//   fftconv::run_op_bench                    bench.hpp:80-145
//   fftconv::random_verify_configs, verify_sweep  bench.hpp:164-222
//   fftconv::preset_network / parse_network_string / init_params /
//     make_batch / run_iteration        layers.hpp:321-609
#include <cstdint>
#include <cstring>
#include <exception>
#include <memory>
#include <string>
#include <vector>

#include "fftconv/bench.hpp"
#include "fftconv/conv_direct.hpp"
#include "fftconv/conv_fft.hpp"
#include "fftconv/cost_model.hpp"
#include "fftconv/fft.hpp"
#include "fftconv/layers.hpp"
#include "fftconv/rng.hpp"

namespace {

thread_local std::string g_last_error;

// errors.hpp class -> status code used across the repo's C ABIs.
template <typename F>
int guarded(F&& f) {
  try {
    f();
    return 0;
  } catch (const fftconv::size_error& e) {
    g_last_error = e.what();
    return 1;
  } catch (const fftconv::shape_error& e) {
    g_last_error = e.what();
    return 2;
  } catch (const fftconv::config_error& e) {
    g_last_error = e.what();
    return 3;
  } catch (const fftconv::capacity_error& e) {
    g_last_error = e.what();
    return 4;
  } catch (const fftconv::plan_error& e) {
    g_last_error = e.what();
    return 5;
  } catch (const std::exception& e) {
    g_last_error = e.what();
    return 9;
  }
}

template <typename T>
fftconv::Tensor4<T> make_tensor(const T* p, size_t S, size_t f, size_t rows, size_t cols) {
  fftconv::Tensor4<T> t(S, f, rows, cols);
  std::memcpy(t.data().data(), p, sizeof(T) * t.size());
  return t;
}

template <typename T>
fftconv::Weights4<T> make_weights(const T* p, size_t fo, size_t fi, size_t k) {
  fftconv::Weights4<T> w(fo, fi, k);
  std::memcpy(w.data().data(), p, sizeof(T) * w.size());
  return w;
}

template <typename T, typename V>
void copy_out(const V& v, T* dst) {
  std::memcpy(dst, v.data().data(), sizeof(T) * v.size());
}

struct RefWs {
  std::unique_ptr<fftconv::ConvWorkspace<float>> f32;
  std::unique_ptr<fftconv::ConvWorkspace<double>> f64;
};

template <typename T>
fftconv::ConvWorkspace<T>& ws_of(RefWs* h);
template <>
fftconv::ConvWorkspace<float>& ws_of<float>(RefWs* h) { return *h->f32; }
template <>
fftconv::ConvWorkspace<double>& ws_of<double>(RefWs* h) { return *h->f64; }

}  // namespace

extern "C" {

const char* ref_last_error() { return g_last_error.c_str(); }

double ref_uniform_at(uint64_t seed, uint64_t role, uint64_t index) {
  return fftconv::uniform_at(seed, role, index);
}

void ref_fill_uniform_f32(float* out, size_t n, uint64_t seed, uint64_t role, uint64_t stream) {
  fftconv::fill_uniform<float>(std::span<float>(out, n), seed,
                               static_cast<fftconv::TensorRole>(role), stream);
}
void ref_fill_uniform_f64(double* out, size_t n, uint64_t seed, uint64_t role, uint64_t stream) {
  fftconv::fill_uniform<double>(std::span<double>(out, n), seed,
                                static_cast<fftconv::TensorRole>(role), stream);
}

// cfgs: count x {k, n, f, f', S}
int ref_ws_create(const uint64_t* cfgs, size_t count, int is_f64, void** out) {
  return guarded([&] {
    std::vector<fftconv::LayerConfig> v;
    for (size_t i = 0; i < count; ++i)
      v.push_back({cfgs[5 * i], cfgs[5 * i + 1], cfgs[5 * i + 2], cfgs[5 * i + 3], cfgs[5 * i + 4]});
    auto* h = new RefWs;
    try {
      if (is_f64)
        h->f64 = std::make_unique<fftconv::ConvWorkspace<double>>(v);
      else
        h->f32 = std::make_unique<fftconv::ConvWorkspace<float>>(v);
    } catch (...) {
      delete h;
      throw;
    }
    *out = h;
  });
}

void ref_ws_destroy(void* h) { delete static_cast<RefWs*>(h); }

// out: max_fft_size, cap_x, cap_w, cap_y, frequency_bytes
void ref_ws_info(void* hv, uint64_t* out) {
  auto* h = static_cast<RefWs*>(hv);
  auto fill = [&](auto& ws) {
    out[0] = ws.max_fft_size();
    out[1] = ws.capacity_x();
    out[2] = ws.capacity_w();
    out[3] = ws.capacity_y();
    out[4] = ws.frequency_bytes();
  };
  if (h->f64) fill(*h->f64); else fill(*h->f32);
}

void ref_ws_counters(void* hv, uint64_t* out) {
  auto* h = static_cast<RefWs*>(hv);
  auto fill = [&](auto& ws) {
    out[0] = ws.counters().forward_transforms;
    out[1] = ws.counters().inverse_transforms;
    out[2] = ws.counters().complex_macs;
  };
  if (h->f64) fill(*h->f64); else fill(*h->f32);
}

void ref_ws_reset_counters(void* hv) {
  auto* h = static_cast<RefWs*>(hv);
  if (h->f64) h->f64->reset_counters(); else h->f32->reset_counters();
}

#define REF_OPS(T, SFX)                                                                       \
  int ref_ws_forward##SFX(void* h, const T* x, size_t S, size_t f, size_t xr, size_t xc,     \
                          const T* w, size_t fo, size_t wi, size_t k, T* y,                  \
                          unsigned threads) {                                               \
    return guarded([&] {                                                                     \
      auto yy = ws_of<T>(static_cast<RefWs*>(h))                                             \
                    .forward(make_tensor(x, S, f, xr, xc), make_weights(w, fo, wi, k),      \
                             threads);                                                      \
      copy_out(yy, y);                                                                       \
    });                                                                                      \
  }                                                                                          \
  int ref_ws_grad_input##SFX(void* h, const T* gy, size_t S, size_t fo, size_t gr,          \
                             size_t gc, const T* w, size_t wo, size_t fi, size_t k, T* gx,   \
                             unsigned threads) {                                            \
    return guarded([&] {                                                                     \
      auto g = ws_of<T>(static_cast<RefWs*>(h))                                              \
                   .grad_input(make_tensor(gy, S, fo, gr, gc), make_weights(w, wo, fi, k),   \
                               threads);                                                    \
      copy_out(g, gx);                                                                       \
    });                                                                                      \
  }                                                                                          \
  int ref_ws_grad_weight##SFX(void* h, const T* gy, size_t Sg, size_t fo, size_t gr,        \
                              size_t gc, const T* x, size_t Sx, size_t fi, size_t xr,        \
                              size_t xc, T* gw, unsigned threads) {                          \
    return guarded([&] {                                                                     \
      auto g = ws_of<T>(static_cast<RefWs*>(h))                                              \
                   .grad_weight(make_tensor(gy, Sg, fo, gr, gc),                             \
                                make_tensor(x, Sx, fi, xr, xc), threads);                    \
      copy_out(g, gw);                                                                       \
    });                                                                                      \
  }                                                                                          \
  int ref_forward_direct##SFX(const T* x, const T* w, T* y, size_t S, size_t f, size_t fo,  \
                              size_t n, size_t k, unsigned threads) {                        \
    return guarded([&] {                                                                     \
      copy_out(fftconv::forward_direct(make_tensor(x, S, f, n, n), make_weights(w, fo, f, k), \
                                       threads),                                            \
               y);                                                                           \
    });                                                                                      \
  }                                                                                          \
  int ref_grad_input_direct##SFX(const T* gy, const T* w, T* gx, size_t S, size_t f,         \
                                 size_t fo, size_t no, size_t k, unsigned threads) {         \
    return guarded([&] {                                                                     \
      copy_out(fftconv::grad_input_direct(make_tensor(gy, S, fo, no, no),                    \
                                          make_weights(w, fo, f, k), threads),               \
               gx);                                                                          \
    });                                                                                      \
  }                                                                                          \
  int ref_grad_weight_direct##SFX(const T* gy, const T* x, T* gw, size_t S, size_t f,        \
                                  size_t fo, size_t n, size_t no, unsigned threads) {        \
    return guarded([&] {                                                                     \
      copy_out(fftconv::grad_weight_direct(make_tensor(gy, S, fo, no, no),                   \
                                           make_tensor(x, S, f, n, n), threads),             \
               gw);                                                                          \
    });                                                                                      \
  }                                                                                          \
  int ref_r2c_plane##SFX(const T* src, size_t rows, size_t cols, size_t m, T* out) {        \
    return guarded([&] {                                                                     \
      fftconv::FftPlan<T> plan(m);                                                           \
      std::vector<std::complex<T>> line(m);                                                  \
      fftconv::detail::r2c_plane(plan, src, rows, cols,                                      \
                                 reinterpret_cast<std::complex<T>*>(out),                    \
                                 std::span<std::complex<T>>(line));                          \
    });                                                                                      \
  }                                                                                          \
  int ref_c2r_plane##SFX(const T* half_in, size_t m, T* dst, size_t rows, size_t cols) {    \
    return guarded([&] {                                                                     \
      fftconv::FftPlan<T> plan(m);                                                           \
      std::vector<std::complex<T>> half(m * (m / 2 + 1)), line(m);                           \
      std::memcpy(half.data(), half_in, sizeof(std::complex<T>) * half.size());              \
      fftconv::detail::c2r_plane(plan, half.data(), dst, rows, cols,                         \
                                 std::span<std::complex<T>>(line));                          \
    });                                                                                      \
  }

REF_OPS(float, _f32)
REF_OPS(double, _f64)

int ref_fft_1d_f64(double* data, size_t m, int inverse) {
  return guarded([&] {
    fftconv::FftPlan<double> plan(m);
    plan.transform(std::span<std::complex<double>>(reinterpret_cast<std::complex<double>*>(data), m),
                   inverse != 0);
  });
}

// run_op_bench<float> (bench.hpp:80-145).  op: 0 output, 1 gradinput,
// 2 gradweight; method: 0 direct, 1 fft.  out: mean, std, min, median ms,
// checksum.
int ref_run_op_bench_f32(size_t k, size_t n, size_t f, size_t fo, size_t S, int op, int method,
                         size_t iters, size_t warmup, unsigned threads, uint64_t seed,
                         double* out) {
  return guarded([&] {
    fftconv::LayerConfig cfg{k, n, f, fo, S};
    auto r = fftconv::run_op_bench<float>(cfg, static_cast<fftconv::BenchOp>(op),
                                          method ? fftconv::Method::fft : fftconv::Method::direct,
                                          iters, warmup, threads, seed);
    out[0] = r.stats.mean_ms;
    out[1] = r.stats.std_ms;
    out[2] = r.stats.min_ms;
    out[3] = r.stats.median_ms;
    out[4] = r.checksum;
  });
}

unsigned ref_resolve_threads(unsigned requested) { return fftconv::resolve_threads(requested); }

// random_verify_configs (bench.hpp:164-183); out: count x {k, n, f, f', S}
void ref_random_verify_configs(size_t count, uint64_t seed, uint64_t* out) {
  auto v = fftconv::random_verify_configs(count, seed);
  for (size_t i = 0; i < v.size(); ++i) {
    out[5 * i + 0] = v[i].kernel;
    out[5 * i + 1] = v[i].image;
    out[5 * i + 2] = v[i].in_maps;
    out[5 * i + 3] = v[i].out_maps;
    out[5 * i + 4] = v[i].batch;
  }
}

// One training iteration of a network (layers.hpp:441-609) with the
// reference's own parameters and batch (init_params / make_batch, seed).
// The network arrives as stage records {kind, k, n, f, f' | fc outputs}
// (kind: 0 conv, 1 relu, 2 pool, 3 fc) and is validated by the reference's
// NetworkSpec::validate; parse_network's istringstream is not used because
// this library carries its own static libstdc++ next to the host process's.
// engine: 0 direct, 1 fft.  out_grads receives, in order, every conv weight
// gradient, then the fc weight and bias gradients (grads_cap floats
// available; the length needed goes to *grads_len).  scalars: loss,
// grad_checksum, update_output_ms, update_grad_input_ms, acc_grad_ms,
// grad_input_calls.
extern "C++" {
template <typename T>
static int ref_run_iteration_t(const uint64_t* stages, size_t nstages, size_t S, uint64_t seed, int engine,
                               unsigned threads, T* out_grads, size_t grads_cap, size_t* grads_len,
                               double* scalars) {
  return guarded([&] {
    fftconv::NetworkSpec net;
    for (size_t i = 0; i < nstages; ++i) {
      const uint64_t* r = stages + 5 * i;
      fftconv::Stage st;
      st.kind = static_cast<fftconv::StageKind>(r[0]);
      if (st.kind == fftconv::StageKind::conv) st.conv = fftconv::LayerConfig{r[1], r[2], r[3], r[4], 1};
      if (st.kind == fftconv::StageKind::fc) st.fc_outputs = r[4];
      net.stages.push_back(st);
    }
    if (!net.stages.empty() && net.stages.front().kind == fftconv::StageKind::conv) {
      net.input_maps = net.stages.front().conv.in_maps;
      net.input_image = net.stages.front().conv.image;
    }
    net.validate();
    auto params = fftconv::init_params<T>(net, seed);
    auto batch = fftconv::make_batch<T>(net, S, seed);
    auto r = fftconv::run_iteration<T>(
        net, params, batch, engine ? fftconv::Engine::fft : fftconv::Engine::direct, nullptr, threads);
    size_t n = 0;
    for (const auto& g : r.conv_weight_grads) n += g.size();
    n += r.fc_weight_grad.size() + r.fc_bias_grad.size();
    *grads_len = n;
    if (out_grads && grads_cap >= n) {
      size_t o = 0;
      for (const auto& g : r.conv_weight_grads) {
        std::memcpy(out_grads + o, g.data().data(), g.size() * sizeof(T));
        o += g.size();
      }
      std::memcpy(out_grads + o, r.fc_weight_grad.data(), r.fc_weight_grad.size() * sizeof(T));
      o += r.fc_weight_grad.size();
      std::memcpy(out_grads + o, r.fc_bias_grad.data(), r.fc_bias_grad.size() * sizeof(T));
    }
    scalars[0] = r.loss;
    scalars[1] = r.grad_checksum;
    scalars[2] = r.times.update_output_ms;
    scalars[3] = r.times.update_grad_input_ms;
    scalars[4] = r.times.acc_grad_ms;
    scalars[5] = (double)r.grad_input_calls;
  });
}
}  // extern "C++"

int ref_run_iteration_f32(const uint64_t* stages, size_t nstages, size_t S, uint64_t seed,
                          int engine, unsigned threads, float* out_grads, size_t grads_cap,
                          size_t* grads_len, double* scalars) {
  return ref_run_iteration_t<float>(stages, nstages, S, seed, engine, threads, out_grads, grads_cap, grads_len,
                                    scalars);
}

// The same iteration in double (run_iteration<double>): the precision
// reference for deep stacks, where two fp32 implementations drift apart.
int ref_run_iteration_f64(const uint64_t* stages, size_t nstages, size_t S, uint64_t seed,
                          int engine, unsigned threads, double* out_grads, size_t grads_cap,
                          size_t* grads_len, double* scalars) {
  return ref_run_iteration_t<double>(stages, nstages, S, seed, engine, threads, out_grads, grads_cap, grads_len,
                                     scalars);
}

// cost_model.hpp:39-110: op 0/1/2 -> {direct, transform, pointwise, inverse}
// counts; out[4] = memory_bytes, out[5] = packed_memory_bytes(4 bytes).
int ref_cost_model(size_t k, size_t n, size_t f, size_t fo, size_t S, double C, int op, double* out) {
  return guarded([&] {
    fftconv::CostParams p{{k, n, f, fo, S}, C};
    fftconv::OpCounts c = op == 0 ? fftconv::ops_forward(p)
                                  : (op == 1 ? fftconv::ops_grad_input(p) : fftconv::ops_grad_weight(p));
    out[0] = c.direct_ops;
    out[1] = c.transform_ops;
    out[2] = c.pointwise_ops;
    out[3] = c.inverse_ops;
    out[4] = (double)fftconv::memory_bytes(p.config);
    out[5] = (double)fftconv::packed_memory_bytes(p.config, 4);
  });
}

}  // extern "C"
