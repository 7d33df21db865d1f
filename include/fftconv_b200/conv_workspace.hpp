// fftconv::b200::ConvWorkspace -- header-only C++ drop-in for
// fftconv::ConvWorkspace<float> (/root/reference/proj/include/fftconv/
// conv_fft.hpp:40-335), running on the B200 kernels through the C ABI in
// fftconv_b200.h.
//
// Same method names, argument order and return-by-value types as the
// reference, on the reference's own Tensor4/Weights4/LayerConfig/OpCounters
// (include the reference headers first -- this is a drop-in for code that
// already uses them).  Failures throw the reference exception classes
// (errors.hpp) in the reference's validation order.  `threads` is accepted
// for signature parity and ignored: parallelism lives on the GPU.
#pragma once

#include <cstdint>
#include <string>
#include <utility>
#include <vector>

#include "fftconv/conv_fft.hpp"  // OpCounters (and the reference CPU path itself)
#include "fftconv/errors.hpp"
#include "fftconv/layer_config.hpp"
#include "fftconv/tensor.hpp"
#include "fftconv_b200.h"

namespace fftconv::b200 {

namespace detail {

inline void throw_status(int code, const char* msg) {
  const std::string m = msg ? msg : "";
  switch (code) {
    case FFTCONV_B200_OK: return;
    case FFTCONV_B200_SIZE_ERROR: throw fftconv::size_error(m);
    case FFTCONV_B200_SHAPE_ERROR: throw fftconv::shape_error(m);
    case FFTCONV_B200_CONFIG_ERROR: throw fftconv::config_error(m);
    case FFTCONV_B200_CAPACITY_ERROR: throw fftconv::capacity_error(m);
    case FFTCONV_B200_PLAN_ERROR: throw fftconv::plan_error(m);
    default: throw fftconv::error("fftconv_b200: " + m);
  }
}

}  // namespace detail

class ConvWorkspace {
 public:
  // conv_fft.hpp:43-58 (config_error on an empty list or an invalid config).
  explicit ConvWorkspace(const std::vector<LayerConfig>& configs, int device = 0) {
    std::vector<fftconv_b200_layer> c;
    c.reserve(configs.size());
    for (const LayerConfig& l : configs)
      c.push_back({l.kernel, l.image, l.in_maps, l.out_maps, l.batch});
    const int code = fftconv_b200_ws_create(c.data(), c.size(), device, &ws_);
    detail::throw_status(code, fftconv_b200_last_error(nullptr));
  }
  ~ConvWorkspace() { fftconv_b200_ws_destroy(ws_); }
  ConvWorkspace(const ConvWorkspace&) = delete;
  ConvWorkspace& operator=(const ConvWorkspace&) = delete;
  ConvWorkspace(ConvWorkspace&& o) noexcept : ws_(std::exchange(o.ws_, nullptr)) {}
  ConvWorkspace& operator=(ConvWorkspace&& o) noexcept {
    std::swap(ws_, o.ws_);
    return *this;
  }

  // conv_fft.hpp:60-69
  std::size_t max_fft_size() const { return static_cast<std::size_t>(info(0)); }
  std::uint64_t capacity_x() const { return info(1); }
  std::uint64_t capacity_w() const { return info(2); }
  std::uint64_t capacity_y() const { return info(3); }
  std::uint64_t frequency_bytes() const { return info(4); }

  // conv_fft.hpp:71-72
  const OpCounters& counters() const {
    std::uint64_t c[3];
    fftconv_b200_counters(ws_, c);
    counters_ = OpCounters{c[0], c[1], c[2]};
    return counters_;
  }
  void reset_counters() { fftconv_b200_reset_counters(ws_); }

  // conv_fft.hpp:74-113
  Tensor4<float> forward(const Tensor4<float>& x, const Weights4<float>& w, unsigned threads = 1) {
    const bool ok = x.rows() == x.cols() && w.in_maps() == x.maps() && w.kernel() <= x.rows();
    if (!ok) call(fftconv_b200_forward_host(ws_, x.data().data(), x.batch(), x.maps(), x.rows(),
                                            x.cols(), w.data().data(), w.out_maps(), w.in_maps(),
                                            w.kernel(), nullptr, threads));
    const std::size_t no = x.rows() - w.kernel() + 1;
    Tensor4<float> y(x.batch(), w.out_maps(), no, no);
    call(fftconv_b200_forward_host(ws_, x.data().data(), x.batch(), x.maps(), x.rows(), x.cols(),
                                   w.data().data(), w.out_maps(), w.in_maps(), w.kernel(),
                                   y.data().data(), threads));
    return y;
  }

  // conv_fft.hpp:115-152
  Tensor4<float> grad_input(const Tensor4<float>& gy, const Weights4<float>& w,
                            unsigned threads = 1) {
    const bool ok = gy.rows() == gy.cols() && w.out_maps() == gy.maps();
    if (!ok) call(fftconv_b200_grad_input_host(ws_, gy.data().data(), gy.batch(), gy.maps(),
                                               gy.rows(), gy.cols(), w.data().data(),
                                               w.out_maps(), w.in_maps(), w.kernel(), nullptr,
                                               threads));
    const std::size_t n = gy.rows() + w.kernel() - 1;
    Tensor4<float> gx(gy.batch(), w.in_maps(), n, n);
    call(fftconv_b200_grad_input_host(ws_, gy.data().data(), gy.batch(), gy.maps(), gy.rows(),
                                      gy.cols(), w.data().data(), w.out_maps(), w.in_maps(),
                                      w.kernel(), gx.data().data(), threads));
    return gx;
  }

  // conv_fft.hpp:154-206
  Weights4<float> grad_weight(const Tensor4<float>& gy, const Tensor4<float>& x,
                              unsigned threads = 1) {
    const bool ok = gy.rows() == gy.cols() && x.rows() == x.cols() && gy.batch() == x.batch() &&
                    gy.rows() <= x.rows();
    if (!ok) call(fftconv_b200_grad_weight_host(ws_, gy.data().data(), gy.batch(), gy.maps(),
                                                gy.rows(), gy.cols(), x.data().data(), x.batch(),
                                                x.maps(), x.rows(), x.cols(), nullptr, threads));
    const std::size_t k = x.rows() - gy.rows() + 1;
    Weights4<float> gw(gy.maps(), x.maps(), k);
    call(fftconv_b200_grad_weight_host(ws_, gy.data().data(), gy.batch(), gy.maps(), gy.rows(),
                                       gy.cols(), x.data().data(), x.batch(), x.maps(), x.rows(),
                                       x.cols(), gw.data().data(), threads));
    return gw;
  }

  // Minibatch-sharded accGrad (BASELINE configs[3] / [4] on N GPUs): `gy`
  // and `x` are this rank's shard of the minibatch; returns the full-batch
  // weight gradient, summed over the ranks of `nccl_comm` (an ncclComm_t,
  // e.g. from nccl_comm_create).  A Tensor4 cannot be empty, so a rank whose
  // shard is empty (world > S) calls fftconv_b200_grad_weight_sharded_host
  // with S_gy = S_x = 0 instead; it contributes zeros to the sum.
  Weights4<float> grad_weight_sharded(const Tensor4<float>& gy, const Tensor4<float>& x, void* nccl_comm,
                                      unsigned threads = 1) {
    const std::size_t k = x.rows() >= gy.rows() ? x.rows() - gy.rows() + 1 : 1;
    Weights4<float> gw(gy.maps(), x.maps(), k);
    call(fftconv_b200_grad_weight_sharded_host(ws_, gy.data().data(), gy.batch(), gy.maps(), gy.rows(),
                                               gy.cols(), x.data().data(), x.batch(), x.maps(), x.rows(),
                                               x.cols(), gw.data().data(), nccl_comm, threads));
    return gw;
  }

  fftconv_b200_ws* native_handle() const { return ws_; }

 private:
  std::uint64_t info(int i) const {
    std::uint64_t v[6] = {};
    fftconv_b200_ws_info(ws_, v);
    return v[i];
  }
  void call(int code) const { detail::throw_status(code, fftconv_b200_last_error(ws_)); }

  fftconv_b200_ws* ws_ = nullptr;
  mutable OpCounters counters_{};
};

// NCCL communicator for grad_weight_sharded without linking NCCL: rank 0
// calls nccl_unique_id, the caller distributes the 128 bytes, every rank
// calls nccl_comm_create.  Throws fftconv::error on failure.
inline std::vector<unsigned char> nccl_unique_id() {
  std::vector<unsigned char> id(128);
  const int code = fftconv_b200_nccl_get_unique_id(id.data());
  detail::throw_status(code, fftconv_b200_last_error(nullptr));
  return id;
}
inline void* nccl_comm_create(const std::vector<unsigned char>& id, int nranks, int rank, int device = 0) {
  void* comm = nullptr;
  const int code = fftconv_b200_nccl_comm_create(id.data(), nranks, rank, device, &comm);
  detail::throw_status(code, fftconv_b200_last_error(nullptr));
  return comm;
}
inline void nccl_comm_destroy(void* comm) { fftconv_b200_nccl_comm_destroy(comm); }

// conv_fft.hpp:314-335
inline ConvWorkspace workspace_for(const std::vector<LayerConfig>& configs, int device = 0) {
  return ConvWorkspace(configs, device);
}
inline Tensor4<float> forward_fft(ConvWorkspace& ws, const Tensor4<float>& x,
                                  const Weights4<float>& w, unsigned threads = 1) {
  return ws.forward(x, w, threads);
}
inline Tensor4<float> grad_input_fft(ConvWorkspace& ws, const Tensor4<float>& gy,
                                     const Weights4<float>& w, unsigned threads = 1) {
  return ws.grad_input(gy, w, threads);
}
inline Weights4<float> grad_weight_fft(ConvWorkspace& ws, const Tensor4<float>& gy,
                                       const Tensor4<float>& x, unsigned threads = 1) {
  return ws.grad_weight(gy, x, threads);
}

}  // namespace fftconv::b200
