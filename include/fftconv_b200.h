/*
 * fftconv_b200 -- C ABI of the B200 (sm_100a) FFT-convolution hot path.
 *
 * Drop-in replacement for the reference fftconv::ConvWorkspace<float>
 * operator interface (/root/reference/proj/include/fftconv/conv_fft.hpp).
 * Plain pointers and sizes only; no C++ or torch types cross this boundary.
 * Each entry point names the reference interface it replaces.
 *
 * Tensor layouts are the reference's (tensor.hpp:13-15, :63-64):
 *   x, gx  [S][f][n][n]      fp32 row-major
 *   y, gy  [S][f'][n'][n']   n' = n - k + 1
 *   w, gw  [f'][f][k][k]
 *
 * Status codes mirror the reference exception classes (errors.hpp:7-41);
 * validation happens before any work, in the reference's order
 * (conv_fft.hpp:76-83, :117-122, :156-164): shape/size checks, then the
 * layer config (config_error), then the workspace capacity.
 *
 * Threading: a workspace serves one invocation at a time (conv_fft.hpp:37-38);
 * calls on one workspace are not reentrant.  Device entry points enqueue on
 * the caller's stream and return without synchronising.  Consecutive calls
 * on one workspace are ordered even across streams: a call on a stream other
 * than the previous call's first waits for that call to finish on the device
 * (the host entry points included; not inside a stream capture).
 */
#ifndef FFTCONV_B200_H_
#define FFTCONV_B200_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Status codes -- fftconv::error subclasses (errors.hpp). */
enum fftconv_b200_status {
  FFTCONV_B200_OK = 0,
  FFTCONV_B200_SIZE_ERROR = 1,     /* fftconv::size_error     */
  FFTCONV_B200_SHAPE_ERROR = 2,    /* fftconv::shape_error    */
  FFTCONV_B200_CONFIG_ERROR = 3,   /* fftconv::config_error   */
  FFTCONV_B200_CAPACITY_ERROR = 4, /* fftconv::capacity_error */
  FFTCONV_B200_PLAN_ERROR = 5,     /* fftconv::plan_error     */
  FFTCONV_B200_CUDA_ERROR = 6,     /* CUDA runtime/driver failure */
  FFTCONV_B200_NCCL_ERROR = 7,     /* NCCL missing or a collective failed */
  FFTCONV_B200_INVALID_ARGUMENT = 8
};

/* fftconv::LayerConfig (layer_config.hpp:22-40): {k, n, f, f', S}. */
typedef struct fftconv_b200_layer {
  size_t kernel;   /* k  */
  size_t image;    /* n  */
  size_t in_maps;  /* f  */
  size_t out_maps; /* f' */
  size_t batch;    /* S  */
} fftconv_b200_layer;

typedef struct fftconv_b200_ws fftconv_b200_ws;

/* ConvWorkspace<T>::ConvWorkspace(configs)  conv_fft.hpp:43-58
 * Capacities are the per-role maxima over `configs` exactly as the
 * reference computes them; device buffers are allocated once here.
 * Empty list or invalid config -> FFTCONV_B200_CONFIG_ERROR. */
int fftconv_b200_ws_create(const fftconv_b200_layer* configs, size_t count, int device,
                           fftconv_b200_ws** out);
void fftconv_b200_ws_destroy(fftconv_b200_ws* ws);

/* Thread-local message of the last failure on this thread, or of the
 * workspace (when non-NULL). */
const char* fftconv_b200_last_error(const fftconv_b200_ws* ws);

/* Precision scheme of the per-bin complex GEMM (K3): the process default
 * (fftconv_b200_set_gemm_kind, atomic) and a per-workspace override
 * (fftconv_b200_ws_set_gemm_kind).  All
 * keep fp32-level accuracy (rel. L2 ~1e-6 against the fp64 oracle):
 *   FFTCONV_B200_GEMM_TF32X3 x = tf32 hi + lo, D = hi.hi + hi.lo + lo.hi
 *       on kind::tf32 -- per-element exponents, the fp32 range;
 *   FFTCONV_B200_GEMM_F16X3 each operand scaled by one power of two from
 *       its max magnitude (found by K1) and split into fp16 hi + mid;
 *       D = hi.hi + hi.mid + mid.hi on kind::f16 (twice the tf32 rate).
 *       Components below ~2^-24 of their operand's maximum lose relative
 *       precision (absolute error ~2^-38 of the maximum);
 *   FFTCONV_B200_GEMM_AUTO (default) 3xTF32 where the GEMM is bound by its
 *       bytes anyway; where it is tensor-bound, an fp16x3 kernel and a
 *       3xTF32 fallback are launched back to back and exactly one runs:
 *       fp16x3 iff every operand row's maximum is within 2^18 of its
 *       operand's maximum (K1 records the per-row maxima).
 * m < 4 always uses 3xTF32.  The environment variable FFTCONV_B200_GEMM
 * = tf32 | f16x3 | auto selects the initial kind.  Returns the previous
 * kind, or -1 for an unknown kind. */
#define FFTCONV_B200_GEMM_F16X3 0
#define FFTCONV_B200_GEMM_TF32X3 1
#define FFTCONV_B200_GEMM_AUTO 2
int fftconv_b200_set_gemm_kind(int kind);
/* Per-workspace override of the above; kind -1 returns the workspace to the
 * process default.  Returns the previous override (-1 = none), or -1 for an
 * unknown kind / NULL workspace. */
int fftconv_b200_ws_set_gemm_kind(fftconv_b200_ws* ws, int kind);
/* Which GEMM kernel ran in the workspace's last operator call (synchronises
 * the device): 1 fp16x3, 0 3xTF32, -1 none yet / error. */
int fftconv_b200_last_gemm_path(fftconv_b200_ws* ws);

/* ConvWorkspace::max_fft_size/capacity_x/capacity_w/capacity_y/
 * frequency_bytes  conv_fft.hpp:60-69.
 * out[0..4] = max_fft_size, cap_x, cap_w, cap_y, frequency_bytes (the
 * reference's accounting); out[5] = device bytes actually held. */
int fftconv_b200_ws_info(const fftconv_b200_ws* ws, uint64_t out[6]);

/* ConvWorkspace::counters / reset_counters  conv_fft.hpp:71-72 (OpCounters
 * :22-28): out = forward_transforms, inverse_transforms, complex_macs. */
int fftconv_b200_counters(const fftconv_b200_ws* ws, uint64_t out[3]);
int fftconv_b200_reset_counters(fftconv_b200_ws* ws);

/* ---- Device-pointer operators (inputs/outputs resident in HBM) ---------- */

/* ConvWorkspace<float>::forward(x, w)  conv_fft.hpp:74-113.
 * x: [S][f][x_rows][x_cols]; w: [w_out][w_in][k][k]; y: [S][w_out][n'][n'].
 * `stream` is a cudaStream_t (NULL = legacy default stream). */
int fftconv_b200_forward(fftconv_b200_ws* ws, const float* x, size_t S, size_t f, size_t x_rows,
                         size_t x_cols, const float* w, size_t w_out, size_t w_in, size_t k,
                         float* y, void* stream);

/* forward followed by the layer stack's relu (layers.hpp:88-97), fused into
 * the inverse transform's stores: y = max(forward(x, w), 0) with the
 * reference's x > 0 ? x : 0.  Same arguments and errors as
 * fftconv_b200_forward; the stack's relu backward can use y as its mask. */
int fftconv_b200_forward_relu(fftconv_b200_ws* ws, const float* x, size_t S, size_t f, size_t x_rows,
                              size_t x_cols, const float* w, size_t w_out, size_t w_in, size_t k,
                              float* y, void* stream);

/* The layer stack's fit_to (layers.hpp:393-407) folded into the operators.
 * forward_fit: x holds the top-left x_rows x x_cols of a layer image of
 * image x image (zeros elsewhere; x_rows <= image), y is the layer's
 * (image - k + 1)^2 output -- the same as fit_to(x, image) then forward,
 * without materialising the padded input.  flags: FFTCONV_B200_FIT_RELU
 * fuses the following relu (as fftconv_b200_forward_relu).
 * grad_input_fit: only the top-left gx_size x gx_size of each input-gradient
 * plane (gx: [S][w_in][gx_size][gx_size], gx_size <= gy_rows + k - 1), i.e.
 * grad_input then fit_to(gx, gx_size) for a crop.
 * grad_weight_fit: x as in forward_fit (k = image - gy_rows + 1). */
#define FFTCONV_B200_FIT_RELU 1u
int fftconv_b200_forward_fit(fftconv_b200_ws* ws, const float* x, size_t S, size_t f, size_t x_rows,
                             size_t x_cols, size_t image, const float* w, size_t w_out, size_t w_in, size_t k,
                             float* y, unsigned flags, void* stream);
int fftconv_b200_grad_input_fit(fftconv_b200_ws* ws, const float* gy, size_t S, size_t fo, size_t gy_rows,
                                size_t gy_cols, const float* w, size_t w_out, size_t w_in, size_t k, float* gx,
                                size_t gx_size, void* stream);
int fftconv_b200_grad_weight_fit(fftconv_b200_ws* ws, const float* gy, size_t Sg, size_t fo, size_t gy_rows,
                                 size_t gy_cols, const float* x, size_t Sx, size_t f, size_t x_rows, size_t x_cols,
                                 size_t image, float* gw, void* stream);

/* ConvWorkspace<float>::grad_input(gy, w)  conv_fft.hpp:115-152.
 * gy: [S][fo][gy_rows][gy_cols]; gx: [S][w_in][n][n], n = gy_rows + k - 1. */
int fftconv_b200_grad_input(fftconv_b200_ws* ws, const float* gy, size_t S, size_t fo,
                            size_t gy_rows, size_t gy_cols, const float* w, size_t w_out,
                            size_t w_in, size_t k, float* gx, void* stream);

/* ConvWorkspace<float>::grad_weight(gy, x)  conv_fft.hpp:154-206.
 * gw: [fo][f][k][k], k = x_rows - gy_rows + 1. */
int fftconv_b200_grad_weight(fftconv_b200_ws* ws, const float* gy, size_t S_gy, size_t fo,
                             size_t gy_rows, size_t gy_cols, const float* x, size_t S_x,
                             size_t f, size_t x_rows, size_t x_cols, float* gw, void* stream);

/* ---- Minibatch-sharded accGrad (BASELINE configs[3] / [4]) ----------------
 * fprop and bprop of a minibatch shard are the plain device entry points on
 * the shard (no communication; batch decomposability, conv_direct_test.cpp:
 * 186-212).  accGrad's weight gradient is the sum over shards:
 * fftconv_b200_grad_weight_sharded runs the local grad_weight (conv_fft.hpp:
 * 154-206) with its final c2r/crop stage in `chunks` f'-row chunks and
 * all-reduces (sum) each chunk's rows of gw over `comm` (an ncclComm_t) on
 * an internal stream as soon as that chunk's launch finishes, so the
 * collective overlaps the remaining chunks.  `stream` waits for the last
 * all-reduce: on return-and-sync every rank holds the full-batch gradient.
 * With flags & FFTCONV_B200_SHARDED_ASYNC the stream does not wait: the
 * collective keeps running behind whatever the caller enqueues next (a
 * training step's remaining backward layers; gw must not be read, and the
 * next sharded call on this workspace orders itself after it) until
 * fftconv_b200_comm_wait(ws, stream) makes `stream` wait for every
 * all-reduce issued so far.
 * A rank whose shard is empty (S_gy == S_x == 0, world > S) contributes
 * zeros.  NCCL is loaded at run time (libnccl.so.2); FFTCONV_B200_NCCL_ERROR
 * if it is missing or a collective fails.
 * The three helpers create the communicator without linking NCCL: rank 0
 * gets a 128-byte unique id, the caller distributes it (MPI, torch.distributed
 * ...), every rank creates its communicator on its device. */
int fftconv_b200_nccl_get_unique_id(void* id /* 128 bytes */);
int fftconv_b200_nccl_comm_create(const void* id, int nranks, int rank, int device, void** comm);
int fftconv_b200_nccl_comm_destroy(void* comm);
int fftconv_b200_grad_weight_sharded(fftconv_b200_ws* ws, const float* gy, size_t S_gy, size_t fo,
                                     size_t gy_rows, size_t gy_cols, const float* x, size_t S_x, size_t f,
                                     size_t x_rows, size_t x_cols, float* gw, void* comm, int chunks,
                                     unsigned flags, void* stream);
#define FFTCONV_B200_SHARDED_ASYNC 1u
int fftconv_b200_comm_wait(fftconv_b200_ws* ws, void* stream);
/* Host-buffer form of the above (the drop-in's Tensor4 storage): this rank's
 * shard is copied in (chunked H2D pipeline), its gw computed, all-reduced
 * over `comm` and copied back; returns with the full-batch gradient in `gw`. */
int fftconv_b200_grad_weight_sharded_host(fftconv_b200_ws* ws, const float* gy, size_t S_gy, size_t fo,
                                          size_t gy_rows, size_t gy_cols, const float* x, size_t S_x,
                                          size_t f, size_t x_rows, size_t x_cols, float* gw, void* comm,
                                          unsigned threads);
/* With stage timing enabled, the last sharded call's all-reduce timing (ms):
 * out[0] = first all-reduce start -> last all-reduce end (collective span),
 * out[1] = end of the local transforms -> last all-reduce end (the part not
 * hidden behind the chunked c2r). */
int fftconv_b200_comm_ms(fftconv_b200_ws* ws, float out[2]);

/* ---- Host-pointer operators (the drop-in: Tensor4/Weights4 storage) ------
 * Same contracts; inputs are copied host->device, the result device->host,
 * and the call returns after the result is in `y`/`gx`/`gw`.  `threads`
 * is accepted for interface parity (conv_fft.hpp:75) and ignored. */
int fftconv_b200_forward_host(fftconv_b200_ws* ws, const float* x, size_t S, size_t f,
                              size_t x_rows, size_t x_cols, const float* w, size_t w_out,
                              size_t w_in, size_t k, float* y, unsigned threads);
int fftconv_b200_grad_input_host(fftconv_b200_ws* ws, const float* gy, size_t S, size_t fo,
                                 size_t gy_rows, size_t gy_cols, const float* w, size_t w_out,
                                 size_t w_in, size_t k, float* gx, unsigned threads);
int fftconv_b200_grad_weight_host(fftconv_b200_ws* ws, const float* gy, size_t S_gy, size_t fo,
                                  size_t gy_rows, size_t gy_cols, const float* x, size_t S_x,
                                  size_t f, size_t x_rows, size_t x_cols, float* gw,
                                  unsigned threads);

/* ---- Packed-spectrum API (fft.hpp:105-152, :209-243) --------------------
 * fft_2d_real_batch: `planes` real m x m planes (already padded to the plan
 * size, fp32, device) -> their packed half spectra in the reference's
 * HalfSpectrum layout, spec[p][u][v] for u < m, v <= m/2 (complex
 * interleaved fp32), unnormalised.  ifft_2d_real_batch: the inverse, full
 * m x m planes scaled by 1/m^2 (as the reference's two 1/m passes); like the
 * reference's c2r it reads only the packed columns and drops the imaginary
 * parts c2r discards.  Both run on the K1 / K4 kernels, enqueued on
 * `stream`; `scratch` is a device buffer of at least
 * fftconv_b200_spectrum_scratch_bytes(planes, m) bytes (0 for an invalid m).
 * m must be a power of two (FFTCONV_B200_PLAN_ERROR, FftPlan) of at most
 * 128 (FFTCONV_B200_SIZE_ERROR). */
size_t fftconv_b200_spectrum_scratch_bytes(size_t planes, size_t m);
int fftconv_b200_fft_2d_real_batch(const float* planes, size_t planes_count, size_t m, float* spec,
                                   void* scratch, size_t scratch_bytes, void* stream);
int fftconv_b200_ifft_2d_real_batch(const float* spec, size_t planes_count, size_t m, float* planes,
                                    void* scratch, size_t scratch_bytes, void* stream);

/* ---- Instrumentation ----------------------------------------------------
 * When enabled, each operator records CUDA events between its stages on
 * the launching stream; fftconv_b200_stage_ms returns the last call's
 * per-stage device times (ms): [0] r2c of operand A (of both operands when
 * one launch transforms both), [1] r2c of operand B (~0 when merged),
 * [2] per-bin complex GEMM, [3] c2r + crop.  Blocks until they are known. */
int fftconv_b200_set_stage_timing(fftconv_b200_ws* ws, int enable);
int fftconv_b200_stage_ms(fftconv_b200_ws* ws, float out[4]);

/* Live kernel spans with the programmatic-dependent-launch chain intact (no
 * events between the kernels): when enabled (synchronises the device and
 * clears up to 128 operator slots), each operator's K1 / K3 / K4 (TMA
 * kernels, m in 4..64) record, on the GPU's global timer, the first CTA past
 * its dependency wait and the last CTA done.  fftconv_b200_span_ms writes
 * out[3 i + k] (ms; -1 where not recorded) for the first min(ops, max_ops)
 * operators since enabling and returns that count (negative status on
 * error). */
int fftconv_b200_set_span_timing(fftconv_b200_ws* ws, int enable);
int fftconv_b200_span_ms(fftconv_b200_ws* ws, float* out, int max_ops);

/* Number of kernel launches the last operator call enqueued. */
int fftconv_b200_last_launch_count(const fftconv_b200_ws* ws);

/* ---- Layer-stack stages (training-step driver, layers.hpp) ---------------
 * Device pointers, enqueued on `stream`.  Used by the stack driver
 * (paper_1312_5851_b200/layers.py) around the convolution operators. */
/* relu_forward / relu_backward  layers.hpp:88-109 (n elements). */
int fftconv_b200_relu_forward(const float* x, float* y, size_t n, void* stream);
int fftconv_b200_relu_backward(const float* gy, const float* x, float* gx, size_t n,
                               void* stream);
/* maxpool_forward  layers.hpp:34-66: 2x2 / stride 2 over `planes` planes of
 * rows x cols (both even, else FFTCONV_B200_SIZE_ERROR); argmax[o] = flat
 * index of the winner inside its input plane (ties: earliest, row-major). */
int fftconv_b200_maxpool_forward(const float* x, size_t planes, size_t rows, size_t cols,
                                 float* y, uint32_t* argmax, void* stream);
/* maxpool_backward  layers.hpp:68-83: gx (planes x rows x cols) = gy routed
 * to each window's winner, zero elsewhere. */
int fftconv_b200_maxpool_backward(const float* gy, const uint32_t* argmax, size_t planes,
                                  size_t rows, size_t cols, float* gx, void* stream);
/* maxpool_backward followed by the relu_backward of the relu the pool
 * consumed (layers.hpp:68-83 then :99-109), in one pass: gx = gy routed to
 * each window's winner where the pooled value y > 0 (the winner's relu
 * output, so relu(x) > 0 exactly where x > 0), zero elsewhere -- what the two
 * kernels produce, bit for bit.  y is maxpool_forward's output. */
int fftconv_b200_maxpool_relu_backward(const float* gy, const uint32_t* argmax, const float* y, size_t planes,
                                       size_t rows, size_t cols, float* gx, void* stream);
/* fit_to  layers.hpp:393-407: every plane padded with zeros or cropped at
 * the top-left corner to size x size. */
int fftconv_b200_fit_to(const float* x, size_t planes, size_t rows, size_t cols, float* y,
                        size_t size, void* stream);

/* ---- Unit-level test hooks (K1 / K4 / K3 in isolation) ------------------ */

/* Forward 2-D real transforms of `planes` square src x src planes
 * (zero-padded to m x m, m = next_pow2 >= src) into the half spectrum
 * out[p][u][v] = F[u][v] (u in [0, m/2], v in [0, m)), complex interleaved.
 * The reference HalfSpectrum (fft.hpp:105-152) keeps the other half,
 * F[u][v] for v <= m/2; the two are related by F[u][v] =
 * conj(F[(m-u)%m][(m-v)%m]) (paper_1312_5851_b200/spectra.py repacks). */
int fftconv_b200_debug_r2c(const float* in, size_t planes, size_t src, size_t m, float* out,
                           void* stream);
/* Inverse of the above with top-left crop x crop, scaled by 1/m^2. */
int fftconv_b200_debug_c2r(const float* in, size_t planes, size_t m, size_t crop, float* out,
                           void* stream);
/* Batched complex GEMM per bin, mode 0 fprop (A.conj(B)^T), 1 bprop
 * (A.B^T), 2 accGrad (conj(A).B^T): a [bins][M][K], b [bins][N][K],
 * out [bins][N][M], all complex interleaved fp32. */
int fftconv_b200_debug_cgemm(const float* a, const float* b, float* out, size_t bins, size_t M,
                             size_t N, size_t K, int mode, void* stream);

#ifdef __cplusplus
}
#endif

#endif /* FFTCONV_B200_H_ */
