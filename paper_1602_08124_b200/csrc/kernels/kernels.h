// Host-side launch interface of the sm_100a kernels (internal to libvdnn).
#pragma once
#include <cstddef>
#include <cstdint>
#include <cuda_runtime.h>

namespace vdnnk {

constexpr int kMaxConvSegs = 8;

// A (possibly channel-concatenated) NHWC conv input and its gradient planes.
// FC layers are passed as 1x1 convs over a 1x1 image whose channels are the
// flattened (h, w, c) features of each input segment.
struct ConvArgs {
  int n = 0, h = 0, w = 0;                 // input spatial dims
  int nseg = 0;
  const float* x[kMaxConvSegs] = {};       // segment inputs (fprop / wgrad)
  float* dx[kMaxConvSegs] = {};            // segment gradient planes (dgrad), may be null
  int c[kMaxConvSegs] = {};                // segment channels
  int cout = 0, kh = 1, kw = 1, stride = 1, pad = 0;
  int relu_out = 0;                        // fprop: fused ReLU on the output (the ACTV that follows)
  int mask_in[kMaxConvSegs] = {};          // dgrad: fused ReLU backward, dX *= (x > 0) per segment
  int ho() const { return (h + 2 * pad - kh) / stride + 1; }
  int wo() const { return (w + 2 * pad - kw) / stride + 1; }
  int cin() const {
    int t = 0;
    for (int i = 0; i < nseg; ++i) t += c[i];
    return t;
  }
};

// Tensor-core conv contractions (kind::tf32, fp32 accumulate). With
// set_precise(true) (per calling thread) every contraction runs as 3xTF32
// (hi*hi + hi*lo + lo*hi), i.e. fp32-accurate products.
void set_precise(bool on);
bool precise();
// TMA producers (im2col / tiled tensor maps) where eligible; off = cp.async gathers everywhere.
void set_tma(bool on);
// `ws` (optional, conv_fprop_ws_bytes(a) bytes) enables a deterministic
// split-K for outputs with fewer tiles than SMs (FC layers).
cudaError_t conv_fprop(const ConvArgs& a, const float* w, const float* bias, float* y, bool accumulate,
                       cudaStream_t st, float* ws = nullptr, size_t ws_bytes = 0);
size_t conv_fprop_ws_bytes(const ConvArgs& a);
// `ws` (optional, conv_dgrad_ws_bytes(a) bytes): deterministic split-K for FC
// layers with fewer output tiles than SMs.
cudaError_t conv_dgrad(const ConvArgs& a, const float* w, const float* dy, bool accumulate, cudaStream_t st,
                       float* ws = nullptr, size_t ws_bytes = 0);
size_t conv_dgrad_ws_bytes(const ConvArgs& a);
// SMs the persistent conv kernels leave free for concurrent SM-driven
// transfers (process-wide; -1 = VDNN_SM_RESERVE or 0).
void set_sm_reserve(int sms);
// Weight gradient. If dw_out is null: fused SGD  w_mut -= lr * dW.
// Otherwise dW is written to dw_out (KRSC layout) and w_mut is untouched.
// `ws` holds split-K partials; pass conv_wgrad_ws_bytes(a) bytes (or less:
// fewer splits are used).
cudaError_t conv_wgrad(const ConvArgs& a, const float* dy, float* w_mut, float lr, float* dw_out, float* ws,
                       size_t ws_bytes, cudaStream_t st);
size_t conv_wgrad_ws_bytes(const ConvArgs& a);

// Memory-bound kernels.
cudaError_t relu_fwd(float* y, size_t n, cudaStream_t st);
// g0 = (g0 + sum extra) * (y > 0); in place on g0.
cudaError_t relu_bwd(float* g0, const float* const* extra, int nextra, const float* y, size_t n, cudaStream_t st);
cudaError_t add_into(float* dst, const float* const* src, int nsrc, size_t n, cudaStream_t st);
// dst = sum src[k] (k < nsrc <= 8), then *= (y > 0) if y; dst may alias src[0]; 16-B aligned.
cudaError_t combine(float* dst, const float* const* src, int nsrc, const float* y, size_t n, cudaStream_t st);
// zero-inserted dY of a stride-s conv: ((ho-1)s+1) x ((wo-1)s+1) x c per image
cudaError_t dilate(float* d, const float* dy, int n, int ho, int wo, int c, int stride, cudaStream_t st);
struct PoolArgs {
  int n = 0, h = 0, w = 0, window = 2, stride = 2;
  int nseg = 0;
  const float* x[kMaxConvSegs] = {};
  float* dx[kMaxConvSegs] = {};
  int c[kMaxConvSegs] = {};
  int mask_in[kMaxConvSegs] = {};          // bwd: fused ReLU backward (x is the ReLU's output)
  int ho() const { return (h - window) / stride + 1; }
  int wo() const { return (w - window) / stride + 1; }
  int ctot() const {
    int t = 0;
    for (int i = 0; i < nseg; ++i) t += c[i];
    return t;
  }
};
cudaError_t maxpool_fwd(const PoolArgs& a, float* y, cudaStream_t st);
// `y` (the reference's operand set: X, Y, dY) is not read: the kernels
// recompute each window's maximum from X with the forward's rule.
cudaError_t maxpool_bwd(const PoolArgs& a, const float* y, const float* dy, cudaStream_t st);
// Mean softmax cross-entropy over n rows of k logits. Writes the gradient
// (softmax - onehot)/n into grad_scratch, the per-row loss into row_loss and
// the mean loss into *loss (all device pointers).
// Labels are taken modulo k (several LOSS heads may share one label vector);
// accumulate: *loss += mean instead of *loss = mean (the total over heads).
cudaError_t softmax_xent_fwd(const float* logits, const int32_t* labels, int n, int k, float* grad_scratch,
                             float* row_loss, float* loss, cudaStream_t st, bool accumulate = false);
// bias -= lr * sum_n dy[n][o]   (or db_out[o] = sum when db_out != null)
cudaError_t bias_grad(const float* dy, int n, int o, float* bias, float lr, float* db_out, cudaStream_t st);
cudaError_t sgd_update(float* w, const float* g, float lr, size_t n, cudaStream_t st);
cudaError_t scale_inplace(float* x, float s, size_t n, cudaStream_t st);
// Deterministic synthetic data: He-normal weights, U[-1,1) images, labels.
cudaError_t fill_normal(float* w, size_t n, float stddev, uint64_t seed, cudaStream_t st);
cudaError_t fill_uniform(float* x, size_t n, float lo, float hi, uint64_t seed, cudaStream_t st);
cudaError_t fill_const(float* x, size_t n, float v, cudaStream_t st);
cudaError_t fill_labels(int32_t* y, size_t n, int classes, uint64_t seed, cudaStream_t st);

// Number of kernel launches issued by the calls above since process start
// (used by bench.py's gpu_launches claim).
uint64_t launch_count();
// Zero-value-compressed transfer between a device buffer and a (zero-copy
// mapped) pinned host slot; lossless, see zvc.cu for the format. `count`
// floats (multiple of 4, 16-B aligned); `wire` (device counter, may be null
// for decompress) accumulates the bytes that crossed the link.
constexpr int kZvcChunk = 1024;
constexpr int kZvcSlot = 128 + 16 + 4 * kZvcChunk;  // mask + header + dense values (worst case)
uint64_t zvc_slot_bytes(uint64_t bytes);
bool zvc_eligible(const void* p, uint64_t bytes);
// tf32 = true: nonzeros may travel TF32-exact (low 13 mantissa bits dropped; zvc.cu mode 2)
cudaError_t zvc_compress(const float* src, uint64_t count, void* host_dst, unsigned long long* wire, cudaStream_t st,
                         bool tf32 = false);
cudaError_t zvc_decompress(const void* host_src, uint64_t count, float* dst, unsigned long long* wire,
                           cudaStream_t st);
// BF16 maps (elem_size = 2): chunks of 2048 bf16, a 64-bit zero mask per lane,
// nonzeros as u16 or (narrow top bytes) 1.5 B each; `count` = bf16 elements
// (multiple of 8). Lossless: every restored bit pattern equals the original.
constexpr int kZvcbChunk = 2048;
constexpr int kZvcbSlot = 256 + 16 + 2 * kZvcbChunk;  // mask + header + dense values (worst case)
uint64_t zvc_slot_bytes_bf16(uint64_t bytes);
cudaError_t zvc_compress_bf16(const void* src, uint64_t count, void* host_dst, unsigned long long* wire,
                              cudaStream_t st);
cudaError_t zvc_decompress_bf16(const void* host_src, uint64_t count, void* dst, unsigned long long* wire,
                                cudaStream_t st);
// Data-parallel exchange over peer memory (peer.cu): barrier flags and the
// fused reduce + SGD + broadcast of the weight gradients.
constexpr int kPeerMaxRanks = 8;
struct PeerChunk {
  uint64_t w_off;   // byte offset of the weights from the arena base (identical on every rank)
  uint64_t g_off;   // float offset into the gradient arena
  uint32_t count;   // floats
  uint32_t pad;
};
struct PeerArgs {
  int world = 1, rank = 0;
  char* arena[kPeerMaxRanks] = {};                 // per-rank arena base (local or IPC-mapped)
  const float* grads[kPeerMaxRanks] = {};          // per-rank gradient arena
  unsigned long long* signal[kPeerMaxRanks] = {};  // per-rank flags [2 phases][kPeerMaxRanks]
  const PeerChunk* chunks = nullptr;               // this rank's share (device memory)
  int nchunks = 0;
  float step = 0.f;                                // lr * grad_scale
  int bf16 = 0;                                    // weights stored as bf16 (elem_size 2); gradients fp32
};
cudaError_t peer_barrier(const PeerArgs& a, unsigned long long epoch, int phase, cudaStream_t st);
cudaError_t peer_reduce_sgd(const PeerArgs& a, cudaStream_t st);
// Measured TF32 tensor-core ceiling (TFLOP/s) of the current device.
cudaError_t tf32_peak_probe(double* tflops);
void count_launch(uint64_t k = 1);

// ---- BF16 storage (the reference's elem_size = 2, cost_model.hpp:69) ------
// Same operations over bf16 tensors (tcb_conv.cuh, conv_bf16.cu,
// elementwise_bf16.cu): tcgen05 kind::f16 contractions with fp32 TMEM
// accumulation, memory-bound ops in fp32 registers, one round-to-nearest-even
// per stored value. ConvArgs / PoolArgs pointers address bf16 data here; the
// split-K workspaces, the optional dW / db outputs and the SGD gradient
// arena are fp32.
cudaError_t conv_fprop_bf16(const ConvArgs& a, const void* w, const void* bias, void* y, bool accumulate,
                            cudaStream_t st, float* ws = nullptr, size_t ws_bytes = 0);
size_t conv_fprop_ws_bytes_bf16(const ConvArgs& a);
cudaError_t conv_dgrad_bf16(const ConvArgs& a, const void* w, const void* dy, bool accumulate, cudaStream_t st,
                            float* ws = nullptr, size_t ws_bytes = 0);
size_t conv_dgrad_ws_bytes_bf16(const ConvArgs& a);
cudaError_t conv_wgrad_bf16(const ConvArgs& a, const void* dy, void* w_mut, float lr, float* dw_out, float* ws,
                            size_t ws_bytes, cudaStream_t st);
size_t conv_wgrad_ws_bytes_bf16(const ConvArgs& a);
// TMA producers where eligible (default) or cp.async gathers everywhere (per thread)
void set_tma_bf16(bool on);
cudaError_t relu_fwd_bf16(void* y, size_t n, cudaStream_t st);
cudaError_t relu_bwd_bf16(void* g0, const void* const* extra, int nextra, const void* y, size_t n, cudaStream_t st);
cudaError_t add_into_bf16(void* dst, const void* const* src, int nsrc, size_t n, cudaStream_t st);
cudaError_t combine_bf16(void* dst, const void* const* src, int nsrc, const void* y, size_t n, cudaStream_t st);
cudaError_t dilate_bf16(void* d, const void* dy, int n, int ho, int wo, int c, int stride, cudaStream_t st);
cudaError_t maxpool_fwd_bf16(const PoolArgs& a, void* y, cudaStream_t st);
cudaError_t maxpool_bwd_bf16(const PoolArgs& a, const void* dy, cudaStream_t st);
cudaError_t softmax_xent_fwd_bf16(const void* logits, const int32_t* labels, int n, int k, void* grad_scratch,
                                  float* row_loss, float* loss, cudaStream_t st, bool accumulate = false);
cudaError_t bias_grad_bf16(const void* dy, int n, int o, void* bias, float lr, float* db_out, cudaStream_t st);
cudaError_t sgd_update_bf16(void* w, const float* g, float lr, size_t n, cudaStream_t st);
cudaError_t fill_normal_bf16(void* w, size_t n, float stddev, uint64_t seed, cudaStream_t st);
cudaError_t fill_uniform_bf16(void* x, size_t n, float lo, float hi, uint64_t seed, cudaStream_t st);
cudaError_t fill_const_bf16(void* x, size_t n, float v, cudaStream_t st);
// The reference's GEMM_WS algorithm as kernels (conv_gemmws.cu): im2col of a
// single-segment conv input into the planned workspace (gemmws_col_bytes),
// the contraction as a 1x1 conv over it (gemmws_args), and col2im of the
// column gradient into dX (fused ReLU-backward mask / accumulation).
uint64_t gemmws_col_bytes(const ConvArgs& a, int es);
cudaError_t im2col(const ConvArgs& a, int es, void* col, cudaStream_t st);
cudaError_t col2im(const ConvArgs& a, int es, const void* dcol, bool accumulate, cudaStream_t st);
ConvArgs gemmws_args(const ConvArgs& a, const void* col, void* dcol);
// First layers (C <= 8, kh*kw*C <= 64) that the dedicated BF16 kernels of
// conv_c3tcb.cu run in fprop and wgrad (no channel padding needed)
bool conv_bf16_c3_native(const ConvArgs& a);
// [rows][c] <-> [rows][cp] channel padding (zeros in c..cp)
cudaError_t pad_channels_bf16(void* dst, const void* src, size_t rows, int c, int cp, cudaStream_t st);
cudaError_t unpad_channels_bf16(void* dst, const void* src, size_t rows, int c, int cp, cudaStream_t st);
cudaError_t unpad_channels_f32(float* dst, const float* src, size_t rows, int c, int cp, cudaStream_t st);
cudaError_t f32_to_bf16(void* dst, const float* src, size_t n, cudaStream_t st);
cudaError_t bf16_to_f32(float* dst, const void* src, size_t n, cudaStream_t st);

}  // namespace vdnnk
