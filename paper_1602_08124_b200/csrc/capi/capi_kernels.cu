// extern "C" kernel-level entry points (plain pointers, no torch types).
#include <cuda_runtime.h>

#include <string>

#include "../kernels/kernels.h"
#include "capi_common.h"

using vdnncapi::fail;

namespace {
bool to_args(const vdnn_conv_desc* d, vdnnk::ConvArgs& a) {
  if (!d || d->nseg < 1 || d->nseg > vdnnk::kMaxConvSegs) return false;
  a.n = d->n;
  a.h = d->h;
  a.w = d->w;
  a.nseg = d->nseg;
  for (int i = 0; i < d->nseg; ++i) {
    a.x[i] = d->x[i];
    a.dx[i] = d->dx[i];
    a.c[i] = d->c[i];
  }
  a.cout = d->cout;
  a.kh = d->kh;
  a.kw = d->kw;
  a.stride = d->stride;
  a.pad = d->pad;
  return true;
}
vdnn_status cuda_status(cudaError_t e, const char* what) {
  if (e == cudaSuccess) return VDNN_OK;
  return fail(VDNN_CUDA_ERROR, std::string(what) + ": " + cudaGetErrorString(e));
}
}  // namespace

extern "C" {

uint64_t vdnn_kernel_launch_count(void) { return vdnnk::launch_count(); }
void vdnn_kernel_set_precise(int32_t on) { vdnnk::set_precise(on != 0); }
void vdnn_kernel_set_tma(int32_t on) {
  vdnnk::set_tma(on != 0);
  vdnnk::set_tma_bf16(on != 0);
}
uint64_t vdnn_kernel_zvc_slot_bytes(uint64_t bytes) { return vdnnk::zvc_slot_bytes(bytes); }
vdnn_status vdnn_kernel_zvc_compress(const float* src, uint64_t count, void* host_dst, uint64_t* wire, void* stream) {
  if (!src || !host_dst || !wire) return fail(VDNN_INVALID_ARGUMENT, "null argument");
  if (!vdnnk::zvc_eligible(src, count * 4) || !vdnnk::zvc_eligible(host_dst, 16))
    return fail(VDNN_INVALID_ARGUMENT, "zvc needs count % 4 == 0 and 16-B aligned buffers");
  return cuda_status(vdnnk::zvc_compress(src, count, host_dst, reinterpret_cast<unsigned long long*>(wire),
                                         static_cast<cudaStream_t>(stream)),
                     "zvc_compress");
}
vdnn_status vdnn_kernel_zvc_compress_tf32(const float* src, uint64_t count, void* host_dst, uint64_t* wire,
                                          void* stream) {
  if (!src || !host_dst || !wire) return fail(VDNN_INVALID_ARGUMENT, "null argument");
  if (!vdnnk::zvc_eligible(src, count * 4) || !vdnnk::zvc_eligible(host_dst, 16))
    return fail(VDNN_INVALID_ARGUMENT, "zvc needs count % 4 == 0 and 16-B aligned buffers");
  return cuda_status(vdnnk::zvc_compress(src, count, host_dst, reinterpret_cast<unsigned long long*>(wire),
                                         static_cast<cudaStream_t>(stream), true),
                     "zvc_compress_tf32");
}
vdnn_status vdnn_kernel_zvc_decompress(const void* host_src, uint64_t count, float* dst, uint64_t* wire,
                                       void* stream) {
  if (!host_src || !dst) return fail(VDNN_INVALID_ARGUMENT, "null argument");
  if (!vdnnk::zvc_eligible(dst, count * 4) || !vdnnk::zvc_eligible(host_src, 16))
    return fail(VDNN_INVALID_ARGUMENT, "zvc needs count % 4 == 0 and 16-B aligned buffers");
  return cuda_status(vdnnk::zvc_decompress(host_src, count, dst, reinterpret_cast<unsigned long long*>(wire),
                                           static_cast<cudaStream_t>(stream)),
                     "zvc_decompress");
}
uint64_t vdnn_kernel_zvc_slot_bytes_bf16(uint64_t bytes) { return vdnnk::zvc_slot_bytes_bf16(bytes); }
vdnn_status vdnn_kernel_zvc_compress_bf16(const void* src, uint64_t count, void* host_dst, uint64_t* wire,
                                          void* stream) {
  if (!src || !host_dst || !wire) return fail(VDNN_INVALID_ARGUMENT, "null argument");
  if (count % 8 != 0 || !vdnnk::zvc_eligible(src, count * 2) || !vdnnk::zvc_eligible(host_dst, 16))
    return fail(VDNN_INVALID_ARGUMENT, "bf16 zvc needs count % 8 == 0 and 16-B aligned buffers");
  return cuda_status(vdnnk::zvc_compress_bf16(src, count, host_dst, reinterpret_cast<unsigned long long*>(wire),
                                              static_cast<cudaStream_t>(stream)),
                     "zvc_compress_bf16");
}
vdnn_status vdnn_kernel_zvc_decompress_bf16(const void* host_src, uint64_t count, void* dst, uint64_t* wire,
                                            void* stream) {
  if (!host_src || !dst) return fail(VDNN_INVALID_ARGUMENT, "null argument");
  if (count % 8 != 0 || !vdnnk::zvc_eligible(dst, count * 2) || !vdnnk::zvc_eligible(host_src, 16))
    return fail(VDNN_INVALID_ARGUMENT, "bf16 zvc needs count % 8 == 0 and 16-B aligned buffers");
  return cuda_status(vdnnk::zvc_decompress_bf16(host_src, count, dst, reinterpret_cast<unsigned long long*>(wire),
                                                static_cast<cudaStream_t>(stream)),
                     "zvc_decompress_bf16");
}
vdnn_status vdnn_kernel_tf32_peak(double* tflops) {
  if (!tflops) return fail(VDNN_INVALID_ARGUMENT, "null output");
  return cuda_status(vdnnk::tf32_peak_probe(tflops), "tf32 peak probe");
}

vdnn_status vdnn_kernel_conv_fprop(const vdnn_conv_desc* d, const float* w, const float* bias, float* y,
                                   void* stream) {
  vdnnk::ConvArgs a;
  if (!to_args(d, a)) return fail(VDNN_INVALID_ARGUMENT, "bad conv descriptor");
  return cuda_status(vdnnk::conv_fprop(a, w, bias, y, false, static_cast<cudaStream_t>(stream)), "conv_fprop");
}

vdnn_status vdnn_kernel_conv_dgrad(const vdnn_conv_desc* d, const float* w, const float* dy, int32_t accumulate,
                                   void* stream) {
  vdnnk::ConvArgs a;
  if (!to_args(d, a)) return fail(VDNN_INVALID_ARGUMENT, "bad conv descriptor");
  if (a.stride != 1) return fail(VDNN_UNSUPPORTED, "dgrad implemented for stride 1 only");
  return cuda_status(vdnnk::conv_dgrad(a, w, dy, accumulate != 0, static_cast<cudaStream_t>(stream)),
                     "conv_dgrad");
}

vdnn_status vdnn_kernel_conv_wgrad(const vdnn_conv_desc* d, const float* dy, float* w, float lr, float* dw_out,
                                   float* ws, size_t ws_bytes, void* stream) {
  vdnnk::ConvArgs a;
  if (!to_args(d, a)) return fail(VDNN_INVALID_ARGUMENT, "bad conv descriptor");
  return cuda_status(vdnnk::conv_wgrad(a, dy, w, lr, dw_out, ws, ws_bytes, static_cast<cudaStream_t>(stream)),
                     "conv_wgrad");
}

vdnn_status vdnn_kernel_conv_fprop_ws(const vdnn_conv_desc* d, const float* w, const float* bias, float* y, float* ws,
                                      size_t ws_bytes, void* stream) {
  vdnnk::ConvArgs a;
  if (!to_args(d, a)) return fail(VDNN_INVALID_ARGUMENT, "bad conv descriptor");
  return cuda_status(vdnnk::conv_fprop(a, w, bias, y, false, static_cast<cudaStream_t>(stream), ws, ws_bytes),
                     "conv_fprop");
}
size_t vdnn_kernel_conv_fprop_ws_bytes(const vdnn_conv_desc* d) {
  vdnnk::ConvArgs a;
  if (!to_args(d, a)) return 0;
  return vdnnk::conv_fprop_ws_bytes(a);
}

vdnn_status vdnn_kernel_conv_dgrad_ws(const vdnn_conv_desc* d, const float* w, const float* dy, int32_t accumulate,
                                      float* ws, size_t ws_bytes, void* stream) {
  vdnnk::ConvArgs a;
  if (!to_args(d, a)) return fail(VDNN_INVALID_ARGUMENT, "bad conv descriptor");
  if (a.stride != 1) return fail(VDNN_UNSUPPORTED, "dgrad implemented for stride 1 only");
  return cuda_status(
      vdnnk::conv_dgrad(a, w, dy, accumulate != 0, static_cast<cudaStream_t>(stream), ws, ws_bytes), "conv_dgrad");
}
size_t vdnn_kernel_conv_dgrad_ws_bytes(const vdnn_conv_desc* d) {
  vdnnk::ConvArgs a;
  if (!to_args(d, a)) return 0;
  return vdnnk::conv_dgrad_ws_bytes(a);
}

size_t vdnn_kernel_conv_wgrad_ws_bytes(const vdnn_conv_desc* d) {
  vdnnk::ConvArgs a;
  if (!to_args(d, a)) return 0;
  return vdnnk::conv_wgrad_ws_bytes(a);
}

static bool to_pool(const vdnn_conv_desc* d, int32_t window, int32_t stride, vdnnk::PoolArgs& p) {
  if (!d || d->nseg < 1 || d->nseg > vdnnk::kMaxConvSegs) return false;
  p.n = d->n;
  p.h = d->h;
  p.w = d->w;
  p.window = window;
  p.stride = stride;
  p.nseg = d->nseg;
  for (int i = 0; i < d->nseg; ++i) {
    p.x[i] = d->x[i];
    p.dx[i] = d->dx[i];
    p.c[i] = d->c[i];
  }
  return true;
}

vdnn_status vdnn_kernel_maxpool_fwd(const vdnn_conv_desc* d, int32_t window, int32_t stride, float* y,
                                    void* stream) {
  vdnnk::PoolArgs p;
  if (!to_pool(d, window, stride, p)) return fail(VDNN_INVALID_ARGUMENT, "bad pool descriptor");
  return cuda_status(vdnnk::maxpool_fwd(p, y, static_cast<cudaStream_t>(stream)), "maxpool_fwd");
}

vdnn_status vdnn_kernel_maxpool_bwd(const vdnn_conv_desc* d, int32_t window, int32_t stride, const float* y,
                                    const float* dy, void* stream) {
  vdnnk::PoolArgs p;
  if (!to_pool(d, window, stride, p)) return fail(VDNN_INVALID_ARGUMENT, "bad pool descriptor");
  return cuda_status(vdnnk::maxpool_bwd(p, y, dy, static_cast<cudaStream_t>(stream)), "maxpool_bwd");
}

vdnn_status vdnn_kernel_relu_fwd(float* y, size_t n, void* stream) {
  return cuda_status(vdnnk::relu_fwd(y, n, static_cast<cudaStream_t>(stream)), "relu_fwd");
}

vdnn_status vdnn_kernel_relu_bwd(float* g, const float* y, size_t n, void* stream) {
  return cuda_status(vdnnk::relu_bwd(g, nullptr, 0, y, n, static_cast<cudaStream_t>(stream)), "relu_bwd");
}

vdnn_status vdnn_kernel_softmax_xent(const float* logits, const int32_t* labels, int32_t n, int32_t k, float* grad,
                                     float* row_loss, float* loss, void* stream) {
  return cuda_status(
      vdnnk::softmax_xent_fwd(logits, labels, n, k, grad, row_loss, loss, static_cast<cudaStream_t>(stream)),
      "softmax_xent");
}

vdnn_status vdnn_kernel_bias_grad(const float* dy, int32_t n, int32_t o, float* bias, float lr, float* db_out,
                                  void* stream) {
  return cuda_status(vdnnk::bias_grad(dy, n, o, bias, lr, db_out, static_cast<cudaStream_t>(stream)),
                     "bias_grad");
}

}  // extern "C"
