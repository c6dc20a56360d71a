// The reference's GEMM_WS convolution algorithm as real kernels
// (cost_model.hpp:163-168: the workspace is the im2col matrix,
// k*k*Cin*Ho*Wo*N elements): im2col of X into the planned workspace, the
// contraction as a 1x1 GEMM over it on the tensor-core engine, and for the
// data gradient the inverse gather (col2im) of the GEMM's column gradient.
// Opt-in (Session option algo_kernels = planned): on the B200 the implicit
// GEMM is faster at every VGG layer (profiles/r02s4_algo_probe.txt), so the
// default executor runs it for every planned algorithm and only reserves the
// workspace.
//
//   col[p][(r*k + s)*C + c] = X[n][oh*stride - pad + r][ow*stride - pad + s][c]
//   (p = (n*Ho + oh)*Wo + ow; zero outside the image) -- the KRSC weight
//   column order, so Y = col x W^T and dW = dY^T x col are 1x1 contractions
//   dX[n][ih][iw][c] = sum over (r, s) with ih = oh*stride - pad + r, iw = ...
//   of dcol[p][(r*k + s)*C + c], then the fused ReLU-backward mask / accumulate
//   of the implicit dgrad
#include <cuda_bf16.h>

#include <algorithm>

#include "kernels.h"

namespace vdnnk {

namespace {

struct ColGeom {
  int n, h, w, c, k, stride, pad, ho, wo;
  int64_t kk;  // k*k*c
};

__device__ __forceinline__ float ld_f(const float* p, int64_t i) { return p[i]; }
__device__ __forceinline__ float ld_f(const __nv_bfloat16* p, int64_t i) { return __bfloat162float(p[i]); }
__device__ __forceinline__ void st_f(float* p, int64_t i, float v) { p[i] = v; }
__device__ __forceinline__ void st_f(__nv_bfloat16* p, int64_t i, float v) { p[i] = __float2bfloat16_rn(v); }

// one thread per (p, column); the channel index is fastest, so a warp reads
// consecutive channels of one input pixel and writes consecutive columns
template <typename T>
__global__ void im2col_kernel(const T* __restrict__ x, T* __restrict__ col, ColGeom g) {
  const int64_t total = static_cast<int64_t>(g.n) * g.ho * g.wo * g.kk;
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < total;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t p = i / g.kk;
    const int q = static_cast<int>(i - p * g.kk);
    const int tap = q / g.c, c = q - tap * g.c;
    const int r = tap / g.k, s = tap - r * g.k;
    const int ow = static_cast<int>(p % g.wo);
    const int64_t t = p / g.wo;
    const int oh = static_cast<int>(t % g.ho);
    const int nn = static_cast<int>(t / g.ho);
    const int ih = oh * g.stride - g.pad + r, iw = ow * g.stride - g.pad + s;
    T v{};
    if (ih >= 0 && ih < g.h && iw >= 0 && iw < g.w)
      v = x[((static_cast<int64_t>(nn) * g.h + ih) * g.w + iw) * g.c + c];
    col[i] = v;
  }
}

// one thread per dX element (gather form: deterministic, no atomics)
template <typename T>
__global__ void col2im_kernel(const T* __restrict__ dcol, T* __restrict__ dx, const T* __restrict__ mask_x,
                              int accumulate, ColGeom g) {
  const int64_t total = static_cast<int64_t>(g.n) * g.h * g.w * g.c;
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < total;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int c = static_cast<int>(i % g.c);
    int64_t t = i / g.c;
    const int iw = static_cast<int>(t % g.w);
    t /= g.w;
    const int ih = static_cast<int>(t % g.h);
    const int nn = static_cast<int>(t / g.h);
    float acc = 0.f;
    for (int r = 0; r < g.k; ++r) {
      const int oy = ih + g.pad - r;
      if (oy < 0 || oy % g.stride != 0) continue;
      const int oh = oy / g.stride;
      if (oh >= g.ho) continue;
      for (int s = 0; s < g.k; ++s) {
        const int ox = iw + g.pad - s;
        if (ox < 0 || ox % g.stride != 0) continue;
        const int ow = ox / g.stride;
        if (ow >= g.wo) continue;
        const int64_t p = (static_cast<int64_t>(nn) * g.ho + oh) * g.wo + ow;
        acc += ld_f(dcol, p * g.kk + (r * g.k + s) * g.c + c);
      }
    }
    if (mask_x && !(ld_f(mask_x, i) > 0.f)) acc = 0.f;
    if (accumulate) acc += ld_f(dx, i);
    st_f(dx, i, acc);
  }
}

ColGeom geom(const ConvArgs& a) {
  ColGeom g;
  g.n = a.n;
  g.h = a.h;
  g.w = a.w;
  g.c = a.c[0];
  g.k = a.kh;
  g.stride = a.stride;
  g.pad = a.pad;
  g.ho = a.ho();
  g.wo = a.wo();
  g.kk = static_cast<int64_t>(a.kh) * a.kw * a.c[0];
  return g;
}

int blocks_for(int64_t n) { return static_cast<int>(std::min<int64_t>((n + 255) / 256, 148 * 16)); }

}  // namespace

uint64_t gemmws_col_bytes(const ConvArgs& a, int es) {
  return static_cast<uint64_t>(a.n) * a.ho() * a.wo() * a.kh * a.kw * a.c[0] * es;
}

cudaError_t im2col(const ConvArgs& a, int es, void* col, cudaStream_t st) {
  const ColGeom g = geom(a);
  const int64_t total = static_cast<int64_t>(g.n) * g.ho * g.wo * g.kk;
  if (total == 0) return cudaSuccess;
  if (es == 2)
    im2col_kernel<__nv_bfloat16><<<blocks_for(total), 256, 0, st>>>(
        reinterpret_cast<const __nv_bfloat16*>(a.x[0]), static_cast<__nv_bfloat16*>(col), g);
  else
    im2col_kernel<float><<<blocks_for(total), 256, 0, st>>>(a.x[0], static_cast<float*>(col), g);
  count_launch();
  return cudaGetLastError();
}

cudaError_t col2im(const ConvArgs& a, int es, const void* dcol, bool accumulate, cudaStream_t st) {
  const ColGeom g = geom(a);
  const int64_t total = static_cast<int64_t>(g.n) * g.h * g.w * g.c;
  if (total == 0 || a.dx[0] == nullptr) return cudaSuccess;
  const void* mask = a.mask_in[0] ? static_cast<const void*>(a.x[0]) : nullptr;
  if (es == 2)
    col2im_kernel<__nv_bfloat16><<<blocks_for(total), 256, 0, st>>>(
        static_cast<const __nv_bfloat16*>(dcol), reinterpret_cast<__nv_bfloat16*>(a.dx[0]),
        static_cast<const __nv_bfloat16*>(mask), accumulate ? 1 : 0, g);
  else
    col2im_kernel<float><<<blocks_for(total), 256, 0, st>>>(static_cast<const float*>(dcol), a.dx[0],
                                                            static_cast<const float*>(mask), accumulate ? 1 : 0, g);
  count_launch();
  return cudaGetLastError();
}

// The 1x1 contraction over a column matrix of `a`: P = N*Ho*Wo "pixels" of
// K = k*k*C channels, the layer's Cout outputs.
ConvArgs gemmws_args(const ConvArgs& a, const void* col, void* dcol) {
  ConvArgs g;
  g.n = a.n * a.ho() * a.wo();
  g.h = g.w = 1;
  g.nseg = 1;
  g.x[0] = static_cast<const float*>(col);
  g.dx[0] = static_cast<float*>(dcol);
  g.c[0] = a.kh * a.kw * a.c[0];
  g.cout = a.cout;
  g.kh = g.kw = 1;
  g.stride = 1;
  g.pad = 0;
  g.relu_out = a.relu_out;
  return g;
}

}  // namespace vdnnk
