// First-layer convolutions (input channels C <= 4, e.g. RGB images): exact
// fp32 SIMT kernels. With C = 3 the implicit-GEMM K dimension (k*k*3 = 27 for
// VGG, 363 for AlexNet/OverFeat) neither fills a 32-wide tensor-core K block
// per tap nor admits TMA (12-byte pixel stride), so the tensor-core engine
// would fall back to 4-byte gathers; these kernels stage the input patch and
// the weights in shared memory instead.
//
//   fprop: Y[n][oh][ow][co] = sum_{r,s,c} X[n][oh*S-P+r][ow*S-P+s][c] * W[co][r][s][c]
//   wgrad: dW[co][r][s][c]  = sum_{n,oh,ow} dY[n][oh][ow][co] * X[...]   (deterministic
//          per-block partials + ordered reduce, fused SGD)
// FLOPs as the reference counts them: 2*k^2*C*Cout*Ho*Wo*N (cost_model.hpp:100-106).
#include <algorithm>

#include "kernels.h"

namespace vdnnk {

namespace {
constexpr int kTW = 64;     // output pixels per fprop block (2 per lane)
constexpr int kCoBlk = 32;  // output channels per fprop block (8 per warp, 4 warps)
}  // namespace

// grid: (ceil(Wo/64), ceil(Ho/RG), N * ceil(Cout/32)), block 128. Each block
// keeps its 32-channel weight slice in shared memory across RG output rows.
constexpr int kRG = 16;
__global__ void __launch_bounds__(128) smallc_fprop_kernel(const float* __restrict__ x, const float* __restrict__ w,
                                                           float* __restrict__ y, int H, int W, int C, int Ho,
                                                           int Wo, int Cout, int k, int stride, int pad, int relu) {
  extern __shared__ float sm[];
  const int ktot = k * k * C;
  const int span = (kTW - 1) * stride + k;
  float* ws = sm;                           // [ktot][32]
  float* patch = sm + ktot * kCoBlk;        // [k][span][C]
  const int ncb = (Cout + kCoBlk - 1) / kCoBlk;
  const int n = blockIdx.z / ncb;
  const int co0 = (blockIdx.z % ncb) * kCoBlk;
  const int ow0 = blockIdx.x * kTW;
  const int tid = threadIdx.x;
  for (int i = tid; i < ktot * kCoBlk; i += blockDim.x) {
    const int co = i / ktot, kk = i - co * ktot;
    ws[kk * kCoBlk + co] = (co0 + co < Cout) ? w[static_cast<size_t>(co0 + co) * ktot + kk] : 0.f;
  }
  const int warp = tid >> 5, lane = tid & 31;
  const int cw = warp * 8;  // 8 channels per warp
  const int cbase = co0 + cw;
  const int p0 = lane, p1 = lane + 32;
  const int prow = span * C;
  const int iw0 = ow0 * stride - pad;
  const int oh_end = min(Ho, (blockIdx.y + 1) * kRG);
  for (int oh = blockIdx.y * kRG; oh < oh_end; ++oh) {
    __syncthreads();  // previous row's patch fully consumed (and weights visible on the first pass)
    const int ih0 = oh * stride - pad;
    for (int i = tid; i < k * prow; i += blockDim.x) {
      const int r = i / prow, rem = i - r * prow;
      const int ih = ih0 + r, iw = iw0 + rem / C;
      patch[i] = (ih >= 0 && ih < H && iw >= 0 && iw < W)
                     ? __ldg(x + ((static_cast<size_t>(n) * H + ih) * W) * C + static_cast<size_t>(iw0) * C + rem)
                     : 0.f;
    }
    __syncthreads();
    float a0[8], a1[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) a0[j] = a1[j] = 0.f;
    for (int r = 0; r < k; ++r) {
      const float* pr = patch + r * prow;
      const float* wr = ws + (r * k * C) * kCoBlk + cw;
      const int q0 = p0 * stride * C, q1 = p1 * stride * C;
      for (int sc = 0; sc < k * C; ++sc) {  // (s, c) is contiguous in the patch row
        const float x0 = pr[q0 + sc], x1 = pr[q1 + sc];
        const float4 wa = *reinterpret_cast<const float4*>(wr + sc * kCoBlk);
        const float4 wb = *reinterpret_cast<const float4*>(wr + sc * kCoBlk + 4);
        const float wv[8] = {wa.x, wa.y, wa.z, wa.w, wb.x, wb.y, wb.z, wb.w};
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          a0[j] = fmaf(x0, wv[j], a0[j]);
          a1[j] = fmaf(x1, wv[j], a1[j]);
        }
      }
    }
    for (int h = 0; h < 2; ++h) {
      const int ow = ow0 + (h ? p1 : p0);
      if (ow >= Wo) continue;
      float* dst = y + ((static_cast<size_t>(n) * Ho + oh) * Wo + ow) * Cout + cbase;
      const float* a = h ? a1 : a0;
      if (cbase + 8 <= Cout && (Cout & 3) == 0) {
        float4 o0 = make_float4(a[0], a[1], a[2], a[3]), o1 = make_float4(a[4], a[5], a[6], a[7]);
        if (relu) {
          o0 = make_float4(fmaxf(o0.x, 0.f), fmaxf(o0.y, 0.f), fmaxf(o0.z, 0.f), fmaxf(o0.w, 0.f));
          o1 = make_float4(fmaxf(o1.x, 0.f), fmaxf(o1.y, 0.f), fmaxf(o1.z, 0.f), fmaxf(o1.w, 0.f));
        }
        reinterpret_cast<float4*>(dst)[0] = o0;
        reinterpret_cast<float4*>(dst)[1] = o1;
      } else {
#pragma unroll
        for (int j = 0; j < 8; ++j)
          if (cbase + j < Cout) dst[j] = relu ? fmaxf(a[j], 0.f) : a[j];
      }
    }
  }
}

// WGRAD partials: block (bx, by, bz) accumulates a 64(co) x 64(kk) tile over
// its pixel range; 256 threads x (4 co x 4 kk). Staged per 32-pixel batch:
// dys[32][64 co] and xs[32][64 kk]. Each thread always loads the same kk
// column (decoded once) and 8 pixel rows whose window origins are decoded
// once per batch by 32 threads into shared memory.
__global__ void __launch_bounds__(256) smallc_wgrad_kernel(const float* __restrict__ x, const float* __restrict__ dy,
                                                           float* __restrict__ part, int N, int H, int W, int C,
                                                           int Ho, int Wo, int Cout, int k, int stride, int pad,
                                                           int64_t pix_per_block) {
  __shared__ float dys[32][64];
  __shared__ float xs[32][64];
  __shared__ int pix_n[32], pix_h[32], pix_w[32];
  const int ktot = k * k * C;
  const int co0 = blockIdx.y * 64;
  const int kk0 = blockIdx.z * 64;
  const int64_t P = static_cast<int64_t>(N) * Ho * Wo;
  const int64_t pb = static_cast<int64_t>(blockIdx.x) * pix_per_block;
  const int64_t pe = std::min<int64_t>(P, pb + pix_per_block);
  const int tid = threadIdx.x;
  const int tco = (tid >> 4) * 4;  // 16 x 4 co
  const int tkk = (tid & 15) * 4;  // 16 x 4 kk
  // this thread's load column
  const int j = tid & 63;
  const int kk = kk0 + j;
  const bool kk_ok = kk < ktot;
  int dr = 0, ds = 0, dc = 0;
  if (kk_ok) {
    const int tap = kk / C;
    dc = kk - tap * C;
    dr = tap / k;
    ds = tap - dr * k;
  }
  const bool co_ok = co0 + j < Cout;
  float acc[4][4] = {};
  for (int64_t p = pb; p < pe; p += 32) {
    if (tid < 32) {
      const int64_t pp = p + tid;
      if (pp < pe) {
        const int ow = static_cast<int>(pp % Wo);
        const int64_t t = pp / Wo;
        pix_w[tid] = ow * stride - pad;
        pix_h[tid] = static_cast<int>(t % Ho) * stride - pad;
        pix_n[tid] = static_cast<int>(t / Ho);
      } else {
        pix_n[tid] = -1;
      }
    }
    __syncthreads();
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      const int pi = (tid >> 6) + 4 * q;
      const int n = pix_n[pi];
      dys[pi][j] = (n >= 0 && co_ok) ? __ldg(dy + (p + pi) * Cout + co0 + j) : 0.f;
      float v = 0.f;
      if (n >= 0 && kk_ok) {
        const int ih = pix_h[pi] + dr, iw = pix_w[pi] + ds;
        if (ih >= 0 && ih < H && iw >= 0 && iw < W) v = __ldg(x + ((static_cast<size_t>(n) * H + ih) * W + iw) * C + dc);
      }
      xs[pi][j] = v;
    }
    __syncthreads();
#pragma unroll 8
    for (int q = 0; q < 32; ++q) {
      const float4 d4 = *reinterpret_cast<const float4*>(&dys[q][tco]);
      const float4 x4 = *reinterpret_cast<const float4*>(&xs[q][tkk]);
      const float dv[4] = {d4.x, d4.y, d4.z, d4.w};
      const float xv[4] = {x4.x, x4.y, x4.z, x4.w};
#pragma unroll
      for (int a = 0; a < 4; ++a)
#pragma unroll
        for (int b = 0; b < 4; ++b) acc[a][b] = fmaf(dv[a], xv[b], acc[a][b]);
    }
    __syncthreads();
  }
  // partial layout: [block x][co][kk] (only the valid rectangle is reduced)
  float* out = part + static_cast<size_t>(blockIdx.x) * Cout * ktot;
#pragma unroll
  for (int a = 0; a < 4; ++a)
#pragma unroll
    for (int b = 0; b < 4; ++b) {
      const int co = co0 + tco + a, kc = kk0 + tkk + b;
      if (co < Cout && kc < ktot) out[static_cast<size_t>(co) * ktot + kc] = acc[a][b];
    }
}

__global__ void smallc_wgrad_reduce(const float* __restrict__ part, int nparts, int64_t count, float* __restrict__ w,
                                    float lr, float* __restrict__ dw_out) {
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < count;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    float s = 0.f;
    for (int b = 0; b < nparts; ++b) s += part[static_cast<size_t>(b) * count + i];
    if (dw_out)
      dw_out[i] = s;
    else
      w[i] -= lr * s;
  }
}

cudaError_t smallc_wgrad_reduce_launch(const float* part, int nparts, int64_t count, float* w, float lr,
                                       float* dw_out, cudaStream_t st) {
  smallc_wgrad_reduce<<<static_cast<int>(std::min<int64_t>((count + 255) / 256, 1184)), 256, 0, st>>>(
      part, nparts, count, w, lr, dw_out);
  count_launch();
  return cudaGetLastError();
}

bool smallc_eligible(const ConvArgs& a) { return a.nseg == 1 && a.c[0] <= 4 && a.cout >= 1 && a.kh == a.kw; }

size_t smallc_fprop_smem(const ConvArgs& a) {
  const int ktot = a.kh * a.kw * a.c[0];
  const int span = (kTW - 1) * a.stride + a.kh;
  return static_cast<size_t>(ktot * kCoBlk + a.kh * span * a.c[0]) * sizeof(float);
}

cudaError_t smallc_fprop(const ConvArgs& a, const float* w, float* y, cudaStream_t st) {
  const size_t smem = smallc_fprop_smem(a);
  static size_t attr = 0;
  if (smem > 48 * 1024 && smem > attr) {
    cudaError_t e = cudaFuncSetAttribute(smallc_fprop_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         static_cast<int>(std::max<size_t>(smem, 160 * 1024)));
    if (e != cudaSuccess) return e;
    attr = std::max<size_t>(smem, 160 * 1024);
  }
  const int Ho = a.ho(), Wo = a.wo();
  const int ncb = (a.cout + kCoBlk - 1) / kCoBlk;
  dim3 grid((Wo + kTW - 1) / kTW, (Ho + kRG - 1) / kRG, a.n * ncb);
  smallc_fprop_kernel<<<grid, 128, smem, st>>>(a.x[0], w, y, a.h, a.w, a.c[0], Ho, Wo, a.cout, a.kh, a.stride,
                                                a.pad, a.relu_out);
  count_launch();
  return cudaGetLastError();
}

size_t smallc_wgrad_ws_bytes(const ConvArgs& a, int* nblocks_out) {
  const int64_t P = static_cast<int64_t>(a.n) * a.ho() * a.wo();
  const int ktot = a.kh * a.kw * a.c[0];
  const int gy = (a.cout + 63) / 64, gz = (ktot + 63) / 64;
  // ~4 blocks per SM in total, at least 256 pixels each
  int nb = std::max(1, (148 * 4) / (gy * gz));
  nb = static_cast<int>(std::min<int64_t>(nb, (P + 255) / 256));
  if (nblocks_out) *nblocks_out = nb;
  return static_cast<size_t>(nb) * a.cout * ktot * sizeof(float);
}

cudaError_t smallc_wgrad(const ConvArgs& a, const float* dy, float* w, float lr, float* dw_out, float* ws,
                         size_t ws_bytes, cudaStream_t st) {
  int nb = 1;
  const size_t need = smallc_wgrad_ws_bytes(a, &nb);
  const int ktot = a.kh * a.kw * a.c[0];
  const size_t per = static_cast<size_t>(a.cout) * ktot * sizeof(float);
  if (ws == nullptr || ws_bytes < per) return cudaErrorInvalidValue;
  if (need > ws_bytes) nb = static_cast<int>(ws_bytes / per);
  const int64_t P = static_cast<int64_t>(a.n) * a.ho() * a.wo();
  int64_t ppb = (P + nb - 1) / nb;
  ppb = (ppb + 31) / 32 * 32;
  nb = static_cast<int>((P + ppb - 1) / ppb);
  dim3 grid(nb, (a.cout + 63) / 64, (ktot + 63) / 64);
  smallc_wgrad_kernel<<<grid, 256, 0, st>>>(a.x[0], dy, ws, a.n, a.h, a.w, a.c[0], a.ho(), a.wo(), a.cout, a.kh,
                                             a.stride, a.pad, ppb);
  const int64_t count = static_cast<int64_t>(a.cout) * ktot;
  smallc_wgrad_reduce<<<static_cast<int>(std::min<int64_t>((count + 255) / 256, 1184)), 256, 0, st>>>(
      ws, nb, count, w, lr, dw_out);
  count_launch(2);
  return cudaGetLastError();
}

}  // namespace vdnnk
