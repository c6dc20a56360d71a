// Debug harness for the tcgen05 conv engine vs a CPU loop (fprop only).
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <vector>
#include "../paper_1602_08124_b200/csrc/kernels/kernels.h"
static float rnd() { return (rand() % 2001 - 1000) / 1000.0f; }
int run(int n, int h, int w, int c, int cout, int k, int stride, int pad) {
  int ho = (h + 2 * pad - k) / stride + 1, wo = (w + 2 * pad - k) / stride + 1;
  std::vector<float> hx((size_t)n * h * w * c), hw((size_t)cout * k * k * c), hy((size_t)n * ho * wo * cout, -7.f);
  for (auto& v : hx) v = rnd();
  for (auto& v : hw) v = rnd();
  float *dx, *dw, *dy;
  cudaMalloc(&dx, hx.size() * 4); cudaMalloc(&dw, hw.size() * 4); cudaMalloc(&dy, hy.size() * 4);
  cudaMemcpy(dx, hx.data(), hx.size() * 4, cudaMemcpyHostToDevice);
  cudaMemcpy(dw, hw.data(), hw.size() * 4, cudaMemcpyHostToDevice);
  cudaMemcpy(dy, hy.data(), hy.size() * 4, cudaMemcpyHostToDevice);
  vdnnk::ConvArgs a; a.n = n; a.h = h; a.w = w; a.nseg = 1; a.x[0] = dx; a.c[0] = c; a.cout = cout;
  a.kh = a.kw = k; a.stride = stride; a.pad = pad;
  cudaError_t e = vdnnk::conv_fprop(a, dw, nullptr, dy, false, 0);
  cudaError_t e2 = cudaDeviceSynchronize();
  cudaMemcpy(hy.data(), dy, hy.size() * 4, cudaMemcpyDeviceToHost);
  double maxerr = 0, maxref = 0; int shown = 0;
  for (int b = 0; b < n; ++b) for (int oh = 0; oh < ho; ++oh) for (int ow = 0; ow < wo; ++ow) for (int o = 0; o < cout; ++o) {
    double s = 0;
    for (int r = 0; r < k; ++r) for (int q = 0; q < k; ++q) {
      int ih = oh * stride - pad + r, iw = ow * stride - pad + q;
      if (ih < 0 || ih >= h || iw < 0 || iw >= w) continue;
      for (int ci = 0; ci < c; ++ci) s += (double)hx[(((size_t)b * h + ih) * w + iw) * c + ci] * hw[(((size_t)o * k + r) * k + q) * c + ci];
    }
    double got = hy[(((size_t)b * ho + oh) * wo + ow) * cout + o];
    maxerr = fmax(maxerr, fabs(got - s)); maxref = fmax(maxref, fabs(s));
    if (fabs(got - s) > 1e-2 * (1 + fabs(s)) && shown < 6) { printf("  y[%d,%d,%d,%d]=%g ref %g\n", b, oh, ow, o, got, s); ++shown; }
  }
  printf("case n%d h%d w%d c%d cout%d k%d s%d p%d: %s/%s maxerr %.3e maxref %.3e\n", n, h, w, c, cout, k, stride, pad,
         cudaGetErrorString(e), cudaGetErrorString(e2), maxerr, maxref);
  cudaFree(dx); cudaFree(dw); cudaFree(dy);
  return 0;
}

int run_bwd(int n, int h, int w, int c, int cout, int k, int pad) {
  int ho = h + 2 * pad - k + 1, wo = w + 2 * pad - k + 1;
  std::vector<float> hx((size_t)n * h * w * c), hw((size_t)cout * k * k * c), hdy((size_t)n * ho * wo * cout);
  for (auto& v : hx) v = rnd();
  for (auto& v : hw) v = rnd();
  for (auto& v : hdy) v = rnd();
  std::vector<float> hdx(hx.size(), -7.f), hdw(hw.size(), -7.f);
  float *dx, *dw, *ddy, *ddx, *ddw;
  cudaMalloc(&dx, hx.size() * 4); cudaMalloc(&dw, hw.size() * 4); cudaMalloc(&ddy, hdy.size() * 4);
  cudaMalloc(&ddx, hx.size() * 4); cudaMalloc(&ddw, hw.size() * 4);
  cudaMemcpy(dx, hx.data(), hx.size() * 4, cudaMemcpyHostToDevice);
  cudaMemcpy(dw, hw.data(), hw.size() * 4, cudaMemcpyHostToDevice);
  cudaMemcpy(ddy, hdy.data(), hdy.size() * 4, cudaMemcpyHostToDevice);
  cudaMemcpy(ddx, hdx.data(), hdx.size() * 4, cudaMemcpyHostToDevice);
  cudaMemcpy(ddw, hdw.data(), hdw.size() * 4, cudaMemcpyHostToDevice);
  vdnnk::ConvArgs a; a.n = n; a.h = h; a.w = w; a.nseg = 1; a.x[0] = dx; a.dx[0] = ddx; a.c[0] = c; a.cout = cout;
  a.kh = a.kw = k; a.stride = 1; a.pad = pad;
  cudaError_t e1 = vdnnk::conv_dgrad(a, dw, ddy, false, 0);
  cudaError_t e2 = vdnnk::conv_wgrad(a, ddy, dw, 0.f, ddw, nullptr, 0, 0);
  cudaError_t e3 = cudaDeviceSynchronize();
  cudaMemcpy(hdx.data(), ddx, hx.size() * 4, cudaMemcpyDeviceToHost);
  cudaMemcpy(hdw.data(), ddw, hw.size() * 4, cudaMemcpyDeviceToHost);
  std::vector<double> rdx(hx.size(), 0), rdw(hw.size(), 0);
  for (int b = 0; b < n; ++b) for (int oh = 0; oh < ho; ++oh) for (int ow = 0; ow < wo; ++ow) for (int o = 0; o < cout; ++o) {
    double g = hdy[(((size_t)b * ho + oh) * wo + ow) * cout + o];
    for (int r = 0; r < k; ++r) for (int q = 0; q < k; ++q) {
      int ih = oh - pad + r, iw = ow - pad + q;
      if (ih < 0 || ih >= h || iw < 0 || iw >= w) continue;
      for (int ci = 0; ci < c; ++ci) {
        size_t xi = (((size_t)b * h + ih) * w + iw) * c + ci, wi = (((size_t)o * k + r) * k + q) * c + ci;
        rdx[xi] += g * hw[wi]; rdw[wi] += g * hx[xi];
      }
    }
  }
  double ex = 0, rx = 0, ew = 0, rw = 0;
  for (size_t i = 0; i < rdx.size(); ++i) { ex = fmax(ex, fabs(hdx[i] - rdx[i])); rx = fmax(rx, fabs(rdx[i])); }
  for (size_t i = 0; i < rdw.size(); ++i) { ew = fmax(ew, fabs(hdw[i] - rdw[i])); rw = fmax(rw, fabs(rdw[i])); }
  printf("bwd n%d h%d w%d c%d cout%d k%d p%d: %s %s %s dgrad err %.3e/%.3e wgrad err %.3e/%.3e  dx0 %g ref %g  dw0 %g ref %g\n",
         n, h, w, c, cout, k, pad, cudaGetErrorString(e1), cudaGetErrorString(e2), cudaGetErrorString(e3), ex, rx, ew, rw,
         hdx[0], rdx[0], hdw[0], rdw[0]);
  run_bwd(1, 1, 32, 32, 32, 1, 0);
  run_bwd(1, 1, 128, 32, 64, 1, 0);
  run_bwd(2, 14, 14, 64, 128, 3, 1);
  run_bwd(2, 8, 8, 5, 7, 3, 1);
  return 0;
}
int main() {
  run(1, 1, 128, 32, 64, 1, 1, 0);
  run(1, 1, 128, 256, 64, 1, 1, 0);   // 8 k-blocks: pipeline wraps
  run(1, 1, 128, 32, 128, 1, 1, 0);   // BN=128
  run(1, 1, 300, 64, 64, 1, 1, 0);    // multiple M tiles, partial
  run(2, 14, 14, 64, 128, 3, 1, 1);   // case0
  run(3, 35, 35, 3, 64, 11, 4, 0);    // scalar
  run_bwd(1, 1, 32, 32, 32, 1, 0);
  run_bwd(1, 1, 128, 32, 64, 1, 0);
  run_bwd(2, 14, 14, 64, 128, 3, 1);
  run_bwd(2, 8, 8, 5, 7, 3, 1);
  return 0;
}
