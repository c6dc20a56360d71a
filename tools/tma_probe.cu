// TMA issue-rate probe: one thread per CTA streams im2col (or tiled) boxes of
// P pixels x 32 fp32 channels into a ring of S stages (mbarrier complete_tx),
// no consumer work. Reports boxes/us per SM and GB/s.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++20 -I paper_1602_08124_b200/csrc/kernels \
//        tools/tma_probe.cu -o /tmp/tma_probe -lcuda
#include <cstdio>
#include <cstring>

#include "tc_conv.cuh"
#include "tma_maps.h"
using namespace vdnnk;

struct Geo {
  int N, H, W, C;
};

__global__ void __launch_bounds__(32, 1) probe(const __grid_constant__ CUtensorMap map, Geo g, int pix, int stages,
                                               int iters, int mode, int ops_per_stage) {
  extern __shared__ uint8_t smem_raw[];
  const uint32_t base = (smem_u32(smem_raw) + 1023u) & ~1023u;
  const uint32_t bars = base + stages * ops_per_stage * pix * 128;
  if (threadIdx.x != 0) return;
  for (int s = 0; s < stages; ++s) mbar_init(bars + 8 * s, 1);
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  int m = 0, w = 0, h = 0, n = 0;
  for (int it = 0; it < iters; ++it) {
    const int s = it % stages;
    if (it >= stages) mbar_wait(bars + 8 * s, ((it / stages) & 1) ^ 1);
    mbar_expect_tx(bars + 8 * s, ops_per_stage * pix * 128);
    for (int o = 0; o < ops_per_stage; ++o) {
      // walk the tensor linearly (cheap address math: the probe must not be issue-bound)
      m += pix;
      w += pix;
      while (w >= g.W) { w -= g.W; ++h; }
      if (h >= g.H) { h = 0; ++n; }
      if (n >= g.N - 1) { n = 0; m = 0; }
      const uint32_t dst = base + (s * ops_per_stage + o) * pix * 128;
      if (mode == 0)
        tma_load_im2col(dst, &map, bars + 8 * s, (o % (g.C / 32)) * 32, w - 1, h - 1, n, 1, 1);
      else
        tma_load_2d(dst, &map, bars + 8 * s, (o % (g.C / 32)) * 32, m);
    }
  }
  for (int it = iters - stages; it < iters; ++it) mbar_wait(bars + 8 * (it % stages), (it / stages) & 1);
}

int main() {
  Geo g{8, 56, 56, 128};
  float* x;
  const size_t n = size_t(g.N) * g.H * g.W * g.C;
  cudaMalloc(&x, n * 4);
  cudaMemset(x, 0, n * 4);
  for (int mode = 0; mode < 2; ++mode)
    for (int cfg = 0; cfg < 6; ++cfg) {
      const int pix = (cfg < 3) ? 32 : 128;
      const int stages = (cfg % 3 == 0) ? 2 : (cfg % 3 == 1) ? 4 : 8;
      alignas(64) CUtensorMap map;
      memset(&map, 0, sizeof(map));
      bool ok;
      if (mode == 0) {
        ok = encode_im2col(&map, x, g.N, g.H, g.W, g.C, 3, 1, 1, pix,
                           pix == 32 ? CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B : CU_TENSOR_MAP_SWIZZLE_128B);
      } else {
        const cuuint64_t dims[2] = {(cuuint64_t)g.C, (cuuint64_t)g.N * g.H * g.W};
        const cuuint64_t strides[1] = {(cuuint64_t)g.C * 4};
        const cuuint32_t box[2] = {32, (cuuint32_t)pix};
        ok = encode_tiled(&map, x, 2, dims, strides, box, CU_TENSOR_MAP_SWIZZLE_128B);
      }
      if (!ok) { printf("encode failed\n"); continue; }
      const int ops = pix == 32 ? 4 : 1, iters = 4000;
      const int smem = stages * ops * pix * 128 + 1024 + 256;
      if (smem > 227 * 1024) continue;
      cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
      probe<<<148, 32, smem>>>(map, g, pix, stages, 50, mode, ops);
      cudaEvent_t a, b;
      cudaEventCreate(&a);
      cudaEventCreate(&b);
      cudaEventRecord(a);
      probe<<<148, 32, smem>>>(map, g, pix, stages, iters, mode, ops);
      cudaEventRecord(b);
      cudaEventSynchronize(b);
      float ms;
      cudaEventElapsedTime(&ms, a, b);
      const double boxes = 148.0 * iters * ops;
      printf("stages %d ops %d ", stages, ops);
      printf("%s pix %3d: %.2f boxes/us/SM  %.0f GB/s  (%s)\n", mode ? "tiled " : "im2col", pix,
             boxes / 148 / (ms * 1e3), boxes * pix * 128 / ms / 1e6, cudaGetErrorString(cudaGetLastError()));
    }
  return 0;
}
