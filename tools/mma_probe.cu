// tcgen05.mma kind::tf32 issue ceiling by operand major-ness and N (tool).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++20 -I paper_1602_08124_b200/csrc/kernels \
//        tools/mma_probe.cu -o /tmp/mma_probe
#include <cstdio>

#include "tc_conv.cuh"
using namespace vdnnk;

__global__ void __launch_bounds__(128, 1) probe(int iters, int n, int amn, int bmn, float* sink) {
  extern __shared__ uint8_t smem_raw[];
  const uint32_t base = (smem_u32(smem_raw) + 1023u) & ~1023u;
  const uint32_t tslot = base + 65536, bar = base + 65536 + 16;
  if (threadIdx.x == 0) {
    mbar_init(bar, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (threadIdx.x < 32) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(tslot), "r"(256)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  uint32_t tmem;
  asm volatile("ld.shared.u32 %0, [%1];" : "=r"(tmem) : "r"(tslot) : "memory");
  if (threadIdx.x == 0) {
    const uint32_t idesc = make_idesc_tf32(n, amn, bmn);
    const uint32_t sa = base, sb = base + 16384;
    for (int i = 0; i < iters; ++i) {
#pragma unroll
      for (int kk = 0; kk < 4; ++kk) {
        const uint64_t ad = amn ? make_sdesc(sa + kk * 1024, 4096, 512, kSw128Base32) : make_sdesc(sa + kk * 32, 16, 1024, kSw128);
        const uint64_t bd = bmn ? make_sdesc(sb + kk * 1024, 4096, 512, kSw128Base32) : make_sdesc(sb + kk * 32, 16, 1024, kSw128);
        tc_mma_tf32(tmem, ad, bd, idesc, 1u);
      }
    }
    tc_commit(bar);
    mbar_wait(bar, 0);
  }
  tc_fence_before();
  __syncthreads();
  if (threadIdx.x < 32) {
    tc_fence_after();
    float v[32];
    tmem_ld32(tmem, v);
    if (v[0] == 12345.f) sink[0] = v[1];
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(256) : "memory");
  }
}

int main() {
  float* sink;
  cudaMalloc(&sink, 4);
  const int smem = 65536 + 1024 + 64;
  cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  for (int amn = 0; amn < 2; ++amn)
    for (int bmn = 0; bmn < 2; ++bmn)
      for (int n : {64, 128, 256}) {
        const int iters = 10000;
        probe<<<148, 128, smem>>>(100, n, amn, bmn, sink);
        cudaEvent_t a, b;
        cudaEventCreate(&a);
        cudaEventCreate(&b);
        cudaEventRecord(a);
        probe<<<148, 128, smem>>>(iters, n, amn, bmn, sink);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms;
        cudaEventElapsedTime(&ms, a, b);
        printf("A %s B %s N %3d: %.1f TFLOP/s %s\n", amn ? "MN" : "K ", bmn ? "MN" : "K ", n,
               2.0 * 128 * n * 32 * double(iters) * 148 / ms / 1e9, cudaGetErrorString(cudaGetLastError()));
      }
  return 0;
}
