// Roofline denominator probe: the tcgen05 kind::tf32 issue ceiling of this
// part (M=128, N=256, K=8 MMAs back to back from one thread per CTA, one CTA
// per SM, operands resident in shared memory, no memory traffic). bench.py
// reports conv-engine TFLOP/s against this measured number rather than a
// datasheet figure.
#include "kernels.h"
#include "tc_conv.cuh"

namespace vdnnk {
namespace {

__global__ void __launch_bounds__(128, 1) tf32_peak_kernel(int iters, float* sink) {
  extern __shared__ uint8_t smem_raw[];
  const uint32_t base = (smem_u32(smem_raw) + 1023u) & ~1023u;
  const uint32_t tslot = base + 49152, bar = base + 49152 + 16;
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
    const uint32_t idesc = make_idesc_tf32(256, false, false);
    for (int i = 0; i < iters; ++i) {
#pragma unroll
      for (int kk = 0; kk < 4; ++kk)
        tc_mma_tf32(tmem, make_sdesc(base + kk * 32, 16, 1024, kSw128),
                    make_sdesc(base + 16384 + kk * 32, 16, 1024, kSw128), idesc, 1u);
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
    if (v[0] == 1234.5f) sink[0] = v[1];  // keep the accumulator live
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(256) : "memory");
  }
}

}  // namespace

cudaError_t tf32_peak_probe(double* tflops) {
  constexpr int kSmem = 49152 + 1024 + 64;
  constexpr int kIters = 20000, kCtas = 148;
  float* sink = nullptr;
  cudaError_t e = cudaMalloc(&sink, sizeof(float));
  if (e != cudaSuccess) return e;
  cudaEvent_t a = nullptr, b = nullptr;
  e = cudaFuncSetAttribute(tf32_peak_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmem);
  if (e == cudaSuccess) e = cudaEventCreate(&a);
  if (e == cudaSuccess) e = cudaEventCreate(&b);
  if (e == cudaSuccess) {
    tf32_peak_kernel<<<kCtas, 128, kSmem>>>(200, sink);  // warm-up
    cudaEventRecord(a);
    tf32_peak_kernel<<<kCtas, 128, kSmem>>>(kIters, sink);
    cudaEventRecord(b);
    count_launch(2);
    e = cudaEventSynchronize(b);
  }
  float ms = 0.f;
  if (e == cudaSuccess) e = cudaEventElapsedTime(&ms, a, b);
  if (e == cudaSuccess) e = cudaGetLastError();
  if (e == cudaSuccess) *tflops = 2.0 * 128 * 256 * 32 * static_cast<double>(kIters) * kCtas / (ms * 1e-3) / 1e12;
  if (a) cudaEventDestroy(a);
  if (b) cudaEventDestroy(b);
  cudaFree(sink);
  return e;
}

}  // namespace vdnnk
