// Probe (tool): CTA-pair (cta_group::2) tcgen05.mma kind::tf32, M=256 x N=256.
// Checks the operand/accumulator split (A rows and D lanes 0-127 in CTA rank
// 0, 128-255 in rank 1; B rows n 0-127 in rank 0, 128-255 in rank 1), the
// cta_group::2 TMEM alloc and the multicast commit, then measures the
// streaming rate (operands walking through smem, no reuse).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++20 -I paper_1602_08124_b200/csrc/kernels \
//        tools/pair_probe.cu -o tools/pair_probe
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "tc_conv.cuh"
using namespace vdnnk;

__device__ __forceinline__ uint32_t cluster_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ void cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
__device__ __forceinline__ void mma2_tf32(uint32_t d, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n"
      " tcgen05.mma.cta_group::2.kind::tf32 [%0], %1, %2, %3, p;\n}\n" ::"r"(d),
      "l"(a), "l"(b), "r"(idesc), "r"(acc)
      : "memory");
}
__device__ __forceinline__ void commit2(uint32_t bar) {
  asm volatile(
      "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(bar),
      "h"(static_cast<uint16_t>(3))
      : "memory");
}
__host__ __device__ constexpr uint32_t idesc_m256(int n) {
  return (make_idesc_tf32(n, false, false) & ~(0x1Fu << 24)) | ((256u >> 4) << 24);
}

constexpr int kStage = 32768;  // A 128 x 128 B + B 128 x 128 B per CTA

__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(128, 1)
    pair_mma(const float* A, const float* B, float* D, int iters, float* sink) {
  extern __shared__ uint8_t smem_raw[];
  const uint32_t base = (smem_u32(smem_raw) + 1023u) & ~1023u;
  const uint32_t tslot = base + 3 * kStage, bar = tslot + 16;
  const uint32_t rank = cluster_rank();
  if (iters == 0) {  // correctness: stage 0 holds this CTA's A rows and B rows
    for (int e = threadIdx.x; e < 128 * 8; e += blockDim.x) {
      const int r = e / 8, j = e % 8;
      const float* a = A + (rank * 128 + r) * 32 + j * 4;
      const float* b = B + (rank * 128 + r) * 32 + j * 4;
      asm volatile("st.shared.v4.f32 [%0], {%1,%2,%3,%4};" ::"r"(kmaj_addr(base, r, j)), "f"(a[0]), "f"(a[1]),
                   "f"(a[2]), "f"(a[3]));
      asm volatile("st.shared.v4.f32 [%0], {%1,%2,%3,%4};" ::"r"(kmaj_addr(base + 16384, r, j)), "f"(b[0]),
                   "f"(b[1]), "f"(b[2]), "f"(b[3]));
    }
    fence_proxy_async();
  }
  if (threadIdx.x == 0) {
    mbar_init(bar, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (threadIdx.x < 32) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(tslot), "r"(256)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
  }
  tc_fence_before();
  __syncthreads();
  cluster_sync_all();
  tc_fence_after();
  uint32_t tmem;
  asm volatile("ld.shared.u32 %0, [%1];" : "=r"(tmem) : "r"(tslot) : "memory");
  if (rank == 0 && threadIdx.x < 32) {
    const bool leader = elect_one();
    if (leader) {
      const uint32_t idesc = idesc_m256(256);
      const int n = iters == 0 ? 1 : iters;
      for (int i = 0; i < n; ++i) {
        const uint32_t st = base + (i % 3) * kStage;
#pragma unroll
        for (int kk = 0; kk < 4; ++kk)
          mma2_tf32(tmem, make_sdesc(st + kk * 32, 16, 1024, kSw128), make_sdesc(st + 16384 + kk * 32, 16, 1024, kSw128),
                    idesc, (i > 0 || kk > 0) ? 1u : 0u);
      }
      commit2(bar);
    }
    __syncwarp();
  }
  mbar_wait(bar, 0);
  tc_fence_after();
  if (iters == 0) {
    const int w = threadIdx.x / 32;
    const int row = rank * 128 + w * 32 + (threadIdx.x & 31);
    for (int cg = 0; cg < 8; ++cg) {
      float v[32];
      tmem_ld32(tmem + ((w * 32) << 16) + cg * 32, v);
      for (int j = 0; j < 32; ++j) D[row * 256 + cg * 32 + j] = v[j];
    }
  } else if (threadIdx.x < 32) {
    float v[32];
    tmem_ld32(tmem, v);
    if (v[0] == 12345.f) sink[0] = v[1];
  }
  tc_fence_before();
  __syncthreads();
  cluster_sync_all();
  if (threadIdx.x < 32)
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(256) : "memory");
}

int main() {
  std::vector<float> A(256 * 32), B(256 * 32), D(256 * 256);
  srand(3);
  for (auto& v : A) v = float(rand() % 17 - 8) / 8.f;
  for (auto& v : B) v = float(rand() % 17 - 8) / 8.f;
  float *dA, *dB, *dD, *sink;
  cudaMalloc(&dA, A.size() * 4);
  cudaMalloc(&dB, B.size() * 4);
  cudaMalloc(&dD, D.size() * 4);
  cudaMalloc(&sink, 4);
  cudaMemcpy(dA, A.data(), A.size() * 4, cudaMemcpyHostToDevice);
  cudaMemcpy(dB, B.data(), B.size() * 4, cudaMemcpyHostToDevice);
  const int smem = 3 * kStage + 1024 + 64;
  cudaFuncSetAttribute(pair_mma, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  pair_mma<<<2, 128, smem>>>(dA, dB, dD, 0, sink);
  cudaError_t e = cudaDeviceSynchronize();
  cudaMemcpy(D.data(), dD, D.size() * 4, cudaMemcpyDeviceToHost);
  int bad = 0;
  for (int i = 0; i < 256; ++i)
    for (int j = 0; j < 256; ++j) {
      float ref = 0;
      for (int k = 0; k < 32; ++k) ref += A[i * 32 + k] * B[j * 32 + k];
      if (D[i * 256 + j] != ref) ++bad;
    }
  printf("pair M256xN256xK32: %s, %d mismatches\n", cudaGetErrorString(e), bad);
  for (int rep = 0; rep < 2; ++rep) {
    const int iters = 4000;
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    cudaEventRecord(a);
    pair_mma<<<148, 128, smem>>>(dA, dB, dD, iters, sink);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    printf("pair streaming rate: %.1f TFLOP/s %s\n", 2.0 * 256 * 256 * 32 * double(iters) * 74 / ms / 1e9,
           cudaGetErrorString(cudaGetLastError()));
  }
  return 0;
}
