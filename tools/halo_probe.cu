// Probe (tool): can a SWIZZLE_128B K-major A operand start at an arbitrary
// 128-B row of a swizzled tile (M shift by s rows, descriptor base-offset
// field = (addr >> 7) & 7)? That is what a halo-reuse conv needs: the 9 taps
// of a 3x3 stride-1 conv read the same staged input rows shifted by s pixels.
// Also measures the kind::tf32 issue rate of M=64 instructions.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++20 -I paper_1602_08124_b200/csrc/kernels \
//        tools/halo_probe.cu -o /tmp/halo_probe
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "tc_conv.cuh"
using namespace vdnnk;

constexpr int ROWS = 144;  // staged A rows (>= 128 + max shift), 18 swizzle atoms
constexpr int NB = 64;     // B rows (N)

__device__ __forceinline__ uint64_t with_base_offset(uint64_t d, uint32_t bo) {
  return d | (static_cast<uint64_t>(bo & 7) << 49);
}

// out[s][i][j] = sum_k A[s + i][k] * B[j][k], k < 32, for shift s (one CTA per (s, variant))
__global__ void __launch_bounds__(128, 1) shift_mma(const float* A, const float* B, float* out, int variant) {
  extern __shared__ uint8_t smem_raw[];
  const uint32_t base = (smem_u32(smem_raw) + 1023u) & ~1023u;
  const uint32_t sa = base, sb = base + ROWS * 128, tslot = sb + NB * 128, bar = tslot + 16;
  const int s = blockIdx.x;
  for (int e = threadIdx.x; e < ROWS * 8; e += blockDim.x) {  // 16-B chunks of A
    const int r = e / 8, j = e % 8;
    const float* src = A + r * 32 + j * 4;
    asm volatile("st.shared.v4.f32 [%0], {%1,%2,%3,%4};" ::"r"(kmaj_addr(sa, r, j)), "f"(src[0]), "f"(src[1]),
                 "f"(src[2]), "f"(src[3]));
  }
  for (int e = threadIdx.x; e < NB * 8; e += blockDim.x) {
    const int r = e / 8, j = e % 8;
    const float* src = B + r * 32 + j * 4;
    asm volatile("st.shared.v4.f32 [%0], {%1,%2,%3,%4};" ::"r"(kmaj_addr(sb, r, j)), "f"(src[0]), "f"(src[1]),
                 "f"(src[2]), "f"(src[3]));
  }
  fence_proxy_async();
  if (threadIdx.x == 0) {
    mbar_init(bar, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (threadIdx.x < 32) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(tslot), "r"(64)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  uint32_t tmem;
  asm volatile("ld.shared.u32 %0, [%1];" : "=r"(tmem) : "r"(tslot) : "memory");
  if (threadIdx.x == 0) {
    const uint32_t idesc = make_idesc_tf32(NB, false, false);
    for (int kk = 0; kk < 4; ++kk) {
      const uint32_t a_start = sa + s * 128 + kk * 32;
      uint64_t ad = make_sdesc(a_start, 16, 1024, kSw128);
      if (variant == 1) ad = with_base_offset(ad, (a_start >> 7) & 7);
      const uint64_t bd = make_sdesc(sb + kk * 32, 16, 1024, kSw128);
      tc_mma_tf32(tmem, ad, bd, idesc, kk > 0 ? 1u : 0u);
    }
    tc_commit(bar);
    mbar_wait(bar, 0);
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const int w = threadIdx.x / 32;
  for (int cg = 0; cg < NB / 32; ++cg) {
    float v[32];
    tmem_ld32(tmem + ((w * 32) << 16) + cg * 32, v);
    const int row = w * 32 + (threadIdx.x & 31);
    for (int j = 0; j < 32; ++j) out[(size_t(blockIdx.x) * 128 + row) * NB + cg * 32 + j] = v[j];
  }
  tc_fence_before();
  __syncthreads();
  if (threadIdx.x < 32)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(64) : "memory");
}

// issue rate of M=128 instructions whose A starts `shift` rows into a swizzled block
__global__ void __launch_bounds__(128, 1) rate_shift(int iters, int shift, float* sink) {
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
    const uint32_t idesc = make_idesc_tf32(128, false, false);
    for (int i = 0; i < iters; ++i)
#pragma unroll
      for (int kk = 0; kk < 4; ++kk)
        tc_mma_tf32(tmem, make_sdesc(base + shift * 128 + kk * 32, 16, 1024, kSw128),
                    make_sdesc(base + 32768 + kk * 32, 16, 1024, kSw128), idesc, 1u);
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

// Tensor-core rate when the operands stream through smem like the conv
// kernels (no operand reuse between consecutive MMAs): stage i uses A at
// base + (i % 4) * 48 KB (two M=128 halves 16 KB apart), B right after;
// shift = tap row offset of A (halo kernel), n = N per MMA.
__global__ void __launch_bounds__(128, 1) rate_stream(int iters, int n, int shift, float* sink) {
  extern __shared__ uint8_t smem_raw[];
  const uint32_t base = (smem_u32(smem_raw) + 1023u) & ~1023u;
  const uint32_t tslot = base + 3 * 67584, bar = tslot + 16;  // ring of 3 x 66 KB
  if (threadIdx.x == 0) {
    mbar_init(bar, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (threadIdx.x < 32) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(tslot), "r"(512)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  uint32_t tmem;
  asm volatile("ld.shared.u32 %0, [%1];" : "=r"(tmem) : "r"(tslot) : "memory");
  if (threadIdx.x == 0) {
    const uint32_t idesc = make_idesc_tf32(n, false, false);
    for (int i = 0; i < iters; ++i) {
      const uint32_t st = base + (i % 3) * 67584;
#pragma unroll
      for (int kk = 0; kk < 4; ++kk)
#pragma unroll
        for (int h = 0; h < 2; ++h)
          tc_mma_tf32(tmem + h * n, make_sdesc(st + h * 16384 + shift * 128 + kk * 32, 16, 1024, kSw128),
                      make_sdesc(st + 33792 + kk * 32, 16, 1024, kSw128), idesc, 1u);
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
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(512) : "memory");
  }
}

// Same streaming pattern, but every `per` K=32 slices (8 MMAs each) the
// issuer does what the conv kernels do between stages: try_wait on a (ready)
// mbarrier, tcgen05 fence, and a tcgen05.commit to a release barrier.
__global__ void __launch_bounds__(128, 1) rate_sync(int iters, int n, int per, float* sink) {
  extern __shared__ uint8_t smem_raw[];
  const uint32_t base = (smem_u32(smem_raw) + 1023u) & ~1023u;
  const uint32_t tslot = base + 3 * 67584, bar = tslot + 16, ready = tslot + 32, rel = tslot + 48;
  if (threadIdx.x == 0) {
    mbar_init(bar, 1);
    mbar_init(ready, 1);
    mbar_init(rel, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (threadIdx.x < 32) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(tslot), "r"(512)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  uint32_t tmem;
  asm volatile("ld.shared.u32 %0, [%1];" : "=r"(tmem) : "r"(tslot) : "memory");
  if (threadIdx.x == 0) {
    mbar_arrive(ready);  // phase 0 of `ready` completes: waits on parity 0 succeed from now on
    const uint32_t idesc = make_idesc_tf32(n, false, false);
    for (int i = 0; i < iters; ++i) {
      const uint32_t st = base + (i % 3) * 67584;
      if (i % per == 0) {
        mbar_wait(ready, 0);
        tc_fence_after();
      }
#pragma unroll
      for (int kk = 0; kk < 4; ++kk)
#pragma unroll
        for (int h = 0; h < 2; ++h)
          tc_mma_tf32(tmem + h * n, make_sdesc(st + h * 16384 + 128 + kk * 32, 16, 1024, kSw128),
                      make_sdesc(st + 33792 + kk * 32, 16, 1024, kSw128), idesc, 1u);
      if (i % per == per - 1) tc_commit(rel);
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
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(512) : "memory");
  }
}

// issue-rate probe of M=64 instructions (idesc M field = 64 >> 4)
__global__ void __launch_bounds__(128, 1) rate_m64(int iters, int n, float* sink) {
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
    const uint32_t idesc = (make_idesc_tf32(n, false, false) & ~(0x1Fu << 24)) | ((64u >> 4) << 24);
    for (int i = 0; i < iters; ++i)
#pragma unroll
      for (int kk = 0; kk < 4; ++kk)
        tc_mma_tf32(tmem, make_sdesc(base + kk * 32, 16, 1024, kSw128), make_sdesc(base + 16384 + kk * 32, 16, 1024, kSw128),
                    idesc, 1u);
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
  std::vector<float> A(ROWS * 32), B(NB * 32);
  srand(1);
  for (auto& v : A) v = float(rand() % 17 - 8) / 8.f;  // exact in tf32
  for (auto& v : B) v = float(rand() % 17 - 8) / 8.f;
  float *dA, *dB, *dO;
  const int S = ROWS - 128 + 1;
  cudaMalloc(&dA, A.size() * 4);
  cudaMalloc(&dB, B.size() * 4);
  cudaMalloc(&dO, size_t(S) * 128 * NB * 4);
  cudaMemcpy(dA, A.data(), A.size() * 4, cudaMemcpyHostToDevice);
  cudaMemcpy(dB, B.data(), B.size() * 4, cudaMemcpyHostToDevice);
  const int smem = ROWS * 128 + NB * 128 + 64 + 1024;
  cudaFuncSetAttribute(shift_mma, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  std::vector<float> O(size_t(S) * 128 * NB);
  for (int variant = 0; variant < 2; ++variant) {
    cudaMemset(dO, 0, O.size() * 4);
    shift_mma<<<S, 128, smem>>>(dA, dB, dO, variant);
    cudaError_t e = cudaDeviceSynchronize();
    cudaMemcpy(O.data(), dO, O.size() * 4, cudaMemcpyDeviceToHost);
    printf("variant %d (%s): %s\n", variant, variant ? "base offset = (addr>>7)&7" : "base offset 0",
           cudaGetErrorString(e));
    for (int s = 0; s < S; ++s) {
      int bad = 0;
      for (int i = 0; i < 128; ++i)
        for (int j = 0; j < NB; ++j) {
          float ref = 0;
          for (int k = 0; k < 32; ++k) ref += A[(s + i) * 32 + k] * B[j * 32 + k];
          if (O[(size_t(s) * 128 + i) * NB + j] != ref) ++bad;
        }
      printf("  shift %2d: %s (%d mismatches)\n", s, bad ? "WRONG" : "exact", bad);
    }
  }
  float* sink;
  cudaMalloc(&sink, 4);
  const int smem2 = 65536 + 1024 + 64;
  cudaFuncSetAttribute(rate_m64, cudaFuncAttributeMaxDynamicSharedMemorySize, smem2);
  const int smem3 = 3 * 67584 + 64 + 1024;
  cudaFuncSetAttribute(rate_stream, cudaFuncAttributeMaxDynamicSharedMemorySize, smem3);
  for (int n : {64, 128, 256})
    for (int shift : {0, 1}) {
      const int iters = 4000;
      rate_stream<<<148, 128, smem3>>>(100, n, shift, sink);
      cudaEvent_t a, b;
      cudaEventCreate(&a);
      cudaEventCreate(&b);
      cudaEventRecord(a);
      rate_stream<<<148, 128, smem3>>>(iters, n, shift, sink);
      cudaEventRecord(b);
      cudaEventSynchronize(b);
      float ms;
      cudaEventElapsedTime(&ms, a, b);
      printf("stream 2x M128 N=%3d shift %d: %.1f TFLOP/s %s\n", n, shift,
             2.0 * 2 * 128 * n * 32 * double(iters) * 148 / ms / 1e9, cudaGetErrorString(cudaGetLastError()));
    }
  cudaFuncSetAttribute(rate_sync, cudaFuncAttributeMaxDynamicSharedMemorySize, smem3);
  for (int n : {128, 256})
    for (int per : {1, 2, 3, 6}) {
      const int iters = 4200;
      rate_sync<<<148, 128, smem3>>>(60, n, per, sink);
      cudaEvent_t a, b;
      cudaEventCreate(&a);
      cudaEventCreate(&b);
      cudaEventRecord(a);
      rate_sync<<<148, 128, smem3>>>(iters, n, per, sink);
      cudaEventRecord(b);
      cudaEventSynchronize(b);
      float ms;
      cudaEventElapsedTime(&ms, a, b);
      printf("sync every %d x 8 MMAs, N=%3d: %.1f TFLOP/s %s\n", per, n,
             2.0 * 2 * 128 * n * 32 * double(iters) * 148 / ms / 1e9, cudaGetErrorString(cudaGetLastError()));
    }
  cudaFuncSetAttribute(rate_shift, cudaFuncAttributeMaxDynamicSharedMemorySize, smem2);
  for (int shift : {0, 1, 2, 3, 8}) {
    const int iters = 10000;
    rate_shift<<<148, 128, smem2>>>(100, shift, sink);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    cudaEventRecord(a);
    rate_shift<<<148, 128, smem2>>>(iters, shift, sink);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    printf("M=128 N=128 A shifted %d rows: %.1f TFLOP/s %s\n", shift, 2.0 * 128 * 128 * 32 * double(iters) * 148 / ms / 1e9,
           cudaGetErrorString(cudaGetLastError()));
  }
  for (int n : {64, 128, 256}) {
    const int iters = 10000;
    rate_m64<<<148, 128, smem2>>>(100, n, sink);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    cudaEventRecord(a);
    rate_m64<<<148, 128, smem2>>>(iters, n, sink);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    printf("M=64 N=%3d: %.1f TFLOP/s %s\n", n, 2.0 * 64 * n * 32 * double(iters) * 148 / ms / 1e9,
           cudaGetErrorString(cudaGetLastError()));
  }
  return 0;
}
