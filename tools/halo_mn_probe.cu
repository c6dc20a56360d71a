// Probe (tool): MN-major (SWIZZLE_128B_BASE32B) A operand whose 32-wide M
// chunks are the SAME staged rows shifted by one 128-B row each (LBO = 128):
// A[(s, ci)][k] = X[k + s][ci]. That is the layout a halo-reuse WGRAD needs
// (the kw taps of one filter row read one staged block of input pixels).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++20 -I paper_1602_08124_b200/csrc/kernels \
//        tools/halo_mn_probe.cu -o tools/halo_mn_probe
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "tc_conv.cuh"
using namespace vdnnk;

constexpr int R = 40;   // staged pixel rows (32 K rows + shifts up to 3, padded to a 1024-B multiple)
constexpr int NB = 32;  // output channels (N)

__global__ void __launch_bounds__(128, 1) probe(const float* X, const float* B, float* D, int lbo) {
  extern __shared__ uint8_t smem_raw[];
  const uint32_t base = (smem_u32(smem_raw) + 1023u) & ~1023u;
  const uint32_t sa = base, sb = base + 8192, tslot = sb + 4096, bar = tslot + 16;
  for (int e = threadIdx.x; e < R * 8; e += blockDim.x) {
    const int r = e / 8, j = e % 8;
    const float* src = X + r * 32 + j * 4;
    asm volatile("st.shared.v4.f32 [%0], {%1,%2,%3,%4};" ::"r"(mnmaj_addr(sa, r, 0, j)), "f"(src[0]), "f"(src[1]),
                 "f"(src[2]), "f"(src[3]));
  }
  for (int e = threadIdx.x; e < 32 * 8; e += blockDim.x) {
    const int k = e / 8, j = e % 8;
    const float* src = B + k * 32 + j * 4;
    asm volatile("st.shared.v4.f32 [%0], {%1,%2,%3,%4};" ::"r"(mnmaj_addr(sb, k, 0, j)), "f"(src[0]), "f"(src[1]),
                 "f"(src[2]), "f"(src[3]));
  }
  fence_proxy_async();
  if (threadIdx.x == 0) {
    mbar_init(bar, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (threadIdx.x < 32) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(tslot), "r"(32)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  uint32_t tmem;
  asm volatile("ld.shared.u32 %0, [%1];" : "=r"(tmem) : "r"(tslot) : "memory");
  if (threadIdx.x == 0) {
    const uint32_t idesc = make_idesc_tf32(NB, true, true);
    for (int kk = 0; kk < 4; ++kk)
      tc_mma_tf32(tmem, make_sdesc(sa + kk * 1024, lbo, 512, kSw128Base32),
                  make_sdesc(sb + kk * 1024, 4096, 512, kSw128Base32), idesc, kk > 0 ? 1u : 0u);
    tc_commit(bar);
    mbar_wait(bar, 0);
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const int w = threadIdx.x / 32;
  float v[32];
  tmem_ld32(tmem + ((w * 32) << 16), v);
  const int row = w * 32 + (threadIdx.x & 31);
  for (int j = 0; j < 32; ++j) D[row * NB + j] = v[j];
  tc_fence_before();
  __syncthreads();
  if (threadIdx.x < 32)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(32) : "memory");
}

int main() {
  std::vector<float> X(R * 32), B(32 * 32), D(128 * NB);
  srand(5);
  for (auto& v : X) v = float(rand() % 17 - 8) / 8.f;
  for (auto& v : B) v = float(rand() % 17 - 8) / 8.f;
  float *dX, *dB, *dD;
  cudaMalloc(&dX, X.size() * 4);
  cudaMalloc(&dB, B.size() * 4);
  cudaMalloc(&dD, D.size() * 4);
  cudaMemcpy(dX, X.data(), X.size() * 4, cudaMemcpyHostToDevice);
  cudaMemcpy(dB, B.data(), B.size() * 4, cudaMemcpyHostToDevice);
  const int smem = 8192 + 4096 + 64 + 1024;
  cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  for (int lbo : {128, 4096}) {
    cudaMemset(dD, 0, D.size() * 4);
    probe<<<1, 128, smem>>>(dX, dB, dD, lbo);
    cudaError_t e = cudaDeviceSynchronize();
    cudaMemcpy(D.data(), dD, D.size() * 4, cudaMemcpyDeviceToHost);
    int bad = 0;
    for (int m = 0; m < 128; ++m) {
      const int s = m / 32, ci = m % 32;
      for (int n = 0; n < NB; ++n) {
        float ref = 0;
        for (int k = 0; k < 32; ++k) {
          // lbo = 128: chunk s = rows shifted by s; lbo = 4096: chunk s at +4096 B = rows 32s.. (reference layout)
          const int row = lbo == 128 ? k + s : k + 32 * s;
          ref += (row < R ? X[row * 32 + ci] : 0.f) * B[k * 32 + n];
        }
        if (lbo == 4096 && s > 0) continue;  // rows beyond the staged block: not checked
        if (D[m * NB + n] != ref) ++bad;
      }
    }
    printf("LBO %4d: %s, %d mismatches\n", lbo, cudaGetErrorString(e), bad);
  }
  return 0;
}
