// Zero-copy PCIe bandwidth with bulk async copies (cp.async.bulk, the
// non-tensor TMA path) between shared memory and pinned mapped host memory,
// vs per-thread 16-B stores/loads: can the compressed transfers go faster
// than the ~50 GB/s of SM stores?
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 tools/zc_bulk.cu -o tools/zc_bulk
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

// each CTA: loop over 16 KB chunks; fill smem (from device memory), bulk-store to host
template <int CHUNK>
__global__ void bulk_store(char* __restrict__ host, const char* __restrict__ src, size_t nchunks) {
  extern __shared__ __align__(128) char sm[];
  const uint32_t s0 = smem_u32(sm);
  int buf = 0;
  for (size_t c = blockIdx.x; c < nchunks; c += gridDim.x, buf ^= 1) {
    // make sure the bulk store that read this buffer two iterations ago is done
    if (threadIdx.x == 0) asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
    __syncthreads();
    const float4* s4 = reinterpret_cast<const float4*>(src + c * CHUNK);
    float4* d4 = reinterpret_cast<float4*>(sm + buf * CHUNK);
    for (int i = threadIdx.x; i < CHUNK / 16; i += blockDim.x) d4[i] = s4[i];
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    __syncthreads();
    if (threadIdx.x == 0) {
      asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(host + c * CHUNK),
                   "r"(s0 + buf * CHUNK), "r"(CHUNK)
                   : "memory");
      asm volatile("cp.async.bulk.commit_group;" ::: "memory");
    }
  }
  if (threadIdx.x == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

__global__ void st_store(float4* __restrict__ dst, const float4* __restrict__ src, size_t n) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x)
    dst[i] = src[i];
}

// bulk loads host -> smem completing on an mbarrier, then smem -> device memory
template <int CHUNK>
__global__ void bulk_load(char* __restrict__ dst, const char* __restrict__ host, size_t nchunks) {
  extern __shared__ __align__(128) char sm[];
  __shared__ __align__(8) uint64_t bar;
  const uint32_t s0 = smem_u32(sm), b = smem_u32(&bar);
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(b));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  uint32_t phase = 0;
  for (size_t c = blockIdx.x; c < nchunks; c += gridDim.x) {
    if (threadIdx.x == 0) {
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(b), "r"(CHUNK) : "memory");
      asm volatile(
          "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(s0),
          "l"(host + c * CHUNK), "r"(CHUNK), "r"(b)
          : "memory");
    }
    asm volatile(
        "{\n .reg .pred p;\n W: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n @!p bra W;\n}\n" ::"r"(b),
        "r"(phase)
        : "memory");
    phase ^= 1;
    const float4* s4 = reinterpret_cast<const float4*>(sm);
    float4* d4 = reinterpret_cast<float4*>(dst + c * CHUNK);
    for (int i = threadIdx.x; i < CHUNK / 16; i += blockDim.x) d4[i] = s4[i];
    __syncthreads();
  }
}

int main() {
  const size_t bytes = 1ull << 30;
  char *h, *hd, *d;
  cudaHostAlloc(&h, bytes, cudaHostAllocMapped);
  cudaHostGetDevicePointer(&hd, h, 0);
  cudaMalloc(&d, bytes);
  cudaMemset(d, 1, bytes);
  cudaEvent_t a, e;
  cudaEventCreate(&a);
  cudaEventCreate(&e);
  float ms;
  constexpr int CH = 16384;
  cudaFuncSetAttribute(bulk_store<CH>, cudaFuncAttributeMaxDynamicSharedMemorySize, 2 * CH);
  for (int grid : {16, 32, 64, 148}) {
    for (int rep = 0; rep < 2; ++rep) {
      cudaEventRecord(a);
      bulk_store<CH><<<grid, 256, 2 * CH>>>(hd, d, bytes / CH);
      cudaEventRecord(e);
      cudaEventSynchronize(e);
      cudaEventElapsedTime(&ms, a, e);
    }
    printf("bulk store   grid %3d: %6.1f GB/s (%s)\n", grid, bytes / ms / 1e6, cudaGetErrorString(cudaGetLastError()));
    for (int rep = 0; rep < 2; ++rep) {
      cudaEventRecord(a);
      st_store<<<grid, 256>>>(reinterpret_cast<float4*>(hd), reinterpret_cast<const float4*>(d), bytes / 16);
      cudaEventRecord(e);
      cudaEventSynchronize(e);
      cudaEventElapsedTime(&ms, a, e);
    }
    printf("16-B stores  grid %3d: %6.1f GB/s\n", grid, bytes / ms / 1e6);
    for (int rep = 0; rep < 2; ++rep) {
      cudaEventRecord(a);
      bulk_load<CH><<<grid, 256, CH>>>(d, hd, bytes / CH);
      cudaEventRecord(e);
      cudaEventSynchronize(e);
      cudaEventElapsedTime(&ms, a, e);
    }
    printf("bulk load    grid %3d: %6.1f GB/s (%s)\n", grid, bytes / ms / 1e6, cudaGetErrorString(cudaGetLastError()));
  }
  for (int rep = 0; rep < 2; ++rep) {
    cudaEventRecord(a);
    cudaMemcpyAsync(h, d, bytes, cudaMemcpyDeviceToHost);
    cudaEventRecord(e);
    cudaEventSynchronize(e);
    cudaEventElapsedTime(&ms, a, e);
  }
  printf("copy engine D2H: %6.1f GB/s\n", bytes / ms / 1e6);
  return 0;
}
