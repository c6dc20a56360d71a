// Zero-copy PCIe bandwidth of SM-driven loads/stores to pinned mapped host
// memory (the transport a compressed offload would use), vs cudaMemcpyAsync.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 tools/zc_bw.cu -o /tmp/zc_bw
#include <cstdio>
#include <cuda_runtime.h>

__global__ void zc_write(float4* __restrict__ dst, const float4* __restrict__ src, size_t n) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x)
    dst[i] = src[i];
}
__global__ void zc_read(float4* __restrict__ dst, const float4* __restrict__ src, size_t n) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x)
    dst[i] = src[i];
}
// each thread keeps 8 independent 16-B loads in flight
__global__ void zc_read8(float4* __restrict__ dst, const float4* __restrict__ src, size_t n) {
  const size_t stride = (size_t)gridDim.x * blockDim.x;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += 8 * stride) {
    float4 v[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) v[k] = (i + k * stride < n) ? src[i + k * stride] : make_float4(0, 0, 0, 0);
#pragma unroll
    for (int k = 0; k < 8; ++k)
      if (i + k * stride < n) dst[i + k * stride] = v[k];
  }
}

int main() {
  const size_t bytes = 1ull << 30, n = bytes / 16;
  float4 *h, *hd, *d;
  cudaHostAlloc(&h, bytes, cudaHostAllocMapped);
  cudaHostGetDevicePointer(&hd, h, 0);
  cudaMalloc(&d, bytes);
  cudaMemset(d, 1, bytes);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  float ms;
  cudaMemcpy(h, d, bytes, cudaMemcpyDeviceToHost);
  cudaEventRecord(a);
  cudaMemcpyAsync(h, d, bytes, cudaMemcpyDeviceToHost);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  cudaEventElapsedTime(&ms, a, b);
  printf("memcpy D2H %.1f GB/s\n", bytes / ms / 1e6);
  cudaEventRecord(a);
  cudaMemcpyAsync(d, h, bytes, cudaMemcpyHostToDevice);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  cudaEventElapsedTime(&ms, a, b);
  printf("memcpy H2D %.1f GB/s\n", bytes / ms / 1e6);
  for (int grid : {16, 32, 64, 148, 296, 592}) {
    for (int kind = 0; kind < 3; ++kind) {
      auto run = [&] {
        if (kind == 0) zc_write<<<grid, 256>>>(hd, d, n);
        else if (kind == 1) zc_read<<<grid, 256>>>(d, hd, n);
        else zc_read8<<<grid, 256>>>(d, hd, n);
      };
      run();
      cudaEventRecord(a);
      run();
      cudaEventRecord(b);
      cudaEventSynchronize(b);
      cudaEventElapsedTime(&ms, a, b);
      printf("grid %4d %-6s %.1f GB/s %s\n", grid, kind == 0 ? "write" : kind == 1 ? "read" : "read8", bytes / ms / 1e6,
             cudaGetErrorString(cudaGetLastError()));
    }
  }
  return 0;
}
