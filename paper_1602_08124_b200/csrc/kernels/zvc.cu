// Zero-value-compressed offload / prefetch (optional session mode).
//
// vDNN's offload set on ReLU networks is mostly ReLU outputs, about half of
// whose values are exactly +0.0, and the vDNN_dyn iteration is bound by the
// host link (2 x 10.6 GB per VGG-16 b256 iteration). These
// kernels move a feature map between its pool extent and its pinned host slot
// *through the SMs* (zero-copy stores / loads over PCIe, which this part
// drives at ~50 GB/s vs ~56 GB/s for the copy engines) in a lossless
// zero-value-compressed form, so only the nonzero values cross the link. The
// schedule, pool offsets and every byte of the restored buffer are unchanged:
// the round trip is bit-exact (a value is "zero" only if its bit pattern is
// 0x00000000; -0.0, NaN and denormals are kept as values).
//
// Format (per 1024-float chunk c, at byte c * kZvcSlot of the host slot):
//   u32 mask[32]   lane l's 32 bits: bit 4j+e <-> float 4*(32j + l) + e of the chunk
//   f32 vals[nnz]  lane-major (lane 0's nonzeros in (j, e) order, then lane 1's ...)
// Only 128 + 4*nnz bytes of a slot are written / read; dense chunks cost
// +3% (the mask), all-zero chunks 128 B.
#include <cstdlib>

#include "kernels.h"

namespace vdnnk {

namespace {

constexpr int kWarps = 8;

__device__ __forceinline__ uint32_t warp_excl_scan(uint32_t v, uint32_t& total) {
  const int lane = threadIdx.x & 31;
  uint32_t x = v;
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
    const uint32_t y = __shfl_up_sync(0xffffffffu, x, d);
    if (lane >= d) x += y;
  }
  total = __shfl_sync(0xffffffffu, x, 31);
  return x - v;
}

__global__ void __launch_bounds__(kWarps * 32) zvc_compress_kernel(const float4* __restrict__ src, int64_t n4,
                                                                   uint8_t* __restrict__ dst,
                                                                   unsigned long long* __restrict__ wire) {
  __shared__ __align__(16) float stage[kWarps][kZvcChunk + 4];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t nchunks = (n4 + kZvcChunk / 4 - 1) / (kZvcChunk / 4);
  unsigned long long bytes = 0;
  float* st = stage[warp];
  for (int64_t c = blockIdx.x * static_cast<int64_t>(kWarps) + warp; c < nchunks;
       c += static_cast<int64_t>(gridDim.x) * kWarps) {
    const int64_t b4 = c * (kZvcChunk / 4);
    float4 v[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      const int64_t i = b4 + j * 32 + lane;
      v[j] = i < n4 ? __ldcs(src + i) : make_float4(0.f, 0.f, 0.f, 0.f);
    }
    uint32_t mask = 0;
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      mask |= (__float_as_uint(v[j].x) != 0u ? 1u : 0u) << (4 * j);
      mask |= (__float_as_uint(v[j].y) != 0u ? 1u : 0u) << (4 * j + 1);
      mask |= (__float_as_uint(v[j].z) != 0u ? 1u : 0u) << (4 * j + 2);
      mask |= (__float_as_uint(v[j].w) != 0u ? 1u : 0u) << (4 * j + 3);
    }
    uint32_t total;
    uint32_t k = warp_excl_scan(__popc(mask), total);
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      if (__float_as_uint(v[j].x) != 0u) st[k++] = v[j].x;
      if (__float_as_uint(v[j].y) != 0u) st[k++] = v[j].y;
      if (__float_as_uint(v[j].z) != 0u) st[k++] = v[j].z;
      if (__float_as_uint(v[j].w) != 0u) st[k++] = v[j].w;
    }
    __syncwarp();
    uint8_t* out = dst + c * kZvcSlot;
    reinterpret_cast<uint32_t*>(out)[lane] = mask;
    const int nf4 = static_cast<int>((total + 3) / 4);
    const float4* st4 = reinterpret_cast<const float4*>(st);
    float4* o4 = reinterpret_cast<float4*>(out + 128);
    for (int i = lane; i < nf4; i += 32) o4[i] = st4[i];
    __syncwarp();
    bytes += 128 + 4ull * total;
  }
  if (lane == 0 && bytes) atomicAdd(wire, bytes);
}

__global__ void __launch_bounds__(kWarps * 32) zvc_decompress_kernel(const uint8_t* __restrict__ srcb, int64_t n4,
                                                                     float4* __restrict__ dst,
                                                                     unsigned long long* __restrict__ wire) {
  __shared__ __align__(16) float stage[kWarps][kZvcChunk + 4];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t nchunks = (n4 + kZvcChunk / 4 - 1) / (kZvcChunk / 4);
  unsigned long long bytes = 0;
  float* st = stage[warp];
  for (int64_t c = blockIdx.x * static_cast<int64_t>(kWarps) + warp; c < nchunks;
       c += static_cast<int64_t>(gridDim.x) * kWarps) {
    const uint8_t* in = srcb + c * kZvcSlot;
    const uint32_t mask = __ldcs(reinterpret_cast<const unsigned int*>(in) + lane);
    uint32_t total;
    uint32_t k = warp_excl_scan(__popc(mask), total);
    const int nf4 = static_cast<int>((total + 3) / 4);
    const float4* i4 = reinterpret_cast<const float4*>(in + 128);
    float4* st4 = reinterpret_cast<float4*>(st);
    for (int i = lane; i < nf4; i += 32) st4[i] = __ldcs(i4 + i);
    __syncwarp();
    const int64_t b4 = c * (kZvcChunk / 4);
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      float4 v;
      v.x = (mask >> (4 * j)) & 1u ? st[k++] : 0.f;
      v.y = (mask >> (4 * j + 1)) & 1u ? st[k++] : 0.f;
      v.z = (mask >> (4 * j + 2)) & 1u ? st[k++] : 0.f;
      v.w = (mask >> (4 * j + 3)) & 1u ? st[k++] : 0.f;
      const int64_t i = b4 + j * 32 + lane;
      if (i < n4) dst[i] = v;
    }
    __syncwarp();
    bytes += 128 + 4ull * total;
  }
  if (lane == 0 && bytes && wire) atomicAdd(wire, bytes);
}

// Enough resident warps to keep ~50 GB/s of PCIe requests in flight, few
// enough (and light enough: 33 KB smem, 256 threads) to co-reside with the
// conv kernels on the compute stream.
int zvc_max_grid() {
  static const int g = [] {
    const char* e = std::getenv("VDNN_ZVC_GRID");
    return e ? std::atoi(e) : 32;
  }();
  return g;
}
int zvc_grid(int64_t nchunks) {
  const int64_t want = (nchunks + kWarps - 1) / kWarps;
  const int cap = zvc_max_grid();
  return static_cast<int>(want < cap ? (want < 1 ? 1 : want) : cap);
}

}  // namespace

uint64_t zvc_slot_bytes(uint64_t bytes) {
  const uint64_t n = bytes / 4;
  return ((n + kZvcChunk - 1) / kZvcChunk) * kZvcSlot;
}

bool zvc_eligible(const void* p, uint64_t bytes) {
  return bytes > 0 && bytes % 16 == 0 && (reinterpret_cast<uintptr_t>(p) & 15u) == 0;
}

cudaError_t zvc_compress(const float* src, uint64_t count, void* dst, unsigned long long* wire, cudaStream_t st) {
  if (count == 0) return cudaSuccess;
  if (count % 4 != 0) return cudaErrorInvalidValue;
  const int64_t n4 = static_cast<int64_t>(count / 4);
  const int64_t nchunks = (n4 + kZvcChunk / 4 - 1) / (kZvcChunk / 4);
  zvc_compress_kernel<<<zvc_grid(nchunks), kWarps * 32, 0, st>>>(reinterpret_cast<const float4*>(src), n4,
                                                                  static_cast<uint8_t*>(dst), wire);
  count_launch();
  return cudaGetLastError();
}

cudaError_t zvc_decompress(const void* src, uint64_t count, float* dst, unsigned long long* wire, cudaStream_t st) {
  if (count == 0) return cudaSuccess;
  if (count % 4 != 0) return cudaErrorInvalidValue;
  const int64_t n4 = static_cast<int64_t>(count / 4);
  const int64_t nchunks = (n4 + kZvcChunk / 4 - 1) / (kZvcChunk / 4);
  zvc_decompress_kernel<<<zvc_grid(nchunks), kWarps * 32, 0, st>>>(static_cast<const uint8_t*>(src), n4,
                                                                    reinterpret_cast<float4*>(dst), wire);
  count_launch();
  return cudaGetLastError();
}

}  // namespace vdnnk
