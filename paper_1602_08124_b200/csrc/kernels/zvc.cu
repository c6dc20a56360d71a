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
//   u32 hdr[4]     hdr[0] = mode, hdr[1] = base top byte
//   mode 0: f32 vals[nnz]  lane-major (lane 0's nonzeros in (j, e) order, then lane 1's ...)
//   mode 1: the same nonzeros split into their low 3 bytes (u8 lo[3*nnz], padded to 16 B) and
//           their top byte (sign + 7 exponent bits) as a 4-bit offset from hdr[1] (u8 nib[(nnz+1)/2],
//           two per byte, padded to 16 B) -- chosen when a chunk's top bytes span <= 15, which
//           holds for every chunk of the VGG-16 offload set measured (tools/zvc_stats.py):
//           3.5 B per nonzero instead of 4, wire 0.44 -> 0.39 of the raw bytes.
//   mode 2 (TF32-exact transfers, only when the caller asks for it): each nonzero as one u16 =
//           (4-bit top-byte offset << 11) | the next 11 bits (exponent LSB + the 10 TF32 mantissa
//           bits). The low 13 mantissa bits are dropped: the tcgen05 kind::tf32 MMA ignores them
//           (measured: tools/tf32_trunc_probe.py -- fprop and wgrad outputs on X and on X with those
//           bits cleared are bit-identical), so for a map whose only backward readers are TF32
//           contractions and ReLU masks the training step is bit-identical. A chunk falls back to
//           mode 1 / 0 if a nonzero would truncate to +-0 (a denormal: the ReLU mask x > 0 must
//           survive) or is Inf/NaN. 2 B per nonzero instead of 3.5.
// Only the header and the padded payload cross the link; a dense chunk costs
// +3.5% (mask + header), an all-zero chunk 144 B.
#include <cstdlib>

#include "kernels.h"

namespace vdnnk {

namespace {

constexpr int kWarps = 8;
constexpr int kHdr = 16;

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

__device__ __forceinline__ uint32_t pad16(uint32_t b) { return (b + 15u) & ~15u; }

// copy `bytes` (multiple of 16) from shared to the (host-mapped) slot with 16-B stores
__device__ __forceinline__ void warp_copy_out(const float* st, uint8_t* out, uint32_t bytes, int lane) {
  const float4* s4 = reinterpret_cast<const float4*>(st);
  float4* o4 = reinterpret_cast<float4*>(out);
  for (uint32_t i = lane; i < bytes / 16; i += 32) o4[i] = s4[i];
}

__global__ void __launch_bounds__(kWarps * 32) zvc_compress_kernel(const float4* __restrict__ src, int64_t n4,
                                                                   uint8_t* __restrict__ dst,
                                                                   unsigned long long* __restrict__ wire, int tf32) {
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
    uint32_t mask = 0, tmin = 255, tmax = 0;
    bool inexact = false;  // a nonzero that TF32 truncation would not represent (denormal -> 0, Inf/NaN)
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      const uint32_t q[4] = {__float_as_uint(v[j].x), __float_as_uint(v[j].y), __float_as_uint(v[j].z),
                             __float_as_uint(v[j].w)};
#pragma unroll
      for (int e = 0; e < 4; ++e)
        if (q[e] != 0u) {
          mask |= 1u << (4 * j + e);
          tmin = min(tmin, q[e] >> 24);
          tmax = max(tmax, q[e] >> 24);
          inexact |= ((q[e] & 0x7FFFE000u) == 0u) || ((q[e] & 0x7F800000u) == 0x7F800000u);
        }
    }
    inexact = __any_sync(0xffffffffu, inexact);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      tmin = min(tmin, __shfl_xor_sync(0xffffffffu, tmin, o));
      tmax = max(tmax, __shfl_xor_sync(0xffffffffu, tmax, o));
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
    const bool narrow = total > 0 && tmax - tmin <= 15u;
    const uint32_t mode = narrow ? ((tf32 && !inexact) ? 2u : 1u) : 0u;
    if (lane == 0)
      *reinterpret_cast<uint4*>(out + 128) = make_uint4(mode, tmin, total, 0u);
    uint32_t payload;
    if (mode == 0) {
      payload = pad16(4 * total);
      warp_copy_out(st, out + 128 + kHdr, payload, lane);
    } else if (mode == 2) {
      // values into registers first, then the u16 codes in place
      uint32_t w[32];
#pragma unroll
      for (int i = 0; i < 32; ++i) {
        const uint32_t k2 = lane + 32u * i;
        w[i] = k2 < total ? __float_as_uint(st[k2]) : 0u;
      }
      __syncwarp();
      uint16_t* pk = reinterpret_cast<uint16_t*>(st);
#pragma unroll
      for (int i = 0; i < 32; ++i) {
        const uint32_t k2 = lane + 32u * i;
        if (k2 < total) pk[k2] = static_cast<uint16_t>((((w[i] >> 24) - tmin) << 11) | ((w[i] >> 13) & 0x7FFu));
      }
      __syncwarp();
      payload = pad16(2 * total);
      warp_copy_out(st, out + 128 + kHdr, payload, lane);
    } else {
      // pack in place: each lane reads its value pairs (2p, 2p+1) into
      // registers first, then writes their 6 low bytes and one nibble byte
      const uint32_t npairs = (total + 1) / 2;
      uint32_t w[32];
#pragma unroll
      for (int i = 0; i < 16; ++i) {
        const uint32_t pr = lane + 32u * i;
        w[2 * i] = pr < npairs ? __float_as_uint(st[2 * pr]) : 0u;
        w[2 * i + 1] = (pr < npairs && 2 * pr + 1 < total) ? __float_as_uint(st[2 * pr + 1]) : 0u;
      }
      __syncwarp();
      uint8_t* pk = reinterpret_cast<uint8_t*>(st);
      const uint32_t off3 = pad16(3 * total);
#pragma unroll
      for (int i = 0; i < 16; ++i) {
        const uint32_t pr = lane + 32u * i;
        if (pr >= npairs) continue;
        const uint32_t a = w[2 * i], b = w[2 * i + 1];
        uint8_t* d = pk + 6 * pr;
        d[0] = a & 0xff;
        d[1] = (a >> 8) & 0xff;
        d[2] = (a >> 16) & 0xff;
        if (2 * pr + 1 < total) {
          d[3] = b & 0xff;
          d[4] = (b >> 8) & 0xff;
          d[5] = (b >> 16) & 0xff;
        }
        const uint32_t hi = (2 * pr + 1 < total) ? ((b >> 24) - tmin) : 0u;
        pk[off3 + pr] = static_cast<uint8_t>(((a >> 24) - tmin) | (hi << 4));
      }
      __syncwarp();
      payload = off3 + pad16(npairs);
      warp_copy_out(st, out + 128 + kHdr, payload, lane);
    }
    __syncwarp();
    bytes += 128 + kHdr + payload;
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
    const uint4 hdr = __ldcs(reinterpret_cast<const uint4*>(in + 128));
    uint32_t total;
    uint32_t k = warp_excl_scan(__popc(mask), total);
    const uint32_t payload = hdr.x == 0   ? pad16(4 * total)
                             : hdr.x == 2 ? pad16(2 * total)
                                          : pad16(3 * total) + pad16((total + 1) / 2);
    {
      const float4* i4 = reinterpret_cast<const float4*>(in + 128 + kHdr);
      float4* st4 = reinterpret_cast<float4*>(st);
      for (uint32_t i = lane; i < payload / 16; i += 32) st4[i] = __ldcs(i4 + i);
    }
    __syncwarp();
    if (hdr.x == 2) {  // u16 codes -> TF32-exact floats in place (codes into registers first)
      const uint16_t* pk = reinterpret_cast<const uint16_t*>(st);
      uint32_t w[32];
#pragma unroll
      for (int i = 0; i < 32; ++i) {
        const uint32_t k2 = lane + 32u * i;
        w[i] = k2 < total ? pk[k2] : 0u;
      }
      __syncwarp();
#pragma unroll
      for (int i = 0; i < 32; ++i) {
        const uint32_t k2 = lane + 32u * i;
        if (k2 < total) st[k2] = __uint_as_float((((w[i] >> 11) + hdr.y) << 24) | ((w[i] & 0x7FFu) << 13));
      }
      __syncwarp();
    } else if (hdr.x == 1) {  // unpack to floats in place (read every pair into registers first)
      const uint8_t* pk = reinterpret_cast<const uint8_t*>(st);
      const uint32_t off3 = pad16(3 * total), npairs = (total + 1) / 2;
      uint32_t w[32];
#pragma unroll
      for (int i = 0; i < 16; ++i) {
        const uint32_t pr = lane + 32u * i;
        if (pr >= npairs) continue;
        const uint8_t* d = pk + 6 * pr;
        const uint32_t nb = pk[off3 + pr];
        w[2 * i] = (static_cast<uint32_t>(d[0]) | (static_cast<uint32_t>(d[1]) << 8) |
                    (static_cast<uint32_t>(d[2]) << 16)) | (((nb & 15u) + hdr.y) << 24);
        w[2 * i + 1] = (static_cast<uint32_t>(d[3]) | (static_cast<uint32_t>(d[4]) << 8) |
                        (static_cast<uint32_t>(d[5]) << 16)) | (((nb >> 4) + hdr.y) << 24);
      }
      __syncwarp();
#pragma unroll
      for (int i = 0; i < 16; ++i) {
        const uint32_t pr = lane + 32u * i;
        if (pr >= npairs) continue;
        st[2 * pr] = __uint_as_float(w[2 * i]);
        if (2 * pr + 1 < total) st[2 * pr + 1] = __uint_as_float(w[2 * i + 1]);
      }
      __syncwarp();
    }
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
    bytes += 128 + kHdr + payload;
  }
  if (lane == 0 && bytes && wire) atomicAdd(wire, bytes);
}

// ---------------------------------------------------------------- BF16 ----
// Per 2048-bf16 chunk c, at byte c * kZvcbSlot of the host slot:
//   u32 mask[64]   lane l's words 2l (bits of its uint4 groups j = 0..3) and
//                  2l + 1 (j = 4..7): bit 8(j & 3) + e <-> bf16 8*(32j + l) + e
//   u32 hdr[4]     hdr[0] = mode, hdr[1] = top byte base, hdr[2] = nonzeros
//   mode 0: u16 vals[nnz] lane-major (lane 0's nonzeros in (j, e) order, ...)
//   mode 1: u8 lo[nnz] (the low byte: exponent LSB + 7 mantissa bits), padded
//           to 16 B, then u8 nib[(nnz+1)/2]: the top byte (sign + 7 exponent
//           bits) as a 4-bit offset from hdr[1], two per byte -- when a
//           chunk's top bytes span <= 15 (ReLU maps: positive, a few octaves).
// A value is "zero" only as the bit pattern 0x0000 (-0.0, NaN, denormals kept).
__global__ void __launch_bounds__(kWarps * 32) zvcb_compress_kernel(const uint4* __restrict__ src, int64_t n8,
                                                                    uint8_t* __restrict__ dst,
                                                                    unsigned long long* __restrict__ wire) {
  __shared__ __align__(16) uint16_t stage[kWarps][kZvcbChunk + 16];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t nchunks = (n8 + kZvcbChunk / 8 - 1) / (kZvcbChunk / 8);
  unsigned long long bytes = 0;
  uint16_t* st = stage[warp];
  for (int64_t c = blockIdx.x * static_cast<int64_t>(kWarps) + warp; c < nchunks;
       c += static_cast<int64_t>(gridDim.x) * kWarps) {
    const int64_t b8 = c * (kZvcbChunk / 8);
    uint4 v[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      const int64_t i = b8 + j * 32 + lane;
      v[j] = i < n8 ? __ldcs(src + i) : make_uint4(0u, 0u, 0u, 0u);
    }
    uint32_t m[2] = {0u, 0u}, tmin = 255, tmax = 0;
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      const uint32_t w[4] = {v[j].x, v[j].y, v[j].z, v[j].w};
#pragma unroll
      for (int e = 0; e < 8; ++e) {
        const uint32_t h = (w[e >> 1] >> (16 * (e & 1))) & 0xFFFFu;
        if (h != 0u) {
          m[j >> 2] |= 1u << (8 * (j & 3) + e);
          tmin = min(tmin, h >> 8);
          tmax = max(tmax, h >> 8);
        }
      }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      tmin = min(tmin, __shfl_xor_sync(0xffffffffu, tmin, o));
      tmax = max(tmax, __shfl_xor_sync(0xffffffffu, tmax, o));
    }
    uint32_t total;
    uint32_t k = warp_excl_scan(__popc(m[0]) + __popc(m[1]), total);
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      const uint32_t w[4] = {v[j].x, v[j].y, v[j].z, v[j].w};
#pragma unroll
      for (int e = 0; e < 8; ++e) {
        const uint32_t h = (w[e >> 1] >> (16 * (e & 1))) & 0xFFFFu;
        if (h != 0u) st[k++] = static_cast<uint16_t>(h);
      }
    }
    __syncwarp();
    uint8_t* out = dst + c * kZvcbSlot;
    reinterpret_cast<uint2*>(out)[lane] = make_uint2(m[0], m[1]);
    const uint32_t mode = (total > 0 && tmax - tmin <= 15u) ? 1u : 0u;
    if (lane == 0) *reinterpret_cast<uint4*>(out + 256) = make_uint4(mode, tmin, total, 0u);
    uint32_t payload;
    if (mode == 0) {
      payload = pad16(2 * total);
    } else {
      // pack in place: every lane reads its values (pairs p = lane + 32i)
      // into registers first, then writes the low bytes and nibble bytes
      const uint32_t npairs = (total + 1) / 2;
      uint32_t w[32];
#pragma unroll
      for (int i = 0; i < 32; ++i) {
        const uint32_t pr = lane + 32u * i;
        w[i] = pr < npairs ? (static_cast<uint32_t>(st[2 * pr]) |
                              (2 * pr + 1 < total ? static_cast<uint32_t>(st[2 * pr + 1]) << 16 : 0u))
                           : 0u;
      }
      __syncwarp();
      uint8_t* pk = reinterpret_cast<uint8_t*>(st);
      const uint32_t off1 = pad16(total);
#pragma unroll
      for (int i = 0; i < 32; ++i) {
        const uint32_t pr = lane + 32u * i;
        if (pr >= npairs) continue;
        const uint32_t a = w[i] & 0xFFFFu, b = w[i] >> 16;
        pk[2 * pr] = static_cast<uint8_t>(a & 0xFFu);
        if (2 * pr + 1 < total) pk[2 * pr + 1] = static_cast<uint8_t>(b & 0xFFu);
        const uint32_t hi = (2 * pr + 1 < total) ? ((b >> 8) - tmin) : 0u;
        pk[off1 + pr] = static_cast<uint8_t>(((a >> 8) - tmin) | (hi << 4));
      }
      __syncwarp();
      payload = off1 + pad16(npairs);
    }
    warp_copy_out(reinterpret_cast<const float*>(st), out + 256 + kHdr, payload, lane);
    __syncwarp();
    bytes += 256 + kHdr + payload;
  }
  if (lane == 0 && bytes) atomicAdd(wire, bytes);
}

__global__ void __launch_bounds__(kWarps * 32) zvcb_decompress_kernel(const uint8_t* __restrict__ srcb, int64_t n8,
                                                                      uint4* __restrict__ dst,
                                                                      unsigned long long* __restrict__ wire) {
  __shared__ __align__(16) uint16_t stage[kWarps][kZvcbChunk + 16];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t nchunks = (n8 + kZvcbChunk / 8 - 1) / (kZvcbChunk / 8);
  unsigned long long bytes = 0;
  uint16_t* st = stage[warp];
  for (int64_t c = blockIdx.x * static_cast<int64_t>(kWarps) + warp; c < nchunks;
       c += static_cast<int64_t>(gridDim.x) * kWarps) {
    const uint8_t* in = srcb + c * kZvcbSlot;
    const uint2 mm = __ldcs(reinterpret_cast<const uint2*>(in) + lane);
    const uint4 hdr = __ldcs(reinterpret_cast<const uint4*>(in + 256));
    const uint32_t m[2] = {mm.x, mm.y};
    uint32_t total;
    uint32_t k = warp_excl_scan(__popc(m[0]) + __popc(m[1]), total);
    const uint32_t payload = hdr.x == 0 ? pad16(2 * total) : pad16(total) + pad16((total + 1) / 2);
    {
      const uint4* i4 = reinterpret_cast<const uint4*>(in + 256 + kHdr);
      uint4* st4 = reinterpret_cast<uint4*>(st);
      for (uint32_t i = lane; i < payload / 16; i += 32) st4[i] = __ldcs(i4 + i);
    }
    __syncwarp();
    if (hdr.x == 1) {  // unpack to u16 in place (read every pair into registers first)
      const uint8_t* pk = reinterpret_cast<const uint8_t*>(st);
      const uint32_t off1 = pad16(total), npairs = (total + 1) / 2;
      uint32_t w[32];
#pragma unroll
      for (int i = 0; i < 32; ++i) {
        const uint32_t pr = lane + 32u * i;
        if (pr >= npairs) continue;
        const uint32_t nb = pk[off1 + pr];
        const uint32_t a = static_cast<uint32_t>(pk[2 * pr]) | (((nb & 15u) + hdr.y) << 8);
        const uint32_t b = (2 * pr + 1 < total) ? (static_cast<uint32_t>(pk[2 * pr + 1]) | (((nb >> 4) + hdr.y) << 8))
                                                : 0u;
        w[i] = a | (b << 16);
      }
      __syncwarp();
#pragma unroll
      for (int i = 0; i < 32; ++i) {
        const uint32_t pr = lane + 32u * i;
        if (pr >= npairs) continue;
        st[2 * pr] = static_cast<uint16_t>(w[i] & 0xFFFFu);
        if (2 * pr + 1 < total) st[2 * pr + 1] = static_cast<uint16_t>(w[i] >> 16);
      }
      __syncwarp();
    }
    const int64_t b8 = c * (kZvcbChunk / 8);
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      uint32_t w[4] = {0u, 0u, 0u, 0u};
#pragma unroll
      for (int e = 0; e < 8; ++e)
        if ((m[j >> 2] >> (8 * (j & 3) + e)) & 1u) w[e >> 1] |= static_cast<uint32_t>(st[k++]) << (16 * (e & 1));
      const int64_t i = b8 + j * 32 + lane;
      if (i < n8) dst[i] = make_uint4(w[0], w[1], w[2], w[3]);
    }
    __syncwarp();
    bytes += 256 + kHdr + payload;
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

uint64_t zvc_slot_bytes_bf16(uint64_t bytes) {
  const uint64_t n = bytes / 2;
  return ((n + kZvcbChunk - 1) / kZvcbChunk) * kZvcbSlot;
}

cudaError_t zvc_compress_bf16(const void* src, uint64_t count, void* dst, unsigned long long* wire,
                              cudaStream_t st) {
  if (count == 0) return cudaSuccess;
  if (count % 8 != 0) return cudaErrorInvalidValue;
  const int64_t n8 = static_cast<int64_t>(count / 8);
  const int64_t nchunks = (n8 + kZvcbChunk / 8 - 1) / (kZvcbChunk / 8);
  zvcb_compress_kernel<<<zvc_grid(nchunks), kWarps * 32, 0, st>>>(static_cast<const uint4*>(src), n8,
                                                                   static_cast<uint8_t*>(dst), wire);
  count_launch();
  return cudaGetLastError();
}

cudaError_t zvc_decompress_bf16(const void* src, uint64_t count, void* dst, unsigned long long* wire,
                                cudaStream_t st) {
  if (count == 0) return cudaSuccess;
  if (count % 8 != 0) return cudaErrorInvalidValue;
  const int64_t n8 = static_cast<int64_t>(count / 8);
  const int64_t nchunks = (n8 + kZvcbChunk / 8 - 1) / (kZvcbChunk / 8);
  zvcb_decompress_kernel<<<zvc_grid(nchunks), kWarps * 32, 0, st>>>(static_cast<const uint8_t*>(src), n8,
                                                                     static_cast<uint4*>(dst), wire);
  count_launch();
  return cudaGetLastError();
}

uint64_t zvc_slot_bytes(uint64_t bytes) {
  const uint64_t n = bytes / 4;
  return ((n + kZvcChunk - 1) / kZvcChunk) * kZvcSlot;
}

bool zvc_eligible(const void* p, uint64_t bytes) {
  return bytes > 0 && bytes % 16 == 0 && (reinterpret_cast<uintptr_t>(p) & 15u) == 0;
}

cudaError_t zvc_compress(const float* src, uint64_t count, void* dst, unsigned long long* wire, cudaStream_t st,
                         bool tf32) {
  if (count == 0) return cudaSuccess;
  if (count % 4 != 0) return cudaErrorInvalidValue;
  const int64_t n4 = static_cast<int64_t>(count / 4);
  const int64_t nchunks = (n4 + kZvcChunk / 4 - 1) / (kZvcChunk / 4);
  zvc_compress_kernel<<<zvc_grid(nchunks), kWarps * 32, 0, st>>>(reinterpret_cast<const float4*>(src), n4,
                                                                  static_cast<uint8_t*>(dst), wire, tf32 ? 1 : 0);
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
