// Data-parallel gradient exchange fused with the SGD update, over peer memory
// (CUDA IPC mappings of every rank's device arena, gradient arena and signal
// words; NVLink / NVSwitch loads and stores between GPUs).
//
// One exchange = three launches on the compute stream:
//   1. peer_barrier(pre):  every rank's wgrad output is complete and visible;
//   2. peer_reduce_sgd:    this rank owns a 1/N share of the flat gradient
//      index space (chunk list built on the host). For each owned element it
//      sums the N ranks' gradients in rank order 0..N-1 (P2P loads), applies
//      w -= step * sum to its local weight and stores the new weight into
//      EVERY rank's arena at the same offset (P2P stores). That is
//      reduce-scatter + SGD + all-gather in one pass: each rank reads
//      (N-1)/N and writes (N-1)/N of the gradient bytes over NVLink, no
//      separate SGD pass over HBM, and all ranks hold bit-identical weights
//      (one rank computes each element, fixed summation order);
//   3. peer_barrier(post): nobody runs its next forward (reading weights) or
//      its next backward (overwriting its gradients) while a peer is still
//      reading / writing them.
// Barriers are flag words: rank r writes `epoch` into slot [phase][r] of every
// rank's signal array with a system-scope release store and waits until all
// N slots of its own array reach `epoch` (acquire loads). A wait that exceeds
// 120 s traps instead of hanging the device.
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cstdint>

#include "kernels.h"

namespace vdnnk {

namespace {

__device__ __forceinline__ void st_release_sys(unsigned long long* p, unsigned long long v) {
  asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

__device__ __forceinline__ unsigned long long ld_acquire_sys(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}

__device__ __forceinline__ unsigned long long globaltimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}

__global__ void peer_barrier_kernel(PeerArgs a, unsigned long long epoch, int phase) {
  const int p = threadIdx.x;
  if (p >= a.world) return;
  // everything this rank wrote before (earlier kernels on the stream, or the
  // reduce pass's peer stores) is visible system-wide before the flag
  __threadfence_system();
  st_release_sys(a.signal[p] + phase * kPeerMaxRanks + a.rank, epoch);
  const unsigned long long* mine = a.signal[a.rank] + phase * kPeerMaxRanks + p;
  const unsigned long long t0 = globaltimer();
  while (ld_acquire_sys(mine) < epoch) {
    if (globaltimer() - t0 > 120ull * 1000000000ull) __trap();  // a peer never arrived
    __nanosleep(64);
  }
}

// BF16 weights (elem_size 2): the same fp32 reduction in rank order, the
// update computed in fp32 and rounded once (nearest even), 4 weights (8 B)
// per access.
template <int W>
__device__ __forceinline__ void reduce_sgd_bf16(const PeerArgs& a, const PeerChunk& ch) {
  const bool vec = (ch.g_off & 3) == 0 && (ch.w_off & 7) == 0;
  const uint32_t nv = vec ? ch.count / 4 : 0;
  for (uint32_t i = threadIdx.x; i < nv; i += blockDim.x) {
    float4 s = reinterpret_cast<const float4*>(a.grads[0] + ch.g_off)[i];
#pragma unroll
    for (int p = 1; p < W; ++p) {
      const float4 g = reinterpret_cast<const float4*>(a.grads[p] + ch.g_off)[i];
      s.x += g.x;
      s.y += g.y;
      s.z += g.z;
      s.w += g.w;
    }
    const uint2 wb = reinterpret_cast<const uint2*>(a.arena[a.rank] + ch.w_off)[i];
    const float w0 = __uint_as_float(wb.x << 16), w1 = __uint_as_float(wb.x & 0xFFFF0000u);
    const float w2 = __uint_as_float(wb.y << 16), w3 = __uint_as_float(wb.y & 0xFFFF0000u);
    const __nv_bfloat162 lo = __floats2bfloat162_rn(w0 - a.step * s.x, w1 - a.step * s.y);
    const __nv_bfloat162 hi = __floats2bfloat162_rn(w2 - a.step * s.z, w3 - a.step * s.w);
    const uint2 out = make_uint2(*reinterpret_cast<const uint32_t*>(&lo), *reinterpret_cast<const uint32_t*>(&hi));
#pragma unroll
    for (int p = 0; p < W; ++p) reinterpret_cast<uint2*>(a.arena[p] + ch.w_off)[i] = out;
  }
  for (uint32_t i = nv * 4 + threadIdx.x; i < ch.count; i += blockDim.x) {
    float s = a.grads[0][ch.g_off + i];
#pragma unroll
    for (int p = 1; p < W; ++p) s += a.grads[p][ch.g_off + i];
    const __nv_bfloat16 w =
        __float2bfloat16_rn(__bfloat162float(reinterpret_cast<const __nv_bfloat16*>(a.arena[a.rank] + ch.w_off)[i]) -
                            a.step * s);
#pragma unroll
    for (int p = 0; p < W; ++p) reinterpret_cast<__nv_bfloat16*>(a.arena[p] + ch.w_off)[i] = w;
  }
}

template <int W>
__global__ void __launch_bounds__(256) peer_reduce_sgd_kernel(PeerArgs a) {
  for (int c = blockIdx.x; c < a.nchunks; c += gridDim.x) {
    const PeerChunk ch = a.chunks[c];
    if (a.bf16) {
      reduce_sgd_bf16<W>(a, ch);
      continue;
    }
    const bool vec = (ch.g_off & 3) == 0 && (ch.w_off & 15) == 0;  // both 16-B aligned
    const uint32_t nv = vec ? ch.count / 4 : 0;
    for (uint32_t i = threadIdx.x; i < nv; i += blockDim.x) {
      float4 s = reinterpret_cast<const float4*>(a.grads[0] + ch.g_off)[i];
#pragma unroll
      for (int p = 1; p < W; ++p) {
        const float4 g = reinterpret_cast<const float4*>(a.grads[p] + ch.g_off)[i];
        s.x += g.x;
        s.y += g.y;
        s.z += g.z;
        s.w += g.w;
      }
      float4 w = reinterpret_cast<const float4*>(a.arena[a.rank] + ch.w_off)[i];
      w.x -= a.step * s.x;
      w.y -= a.step * s.y;
      w.z -= a.step * s.z;
      w.w -= a.step * s.w;
#pragma unroll
      for (int p = 0; p < W; ++p) reinterpret_cast<float4*>(a.arena[p] + ch.w_off)[i] = w;
    }
    for (uint32_t i = nv * 4 + threadIdx.x; i < ch.count; i += blockDim.x) {
      float s = a.grads[0][ch.g_off + i];
#pragma unroll
      for (int p = 1; p < W; ++p) s += a.grads[p][ch.g_off + i];
      const float w = reinterpret_cast<const float*>(a.arena[a.rank] + ch.w_off)[i] - a.step * s;
#pragma unroll
      for (int p = 0; p < W; ++p) reinterpret_cast<float*>(a.arena[p] + ch.w_off)[i] = w;
    }
  }
}

template <int W>
cudaError_t launch_reduce(const PeerArgs& a, int grid, cudaStream_t st) {
  peer_reduce_sgd_kernel<W><<<grid, 256, 0, st>>>(a);
  return cudaGetLastError();
}

}  // namespace

cudaError_t peer_barrier(const PeerArgs& a, unsigned long long epoch, int phase, cudaStream_t st) {
  if (a.world < 1 || a.world > kPeerMaxRanks || phase < 0 || phase > 1) return cudaErrorInvalidValue;
  peer_barrier_kernel<<<1, 32, 0, st>>>(a, epoch, phase);
  count_launch();
  return cudaGetLastError();
}

cudaError_t peer_reduce_sgd(const PeerArgs& a, cudaStream_t st) {
  if (a.nchunks == 0) return cudaSuccess;
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int grid = a.nchunks < 8 * sms ? a.nchunks : 8 * sms;
  cudaError_t e = cudaErrorInvalidValue;
  switch (a.world) {
    case 1: e = launch_reduce<1>(a, grid, st); break;
    case 2: e = launch_reduce<2>(a, grid, st); break;
    case 3: e = launch_reduce<3>(a, grid, st); break;
    case 4: e = launch_reduce<4>(a, grid, st); break;
    case 5: e = launch_reduce<5>(a, grid, st); break;
    case 6: e = launch_reduce<6>(a, grid, st); break;
    case 7: e = launch_reduce<7>(a, grid, st); break;
    case 8: e = launch_reduce<8>(a, grid, st); break;
    default: break;
  }
  count_launch();
  return e;
}

}  // namespace vdnnk
