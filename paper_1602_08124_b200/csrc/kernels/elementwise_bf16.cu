// Memory-bound kernels over BF16 storage (the reference's elem_size = 2,
// cost_model.hpp:69): the same operations and dataflow contracts as
// elementwise.cu (ReLU in place on the producer's Y, masked by Y > 0; pool
// backward from X and dY with the forward's first-maximum rule; softmax
// gradient produced during LOSS FWD), computed in fp32 and rounded once
// (round-to-nearest-even) where a bf16 value is stored. 16-byte accesses
// (8 bf16) wherever the element count and alignment allow.
#include <cfloat>

#include <cuda_bf16.h>

#include "kernels.h"

namespace vdnnk {

namespace {
using bf16 = __nv_bfloat16;
constexpr int kThreads = 256;
constexpr int kNumSms = 148;

inline int grid_for(size_t n, int per_thread = 1) {
  size_t blocks = (n + static_cast<size_t>(kThreads) * per_thread - 1) / (static_cast<size_t>(kThreads) * per_thread);
  if (blocks < 1) blocks = 1;
  if (blocks > static_cast<size_t>(kNumSms) * 16) blocks = static_cast<size_t>(kNumSms) * 16;
  return static_cast<int>(blocks);
}

__device__ __forceinline__ float f(bf16 v) { return __bfloat162float(v); }
__device__ __forceinline__ bf16 b(float v) { return __float2bfloat16_rn(v); }

struct V8 {
  float v[8];
};
__device__ __forceinline__ V8 ld8(const bf16* p) {
  const uint4 u = *reinterpret_cast<const uint4*>(p);
  const uint32_t w[4] = {u.x, u.y, u.z, u.w};
  V8 r;
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    r.v[2 * i] = __uint_as_float(w[i] << 16);
    r.v[2 * i + 1] = __uint_as_float(w[i] & 0xFFFF0000u);
  }
  return r;
}
__device__ __forceinline__ void st8(bf16* p, const V8& r) {
  uint32_t w[4];
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const __nv_bfloat162 h = __floats2bfloat162_rn(r.v[2 * i], r.v[2 * i + 1]);
    w[i] = *reinterpret_cast<const uint32_t*>(&h);
  }
  *reinterpret_cast<uint4*>(p) = make_uint4(w[0], w[1], w[2], w[3]);
}

bool al16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15) == 0; }

__device__ __forceinline__ uint64_t splitmix64(uint64_t x) {
  x += 0x9E3779B97F4A7C15ull;
  x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
  x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
  return x ^ (x >> 31);
}
__device__ __forceinline__ float u01(uint64_t bits) { return static_cast<float>(bits >> 40) * (1.0f / 16777216.0f); }

struct PtrListB {
  const bf16* p[8];
};
}  // namespace

// ------------------------------------------------------------- ReLU -------
__global__ void relu_fwd_b_kernel(bf16* __restrict__ y, size_t n) {
  const size_t n8 = n / 8;
  for (size_t i = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; i < n8;
       i += static_cast<size_t>(gridDim.x) * blockDim.x) {
    V8 v = ld8(y + 8 * i);
#pragma unroll
    for (int k = 0; k < 8; ++k) v.v[k] = fmaxf(v.v[k], 0.f);
    st8(y + 8 * i, v);
  }
  for (size_t i = n8 * 8 + blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<size_t>(gridDim.x) * blockDim.x)
    y[i] = b(fmaxf(f(y[i]), 0.f));
}

cudaError_t relu_fwd_bf16(void* y, size_t n, cudaStream_t st) {
  if (n == 0) return cudaSuccess;
  if (!al16(y)) return cudaErrorMisalignedAddress;
  relu_fwd_b_kernel<<<grid_for(n, 32), kThreads, 0, st>>>(static_cast<bf16*>(y), n);
  count_launch();
  return cudaGetLastError();
}

// dst = sum src[k] (k < nsrc), masked by (y > 0) when y; dst may alias src[0].
__global__ void combine_b_kernel(bf16* __restrict__ dst, PtrListB src, int nsrc, const bf16* __restrict__ y,
                                 size_t n) {
  const size_t n8 = n / 8;
  for (size_t i = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; i < n8;
       i += static_cast<size_t>(gridDim.x) * blockDim.x) {
    V8 v = ld8(src.p[0] + 8 * i);
    for (int k = 1; k < nsrc; ++k) {
      const V8 e = ld8(src.p[k] + 8 * i);
#pragma unroll
      for (int t = 0; t < 8; ++t) v.v[t] += e.v[t];
    }
    if (y) {
      const V8 a = ld8(y + 8 * i);
#pragma unroll
      for (int t = 0; t < 8; ++t) v.v[t] = a.v[t] > 0.f ? v.v[t] : 0.f;
    }
    st8(dst + 8 * i, v);
  }
  for (size_t i = n8 * 8 + blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<size_t>(gridDim.x) * blockDim.x) {
    float v = f(src.p[0][i]);
    for (int k = 1; k < nsrc; ++k) v += f(src.p[k][i]);
    if (y) v = f(y[i]) > 0.f ? v : 0.f;
    dst[i] = b(v);
  }
}

cudaError_t combine_bf16(void* dst, const void* const* src, int nsrc, const void* y, size_t n, cudaStream_t st) {
  if (n == 0) return cudaSuccess;
  if (nsrc < 1 || nsrc > 8) return cudaErrorInvalidValue;
  PtrListB pl{};
  for (int i = 0; i < nsrc; ++i) {
    if (!al16(src[i])) return cudaErrorMisalignedAddress;
    pl.p[i] = static_cast<const bf16*>(src[i]);
  }
  if (!al16(dst) || (y && !al16(y))) return cudaErrorMisalignedAddress;
  combine_b_kernel<<<grid_for(n, 32), kThreads, 0, st>>>(static_cast<bf16*>(dst), pl, nsrc,
                                                        static_cast<const bf16*>(y), n);
  count_launch();
  return cudaGetLastError();
}

// g0 = (g0 + sum extra) * (y > 0), in place
cudaError_t relu_bwd_bf16(void* g0, const void* const* extra, int nextra, const void* y, size_t n, cudaStream_t st) {
  if (nextra > 7) return cudaErrorInvalidValue;
  const void* src[8] = {g0};
  for (int i = 0; i < nextra; ++i) src[i + 1] = extra[i];
  return combine_bf16(g0, src, nextra + 1, y, n, st);
}

// dst += sum src
cudaError_t add_into_bf16(void* dst, const void* const* src, int nsrc, size_t n, cudaStream_t st) {
  if (n == 0 || nsrc == 0) return cudaSuccess;
  if (nsrc > 7) return cudaErrorInvalidValue;
  const void* all[8] = {dst};
  for (int i = 0; i < nsrc; ++i) all[i + 1] = src[i];
  return combine_bf16(dst, all, nsrc + 1, nullptr, n, st);
}

// Zero-inserted dY of a stride-s conv (elementwise.cu dilate semantics).
__global__ void dilate_b_kernel(bf16* __restrict__ d, const bf16* __restrict__ dy, int n, int ho, int wo, int c,
                                int s, int hd, int wd) {
  const size_t total = static_cast<size_t>(n) * hd * wd * c;
  for (size_t e = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; e < total;
       e += static_cast<size_t>(gridDim.x) * blockDim.x) {
    const int ch = static_cast<int>(e % c);
    size_t r = e / c;
    const int j = static_cast<int>(r % wd);
    r /= wd;
    const int i = static_cast<int>(r % hd);
    const size_t img = r / hd;
    bf16 v = b(0.f);
    if (i % s == 0 && j % s == 0) v = dy[((img * ho + i / s) * wo + j / s) * c + ch];
    d[e] = v;
  }
}

cudaError_t dilate_bf16(void* d, const void* dy, int n, int ho, int wo, int c, int stride, cudaStream_t st) {
  const int hd = (ho - 1) * stride + 1, wd = (wo - 1) * stride + 1;
  const size_t total = static_cast<size_t>(n) * hd * wd * c;
  if (total == 0) return cudaSuccess;
  dilate_b_kernel<<<grid_for(total, 8), kThreads, 0, st>>>(static_cast<bf16*>(d), static_cast<const bf16*>(dy), n,
                                                          ho, wo, c, stride, hd, wd);
  count_launch();
  return cudaGetLastError();
}

// ---------------------------------------------------------- max-pool -----
namespace {
struct PoolDevB {
  int n, h, w, window, stride, ho, wo, nseg, ctot;
  const bf16* x[kMaxConvSegs];
  bf16* dx[kMaxConvSegs];
  int c[kMaxConvSegs];
  int cbase[kMaxConvSegs];
  int mask[kMaxConvSegs];
};

PoolDevB to_dev_b(const PoolArgs& a) {
  PoolDevB d{};
  d.n = a.n;
  d.h = a.h;
  d.w = a.w;
  d.window = a.window;
  d.stride = a.stride;
  d.ho = a.ho();
  d.wo = a.wo();
  d.nseg = a.nseg;
  int cb = 0;
  for (int i = 0; i < a.nseg; ++i) {
    d.x[i] = reinterpret_cast<const bf16*>(a.x[i]);
    d.dx[i] = reinterpret_cast<bf16*>(a.dx[i]);
    d.c[i] = a.c[i];
    d.cbase[i] = cb;
    d.mask[i] = a.mask_in[i];
    cb += a.c[i];
  }
  d.ctot = cb;
  return d;
}

bool vec8(const PoolDevB& d) {
  for (int i = 0; i < d.nseg; ++i)
    if (d.c[i] % 8 != 0) return false;
  return true;
}

__device__ __forceinline__ int pool_seg_b(const PoolDevB& d, int c) {
  int s = 0;
  for (int i = 1; i < d.nseg; ++i)
    if (c >= d.cbase[i]) s = i;
  return s;
}

template <int VEC>
__device__ __forceinline__ void load_vec(const bf16* p, float (&v)[VEC]) {
  if constexpr (VEC == 8) {
    const V8 r = ld8(p);
#pragma unroll
    for (int k = 0; k < 8; ++k) v[k] = r.v[k];
  } else {
    v[0] = f(p[0]);
  }
}
template <int VEC>
__device__ __forceinline__ void store_vec(bf16* p, const float (&v)[VEC]) {
  if constexpr (VEC == 8) {
    V8 r;
#pragma unroll
    for (int k = 0; k < 8; ++k) r.v[k] = v[k];
    st8(p, r);
  } else {
    p[0] = b(v[0]);
  }
}

// window maximum in row-major scan order, strict '>' (first maximum wins)
template <int VEC>
__device__ __forceinline__ void window_max_b(const bf16* x, size_t rowoff0, size_t row_pitch, int C, int window,
                                             float (&m)[VEC]) {
  bool first = true;
  for (int r = 0; r < window; ++r)
    for (int q = 0; q < window; ++q) {
      float v[VEC];
      load_vec<VEC>(x + rowoff0 + r * row_pitch + static_cast<size_t>(q) * C, v);
#pragma unroll
      for (int k = 0; k < VEC; ++k)
        if (first || v[k] > m[k]) m[k] = v[k];
      first = false;
    }
}
}  // namespace

template <int VEC>
__global__ void maxpool_fwd_b_kernel(const __grid_constant__ PoolDevB d, bf16* __restrict__ y) {
  const int cv = d.ctot / VEC;
  const size_t total = static_cast<size_t>(d.n) * d.ho * d.wo * cv;
  for (size_t i = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; i < total;
       i += static_cast<size_t>(gridDim.x) * blockDim.x) {
    const int c = static_cast<int>(i % cv) * VEC;
    size_t t = i / cv;
    const int ow = static_cast<int>(t % d.wo);
    t /= d.wo;
    const int oh = static_cast<int>(t % d.ho);
    const int n = static_cast<int>(t / d.ho);
    const int s = pool_seg_b(d, c);
    const int C = d.c[s];
    float m[VEC];
    window_max_b<VEC>(d.x[s], ((static_cast<size_t>(n) * d.h + oh * d.stride) * d.w + ow * d.stride) * C + (c - d.cbase[s]),
                      static_cast<size_t>(d.w) * C, C, d.window, m);
    store_vec<VEC>(y + ((static_cast<size_t>(n) * d.ho + oh) * d.wo + ow) * d.ctot + c, m);
  }
}

// 2x2 / stride-2 pooling over one segment with no edge gaps (VGG): 32-bit
// index math, the four 16-B window loads issued together, max / scatter from
// registers (the generic kernels decode 64-bit indices and, backward, read
// the window twice).
namespace {
bool pool2x2_fast(const PoolDevB& d) {
  const int64_t outs8 = static_cast<int64_t>(d.n) * d.ho * d.wo * (d.ctot / 8);
  return d.nseg == 1 && d.window == 2 && d.stride == 2 && d.h == 2 * d.ho && d.w == 2 * d.wo && d.c[0] % 8 == 0 &&
         outs8 < (int64_t{1} << 31) && static_cast<int64_t>(d.n) * d.h * d.w * d.c[0] < (int64_t{1} << 40);
}
}  // namespace

__global__ void maxpool2x2_fwd_b_kernel(const bf16* __restrict__ x, bf16* __restrict__ y, uint32_t total,
                                        uint32_t cv, uint32_t wo, int w, int C) {
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < total; i += gridDim.x * blockDim.x) {
    const uint32_t c8 = i % cv, t = i / cv;
    const uint32_t ow = t % wo, nh = t / wo;  // nh = n * ho + oh: input rows 2nh, 2nh + 1
    const size_t pitch = static_cast<size_t>(w) * C;
    const bf16* p = x + (static_cast<size_t>(2 * nh) * w + 2 * ow) * C + c8 * 8;
    const V8 a = ld8(p), b2 = ld8(p + C), c = ld8(p + pitch), e = ld8(p + pitch + C);
    V8 m;
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      float v = a.v[k];
      if (b2.v[k] > v) v = b2.v[k];
      if (c.v[k] > v) v = c.v[k];
      if (e.v[k] > v) v = e.v[k];
      m.v[k] = v;
    }
    st8(y + static_cast<size_t>(i) * 8, m);
  }
}

// first maximum in scan order gets dY (masked by x > 0 for a fused ReLU
// backward), the other three positions 0 -- maxpool_bwd_scatter_b_kernel's rule
__global__ void maxpool2x2_bwd_b_kernel(const bf16* __restrict__ x, const bf16* __restrict__ dy,
                                        bf16* __restrict__ dx, uint32_t total, uint32_t cv, uint32_t wo, int w, int C,
                                        int msk) {
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < total; i += gridDim.x * blockDim.x) {
    const uint32_t c8 = i % cv, t = i / cv;
    const uint32_t ow = t % wo, nh = t / wo;
    const size_t pitch = static_cast<size_t>(w) * C;
    const size_t o = (static_cast<size_t>(2 * nh) * w + 2 * ow) * C + c8 * 8;
    V8 v[4];
    v[0] = ld8(x + o);
    v[1] = ld8(x + o + C);
    v[2] = ld8(x + o + pitch);
    v[3] = ld8(x + o + pitch + C);
    const V8 g = ld8(dy + static_cast<size_t>(i) * 8);
    V8 out[4];
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      float m = v[0].v[k];
#pragma unroll
      for (int j = 1; j < 4; ++j)
        if (v[j].v[k] > m) m = v[j].v[k];
      bool done = false;
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const bool hit = !done && v[j].v[k] == m;
        out[j].v[k] = (hit && (!msk || v[j].v[k] > 0.f)) ? g.v[k] : 0.f;
        done = done || hit;
      }
    }
    st8(dx + o, out[0]);
    st8(dx + o + C, out[1]);
    st8(dx + o + pitch, out[2]);
    st8(dx + o + pitch + C, out[3]);
  }
}

cudaError_t maxpool_fwd_bf16(const PoolArgs& a, void* y, cudaStream_t st) {
  const PoolDevB d = to_dev_b(a);
  const size_t outs = static_cast<size_t>(d.n) * d.ho * d.wo * d.ctot;
  if (outs == 0) return cudaSuccess;
  if (pool2x2_fast(d)) {
    const uint32_t cv = static_cast<uint32_t>(d.ctot / 8), total = static_cast<uint32_t>(outs / 8);
    maxpool2x2_fwd_b_kernel<<<grid_for(total, 2), kThreads, 0, st>>>(d.x[0], static_cast<bf16*>(y), total, cv,
                                                                     static_cast<uint32_t>(d.wo), d.w, d.c[0]);
    count_launch();
    return cudaGetLastError();
  }
  if (vec8(d))
    maxpool_fwd_b_kernel<8><<<grid_for(outs / 8, 2), kThreads, 0, st>>>(d, static_cast<bf16*>(y));
  else
    maxpool_fwd_b_kernel<1><<<grid_for(outs, 4), kThreads, 0, st>>>(d, static_cast<bf16*>(y));
  count_launch();
  return cudaGetLastError();
}

// Non-overlapping windows: one thread per output (x VEC channels) scatters dY
// to the window's first maximum and zeros to the rest of the window.
template <int VEC>
__global__ void maxpool_bwd_scatter_b_kernel(const __grid_constant__ PoolDevB d, const bf16* __restrict__ dy) {
  const int cv = d.ctot / VEC;
  const size_t total = static_cast<size_t>(d.n) * d.ho * d.wo * cv;
  for (size_t i = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; i < total;
       i += static_cast<size_t>(gridDim.x) * blockDim.x) {
    const int c = static_cast<int>(i % cv) * VEC;
    size_t t = i / cv;
    const int ow = static_cast<int>(t % d.wo);
    t /= d.wo;
    const int oh = static_cast<int>(t % d.ho);
    const int n = static_cast<int>(t / d.ho);
    const int s = pool_seg_b(d, c);
    bf16* dx = d.dx[s];
    if (dx == nullptr) continue;
    const int C = d.c[s];
    const size_t base = ((static_cast<size_t>(n) * d.h + oh * d.stride) * d.w + ow * d.stride) * C + (c - d.cbase[s]);
    const size_t pitch = static_cast<size_t>(d.w) * C;
    float ym[VEC], g[VEC];
    bool done[VEC];
    window_max_b<VEC>(d.x[s], base, pitch, C, d.window, ym);
    load_vec<VEC>(dy + ((static_cast<size_t>(n) * d.ho + oh) * d.wo + ow) * d.ctot + c, g);
#pragma unroll
    for (int k = 0; k < VEC; ++k) done[k] = false;
    const bool msk = d.mask[s] != 0;
    for (int r = 0; r < d.window; ++r)
      for (int q = 0; q < d.window; ++q) {
        const size_t off = base + r * pitch + static_cast<size_t>(q) * C;
        float v[VEC], o[VEC];
        load_vec<VEC>(d.x[s] + off, v);
#pragma unroll
        for (int k = 0; k < VEC; ++k) {
          const bool hit = !done[k] && v[k] == ym[k];
          o[k] = (hit && (!msk || v[k] > 0.f)) ? g[k] : 0.f;
          done[k] = done[k] || hit;
        }
        store_vec<VEC>(dx + off, o);
      }
  }
}

// Overlapping windows: gather form (deterministic); every input sums dY over
// the windows whose first-maximum position it is.
template <int VEC>
__global__ void maxpool_bwd_gather_b_kernel(const __grid_constant__ PoolDevB d, const bf16* __restrict__ dy) {
  const int cv = d.ctot / VEC;
  const size_t total = static_cast<size_t>(d.n) * d.h * d.w * cv;
  for (size_t i = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; i < total;
       i += static_cast<size_t>(gridDim.x) * blockDim.x) {
    const int c = static_cast<int>(i % cv) * VEC;
    size_t t = i / cv;
    const int iw = static_cast<int>(t % d.w);
    t /= d.w;
    const int ih = static_cast<int>(t % d.h);
    const int n = static_cast<int>(t / d.h);
    const int s = pool_seg_b(d, c);
    if (d.dx[s] == nullptr) continue;
    const int cl = c - d.cbase[s];
    const bf16* x = d.x[s];
    const int C = d.c[s];
    const size_t pitch = static_cast<size_t>(d.w) * C;
    int oh_lo = ih - d.window + 1;
    oh_lo = oh_lo <= 0 ? 0 : (oh_lo + d.stride - 1) / d.stride;
    const int oh_hi = min(ih / d.stride, d.ho - 1);
    int ow_lo = iw - d.window + 1;
    ow_lo = ow_lo <= 0 ? 0 : (ow_lo + d.stride - 1) / d.stride;
    const int ow_hi = min(iw / d.stride, d.wo - 1);
    float g[VEC];
#pragma unroll
    for (int k = 0; k < VEC; ++k) g[k] = 0.f;
    for (int oh = oh_lo; oh <= oh_hi; ++oh)
      for (int ow = ow_lo; ow <= ow_hi; ++ow) {
        const size_t base = ((static_cast<size_t>(n) * d.h + oh * d.stride) * d.w + ow * d.stride) * C + cl;
        float ym[VEC];
        window_max_b<VEC>(x, base, pitch, C, d.window, ym);
        int arg[VEC];
#pragma unroll
        for (int k = 0; k < VEC; ++k) arg[k] = -1;
        for (int r = 0; r < d.window; ++r)
          for (int q = 0; q < d.window; ++q) {
            float v[VEC];
            load_vec<VEC>(x + base + r * pitch + static_cast<size_t>(q) * C, v);
#pragma unroll
            for (int k = 0; k < VEC; ++k)
              if (arg[k] < 0 && v[k] == ym[k]) arg[k] = r * d.window + q;
          }
        const int here = (ih - oh * d.stride) * d.window + (iw - ow * d.stride);
        float dv[VEC];
        load_vec<VEC>(dy + ((static_cast<size_t>(n) * d.ho + oh) * d.wo + ow) * d.ctot + c, dv);
#pragma unroll
        for (int k = 0; k < VEC; ++k)
          if (arg[k] == here) g[k] += dv[k];
      }
    const size_t xo = ((static_cast<size_t>(n) * d.h + ih) * d.w + iw) * C + cl;
    if (d.mask[s]) {
      float xv[VEC];
      load_vec<VEC>(x + xo, xv);
#pragma unroll
      for (int k = 0; k < VEC; ++k)
        if (!(xv[k] > 0.f)) g[k] = 0.f;
    }
    store_vec<VEC>(d.dx[s] + xo, g);
  }
}

cudaError_t maxpool_bwd_bf16(const PoolArgs& a, const void* dy, cudaStream_t st) {
  const PoolDevB d = to_dev_b(a);
  const size_t total = static_cast<size_t>(d.n) * d.h * d.w * d.ctot;
  if (total == 0) return cudaSuccess;
  const bf16* g = static_cast<const bf16*>(dy);
  const bool v8 = vec8(d);
  if (d.stride >= d.window) {
    const bool gaps = d.stride > d.window || d.ho * d.stride < d.h || d.wo * d.stride < d.w;
    if (gaps)
      for (int i = 0; i < d.nseg; ++i)
        if (d.dx[i]) {
          const cudaError_t e =
              cudaMemsetAsync(d.dx[i], 0, static_cast<size_t>(d.n) * d.h * d.w * d.c[i] * sizeof(bf16), st);
          if (e != cudaSuccess) return e;
        }
    const size_t outs = static_cast<size_t>(d.n) * d.ho * d.wo * d.ctot;
    if (pool2x2_fast(d) && d.dx[0]) {
      const uint32_t cv = static_cast<uint32_t>(d.ctot / 8), total = static_cast<uint32_t>(outs / 8);
      maxpool2x2_bwd_b_kernel<<<grid_for(total, 2), kThreads, 0, st>>>(
          d.x[0], g, d.dx[0], total, cv, static_cast<uint32_t>(d.wo), d.w, d.c[0], d.mask[0]);
      count_launch();
      return cudaGetLastError();
    }
    if (v8)
      maxpool_bwd_scatter_b_kernel<8><<<grid_for(outs / 8, 2), kThreads, 0, st>>>(d, g);
    else
      maxpool_bwd_scatter_b_kernel<1><<<grid_for(outs, 4), kThreads, 0, st>>>(d, g);
  } else if (v8) {
    maxpool_bwd_gather_b_kernel<8><<<grid_for(total / 8, 2), kThreads, 0, st>>>(d, g);
  } else {
    maxpool_bwd_gather_b_kernel<1><<<grid_for(total, 4), kThreads, 0, st>>>(d, g);
  }
  count_launch();
  return cudaGetLastError();
}

// --------------------------------------------------- softmax x-entropy ----
// One warp per row of bf16 logits; gradient (softmax - onehot)/n stored bf16,
// per-row loss fp32, mean over rows by one block (deterministic).
__global__ void softmax_xent_b_kernel(const bf16* __restrict__ logits, const int32_t* __restrict__ labels, int n,
                                      int k, bf16* __restrict__ grad, float* __restrict__ row_loss) {
  const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (warp >= n) return;
  const bf16* z = logits + static_cast<size_t>(warp) * k;
  float m = -FLT_MAX;
  for (int i = lane; i < k; i += 32) m = fmaxf(m, f(z[i]));
  for (int o = 16; o > 0; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
  float s = 0.f;
  for (int i = lane; i < k; i += 32) s += expf(f(z[i]) - m);
  for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  const float lse = m + logf(s);
  const int lab = labels[warp] % k;
  const float inv_n = 1.0f / static_cast<float>(n);
  for (int i = lane; i < k; i += 32) {
    const float pr = expf(f(z[i]) - lse);
    grad[static_cast<size_t>(warp) * k + i] = b((pr - (i == lab ? 1.f : 0.f)) * inv_n);
  }
  if (lane == 0) row_loss[warp] = lse - f(z[lab]);
}

__global__ void mean_b_kernel(const float* __restrict__ v, int n, float* __restrict__ out, int accumulate) {
  __shared__ float part[256];
  float s = 0.f;
  for (int i = threadIdx.x; i < n; i += blockDim.x) s += v[i];
  part[threadIdx.x] = s;
  __syncthreads();
  for (int w = blockDim.x / 2; w > 0; w >>= 1) {
    if (threadIdx.x < w) part[threadIdx.x] += part[threadIdx.x + w];
    __syncthreads();
  }
  if (threadIdx.x == 0) *out = (accumulate ? *out : 0.f) + part[0] / static_cast<float>(n);
}

cudaError_t softmax_xent_fwd_bf16(const void* logits, const int32_t* labels, int n, int k, void* grad_scratch,
                                  float* row_loss, float* loss, cudaStream_t st, bool accumulate) {
  if (n <= 0) return cudaSuccess;
  softmax_xent_b_kernel<<<(n * 32 + 255) / 256, 256, 0, st>>>(static_cast<const bf16*>(logits), labels, n, k,
                                                               static_cast<bf16*>(grad_scratch), row_loss);
  mean_b_kernel<<<1, 256, 0, st>>>(row_loss, n, loss, accumulate ? 1 : 0);
  count_launch(2);
  return cudaGetLastError();
}

// ------------------------------------------------------- bias / SGD -------
// bias -= lr * sum_n dy[n][o] (bf16 bias) or db[o] = sum (fp32)
__global__ void bias_grad_b_kernel(const bf16* __restrict__ dy, int n, int o, bf16* __restrict__ bias, float lr,
                                   float* __restrict__ db) {
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= o) return;
  float s = 0.f;
  for (int i = 0; i < n; ++i) s += f(dy[static_cast<size_t>(i) * o + j]);
  if (db)
    db[j] = s;
  else
    bias[j] = b(f(bias[j]) - lr * s);
}

cudaError_t bias_grad_bf16(const void* dy, int n, int o, void* bias, float lr, float* db_out, cudaStream_t st) {
  if (o <= 0) return cudaSuccess;
  bias_grad_b_kernel<<<(o + 255) / 256, 256, 0, st>>>(static_cast<const bf16*>(dy), n, o, static_cast<bf16*>(bias),
                                                       lr, db_out);
  count_launch();
  return cudaGetLastError();
}

// w (bf16) -= lr * g (fp32 gradient arena)
__global__ void sgd_b_kernel(bf16* __restrict__ w, const float* __restrict__ g, float lr, size_t n) {
  for (size_t i = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<size_t>(gridDim.x) * blockDim.x)
    w[i] = b(f(w[i]) - lr * g[i]);
}

cudaError_t sgd_update_bf16(void* w, const float* g, float lr, size_t n, cudaStream_t st) {
  if (n == 0) return cudaSuccess;
  sgd_b_kernel<<<grid_for(n, 8), kThreads, 0, st>>>(static_cast<bf16*>(w), g, lr, n);
  count_launch();
  return cudaGetLastError();
}

// ---------------------------------------------------------- fills ---------
// Same generators as the fp32 fills (elementwise.cu), rounded to bf16.
__global__ void fill_normal_b_kernel(bf16* __restrict__ w, size_t n, float stddev, uint64_t seed) {
  for (size_t i = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<size_t>(gridDim.x) * blockDim.x) {
    const uint64_t a = splitmix64(seed * 0x100000001B3ull + 2 * i);
    const uint64_t c = splitmix64(seed * 0x100000001B3ull + 2 * i + 1);
    const float u1 = 1.0f - u01(a);
    const float u2 = u01(c);
    w[i] = b(stddev * sqrtf(-2.0f * logf(u1)) * cospif(2.0f * u2));
  }
}

cudaError_t fill_normal_bf16(void* w, size_t n, float stddev, uint64_t seed, cudaStream_t st) {
  if (n == 0) return cudaSuccess;
  fill_normal_b_kernel<<<grid_for(n, 8), kThreads, 0, st>>>(static_cast<bf16*>(w), n, stddev, seed);
  count_launch();
  return cudaGetLastError();
}

__global__ void fill_uniform_b_kernel(bf16* __restrict__ x, size_t n, float lo, float hi, uint64_t seed) {
  for (size_t i = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<size_t>(gridDim.x) * blockDim.x)
    x[i] = b(lo + (hi - lo) * u01(splitmix64(seed * 0x9E3779B97F4A7C15ull + i)));
}

cudaError_t fill_uniform_bf16(void* x, size_t n, float lo, float hi, uint64_t seed, cudaStream_t st) {
  if (n == 0) return cudaSuccess;
  fill_uniform_b_kernel<<<grid_for(n, 8), kThreads, 0, st>>>(static_cast<bf16*>(x), n, lo, hi, seed);
  count_launch();
  return cudaGetLastError();
}

__global__ void fill_const_b_kernel(bf16* __restrict__ x, size_t n, float v) {
  for (size_t i = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<size_t>(gridDim.x) * blockDim.x)
    x[i] = b(v);
}

cudaError_t fill_const_bf16(void* x, size_t n, float v, cudaStream_t st) {
  if (n == 0) return cudaSuccess;
  fill_const_b_kernel<<<grid_for(n, 8), kThreads, 0, st>>>(static_cast<bf16*>(x), n, v);
  count_launch();
  return cudaGetLastError();
}

// Channel padding of a [rows][c] bf16 tensor to [rows][cp] (zeros in c..cp)
// and back, for layers whose channel count is not a multiple of 8 (the first
// layer's C = 3): the padded copy feeds the TMA producers.
__global__ void pad_channels_b_kernel(bf16* __restrict__ dst, const bf16* __restrict__ src, size_t rows, int c,
                                      int cp) {
  const size_t total = rows * cp;
  for (size_t e = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; e < total;
       e += static_cast<size_t>(gridDim.x) * blockDim.x) {
    const size_t r = e / cp;
    const int ch = static_cast<int>(e - r * cp);
    dst[e] = ch < c ? src[r * c + ch] : b(0.f);
  }
}
__global__ void unpad_channels_b_kernel(bf16* __restrict__ dst, const bf16* __restrict__ src, size_t rows, int c,
                                        int cp) {
  const size_t total = rows * c;
  for (size_t e = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; e < total;
       e += static_cast<size_t>(gridDim.x) * blockDim.x) {
    const size_t r = e / c;
    dst[e] = src[r * cp + (e - r * c)];
  }
}
__global__ void unpad_channels_f_kernel(float* __restrict__ dst, const float* __restrict__ src, size_t rows, int c,
                                        int cp) {
  const size_t total = rows * c;
  for (size_t e = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; e < total;
       e += static_cast<size_t>(gridDim.x) * blockDim.x) {
    const size_t r = e / c;
    dst[e] = src[r * cp + (e - r * c)];
  }
}

cudaError_t pad_channels_bf16(void* dst, const void* src, size_t rows, int c, int cp, cudaStream_t st) {
  if (rows == 0) return cudaSuccess;
  pad_channels_b_kernel<<<grid_for(rows * cp, 8), kThreads, 0, st>>>(static_cast<bf16*>(dst),
                                                                     static_cast<const bf16*>(src), rows, c, cp);
  count_launch();
  return cudaGetLastError();
}
cudaError_t unpad_channels_bf16(void* dst, const void* src, size_t rows, int c, int cp, cudaStream_t st) {
  if (rows == 0) return cudaSuccess;
  unpad_channels_b_kernel<<<grid_for(rows * c, 8), kThreads, 0, st>>>(static_cast<bf16*>(dst),
                                                                      static_cast<const bf16*>(src), rows, c, cp);
  count_launch();
  return cudaGetLastError();
}
cudaError_t unpad_channels_f32(float* dst, const float* src, size_t rows, int c, int cp, cudaStream_t st) {
  if (rows == 0) return cudaSuccess;
  unpad_channels_f_kernel<<<grid_for(rows * c, 8), kThreads, 0, st>>>(dst, src, rows, c, cp);
  count_launch();
  return cudaGetLastError();
}

// fp32 <-> bf16 (host-format conversions on the device: weight upload /
// readback, feature probes)
__global__ void to_bf16_kernel(bf16* __restrict__ d, const float* __restrict__ s, size_t n) {
  for (size_t i = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<size_t>(gridDim.x) * blockDim.x)
    d[i] = b(s[i]);
}
__global__ void from_bf16_kernel(float* __restrict__ d, const bf16* __restrict__ s, size_t n) {
  for (size_t i = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<size_t>(gridDim.x) * blockDim.x)
    d[i] = f(s[i]);
}

cudaError_t f32_to_bf16(void* dst, const float* src, size_t n, cudaStream_t st) {
  if (n == 0) return cudaSuccess;
  to_bf16_kernel<<<grid_for(n, 8), kThreads, 0, st>>>(static_cast<bf16*>(dst), src, n);
  count_launch();
  return cudaGetLastError();
}
cudaError_t bf16_to_f32(float* dst, const void* src, size_t n, cudaStream_t st) {
  if (n == 0) return cudaSuccess;
  from_bf16_kernel<<<grid_for(n, 8), kThreads, 0, st>>>(dst, static_cast<const bf16*>(src), n);
  count_launch();
  return cudaGetLastError();
}

}  // namespace vdnnk
