// Memory-bound kernels: in-place ReLU fwd/bwd, gradient folding, max-pool
// fwd/bwd (floor mode, no padding), softmax cross-entropy, bias gradient,
// SGD, and deterministic synthetic-data fills.
//
// Dataflow contracts (reference file:line):
//  * ACTV is in place on the producer's Y and its BWD is in place on the
//    gradient buffer, masked by Y > 0 (net_graph.hpp:384-389,
//    simulator.hpp:102-104, footprint.hpp:62).
//  * POOL BWD reads X and its own Y (simulator.hpp:97-100); pooling is floor
//    mode with no padding (net_graph.hpp:325-334).
//  * LOSS reads nothing in BWD (simulator.hpp:105-107); the softmax gradient
//    is produced during LOSS FWD into a non-pool scratch.
#include <cfloat>

#include "kernels.h"

namespace vdnnk {

namespace {
constexpr int kThreads = 256;
constexpr int kNumSms = 148;

inline int grid_for(size_t n, int per_thread = 1) {
  size_t blocks = (n + static_cast<size_t>(kThreads) * per_thread - 1) / (static_cast<size_t>(kThreads) * per_thread);
  if (blocks < 1) blocks = 1;
  if (blocks > static_cast<size_t>(kNumSms) * 16) blocks = static_cast<size_t>(kNumSms) * 16;
  return static_cast<int>(blocks);
}

__device__ __forceinline__ uint64_t splitmix64(uint64_t x) {
  x += 0x9E3779B97F4A7C15ull;
  x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
  x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
  return x ^ (x >> 31);
}
__device__ __forceinline__ float u01(uint64_t bits) {  // [0, 1)
  return static_cast<float>(bits >> 40) * (1.0f / 16777216.0f);
}
}  // namespace

// ------------------------------------------------------------- ReLU -------
__global__ void relu_fwd_kernel(float* __restrict__ y, size_t n) {
  const size_t n4 = n / 4;
  float4* y4 = reinterpret_cast<float4*>(y);
  for (size_t i = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; i < n4;
       i += static_cast<size_t>(gridDim.x) * blockDim.x) {
    float4 v = y4[i];
    v.x = fmaxf(v.x, 0.f);
    v.y = fmaxf(v.y, 0.f);
    v.z = fmaxf(v.z, 0.f);
    v.w = fmaxf(v.w, 0.f);
    y4[i] = v;
  }
  for (size_t i = n4 * 4 + blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<size_t>(gridDim.x) * blockDim.x)
    y[i] = fmaxf(y[i], 0.f);
}

cudaError_t relu_fwd(float* y, size_t n, cudaStream_t st) {
  if (n == 0) return cudaSuccess;
  relu_fwd_kernel<<<grid_for(n, 16), kThreads, 0, st>>>(y, n);
  count_launch();
  return cudaGetLastError();
}

struct PtrList {
  const float* p[8];
};

__global__ void relu_bwd_kernel(float* __restrict__ g, PtrList extra, int nextra, const float* __restrict__ y,
                                size_t n) {
  const size_t n4 = n / 4;
  for (size_t i = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; i < n4;
       i += static_cast<size_t>(gridDim.x) * blockDim.x) {
    float4 v = reinterpret_cast<float4*>(g)[i];
    for (int k = 0; k < nextra; ++k) {
      const float4 e = reinterpret_cast<const float4*>(extra.p[k])[i];
      v.x += e.x;
      v.y += e.y;
      v.z += e.z;
      v.w += e.w;
    }
    const float4 a = reinterpret_cast<const float4*>(y)[i];
    v.x = a.x > 0.f ? v.x : 0.f;
    v.y = a.y > 0.f ? v.y : 0.f;
    v.z = a.z > 0.f ? v.z : 0.f;
    v.w = a.w > 0.f ? v.w : 0.f;
    reinterpret_cast<float4*>(g)[i] = v;
  }
  for (size_t i = n4 * 4 + blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<size_t>(gridDim.x) * blockDim.x) {
    float v = g[i];
    for (int k = 0; k < nextra; ++k) v += extra.p[k][i];
    g[i] = y[i] > 0.f ? v : 0.f;
  }
}

cudaError_t relu_bwd(float* g0, const float* const* extra, int nextra, const float* y, size_t n, cudaStream_t st) {
  if (n == 0) return cudaSuccess;
  if (nextra > 8) return cudaErrorInvalidValue;
  PtrList pl{};
  for (int i = 0; i < nextra; ++i) pl.p[i] = extra[i];
  relu_bwd_kernel<<<grid_for(n, 16), kThreads, 0, st>>>(g0, pl, nextra, y, n);
  count_launch();
  return cudaGetLastError();
}

__global__ void add_into_kernel(float* __restrict__ dst, PtrList src, int nsrc, size_t n) {
  for (size_t i = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<size_t>(gridDim.x) * blockDim.x) {
    float v = dst[i];
    for (int k = 0; k < nsrc; ++k) v += src.p[k][i];
    dst[i] = v;
  }
}

cudaError_t add_into(float* dst, const float* const* src, int nsrc, size_t n, cudaStream_t st) {
  if (n == 0 || nsrc == 0) return cudaSuccess;
  if (nsrc > 8) return cudaErrorInvalidValue;
  PtrList pl{};
  for (int i = 0; i < nsrc; ++i) pl.p[i] = src[i];
  add_into_kernel<<<grid_for(n, 4), kThreads, 0, st>>>(dst, pl, nsrc, n);
  count_launch();
  return cudaGetLastError();
}

// dst = sum_k src[k], masked by (y > 0) when y != null; dst may be src[0]
// (element-wise in place). Used for shared gradient planes (an elementwise
// join's one map is read-only: its readers sum / mask into their own
// buffer) and for the summed input of an elementwise join.
__global__ void combine_kernel(float* __restrict__ dst, PtrList src, int nsrc, const float* __restrict__ y, size_t n) {
  const size_t n4 = n / 4;
  for (size_t i = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; i < n4;
       i += static_cast<size_t>(gridDim.x) * blockDim.x) {
    float4 v = reinterpret_cast<const float4*>(src.p[0])[i];
    for (int k = 1; k < nsrc; ++k) {
      const float4 e = reinterpret_cast<const float4*>(src.p[k])[i];
      v.x += e.x;
      v.y += e.y;
      v.z += e.z;
      v.w += e.w;
    }
    if (y) {
      const float4 a = reinterpret_cast<const float4*>(y)[i];
      v.x = a.x > 0.f ? v.x : 0.f;
      v.y = a.y > 0.f ? v.y : 0.f;
      v.z = a.z > 0.f ? v.z : 0.f;
      v.w = a.w > 0.f ? v.w : 0.f;
    }
    reinterpret_cast<float4*>(dst)[i] = v;
  }
  for (size_t i = n4 * 4 + blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<size_t>(gridDim.x) * blockDim.x) {
    float v = src.p[0][i];
    for (int k = 1; k < nsrc; ++k) v += src.p[k][i];
    if (y) v = y[i] > 0.f ? v : 0.f;
    dst[i] = v;
  }
}

cudaError_t combine(float* dst, const float* const* src, int nsrc, const float* y, size_t n, cudaStream_t st) {
  if (n == 0) return cudaSuccess;
  if (nsrc < 1 || nsrc > 8) return cudaErrorInvalidValue;
  for (int i = 0; i < nsrc; ++i)
    if (reinterpret_cast<uintptr_t>(src[i]) % 16) return cudaErrorMisalignedAddress;
  if (reinterpret_cast<uintptr_t>(dst) % 16 || (y && reinterpret_cast<uintptr_t>(y) % 16))
    return cudaErrorMisalignedAddress;
  PtrList pl{};
  for (int i = 0; i < nsrc; ++i) pl.p[i] = src[i];
  combine_kernel<<<grid_for(n, 16), kThreads, 0, st>>>(dst, pl, nsrc, y, n);
  count_launch();
  return cudaGetLastError();
}

// Zero insertion for the data gradient of a strided conv: d[n][i][j][c] =
// dy[n][i/s][j/s][c] where s divides i and j, else 0, over (hd, wd) =
// ((ho-1)s+1, (wo-1)s+1); a stride-1 dgrad over d with the conv's own pad
// and kernel then equals the strided conv's dgrad.
__global__ void dilate_kernel(float* __restrict__ d, const float* __restrict__ dy, int n, int ho, int wo, int c,
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
    float v = 0.f;
    if (i % s == 0 && j % s == 0) v = dy[((img * ho + i / s) * wo + j / s) * c + ch];
    d[e] = v;
  }
}

cudaError_t dilate(float* d, const float* dy, int n, int ho, int wo, int c, int stride, cudaStream_t st) {
  const int hd = (ho - 1) * stride + 1, wd = (wo - 1) * stride + 1;
  const size_t total = static_cast<size_t>(n) * hd * wd * c;
  if (total == 0) return cudaSuccess;
  dilate_kernel<<<grid_for(total, 4), kThreads, 0, st>>>(d, dy, n, ho, wo, c, stride, hd, wd);
  count_launch();
  return cudaGetLastError();
}

// ---------------------------------------------------------- max-pool -----
struct PoolDev {
  int n, h, w, window, stride, ho, wo, nseg, ctot;
  const float* x[kMaxConvSegs];
  float* dx[kMaxConvSegs];
  int c[kMaxConvSegs];
  int cbase[kMaxConvSegs];
  int mask[kMaxConvSegs];  // fused ReLU backward: zero where x <= 0
};

static PoolDev to_dev(const PoolArgs& a) {
  PoolDev d{};
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
    d.x[i] = a.x[i];
    d.dx[i] = a.dx[i];
    d.c[i] = a.c[i];
    d.cbase[i] = cb;
    d.mask[i] = a.mask_in[i];
    cb += a.c[i];
  }
  d.ctot = cb;
  return d;
}

__device__ __forceinline__ int pool_seg(const PoolDev& d, int c) {
  int s = 0;
  for (int i = 1; i < d.nseg; ++i)
    if (c >= d.cbase[i]) s = i;
  return s;
}

// Y[n][oh][ow][c] = max over the window (row-major scan, first max wins).
// Vectorised over 4 channels when every segment's C % 4 == 0 (VEC=4).
template <int VEC>
__global__ void maxpool_fwd_kernel(const __grid_constant__ PoolDev d, float* __restrict__ y) {
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
    const int s = pool_seg(d, c);
    const int cl = c - d.cbase[s];
    const float* x = d.x[s];
    const int C = d.c[s];
    float m[VEC];
    bool first = true;
    for (int r = 0; r < d.window; ++r) {
      const float* row = x + ((static_cast<size_t>(n) * d.h + oh * d.stride + r) * d.w + ow * d.stride) * C + cl;
      for (int q = 0; q < d.window; ++q) {
        float v[VEC];
        if constexpr (VEC == 4) {
          const float4 f = *reinterpret_cast<const float4*>(row + static_cast<size_t>(q) * C);
          v[0] = f.x; v[1] = f.y; v[2] = f.z; v[3] = f.w;
        } else {
          v[0] = row[static_cast<size_t>(q) * C];
        }
#pragma unroll
        for (int k = 0; k < VEC; ++k)
          if (first || v[k] > m[k]) m[k] = v[k];
        first = false;
      }
    }
    float* out = y + (((static_cast<size_t>(n) * d.ho + oh) * d.wo + ow) * d.ctot + c);
    if constexpr (VEC == 4)
      *reinterpret_cast<float4*>(out) = make_float4(m[0], m[1], m[2], m[3]);
    else
      out[0] = m[0];
  }
}

// 2x2 / stride-2 windows over one NHWC tensor (every VGG pool): one output
// row per blockIdx.y, 4 channels per thread, the four window loads issued
// before any compare (the generic loop serialises them), 32-bit index math.
// Same scan order and strict '>' as the generic kernel: bit-identical output.
__global__ void __launch_bounds__(256) maxpool2x2_fwd_kernel(const float* __restrict__ x, float* __restrict__ y, int h,
                                                            int w, int c, int ho, int wo) {
  const int cv = c >> 2;
  const int row = blockIdx.y;  // n * ho + oh
  const int n = row / ho, oh = row - n * ho;
  const float4* x0 = reinterpret_cast<const float4*>(x + (static_cast<size_t>(n) * h + 2 * oh) * w * c);
  const float4* x1 = x0 + static_cast<size_t>(w) * cv;
  float4* yr = reinterpret_cast<float4*>(y + static_cast<size_t>(row) * wo * c);
  const int per_row = wo * cv;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < per_row; i += gridDim.x * blockDim.x) {
    const int ow = i / cv, c4 = i - ow * cv;
    const int off = 2 * ow * cv + c4;
    const float4 a = __ldcs(x0 + off), b = __ldcs(x0 + off + cv), e = __ldcs(x1 + off), f = __ldcs(x1 + off + cv);
    float4 m = a;
    m.x = b.x > m.x ? b.x : m.x;
    m.y = b.y > m.y ? b.y : m.y;
    m.z = b.z > m.z ? b.z : m.z;
    m.w = b.w > m.w ? b.w : m.w;
    m.x = e.x > m.x ? e.x : m.x;
    m.y = e.y > m.y ? e.y : m.y;
    m.z = e.z > m.z ? e.z : m.z;
    m.w = e.w > m.w ? e.w : m.w;
    m.x = f.x > m.x ? f.x : m.x;
    m.y = f.y > m.y ? f.y : m.y;
    m.z = f.z > m.z ? f.z : m.z;
    m.w = f.w > m.w ? f.w : m.w;
    yr[i] = m;
  }
}

static bool pool_vec4(const PoolDev& d) {
  for (int i = 0; i < d.nseg; ++i)
    if (d.c[i] % 4 != 0) return false;
  return true;
}

cudaError_t maxpool_fwd(const PoolArgs& a, float* y, cudaStream_t st) {
  const PoolDev d = to_dev(a);
  const size_t total = static_cast<size_t>(d.n) * d.ho * d.wo * d.ctot;
  if (total == 0) return cudaSuccess;
  if (d.nseg == 1 && d.window == 2 && d.stride == 2 && d.c[0] % 4 == 0 &&
      static_cast<int64_t>(d.n) * d.ho <= 65535) {
    const int per_row = d.wo * d.c[0] / 4;
    const dim3 grid(static_cast<unsigned>((per_row + 255) / 256), static_cast<unsigned>(d.n * d.ho));
    maxpool2x2_fwd_kernel<<<grid, 256, 0, st>>>(d.x[0], y, d.h, d.w, d.c[0], d.ho, d.wo);
    count_launch();
    return cudaGetLastError();
  }
  if (pool_vec4(d))
    maxpool_fwd_kernel<4><<<grid_for(total / 4, 2), kThreads, 0, st>>>(d, y);
  else
    maxpool_fwd_kernel<1><<<grid_for(total, 4), kThreads, 0, st>>>(d, y);
  count_launch();
  return cudaGetLastError();
}

// The backward kernels do not read Y: each recomputes its window's maximum
// from X with the forward's rule (row-major scan, strict '>'), which gives
// Y's exact value, and routes dY to the first position equal to it -- the
// same position as comparing with the stored Y (a NaN maximum matches
// nothing either way). Saves the Y read, and a pool output whose other
// backward readers are TF32 contractions may travel TF32-exact (zvc.cu).
template <int VEC>
__device__ __forceinline__ void window_max(const float* x, size_t rowoff0, size_t row_pitch, int C, int window,
                                           float (&m)[VEC]) {
  bool first = true;
  for (int r = 0; r < window; ++r) {
    const size_t rowoff = rowoff0 + static_cast<size_t>(r) * row_pitch;
    for (int q = 0; q < window; ++q) {
      float v[VEC];
      if constexpr (VEC == 4) {
        const float4 f = *reinterpret_cast<const float4*>(x + rowoff + static_cast<size_t>(q) * C);
        v[0] = f.x; v[1] = f.y; v[2] = f.z; v[3] = f.w;
      } else {
        v[0] = x[rowoff + static_cast<size_t>(q) * C];
      }
#pragma unroll
      for (int k = 0; k < VEC; ++k)
        if (first || v[k] > m[k]) m[k] = v[k];
      first = false;
    }
  }
}

// 2x2 / stride 2 over one NHWC tensor (every VGG pool): the four window loads
// in registers, the forward's compare order, first equal position wins.
__global__ void __launch_bounds__(256) maxpool2x2_bwd_kernel(const float* __restrict__ x, float* __restrict__ dx,
                                                            const float* __restrict__ dy, int h, int w, int c,
                                                            int ho, int wo, int msk) {
  const int cv = c >> 2;
  const int row = blockIdx.y;  // n * ho + oh
  const int n = row / ho, oh = row - n * ho;
  const size_t base0 = (static_cast<size_t>(n) * h + 2 * oh) * w * cv;
  const float4* x0 = reinterpret_cast<const float4*>(x) + base0;
  const float4* x1 = x0 + static_cast<size_t>(w) * cv;
  float4* d0 = reinterpret_cast<float4*>(dx) + base0;
  float4* d1 = d0 + static_cast<size_t>(w) * cv;
  const float4* dyr = reinterpret_cast<const float4*>(dy + static_cast<size_t>(row) * wo * c);
  const int per_row = wo * cv;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < per_row; i += gridDim.x * blockDim.x) {
    const int ow = i / cv, c4 = i - ow * cv;
    const int off = 2 * ow * cv + c4;
    const float4 a = __ldcs(x0 + off), b = __ldcs(x0 + off + cv), e = __ldcs(x1 + off), f = __ldcs(x1 + off + cv);
    const float4 g = __ldcs(dyr + i);
    const float av[4] = {a.x, a.y, a.z, a.w}, bv[4] = {b.x, b.y, b.z, b.w}, ev[4] = {e.x, e.y, e.z, e.w},
                fv[4] = {f.x, f.y, f.z, f.w}, gv[4] = {g.x, g.y, g.z, g.w};
    float oa[4], ob[4], oe[4], of[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      float m = av[k];
      m = bv[k] > m ? bv[k] : m;
      m = ev[k] > m ? ev[k] : m;
      m = fv[k] > m ? fv[k] : m;
      const bool ha = av[k] == m, hb = !ha && bv[k] == m, he = !ha && !hb && ev[k] == m,
                 hf = !ha && !hb && !he && fv[k] == m;
      oa[k] = (ha && (!msk || av[k] > 0.f)) ? gv[k] : 0.f;
      ob[k] = (hb && (!msk || bv[k] > 0.f)) ? gv[k] : 0.f;
      oe[k] = (he && (!msk || ev[k] > 0.f)) ? gv[k] : 0.f;
      of[k] = (hf && (!msk || fv[k] > 0.f)) ? gv[k] : 0.f;
    }
    d0[off] = make_float4(oa[0], oa[1], oa[2], oa[3]);
    d0[off + cv] = make_float4(ob[0], ob[1], ob[2], ob[3]);
    d1[off] = make_float4(oe[0], oe[1], oe[2], oe[3]);
    d1[off + cv] = make_float4(of[0], of[1], of[2], of[3]);
  }
}

// Non-overlapping windows (stride >= window): one thread per output element
// (x VEC channels) finds the first maximum and scatters dY to it, zeros to the
// rest of its window -- every covered input written exactly once, no atomics.
template <int VEC>
__global__ void maxpool_bwd_scatter_kernel(const __grid_constant__ PoolDev d, const float* __restrict__ dy) {
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
    const int s = pool_seg(d, c);
    float* dx = d.dx[s];
    if (dx == nullptr) continue;
    const int cl = c - d.cbase[s];
    const float* x = d.x[s];
    const int C = d.c[s];
    const size_t oidx = ((static_cast<size_t>(n) * d.ho + oh) * d.wo + ow) * d.ctot + c;
    float ym[VEC], g[VEC];
    bool done[VEC];
    window_max<VEC>(x, ((static_cast<size_t>(n) * d.h + oh * d.stride) * d.w + ow * d.stride) * C + cl,
                    static_cast<size_t>(d.w) * C, C, d.window, ym);
#pragma unroll
    for (int k = 0; k < VEC; ++k) {
      g[k] = dy[oidx + k];
      done[k] = false;
    }
    for (int r = 0; r < d.window; ++r) {
      const size_t rowoff = ((static_cast<size_t>(n) * d.h + oh * d.stride + r) * d.w + ow * d.stride) * C + cl;
      for (int q = 0; q < d.window; ++q) {
        const size_t off = rowoff + static_cast<size_t>(q) * C;
        float v[VEC], o[VEC];
        if constexpr (VEC == 4) {
          const float4 f = *reinterpret_cast<const float4*>(x + off);
          v[0] = f.x; v[1] = f.y; v[2] = f.z; v[3] = f.w;
        } else {
          v[0] = x[off];
        }
        const bool msk = d.mask[s] != 0;
#pragma unroll
        for (int k = 0; k < VEC; ++k) {
          const bool hit = !done[k] && v[k] == ym[k];
          o[k] = (hit && (!msk || v[k] > 0.f)) ? g[k] : 0.f;
          done[k] = done[k] || hit;
        }
        if constexpr (VEC == 4)
          *reinterpret_cast<float4*>(dx + off) = make_float4(o[0], o[1], o[2], o[3]);
        else
          dx[off] = o[0];
      }
    }
  }
}

// Overlapping windows: gather form (deterministic): every input element sums
// dY over the windows whose first-maximum position it is.
__global__ void maxpool_bwd_kernel(const __grid_constant__ PoolDev d, const float* __restrict__ dy) {
  const size_t total = static_cast<size_t>(d.n) * d.h * d.w * d.ctot;
  for (size_t i = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; i < total;
       i += static_cast<size_t>(gridDim.x) * blockDim.x) {
    const int c = static_cast<int>(i % d.ctot);
    size_t t = i / d.ctot;
    const int iw = static_cast<int>(t % d.w);
    t /= d.w;
    const int ih = static_cast<int>(t % d.h);
    const int n = static_cast<int>(t / d.h);
    const int s = pool_seg(d, c);
    if (d.dx[s] == nullptr) continue;
    const int cl = c - d.cbase[s];
    const float* x = d.x[s];
    const int C = d.c[s];
    // windows oh with oh*stride <= ih < oh*stride + window
    int oh_lo = ih - d.window + 1;
    oh_lo = oh_lo <= 0 ? 0 : (oh_lo + d.stride - 1) / d.stride;
    int oh_hi = ih / d.stride;
    if (oh_hi > d.ho - 1) oh_hi = d.ho - 1;
    int ow_lo = iw - d.window + 1;
    ow_lo = ow_lo <= 0 ? 0 : (ow_lo + d.stride - 1) / d.stride;
    int ow_hi = iw / d.stride;
    if (ow_hi > d.wo - 1) ow_hi = d.wo - 1;
    float g = 0.f;
    for (int oh = oh_lo; oh <= oh_hi; ++oh) {
      for (int ow = ow_lo; ow <= ow_hi; ++ow) {
        const size_t oidx = ((static_cast<size_t>(n) * d.ho + oh) * d.wo + ow) * d.ctot + c;
        float ymv[1];
        window_max<1>(x, ((static_cast<size_t>(n) * d.h + oh * d.stride) * d.w + ow * d.stride) * C + cl,
                      static_cast<size_t>(d.w) * C, C, d.window, ymv);
        const float ym = ymv[0];
        // first position in row-major window order holding the max
        int ar = -1, aq = -1;
        for (int r = 0; r < d.window && ar < 0; ++r) {
          for (int q = 0; q < d.window; ++q) {
            const float v =
                x[((static_cast<size_t>(n) * d.h + oh * d.stride + r) * d.w + ow * d.stride + q) * C + cl];
            if (v == ym) {
              ar = r;
              aq = q;
              break;
            }
          }
        }
        if (oh * d.stride + ar == ih && ow * d.stride + aq == iw) g += dy[oidx];
      }
    }
    if (d.mask[s] && x[((static_cast<size_t>(n) * d.h + ih) * d.w + iw) * C + cl] <= 0.f) g = 0.f;
    d.dx[s][((static_cast<size_t>(n) * d.h + ih) * d.w + iw) * C + cl] = g;
  }
}

// Overlapping windows, 4 channels per thread (every segment C % 4 == 0): the
// same first-maximum rule per channel, float4 loads of the window, early exit
// once all four channels found their argmax. The scalar kernel rescanned up to
// 9 window elements per covering window with 4-byte loads (AlexNet 55x55x64
// pool: 1.05 ms for ~0.25 GB of traffic).
__global__ void maxpool_bwd_gather4_kernel(const __grid_constant__ PoolDev d, const float* __restrict__ dy) {
  const int cv = d.ctot / 4;
  const size_t total = static_cast<size_t>(d.n) * d.h * d.w * cv;
  for (size_t i = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; i < total;
       i += static_cast<size_t>(gridDim.x) * blockDim.x) {
    const int c = static_cast<int>(i % cv) * 4;
    size_t t = i / cv;
    const int iw = static_cast<int>(t % d.w);
    t /= d.w;
    const int ih = static_cast<int>(t % d.h);
    const int n = static_cast<int>(t / d.h);
    const int s = pool_seg(d, c);
    if (d.dx[s] == nullptr) continue;
    const int cl = c - d.cbase[s];
    const float* x = d.x[s];
    const int C = d.c[s];
    int oh_lo = ih - d.window + 1;
    oh_lo = oh_lo <= 0 ? 0 : (oh_lo + d.stride - 1) / d.stride;
    int oh_hi = ih / d.stride;
    if (oh_hi > d.ho - 1) oh_hi = d.ho - 1;
    int ow_lo = iw - d.window + 1;
    ow_lo = ow_lo <= 0 ? 0 : (ow_lo + d.stride - 1) / d.stride;
    int ow_hi = iw / d.stride;
    if (ow_hi > d.wo - 1) ow_hi = d.wo - 1;
    float g[4] = {0.f, 0.f, 0.f, 0.f};
    for (int oh = oh_lo; oh <= oh_hi; ++oh) {
      for (int ow = ow_lo; ow <= ow_hi; ++ow) {
        const size_t oidx = ((static_cast<size_t>(n) * d.ho + oh) * d.wo + ow) * d.ctot + c;
        float ym[4];
        window_max<4>(x, ((static_cast<size_t>(n) * d.h + oh * d.stride) * d.w + ow * d.stride) * C + cl,
                      static_cast<size_t>(d.w) * C, C, d.window, ym);
        int arg[4] = {-1, -1, -1, -1};  // r * window + q of the first maximum, per channel
        int left = 4;
        for (int r = 0; r < d.window && left > 0; ++r) {
          const float* row = x + ((static_cast<size_t>(n) * d.h + oh * d.stride + r) * d.w + ow * d.stride) * C + cl;
          for (int q = 0; q < d.window && left > 0; ++q) {
            const float4 v4 = *reinterpret_cast<const float4*>(row + static_cast<size_t>(q) * C);
            const float v[4] = {v4.x, v4.y, v4.z, v4.w};
#pragma unroll
            for (int k = 0; k < 4; ++k)
              if (arg[k] < 0 && v[k] == ym[k]) {
                arg[k] = r * d.window + q;
                --left;
              }
          }
        }
        const int here = (ih - oh * d.stride) * d.window + (iw - ow * d.stride);
        const float4 d4 = *reinterpret_cast<const float4*>(dy + oidx);
        const float dv[4] = {d4.x, d4.y, d4.z, d4.w};
#pragma unroll
        for (int k = 0; k < 4; ++k)
          if (arg[k] == here) g[k] += dv[k];
      }
    }
    const size_t xo = ((static_cast<size_t>(n) * d.h + ih) * d.w + iw) * C + cl;
    if (d.mask[s]) {
      const float4 xv = *reinterpret_cast<const float4*>(x + xo);
      if (xv.x <= 0.f) g[0] = 0.f;
      if (xv.y <= 0.f) g[1] = 0.f;
      if (xv.z <= 0.f) g[2] = 0.f;
      if (xv.w <= 0.f) g[3] = 0.f;
    }
    *reinterpret_cast<float4*>(d.dx[s] + xo) = make_float4(g[0], g[1], g[2], g[3]);
  }
}

// Overlapping windows with window <= 2*stride (AlexNet/OverFeat 3x3/2):
// deterministic scatter in four passes over the window parity classes
// (oh % 2, ow % 2) -- windows of one class never overlap, so each pass adds
// dY to its windows' first-maximum positions without races, in a fixed
// order. 4 channels per thread; dX zeroed first. The fused ReLU backward
// skips positions whose input is <= 0 (they end 0, as the mask demands).
__global__ void maxpool_bwd_class_kernel(const __grid_constant__ PoolDev d, const float* __restrict__ dy, int ph,
                                         int pw) {
  const int cv = d.ctot / 4;
  const int hoc = (d.ho - ph + 1) / 2, woc = (d.wo - pw + 1) / 2;  // windows of this class
  const size_t total = static_cast<size_t>(d.n) * hoc * woc * cv;
  for (size_t i = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; i < total;
       i += static_cast<size_t>(gridDim.x) * blockDim.x) {
    const int c = static_cast<int>(i % cv) * 4;
    size_t t = i / cv;
    const int ow = 2 * static_cast<int>(t % woc) + pw;
    t /= woc;
    const int oh = 2 * static_cast<int>(t % hoc) + ph;
    const int n = static_cast<int>(t / hoc);
    const int s = pool_seg(d, c);
    float* dx = d.dx[s];
    if (dx == nullptr) continue;
    const int cl = c - d.cbase[s];
    const float* x = d.x[s];
    const int C = d.c[s];
    float m[4];
    int arg[4] = {0, 0, 0, 0};
    for (int r = 0; r < d.window; ++r) {
      const float* row = x + ((static_cast<size_t>(n) * d.h + oh * d.stride + r) * d.w + ow * d.stride) * C + cl;
      for (int q = 0; q < d.window; ++q) {
        const float4 v4 = *reinterpret_cast<const float4*>(row + static_cast<size_t>(q) * C);
        const float v[4] = {v4.x, v4.y, v4.z, v4.w};
        const int pos = r * d.window + q;
#pragma unroll
        for (int k = 0; k < 4; ++k)
          if (pos == 0 || v[k] > m[k]) {
            m[k] = v[k];
            arg[k] = pos;
          }
      }
    }
    const size_t oidx = ((static_cast<size_t>(n) * d.ho + oh) * d.wo + ow) * d.ctot + c;
    const float4 d4 = *reinterpret_cast<const float4*>(dy + oidx);
    const float dv[4] = {d4.x, d4.y, d4.z, d4.w};
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      if (m[k] != m[k]) continue;  // NaN maximum: no position equals it
      if (d.mask[s] && m[k] <= 0.f) continue;
      const int r = arg[k] / d.window, q = arg[k] - r * d.window;
      float* dst = dx + ((static_cast<size_t>(n) * d.h + oh * d.stride + r) * d.w + ow * d.stride + q) * C + cl + k;
      *dst += dv[k];
    }
  }
}

cudaError_t maxpool_bwd(const PoolArgs& a, const float* y, const float* dy, cudaStream_t st) {
  const PoolDev d = to_dev(a);
  const size_t total = static_cast<size_t>(d.n) * d.h * d.w * d.ctot;
  if (total == 0) return cudaSuccess;
  if (d.stride >= d.window) {
    // inputs no window covers (floor-mode remainder, or stride > window) get 0
    const bool gaps = d.stride > d.window || (d.h - d.window) % d.stride != 0 || (d.w - d.window) % d.stride != 0 ||
                      d.ho * d.stride + (d.window - d.stride) < d.h || d.wo * d.stride + (d.window - d.stride) < d.w;
    if (gaps)
      for (int i = 0; i < d.nseg; ++i)
        if (d.dx[i]) {
          cudaError_t e = cudaMemsetAsync(d.dx[i], 0, static_cast<size_t>(d.n) * d.h * d.w * d.c[i] * sizeof(float), st);
          if (e != cudaSuccess) return e;
        }
    const size_t outs = static_cast<size_t>(d.n) * d.ho * d.wo * d.ctot;
    if (!gaps && d.nseg == 1 && d.window == 2 && d.stride == 2 && d.c[0] % 4 == 0 && d.dx[0] &&
        static_cast<int64_t>(d.n) * d.ho <= 65535) {
      const int per_row = d.wo * d.c[0] / 4;
      const dim3 grid(static_cast<unsigned>((per_row + 255) / 256), static_cast<unsigned>(d.n * d.ho));
      maxpool2x2_bwd_kernel<<<grid, 256, 0, st>>>(d.x[0], d.dx[0], dy, d.h, d.w, d.c[0], d.ho, d.wo, d.mask[0]);
    } else if (pool_vec4(d)) {
      maxpool_bwd_scatter_kernel<4><<<grid_for(outs / 4, 2), kThreads, 0, st>>>(d, dy);
    } else {
      maxpool_bwd_scatter_kernel<1><<<grid_for(outs, 4), kThreads, 0, st>>>(d, dy);
    }
  } else if (pool_vec4(d) && d.window <= 2 * d.stride) {
    for (int i = 0; i < d.nseg; ++i)
      if (d.dx[i]) {
        cudaError_t e = cudaMemsetAsync(d.dx[i], 0, static_cast<size_t>(d.n) * d.h * d.w * d.c[i] * sizeof(float), st);
        if (e != cudaSuccess) return e;
      }
    const size_t wins = static_cast<size_t>(d.n) * d.ho * d.wo * d.ctot / 4;
    for (int ph = 0; ph < 2; ++ph)
      for (int pw = 0; pw < 2; ++pw) {
        maxpool_bwd_class_kernel<<<grid_for(wins / 4 + 1, 2), kThreads, 0, st>>>(d, dy, ph, pw);
        count_launch();
      }
    return cudaGetLastError();
  } else if (pool_vec4(d)) {
    maxpool_bwd_gather4_kernel<<<grid_for(total / 4, 2), kThreads, 0, st>>>(d, dy);
  } else {
    maxpool_bwd_kernel<<<grid_for(total, 4), kThreads, 0, st>>>(d, dy);
  }
  count_launch();
  return cudaGetLastError();
}

// --------------------------------------------------- softmax x-entropy ----
// One warp per row; loss averaged over rows by a single-block deterministic
// reduction.
__global__ void softmax_xent_kernel(const float* __restrict__ logits, const int32_t* __restrict__ labels, int n,
                                    int k, float* __restrict__ grad, float* __restrict__ row_loss) {
  const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (warp >= n) return;
  const float* z = logits + static_cast<size_t>(warp) * k;
  float m = -FLT_MAX;
  for (int i = lane; i < k; i += 32) m = fmaxf(m, z[i]);
  for (int o = 16; o > 0; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
  float s = 0.f;
  for (int i = lane; i < k; i += 32) s += expf(z[i] - m);
  for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  const float lse = m + logf(s);
  const int lab = labels[warp] % k;  // several LOSS heads share one label vector
  const float inv_n = 1.0f / static_cast<float>(n);
  for (int i = lane; i < k; i += 32) {
    const float pr = expf(z[i] - lse);
    grad[static_cast<size_t>(warp) * k + i] = (pr - (i == lab ? 1.f : 0.f)) * inv_n;
  }
  if (lane == 0) row_loss[warp] = lse - z[lab];
}

__global__ void mean_kernel(const float* __restrict__ v, int n, float* __restrict__ out, int accumulate) {
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

cudaError_t softmax_xent_fwd(const float* logits, const int32_t* labels, int n, int k, float* grad_scratch,
                             float* row_loss, float* loss, cudaStream_t st, bool accumulate) {
  if (n <= 0) return cudaSuccess;
  const int threads = 256;
  const int blocks = (n * 32 + threads - 1) / threads;
  softmax_xent_kernel<<<blocks, threads, 0, st>>>(logits, labels, n, k, grad_scratch, row_loss);
  mean_kernel<<<1, 256, 0, st>>>(row_loss, n, loss, accumulate ? 1 : 0);
  count_launch(2);
  return cudaGetLastError();
}

// ------------------------------------------------------- bias / SGD -------
__global__ void bias_grad_kernel(const float* __restrict__ dy, int n, int o, float* __restrict__ bias, float lr,
                                 float* __restrict__ db) {
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= o) return;
  float s = 0.f;
  for (int i = 0; i < n; ++i) s += dy[static_cast<size_t>(i) * o + j];
  if (db)
    db[j] = s;
  else
    bias[j] -= lr * s;
}

cudaError_t bias_grad(const float* dy, int n, int o, float* bias, float lr, float* db_out, cudaStream_t st) {
  if (o <= 0) return cudaSuccess;
  bias_grad_kernel<<<(o + 255) / 256, 256, 0, st>>>(dy, n, o, bias, lr, db_out);
  count_launch();
  return cudaGetLastError();
}

__global__ void sgd_kernel(float* __restrict__ w, const float* __restrict__ g, float lr, size_t n) {
  for (size_t i = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<size_t>(gridDim.x) * blockDim.x)
    w[i] -= lr * g[i];
}

cudaError_t sgd_update(float* w, const float* g, float lr, size_t n, cudaStream_t st) {
  if (n == 0) return cudaSuccess;
  sgd_kernel<<<grid_for(n, 8), kThreads, 0, st>>>(w, g, lr, n);
  count_launch();
  return cudaGetLastError();
}

__global__ void scale_kernel(float* __restrict__ x, float s, size_t n) {
  for (size_t i = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<size_t>(gridDim.x) * blockDim.x)
    x[i] *= s;
}

cudaError_t scale_inplace(float* x, float s, size_t n, cudaStream_t st) {
  if (n == 0) return cudaSuccess;
  scale_kernel<<<grid_for(n, 8), kThreads, 0, st>>>(x, s, n);
  count_launch();
  return cudaGetLastError();
}

// ---------------------------------------------------------- fills ---------
__global__ void fill_normal_kernel(float* __restrict__ w, size_t n, float stddev, uint64_t seed) {
  for (size_t i = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<size_t>(gridDim.x) * blockDim.x) {
    const uint64_t a = splitmix64(seed * 0x100000001B3ull + 2 * i);
    const uint64_t b = splitmix64(seed * 0x100000001B3ull + 2 * i + 1);
    const float u1 = 1.0f - u01(a);  // (0, 1]
    const float u2 = u01(b);
    w[i] = stddev * sqrtf(-2.0f * logf(u1)) * cospif(2.0f * u2);
  }
}

cudaError_t fill_normal(float* w, size_t n, float stddev, uint64_t seed, cudaStream_t st) {
  if (n == 0) return cudaSuccess;
  fill_normal_kernel<<<grid_for(n, 8), kThreads, 0, st>>>(w, n, stddev, seed);
  count_launch();
  return cudaGetLastError();
}

__global__ void fill_uniform_kernel(float* __restrict__ x, size_t n, float lo, float hi, uint64_t seed) {
  for (size_t i = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<size_t>(gridDim.x) * blockDim.x)
    x[i] = lo + (hi - lo) * u01(splitmix64(seed * 0x9E3779B97F4A7C15ull + i));
}

cudaError_t fill_uniform(float* x, size_t n, float lo, float hi, uint64_t seed, cudaStream_t st) {
  if (n == 0) return cudaSuccess;
  fill_uniform_kernel<<<grid_for(n, 8), kThreads, 0, st>>>(x, n, lo, hi, seed);
  count_launch();
  return cudaGetLastError();
}

__global__ void fill_const_kernel(float* __restrict__ x, size_t n, float v) {
  for (size_t i = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<size_t>(gridDim.x) * blockDim.x)
    x[i] = v;
}

cudaError_t fill_const(float* x, size_t n, float v, cudaStream_t st) {
  if (n == 0) return cudaSuccess;
  fill_const_kernel<<<grid_for(n, 8), kThreads, 0, st>>>(x, n, v);
  count_launch();
  return cudaGetLastError();
}

__global__ void fill_labels_kernel(int32_t* __restrict__ y, size_t n, int classes, uint64_t seed) {
  for (size_t i = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<size_t>(gridDim.x) * blockDim.x)
    y[i] = static_cast<int32_t>(splitmix64(seed * 0x9E3779B97F4A7C15ull + i) % static_cast<uint64_t>(classes));
}

cudaError_t fill_labels(int32_t* y, size_t n, int classes, uint64_t seed, cudaStream_t st) {
  if (n == 0) return cudaSuccess;
  fill_labels_kernel<<<grid_for(n), kThreads, 0, st>>>(y, n, classes, seed);
  count_launch();
  return cudaGetLastError();
}

}  // namespace vdnnk
