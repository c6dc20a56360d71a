// First-layer convolutions on the tensor cores (TF32 mode): C <= 4 input
// channels and a whole filter window that fits one 32-wide K block
// (kh*kw*C <= 32, e.g. VGG's 3x3x3 = 27). The im2col row of a pixel is only
// 27 floats at a 12-byte pixel stride, which TMA cannot address, so threads
// build the operand rows and the tensor core does the contraction; both
// kernels are then bound by their one big HBM stream (Y written / dY read).
//
//   fprop  Y[p][co] = relu?( sum_k A[p][k] * W[co][k] ),  A[p][k] = im2col(X)
//          persistent CTAs, 128-pixel tiles: 4 builder warps write A rows
//          (K-major SWIZZLE_128B) into a 4-stage ring, one thread issues
//          4 x tcgen05.mma (M=128, N=Cout, K=8) into one of two TMEM
//          accumulators, 4 epilogue warps drain TMEM -> ReLU -> swizzled smem
//          -> TMA store, overlapping the next tiles' build and MMA.
//   wgrad  dW[co][k] = sum_p dY[p][co] * A[p][k]
//          D[co][k] (M = 128 rows, co < Cout live; N = 32) accumulates over a
//          contiguous pixel range per CTA: dY tiles arrive by TMA (MN-major
//          32x32 boxes), eight builder warps each write the A^T rows of every
//          eighth 32-pixel stage (MN-major SWIZZLE_128B_BASE32B), partials per
//          CTA are reduced in order (deterministic) with the SGD update fused.
// The exact-fp32 mode (3xTF32 elsewhere) keeps the SIMT kernels of
// conv_smallc.cu. FLOPs as the reference counts them:
// 2*k^2*C*Cout*Ho*Wo*N per pass (cost_model.hpp:100-106).
#include <algorithm>
#include <cstdlib>

#include "kernels.h"
#include "tc_conv.cuh"
#include "tma_maps.h"

namespace vdnnk {

bool precise();
cudaError_t smallc_wgrad_reduce_launch(const float* part, int nparts, int64_t count, float* w, float lr,
                                       float* dw_out, cudaStream_t st);

namespace {

constexpr int kSms = 148;
constexpr int kFpStages = 4;
constexpr int kWgStages = 10;
constexpr int kPrefetch = 24;  // wgrad: dY stages prefetched into L2 ahead of the ring

struct C3Geom {
  int N, H, W, C, Ho, Wo, Cout, k, stride, pad, KK;
  int P, HoWo;  // output pixels (host checks P < 2^31)
};

// Window table (shared memory): element offset of im2col column i relative
// to the window's top-left input element, and its tap (r, s) for clipping.
__device__ __forceinline__ void c3_table(const C3Geom& g, int* off, int* rs) {
  const int i = threadIdx.x;
  if (i < 32) {
    if (i < g.KK) {
      const int tap = i / g.C, c = i - tap * g.C;
      const int r = tap / g.k, s = tap - r * g.k;
      off[i] = (r * g.W + s) * g.C + c;
      rs[i] = r | (s << 8);
    } else {
      off[i] = 0;
      rs[i] = 0;
    }
  }
}

// im2col row of output pixel m: 32 values (columns >= KK and padding -> 0).
__device__ __forceinline__ void c3_row(const float* __restrict__ x, const C3Geom& g, const int* off, const int* rs,
                                       int m, float (&v)[32]) {
#pragma unroll
  for (int i = 0; i < 32; ++i) v[i] = 0.f;
  if (m >= g.P) return;
  const int n = m / g.HoWo;
  const int rem = m - n * g.HoWo;
  const int oh = rem / g.Wo, ow = rem - oh * g.Wo;
  const int ih0 = oh * g.stride - g.pad, iw0 = ow * g.stride - g.pad;
  const int64_t base = ((static_cast<int64_t>(n) * g.H + ih0) * g.W + iw0) * g.C;
  if (ih0 >= 0 && ih0 + g.k <= g.H && iw0 >= 0 && iw0 + g.k <= g.W) {
#pragma unroll
    for (int i = 0; i < 32; ++i)
      if (i < g.KK) v[i] = __ldg(x + base + off[i]);
  } else {
#pragma unroll
    for (int i = 0; i < 32; ++i) {
      if (i < g.KK) {
        const int ih = ih0 + (rs[i] & 0xff), iw = iw0 + (rs[i] >> 8);
        if (ih >= 0 && ih < g.H && iw >= 0 && iw < g.W) v[i] = __ldg(x + base + off[i]);
      }
    }
  }
}

// Compile-time window (KT x KT taps of CT channels, e.g. VGG's 3 x 3 x 3):
// the 27 loads sit at constant offsets from KT row pointers and clipping is
// two KT-bit masks -- no table reads and no per-element address arithmetic
// (the table-driven row issues ~10 instructions per element; the builders
// are then issue-bound, not HBM-bound). KT = 0: the table-driven row.
template <int KT, int CT>
__device__ __forceinline__ void c3_row_t(const float* __restrict__ x, const C3Geom& g, const int* off, const int* rs,
                                         int m, float (&v)[32]) {
  if constexpr (KT == 0) {
    c3_row(x, g, off, rs, m, v);
  } else {
    static_assert(KT * KT * CT <= 32, "window must fit one K block");
#pragma unroll
    for (int i = 0; i < 32; ++i) v[i] = 0.f;
    if (m >= g.P) return;
    const int n = m / g.HoWo;
    const int rem = m - n * g.HoWo;
    const int oh = rem / g.Wo, ow = rem - oh * g.Wo;
    const int ih0 = oh * g.stride - g.pad, iw0 = ow * g.stride - g.pad;
    uint32_t rmask = 0, cmask = 0;
#pragma unroll
    for (int r = 0; r < KT; ++r) rmask |= (ih0 + r >= 0 && ih0 + r < g.H) ? (1u << r) : 0u;
#pragma unroll
    for (int s = 0; s < KT; ++s) cmask |= (iw0 + s >= 0 && iw0 + s < g.W) ? (1u << s) : 0u;
    const float* x0 = x + ((static_cast<int64_t>(n) * g.H + ih0) * g.W + iw0) * CT;
    const int64_t rstride = static_cast<int64_t>(g.W) * CT;
    const bool full = rmask == (1u << KT) - 1 && cmask == (1u << KT) - 1;
#pragma unroll
    for (int r = 0; r < KT; ++r) {
      const float* xr = x0 + r * rstride;
#pragma unroll
      for (int s = 0; s < KT; ++s) {
#pragma unroll
        for (int c = 0; c < CT; ++c)
          if (full || (((rmask >> r) & (cmask >> s)) & 1u)) v[(r * KT + s) * CT + c] = __ldg(xr + s * CT + c);
      }
    }
  }
}

// Multi-K-block variant (kh*kw*C > 32, e.g. AlexNet / OverFeat 11x11x3 =
// 363 = 12 K blocks): table entries for all KB*32 im2col columns.
constexpr int kMkMaxKB = 12;
__device__ __forceinline__ void c3_table_mk(const C3Geom& g, int kb_count, int* off, int* rs) {
  for (int i = threadIdx.x; i < kb_count * 32; i += blockDim.x) {
    if (i < g.KK) {
      const int tap = i / g.C, c = i - tap * g.C;
      const int r = tap / g.k, s = tap - r * g.k;
      off[i] = (r * g.W + s) * g.C + c;
      rs[i] = r | (s << 8);
    } else {
      off[i] = 0;
      rs[i] = 0;
    }
  }
}

// Window origin of output pixel m (decoded once, then reused for every K block).
struct C3Pix {
  int64_t base;
  int ih0, iw0;
  bool valid, interior;
};
__device__ __forceinline__ C3Pix c3_pix(const C3Geom& g, int m) {
  C3Pix q;
  q.valid = m < g.P;
  const int mm = q.valid ? m : 0;
  const int n = mm / g.HoWo;
  const int rem = mm - n * g.HoWo;
  const int oh = rem / g.Wo, ow = rem - oh * g.Wo;
  q.ih0 = oh * g.stride - g.pad;
  q.iw0 = ow * g.stride - g.pad;
  q.base = ((static_cast<int64_t>(n) * g.H + q.ih0) * g.W + q.iw0) * g.C;
  q.interior = q.ih0 >= 0 && q.ih0 + g.k <= g.H && q.iw0 >= 0 && q.iw0 + g.k <= g.W;
  return q;
}
// the 32 im2col values of K block kb for pixel q (columns >= KK and padding -> 0)
__device__ __forceinline__ void c3_row_kb(const float* __restrict__ x, const C3Geom& g, const int* off,
                                          const int* rs, const C3Pix& q, int kb, float (&v)[32]) {
  const int k0 = kb * 32;
#pragma unroll
  for (int i = 0; i < 32; ++i) v[i] = 0.f;
  if (!q.valid) return;
  if (q.interior) {
#pragma unroll
    for (int i = 0; i < 32; ++i)
      if (k0 + i < g.KK) v[i] = __ldg(x + q.base + off[k0 + i]);
  } else {
#pragma unroll
    for (int i = 0; i < 32; ++i) {
      if (k0 + i < g.KK) {
        const int t = rs[k0 + i];
        const int ih = q.ih0 + (t & 0xff), iw = q.iw0 + (t >> 8);
        if (ih >= 0 && ih < g.H && iw >= 0 && iw < g.W) v[i] = __ldg(x + q.base + off[k0 + i]);
      }
    }
  }
}

// ------------------------------------------------------------ fprop ------
// smem: [B: NB rows x 128 B][A: kFpStages x 16 KB][OUT: 2 x NB/32 x 16 KB][barriers][table]
// warps 0-3 epilogue, 4-11 builders (two groups of 4 warps taking alternate
// tiles, one pixel row per thread), 12 MMA (+ TMEM owner). TMEM: 2 x NBP columns.
constexpr int kFpThreads = 416;
template <int KT, int CT>
__global__ void __launch_bounds__(kFpThreads, 1) c3tc_fprop_kernel(const float* __restrict__ x,
                                                                   const float* __restrict__ w,
                                                                   const __grid_constant__ CUtensorMap tma_y,
                                                                   C3Geom g, int NB, int NBP, int relu) {
  extern __shared__ uint8_t smem_raw[];
  const uint32_t raw = smem_u32(smem_raw);
  const uint32_t base = (raw + 1023u) & ~1023u;
  const uint32_t sb = base;
  const uint32_t sa0 = sb + ((NB * 128 + 1023) & ~1023);
  const uint32_t so = sa0 + kFpStages * 16384;
  const uint32_t obytes = (NB / 32) * 16384;  // one output staging buffer (double-buffered)
  const uint32_t bars = so + 2 * obytes;
  auto full_bar = [&](int s) { return bars + 8u * s; };
  auto empty_bar = [&](int s) { return bars + 8u * (kFpStages + s); };
  auto tfull_bar = [&](int a) { return bars + 8u * (2 * kFpStages + a); };
  auto tempty_bar = [&](int a) { return bars + 8u * (2 * kFpStages + 2 + a); };
  const uint32_t tmem_slot = bars + 8u * (2 * kFpStages + 4);
  int* tab = reinterpret_cast<int*>(smem_raw + (bars + 8u * (2 * kFpStages + 6) - raw));

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int ntiles = (g.P + kBM - 1) / kBM;

  if (threadIdx.x == 0) {
    for (int s = 0; s < kFpStages; ++s) {
      mbar_init(full_bar(s), 128);
      mbar_init(empty_bar(s), 1);
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(tfull_bar(a), 1);
      mbar_init(tempty_bar(a), 128);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  c3_table(g, tab, tab + 32);
  // weights -> B (row co, K-major swizzled; rows >= Cout and k >= KK are 0)
  for (int i = threadIdx.x; i < NB * 8; i += blockDim.x) {
    const int co = i >> 3, j = i & 7;
    float q[4];
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      const int k = j * 4 + e;
      q[e] = (co < g.Cout && k < g.KK) ? w[static_cast<int64_t>(co) * g.KK + k] : 0.f;
    }
    asm volatile("st.shared.v4.f32 [%0], {%1, %2, %3, %4};" ::"r"(kmaj_addr(sb, co, j)), "f"(q[0]), "f"(q[1]),
                 "f"(q[2]), "f"(q[3])
                 : "memory");
  }
  fence_proxy_async();
  if (warp == 12) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(tmem_slot),
                 "r"(2 * NBP)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  uint32_t tmem;
  asm volatile("ld.shared.u32 %0, [%1];" : "=r"(tmem) : "r"(tmem_slot) : "memory");

  if (warp >= 4 && warp < 12) {
    // ---------------- builders ----------------
    const int grp = (warp - 4) >> 2;
    const int row = (threadIdx.x - 128) & 127;
    int it = grp;
    // software-pipelined: the next tile's loads are in flight while this
    // tile's row waits for its stage and is stored
    float v[32], nv[32];
    const int tile0 = blockIdx.x + grp * gridDim.x;
    if (tile0 < ntiles) c3_row_t<KT, CT>(x, g, tab, tab + 32, tile0 * kBM + row, v);
    for (int tile = tile0; tile < ntiles; tile += 2 * gridDim.x, it += 2) {
      const int s = it % kFpStages;
      const int nt = tile + 2 * gridDim.x;
      if (nt < ntiles) c3_row_t<KT, CT>(x, g, tab, tab + 32, nt * kBM + row, nv);
      if (it >= kFpStages) mbar_wait(empty_bar(s), ((it / kFpStages) & 1) ^ 1);
      const uint32_t sa = sa0 + s * 16384;
#pragma unroll
      for (int j = 0; j < 8; ++j)
        asm volatile("st.shared.v4.f32 [%0], {%1, %2, %3, %4};" ::"r"(kmaj_addr(sa, row, j)), "f"(v[4 * j]),
                     "f"(v[4 * j + 1]), "f"(v[4 * j + 2]), "f"(v[4 * j + 3])
                     : "memory");
      fence_proxy_async();
      mbar_arrive(full_bar(s));
#pragma unroll
      for (int i = 0; i < 32; ++i) v[i] = nv[i];
    }
  } else if (warp == 12) {
    // ---------------- MMA issuer ----------------
    // whole warp in the loop, one elected lane issues; descriptors advanced
    // by constants, running stage / phase counters (see c3tc_wgrad_kernel)
    const uint32_t idesc = make_idesc_tf32(NB, false, false);
    const bool leader = elect_one();
    const uint64_t ad0 = make_sdesc(sa0, 16, 1024, kSw128), bd = make_sdesc(sb, 16, 1024, kSw128);
    int it = 0, s = 0;
    uint32_t ph = 0;
    for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x, ++it) {
      const int acc = it & 1;
      mbar_wait(full_bar(s), ph);
      if (it >= 2) mbar_wait(tempty_bar(acc), ((it >> 1) & 1) ^ 1);
      tc_fence_after();
      if (leader) {
        const uint64_t ad = ad0 + static_cast<uint64_t>(s) * (16384 >> 4);
#pragma unroll
        for (int kk = 0; kk < kBK / 8; ++kk)
          tc_mma_tf32(tmem + acc * NBP, ad + kk * 2, bd + kk * 2, idesc, kk > 0 ? 1u : 0u);
        tc_commit(empty_bar(s));
        tc_commit(tfull_bar(acc));
      }
      __syncwarp();
      if (++s == kFpStages) {
        s = 0;
        ph ^= 1;
      }
    }
  } else {
    // ---------------- epilogue ----------------
    const int row = warp * 32 + lane;
    int it = 0;
    for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x, ++it) {
      const int acc = it & 1;
      // the staging buffer of tile it-2 has been read out by its TMA store
      if (threadIdx.x == 0) asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
      const uint32_t ob = so + (it & 1) * obytes;
      asm volatile("bar.sync 1, 128;" ::: "memory");
      mbar_wait(tfull_bar(acc), (it >> 1) & 1);
      tc_fence_after();
      const uint32_t taddr = tmem + acc * NBP + (static_cast<uint32_t>(warp * 32) << 16);
      for (int cg = 0; cg < NB / 32; ++cg) {
        float v[32];
        tmem_ld32(taddr + cg * 32, v);
        if (relu) {
#pragma unroll
          for (int i = 0; i < 32; ++i) v[i] = fmaxf(v[i], 0.f);
        }
        const uint32_t rowaddr = ob + cg * 16384 + row * 128;
#pragma unroll
        for (int j = 0; j < 8; ++j)
          asm volatile("st.shared.v4.f32 [%0], {%1, %2, %3, %4};" ::"r"(rowaddr + (((j ^ (row & 7)) & 7) << 4)),
                       "f"(v[4 * j]), "f"(v[4 * j + 1]), "f"(v[4 * j + 2]), "f"(v[4 * j + 3])
                       : "memory");
      }
      tc_fence_before();
      mbar_arrive(tempty_bar(acc));
      fence_proxy_async();
      asm volatile("bar.sync 1, 128;" ::: "memory");
      if (threadIdx.x == 0) {
        for (int cg = 0; cg < NB / 32; ++cg)
          if (cg * 32 < g.Cout) tma_store_2d(&tma_y, ob + cg * 16384, cg * 32, tile * kBM, false);
        asm volatile("cp.async.bulk.commit_group;" ::: "memory");
      }
    }
    if (threadIdx.x == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 12) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(2 * NBP) : "memory");
  }
}

// ------------------------------------------------------------ wgrad ------
// D[co][k] (M = 128 rows, co < Cout <= 128 live; N = 32 columns = k).
// smem per stage: [A = dY^T: 4 MN-chunks x 4 KB by one TMA (chunks >= Cout/32 stay 0)]
//                 [B = im2col^T: 1 MN-chunk x 4 KB, one pixel row per builder lane]
// warps 0-7 builders (warp w builds stages it = w mod 8; warps < Cout/32 then
// drain TMEM), warp 8 lane 0 TMA, warp 9 MMA + TMEM.
constexpr int kWgThreads = 320;
constexpr uint32_t kWgStage = 16384 + 4096;
template <int KT, int CT>
__global__ void __launch_bounds__(kWgThreads, 1) c3tc_wgrad_kernel(const float* __restrict__ x,
                                                                   const __grid_constant__ CUtensorMap tma_dy,
                                                                   C3Geom g, int ppb, int pf, float* __restrict__ part) {
  extern __shared__ uint8_t smem_raw[];
  const uint32_t raw = smem_u32(smem_raw);
  const uint32_t base = (raw + 1023u) & ~1023u;
  const uint32_t bars = base + kWgStages * kWgStage;
  auto full_bar = [&](int s) { return bars + 8u * s; };
  auto empty_bar = [&](int s) { return bars + 8u * (kWgStages + s); };
  const uint32_t done_bar = bars + 8u * (2 * kWgStages);
  const uint32_t tmem_slot = bars + 8u * (2 * kWgStages + 1);
  int* tab = reinterpret_cast<int*>(smem_raw + (bars + 8u * (2 * kWgStages + 2) - raw));

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int p_begin = blockIdx.x * ppb;
  const int p_end = min(p_begin + ppb, g.P);
  const int nkb = p_end > p_begin ? (p_end - p_begin + kBK - 1) / kBK : 0;
  const int nchunk = g.Cout / 32;

  if (threadIdx.x == 0) {
    for (int s = 0; s < kWgStages; ++s) {
      mbar_init(full_bar(s), 33);  // the building warp's 32 lanes + the TMA thread's expect_tx arrival
      mbar_init(empty_bar(s), 1);
    }
    mbar_init(done_bar, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  c3_table(g, tab, tab + 32);
  // A chunks >= Cout/32 (M rows the TMA never writes) are zero in every stage
  const int zbytes = (4 - nchunk) * 4096;
  for (int s = 0; s < kWgStages; ++s)
    for (int off = threadIdx.x * 16; off < zbytes; off += blockDim.x * 16)
      asm volatile("st.shared.v4.u32 [%0], {%1, %1, %1, %1};" ::"r"(base + s * kWgStage + nchunk * 4096 + off),
                   "r"(0)
                   : "memory");
  fence_proxy_async();
  if (warp == 9) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(tmem_slot), "r"(32)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  uint32_t tmem;
  asm volatile("ld.shared.u32 %0, [%1];" : "=r"(tmem) : "r"(tmem_slot) : "memory");

  if (warp < 8) {
    // ---------------- builders ----------------
    // software-pipelined: stage it + 8's loads are in flight while stage it
    // waits for its slot and is stored
    auto pix = [&](int i) {
      const int m = p_begin + i * kBK + lane;
      return m < p_end ? m : g.P;
    };
    float v[32], nv[32];
    if (warp < nkb) c3_row_t<KT, CT>(x, g, tab, tab + 32, pix(warp), v);
    for (int it = warp; it < nkb; it += 8) {
      const int s = it % kWgStages;
      if (it + 8 < nkb) c3_row_t<KT, CT>(x, g, tab, tab + 32, pix(it + 8), nv);
      if (it >= kWgStages) mbar_wait(empty_bar(s), ((it / kWgStages) & 1) ^ 1);
      const uint32_t sbb = base + s * kWgStage + 16384;
#pragma unroll
      for (int j = 0; j < 8; ++j)
        asm volatile("st.shared.v4.f32 [%0], {%1, %2, %3, %4};" ::"r"(mnmaj_addr(sbb, lane, 0, j)), "f"(v[4 * j]),
                     "f"(v[4 * j + 1]), "f"(v[4 * j + 2]), "f"(v[4 * j + 3])
                     : "memory");
      fence_proxy_async();
      mbar_arrive(full_bar(s));
#pragma unroll
      for (int i = 0; i < 32; ++i) v[i] = nv[i];
    }
    // ---------------- epilogue: warp w owns TMEM lanes 32w.. = co ----------------
    if (warp < nchunk) {
      mbar_wait_sleep(done_bar, 0);
      tc_fence_after();
      float v[32];
      tmem_ld32(tmem + (static_cast<uint32_t>(warp * 32) << 16), v);
      if (nkb <= 0) {
#pragma unroll
        for (int i = 0; i < 32; ++i) v[i] = 0.f;
      }
      float* dst = part + (static_cast<int64_t>(blockIdx.x) * g.Cout + warp * 32 + lane) * g.KK;
#pragma unroll
      for (int i = 0; i < 32; ++i)
        if (i < g.KK) dst[i] = v[i];
    }
  } else if (warp == 8) {
    // ---------------- TMA producer (dY tiles) ----------------
    if (lane == 0) {
      asm volatile("prefetch.tensormap [%0];" ::"l"(&tma_dy) : "memory");
      for (int it = 0; it < nkb; ++it) {
        const int s = it % kWgStages;
        // warm L2 with the tile `pf` stages ahead: the ring's loads then hit L2
        if (pf > 0 && it + pf < nkb)
          asm volatile("cp.async.bulk.prefetch.tensor.3d.L2.global [%0, {%1, %2, %3}];" ::"l"(&tma_dy), "r"(0),
                       "r"(p_begin + (it + pf) * kBK), "r"(0)
                       : "memory");
        if (it >= kWgStages) mbar_wait(empty_bar(s), ((it / kWgStages) & 1) ^ 1);
        mbar_expect_tx(full_bar(s), static_cast<uint32_t>(nchunk * 4096));
        tma_load_3d(base + s * kWgStage, &tma_dy, full_bar(s), 0, p_begin + it * kBK, 0);
      }
    }
    __syncwarp();
  } else {
    // ---------------- MMA issuer ----------------
    // N = 32 MMAs are short (one per 8 pixels), so the issue loop itself is
    // the limiter (ncu: the MMA warp never waited for a full stage and spent
    // ~575 cycles per stage on dependent uniform-datapath instructions): the
    // descriptors are built once and advanced by constants, the stage and
    // phase are running counters (no division), and the whole warp runs the
    // loop with one elected lane issuing
    const uint32_t idesc = make_idesc_tf32(32, true, true);
    const bool leader = elect_one();
    const uint64_t ad0 = make_sdesc(base, 4096, 512, kSw128Base32);
    const uint64_t bd0 = make_sdesc(base + 16384, 4096, 512, kSw128Base32);
    constexpr uint64_t kStageLo = kWgStage >> 4, kKkLo = 1024 >> 4;
    int s = 0;
    uint32_t ph = 0;
    for (int it = 0; it < nkb; ++it) {
      mbar_wait(full_bar(s), ph);
      tc_fence_after();
      if (leader) {
        const uint64_t so = static_cast<uint64_t>(s) * kStageLo;
        const uint64_t ad = ad0 + so, bd = bd0 + so;
        tc_mma_tf32(tmem, ad, bd, idesc, it > 0 ? 1u : 0u);
#pragma unroll
        for (int kk = 1; kk < kBK / 8; ++kk) tc_mma_tf32(tmem, ad + kk * kKkLo, bd + kk * kKkLo, idesc, 1u);
        tc_commit(empty_bar(s));
      }
      __syncwarp();
      if (++s == kWgStages) {
        s = 0;
        ph ^= 1;
      }
    }
    if (leader) {
      if (nkb > 0)
        tc_commit(done_bar);
      else
        mbar_arrive(done_bar);
    }
    __syncwarp();
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 9) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(32) : "memory");
  }
}

// ------------------------------------------------------ multi-K fprop ------
// Same warp roles as c3tc_fprop_kernel; a tile is KB pipeline stages (one
// per 32-column K block). A stage holds the A block built from the input
// (one pixel row per builder thread) and the matching K block of W (copied by
// the same builders: W [Cout][KK] rows are not 16-B aligned at KK = 363, so
// it is not resident -- 12 x NB x 128 B would not fit next to the ring).
constexpr int kMkFpStages = 4;
// builder groups take stages round-robin: group spacing (kMkGroups) must not
// exceed the ring depth for the parity waits to stay unambiguous
constexpr int kMkGroups = 4;
constexpr int kMkMmaWarp = 4 + 4 * kMkGroups;
constexpr int kFpMkThreads = 32 * (kMkMmaWarp + 1);
static_assert(kMkGroups <= kMkFpStages, "builder spacing must fit the ring");
__global__ void __launch_bounds__(kFpMkThreads, 1) c3tc_fprop_mk_kernel(const float* __restrict__ x,
                                                                      const float* __restrict__ w,
                                                                      const __grid_constant__ CUtensorMap tma_y,
                                                                      C3Geom g, int NB, int NBP, int KB, int relu) {
  extern __shared__ uint8_t smem_raw[];
  const uint32_t raw = smem_u32(smem_raw);
  const uint32_t base = (raw + 1023u) & ~1023u;
  const uint32_t bbytes = (static_cast<uint32_t>(NB) * 128 + 1023u) & ~1023u;
  const uint32_t stage = 16384 + bbytes;
  const uint32_t so = base + kMkFpStages * stage;
  const uint32_t obytes = (NB / 32) * 16384;
  const uint32_t bars = so + 2 * obytes;
  auto full_bar = [&](int s) { return bars + 8u * s; };
  auto empty_bar = [&](int s) { return bars + 8u * (kMkFpStages + s); };
  auto tfull_bar = [&](int a) { return bars + 8u * (2 * kMkFpStages + a); };
  auto tempty_bar = [&](int a) { return bars + 8u * (2 * kMkFpStages + 2 + a); };
  const uint32_t tmem_slot = bars + 8u * (2 * kMkFpStages + 4);
  int* tab = reinterpret_cast<int*>(smem_raw + (bars + 8u * (2 * kMkFpStages + 6) - raw));

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int ntiles = (g.P + kBM - 1) / kBM;

  if (threadIdx.x == 0) {
    for (int s = 0; s < kMkFpStages; ++s) {
      mbar_init(full_bar(s), 128);
      mbar_init(empty_bar(s), 1);
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(tfull_bar(a), 1);
      mbar_init(tempty_bar(a), 128);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  c3_table_mk(g, KB, tab, tab + kMkMaxKB * 32);
  if (warp == kMkMmaWarp) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(tmem_slot),
                 "r"(2 * NBP)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  uint32_t tmem;
  asm volatile("ld.shared.u32 %0, [%1];" : "=r"(tmem) : "r"(tmem_slot) : "memory");
  const int* off = tab;
  const int* rs = tab + kMkMaxKB * 32;

  if (warp >= 4 && warp < kMkMmaWarp) {
    // ---------------- builders: kMkGroups groups of 4 warps take stages round-robin ----------------
    // (mbarrier parity waits are only unambiguous if a builder's consecutive
    // stages are at most kMkFpStages apart: alternating whole 12-stage tiles
    // let a group wait on a slot two phases back -- wrong data, measured)
    const int grp = (warp - 4) >> 2;
    const int t = (threadIdx.x - 128) & 127;
    int cur_tl = -1;
    C3Pix q{};
    const int total = ((ntiles - static_cast<int>(blockIdx.x) + static_cast<int>(gridDim.x) - 1) /
                       static_cast<int>(gridDim.x)) * KB;
    for (int it = grp; it < total; it += kMkGroups) {
      const int tl = it / KB, kb = it - tl * KB;
      if (tl != cur_tl) {
        cur_tl = tl;
        q = c3_pix(g, (static_cast<int>(blockIdx.x) + tl * static_cast<int>(gridDim.x)) * kBM + t);
      }
      const int s = it % kMkFpStages;
      float v[32];
      c3_row_kb(x, g, off, rs, q, kb, v);  // loads in flight while the stage drains
      if (it >= kMkFpStages) mbar_wait(empty_bar(s), ((it / kMkFpStages) & 1) ^ 1);
      const uint32_t sa = base + s * stage, sb = sa + 16384;
#pragma unroll
      for (int j = 0; j < 8; ++j)
        asm volatile("st.shared.v4.f32 [%0], {%1, %2, %3, %4};" ::"r"(kmaj_addr(sa, t, j)), "f"(v[4 * j]),
                     "f"(v[4 * j + 1]), "f"(v[4 * j + 2]), "f"(v[4 * j + 3])
                     : "memory");
      // this K block of W (rows co < NB; co >= Cout and k >= KK are 0)
      for (int e = t; e < NB * 32; e += 128) {
        const int co = e >> 5, k = e & 31;
        const int kk = kb * 32 + k;
        const float wv = (co < g.Cout && kk < g.KK) ? __ldg(w + static_cast<int64_t>(co) * g.KK + kk) : 0.f;
        asm volatile("st.shared.f32 [%0], %1;" ::"r"(kmaj_addr(sb, co, k >> 2) + (k & 3) * 4), "f"(wv)
                     : "memory");
      }
      fence_proxy_async();
      mbar_arrive(full_bar(s));
    }
  } else if (warp == kMkMmaWarp) {
    // ---------------- MMA issuer (whole warp, one elected lane issues) ----------------
    const uint32_t idesc = make_idesc_tf32(NB, false, false);
    const bool leader = elect_one();
    int it = 0, lt = 0;
    for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x, ++lt) {
      const int acc = lt & 1;
      if (lt >= 2) mbar_wait(tempty_bar(acc), ((lt >> 1) & 1) ^ 1);
      tc_fence_after();
      for (int kb = 0; kb < KB; ++kb, ++it) {
        const int s = it % kMkFpStages;
        mbar_wait(full_bar(s), (it / kMkFpStages) & 1);
        tc_fence_after();
        const uint32_t sa = base + s * stage, sb = sa + 16384;
        if (leader) {
#pragma unroll
          for (int kk = 0; kk < kBK / 8; ++kk)
            tc_mma_tf32(tmem + acc * NBP, make_sdesc(sa + kk * 32, 16, 1024, kSw128),
                        make_sdesc(sb + kk * 32, 16, 1024, kSw128), idesc, (kb > 0 || kk > 0) ? 1u : 0u);
          tc_commit(empty_bar(s));
        }
        __syncwarp();
      }
      if (leader) tc_commit(tfull_bar(acc));
      __syncwarp();
    }
  } else {
    // ---------------- epilogue (as c3tc_fprop_kernel) ----------------
    const int row = warp * 32 + lane;
    int it = 0;
    for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x, ++it) {
      const int acc = it & 1;
      if (threadIdx.x == 0) asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
      const uint32_t ob = so + (it & 1) * obytes;
      asm volatile("bar.sync 1, 128;" ::: "memory");
      mbar_wait_sleep(tfull_bar(acc), (it >> 1) & 1);
      tc_fence_after();
      const uint32_t taddr = tmem + acc * NBP + (static_cast<uint32_t>(warp * 32) << 16);
      for (int cg = 0; cg < NB / 32; ++cg) {
        float v[32];
        tmem_ld32(taddr + cg * 32, v);
        if (relu) {
#pragma unroll
          for (int i = 0; i < 32; ++i) v[i] = fmaxf(v[i], 0.f);
        }
        const uint32_t rowaddr = ob + cg * 16384 + row * 128;
#pragma unroll
        for (int j = 0; j < 8; ++j)
          asm volatile("st.shared.v4.f32 [%0], {%1, %2, %3, %4};" ::"r"(rowaddr + (((j ^ (row & 7)) & 7) << 4)),
                       "f"(v[4 * j]), "f"(v[4 * j + 1]), "f"(v[4 * j + 2]), "f"(v[4 * j + 3])
                       : "memory");
      }
      tc_fence_before();
      mbar_arrive(tempty_bar(acc));
      fence_proxy_async();
      asm volatile("bar.sync 1, 128;" ::: "memory");
      if (threadIdx.x == 0) {
        for (int cg = 0; cg < NB / 32; ++cg)
          if (cg * 32 < g.Cout) tma_store_2d(&tma_y, ob + cg * 16384, cg * 32, tile * kBM, false);
        asm volatile("cp.async.bulk.commit_group;" ::: "memory");
      }
    }
    if (threadIdx.x == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
  }
  tc_fence_before();
  __syncthreads();
  if (warp == kMkMmaWarp) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(2 * NBP) : "memory");
  }
}

// ------------------------------------------------------ multi-K wgrad ------
// D[co][k] over all KB*32 im2col columns at once (N = KB*32 <= 384: two MMAs
// of N <= 256 per K step), 32 pixels per stage: A = dY^T by TMA (as the
// single-block kernel), B = KB MN-major chunks of im2col^T, one pixel row per
// builder lane for every K block.
constexpr int kMkWgStages = 3;
constexpr int kMkWgBuilders = 3;
__global__ void __launch_bounds__(kWgThreads, 1) c3tc_wgrad_mk_kernel(const float* __restrict__ x,
                                                                      const __grid_constant__ CUtensorMap tma_dy,
                                                                      C3Geom g, int ppb, int KB, int ncols,
                                                                      float* __restrict__ part) {
  extern __shared__ uint8_t smem_raw[];
  const uint32_t raw = smem_u32(smem_raw);
  const uint32_t base = (raw + 1023u) & ~1023u;
  const uint32_t stage = 16384 + static_cast<uint32_t>(KB) * 4096;
  const uint32_t bars = base + kMkWgStages * stage;
  auto full_bar = [&](int s) { return bars + 8u * s; };
  auto empty_bar = [&](int s) { return bars + 8u * (kMkWgStages + s); };
  const uint32_t done_bar = bars + 8u * (2 * kMkWgStages);
  const uint32_t tmem_slot = bars + 8u * (2 * kMkWgStages + 1);
  int* tab = reinterpret_cast<int*>(smem_raw + (bars + 8u * (2 * kMkWgStages + 2) - raw));

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int p_begin = blockIdx.x * ppb;
  const int p_end = min(p_begin + ppb, g.P);
  const int nkb = p_end > p_begin ? (p_end - p_begin + kBK - 1) / kBK : 0;
  const int nchunk = g.Cout / 32;
  const int n1 = KB * 32 <= 256 ? KB * 32 : 256, n2 = KB * 32 - n1;

  if (threadIdx.x == 0) {
    for (int s = 0; s < kMkWgStages; ++s) {
      mbar_init(full_bar(s), 33);
      mbar_init(empty_bar(s), 1);
    }
    mbar_init(done_bar, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  c3_table_mk(g, KB, tab, tab + kMkMaxKB * 32);
  const int zbytes = (4 - nchunk) * 4096;
  for (int s = 0; s < kMkWgStages; ++s)
    for (int o = threadIdx.x * 16; o < zbytes; o += blockDim.x * 16)
      asm volatile("st.shared.v4.u32 [%0], {%1, %1, %1, %1};" ::"r"(base + s * stage + nchunk * 4096 + o), "r"(0)
                   : "memory");
  fence_proxy_async();
  if (warp == 9) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(tmem_slot),
                 "r"(ncols)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  uint32_t tmem;
  asm volatile("ld.shared.u32 %0, [%1];" : "=r"(tmem) : "r"(tmem_slot) : "memory");
  const int* off = tab;
  const int* rs = tab + kMkMaxKB * 32;

  if (warp < 8) {
    // ---------------- builders: kMkWgBuilders warps, stage it by warp it % kMkWgBuilders ----------------
    // (a builder's consecutive stages must be <= kMkWgStages apart for the
    // parity waits on the ring to be unambiguous)
    for (int it = warp; warp < kMkWgBuilders && it < nkb; it += kMkWgBuilders) {
      const int s = it % kMkWgStages;
      const int m = p_begin + it * kBK + lane;
      const C3Pix q = c3_pix(g, m < p_end ? m : g.P);
      if (it >= kMkWgStages) mbar_wait(empty_bar(s), ((it / kMkWgStages) & 1) ^ 1);
      const uint32_t sbb = base + s * stage + 16384;
      for (int kb = 0; kb < KB; ++kb) {
        float v[32];
        c3_row_kb(x, g, off, rs, q, kb, v);
#pragma unroll
        for (int j = 0; j < 8; ++j)
          asm volatile("st.shared.v4.f32 [%0], {%1, %2, %3, %4};" ::"r"(mnmaj_addr(sbb, lane, kb, j)),
                       "f"(v[4 * j]), "f"(v[4 * j + 1]), "f"(v[4 * j + 2]), "f"(v[4 * j + 3])
                       : "memory");
      }
      fence_proxy_async();
      mbar_arrive(full_bar(s));
    }
    // ---------------- epilogue: warp w owns TMEM lanes 32w.. = co ----------------
    if (warp < nchunk) {
      mbar_wait_sleep(done_bar, 0);
      tc_fence_after();
      float* dst = part + (static_cast<int64_t>(blockIdx.x) * g.Cout + warp * 32 + lane) * g.KK;
      for (int cg = 0; cg < KB; ++cg) {
        float v[32];
        tmem_ld32(tmem + (static_cast<uint32_t>(warp * 32) << 16) + cg * 32, v);
        if (nkb <= 0) {
#pragma unroll
          for (int i = 0; i < 32; ++i) v[i] = 0.f;
        }
#pragma unroll
        for (int i = 0; i < 32; ++i)
          if (cg * 32 + i < g.KK) dst[cg * 32 + i] = v[i];
      }
    }
  } else if (warp == 8) {
    // ---------------- TMA producer (dY tiles) ----------------
    if (lane == 0) {
      asm volatile("prefetch.tensormap [%0];" ::"l"(&tma_dy) : "memory");
      for (int it = 0; it < nkb; ++it) {
        const int s = it % kMkWgStages;
        if (it + kPrefetch < nkb)
          asm volatile("cp.async.bulk.prefetch.tensor.3d.L2.global [%0, {%1, %2, %3}];" ::"l"(&tma_dy), "r"(0),
                       "r"(p_begin + (it + kPrefetch) * kBK), "r"(0)
                       : "memory");
        if (it >= kMkWgStages) mbar_wait(empty_bar(s), ((it / kMkWgStages) & 1) ^ 1);
        mbar_expect_tx(full_bar(s), static_cast<uint32_t>(nchunk * 4096));
        tma_load_3d(base + s * stage, &tma_dy, full_bar(s), 0, p_begin + it * kBK, 0);
      }
    }
    __syncwarp();
  } else {
    // ---------------- MMA issuer ----------------
    const uint32_t idesc1 = make_idesc_tf32(n1, true, true);
    const uint32_t idesc2 = make_idesc_tf32(n2 > 0 ? n2 : 16, true, true);
    const bool leader = elect_one();
    for (int it = 0; it < nkb; ++it) {
      const int s = it % kMkWgStages;
      mbar_wait(full_bar(s), (it / kMkWgStages) & 1);
      tc_fence_after();
      const uint32_t sa = base + s * stage;
      const uint32_t sbb = sa + 16384;
      if (leader) {
#pragma unroll
        for (int kk = 0; kk < kBK / 8; ++kk) {
          const uint64_t ad = make_sdesc(sa + kk * 1024, 4096, 512, kSw128Base32);
          tc_mma_tf32(tmem, ad, make_sdesc(sbb + kk * 1024, 4096, 512, kSw128Base32), idesc1,
                      (it > 0 || kk > 0) ? 1u : 0u);
          if (n2 > 0)
            tc_mma_tf32(tmem + n1, ad, make_sdesc(sbb + (n1 / 32) * 4096 + kk * 1024, 4096, 512, kSw128Base32),
                        idesc2, (it > 0 || kk > 0) ? 1u : 0u);
        }
        tc_commit(empty_bar(s));
      }
      __syncwarp();
    }
    if (leader) {
      if (nkb > 0)
        tc_commit(done_bar);
      else
        mbar_arrive(done_bar);
    }
    __syncwarp();
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 9) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(ncols) : "memory");
  }
}

C3Geom geom_of(const ConvArgs& a) {
  C3Geom g;
  g.N = a.n;
  g.H = a.h;
  g.W = a.w;
  g.C = a.c[0];
  g.Ho = a.ho();
  g.Wo = a.wo();
  g.Cout = a.cout;
  g.k = a.kh;
  g.stride = a.stride;
  g.pad = a.pad;
  g.KK = a.kh * a.kw * a.c[0];
  g.HoWo = g.Ho * g.Wo;
  g.P = a.n * g.HoWo;
  return g;
}

int pow2_at_least(int v) {
  int p = 32;
  while (p < v) p <<= 1;
  return p;
}

size_t fprop_smem(int NB) {
  return 1024 + static_cast<size_t>((NB * 128 + 1023) & ~1023) + kFpStages * 16384 + 2 * (NB / 32) * 16384 + 512;
}
size_t wgrad_smem() { return 1024 + static_cast<size_t>(kWgStages) * kWgStage + 512; }

int wgrad_blocks(const C3Geom& g) {
  // one CTA per SM, at least 256 pixel rows each
  return std::max(1, std::min(kSms, (g.P + 255) / 256));
}

bool c3_common(const ConvArgs& a) {
  const int64_t P = static_cast<int64_t>(a.n) * a.ho() * a.wo();
  const int64_t X = static_cast<int64_t>(a.n) * a.h * a.w * a.c[0];
  return !precise() && a.nseg == 1 && a.c[0] <= 4 && a.kh == a.kw && a.kh * a.kw * a.c[0] <= 32 * kMkMaxKB &&
         P > 0 && P < (int64_t{1} << 31) - kBM && X < (int64_t{1} << 40);
}
int kblocks_of(const ConvArgs& a) { return (a.kh * a.kw * a.c[0] + 31) / 32; }
size_t fprop_mk_smem(int NB) {
  const size_t bbytes = (static_cast<size_t>(NB) * 128 + 1023) & ~size_t{1023};
  return 1024 + kMkFpStages * (16384 + bbytes) + 2 * (NB / 32) * 16384 + 8 * (2 * kMkFpStages + 6) +
         2 * kMkMaxKB * 32 * sizeof(int) + 64;
}
size_t wgrad_mk_smem(int KB) {
  return 1024 + kMkWgStages * (16384 + static_cast<size_t>(KB) * 4096) + 8 * (2 * kMkWgStages + 2) +
         2 * kMkMaxKB * 32 * sizeof(int) + 64;
}

}  // namespace

// TF32 tensor-core eligibility (precise mode stays on the exact SIMT kernels).
bool c3tc_fprop_eligible(const ConvArgs& a) {
  // multi-K blocks stream W through the ring: up to 96 output channels fit
  return c3_common(a) && a.cout % 4 == 0 && a.cout <= (kblocks_of(a) > 1 ? 96 : 128);
}
bool c3tc_wgrad_eligible(const ConvArgs& a) { return c3_common(a) && a.cout % 32 == 0 && a.cout <= 128; }
size_t c3tc_wgrad_ws_bytes(const ConvArgs& a) {
  const C3Geom g = geom_of(a);
  return static_cast<size_t>(wgrad_blocks(g)) * g.Cout * g.KK * sizeof(float);
}

cudaError_t c3tc_fprop(const ConvArgs& a, const float* w, float* y, cudaStream_t st) {
  const C3Geom g = geom_of(a);
  if (g.P <= 0) return cudaSuccess;
  const int NB = (g.Cout + 31) / 32 * 32, NBP = pow2_at_least(NB);
  alignas(64) CUtensorMap ty;
  if (!encode_out(&ty, y, g.P, g.Cout)) return cudaErrorInvalidValue;
  const int KB = kblocks_of(a);
  if (KB > 1) {
    const size_t smem = fprop_mk_smem(NB);
    static size_t attr_mk = 0;
    if (smem > attr_mk) {
      cudaError_t e = cudaFuncSetAttribute(c3tc_fprop_mk_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                           static_cast<int>(smem));
      if (e != cudaSuccess) return e;
      attr_mk = smem;
    }
    const int ntiles = (g.P + kBM - 1) / kBM;
    c3tc_fprop_mk_kernel<<<std::min(kSms, ntiles), kFpMkThreads, smem, st>>>(a.x[0], w, ty, g, NB, NBP, KB,
                                                                            a.relu_out);
    count_launch();
    return cudaGetLastError();
  }
  const size_t smem = fprop_smem(NB);
  const bool k3c3 = g.k == 3 && g.C == 3;
  auto kern = k3c3 ? c3tc_fprop_kernel<3, 3> : c3tc_fprop_kernel<0, 0>;
  static size_t attr[2] = {0, 0};
  if (smem > attr[k3c3]) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
    if (e != cudaSuccess) return e;
    attr[k3c3] = smem;
  }
  const int ntiles = (g.P + kBM - 1) / kBM;
  const int grid = std::min(kSms, ntiles);
  kern<<<grid, kFpThreads, smem, st>>>(a.x[0], w, ty, g, NB, NBP, a.relu_out);
  count_launch();
  return cudaGetLastError();
}

cudaError_t c3tc_wgrad(const ConvArgs& a, const float* dy, float* w, float lr, float* dw_out, float* ws,
                       size_t ws_bytes, cudaStream_t st) {
  const C3Geom g = geom_of(a);
  const size_t per = static_cast<size_t>(g.Cout) * g.KK * sizeof(float);
  int nb = wgrad_blocks(g);
  if (ws == nullptr || ws_bytes < per) return cudaErrorInvalidValue;
  nb = static_cast<int>(std::min<size_t>(nb, ws_bytes / per));
  int ppb = (g.P + nb - 1) / nb;
  ppb = (ppb + kBK - 1) / kBK * kBK;
  nb = static_cast<int>((g.P + ppb - 1) / ppb);
  // dY [P][Cout] as (32 co, pixel, co-chunk): one 32-pixel x NB box per stage, MN-major chunks
  alignas(64) CUtensorMap tdy;
  const cuuint64_t d3[3] = {32, static_cast<cuuint64_t>(g.P), static_cast<cuuint64_t>(g.Cout / 32)};
  const cuuint64_t s3[2] = {static_cast<cuuint64_t>(g.Cout) * 4, 128};
  const cuuint32_t b3[3] = {32, 32, static_cast<cuuint32_t>(g.Cout / 32)};
  if (!encode_tiled(&tdy, dy, 3, d3, s3, b3, CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B)) return cudaErrorInvalidValue;
  const size_t smem = wgrad_smem();
  const bool k3c3 = g.k == 3 && g.C == 3;
  auto kern = k3c3 ? c3tc_wgrad_kernel<3, 3> : c3tc_wgrad_kernel<0, 0>;
  static size_t attr[2] = {0, 0};
  if (smem > attr[k3c3]) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
    if (e != cudaSuccess) return e;
    attr[k3c3] = smem;
  }
  const int KB = kblocks_of(a);
  if (KB > 1) {
    const size_t smk = wgrad_mk_smem(KB);
    static size_t attr_mk = 0;
    if (smk > attr_mk) {
      cudaError_t e = cudaFuncSetAttribute(c3tc_wgrad_mk_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                           static_cast<int>(smk));
      if (e != cudaSuccess) return e;
      attr_mk = smk;
    }
    c3tc_wgrad_mk_kernel<<<nb, kWgThreads, smk, st>>>(a.x[0], tdy, g, ppb, KB, pow2_at_least(KB * 32), ws);
  } else {
    static const int pf = [] {  // VDNN_C3_PREFETCH: dY stages prefetched into L2 ahead of the ring (A/B)
      const char* e = std::getenv("VDNN_C3_PREFETCH");
      return e ? std::atoi(e) : kPrefetch;
    }();
    kern<<<nb, kWgThreads, smem, st>>>(a.x[0], tdy, g, ppb, pf, ws);
  }
  count_launch();
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  return smallc_wgrad_reduce_launch(ws, nb, static_cast<int64_t>(g.Cout) * g.KK, w, lr, dw_out, st);
}

}  // namespace vdnnk
