// First-layer convolutions of the BF16 engine on the tensor cores: few input
// channels (the raw image, C = 3) and a whole filter window that fits one
// 64-wide bf16 K block (kh*kw*C <= 64, e.g. VGG's 3x3x3 = 27). A pixel's
// im2col row is 27 bf16 at a 6-byte pixel stride -- no TMA box or 16-B
// gather can address it -- so builder threads assemble the operand rows from
// 2-byte loads and the tensor core does the contraction; both kernels are
// then bound by their one big HBM stream (Y written / dY read), the same
// split of work as the TF32 kernels of conv_c3tc.cu at half the bytes.
//
//   fprop  Y[p][co] = relu?( sum_k A[p][k] * W[co][k] ),  A[p][k] = im2col(X)
//          persistent CTAs over 128-pixel tiles: 8 builder warps (two groups
//          taking alternate tiles, one pixel row per thread) write 128-byte
//          A rows (K-major SWIZZLE_128B) into a 4-stage ring; one thread
//          issues ceil(KK/16) x tcgen05.mma kind::f16 (M = 128, N = Cout,
//          K = 16) into one of two TMEM accumulators; 4 epilogue warps drain
//          TMEM -> ReLU -> bf16 (RNE) -> swizzled smem -> TMA store of
//          64-channel boxes, overlapping the next tiles' build and MMAs.
//   wgrad  dW[co][k] = sum_p dY[p][co] * A[p][k]
//          D[co][k] (M = 128 rows, co < Cout live; N = 64 = k) accumulates
//          over a contiguous pixel range per CTA, 64 pixels per stage: dY
//          arrives by TMA as MN-major 64 x 64 boxes (one per 64 output
//          channels), eight builder warps each write the im2col^T rows of
//          every eighth stage (MN-major SWIZZLE_128B, two pixels per lane);
//          per-CTA fp32 partials are reduced in a fixed order (deterministic,
//          independent of the plan) with the bf16 SGD update or the fp32 dW.
// Numerics are the BF16 engine's (tcb_conv.cuh): exact bf16 products, fp32
// accumulation, one rounding per stored value.
#include <algorithm>
#include <cstdlib>

#include "kernels.h"
#include "tcb_conv.cuh"
#include "tma_maps.h"

namespace vdnnk {

namespace {

constexpr int kSmsC3 = 148;
constexpr int kFbStages = 8;
constexpr int kWbStages = 8;
constexpr int kWbPrefetch = 16;  // wgrad: dY stages prefetched into L2 ahead of the ring
constexpr int kKb = 64;          // bf16 per K block (one 128-B operand row)

struct C3B {
  int N, H, W, C, Ho, Wo, Cout, k, stride, pad, KK;
  int P, HoWo;  // output pixels (host checks P < 2^31 - 128)
};

// Window table (shared memory): element offset of im2col column i relative to
// the window's top-left input element, and its tap (r, s) for clipping.
__device__ __forceinline__ void c3b_table(const C3B& g, int* off, int* rs) {
  for (int i = threadIdx.x; i < kKb; i += blockDim.x) {
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

// im2col row of output pixel m as 32 packed bf16 pairs (columns >= KK and
// padding -> 0).
__device__ __forceinline__ void c3b_row(const uint16_t* __restrict__ x, const C3B& g, const int* off, const int* rs,
                                        int m, uint32_t (&u)[32]) {
#pragma unroll
  for (int i = 0; i < 32; ++i) u[i] = 0u;
  if (m >= g.P) return;
  const int n = m / g.HoWo;
  const int rem = m - n * g.HoWo;
  const int oh = rem / g.Wo, ow = rem - oh * g.Wo;
  const int ih0 = oh * g.stride - g.pad, iw0 = ow * g.stride - g.pad;
  const int64_t base = ((static_cast<int64_t>(n) * g.H + ih0) * g.W + iw0) * g.C;
  const uint16_t* xb = x + base;
  if (ih0 >= 0 && ih0 + g.k <= g.H && iw0 >= 0 && iw0 + g.k <= g.W) {
#pragma unroll
    for (int i = 0; i < kKb; ++i)
      if (i < g.KK) u[i >> 1] |= static_cast<uint32_t>(__ldg(xb + off[i])) << ((i & 1) * 16);
  } else {
#pragma unroll
    for (int i = 0; i < kKb; ++i) {
      if (i < g.KK) {
        const int ih = ih0 + (rs[i] & 0xff), iw = iw0 + (rs[i] >> 8);
        if (ih >= 0 && ih < g.H && iw >= 0 && iw < g.W)
          u[i >> 1] |= static_cast<uint32_t>(__ldg(xb + off[i])) << ((i & 1) * 16);
      }
    }
  }
}

// Compile-time window (KT x KT taps of CT channels, e.g. VGG's 3 x 3 x 3):
// the 27 loads sit at constant offsets from three row pointers, clipping is
// two 3-bit masks, no table and no per-element address arithmetic.
// KT = 0: the table-driven row above (any window with kh*kw*C <= 64).
template <int KT, int CT>
__device__ __forceinline__ void c3b_row_t(const uint16_t* __restrict__ x, const C3B& g, const int* off, const int* rs,
                                          int m, uint32_t (&u)[32]) {
  if constexpr (KT == 0) {
    c3b_row(x, g, off, rs, m, u);
  } else {
    static_assert(KT * KT * CT <= kKb, "window must fit one K block");
#pragma unroll
    for (int i = 0; i < 32; ++i) u[i] = 0u;
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
    const uint16_t* x0 = x + ((static_cast<int64_t>(n) * g.H + ih0) * g.W + iw0) * CT;
    const int64_t rstride = static_cast<int64_t>(g.W) * CT;
    const bool full = rmask == (1u << KT) - 1 && cmask == (1u << KT) - 1;
#pragma unroll
    for (int r = 0; r < KT; ++r) {
      const uint16_t* xr = x0 + r * rstride;
#pragma unroll
      for (int s = 0; s < KT; ++s) {
#pragma unroll
        for (int c = 0; c < CT; ++c) {
          const int i = (r * KT + s) * CT + c;
          if (full || (((rmask >> r) & (cmask >> s)) & 1u))
            u[i >> 1] |= static_cast<uint32_t>(__ldg(xr + s * CT + c)) << ((i & 1) * 16);
        }
      }
    }
  }
}

__device__ __forceinline__ void st_shared_v4(uint32_t addr, uint32_t a, uint32_t b, uint32_t c, uint32_t d) {
  asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(addr), "r"(a), "r"(b), "r"(c), "r"(d) : "memory");
}

// ------------------------------------------------------------ fprop ------
// smem: [B: NB rows x 128 B][A: kFbStages x 16 KB][OUT: 2 x NG x 16 KB][barriers][table]
// (NG = 64-channel output groups). warps 0-3 epilogue, 4-11 builders, 12 MMA
// (+ TMEM owner). TMEM: 2 x NBP columns.
// kFbGroups builder groups of 4 warps take alternate tiles (stage spacing
// kFbGroups <= ring depth): the builders are latency-bound (27 loads per row,
// then one stage), so more groups keep more tiles' loads in flight.
constexpr int kFbGroups = 4;
constexpr int kFbMmaWarp = 4 + 4 * kFbGroups;
constexpr int kFbThreads = 32 * (kFbMmaWarp + 1);
constexpr int kFbmThreads = 416;  // the multi-K kernel: 2 groups, MMA warp 12
static_assert(kFbGroups <= kFbStages, "builder spacing must fit the ring");
template <int KT, int CT>
__global__ void __launch_bounds__(kFbThreads, 1) c3b_fprop_kernel(const uint16_t* __restrict__ x,
                                                                  const uint16_t* __restrict__ w,
                                                                  const __grid_constant__ CUtensorMap tma_y, C3B g,
                                                                  int NB, int NBP, int relu) {
  extern __shared__ uint8_t smem_raw[];
  const uint32_t raw = smem_u32(smem_raw);
  const uint32_t base = (raw + 1023u) & ~1023u;
  const uint32_t sb = base;
  const uint32_t sa0 = sb + ((NB * 128 + 1023) & ~1023);
  const uint32_t so = sa0 + kFbStages * 16384;
  const int NG = (NB + 63) / 64;
  const uint32_t obytes = NG * 16384;  // one output staging buffer (double-buffered)
  const uint32_t bars = so + 2 * obytes;
  auto full_bar = [&](int s) { return bars + 8u * s; };
  auto empty_bar = [&](int s) { return bars + 8u * (kFbStages + s); };
  auto tfull_bar = [&](int a) { return bars + 8u * (2 * kFbStages + a); };
  auto tempty_bar = [&](int a) { return bars + 8u * (2 * kFbStages + 2 + a); };
  const uint32_t tmem_slot = bars + 8u * (2 * kFbStages + 4);
  int* tab = reinterpret_cast<int*>(smem_raw + (bars + 8u * (2 * kFbStages + 6) - raw));

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int ntiles = (g.P + kBM - 1) / kBM;

  if (threadIdx.x == 0) {
    for (int s = 0; s < kFbStages; ++s) {
      mbar_init(full_bar(s), 128);
      mbar_init(empty_bar(s), 1);
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(tfull_bar(a), 1);
      mbar_init(tempty_bar(a), 128);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  c3b_table(g, tab, tab + kKb);
  // weights -> B (row co, K-major swizzled; rows >= Cout and k >= KK are 0)
  for (int i = threadIdx.x; i < NB * 8; i += blockDim.x) {
    const int co = i >> 3, j = i & 7;
    uint32_t q[4];
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      const int k0 = j * 8 + 2 * e;
      const uint32_t lo = (co < g.Cout && k0 < g.KK) ? w[static_cast<int64_t>(co) * g.KK + k0] : 0u;
      const uint32_t hi = (co < g.Cout && k0 + 1 < g.KK) ? w[static_cast<int64_t>(co) * g.KK + k0 + 1] : 0u;
      q[e] = lo | (hi << 16);
    }
    st_shared_v4(kmaj_addr(sb, co, j), q[0], q[1], q[2], q[3]);
  }
  fence_proxy_async();
  if (warp == kFbMmaWarp) {
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

  if (warp >= 4 && warp < kFbMmaWarp) {
    // ---------------- builders ----------------
    const int grp = (warp - 4) >> 2;
    const int row = (threadIdx.x - 128) & 127;
    int it = grp;
    // software-pipelined: the next tile's loads are in flight while this
    // tile's row waits for its stage and is stored
    uint32_t u[32], nu[32];
    const int tile0 = blockIdx.x + grp * gridDim.x;
    if (tile0 < ntiles) c3b_row_t<KT, CT>(x, g, tab, tab + kKb, tile0 * kBM + row, u);
    for (int tile = tile0; tile < ntiles; tile += kFbGroups * gridDim.x, it += kFbGroups) {
      const int s = it % kFbStages;
      const int nt = tile + kFbGroups * gridDim.x;
      if (nt < ntiles) c3b_row_t<KT, CT>(x, g, tab, tab + kKb, nt * kBM + row, nu);
      if (it >= kFbStages) mbar_wait(empty_bar(s), ((it / kFbStages) & 1) ^ 1);
      const uint32_t sa = sa0 + s * 16384;
#pragma unroll
      for (int j = 0; j < 8; ++j) st_shared_v4(kmaj_addr(sa, row, j), u[4 * j], u[4 * j + 1], u[4 * j + 2], u[4 * j + 3]);
      fence_proxy_async();
      mbar_arrive(full_bar(s));
#pragma unroll
      for (int i = 0; i < 32; ++i) u[i] = nu[i];
    }
  } else if (warp == kFbMmaWarp) {
    // ---------------- MMA issuer ----------------
    // whole warp in the loop, one elected lane issues; descriptors advanced
    // by constants, running stage / phase counters (see c3b_wgrad_kernel)
    const uint32_t idesc = make_idesc_bf16(NB, false, false);
    const int nk = (g.KK + 15) / 16;  // K = 16 steps that hold live columns
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
        for (int kk = 0; kk < nk; ++kk)
          tc_mma_bf16(tmem + acc * NBP, ad + kk * 2, bd + kk * 2, idesc, kk > 0 ? 1u : 0u);
        tc_commit(empty_bar(s));
        tc_commit(tfull_bar(acc));
      }
      __syncwarp();
      if (++s == kFbStages) {
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
        // 32 channels = 4 granules of the group's 128-byte row
        const uint32_t rowaddr = ob + (cg >> 1) * 16384 + row * 128;
#pragma unroll
        for (int jj = 0; jj < 4; ++jj) {
          const int j = (cg & 1) * 4 + jj;
          st_shared_v4(rowaddr + (((j ^ (row & 7)) & 7) << 4), pack_bf16x2(v[8 * jj], v[8 * jj + 1]),
                       pack_bf16x2(v[8 * jj + 2], v[8 * jj + 3]), pack_bf16x2(v[8 * jj + 4], v[8 * jj + 5]),
                       pack_bf16x2(v[8 * jj + 6], v[8 * jj + 7]));
        }
      }
      tc_fence_before();
      mbar_arrive(tempty_bar(acc));
      fence_proxy_async();
      asm volatile("bar.sync 1, 128;" ::: "memory");
      if (threadIdx.x == 0) {
        for (int gi = 0; gi < NG; ++gi) tma_store_2d(&tma_y, ob + gi * 16384, gi * 64, tile * kBM, false);
        asm volatile("cp.async.bulk.commit_group;" ::: "memory");
      }
    }
    if (threadIdx.x == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
  }
  tc_fence_before();
  __syncthreads();
  if (warp == kFbMmaWarp) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(2 * NBP) : "memory");
  }
}

// ------------------------------------------------------------ wgrad ------
// D[co][k] (M = 128 rows, co < Cout <= 128 live; N = 64 columns = k).
// smem per stage: [A = dY^T: 2 MN-chunks x 8 KB by one TMA (chunks >= Cout/64 stay 0)]
//                 [B = im2col^T: 1 MN-chunk x 8 KB, two pixel rows per builder lane]
// warps 0-7 builders (warp w builds stages it = w mod 8; warps < Cout/32 then
// drain TMEM), warp 8 lane 0 TMA, warp 9 MMA + TMEM.
constexpr int kWbThreads = 320;
constexpr uint32_t kWbStage = 16384 + 8192;
template <int KT, int CT>
__global__ void __launch_bounds__(kWbThreads, 1) c3b_wgrad_kernel(const uint16_t* __restrict__ x,
                                                                  const __grid_constant__ CUtensorMap tma_dy, C3B g,
                                                                  int ppb, int pf, float* __restrict__ part) {
  extern __shared__ uint8_t smem_raw[];
  const uint32_t raw = smem_u32(smem_raw);
  const uint32_t base = (raw + 1023u) & ~1023u;
  const uint32_t bars = base + kWbStages * kWbStage;
  auto full_bar = [&](int s) { return bars + 8u * s; };
  auto empty_bar = [&](int s) { return bars + 8u * (kWbStages + s); };
  const uint32_t done_bar = bars + 8u * (2 * kWbStages);
  const uint32_t tmem_slot = bars + 8u * (2 * kWbStages + 1);
  int* tab = reinterpret_cast<int*>(smem_raw + (bars + 8u * (2 * kWbStages + 2) - raw));

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int p_begin = blockIdx.x * ppb;
  const int p_end = min(p_begin + ppb, g.P);
  const int nkb = p_end > p_begin ? (p_end - p_begin + kKb - 1) / kKb : 0;
  const int nchunk = g.Cout / 64;

  if (threadIdx.x == 0) {
    for (int s = 0; s < kWbStages; ++s) {
      mbar_init(full_bar(s), 33);  // the building warp's 32 lanes + the TMA thread's expect_tx arrival
      mbar_init(empty_bar(s), 1);
    }
    mbar_init(done_bar, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  c3b_table(g, tab, tab + kKb);
  // A chunks >= Cout/64 (M rows the TMA never writes) are zero in every stage
  const int zbytes = (2 - nchunk) * 8192;
  for (int s = 0; s < kWbStages; ++s)
    for (int o = threadIdx.x * 16; o < zbytes; o += blockDim.x * 16)
      st_shared_v4(base + s * kWbStage + nchunk * 8192 + o, 0u, 0u, 0u, 0u);
  fence_proxy_async();
  if (warp == 9) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(tmem_slot), "r"(64)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  uint32_t tmem;
  asm volatile("ld.shared.u32 %0, [%1];" : "=r"(tmem) : "r"(tmem_slot) : "memory");

  if (warp < 8) {
    // ---------------- builders: lane builds pixel rows lane and lane + 32 ----------------
    // software-pipelined: stage it + 8's loads are in flight while stage it
    // waits for its slot and is stored
    auto pix = [&](int i, int half) {
      const int m = p_begin + i * kKb + half * 32 + lane;
      return m < p_end ? m : g.P;
    };
    uint32_t u0[32], u1[32], n0[32], n1[32];
    if (warp < nkb) {
      c3b_row_t<KT, CT>(x, g, tab, tab + kKb, pix(warp, 0), u0);
      c3b_row_t<KT, CT>(x, g, tab, tab + kKb, pix(warp, 1), u1);
    }
    for (int it = warp; it < nkb; it += 8) {
      const int s = it % kWbStages;
      if (it + 8 < nkb) {
        c3b_row_t<KT, CT>(x, g, tab, tab + kKb, pix(it + 8, 0), n0);
        c3b_row_t<KT, CT>(x, g, tab, tab + kKb, pix(it + 8, 1), n1);
      }
      if (it >= kWbStages) mbar_wait(empty_bar(s), ((it / kWbStages) & 1) ^ 1);
      const uint32_t sbb = base + s * kWbStage + 16384;
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        st_shared_v4(mnb_addr(sbb, lane, 0, j), u0[4 * j], u0[4 * j + 1], u0[4 * j + 2], u0[4 * j + 3]);
        st_shared_v4(mnb_addr(sbb, lane + 32, 0, j), u1[4 * j], u1[4 * j + 1], u1[4 * j + 2], u1[4 * j + 3]);
      }
      fence_proxy_async();
      mbar_arrive(full_bar(s));
#pragma unroll
      for (int i = 0; i < 32; ++i) {
        u0[i] = n0[i];
        u1[i] = n1[i];
      }
    }
    // ---------------- epilogue: warp w owns TMEM lanes 32w.. = co ----------------
    if (warp < g.Cout / 32) {
      mbar_wait_sleep(done_bar, 0);
      tc_fence_after();
      float* dst = part + (static_cast<int64_t>(blockIdx.x) * g.Cout + warp * 32 + lane) * g.KK;
#pragma unroll 1
      for (int cg = 0; cg < 2; ++cg) {
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
        const int s = it % kWbStages;
        // warm L2 with the tile `pf` stages ahead: the ring's loads then hit L2
        if (pf > 0 && it + pf < nkb)
          asm volatile("cp.async.bulk.prefetch.tensor.3d.L2.global [%0, {%1, %2, %3}];" ::"l"(&tma_dy), "r"(0),
                       "r"(p_begin + (it + pf) * kKb), "r"(0)
                       : "memory");
        if (it >= kWbStages) mbar_wait(empty_bar(s), ((it / kWbStages) & 1) ^ 1);
        mbar_expect_tx(full_bar(s), static_cast<uint32_t>(nchunk * 8192));
        tma_load_3d(base + s * kWbStage, &tma_dy, full_bar(s), 0, p_begin + it * kKb, 0);
      }
    }
    __syncwarp();
  } else {
    // ---------------- MMA issuer ----------------
    // (as c3tc_wgrad_kernel: descriptors built once and advanced by
    // constants, running stage / phase counters, whole warp + elected lane --
    // the short N = 64 MMAs leave the issue loop as the limiter otherwise)
    const uint32_t idesc = make_idesc_bf16(64, true, true);
    const bool leader = elect_one();
    const uint64_t ad0 = make_sdesc(base, 8192, 1024, kSw128);
    const uint64_t bd0 = make_sdesc(base + 16384, 8192, 1024, kSw128);
    constexpr uint64_t kStageLo = kWbStage >> 4, kKkLo = 2048 >> 4;
    int s = 0;
    uint32_t ph = 0;
    for (int it = 0; it < nkb; ++it) {
      mbar_wait(full_bar(s), ph);
      tc_fence_after();
      if (leader) {
        const uint64_t so = static_cast<uint64_t>(s) * kStageLo;
        const uint64_t ad = ad0 + so, bd = bd0 + so;
        tc_mma_bf16(tmem, ad, bd, idesc, it > 0 ? 1u : 0u);
#pragma unroll
        for (int kk = 1; kk < kKb / 16; ++kk) tc_mma_bf16(tmem, ad + kk * kKkLo, bd + kk * kKkLo, idesc, 1u);
        tc_commit(empty_bar(s));
      }
      __syncwarp();
      if (++s == kWbStages) {
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
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(64) : "memory");
  }
}

// ------------------------------------------------------ multi-K fprop ------
// Windows past one K block (AlexNet / OverFeat 11x11x3 = 363 = 6 K blocks of
// 64): same warp roles as c3b_fprop_kernel, a tile is KB stages (one per K
// block), W stays resident (KB x NB rows x 128 B: 72 KB at 96 channels).
// Builder groups take stages round-robin (stage it -> group it % 2) so a
// group's consecutive stages are 2 <= ring depth apart (parity waits stay
// unambiguous; alternating whole tiles would put them KB stages apart).
constexpr int kMkMaxKB = 6;
constexpr int kFbmStages = 4;
__device__ __forceinline__ void c3b_table_mk(const C3B& g, int kbn, int* off, int* rs) {
  for (int i = threadIdx.x; i < kbn * kKb; i += blockDim.x) {
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
struct C3BPix {
  int64_t base;
  int ih0, iw0;
  bool valid, interior;
};
__device__ __forceinline__ C3BPix c3b_pix(const C3B& g, int m) {
  C3BPix q;
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
// the 64 im2col values of K block kb for pixel q, packed in bf16 pairs
__device__ __forceinline__ void c3b_row_kb(const uint16_t* __restrict__ x, const C3B& g, const int* off, const int* rs,
                                           const C3BPix& q, int kb, uint32_t (&u)[32]) {
#pragma unroll
  for (int i = 0; i < 32; ++i) u[i] = 0u;
  if (!q.valid) return;
  const int k0 = kb * kKb;
  const uint16_t* xb = x + q.base;
  if (q.interior) {
#pragma unroll
    for (int i = 0; i < kKb; ++i)
      if (k0 + i < g.KK) u[i >> 1] |= static_cast<uint32_t>(__ldg(xb + off[k0 + i])) << ((i & 1) * 16);
  } else {
#pragma unroll
    for (int i = 0; i < kKb; ++i) {
      if (k0 + i < g.KK) {
        const int t = rs[k0 + i];
        const int ih = q.ih0 + (t & 0xff), iw = q.iw0 + (t >> 8);
        if (ih >= 0 && ih < g.H && iw >= 0 && iw < g.W)
          u[i >> 1] |= static_cast<uint32_t>(__ldg(xb + off[k0 + i])) << ((i & 1) * 16);
      }
    }
  }
}

__global__ void __launch_bounds__(kFbmThreads, 1) c3b_fprop_mk_kernel(const uint16_t* __restrict__ x,
                                                                     const uint16_t* __restrict__ w,
                                                                     const __grid_constant__ CUtensorMap tma_y, C3B g,
                                                                     int NB, int NBP, int KB, int relu) {
  extern __shared__ uint8_t smem_raw[];
  const uint32_t raw = smem_u32(smem_raw);
  const uint32_t base = (raw + 1023u) & ~1023u;
  const uint32_t bblk = (static_cast<uint32_t>(NB) * 128 + 1023u) & ~1023u;  // one K block of W
  const uint32_t sb = base;
  const uint32_t sa0 = sb + KB * bblk;
  const uint32_t so = sa0 + kFbmStages * 16384;
  const int NG = (NB + 63) / 64;
  const uint32_t obytes = NG * 16384;
  const uint32_t bars = so + 2 * obytes;
  auto full_bar = [&](int s) { return bars + 8u * s; };
  auto empty_bar = [&](int s) { return bars + 8u * (kFbmStages + s); };
  auto tfull_bar = [&](int a) { return bars + 8u * (2 * kFbmStages + a); };
  auto tempty_bar = [&](int a) { return bars + 8u * (2 * kFbmStages + 2 + a); };
  const uint32_t tmem_slot = bars + 8u * (2 * kFbmStages + 4);
  int* tab = reinterpret_cast<int*>(smem_raw + (bars + 8u * (2 * kFbmStages + 6) - raw));
  const int* off = tab;
  const int* rs = tab + kMkMaxKB * kKb;

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int ntiles = (g.P + kBM - 1) / kBM;

  if (threadIdx.x == 0) {
    for (int s = 0; s < kFbmStages; ++s) {
      mbar_init(full_bar(s), 128);
      mbar_init(empty_bar(s), 1);
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(tfull_bar(a), 1);
      mbar_init(tempty_bar(a), 128);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  c3b_table_mk(g, KB, tab, tab + kMkMaxKB * kKb);
  // W -> KB resident K-major blocks (rows >= Cout and k >= KK are 0)
  for (int i = threadIdx.x; i < KB * NB * 8; i += blockDim.x) {
    const int kb = i / (NB * 8), r = i - kb * NB * 8;
    const int co = r >> 3, j = r & 7;
    uint32_t q[4];
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      const int k0 = kb * kKb + j * 8 + 2 * e;
      const uint32_t lo = (co < g.Cout && k0 < g.KK) ? w[static_cast<int64_t>(co) * g.KK + k0] : 0u;
      const uint32_t hi = (co < g.Cout && k0 + 1 < g.KK) ? w[static_cast<int64_t>(co) * g.KK + k0 + 1] : 0u;
      q[e] = lo | (hi << 16);
    }
    st_shared_v4(kmaj_addr(sb + kb * bblk, co, j), q[0], q[1], q[2], q[3]);
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
    // ---------------- builders: 2 groups take stages round-robin ----------------
    const int grp = (warp - 4) >> 2;
    const int t = (threadIdx.x - 128) & 127;
    int cur_tl = -1;
    C3BPix q{};
    const int total = ((ntiles - static_cast<int>(blockIdx.x) + static_cast<int>(gridDim.x) - 1) /
                       static_cast<int>(gridDim.x)) * KB;
    for (int it = grp; it < total; it += 2) {
      const int tl = it / KB, kb = it - tl * KB;
      if (tl != cur_tl) {
        cur_tl = tl;
        q = c3b_pix(g, (static_cast<int>(blockIdx.x) + tl * static_cast<int>(gridDim.x)) * kBM + t);
      }
      const int s = it % kFbmStages;
      uint32_t u[32];
      c3b_row_kb(x, g, off, rs, q, kb, u);  // loads in flight while the stage drains
      if (it >= kFbmStages) mbar_wait(empty_bar(s), ((it / kFbmStages) & 1) ^ 1);
      const uint32_t sa = sa0 + s * 16384;
#pragma unroll
      for (int j = 0; j < 8; ++j) st_shared_v4(kmaj_addr(sa, t, j), u[4 * j], u[4 * j + 1], u[4 * j + 2], u[4 * j + 3]);
      fence_proxy_async();
      mbar_arrive(full_bar(s));
    }
  } else if (warp == 12) {
    // ---------------- MMA issuer ----------------
    const uint32_t idesc = make_idesc_bf16(NB, false, false);
    const bool leader = elect_one();
    int it = 0, lt = 0;
    for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x, ++lt) {
      const int acc = lt & 1;
      if (lt >= 2) mbar_wait(tempty_bar(acc), ((lt >> 1) & 1) ^ 1);
      tc_fence_after();
      for (int kb = 0; kb < KB; ++kb, ++it) {
        const int s = it % kFbmStages;
        mbar_wait(full_bar(s), (it / kFbmStages) & 1);
        tc_fence_after();
        const uint32_t sa = sa0 + s * 16384;
        if (leader) {
#pragma unroll
          for (int kk = 0; kk < kKb / 16; ++kk)
            tc_mma_bf16(tmem + acc * NBP, make_sdesc(sa + kk * 32, 16, 1024, kSw128),
                        make_sdesc(sb + kb * bblk + kk * 32, 16, 1024, kSw128), idesc, (kb > 0 || kk > 0) ? 1u : 0u);
          tc_commit(empty_bar(s));
        }
        __syncwarp();
      }
      if (leader) tc_commit(tfull_bar(acc));
      __syncwarp();
    }
  } else {
    // ---------------- epilogue (as c3b_fprop_kernel) ----------------
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
        const uint32_t rowaddr = ob + (cg >> 1) * 16384 + row * 128;
#pragma unroll
        for (int jj = 0; jj < 4; ++jj) {
          const int j = (cg & 1) * 4 + jj;
          st_shared_v4(rowaddr + (((j ^ (row & 7)) & 7) << 4), pack_bf16x2(v[8 * jj], v[8 * jj + 1]),
                       pack_bf16x2(v[8 * jj + 2], v[8 * jj + 3]), pack_bf16x2(v[8 * jj + 4], v[8 * jj + 5]),
                       pack_bf16x2(v[8 * jj + 6], v[8 * jj + 7]));
        }
      }
      tc_fence_before();
      mbar_arrive(tempty_bar(acc));
      fence_proxy_async();
      asm volatile("bar.sync 1, 128;" ::: "memory");
      if (threadIdx.x == 0) {
        for (int gi = 0; gi < NG; ++gi) tma_store_2d(&tma_y, ob + gi * 16384, gi * 64, tile * kBM, false);
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

// ------------------------------------------------------ multi-K wgrad ------
// D[co][k] over all KB*64 im2col columns at once (N = KB*64 <= 384: MMAs of
// N <= 256 and the rest), 64 pixels per stage: A = dY^T (two 64-co MN-major
// chunks by two 2D TMA boxes; channels past Cout are zero fill), B = KB
// MN-major chunks of im2col^T built by a warp pair per stage (warp h of the
// pair: pixel rows 32h + lane). kMkWbStages pairs and a ring of the same
// depth: a builder's consecutive stages are exactly one ring apart.
constexpr int kMkWbStages = 3;
__global__ void __launch_bounds__(kWbThreads, 1) c3b_wgrad_mk_kernel(const uint16_t* __restrict__ x,
                                                                     const __grid_constant__ CUtensorMap tma_dy, C3B g,
                                                                     int ppb, int KB, int ncols,
                                                                     float* __restrict__ part) {
  extern __shared__ uint8_t smem_raw[];
  const uint32_t raw = smem_u32(smem_raw);
  const uint32_t base = (raw + 1023u) & ~1023u;
  const uint32_t stage = 16384 + static_cast<uint32_t>(KB) * 8192;
  const uint32_t bars = base + kMkWbStages * stage;
  auto full_bar = [&](int s) { return bars + 8u * s; };
  auto empty_bar = [&](int s) { return bars + 8u * (kMkWbStages + s); };
  const uint32_t done_bar = bars + 8u * (2 * kMkWbStages);
  const uint32_t tmem_slot = bars + 8u * (2 * kMkWbStages + 1);
  int* tab = reinterpret_cast<int*>(smem_raw + (bars + 8u * (2 * kMkWbStages + 2) - raw));
  const int* off = tab;
  const int* rs = tab + kMkMaxKB * kKb;

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int p_begin = blockIdx.x * ppb;
  const int p_end = min(p_begin + ppb, g.P);
  const int nkb = p_end > p_begin ? (p_end - p_begin + kKb - 1) / kKb : 0;
  const int nt = KB * kKb;
  const int n1 = nt <= 256 ? nt : 256, n2 = nt - n1;

  if (threadIdx.x == 0) {
    for (int s = 0; s < kMkWbStages; ++s) {
      mbar_init(full_bar(s), 65);  // the building pair's 64 lanes + the TMA thread's expect_tx arrival
      mbar_init(empty_bar(s), 1);
    }
    mbar_init(done_bar, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  c3b_table_mk(g, KB, tab, tab + kMkMaxKB * kKb);
  if (warp == 9) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(tmem_slot), "r"(ncols)
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
    const int pr = warp >> 1, half = warp & 1;
    for (int it = pr; warp < 2 * kMkWbStages && it < nkb; it += kMkWbStages) {
      const int s = it % kMkWbStages;
      const int row = half * 32 + lane;
      const int m = p_begin + it * kKb + row;
      const C3BPix q = c3b_pix(g, m < p_end ? m : g.P);
      if (it >= kMkWbStages) mbar_wait(empty_bar(s), ((it / kMkWbStages) & 1) ^ 1);
      const uint32_t sbb = base + s * stage + 16384;
      for (int kb = 0; kb < KB; ++kb) {
        uint32_t u[32];
        c3b_row_kb(x, g, off, rs, q, kb, u);
#pragma unroll
        for (int j = 0; j < 8; ++j) st_shared_v4(mnb_addr(sbb, row, kb, j), u[4 * j], u[4 * j + 1], u[4 * j + 2], u[4 * j + 3]);
      }
      fence_proxy_async();
      mbar_arrive(full_bar(s));
    }
    // ---------------- epilogue: warp w owns TMEM lanes 32w.. = co ----------------
    if (warp < 4 && warp * 32 < g.Cout) {
      mbar_wait_sleep(done_bar, 0);
      tc_fence_after();
      const int co = warp * 32 + lane;
      float* dst = part + (static_cast<int64_t>(blockIdx.x) * g.Cout + co) * g.KK;
      for (int cg = 0; cg < nt / 32; ++cg) {
        float v[32];
        tmem_ld32(tmem + (static_cast<uint32_t>(warp * 32) << 16) + cg * 32, v);
        if (nkb <= 0) {
#pragma unroll
          for (int i = 0; i < 32; ++i) v[i] = 0.f;
        }
        if (co < g.Cout) {
#pragma unroll
          for (int i = 0; i < 32; ++i)
            if (cg * 32 + i < g.KK) dst[cg * 32 + i] = v[i];
        }
      }
    }
  } else if (warp == 8) {
    // ---------------- TMA producer (dY tiles: two 64-co boxes per stage) ----------------
    if (lane == 0) {
      asm volatile("prefetch.tensormap [%0];" ::"l"(&tma_dy) : "memory");
      for (int it = 0; it < nkb; ++it) {
        const int s = it % kMkWbStages;
        if (it >= kMkWbStages) mbar_wait(empty_bar(s), ((it / kMkWbStages) & 1) ^ 1);
        mbar_expect_tx(full_bar(s), 16384u);
        tma_load_2d(base + s * stage, &tma_dy, full_bar(s), 0, p_begin + it * kKb);
        tma_load_2d(base + s * stage + 8192, &tma_dy, full_bar(s), 64, p_begin + it * kKb);
      }
    }
    __syncwarp();
  } else {
    // ---------------- MMA issuer ----------------
    const uint32_t idesc1 = make_idesc_bf16(n1, true, true);
    const uint32_t idesc2 = make_idesc_bf16(n2 > 0 ? n2 : 16, true, true);
    const bool leader = elect_one();
    for (int it = 0; it < nkb; ++it) {
      const int s = it % kMkWbStages;
      mbar_wait(full_bar(s), (it / kMkWbStages) & 1);
      tc_fence_after();
      const uint32_t sa = base + s * stage;
      const uint32_t sbb = sa + 16384;
      if (leader) {
#pragma unroll
        for (int kk = 0; kk < kKb / 16; ++kk) {
          const uint64_t ad = make_sdesc(sa + kk * 2048, 8192, 1024, kSw128);
          tc_mma_bf16(tmem, ad, make_sdesc(sbb + kk * 2048, 8192, 1024, kSw128), idesc1, (it > 0 || kk > 0) ? 1u : 0u);
          if (n2 > 0)
            tc_mma_bf16(tmem + n1, ad, make_sdesc(sbb + (n1 / 64) * 8192 + kk * 2048, 8192, 1024, kSw128), idesc2,
                        (it > 0 || kk > 0) ? 1u : 0u);
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

// Partials [nparts][count] summed in part order; bf16 SGD update (one
// rounding) or the fp32 dW.
__global__ void c3b_reduce_kernel(const float* __restrict__ part, int nparts, int64_t count, bf16* __restrict__ w,
                                  float lr, float* __restrict__ dw_out) {
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < count;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    float s = 0.f;
    for (int b = 0; b < nparts; ++b) s += part[static_cast<size_t>(b) * count + i];
    if (dw_out)
      dw_out[i] = s;
    else
      w[i] = __float2bfloat16_rn(__bfloat162float(w[i]) - lr * s);
  }
}

C3B geom_of(const ConvArgs& a) {
  C3B g;
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
  return 1024 + static_cast<size_t>((NB * 128 + 1023) & ~1023) + kFbStages * 16384 +
         2 * static_cast<size_t>((NB + 63) / 64) * 16384 + 8 * (2 * kFbStages + 6) + 2 * kKb * sizeof(int) + 64;
}
size_t wgrad_smem() {
  return 1024 + static_cast<size_t>(kWbStages) * kWbStage + 8 * (2 * kWbStages + 2) + 2 * kKb * sizeof(int) + 64;
}

int wgrad_blocks(const C3B& g) { return std::max(1, std::min(kSmsC3, (g.P + 255) / 256)); }

bool c3b_common(const ConvArgs& a) {
  const int64_t P = static_cast<int64_t>(a.n) * a.ho() * a.wo();
  const int64_t X = static_cast<int64_t>(a.n) * a.h * a.w * a.c[0];
  return a.nseg == 1 && a.c[0] <= 8 && a.kh == a.kw && a.kh * a.kw * a.c[0] <= kMkMaxKB * kKb && a.kh < 256 &&
         P > 0 && P < (int64_t{1} << 31) - kBM && X < (int64_t{1} << 40);
}
int kblocks_of(const ConvArgs& a) { return (a.kh * a.kw * a.c[0] + kKb - 1) / kKb; }
size_t fprop_mk_smem(int NB, int KB) {
  const size_t bblk = (static_cast<size_t>(NB) * 128 + 1023) & ~size_t{1023};
  return 1024 + KB * bblk + kFbmStages * 16384 + 2 * static_cast<size_t>((NB + 63) / 64) * 16384 +
         8 * (2 * kFbmStages + 6) + 2 * kMkMaxKB * kKb * sizeof(int) + 64;
}
size_t wgrad_mk_smem(int KB) {
  return 1024 + kMkWbStages * (16384 + static_cast<size_t>(KB) * 8192) + 8 * (2 * kMkWbStages + 2) +
         2 * kMkMaxKB * kKb * sizeof(int) + 64;
}

}  // namespace

bool c3b_fprop_eligible(const ConvArgs& a) {
  return c3b_common(a) && a.cout % 8 == 0 && a.cout <= 128 &&
         (kblocks_of(a) == 1 || fprop_mk_smem((a.cout + 31) / 32 * 32, kblocks_of(a)) <= 227 * 1024);
}
bool c3b_wgrad_eligible(const ConvArgs& a) {
  return c3b_common(a) && (kblocks_of(a) == 1 ? (a.cout == 64 || a.cout == 128) : (a.cout % 8 == 0 && a.cout <= 128));
}
size_t c3b_wgrad_ws_bytes(const ConvArgs& a) {
  const C3B g = geom_of(a);
  return static_cast<size_t>(wgrad_blocks(g)) * g.Cout * g.KK * sizeof(float);
}

cudaError_t c3b_fprop(const ConvArgs& a, const void* w, void* y, cudaStream_t st) {
  const C3B g = geom_of(a);
  if (g.P <= 0) return cudaSuccess;
  const int NB = (g.Cout + 31) / 32 * 32, NBP = pow2_at_least(NB);
  // Y [P][Cout] bf16 in 128-pixel x 64-channel SWIZZLE_128B boxes
  alignas(64) CUtensorMap ty;
  const cuuint64_t dims[2] = {static_cast<cuuint64_t>(g.Cout), static_cast<cuuint64_t>(g.P)};
  const cuuint64_t strides[1] = {static_cast<cuuint64_t>(g.Cout) * 2};
  const cuuint32_t box[2] = {64, static_cast<cuuint32_t>(kBM)};
  if (!encode_tiled(&ty, y, 2, dims, strides, box, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16))
    return cudaErrorInvalidValue;
  const int KB = kblocks_of(a);
  if (KB > 1) {
    const size_t smk = fprop_mk_smem(NB, KB);
    static size_t attr_mk = 0;
    if (smk > attr_mk) {
      cudaError_t e = cudaFuncSetAttribute(c3b_fprop_mk_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                           static_cast<int>(smk));
      if (e != cudaSuccess) return e;
      attr_mk = smk;
    }
    const int ntiles = (g.P + kBM - 1) / kBM;
    c3b_fprop_mk_kernel<<<std::min(kSmsC3, ntiles), kFbmThreads, smk, st>>>(
        static_cast<const uint16_t*>(static_cast<const void*>(a.x[0])), static_cast<const uint16_t*>(w), ty, g, NB,
        NBP, KB, a.relu_out);
    count_launch();
    return cudaGetLastError();
  }
  const size_t smem = fprop_smem(NB);
  const bool k3c3 = g.k == 3 && g.C == 3;
  auto kern = k3c3 ? c3b_fprop_kernel<3, 3> : c3b_fprop_kernel<0, 0>;
  static size_t attr[2] = {0, 0};
  if (smem > attr[k3c3]) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
    if (e != cudaSuccess) return e;
    attr[k3c3] = smem;
  }
  const int ntiles = (g.P + kBM - 1) / kBM;
  kern<<<std::min(kSmsC3, ntiles), kFbThreads, smem, st>>>(
      static_cast<const uint16_t*>(static_cast<const void*>(a.x[0])), static_cast<const uint16_t*>(w), ty, g, NB, NBP,
      a.relu_out);
  count_launch();
  return cudaGetLastError();
}

cudaError_t c3b_wgrad(const ConvArgs& a, const void* dy, void* w, float lr, float* dw_out, float* ws, size_t ws_bytes,
                      cudaStream_t st) {
  const C3B g = geom_of(a);
  const size_t per = static_cast<size_t>(g.Cout) * g.KK * sizeof(float);
  int nb = wgrad_blocks(g);
  if (ws == nullptr || ws_bytes < per) return cudaErrorInvalidValue;
  nb = static_cast<int>(std::min<size_t>(nb, ws_bytes / per));
  int ppb = (g.P + nb - 1) / nb;
  ppb = (ppb + kKb - 1) / kKb * kKb;
  nb = static_cast<int>((g.P + ppb - 1) / ppb);
  const int KB = kblocks_of(a);
  if (KB > 1) {
    // dY [P][Cout]: 64 co x 64 pixel boxes (MN-major chunks), co past Cout zero-filled
    alignas(64) CUtensorMap t2;
    const cuuint64_t d2[2] = {static_cast<cuuint64_t>(g.Cout), static_cast<cuuint64_t>(g.P)};
    const cuuint64_t s2[1] = {static_cast<cuuint64_t>(g.Cout) * 2};
    const cuuint32_t b2[2] = {64, 64};
    if (!encode_tiled(&t2, dy, 2, d2, s2, b2, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16))
      return cudaErrorInvalidValue;
    const size_t smk = wgrad_mk_smem(KB);
    static size_t attr_mk = 0;
    if (smk > attr_mk) {
      cudaError_t e = cudaFuncSetAttribute(c3b_wgrad_mk_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                           static_cast<int>(smk));
      if (e != cudaSuccess) return e;
      attr_mk = smk;
    }
    c3b_wgrad_mk_kernel<<<nb, kWbThreads, smk, st>>>(static_cast<const uint16_t*>(static_cast<const void*>(a.x[0])),
                                                     t2, g, ppb, KB, pow2_at_least(KB * kKb), ws);
  } else {
  // dY [P][Cout] as (64 co, pixel, co-chunk): one 64-pixel box per stage, MN-major 8 KB chunks
  alignas(64) CUtensorMap tdy;
  const cuuint64_t d3[3] = {64, static_cast<cuuint64_t>(g.P), static_cast<cuuint64_t>(g.Cout / 64)};
  const cuuint64_t s3[2] = {static_cast<cuuint64_t>(g.Cout) * 2, 128};
  const cuuint32_t b3[3] = {64, 64, static_cast<cuuint32_t>(g.Cout / 64)};
  if (!encode_tiled(&tdy, dy, 3, d3, s3, b3, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16))
    return cudaErrorInvalidValue;
  const size_t smem = wgrad_smem();
  const bool k3c3 = g.k == 3 && g.C == 3;
  auto kern = k3c3 ? c3b_wgrad_kernel<3, 3> : c3b_wgrad_kernel<0, 0>;
  static size_t attr[2] = {0, 0};
  if (smem > attr[k3c3]) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
    if (e != cudaSuccess) return e;
    attr[k3c3] = smem;
  }
  static const int pf = [] {  // VDNN_C3_PREFETCH: dY stages prefetched into L2 ahead of the ring (A/B)
    const char* e = std::getenv("VDNN_C3_PREFETCH");
    return e ? std::atoi(e) : kWbPrefetch;
  }();
  kern<<<nb, kWbThreads, smem, st>>>(static_cast<const uint16_t*>(static_cast<const void*>(a.x[0])), tdy,
                                                 g, ppb, pf, ws);
  }
  count_launch();
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  const int64_t count = static_cast<int64_t>(g.Cout) * g.KK;
  c3b_reduce_kernel<<<static_cast<int>(std::min<int64_t>((count + 255) / 256, 1184)), 256, 0, st>>>(
      ws, nb, count, static_cast<bf16*>(w), lr, dw_out);
  count_launch();
  return cudaGetLastError();
}

}  // namespace vdnnk
