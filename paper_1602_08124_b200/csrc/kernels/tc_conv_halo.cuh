// Halo-reuse variant of the tcgen05 conv engine for stride-1 FPROP / DGRAD
// (included by conv.cu after tc_conv.cuh).
//
// The im2col producer stages every input pixel once per filter tap (9x for a
// 3x3 conv): at 64-128 output channels the L2 -> SM fill rate, not the tensor
// pipe, bounds those layers (26-44 FLOP per staged byte). Here the A operand
// of tap (r, s) is read straight out of ONE staged block of input rows:
//
//   Output pixels are indexed on a "virtual" grid whose row pitch is the
//   padded input width P = Win + 2*pad (columns >= Wout are garbage). Then
//   the input pixel of output v = y*P + x under tap (r, s) is the padded
//   input pixel v + r*P + s: an affine shift. A tile is TH = 256 / P output
//   rows (two M=128 MMAs, virtual rows 0..255); the stage of (channel chunk c,
//   tap row r) is the TMA box of TH padded input rows x P pixels x 32
//   channels (zero fill does the padding), and the MMA of tap (r, s) uses an
//   A descriptor whose start address is advanced by s rows of 128 B. The
//   SWIZZLE_128B pattern is a function of the absolute shared-memory address
//   (measured: tools/halo_probe.cu, descriptor base offset 0), so a start at
//   any 128-B row of the swizzled block is a valid K-major operand.
//
// Per (c, r) stage the A fill is TH*P rows for kw taps: ~3 rows per output
// pixel instead of 9; B (weights) streams per tap through its own ring.
//   BN=128: 82 FLOP per staged byte (im2col tall tiles: 43); BN=64: 59 (26).
// Valid outputs per tile: TH*Wout of 256 virtual rows (VGG: 224 = 87.5%).
//
//   warps 0-3 : epilogue (warp w drains TMEM lanes 32w..32w+31): fused ReLU
//               (fprop) / ReLU-backward mask (dgrad), accumulate, stores
//   warp 4    : TMEM owner + single-thread tcgen05.mma issuer
//   warp 5    : single-thread TMA producer
// Persistent (one CTA per SM, static round-robin over tiles), two TMEM
// accumulator sets so tile t's epilogue overlaps tile t+1's main loop.
#pragma once

namespace vdnnk {

struct HaloParams {
  int kind;               // kFprop or kDgrad
  int N, Hin, Win, Cin;   // A source: fprop X, dgrad dY (NHWC)
  int pad;                // fprop: pad; dgrad: kh - 1 - pad
  int kh, kw;
  int Hout, Wout, Cout;   // output: fprop Y, dgrad dX (NHWC)
  int P, TH, nck, tiles_h, ntn, ntiles;
  int relu, accum;
  int epi_t;              // halo pair: stores transposed through shared memory (store_half32_f32)
  float* out;
  const float* mask_x;    // dgrad: dX *= (x > 0), x laid out like out; null = none
};

template <int BN, int AS, int BS>
struct HaloSmem {
  static constexpr int kASlot = 33 * 1024;  // >= 258 rows x 128 B (256 virtual rows + 2 tap shifts)
  static constexpr int kBSlot = BN * 128;
  static constexpr int kTotal = AS * kASlot + BS * kBSlot + 1024 + 256;
  static constexpr int kAccCols = 2 * BN;  // two M=128 halves
  static_assert(2 * kAccCols <= 512, "two accumulator sets must fit TMEM");
};

template <int BN, int AS, int BS, int KW>
__global__ void __launch_bounds__(192, 1) tc_conv_halo_kernel(const __grid_constant__ HaloParams p,
                                                              const __grid_constant__ CUtensorMap tma_a,
                                                              const __grid_constant__ CUtensorMap tma_b) {
  using L = HaloSmem<BN, AS, BS>;
  constexpr int kTmemCols = 2 * L::kAccCols;
  extern __shared__ uint8_t smem_raw[];
  const uint32_t base = (smem_u32(smem_raw) + 1023u) & ~1023u;
  const uint32_t bslots = base + AS * L::kASlot;
  const uint32_t bars = bslots + BS * L::kBSlot;
  auto full_a = [&](int s) { return bars + 8u * s; };
  auto empty_a = [&](int s) { return bars + 8u * (AS + s); };
  auto full_b = [&](int s) { return bars + 8u * (2 * AS + s); };
  auto empty_b = [&](int s) { return bars + 8u * (2 * AS + BS + s); };
  auto tfull = [&](int a) { return bars + 8u * (2 * AS + 2 * BS + a); };
  auto tempty = [&](int a) { return bars + 8u * (2 * AS + 2 * BS + 2 + a); };
  const uint32_t tmem_slot = bars + 8u * (2 * AS + 2 * BS + 4);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

  if (threadIdx.x == 0) {
    for (int s = 0; s < AS; ++s) {
      mbar_init(full_a(s), 1);
      mbar_init(empty_a(s), 1);
    }
    for (int s = 0; s < BS; ++s) {
      mbar_init(full_b(s), 1);
      mbar_init(empty_b(s), 1);
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(tfull(a), 1);
      mbar_init(tempty(a), 128);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 4) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(tmem_slot),
                 "r"(kTmemCols)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  uint32_t tmem;
  asm volatile("ld.shared.u32 %0, [%1];" : "=r"(tmem) : "r"(tmem_slot) : "memory");

  const uint32_t abytes = static_cast<uint32_t>(p.TH * p.P * 128);
  if (warp == 5) {
    // ---------------- TMA producer ----------------
    if (lane == 0) {
      asm volatile("prefetch.tensormap [%0];" ::"l"(&tma_a) : "memory");
      asm volatile("prefetch.tensormap [%0];" ::"l"(&tma_b) : "memory");
      int sa = 0, sb = 0;
      uint32_t pha = 1, phb = 1;  // the first pass over each ring does not wait
      for (int tile = blockIdx.x; tile < p.ntiles; tile += gridDim.x) {
        const int tn = tile % p.ntn, t2 = tile / p.ntn;
        const int th = t2 % p.tiles_h, n = t2 / p.tiles_h;
        const int y0 = th * p.TH, n0 = tn * BN;
        if (p.mask_x && tn == 0 && y0 < p.Hout)  // the dgrad ReLU mask into L2 (tc_conv_halo_pair.cuh)
          prefetch_l2_bulk(p.mask_x + (static_cast<int64_t>(n) * p.Hout + y0) * p.Wout * p.Cout,
                           static_cast<uint64_t>(min(p.TH, p.Hout - y0)) * p.Wout * p.Cout * sizeof(float));
        for (int c = 0; c < p.nck; ++c) {
          for (int r = 0; r < p.kh; ++r) {
            mbar_wait(empty_a(sa), pha);
            mbar_expect_tx(full_a(sa), abytes);
            tma_load_4d(base + sa * L::kASlot, &tma_a, full_a(sa), c * 32, -p.pad, y0 + r - p.pad, n);
            if (++sa == AS) {
              sa = 0;
              pha ^= 1;
            }
#pragma unroll
            for (int s = 0; s < KW; ++s) {
              mbar_wait(empty_b(sb), phb);
              mbar_expect_tx(full_b(sb), L::kBSlot);
              if (p.kind == kFprop) {
                tma_load_2d(bslots + sb * L::kBSlot, &tma_b, full_b(sb), (r * KW + s) * p.Cin + c * 32, n0);
              } else {
                const int ftap = (p.kh - 1 - r) * KW + (KW - 1 - s);
                tma_load_4d(bslots + sb * L::kBSlot, &tma_b, full_b(sb), 0, c * 32, n0 >> 5, ftap);
              }
              if (++sb == BS) {
                sb = 0;
                phb ^= 1;
              }
            }
          }
        }
      }
    }
    __syncwarp();
  } else if (warp == 4) {
    // ---------------- MMA issuer ----------------
    // Issue-bound if written naively: a B sub-stage is only 8 MMAs (~120
    // cycles of tensor work at N=128), so descriptors are precomputed (the
    // 14-bit start-address field is advanced by adding (offset >> 4)), the
    // taps are unrolled (KW is a template parameter) and the ring indices
    // wrap instead of using / and %.
    // The whole warp runs the loop (warp-uniform control flow and
    // descriptors, so they live in uniform registers); one elected lane
    // issues the MMAs and commits.
    const bool leader = elect_one();
    const bool b_mn = p.kind != kFprop;
    const uint32_t idesc = make_idesc_tf32(BN, false, b_mn);
    const uint64_t adesc0 = make_sdesc(base, 16, 1024, kSw128);
    const uint64_t bdesc0 = b_mn ? make_sdesc(bslots, 4096, 512, kSw128Base32) : make_sdesc(bslots, 16, 1024, kSw128);
    const uint32_t kstep_b = b_mn ? (1024 >> 4) : (32 >> 4);  // next K=8 slice of B
    int sa = 0, sb = 0, lt = 0;
    uint32_t pha = 0, phb = 0;
    const int nstage = p.nck * p.kh;
    for (int tile = blockIdx.x; tile < p.ntiles; tile += gridDim.x, ++lt) {
      const int acc = lt & 1;
      if (lt >= 2) mbar_wait(tempty(acc), ((lt >> 1) & 1) ^ 1);
      tc_fence_after();
      const uint32_t d0 = tmem + acc * L::kAccCols;
      uint32_t first = 1;
      for (int st = 0; st < nstage; ++st) {
        mbar_wait(full_a(sa), pha);
        tc_fence_after();
        const uint64_t ad = adesc0 + static_cast<uint64_t>((sa * L::kASlot) >> 4);
#pragma unroll
        for (int s = 0; s < KW; ++s) {
          mbar_wait(full_b(sb), phb);
          tc_fence_after();
          const uint64_t bd = bdesc0 + static_cast<uint64_t>((sb * L::kBSlot) >> 4);
          if (leader) {
#pragma unroll
            for (int kk = 0; kk < kBK / 8; ++kk) {
#pragma unroll
              for (int h = 0; h < 2; ++h)
                tc_mma_tf32(d0 + h * BN, ad + static_cast<uint64_t>(((h * kBM + s) * 128 + kk * 32) >> 4),
                            bd + static_cast<uint64_t>(kk * kstep_b), idesc, (first && kk == 0) ? 0u : 1u);
            }
            tc_commit(empty_b(sb));
          }
          __syncwarp();
          first = 0;
          if (++sb == BS) {
            sb = 0;
            phb ^= 1;
          }
        }
        if (leader) tc_commit(empty_a(sa));
        __syncwarp();
        if (++sa == AS) {
          sa = 0;
          pha ^= 1;
        }
      }
      if (leader) tc_commit(tfull(acc));
      __syncwarp();
    }
  } else {
    // ---------------- epilogue ----------------
    const int row = warp * 32 + lane;
    int lt = 0;
    for (int tile = blockIdx.x; tile < p.ntiles; tile += gridDim.x, ++lt) {
      const int acc = lt & 1;
      const int tn = tile % p.ntn, t2 = tile / p.ntn;
      const int th = t2 % p.tiles_h, n = t2 / p.tiles_h;
      const int y0 = th * p.TH, n0 = tn * BN;
      mbar_wait_sleep(tfull(acc), (lt >> 1) & 1);
      tc_fence_after();
#pragma unroll 1
      for (int h = 0; h < 2; ++h) {
        const int v = h * kBM + row;
        const int yl = v / p.P, x = v - yl * p.P, y = y0 + yl;
        const bool valid = yl < p.TH && x < p.Wout && y < p.Hout;
        const int64_t pix = (static_cast<int64_t>(n) * p.Hout + y) * p.Wout + x;
        const uint32_t taddr = tmem + acc * L::kAccCols + h * BN + (static_cast<uint32_t>(warp * 32) << 16);
#pragma unroll 1
        for (int cg = 0; cg < BN / 32; ++cg) {
          float vals[32];
          tmem_ld32(taddr + cg * 32, vals);
          if (h == 1 && cg == BN / 32 - 1) {
            // last TMEM read of this accumulator set: hand it back to the MMA warp
            tc_fence_before();
            mbar_arrive(tempty(acc));
          }
          const int nb = n0 + cg * 32;
          if (!valid || nb >= p.Cout) continue;
          if (p.relu) {
#pragma unroll
            for (int i = 0; i < 32; ++i) vals[i] = fmaxf(vals[i], 0.f);
          }
          if (p.mask_x) {
            const float4* xr = reinterpret_cast<const float4*>(p.mask_x + pix * p.Cout + nb);
            float4 xv[8];
#pragma unroll
            for (int i = 0; i < 8; ++i) xv[i] = __ldg(xr + i);
#pragma unroll
            for (int i = 0; i < 8; ++i) {
              vals[4 * i] = xv[i].x > 0.f ? vals[4 * i] : 0.f;
              vals[4 * i + 1] = xv[i].y > 0.f ? vals[4 * i + 1] : 0.f;
              vals[4 * i + 2] = xv[i].z > 0.f ? vals[4 * i + 2] : 0.f;
              vals[4 * i + 3] = xv[i].w > 0.f ? vals[4 * i + 3] : 0.f;
            }
          }
          float4* dst = reinterpret_cast<float4*>(p.out + pix * p.Cout + nb);
          if (p.accum) {
            float4 a[8];  // loads in flight together, then the stores
#pragma unroll
            for (int i = 0; i < 8; ++i) a[i] = dst[i];
#pragma unroll
            for (int i = 0; i < 8; ++i) {
              vals[4 * i] += a[i].x;
              vals[4 * i + 1] += a[i].y;
              vals[4 * i + 2] += a[i].z;
              vals[4 * i + 3] += a[i].w;
            }
          }
#pragma unroll
          for (int i = 0; i < 8; ++i)
            dst[i] = make_float4(vals[4 * i], vals[4 * i + 1], vals[4 * i + 2], vals[4 * i + 3]);
        }
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 4) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(kTmemCols) : "memory");
  }
}

}  // namespace vdnnk

namespace vdnnk {

// ------------------------------------------------------- halo WGRAD -------
// dW[co][r][s][ci] = sum_p dY[p][co] * X[p + r*P + s][ci] on the virtual
// pixel grid (pitch P = W + 2*pad; dY is 0 on the garbage columns x >= Wout,
// which TMA's out-of-bounds fill provides). One pipeline unit is one virtual
// output row: B = that dY row (Cout/32 MN-major chunks of P pixel rows), and
// per (tap row r, 32-channel chunk c) of this CTA's group one TMA box of the
// padded input row y + r. The M = 128 rows of an MMA are the four shifted
// views s = 0..3 of that ONE staged box (MN-major chunks LBO = 128 B apart:
// A[(s, ci)][k] = X[k + s][ci]; tools/halo_mn_probe.cu) -- s = 3 is unused
// for 3x3, so 96 of 128 rows are useful, but every input row is staged once
// per (r, c) instead of once per tap (the im2col wgrad stages it 9 times).
// A CTA owns a group of (r, c) blocks (G x Cout TMEM columns) and a range of
// rows, and writes its split-K partial; wgrad_reduce_kernel sums them.
struct HaloWgParams {
  int N, H, W, C, Cout, kh, kw, pad, P, Kp, Hout, Wout, nck;
  int G, ngroups, rows_per, nrows, M;
  int AS, BS;              // ring depths (A: one padded input row per (r, c); B: one dY row)
  int pair;                // 1: tc_wgrad_halo_pair_kernel (G blocks per CTA, splits = pairs)
  uint32_t a_slot, b_slot; // bytes per slot (1024-aligned)
  float* part;             // [splits][Cout][M]
};
constexpr int kHwMaxAS = 4, kHwMaxBS = 2;
inline uint32_t halo_wg_a_slot(int Kp) { return ((static_cast<uint32_t>(Kp) + 8) * 128 + 1023u) & ~1023u; }
inline uint32_t halo_wg_b_slot(int Kp, int bn) { return ((static_cast<uint32_t>(bn / 32) * Kp * 128) + 1023u) & ~1023u; }

template <int BN>
__global__ void __launch_bounds__(192, 1) tc_wgrad_halo_kernel(const __grid_constant__ HaloWgParams p,
                                                               const __grid_constant__ CUtensorMap tma_x,
                                                               const __grid_constant__ CUtensorMap tma_dy) {
  const int AS = p.AS, BS = p.BS;
  extern __shared__ uint8_t smem_raw[];
  const uint32_t base = (smem_u32(smem_raw) + 1023u) & ~1023u;
  const uint32_t bslots = base + AS * p.a_slot;
  const uint32_t bars = bslots + BS * p.b_slot;
  auto full_a = [&](int s) { return bars + 8u * s; };
  auto empty_a = [&](int s) { return bars + 8u * (AS + s); };
  auto full_b = [&](int s) { return bars + 8u * (2 * AS + s); };
  auto empty_b = [&](int s) { return bars + 8u * (2 * AS + BS + s); };
  const uint32_t done_bar = bars + 8u * (2 * AS + 2 * BS);
  const uint32_t tmem_slot = bars + 8u * (2 * AS + 2 * BS + 1);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int z = blockIdx.x / p.ngroups, grp = blockIdx.x - z * p.ngroups;
  const int g0 = grp * p.G;
  const int G = min(p.G, p.kh * p.nck - g0);  // (r, c) blocks of this CTA: index j -> block g0 + j
  const int row0 = z * p.rows_per;
  const int row1 = min(row0 + p.rows_per, p.nrows);
  const int nrows = max(0, row1 - row0);
  const int ncol = G * BN;
  int tcols = 32;
  while (tcols < ncol) tcols <<= 1;

  if (threadIdx.x == 0) {
    for (int s = 0; s < AS; ++s) {
      mbar_init(full_a(s), 1);
      mbar_init(empty_a(s), 1);
    }
    for (int s = 0; s < BS; ++s) {
      mbar_init(full_b(s), 1);
      mbar_init(empty_b(s), 1);
    }
    mbar_init(done_bar, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  // rows the boxes never write: B rows [P, Kp) must be 0 (they meet A rows of
  // garbage pixels), A rows [P, Kp + 8) must be finite
  for (int s = 0; s < AS; ++s)
    for (uint32_t o = p.P * 128 + threadIdx.x * 16; o < p.a_slot; o += blockDim.x * 16)
      asm volatile("st.shared.v4.u32 [%0], {%1, %1, %1, %1};" ::"r"(base + s * p.a_slot + o), "r"(0) : "memory");
  for (int s = 0; s < BS; ++s)
    for (int ch = 0; ch < BN / 32; ++ch)
      for (int o = p.P * 128 + threadIdx.x * 16; o < p.Kp * 128; o += blockDim.x * 16)
        asm volatile("st.shared.v4.u32 [%0], {%1, %1, %1, %1};" ::"r"(bslots + s * p.b_slot + ch * p.Kp * 128 + o),
                     "r"(0)
                     : "memory");
  fence_proxy_async();
  if (warp == 4) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(tmem_slot), "r"(tcols)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  uint32_t tmem;
  asm volatile("ld.shared.u32 %0, [%1];" : "=r"(tmem) : "r"(tmem_slot) : "memory");

  if (warp == 5) {
    // ---------------- TMA producer (one thread, in consumption order) ----------------
    if (lane == 0) {
      asm volatile("prefetch.tensormap [%0];" ::"l"(&tma_x) : "memory");
      asm volatile("prefetch.tensormap [%0];" ::"l"(&tma_dy) : "memory");
      int sa = 0, sb = 0;
      uint32_t pha = 1, phb = 1;
      const uint32_t abytes = static_cast<uint32_t>(p.P) * 128, bbytes = (BN / 32) * abytes;
      for (int row = row0; row < row1; ++row) {
        const int n = row / p.Hout, y = row - n * p.Hout;
        mbar_wait(empty_b(sb), phb);
        mbar_expect_tx(full_b(sb), bbytes);
        for (int ch = 0; ch < BN / 32; ++ch)
          tma_load_4d(bslots + sb * p.b_slot + ch * p.Kp * 128, &tma_dy, full_b(sb), ch * 32, 0, y, n);
        if (++sb == BS) {
          sb = 0;
          phb ^= 1;
        }
        for (int j = 0; j < G; ++j) {
          const int blk = g0 + j, r = blk / p.nck, c = blk - r * p.nck;
          mbar_wait(empty_a(sa), pha);
          mbar_expect_tx(full_a(sa), abytes);
          tma_load_4d(base + sa * p.a_slot, &tma_x, full_a(sa), c * 32, -p.pad, y + r - p.pad, n);
          if (++sa == AS) {
            sa = 0;
            pha ^= 1;
          }
        }
      }
    }
    __syncwarp();
  } else if (warp == 4) {
    // ---------------- MMA issuer ----------------
    const uint32_t idesc = make_idesc_tf32(BN, true, true);
    const bool leader = elect_one();
    const int ksteps = p.Kp / 8;
    const uint32_t lbo_b = static_cast<uint32_t>(p.Kp) * 128;
    int sa = 0, sb = 0;
    uint32_t pha = 0, phb = 0;
    for (int i = 0; i < nrows; ++i) {
      mbar_wait(full_b(sb), phb);
      tc_fence_after();
      const uint32_t b0 = bslots + sb * p.b_slot;
      for (int j = 0; j < G; ++j) {
        mbar_wait(full_a(sa), pha);
        tc_fence_after();
        const uint32_t a0 = base + sa * p.a_slot;
        if (leader) {
          for (int kk = 0; kk < ksteps; ++kk)
            tc_mma_tf32(tmem + j * BN, make_sdesc(a0 + kk * 1024, 128, 512, kSw128Base32),
                        make_sdesc(b0 + kk * 1024, lbo_b, 512, kSw128Base32), idesc, (i > 0 || kk > 0) ? 1u : 0u);
          tc_commit(empty_a(sa));
        }
        __syncwarp();
        if (++sa == AS) {
          sa = 0;
          pha ^= 1;
        }
      }
      if (leader) tc_commit(empty_b(sb));
      __syncwarp();
      if (++sb == BS) {
        sb = 0;
        phb ^= 1;
      }
    }
    if (leader) {
      if (nrows > 0)
        tc_commit(done_bar);
      else
        mbar_arrive(done_bar);
    }
    __syncwarp();
  } else {
    // ---------------- epilogue: warp w = shift s, lane = ci ----------------
    mbar_wait_sleep(done_bar, 0);
    tc_fence_after();
    const int s = warp;
    for (int j = 0; j < G; ++j) {
      const int blk = g0 + j, r = blk / p.nck, c = blk - r * p.nck;
      const int m = ((r * p.kw + s) * p.nck + c) * 32 + lane;
      for (int cg = 0; cg < BN / 32; ++cg) {
        float v[32];
        tmem_ld32(tmem + j * BN + cg * 32 + (static_cast<uint32_t>(warp * 32) << 16), v);
        if (s >= p.kw) continue;  // the fourth shifted view (taps past the kernel)
        if (nrows <= 0) {
#pragma unroll
          for (int q = 0; q < 32; ++q) v[q] = 0.f;
        }
        float* dst = p.part + static_cast<int64_t>(z) * p.Cout * p.M;
#pragma unroll
        for (int q = 0; q < 32; ++q)
          if (cg * 32 + q < p.Cout) dst[static_cast<int64_t>(cg * 32 + q) * p.M + m] = v[q];
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 4) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(tcols) : "memory");
  }
}

}  // namespace vdnnk
