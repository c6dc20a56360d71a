// Halo-reuse FPROP / DGRAD for the BF16 engine (included by conv_bf16.cu
// after tcb_conv.cuh): stride-1 k x k convolutions with 64-multiple channel
// counts and narrow outputs (<= 128 columns), i.e. VGG's 224x224x64 and
// 112x112x128 layers.
//
// Why: the im2col TMA producer (tcb_conv.cuh) stages every input pixel once
// per filter tap -- 9 x 16 KB boxes per 128 output pixels for a 3x3 conv over
// 64 channels -- and at N = 64 / 128 columns that fill, not the tensor pipe,
// bounds the layer (ncu, 224x224x64 fprop: L1/TMA throughput 87% of peak,
// 22 GB through the xbar for 3.3 GB of X and Y, tensor pipe 21% active).
// Here, as in the TF32 halo kernel (tc_conv_halo.cuh), output pixels live on
// a virtual grid whose row pitch is the padded input width P = Win + 2*pad:
// the input pixel of output v = y*P + x under tap (r, s) is padded input pixel
// v + r*P + s, so one TMA box of TH padded input rows x P pixels x 64 channels
// (zero fill = padding) serves the kw taps of filter row r through A
// descriptors advanced by s rows of 128 B (SWIZZLE_128B is a function of the
// absolute shared-memory address: tools/halo_probe.cu). A fill per 256
// virtual rows: kh boxes of <= 33 KB per 64 channels instead of kh*kw boxes.
//
//   FPROP  A = X box (K-major), B = W[co][r][s][c0:c0+64] (K-major, one 2D box)
//   DGRAD  A = dY box (K-major, pad' = k-1-pad), B[k = co][n = ci] =
//          W[co][flipped tap][ci] (MN-major: 64 ci x 64 co boxes), fused
//          ReLU backward (dX *= x > 0) and accumulation in the epilogue.
// Tile = 256 virtual rows (two M = 128 MMAs per tap, h = 0, 1) x BN columns;
// persistent CTAs (one per SM), two TMEM accumulator sets (4 x BN columns)
// so tile t's epilogue overlaps tile t+1's main loop.
//   warps 0-3, 6-9 : epilogue, one M half per warpgroup (TMEM lane quarter
//               = warp % 4): bf16 RNE stores, fused ReLU / mask / accumulate
//   warp 4    : TMEM owner + MMA issuer (one elected lane)
//   warp 5    : TMA producer (one lane), in consumption order
#pragma once

namespace vdnnk {

struct HaloParamsB {
  int kind;               // kFprop or kDgrad
  int N, Hin, Win, Cin;   // A source: fprop X, dgrad dY (NHWC bf16)
  int pad;                // fprop: pad; dgrad: kh - 1 - pad
  int kh, kw;
  int Hout, Wout, Cout;   // output: fprop Y, dgrad dX (NHWC bf16)
  int P, TH, nck, tiles_h, ntn, ntiles;
  int relu, accum;
  int epi_t;              // 1: stores transposed through shared memory (store_tile32_t)
  bf16* out;
  const bf16* mask_x;     // dgrad: dX *= (x > 0), x laid out like out; null = none
};

template <int BN, int AS, int BS>
struct HaloSmemB {
  static constexpr int kASlot = 33 * 1024;  // >= 258 rows x 128 B (256 virtual rows + 2 tap shifts)
  static constexpr int kBSlot = BN * 128;
  static constexpr int kEpiScratch = 8 * 2048;  // store_tile32_t transpose, one 2 KB block per epilogue warp
  static constexpr int kTotal = AS * kASlot + BS * kBSlot + 1024 + 256 + kEpiScratch;
  static constexpr int kAccCols = 2 * BN;   // two M = 128 halves
  static_assert(2 * kAccCols <= 512, "two accumulator sets must fit TMEM");
};

// RESB: the whole filter (nck x kh x KW slots of BN x 64) is loaded once per
// CTA and stays resident (BS = that slot count): the per-tile B stream --
// 72 KB per 256 virtual rows at 64 -> 64 channels, 45% of the L2 -> SM fill
// -- disappears (224x224x64 fprop / dgrad).
// Two epilogue warpgroups (warps 0-3: M half 0, warps 6-9: M half 1; TMEM
// lane quarter = warp % 4) keep the dgrad's ReLU-mask loads and the stores of
// both halves in flight together (as tc_conv_halo_pair.cuh).
constexpr int kHaloBThreads = 320;
template <int BN, int AS, int BS, int KW, bool RESB = false>
__global__ void __launch_bounds__(kHaloBThreads, 1) tcb_halo_kernel(const __grid_constant__ HaloParamsB p,
                                                          const __grid_constant__ CUtensorMap tma_a,
                                                          const __grid_constant__ CUtensorMap tma_b) {
  using L = HaloSmemB<BN, AS, BS>;
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
      mbar_init(tempty(a), 256);  // both epilogue warpgroups
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
      if constexpr (RESB) {  // the whole filter, once, on full_b(0) (host: ntn == 1)
        mbar_expect_tx(full_b(0), static_cast<uint32_t>(BS) * L::kBSlot);
        for (int c = 0; c < p.nck; ++c)
          for (int r = 0; r < p.kh; ++r)
            for (int s = 0; s < KW; ++s) {
              const uint32_t bdst = bslots + ((c * p.kh + r) * KW + s) * L::kBSlot;
              if (p.kind == kFprop) {
                tma_load_2d(bdst, &tma_b, full_b(0), (r * KW + s) * p.Cin + c * 64, 0);
              } else {
                const int ftap = (p.kh - 1 - r) * KW + (KW - 1 - s);
                for (int mc = 0; mc < BN / 64; ++mc)
                  tma_load_3d(bdst + mc * 8192, &tma_b, full_b(0), mc * 64, ftap, c * 64);
              }
            }
      }
      for (int tile = blockIdx.x; tile < p.ntiles; tile += gridDim.x) {
        const int tn = tile % p.ntn, t2 = tile / p.ntn;
        const int th = t2 % p.tiles_h, n = t2 / p.tiles_h;
        const int y0 = th * p.TH, n0 = tn * BN;
        if (p.mask_x && tn == 0 && y0 < p.Hout)  // the dgrad ReLU mask into L2 while the main loop runs
          prefetch_l2_bulk(p.mask_x + (static_cast<int64_t>(n) * p.Hout + y0) * p.Wout * p.Cout,
                           static_cast<uint64_t>(min(p.TH, p.Hout - y0)) * p.Wout * p.Cout * sizeof(bf16));
        for (int c = 0; c < p.nck; ++c) {
          for (int r = 0; r < p.kh; ++r) {
            mbar_wait(empty_a(sa), pha);
            mbar_expect_tx(full_a(sa), abytes);
            tma_load_4d(base + sa * L::kASlot, &tma_a, full_a(sa), c * 64, -p.pad, y0 + r - p.pad, n);
            if (++sa == AS) {
              sa = 0;
              pha ^= 1;
            }
#pragma unroll
            for (int s = 0; s < KW; ++s) {
              if constexpr (RESB) continue;
              mbar_wait(empty_b(sb), phb);
              mbar_expect_tx(full_b(sb), L::kBSlot);
              const uint32_t bdst = bslots + sb * L::kBSlot;
              if (p.kind == kFprop) {
                tma_load_2d(bdst, &tma_b, full_b(sb), (r * KW + s) * p.Cin + c * 64, n0);
              } else {
                const int ftap = (p.kh - 1 - r) * KW + (KW - 1 - s);
#pragma unroll
                for (int mc = 0; mc < BN / 64; ++mc)
                  tma_load_3d(bdst + mc * 8192, &tma_b, full_b(sb), n0 + mc * 64, ftap, c * 64);
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
    // Descriptors precomputed (the 14-bit start-address field advances by
    // offset >> 4), taps unrolled, ring indices wrapped: a B sub-stage is
    // only 8 MMAs. The whole warp runs the loop; one elected lane issues.
    const bool leader = elect_one();
    const bool b_mn = p.kind != kFprop;
    const uint32_t idesc = make_idesc_bf16(BN, false, b_mn);
    const uint64_t adesc0 = make_sdesc(base, 16, 1024, kSw128);
    const uint64_t bdesc0 = b_mn ? make_sdesc(bslots, 8192, 1024, kSw128) : make_sdesc(bslots, 16, 1024, kSw128);
    const uint32_t kstep_b = b_mn ? (2048 >> 4) : (32 >> 4);  // next K = 16 slice of B
    int sa = 0, sb = 0, lt = 0;
    uint32_t pha = 0, phb = 0;
    const int nstage = p.nck * p.kh;
    if constexpr (RESB) mbar_wait(full_b(0), 0);
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
          if constexpr (RESB) {
            sb = st * KW + s;
          } else {
            mbar_wait(full_b(sb), phb);
            tc_fence_after();
          }
          const uint64_t bd = bdesc0 + static_cast<uint64_t>((sb * L::kBSlot) >> 4);
          if (leader) {
#pragma unroll
            for (int kk = 0; kk < kBKb / 16; ++kk) {
#pragma unroll
              for (int h = 0; h < 2; ++h)
                tc_mma_bf16(d0 + h * BN, ad + static_cast<uint64_t>(((h * kBM + s) * 128 + kk * 32) >> 4),
                            bd + static_cast<uint64_t>(kk * kstep_b), idesc, (first && kk == 0) ? 0u : 1u);
            }
            if constexpr (!RESB) tc_commit(empty_b(sb));
          }
          __syncwarp();
          first = 0;
          if (RESB) continue;
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
  } else if (warp < 4 || warp >= 6) {
    // ---------------- epilogue ----------------
    const int hsel = warp < 4 ? 0 : 1;
    const int qw = warp & 3;
    const int row = qw * 32 + lane;
    int lt = 0;
    for (int tile = blockIdx.x; tile < p.ntiles; tile += gridDim.x, ++lt) {
      const int acc = lt & 1;
      const int tn = tile % p.ntn, t2 = tile / p.ntn;
      const int th = t2 % p.tiles_h, n = t2 / p.tiles_h;
      const int y0 = th * p.TH, n0 = tn * BN;
      mbar_wait_sleep(tfull(acc), (lt >> 1) & 1);
      tc_fence_after();
      {
        const int h = hsel;
        const int v = h * kBM + row;
        const int yl = v / p.P, x = v - yl * p.P, y = y0 + yl;
        const bool valid = yl < p.TH && x < p.Wout && y < p.Hout;
        const int64_t pix = (static_cast<int64_t>(n) * p.Hout + y) * p.Wout + x;
        const uint32_t taddr = tmem + acc * L::kAccCols + h * BN + (static_cast<uint32_t>(qw * 32) << 16);
#pragma unroll 1
        for (int cg = 0; cg < BN / 32; ++cg) {
          float vals[32];
          tmem_ld32(taddr + cg * 32, vals);
          if (cg == BN / 32 - 1) {
            // last TMEM read of this accumulator set: hand it back to the MMA warp
            tc_fence_before();
            mbar_arrive(tempty(acc));
          }
          const int nb = n0 + cg * 32;
          if (p.relu) {
#pragma unroll
            for (int i = 0; i < 32; ++i) vals[i] = fmaxf(vals[i], 0.f);
          }
          if (p.epi_t && !p.accum && nb < p.Cout) {  // warp-uniform; rows of invalid pixels store nothing
            const int64_t at = pix * p.Cout + nb;
            store_tile32_t(bars + 256 + (hsel * 4 + qw) * 2048, vals, valid ? p.out + at : nullptr,
                           p.mask_x ? p.mask_x + at : nullptr);
            continue;
          }
          if (!valid || nb >= p.Cout) continue;
          if (p.mask_x) {
            const uint4* xr = reinterpret_cast<const uint4*>(p.mask_x + pix * p.Cout + nb);
            uint4 xa[4];  // loads in flight together, then the selects
#pragma unroll
            for (int i = 0; i < 4; ++i) xa[i] = __ldg(xr + i);
#pragma unroll
            for (int i = 0; i < 4; ++i) {
              float f[8];
              unpack_bf16x8(xa[i], f);
#pragma unroll
              for (int t = 0; t < 8; ++t) vals[8 * i + t] = f[t] > 0.f ? vals[8 * i + t] : 0.f;
            }
          }
          store_row32(p.out + pix * p.Cout + nb, vals, 32, p.accum != 0);
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
// dW[co][r][s][ci] = sum_p dY[p][co] * X[p + r*P + s][ci] on the virtual pixel
// grid (pitch P = W + 2*pad; dY is 0 on the garbage columns x >= Wout, which
// the TMA box's out-of-bounds fill provides). One pipeline unit is one output
// row: B = that dY row (Cout/64 MN-major chunks of Kp pixel rows), and per
// block (tap row r, 64-channel chunk c) of this CTA's group one TMA box of the
// padded input row y + r - pad. A K = 16 MMA reads M = 128 rows = two
// shifted views of that ONE staged box: MN-major chunks LBO = 128 B apart, so
// A[(v, ci)][k] = X[k + s0 + v][ci] (SWIZZLE_128B is address-based, as for
// the fprop halo kernel); two MMAs per K step cover the views s = 0..3 (s = 3
// unused for 3x3: 75% of the rows useful), and every input row is staged
// once per (r, c) instead of once per tap (the im2col wgrad stages it 9
// times). A CTA owns G blocks (G x 2 x Cout TMEM columns) and a range of
// rows; its fp32 partial [Cout][M] (M rows = (tap, 64-chunk, ci), the layout
// wgrad_reduce_b_kernel sums) goes to slab z.
struct HaloWgParamsB {
  int N, H, W, C, Cout, kh, kw, pad, P, Kp, Hout, Wout, nck;
  int G, ngroups, rows_per, nrows, M;
  int AS, BS;               // ring depths (A: one padded input row per (r, c); B: one dY row)
  uint32_t a_slot, b_slot;  // bytes per slot (1024-aligned)
  float* part;              // [splits][Cout][M]
};
constexpr int kHwbMaxAS = 4;
inline uint32_t halo_wgb_a_slot(int Kp) { return ((static_cast<uint32_t>(Kp) + 8) * 128 + 1023u) & ~1023u; }
inline uint32_t halo_wgb_b_slot(int Kp, int bn) {
  return ((static_cast<uint32_t>(bn / 64) * Kp * 128) + 1023u) & ~1023u;
}

template <int BN>
__global__ void __launch_bounds__(192, 1) tcb_wgrad_halo_kernel(const __grid_constant__ HaloWgParamsB p,
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
  const int ncol = G * 2 * BN;
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
  // garbage pixels), A rows [P, a_slot / 128) must be finite
  for (int s = 0; s < AS; ++s)
    for (uint32_t o = p.P * 128 + threadIdx.x * 16; o < p.a_slot; o += blockDim.x * 16)
      asm volatile("st.shared.v4.u32 [%0], {%1, %1, %1, %1};" ::"r"(base + s * p.a_slot + o), "r"(0) : "memory");
  for (int s = 0; s < BS; ++s)
    for (int ch = 0; ch < BN / 64; ++ch)
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
      const uint32_t abytes = static_cast<uint32_t>(p.P) * 128, bbytes = (BN / 64) * abytes;
      for (int row = row0; row < row1; ++row) {
        const int n = row / p.Hout, y = row - n * p.Hout;
        mbar_wait(empty_b(sb), phb);
        mbar_expect_tx(full_b(sb), bbytes);
        for (int ch = 0; ch < BN / 64; ++ch)
          tma_load_4d(bslots + sb * p.b_slot + ch * p.Kp * 128, &tma_dy, full_b(sb), ch * 64, 0, y, n);
        if (++sb == BS) {
          sb = 0;
          phb ^= 1;
        }
        for (int j = 0; j < G; ++j) {
          const int blk = g0 + j, r = blk / p.nck, c = blk - r * p.nck;
          mbar_wait(empty_a(sa), pha);
          mbar_expect_tx(full_a(sa), abytes);
          tma_load_4d(base + sa * p.a_slot, &tma_x, full_a(sa), c * 64, -p.pad, y + r - p.pad, n);
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
    const uint32_t idesc = make_idesc_bf16(BN, true, true);
    const bool leader = elect_one();
    const int ksteps = p.Kp / 16;
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
          for (int kk = 0; kk < ksteps; ++kk) {
            const uint64_t bd = make_sdesc(b0 + kk * 2048, lbo_b, 1024, kSw128);
#pragma unroll
            for (int q = 0; q < 2; ++q)
              tc_mma_bf16(tmem + (j * 2 + q) * BN, make_sdesc(a0 + q * 256 + kk * 2048, 128, 1024, kSw128), bd, idesc,
                          (i > 0 || kk > 0) ? 1u : 0u);
          }
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
    // ---------------- epilogue: TMEM lane l = (view l / 64, ci = l % 64) ----------------
    mbar_wait_sleep(done_bar, 0);
    tc_fence_after();
    const int l = warp * 32 + lane;
    const int ci = l & 63;
    float* dst = p.part + static_cast<int64_t>(z) * p.Cout * p.M;
    for (int j = 0; j < G; ++j) {
      const int blk = g0 + j, r = blk / p.nck, c = blk - r * p.nck;
#pragma unroll 1
      for (int q = 0; q < 2; ++q) {
        const int s = 2 * q + (l >> 6);
        const int m = ((r * p.kw + s) * p.nck + c) * 64 + ci;
#pragma unroll 1
        for (int cg = 0; cg < BN / 32; ++cg) {
          float v[32];
          tmem_ld32(tmem + (j * 2 + q) * BN + cg * 32 + (static_cast<uint32_t>(warp * 32) << 16), v);
          if (s >= p.kw) continue;  // the fourth shifted view (taps past the kernel)
          if (nrows <= 0) {
#pragma unroll
            for (int t = 0; t < 32; ++t) v[t] = 0.f;
          }
#pragma unroll
          for (int t = 0; t < 32; ++t)
            if (cg * 32 + t < p.Cout) dst[static_cast<int64_t>(cg * 32 + t) * p.M + m] = v[t];
        }
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
