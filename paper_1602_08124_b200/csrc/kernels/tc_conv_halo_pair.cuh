// CTA-pair (cta_group::2) variant of the halo-reuse FPROP / DGRAD kernel
// (tc_conv_halo.cuh; included by conv.cu after tc_conv_pair.cuh).
//
// Why: the halo kernel's N = 64 / 128 MMAs are bound by the tensor core's
// shared-memory operand reads (ncu: TC wavefronts 78-83% busy, tensor pipe
// 48-56%): per M128 x N x K8 MMA a single SM reads 4 KB of A and N x 32 B of
// B. On a CTA pair each SM keeps its own 128 A rows but only HALF of B (the
// pair exchanges the halves), so per SM and MMA of the same FLOPs it reads
// 4 KB + N x 16 B: 6 -> 5 KB at N = 64, 8 -> 6 KB at N = 128.
//
//   cluster (2,1,1); rank 0 = leader. Pair tile = (image n, row-tile pair
//   thp, column block tn): CTA rank r owns output rows th = 2*thp + r (TH rows
//   of the virtual pitch-P grid, two M=256 pair MMAs per tap: h = 0, 1) and
//   stages its own padded input box plus B rows n0 + r*BN/2. A rank-1 tile past
//   the last row tile computes on TMA zero fill and stores nothing.
//   warps 0-3, 6-9 : epilogue of this CTA's 256 virtual rows, one M half per
//               warpgroup (kHaloEpiGroups; TMEM lane quarter = warp % 4)
//   warp 4    : TMEM alloc (cta_group::2); in the leader the MMA issuer
//   warp 5    : TMA producer; both CTAs' loads complete on the LEADER's full
//               barriers (.cta_group::2 TMA), the leader's single arrive
//               expects both CTAs' bytes; empty / tfull barriers are
//               multicast commits; tempty counts 256 arrivals per epilogue
//               warpgroup in the leader (kHaloEpiGroups, both CTAs).
// RESB: when one CTA's half of the whole filter fits next to the A ring
// (64 -> 64 channels: 9 taps x 2 chunks x 4 KB = 72 KB), B is loaded once per
// CTA and stays resident: the per-tile B stream (as many L2 -> SM bytes as
// the A boxes at 64 columns) disappears.
#pragma once

namespace vdnnk {

// Warp-cooperative store of 16 fp32 columns of 32 rows (row r in lane r, the
// TMEM lane layout) through a 2 KB per-warp shared-memory transpose: a warp's
// 16-B st.global then covers 8 rows x 64 B (full sectors) instead of 32 rows
// x 16 B. dst / mask: this lane's row at the first column (null: row not
// stored / no ReLU mask); the mask chunks are loaded before the transpose and
// selected per element after it (the same x > 0 select as the per-lane path,
// so the stored values are bit-identical). Chunk index XOR (row >> 1) & 3:
// conflict-free row writes and chunk reads.
__device__ __forceinline__ void store_half32_f32(uint32_t scratch, const float* v, float* dst, const float* mask) {
  const int lane = threadIdx.x & 31;
  const int q = lane & 3;
  float* d[4];
  float4 x[4];
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int r = 8 * i + (lane >> 2);
    d[i] = reinterpret_cast<float*>(__shfl_sync(0xffffffffu, reinterpret_cast<uintptr_t>(dst), r));
    const float* mk = reinterpret_cast<const float*>(__shfl_sync(0xffffffffu, reinterpret_cast<uintptr_t>(mask), r));
    x[i] = make_float4(1.f, 1.f, 1.f, 1.f);
    if (mk && d[i]) x[i] = __ldg(reinterpret_cast<const float4*>(mk) + q);
  }
  __syncwarp();  // the previous block's chunk reads are done
#pragma unroll
  for (int c = 0; c < 4; ++c)
    asm volatile("st.shared.v4.f32 [%0], {%1, %2, %3, %4};" ::"r"(scratch + lane * 64 + ((c ^ ((lane >> 1) & 3)) << 4)),
                 "f"(v[4 * c]), "f"(v[4 * c + 1]), "f"(v[4 * c + 2]), "f"(v[4 * c + 3])
                 : "memory");
  __syncwarp();
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int r = 8 * i + (lane >> 2);
    float4 w;
    asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];"
                 : "=f"(w.x), "=f"(w.y), "=f"(w.z), "=f"(w.w)
                 : "r"(scratch + r * 64 + ((q ^ ((r >> 1) & 3)) << 4))
                 : "memory");
    if (d[i])
      reinterpret_cast<float4*>(d[i])[q] = make_float4(x[i].x > 0.f ? w.x : 0.f, x[i].y > 0.f ? w.y : 0.f,
                                                       x[i].z > 0.f ? w.z : 0.f, x[i].w > 0.f ? w.w : 0.f);
  }
}

template <int BN, int AS, int BS>
struct HaloPairSmem {
  static constexpr int kASlot = 33 * 1024;       // >= 258 rows x 128 B
  static constexpr int kBSlot = (BN / 2) * 128;  // this CTA's half of B
  static constexpr int kEpiScratch = 8 * 2048;  // store_half32_f32 transpose, one 2 KB block per epilogue warp
  static constexpr int kTotal = AS * kASlot + BS * kBSlot + 1024 + 256 + kEpiScratch;
  static int total(int nbslots) { return AS * kASlot + nbslots * kBSlot + 1024 + 256 + kEpiScratch; }
  static constexpr int kAccCols = 2 * BN;  // h = 0, 1
  static_assert(2 * kAccCols <= 512, "two accumulator sets must fit TMEM");
};

// Epilogue warpgroups: group 0 = warps 0-3, group g >= 1 = warps 6 + 4(g-1)
// .. (TMEM lane quarter = warp % 4); group g drains M half g % 2 and column
// half g / 2 of the tile, so the dgrad's ReLU-mask loads and the stores of
// the whole tile are in flight together (with one warpgroup the epilogue --
// four serial DRAM round trips per tile -- bounded the 224x224x64 dgrad:
// tensor pipe 36% active, long-scoreboard stalls; 2.73 -> 2.43 ms with two;
// four measured slower, 2.86).
constexpr int kHaloEpiGroups = 2;
constexpr int kHaloPairThreads = 32 * (6 + 4 * (kHaloEpiGroups - 1));
template <int BN, int AS, int BS, int KW, bool RESB = false>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(kHaloPairThreads, 1)
    tc_conv_halo_pair_kernel(const __grid_constant__ HaloParams p, const __grid_constant__ CUtensorMap tma_a,
                             const __grid_constant__ CUtensorMap tma_b) {
  using L = HaloPairSmem<BN, AS, BS>;
  constexpr int kTmemCols = 2 * L::kAccCols;
  extern __shared__ uint8_t smem_raw[];
  const uint32_t base = (smem_u32(smem_raw) + 1023u) & ~1023u;
  const uint32_t bslots = base + AS * L::kASlot;
  const int nbslots = RESB ? p.nck * p.kh * KW : BS;
  const uint32_t bars = bslots + static_cast<uint32_t>(nbslots) * L::kBSlot;
  auto full_a = [&](int s) { return bars + 8u * s; };
  auto empty_a = [&](int s) { return bars + 8u * (AS + s); };
  auto full_b = [&](int s) { return bars + 8u * (2 * AS + s); };
  auto empty_b = [&](int s) { return bars + 8u * (2 * AS + BS + s); };
  auto tfull = [&](int a) { return bars + 8u * (2 * AS + 2 * BS + a); };
  auto tempty = [&](int a) { return bars + 8u * (2 * AS + 2 * BS + 2 + a); };
  const uint32_t tmem_slot = bars + 8u * (2 * AS + 2 * BS + 4);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t rank = cluster_ctarank();
  const int pair = static_cast<int>(blockIdx.x >> 1), npairs = static_cast<int>(gridDim.x >> 1);
  const int tiles_hp = (p.tiles_h + 1) >> 1;
  const int ntiles = p.N * tiles_hp * p.ntn;

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
      mbar_init(tempty(a), 256 * kHaloEpiGroups);  // both CTAs' epilogue warpgroups
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 4) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(tmem_slot),
                 "r"(kTmemCols)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
  }
  tc_fence_before();
  __syncthreads();
  cluster_sync_all();
  tc_fence_after();
  uint32_t tmem;
  asm volatile("ld.shared.u32 %0, [%1];" : "=r"(tmem) : "r"(tmem_slot) : "memory");

  const uint32_t abytes = static_cast<uint32_t>(p.TH * p.P * 128);
  if (warp == 5) {
    // ---------------- TMA producer (this CTA's rows and B half) ----------------
    if (lane == 0) {
      asm volatile("prefetch.tensormap [%0];" ::"l"(&tma_a) : "memory");
      asm volatile("prefetch.tensormap [%0];" ::"l"(&tma_b) : "memory");
      int sa = 0, sb = 0;
      uint32_t pha = 1, phb = 1;  // the first pass over each ring does not wait
      if constexpr (RESB) {  // the whole filter half, once, on full_b(0)
        const int nb = static_cast<int>(rank) * (BN / 2);
        if (rank == 0) mbar_expect_tx(full_b(0), 2u * nbslots * L::kBSlot);
        const uint32_t lb = map_to_rank(full_b(0), 0);
        for (int c = 0; c < p.nck; ++c)
          for (int r = 0; r < p.kh; ++r)
            for (int s = 0; s < KW; ++s) {
              const uint32_t dst = bslots + ((c * p.kh + r) * KW + s) * L::kBSlot;
              if (p.kind == kFprop) {
                tma_load_2d_pair(dst, &tma_b, lb, (r * KW + s) * p.Cin + c * 32, nb);
              } else {
                const int ftap = (p.kh - 1 - r) * KW + (KW - 1 - s);
                tma_load_4d_pair(dst, &tma_b, lb, 0, c * 32, nb >> 5, ftap);
              }
            }
      }
      for (int tile = pair; tile < ntiles; tile += npairs) {
        const int tn = tile % p.ntn, t2 = tile / p.ntn;
        const int thp = t2 % tiles_hp, n = t2 / tiles_hp;
        const int y0 = (2 * thp + static_cast<int>(rank)) * p.TH;
        const int nb = tn * BN + static_cast<int>(rank) * (BN / 2);
        if (p.mask_x && tn == 0 && y0 < p.Hout) {
          // the dgrad epilogue's ReLU mask (x rows of this CTA's output rows,
          // every channel) into L2 while the main loop runs: its loads then
          // hit L2 instead of serialising DRAM round trips per column group
          const int rows = min(p.TH, p.Hout - y0);
          prefetch_l2_bulk(p.mask_x + (static_cast<int64_t>(n) * p.Hout + y0) * p.Wout * p.Cout,
                           static_cast<uint64_t>(rows) * p.Wout * p.Cout * sizeof(float));
        }
        for (int c = 0; c < p.nck; ++c) {
          for (int r = 0; r < p.kh; ++r) {
            mbar_wait(empty_a(sa), pha);
            // only the leader arrives (expecting both CTAs' bytes); see tc_conv_pair.cuh
            if (rank == 0) mbar_expect_tx(full_a(sa), 2 * abytes);
            tma_load_4d_pair(base + sa * L::kASlot, &tma_a, map_to_rank(full_a(sa), 0), c * 32, -p.pad,
                             y0 + r - p.pad, n);
            if (++sa == AS) {
              sa = 0;
              pha ^= 1;
            }
            if constexpr (!RESB) {
#pragma unroll
              for (int s = 0; s < KW; ++s) {
                mbar_wait(empty_b(sb), phb);
                if (rank == 0) mbar_expect_tx(full_b(sb), 2 * L::kBSlot);
                const uint32_t lb = map_to_rank(full_b(sb), 0);
                if (p.kind == kFprop) {
                  tma_load_2d_pair(bslots + sb * L::kBSlot, &tma_b, lb, (r * KW + s) * p.Cin + c * 32, nb);
                } else {
                  const int ftap = (p.kh - 1 - r) * KW + (KW - 1 - s);
                  tma_load_4d_pair(bslots + sb * L::kBSlot, &tma_b, lb, 0, c * 32, nb >> 5, ftap);
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
    }
    __syncwarp();
  } else if (warp == 4) {
    // ---------------- MMA issuer (leader CTA) ----------------
    if (rank == 0) {
      const bool leader = elect_one();
      const bool b_mn = p.kind != kFprop;
      const uint32_t idesc = (make_idesc_tf32(BN, false, b_mn) & ~(0x1Fu << 24)) | ((256u >> 4) << 24);
      const uint64_t adesc0 = make_sdesc(base, 16, 1024, kSw128);
      const uint64_t bdesc0 =
          b_mn ? make_sdesc(bslots, 4096, 512, kSw128Base32) : make_sdesc(bslots, 16, 1024, kSw128);
      const uint32_t kstep_b = b_mn ? (1024 >> 4) : (32 >> 4);
      int sa = 0, sb = 0, lt = 0;
      uint32_t pha = 0, phb = 0;
      const int nstage = p.nck * p.kh;
      if constexpr (RESB) mbar_wait(full_b(0), 0);
      for (int tile = pair; tile < ntiles; tile += npairs, ++lt) {
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
            }
            tc_fence_after();
            const uint64_t bd = bdesc0 + static_cast<uint64_t>((sb * L::kBSlot) >> 4);
            if (leader) {
#pragma unroll
              for (int kk = 0; kk < kBK / 8; ++kk) {
#pragma unroll
                for (int h = 0; h < 2; ++h)
                  tc_mma_tf32_pair(d0 + h * BN, ad + static_cast<uint64_t>(((h * kBM + s) * 128 + kk * 32) >> 4),
                                   bd + static_cast<uint64_t>(kk * kstep_b), idesc,
                                   (first && kk == 0) ? 0u : 1u);
              }
              if constexpr (!RESB) tc_commit_pair(empty_b(sb));
            }
            __syncwarp();
            first = 0;
            if (RESB) continue;
            if (++sb == BS) {
              sb = 0;
              phb ^= 1;
            }
          }
          if (leader) tc_commit_pair(empty_a(sa));
          __syncwarp();
          if (++sa == AS) {
            sa = 0;
            pha ^= 1;
          }
        }
        if (leader) tc_commit_pair(tfull(acc));
        __syncwarp();
      }
    }
  } else if (warp < 4 || warp >= 6) {
    // ---------------- epilogue (this CTA's 256 virtual rows) ----------------
    const int gi = warp < 4 ? 0 : 1 + (warp - 6) / 4;
    const int hsel = gi & 1;
    const int cgs = (BN / 32) / (kHaloEpiGroups / 2);  // column groups per warpgroup
    const int cg0 = (gi >> 1) * cgs;
    const int qw = warp & 3;
    const int row = qw * 32 + lane;
    const uint32_t ltempty0 = map_to_rank(tempty(0), 0), ltempty1 = map_to_rank(tempty(1), 0);
    int lt = 0;
    for (int tile = pair; tile < ntiles; tile += npairs, ++lt) {
      const int acc = lt & 1;
      const int tn = tile % p.ntn, t2 = tile / p.ntn;
      const int thp = t2 % tiles_hp, n = t2 / tiles_hp;
      const int y0 = (2 * thp + static_cast<int>(rank)) * p.TH, n0 = tn * BN;
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
        for (int cg = cg0; cg < cg0 + cgs; ++cg) {
          float vals[32];
          tmem_ld32(taddr + cg * 32, vals);
          if (cg == cg0 + cgs - 1) {
            // last TMEM read of this accumulator set: release it to the leader's MMA warp
            tc_fence_before();
            mbar_arrive_cluster(acc ? ltempty1 : ltempty0);
          }
          const int nb = n0 + cg * 32;
          if (p.relu) {
#pragma unroll
            for (int i = 0; i < 32; ++i) vals[i] = fmaxf(vals[i], 0.f);
          }
          // 64-column tiles only: at BN = 128 the A/B of tools/ab_halo_epi_t.sh measured no gain
          // (112^2 layers 0.89-0.92 -> 0.94 ms), at BN = 64 224^2x64 fprop 2.05-2.11 -> 1.90-1.93 ms
          if (BN == 64 && p.epi_t && !p.accum && nb < p.Cout) {  // warp-uniform; invalid pixels store nothing
            const int64_t at = pix * p.Cout + nb;
            const uint32_t scr = bars + 256 + ((warp < 4 ? warp : warp - 2) * 2048);
#pragma unroll
            for (int hh = 0; hh < 2; ++hh)
              store_half32_f32(scr, vals + 16 * hh, valid ? p.out + at + 16 * hh : nullptr,
                               p.mask_x ? p.mask_x + at + 16 * hh : nullptr);
            continue;
          }
          if (!valid || nb >= p.Cout) continue;
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
            float4 a[8];
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
  cluster_sync_all();  // the peer's MMAs / barrier traffic into this CTA are over
  if (warp == 4) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(kTmemCols) : "memory");
  }
}

}  // namespace vdnnk

namespace vdnnk {

// Halo WGRAD (tc_conv_halo.cuh) on a CTA pair, 64 output channels: a work
// item is a range of rows; CTA rank r of the pair owns (r, c) blocks
// g0 = r*G .. (its 128 M rows per MMA: the four shifted views of its staged
// input row) and stages dY channels 32r..32r+31 of each row (its half of B).
// One M256 x N64 pair MMA per K step covers two blocks: per SM the tensor
// core reads 4 KB of A + 1 KB of B instead of 4 + 2 KB (the single-CTA
// kernel is operand-read bound: ncu TC wavefronts 83%, tensor pipe 55%).
// Persistent over a FIXED number of items (the split-K partials and their
// reduce order do not depend on how many SMs the grid got, e.g. with an SM
// reserve for compressed transfers), two TMEM accumulator sets so item i's
// epilogue overlaps item i+1's main loop. Both CTAs walk the same items and
// G blocks per row in lockstep; loads complete on the leader's barriers,
// releases are multicast commits (see tc_conv_pair.cuh).
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(192, 1)
    tc_wgrad_halo_pair_kernel(const __grid_constant__ HaloWgParams p, const __grid_constant__ CUtensorMap tma_x,
                              const __grid_constant__ CUtensorMap tma_dy, int nitems) {
  constexpr int BN = 64;
  const int AS = p.AS, BS = p.BS;
  extern __shared__ uint8_t smem_raw[];
  const uint32_t base = (smem_u32(smem_raw) + 1023u) & ~1023u;
  const uint32_t bslots = base + AS * p.a_slot;
  const uint32_t bars = bslots + BS * p.b_slot;
  auto full_a = [&](int s) { return bars + 8u * s; };
  auto empty_a = [&](int s) { return bars + 8u * (AS + s); };
  auto full_b = [&](int s) { return bars + 8u * (2 * AS + s); };
  auto empty_b = [&](int s) { return bars + 8u * (2 * AS + BS + s); };
  auto tfull = [&](int a) { return bars + 8u * (2 * AS + 2 * BS + a); };
  auto tempty = [&](int a) { return bars + 8u * (2 * AS + 2 * BS + 2 + a); };
  const uint32_t tmem_slot = bars + 8u * (2 * AS + 2 * BS + 4);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t rank = cluster_ctarank();
  const int pair = static_cast<int>(blockIdx.x >> 1), npairs = static_cast<int>(gridDim.x >> 1);
  const int G = p.G;
  const int g0 = static_cast<int>(rank) * G;
  int acc_cols = 32;
  while (acc_cols < G * BN) acc_cols <<= 1;
  const int tcols = 2 * acc_cols;

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
      mbar_init(tempty(a), 256);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  // rows the boxes never write: B rows [P, Kp) must be 0, A rows [P, Kp + 8) finite
  for (int s = 0; s < AS; ++s)
    for (uint32_t o = p.P * 128 + threadIdx.x * 16; o < p.a_slot; o += blockDim.x * 16)
      asm volatile("st.shared.v4.u32 [%0], {%1, %1, %1, %1};" ::"r"(base + s * p.a_slot + o), "r"(0) : "memory");
  for (int s = 0; s < BS; ++s)
    for (int o = p.P * 128 + threadIdx.x * 16; o < p.Kp * 128; o += blockDim.x * 16)
      asm volatile("st.shared.v4.u32 [%0], {%1, %1, %1, %1};" ::"r"(bslots + s * p.b_slot + o), "r"(0) : "memory");
  fence_proxy_async();
  if (warp == 4) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(tmem_slot), "r"(tcols)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
  }
  tc_fence_before();
  __syncthreads();
  cluster_sync_all();
  tc_fence_after();
  uint32_t tmem;
  asm volatile("ld.shared.u32 %0, [%1];" : "=r"(tmem) : "r"(tmem_slot) : "memory");

  if (warp == 5) {
    // ---------------- TMA producer (this CTA's dY half and input rows) ----------------
    if (lane == 0) {
      asm volatile("prefetch.tensormap [%0];" ::"l"(&tma_x) : "memory");
      asm volatile("prefetch.tensormap [%0];" ::"l"(&tma_dy) : "memory");
      int sa = 0, sb = 0;
      uint32_t pha = 1, phb = 1;
      const uint32_t bytes = static_cast<uint32_t>(p.P) * 128;
      for (int item = pair; item < nitems; item += npairs) {
        const int row0 = item * p.rows_per, row1 = min(row0 + p.rows_per, p.nrows);
        for (int row = row0; row < row1; ++row) {
          const int n = row / p.Hout, y = row - n * p.Hout;
          mbar_wait(empty_b(sb), phb);
          if (rank == 0) mbar_expect_tx(full_b(sb), 2 * bytes);
          tma_load_4d_pair(bslots + sb * p.b_slot, &tma_dy, map_to_rank(full_b(sb), 0),
                           static_cast<int>(rank) * 32, 0, y, n);
          if (++sb == BS) {
            sb = 0;
            phb ^= 1;
          }
          for (int j = 0; j < G; ++j) {
            const int blk = g0 + j, r = blk / p.nck, c = blk - r * p.nck;
            mbar_wait(empty_a(sa), pha);
            if (rank == 0) mbar_expect_tx(full_a(sa), 2 * bytes);
            tma_load_4d_pair(base + sa * p.a_slot, &tma_x, map_to_rank(full_a(sa), 0), c * 32, -p.pad,
                             y + r - p.pad, n);
            if (++sa == AS) {
              sa = 0;
              pha ^= 1;
            }
          }
        }
      }
    }
    __syncwarp();
  } else if (warp == 4) {
    // ---------------- MMA issuer (leader) ----------------
    if (rank == 0) {
      const uint32_t idesc = (make_idesc_tf32(BN, true, true) & ~(0x1Fu << 24)) | ((256u >> 4) << 24);
      const bool leader = elect_one();
      const int ksteps = p.Kp / 8;
      const uint32_t lbo_b = static_cast<uint32_t>(p.Kp) * 128;
      int sa = 0, sb = 0, lt = 0;
      uint32_t pha = 0, phb = 0;
      for (int item = pair; item < nitems; item += npairs, ++lt) {
        const int acc = lt & 1;
        if (lt >= 2) mbar_wait(tempty(acc), ((lt >> 1) & 1) ^ 1);
        tc_fence_after();
        const uint32_t d0 = tmem + acc * acc_cols;
        const int nrows = min(p.rows_per, p.nrows - item * p.rows_per);
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
                tc_mma_tf32_pair(d0 + j * BN, make_sdesc(a0 + kk * 1024, 128, 512, kSw128Base32),
                                 make_sdesc(b0 + kk * 1024, lbo_b, 512, kSw128Base32), idesc,
                                 (i > 0 || kk > 0) ? 1u : 0u);
              tc_commit_pair(empty_a(sa));
            }
            __syncwarp();
            if (++sa == AS) {
              sa = 0;
              pha ^= 1;
            }
          }
          if (leader) tc_commit_pair(empty_b(sb));
          __syncwarp();
          if (++sb == BS) {
            sb = 0;
            phb ^= 1;
          }
        }
        if (leader) tc_commit_pair(tfull(acc));
        __syncwarp();
      }
    }
  } else {
    // ---------------- epilogue: warp w = shift s, lane = ci ----------------
    const uint32_t lt0 = map_to_rank(tempty(0), 0), lt1 = map_to_rank(tempty(1), 0);
    const int s = warp;
    int lt = 0;
    for (int item = pair; item < nitems; item += npairs, ++lt) {
      const int acc = lt & 1;
      mbar_wait_sleep(tfull(acc), (lt >> 1) & 1);
      tc_fence_after();
      float* dst = p.part + static_cast<int64_t>(item) * p.Cout * p.M;
      for (int j = 0; j < G; ++j) {
        const int blk = g0 + j, r = blk / p.nck, c = blk - r * p.nck;
        const int m = ((r * p.kw + s) * p.nck + c) * 32 + lane;
        for (int cg = 0; cg < BN / 32; ++cg) {
          float v[32];
          tmem_ld32(tmem + acc * acc_cols + j * BN + cg * 32 + (static_cast<uint32_t>(warp * 32) << 16), v);
          if (j == G - 1 && cg == BN / 32 - 1) {
            // last TMEM read of this accumulator set: release it to the leader's MMA warp
            tc_fence_before();
            mbar_arrive_cluster(acc ? lt1 : lt0);
          }
          if (s >= p.kw) continue;  // the fourth shifted view (taps past the kernel)
#pragma unroll
          for (int q = 0; q < 32; ++q)
            if (cg * 32 + q < p.Cout) dst[static_cast<int64_t>(cg * 32 + q) * p.M + m] = v[q];
        }
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  cluster_sync_all();
  if (warp == 4) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(tcols) : "memory");
  }
}

}  // namespace vdnnk
