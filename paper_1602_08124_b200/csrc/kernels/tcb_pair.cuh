// CTA-pair (cta_group::2) variant of the BF16 engine's persistent kernel for
// TMA-fed layers with >= 256 output columns (included by conv_bf16.cu after
// tcb_conv.cuh and tc_conv_pair.cuh, whose cluster / pair-TMA / multicast
// commit helpers it uses).
//
// Why: a single-SM M128 x N256 x K16 kind::f16 MMA reads A (4 KB) + B (8 KB)
// from its own shared memory and the stage fill is A 16 KB + B 32 KB per 64
// channels: the same operand-read / fill ratio that capped the fp32 engine's
// single-CTA N = 256 tiles (tc_conv_pair.cuh). On a CTA pair each SM holds its
// own 128 A rows and HALF of B (128 of 256 columns), the pair's M256 x N256
// MMA exchanges the B halves: per SM and K step 4 KB + 4 KB of operand reads
// for the FLOPs of an N = 256 tile, and 32 KB of fill per stage instead of 48.
//
//   cluster (2,1,1); rank 0 = leader. A pair walks (split, 256-row M tile,
//   256-column N tile) items; CTA rank r stages A rows m0 + 128r and B
//   columns n0 + 128r (fprop: 128 K-major W rows; dgrad: two 64-ci MN-major
//   W^T chunks; wgrad: two 64-co MN-major dY chunks).
//   warps 0-3, 6-9 : epilogue of this CTA's 128 rows, one column half per
//               warpgroup (tcb_epilogue: fused bias / ReLU / ReLU-backward
//               mask / accumulate, SGD / dW, partials)
//   warp 4    : TMEM alloc (cta_group::2, both CTAs); in the leader the MMA
//               issuer (tcgen05.mma.cta_group::2.kind::f16, M256 N256 K16)
//   warp 5    : TMA producer of this CTA's halves; both CTAs' loads complete
//               on the LEADER's full barrier, whose single expect_tx arrive
//               covers both CTAs' bytes; empty / tfull: multicast commits;
//               tempty: 512 arrivals in the leader (both CTAs' two epilogue
//               warpgroups, warps 0-3 and 6-9).
// Two TMEM accumulator sets (2 x 256 columns per SM): tile t's epilogue
// overlaps tile t+1's main loop.
#pragma once

namespace vdnnk {

__device__ __forceinline__ void tc_mma_bf16_pair(uint32_t d_tmem, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                                 uint32_t accumulate) {
  asm volatile(
      "{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n"
      " tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n}\n" ::"r"(d_tmem),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate)
      : "memory");
}

template <int STAGES>
struct TcbPairSmem {
  static constexpr int kABytes = kBM * 128;  // this CTA's 128 A rows (or 2 MN chunks) x 64 bf16
  static constexpr int kBBytes = 128 * 128;  // this CTA's half of B: 128 rows (or 2 MN chunks) x 64 bf16
  static constexpr int kStage = kABytes + kBBytes;
  static constexpr int kEpiScratch = 8 * 2048;  // store_tile32_t transpose, one 2 KB block per epilogue warp
  static constexpr int kTotal = STAGES * kStage + 1024 + 256 + kEpiScratch;
};

// Two epilogue warpgroups (warps 0-3: columns [0, 128), warps 6-9: columns
// [128, 256) of the tile; TMEM lane quarter = warp % 4): the stores -- and
// the W round trips of a fused-SGD wgrad -- of both column halves are in
// flight together.
constexpr int kTcbPairThreads = 320;
template <int STAGES>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(kTcbPairThreads, 1)
    tcb_pair_kernel(const __grid_constant__ ConvParamsB p, const __grid_constant__ CUtensorMap tma_a,
                    const __grid_constant__ CUtensorMap tma_b, int splits, int epi_t) {
  using L = TcbPairSmem<STAGES>;
  constexpr int BN = 256;
  constexpr int kTmemCols = 2 * BN;
  extern __shared__ uint8_t smem_raw[];
  const uint32_t base = (smem_u32(smem_raw) + 1023u) & ~1023u;
  const uint32_t bars = base + STAGES * L::kStage;
  auto full_bar = [&](int s) { return bars + 8u * s; };
  auto empty_bar = [&](int s) { return bars + 8u * (STAGES + s); };
  auto tfull = [&](int a) { return bars + 8u * (2 * STAGES + a); };
  auto tempty = [&](int a) { return bars + 8u * (2 * STAGES + 2 + a); };
  const uint32_t tmem_slot = bars + 8u * (2 * STAGES + 4);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t rank = cluster_ctarank();
  const int pair = static_cast<int>(blockIdx.x >> 1), npairs = static_cast<int>(gridDim.x >> 1);
  const int ntn = (p.Ncols + BN - 1) / BN;
  const int mt = (p.M + 255) / 256;
  const int ntiles = mt * ntn * splits;
  // item -> (split z, this CTA's m0, n0, K-block range); the N tiles of one M
  // tile are adjacent (the A rows are re-hit in L2)
  auto decode = [&](int t, int& z, int& m0, int& n0, int& kb0, int& nkb) {
    z = t / (mt * ntn);
    const int r = t - z * mt * ntn;
    m0 = (r / ntn) * 256 + static_cast<int>(rank) * kBM;
    n0 = (r % ntn) * BN;
    kb0 = z * p.kb_per_split;
    nkb = min(p.kblocks, kb0 + p.kb_per_split) - kb0;
  };

  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(full_bar(s), 1);  // the leader's expect_tx arrive (covers both CTAs' bytes)
      mbar_init(empty_bar(s), 1);
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(tfull(a), 1);
      mbar_init(tempty(a), 512);  // both CTAs' two epilogue warpgroups
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

  if (warp == 5) {
    // ---------------- TMA producer (this CTA's A rows and B half) ----------------
    if (lane == 0) {
      asm volatile("prefetch.tensormap [%0];" ::"l"(&tma_a) : "memory");
      asm volatile("prefetch.tensormap [%0];" ::"l"(&tma_b) : "memory");
      int s = 0;
      uint32_t ph = 1;  // the first pass over the ring does not wait
      for (int t = pair; t < ntiles; t += npairs) {
        int z, m0, n0, kb0, nkb;
        decode(t, z, m0, n0, kb0, nkb);
        const int nb = n0 + static_cast<int>(rank) * 128;  // this CTA's B columns
        TmaProducerB<BN> tp;
        tp.init(p, m0, kb0);
        for (int it = 0; it < nkb; ++it) {
          mbar_wait(empty_bar(s), ph);
          const uint32_t sa = base + s * L::kStage, sb = sa + L::kABytes;
          // only the leader arrives, expecting both CTAs' bytes (tc_conv_pair.cuh)
          const uint32_t lbar = map_to_rank(full_bar(s), 0);
          if (rank == 0) mbar_expect_tx(full_bar(s), 2 * L::kStage);
          if (p.kind == kFprop) {
            tma_load_im2col_pair(sa, &tma_a, lbar, tp.ck * 64, tp.qw, tp.qh, tp.qn, static_cast<uint16_t>(tp.s),
                                 static_cast<uint16_t>(tp.r));
            tma_load_3d_pair(sb, &tma_b, lbar, tp.ck * 64, tp.r * p.kw + tp.s, nb);
          } else if (p.kind == kDgrad) {
            tma_load_im2col_pair(sa, &tma_a, lbar, tp.ck * 64, tp.qw, tp.qh, tp.qn, static_cast<uint16_t>(tp.s),
                                 static_cast<uint16_t>(tp.r));
            const int ftap = (p.kh - 1 - tp.r) * p.kw + (p.kw - 1 - tp.s);
#pragma unroll
            for (int mc = 0; mc < 2; ++mc) tma_load_3d_pair(sb + mc * 8192, &tma_b, lbar, nb + mc * 64, ftap, tp.ck * 64);
          } else {
            // wgrad (host: M % 256 == 0, so both A chunks of every CTA are real)
            const int iw = tp.pw * p.stride - p.pad, ih = tp.ph * p.stride - p.pad;
#pragma unroll
            for (int mc = 0; mc < 2; ++mc)
              tma_load_im2col_pair(sa + mc * 8192, &tma_a, lbar, tp.wch[mc], iw, ih, tp.pn,
                                   static_cast<uint16_t>(tp.ws[mc]), static_cast<uint16_t>(tp.wr[mc]));
#pragma unroll
            for (int mc = 0; mc < 2; ++mc) tma_load_2d_pair(sb + mc * 8192, &tma_b, lbar, nb + mc * 64, tp.p0);
          }
          tp.next(p);
          if (++s == STAGES) {
            s = 0;
            ph ^= 1;
          }
        }
      }
    }
    __syncwarp();
  } else if (warp == 4) {
    // ---------------- MMA issuer (leader CTA) ----------------
    if (rank == 0) {
      const bool a_mn = p.kind == kWgrad;
      const bool b_mn = p.kind != kFprop;
      const uint32_t idesc = (make_idesc_bf16(BN, a_mn, b_mn) & ~(0x1Fu << 24)) | ((256u >> 4) << 24);
      const bool leader = elect_one();
      int s = 0, lt = 0;
      uint32_t ph = 0;
      for (int t = pair; t < ntiles; t += npairs, ++lt) {
        int z, m0, n0, kb0, nkb;
        decode(t, z, m0, n0, kb0, nkb);
        const int acc = lt & 1;
        if (lt >= 2) mbar_wait(tempty(acc), ((lt >> 1) & 1) ^ 1);
        tc_fence_after();
        const uint32_t d = tmem + acc * BN;
        for (int it = 0; it < nkb; ++it) {
          mbar_wait(full_bar(s), ph);
          tc_fence_after();
          const uint32_t sa = base + s * L::kStage, sb = sa + L::kABytes;
          if (leader) {
#pragma unroll
            for (int kk = 0; kk < kBKb / 16; ++kk) {
              const uint64_t ad = a_mn ? make_sdesc(sa + kk * 2048, 8192, 1024, kSw128)
                                       : make_sdesc(sa + kk * 32, 16, 1024, kSw128);
              const uint64_t bd = b_mn ? make_sdesc(sb + kk * 2048, 8192, 1024, kSw128)
                                       : make_sdesc(sb + kk * 32, 16, 1024, kSw128);
              tc_mma_bf16_pair(d, ad, bd, idesc, (it > 0 || kk > 0) ? 1u : 0u);
            }
            tc_commit_pair(empty_bar(s));
          }
          __syncwarp();
          if (++s == STAGES) {
            s = 0;
            ph ^= 1;
          }
        }
        if (leader) tc_commit_pair(tfull(acc));
        __syncwarp();
      }
    }
  } else if (warp < 4 || warp >= 6) {
    // ---------------- epilogue (this CTA's 128 rows, one column half per warpgroup) ----------------
    const int qw = warp & 3, chalf = warp < 4 ? 0 : 1;
    const uint32_t lt0 = map_to_rank(tempty(0), 0), lt1 = map_to_rank(tempty(1), 0);
    int lt = 0;
    for (int t = pair; t < ntiles; t += npairs, ++lt) {
      int z, m0, n0, kb0, nkb;
      decode(t, z, m0, n0, kb0, nkb);
      const int acc = lt & 1;
      mbar_wait_sleep(tfull(acc), (lt >> 1) & 1);
      tc_fence_after();
      const uint32_t ta = tmem + acc * BN + (static_cast<uint32_t>(qw * 32) << 16);
      tcb_epilogue<BN>(p, ta, m0, n0, z, qw * 32 + lane, nkb <= 0, [&] {
        // last TMEM read of this accumulator set: release it to the leader's MMA warp
        tc_fence_before();
        mbar_arrive_cluster(acc ? lt1 : lt0);
      }, chalf * (BN / 64), (chalf + 1) * (BN / 64),
                     epi_t ? bars + 256 + (chalf * 4 + qw) * 2048 : 0u);
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
