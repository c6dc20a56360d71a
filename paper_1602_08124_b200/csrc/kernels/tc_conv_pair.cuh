// CTA-pair (cta_group::2) variant of the tcgen05 conv engine for FPROP /
// DGRAD with >= 256 output columns (included by conv.cu after tc_conv.cuh).
//
// Why: at N = 256 a single-SM M128 MMA reads A (4 KB) + B (8 KB) from its own
// shared memory per K=8 step, and the tensor core's operand reads saturate
// (ncu l1tex__data_pipe_tc_wavefronts 87%) well below the MMA rate. A CTA pair
// on the two SMs of a TPC runs M = 256 x N = 256 MMAs in which each SM holds
// its own 128 A rows and HALF of B (128 of the 256 columns) and the B halves
// are exchanged between the pair: per SM and K step 4 KB + 4 KB for twice the
// FLOPs of an N=128 MMA (tools/pair_probe.cu: 1,104 TFLOP/s streaming).
//
//   cluster (2,1,1); rank 0 = leader. A pair walks output tiles of 256 rows x
//   256 columns: CTA rank r stages A rows m0 + 128r and B rows n0 + 128r.
//   warps 0-3 : epilogue of this CTA's 128 rows (TMEM lanes = its rows)
//   warp 4    : TMEM alloc (cta_group::2, both CTAs); in the leader the MMA
//               issuer (tcgen05.mma.cta_group::2, M256 N256 K8)
//   warp 5    : TMA producer of this CTA's halves; both CTAs' loads complete
//               on the LEADER's full barrier (.cta_group::2 TMA), which
//               expects 2 x stage bytes from the leader's single arrive
//   empty / tfull barriers: one tcgen05.commit multicast to both CTAs.
//   tempty: in the leader, 256 arrivals (both CTAs' epilogue threads).
// Persistent over tiles, two TMEM accumulator sets (2 x 256 columns per SM).
#pragma once

namespace vdnnk {

__device__ __forceinline__ uint32_t cluster_ctarank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ void cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
// shared::cluster address of the same smem offset in CTA `rank` of the cluster
__device__ __forceinline__ uint32_t map_to_rank(uint32_t addr, uint32_t rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(addr), "r"(rank));
  return r;
}
__device__ __forceinline__ void mbar_arrive_cluster(uint32_t cluster_addr) {
  asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(cluster_addr) : "memory");
}
__device__ __forceinline__ void tc_mma_tf32_pair(uint32_t d_tmem, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                                 uint32_t accumulate) {
  asm volatile(
      "{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n"
      " tcgen05.mma.cta_group::2.kind::tf32 [%0], %1, %2, %3, p;\n}\n" ::"r"(d_tmem),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate)
      : "memory");
}
__device__ __forceinline__ void tc_commit_pair(uint32_t bar) {
  asm volatile(
      "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(bar),
      "h"(static_cast<uint16_t>(3))
      : "memory");
}
// TMA loads into this CTA's smem that complete on a barrier of either pair CTA
__device__ __forceinline__ void tma_load_2d_pair(uint32_t dst, const CUtensorMap* map, uint32_t bar, int x, int y) {
  asm volatile(
      "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%3, "
      "%4}], [%2];" ::"r"(dst),
      "l"(map), "r"(bar), "r"(x), "r"(y)
      : "memory");
}
__device__ __forceinline__ void tma_load_4d_pair(uint32_t dst, const CUtensorMap* map, uint32_t bar, int x, int y,
                                                 int z, int w) {
  asm volatile(
      "cp.async.bulk.tensor.4d.cta_group::2.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%3, "
      "%4, %5, %6}], [%2];" ::"r"(dst),
      "l"(map), "r"(bar), "r"(x), "r"(y), "r"(z), "r"(w)
      : "memory");
}
__device__ __forceinline__ void tma_load_im2col_pair(uint32_t dst, const CUtensorMap* map, uint32_t bar, int c, int w,
                                                     int h, int n, uint16_t ow, uint16_t oh) {
  asm volatile(
      "cp.async.bulk.tensor.4d.cta_group::2.shared::cluster.global.im2col.mbarrier::complete_tx::bytes [%0], [%1, "
      "{%3, %4, %5, %6}], [%2], {%7, %8};" ::"r"(dst),
      "l"(map), "r"(bar), "r"(c), "r"(w), "r"(h), "r"(n), "h"(ow), "h"(oh)
      : "memory");
}

__device__ __forceinline__ void tma_load_3d_pair(uint32_t dst, const CUtensorMap* map, uint32_t bar, int x, int y,
                                                 int z) {
  asm volatile(
      "cp.async.bulk.tensor.3d.cta_group::2.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%3, "
      "%4, %5}], [%2];" ::"r"(dst),
      "l"(map), "r"(bar), "r"(x), "r"(y), "r"(z)
      : "memory");
}

template <int STAGES, int KB = 1, int NOUT = 2>
struct PairSmem {
  static constexpr int kABytes = KB * kBM * 128;  // this CTA's 128 A rows x 32 fp32, per k-block
  static constexpr int kBBytes = KB * 128 * 128;  // this CTA's half of B: 128 rows (or 4 MN chunks) x 32 fp32
  static constexpr int kStage = kABytes + kBBytes;
  static constexpr int kOut = NOUT * 16384;  // TMA-store staging boxes (128 rows x 32 columns)
  static constexpr int kTotal = STAGES * kStage + kOut + 1024 + 256;
  static constexpr int kAccCols = 256;
};

// KB = k-blocks (32 channels each) per pipeline stage; p.kblocks % KB == 0.
template <int STAGES, int KB, int NOUT>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(192, 1)
    tc_conv_pair_kernel(const __grid_constant__ ConvParams p, const __grid_constant__ CUtensorMap tma_a,
                        const __grid_constant__ CUtensorMap tma_b, const __grid_constant__ CUtensorMap tma_c) {
  using L = PairSmem<STAGES, KB, NOUT>;
  constexpr int BN = 256;
  constexpr int kTmemCols = 2 * L::kAccCols;
  extern __shared__ uint8_t smem_raw[];
  const uint32_t raw = smem_u32(smem_raw);
  const uint32_t base = (raw + 1023u) & ~1023u;
  const uint32_t obuf = base + STAGES * L::kStage;
  const uint32_t bars = obuf + L::kOut;
  auto full_bar = [&](int s) { return bars + 8u * s; };
  auto empty_bar = [&](int s) { return bars + 8u * (STAGES + s); };
  auto tfull_bar = [&](int a) { return bars + 8u * (2 * STAGES + a); };
  auto tempty_bar = [&](int a) { return bars + 8u * (2 * STAGES + 2 + a); };
  const uint32_t tmem_slot = bars + 8u * (2 * STAGES + 4);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t rank = cluster_ctarank();
  const int pair = static_cast<int>(blockIdx.x >> 1), npairs = static_cast<int>(gridDim.x >> 1);
  const int ntn = (p.Ncols + BN - 1) / BN;
  const int ntiles = ((p.M + 255) / 256) * ntn;
  const int nkb = p.kblocks / KB;  // pipeline stages per tile

  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(full_bar(s), 1);  // leader's expect_tx arrive (covers both CTAs' bytes)
      mbar_init(empty_bar(s), 1);
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(tfull_bar(a), 1);
      mbar_init(tempty_bar(a), 256);
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
      int it = 0;
      for (int tile = pair; tile < ntiles; tile += npairs) {
        const int m0 = (tile / ntn) * 256 + static_cast<int>(rank) * kBM;
        const int n0 = (tile % ntn) * BN;
        const int nb = n0 + static_cast<int>(rank) * 128;  // this CTA's B rows / MN chunks
        TmaProducer<128, kBM, kBK> tp;
        tp.init(p, m0, 0);
        for (int kb = 0; kb < nkb; ++kb, ++it) {
          const int s = it % STAGES;
          if (it >= STAGES) mbar_wait(empty_bar(s), ((it / STAGES) & 1) ^ 1);
          const uint32_t sa = base + s * L::kStage, sb = sa + L::kABytes;
          // Only the leader arrives (expecting both CTAs' bytes). The peer's
          // complete_tx may land before that arrive; the phase cannot
          // complete early (the arrival is pending), and the peer cannot run
          // a phase ahead (it waited on empty[s], i.e. on the MMAs that
          // consumed the previous phase). A remote arrive here needs
          // .release.cluster, which waits for the CTA's earlier TMA loads and
          // serialised the ring (measured 0.9 us per stage).
          const uint32_t lbar = map_to_rank(full_bar(s), 0);
          if (rank == 0) mbar_expect_tx(full_bar(s), 2 * L::kStage);
#pragma unroll
          for (int j = 0; j < KB; ++j) {
            if (j > 0) tp.next(p);
            // A: im2col rows of this CTA's half; B: this CTA's half of the columns
            tma_load_im2col_pair(sa + j * 16384, &tma_a, lbar, tp.ck * 32, tp.qw[0], tp.qh[0], tp.qn[0],
                                 static_cast<uint16_t>(tp.s), static_cast<uint16_t>(tp.r));
            if (p.kind == kFprop) {
              tma_load_2d_pair(sb + j * 16384, &tma_b, lbar, (tp.r * p.kw + tp.s) * p.C + tp.ck * 32, nb);
            } else {
              const int ftap = (p.kh - 1 - tp.r) * p.kw + (p.kw - 1 - tp.s);
              tma_load_4d_pair(sb + j * 16384, &tma_b, lbar, 0, tp.ck * 32, nb >> 5, ftap);
            }
          }
          tp.next(p);
        }
      }
    }
    __syncwarp();
  } else if (warp == 4) {
    // ---------------- MMA issuer (leader CTA) ----------------
    if (rank == 0) {
      const bool b_mn = p.kind != kFprop;
      const uint32_t idesc = (make_idesc_tf32(BN, false, b_mn) & ~(0x1Fu << 24)) | ((256u >> 4) << 24);
      const bool leader = elect_one();
      int it = 0, lt = 0;
      for (int tile = pair; tile < ntiles; tile += npairs, ++lt) {
        const int acc = lt & 1;
        if (lt >= 2) mbar_wait(tempty_bar(acc), ((lt >> 1) & 1) ^ 1);
        tc_fence_after();
        const uint32_t d0 = tmem + acc * L::kAccCols;
        for (int kb = 0; kb < nkb; ++kb, ++it) {
          const int s = it % STAGES;
          mbar_wait(full_bar(s), (it / STAGES) & 1);
          tc_fence_after();
          const uint32_t sa = base + s * L::kStage, sb = sa + L::kABytes;
          if (leader) {
#pragma unroll
            for (int j = 0; j < KB; ++j)
#pragma unroll
              for (int kk = 0; kk < kBK / 8; ++kk) {
                const uint64_t ad = make_sdesc(sa + j * 16384 + kk * 32, 16, 1024, kSw128);
                const uint64_t bd = b_mn ? make_sdesc(sb + j * 16384 + kk * 1024, 4096, 512, kSw128Base32)
                                         : make_sdesc(sb + j * 16384 + kk * 32, 16, 1024, kSw128);
                tc_mma_tf32_pair(d0, ad, bd, idesc, (kb > 0 || j > 0 || kk > 0) ? 1u : 0u);
              }
            tc_commit_pair(empty_bar(s));
          }
          __syncwarp();
        }
        if (leader) tc_commit_pair(tfull_bar(acc));
        __syncwarp();
      }
    }
  } else {
    // ---------------- epilogue (this CTA's 128 rows) ----------------
    const int row = warp * 32 + lane;
    const uint32_t ltempty0 = map_to_rank(tempty_bar(0), 0), ltempty1 = map_to_rank(tempty_bar(1), 0);
    int lt = 0, box = 0;
    for (int tile = pair; tile < ntiles; tile += npairs, ++lt) {
      const int acc = lt & 1;
      const int m0 = (tile / ntn) * 256 + static_cast<int>(rank) * kBM;
      const int n0 = (tile % ntn) * BN;
      mbar_wait_sleep(tfull_bar(acc), (lt >> 1) & 1);
      tc_fence_after();
      const int m = m0 + row;
      const uint32_t taddr = tmem + acc * L::kAccCols + (static_cast<uint32_t>(warp * 32) << 16);
#pragma unroll 1
      for (int cg = 0; cg < BN / 32; ++cg, ++box) {
        const int nb = n0 + cg * 32;
        float v[32];
        tmem_ld32(taddr + cg * 32, v);
        if (cg == BN / 32 - 1) {
          // last TMEM read of this accumulator set: release it to the leader's MMA warp
          tc_fence_before();
          mbar_arrive_cluster(acc ? ltempty1 : ltempty0);
        }
        if (p.kind == kFprop && p.bias) {
#pragma unroll
          for (int i = 0; i < 32; ++i) v[i] += (nb + i < p.Cout) ? p.bias[nb + i] : 0.f;
        }
        if (p.kind == kFprop && p.relu) {
#pragma unroll
          for (int i = 0; i < 32; ++i) v[i] = fmaxf(v[i], 0.f);
        }
        if (p.kind == kDgrad && p.seg[0].mask && m < p.M && nb < p.C) {
          const float* xr = p.seg[0].x + static_cast<int64_t>(m) * p.C + nb;
          if (nb + 32 <= p.C) {
#pragma unroll
            for (int i = 0; i < 32; i += 4) {
              const float4 xv = __ldg(reinterpret_cast<const float4*>(xr + i));
              v[i] = xv.x > 0.f ? v[i] : 0.f;
              v[i + 1] = xv.y > 0.f ? v[i + 1] : 0.f;
              v[i + 2] = xv.z > 0.f ? v[i + 2] : 0.f;
              v[i + 3] = xv.w > 0.f ? v[i + 3] : 0.f;
            }
          } else {
#pragma unroll
            for (int i = 0; i < 32; ++i)
              if (nb + i < p.C) v[i] = xr[i] > 0.f ? v[i] : 0.f;
          }
        }
        // box buffer (box % NOUT) was last used NOUT boxes ago: its TMA store must have read it
        if (threadIdx.x == 0) {
          if constexpr (NOUT == 4)
            asm volatile("cp.async.bulk.wait_group.read 3;" ::: "memory");
          else
            asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
        }
        asm volatile("bar.sync 1, 128;" ::: "memory");
        const uint32_t ob = obuf + (box % NOUT) * 16384;
        const uint32_t rowaddr = ob + row * 128;
#pragma unroll
        for (int j = 0; j < 8; ++j)
          asm volatile("st.shared.v4.f32 [%0], {%1, %2, %3, %4};" ::"r"(rowaddr + (((j ^ (row & 7)) & 7) << 4)),
                       "f"(v[4 * j]), "f"(v[4 * j + 1]), "f"(v[4 * j + 2]), "f"(v[4 * j + 3])
                       : "memory");
        fence_proxy_async();
        asm volatile("bar.sync 1, 128;" ::: "memory");
        if (threadIdx.x == 0) {
          if (nb < p.Ncols && m0 < p.M) tma_store_2d(&tma_c, ob, nb, m0, p.epi == kEpiAccum);
          asm volatile("cp.async.bulk.commit_group;" ::: "memory");
        }
      }
    }
    if (threadIdx.x == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
  }
  tc_fence_before();
  __syncthreads();
  cluster_sync_all();  // the peer's MMAs / barrier traffic into this CTA are over
  if (warp == 4) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(kTmemCols) : "memory");
  }
}

// WGRAD on a CTA pair: D[(tap, ci)][co] over M = 256 weight rows (CTA rank r
// holds rows m0 + 128r: four 32-row MN chunks of X im2col boxes) x N = 256
// output channels (rank r holds dY columns n0 + 128r), K = KW pixels per
// stage, both operands MN-major. Work items are (tile, split) pairs walked
// persistently; the epilogue writes split-K partials or applies SGD / writes
// dW exactly like tc_conv_kernel's WGRAD epilogue.
template <int STAGES, int KW, int PN>
struct WgradPairSmem {
  static constexpr int kABytes = kBM * KW * 4;
  static constexpr int kBBytes = (PN / 2) * KW * 4;  // this CTA's half of the PN output channels
  static constexpr int kStage = kABytes + kBBytes;
  static constexpr int kTotal = STAGES * kStage + 1024 + 256;
  static constexpr int kAccCols = PN < 32 ? 32 : PN;
};

// PN = output channels per pair MMA (N): 256, 128 or 64; each CTA stages PN/2.
template <int STAGES, int KW, int PN>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(192, 1)
    tc_wgrad_pair_kernel(const __grid_constant__ ConvParams p, const __grid_constant__ CUtensorMap tma_a,
                         const __grid_constant__ CUtensorMap tma_b, int splits) {
  using L = WgradPairSmem<STAGES, KW, PN>;
  constexpr int BN = PN;
  constexpr int kTmemCols = 2 * L::kAccCols;
  extern __shared__ uint8_t smem_raw[];
  const uint32_t base = (smem_u32(smem_raw) + 1023u) & ~1023u;
  const uint32_t bars = base + STAGES * L::kStage;
  auto full_bar = [&](int s) { return bars + 8u * s; };
  auto empty_bar = [&](int s) { return bars + 8u * (STAGES + s); };
  auto tfull_bar = [&](int a) { return bars + 8u * (2 * STAGES + a); };
  auto tempty_bar = [&](int a) { return bars + 8u * (2 * STAGES + 2 + a); };
  const uint32_t tmem_slot = bars + 8u * (2 * STAGES + 4);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t rank = cluster_ctarank();
  const int pair = static_cast<int>(blockIdx.x >> 1), npairs = static_cast<int>(gridDim.x >> 1);
  const int ntn = (p.Ncols + BN - 1) / BN;
  const int nwork = ((p.M + 255) / 256) * ntn * splits;

  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(full_bar(s), 1);
      mbar_init(empty_bar(s), 1);
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(tfull_bar(a), 1);
      mbar_init(tempty_bar(a), 256);
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

  // split-major order: the pairs running concurrently share one pixel range
  // (same split) across tiles, so its X / dY rows are read from DRAM once and
  // re-hit in L2 (tile-major order re-read them once per tile)
  const int ntiles = ((p.M + 255) / 256) * ntn;
  auto decode = [&](int w, int& m0, int& n0, int& z, int& kb0, int& kb1) {
    z = w / ntiles;
    const int tile = w - z * ntiles;
    m0 = (tile / ntn) * 256 + static_cast<int>(rank) * kBM;
    n0 = (tile % ntn) * BN;
    kb0 = z * p.kb_per_split;
    kb1 = kb0 + p.kb_per_split < p.kblocks ? kb0 + p.kb_per_split : p.kblocks;
  };

  if (warp == 5) {
    // ---------------- TMA producer ----------------
    if (lane == 0) {
      asm volatile("prefetch.tensormap [%0];" ::"l"(&tma_a) : "memory");
      asm volatile("prefetch.tensormap [%0];" ::"l"(&tma_b) : "memory");
      int it = 0;
      for (int w = pair; w < nwork; w += npairs) {
        int m0, n0, z, kb0, kb1;
        decode(w, m0, n0, z, kb0, kb1);
        const int nb = n0 + static_cast<int>(rank) * (PN / 2);
        TmaProducer<PN / 2, kBM, KW> tp;
        tp.init(p, m0, kb0);
        for (int kb = kb0; kb < kb1; ++kb, ++it) {
          const int s = it % STAGES;
          if (it >= STAGES) mbar_wait(empty_bar(s), ((it / STAGES) & 1) ^ 1);
          const uint32_t sa = base + s * L::kStage, sb = sa + L::kABytes;
          const uint32_t lbar = map_to_rank(full_bar(s), 0);
          if (rank == 0) mbar_expect_tx(full_bar(s), 2 * L::kStage);
          const int iw = tp.pw * p.stride - p.pad, ih = tp.ph * p.stride - p.pad;
#pragma unroll
          for (int mc = 0; mc < kBM / 32; ++mc)
            tma_load_im2col_pair(sa + mc * (KW * 128), &tma_a, lbar, tp.wch[mc], iw, ih, tp.pn, tp.ws[mc],
                                 tp.wr[mc]);
          if (p.tma_b_merged)
            tma_load_3d_pair(sb, &tma_b, lbar, 0, tp.p0, nb >> 5);
          else
            for (int mc = 0; mc < PN / 64; ++mc)
              tma_load_2d_pair(sb + mc * (KW * 128), &tma_b, lbar, nb + mc * 32, tp.p0);
          tp.next(p);
        }
      }
    }
    __syncwarp();
  } else if (warp == 4) {
    // ---------------- MMA issuer (leader CTA) ----------------
    if (rank == 0) {
      const uint32_t idesc = (make_idesc_tf32(BN, true, true) & ~(0x1Fu << 24)) | ((256u >> 4) << 24);
      const bool leader = elect_one();
      int it = 0, lt = 0;
      for (int w = pair; w < nwork; w += npairs, ++lt) {
        int m0, n0, z, kb0, kb1;
        decode(w, m0, n0, z, kb0, kb1);
        const int acc = lt & 1;
        if (lt >= 2) mbar_wait(tempty_bar(acc), ((lt >> 1) & 1) ^ 1);
        tc_fence_after();
        const uint32_t d0 = tmem + acc * L::kAccCols;
        for (int kb = kb0; kb < kb1; ++kb, ++it) {
          const int s = it % STAGES;
          mbar_wait(full_bar(s), (it / STAGES) & 1);
          tc_fence_after();
          const uint32_t sa = base + s * L::kStage, sb = sa + L::kABytes;
          if (leader) {
#pragma unroll
            for (int kk = 0; kk < KW / 8; ++kk)
              tc_mma_tf32_pair(d0, make_sdesc(sa + kk * 1024, KW * 128, 512, kSw128Base32),
                               make_sdesc(sb + kk * 1024, KW * 128, 512, kSw128Base32), idesc,
                               (kb > kb0 || kk > 0) ? 1u : 0u);
            tc_commit_pair(empty_bar(s));
          }
          __syncwarp();
        }
        if (leader) tc_commit_pair(tfull_bar(acc));
        __syncwarp();
      }
    }
  } else {
    // ---------------- epilogue ----------------
    const int row = warp * 32 + lane;
    const uint32_t ltempty0 = map_to_rank(tempty_bar(0), 0), ltempty1 = map_to_rank(tempty_bar(1), 0);
    int lt = 0;
    for (int w = pair; w < nwork; w += npairs, ++lt) {
      int m0, n0, z, kb0, kb1;
      decode(w, m0, n0, z, kb0, kb1);
      const int acc = lt & 1;
      mbar_wait_sleep(tfull_bar(acc), (lt >> 1) & 1);
      tc_fence_after();
      const int m = m0 + row;
      const uint32_t taddr = tmem + acc * L::kAccCols + (static_cast<uint32_t>(warp * 32) << 16);
#pragma unroll 1
      for (int cg = 0; cg < BN / 32; ++cg) {
        float v[32];
        tmem_ld32(taddr + cg * 32, v);
        if (cg == BN / 32 - 1) {
          tc_fence_before();
          mbar_arrive_cluster(acc ? ltempty1 : ltempty0);
        }
        if (kb1 <= kb0) {
#pragma unroll
          for (int i = 0; i < 32; ++i) v[i] = 0.f;
        }
        if (m >= p.M) continue;
        const int nb = n0 + cg * 32;
        if (nb >= p.Cout) continue;
        if (p.epi == kEpiPartial) {
          float* dst = p.out + static_cast<int64_t>(z) * p.Ncols * p.M;
#pragma unroll
          for (int i = 0; i < 32; ++i)
            if (nb + i < p.Cout) dst[static_cast<int64_t>(nb + i) * p.M + m] = v[i];
        } else {
          bool valid;
          const int widx = wgrad_widx(p, m, valid);
          if (!valid) continue;
          if (p.epi == kEpiSgd) {
            float* wcol = p.w_mut + static_cast<int64_t>(nb) * p.KK + widx;
            float wv[32];
#pragma unroll
            for (int i = 0; i < 32; ++i) wv[i] = (nb + i < p.Cout) ? wcol[static_cast<int64_t>(i) * p.KK] : 0.f;
#pragma unroll
            for (int i = 0; i < 32; ++i)
              if (nb + i < p.Cout) wcol[static_cast<int64_t>(i) * p.KK] = wv[i] - p.lr * v[i];
          } else {
#pragma unroll
            for (int i = 0; i < 32; ++i)
              if (nb + i < p.Cout) p.out[static_cast<int64_t>(nb + i) * p.KK + widx] = v[i];
          }
        }
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  cluster_sync_all();
  if (warp == 4) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(kTmemCols) : "memory");
  }
}

}  // namespace vdnnk
