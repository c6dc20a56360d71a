// Persistent variant of the tcgen05 conv engine for FPROP / DGRAD on the TMA
// path (included by conv.cu after tc_conv.cuh).
//
// Short reduction loops (a 3x3 conv over 64 channels is 18 K blocks) leave
// the one-tile-per-CTA kernel paying, per tile, a CTA launch, a pipeline fill
// (first TMA round trip) and an epilogue that only the other resident CTA can
// hide. Here one CTA per SM walks a static round-robin of tiles with a
// continuous stage ring and TWO TMEM accumulator sets, so the epilogue of
// tile t (TMEM -> registers -> fused bias/ReLU/ReLU-mask -> swizzled smem ->
// TMA store) runs while tile t+1's loads and MMAs proceed.
//
//   warps 0-3 : epilogue (warp w drains TMEM lanes 32w..32w+31)
//   warp 4    : TMEM owner + single-thread tcgen05.mma issuer
//   warp 5    : single-thread TMA producer (TmaProducer, incremental coords)
//
// smem: [STAGES x (A BM x 128 B | B BN x 128 B)] [2 x 16 KB output boxes] [barriers]
// TMEM: 2 x (BM/128) x BN fp32 columns (<= 512).
//
// WG = true: WGRAD with a short reduction (FC layers: K = batch, 8 K blocks
// at b256), unsplit. One tile per CTA paid a launch, a pipeline fill and
// TMEM setup for every 256 x 128 block of weights; here the fused SGD
// epilogue (w -= lr * dW, the weight read + write that bounds these layers)
// of tile t overlaps tile t+1's loads and MMAs. Both operands MN-major.
#pragma once

namespace vdnnk {

template <int BN, int BM, int STAGES, int NOUT = 2>
struct PersistSmem {
  static constexpr int kABytes = BM * 128;
  static constexpr int kBBytes = BN * 128;
  static constexpr int kStage = kABytes + kBBytes;
  static constexpr int kOut = NOUT * 16384;
  static constexpr int kTotal = STAGES * kStage + kOut + 1024 + 256;
  static constexpr int kAccCols = (BM / kBM) * BN;  // one accumulator set
  static_assert(2 * kAccCols <= 512, "two accumulator sets must fit TMEM");
};

template <int BN, int BM, int STAGES, bool WG = false>
__global__ void __launch_bounds__(192, 1) tc_conv_persist_kernel(const __grid_constant__ ConvParams p,
                                                                 const __grid_constant__ CUtensorMap tma_a,
                                                                 const __grid_constant__ CUtensorMap tma_b,
                                                                 const __grid_constant__ CUtensorMap tma_c) {
  // WG: four 16 KB W boxes (three loads ahead of the SGD math)
  constexpr int kNout = WG ? 4 : 2;
  using L = PersistSmem<BN, BM, STAGES, kNout>;
  constexpr int kHalves = BM / kBM;
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
  auto wbar = [&](int b) { return bars + 8u * (2 * STAGES + 5 + b); };  // WG + sgd_tma: W box loads (4)

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int ntn = (p.Ncols + BN - 1) / BN;
  const int ntiles = ((p.M + BM - 1) / BM) * ntn;
  const int nkb = p.kblocks;

  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(full_bar(s), 1);
      mbar_init(empty_bar(s), 1);
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(tfull_bar(a), 1);
      mbar_init(tempty_bar(a), 128);
    }
    for (int b = 0; b < 4; ++b) mbar_init(wbar(b), 1);
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

  if (warp == 5) {
    // ---------------- TMA producer ----------------
    if (lane == 0) {
      asm volatile("prefetch.tensormap [%0];" ::"l"(&tma_a) : "memory");
      asm volatile("prefetch.tensormap [%0];" ::"l"(&tma_b) : "memory");
      int it = 0;
      for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
        const int m0 = (tile / ntn) * BM, n0 = (tile % ntn) * BN;
        TmaProducer<BN, BM, kBK> tp;
        tp.init(p, m0, 0);
        for (int kb = 0; kb < nkb; ++kb, ++it) {
          const int s = it % STAGES;
          if (it >= STAGES) mbar_wait(empty_bar(s), ((it / STAGES) & 1) ^ 1);
          const uint32_t sa = base + s * L::kStage;
          mbar_expect_tx(full_bar(s), L::kStage);
          tp.issue(p, &tma_a, &tma_b, n0, sa, sa + L::kABytes, full_bar(s));
          tp.next(p);
        }
      }
    }
    __syncwarp();
  } else if (warp == 4) {
    // ---------------- MMA issuer ----------------
    // whole warp in the loop (warp-uniform descriptors), one elected lane issues
    const uint32_t idesc = make_idesc_tf32(BN, WG, p.kind != kFprop);
    const bool b_mn = p.kind != kFprop;
    const bool leader = elect_one();
    int it = 0, lt = 0;
    for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x, ++lt) {
      const int acc = lt & 1;
      if (lt >= 2) mbar_wait(tempty_bar(acc), ((lt >> 1) & 1) ^ 1);
      tc_fence_after();
      const uint32_t d0 = tmem + acc * L::kAccCols;
      for (int kb = 0; kb < nkb; ++kb, ++it) {
        const int s = it % STAGES;
        mbar_wait(full_bar(s), (it / STAGES) & 1);
        tc_fence_after();
        const uint32_t sa = base + s * L::kStage;
        const uint32_t sb = sa + L::kABytes;
        if (leader) {
#pragma unroll
          for (int kk = 0; kk < kBK / 8; ++kk) {
            const uint64_t ad = WG ? make_sdesc(sa + kk * 1024, kBK * 128, 512, kSw128Base32)
                                   : make_sdesc(sa + kk * 32, 16, 1024, kSw128);
            const uint64_t bd = b_mn ? make_sdesc(sb + kk * 1024, 4096, 512, kSw128Base32)
                                     : make_sdesc(sb + kk * 32, 16, 1024, kSw128);
#pragma unroll
            for (int h = 0; h < kHalves; ++h)
              tc_mma_tf32(d0 + h * BN, ad + static_cast<uint64_t>(h * (16384 >> 4)), bd, idesc,
                          (kb > 0 || kk > 0) ? 1u : 0u);
          }
          tc_commit(empty_bar(s));
        }
        __syncwarp();
      }
      if (leader) tc_commit(tfull_bar(acc));
      __syncwarp();
    }
  } else {
    // ---------------- epilogue ----------------
    const int row = warp * 32 + lane;
    int lt = 0, box = 0;
    // WG + sgd_tma: W box g (global order: tile, half, 32-column group) goes
    // to buffer g % 4; the load of box g + 3 is issued once box g's store is out
    constexpr int kPerTile = kHalves * (BN / 32);
    auto issue_w = [&](int g) {
      const int t = static_cast<int>(blockIdx.x) + (g / kPerTile) * static_cast<int>(gridDim.x);
      if (t >= ntiles) return;
      const int j = g % kPerTile, hh = j / (BN / 32), cc = j - hh * (BN / 32);
      const int km = (t / ntn) * BM + hh * kBM, co = (t % ntn) * BN + cc * 32;
      mbar_expect_tx(wbar(g & 3), 16384);
      tma_load_2d(obuf + (g & 3) * 16384, &tma_c, wbar(g & 3), km, co);
    };
    if (WG && p.sgd_tma && threadIdx.x == 0)
      for (int g = 0; g < 3; ++g) issue_w(g);
    for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x, ++lt) {
      const int acc = lt & 1;
      const int m0 = (tile / ntn) * BM, n0 = (tile % ntn) * BN;
      mbar_wait_sleep(tfull_bar(acc), (lt >> 1) & 1);
      tc_fence_after();
#pragma unroll 1
      for (int h = 0; h < kHalves; ++h) {
        const int m = m0 + h * kBM + row;
        const uint32_t taddr = tmem + acc * L::kAccCols + h * BN + (static_cast<uint32_t>(warp * 32) << 16);
#pragma unroll 1
        for (int cg = 0; cg < BN / 32; ++cg, ++box) {
          const int nb = n0 + cg * 32;
          float v[32];
          tmem_ld32(taddr + cg * 32, v);
          if (h == kHalves - 1 && cg == BN / 32 - 1) {
            // last TMEM read of this accumulator set: hand it back to the MMA warp
            tc_fence_before();
            mbar_arrive(tempty_bar(acc));
          }
          if constexpr (WG) {
            if (p.sgd_tma) {
              // FC layer: W[nb .. nb+31][m0 + h*128 .. +127] as one TMA box
              // (16 KB, unswizzled [32 co][128 k]); SGD in shared memory, TMA
              // store back -- the weight traffic runs asynchronously (three
              // box loads in flight) instead of 32 dependent loads per thread
              const int b = box & 3;
              const uint32_t ob = obuf + b * 16384;
              mbar_wait(wbar(b), (box >> 2) & 1);
              const uint32_t col = ob + row * 4;
#pragma unroll
              for (int i = 0; i < 32; ++i) {
                float w;
                asm volatile("ld.shared.f32 %0, [%1];" : "=f"(w) : "r"(col + i * 512) : "memory");
                asm volatile("st.shared.f32 [%0], %1;" ::"r"(col + i * 512), "f"(w - p.lr * v[i]) : "memory");
              }
              fence_proxy_async();
              asm volatile("bar.sync 1, 128;" ::: "memory");
              if (threadIdx.x == 0) {
                tma_store_2d(&tma_c, ob, m0 + h * kBM, nb, false);
                asm volatile("cp.async.bulk.commit_group;" ::: "memory");
                // buffer (box + 3) & 3 held box - 1, whose store must have read it
                asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
                issue_w(box + 3);
              }
              continue;
            }
            // row m = weight column, v[i] = dW of output channel nb + i
            bool valid;
            const int widx = wgrad_widx(p, m, valid);
            if (valid) {
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
            continue;
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
          // box buffer (box & 1) was last used two boxes ago: its TMA store must have read it
          if (threadIdx.x == 0) asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
          asm volatile("bar.sync 1, 128;" ::: "memory");
          const uint32_t ob = obuf + (box & 1) * 16384;
          const uint32_t rowaddr = ob + row * 128;
#pragma unroll
          for (int j = 0; j < 8; ++j)
            asm volatile("st.shared.v4.f32 [%0], {%1, %2, %3, %4};" ::"r"(rowaddr + (((j ^ (row & 7)) & 7) << 4)),
                         "f"(v[4 * j]), "f"(v[4 * j + 1]), "f"(v[4 * j + 2]), "f"(v[4 * j + 3])
                         : "memory");
          fence_proxy_async();
          asm volatile("bar.sync 1, 128;" ::: "memory");
          if (threadIdx.x == 0) {
            if (nb < p.Ncols) tma_store_2d(&tma_c, ob, nb, m0 + h * kBM, p.epi == kEpiAccum);
            asm volatile("cp.async.bulk.commit_group;" ::: "memory");
          }
        }
      }
    }
    if ((!WG || p.sgd_tma) && threadIdx.x == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 4) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(kTmemCols) : "memory");
  }
}

}  // namespace vdnnk
