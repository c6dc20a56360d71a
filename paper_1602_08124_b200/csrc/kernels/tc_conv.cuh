// tcgen05 / TMEM implicit-GEMM convolution engine for sm_100a (B200).
//
// One kernel template computes the three contractions a CONV (and an FC,
// which is a 1x1 conv over a 1x1 "image" whose channels are the flattened
// input) needs in training:
//   FPROP  Y[p][co]            = sum_{r,s,ci} X[p@(r,s)][ci] * W[co][r][s][ci]
//   DGRAD  dX[p][ci]           = sum_{r,s,co} dY[p@(r',s')][co] * W[co][k-1-r'][k-1-s'][ci]
//   WGRAD  dW[(r,s,ci)][co]    = sum_{p} X[p@(r,s)][ci] * dY[p][co]
// Activations are NHWC fp32, weights KRSC ([Cout][kh][kw][Cin]) fp32; the MMA
// runs kind::tf32 with fp32 accumulation in TMEM.
//
// The reference (vdnnsim) only *times* these events: FLOPs are
// 2*k^2*Cin*Cout*Ho*Wo*N for FWD and 2x that for BWD
// (/root/reference/proj/include/vdnnsim/cost_model.hpp:95-121); the operand
// sets (CONV/FC BWD read X, no conv bias, no gradient w.r.t. raw input) are
// fixed by simulator.hpp:90-131 and footprint.hpp:58-71.
//
// Structure (one output tile of 128 x BN per CTA, split-K over grid.z):
//   warps 0-3 : producers. Each 128-byte operand row (32 fp32 along the
//               contiguous dimension) is gathered with cp.async (zero-fill for
//               padding / out-of-range) straight into the UMMA SWIZZLE_128B
//               canonical layout; completion is signalled with
//               cp.async.mbarrier.arrive.noinc on the stage's FULL barrier.
//               After the main loop the same warps are the epilogue
//               (tcgen05.ld 32x32b: warp w owns TMEM lanes 32w..32w+31).
//   warp 4    : TMEM allocator + single-thread tcgen05.mma issuer; each
//               stage is released with tcgen05.commit -> EMPTY barrier.
#pragma once
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdint>

namespace vdnnk {

constexpr int kBM = 128;            // UMMA M (cta_group::1)
constexpr int kBK = 32;             // fp32 elements per K block = one 128-B swizzle row
constexpr int kMaxSegs = 8;
constexpr int kMaxChunks = 96;

enum GemmKind : int { kFprop = 0, kDgrad = 1, kWgrad = 2 };
enum EpiMode : int { kEpiStore = 0, kEpiAccum = 1, kEpiSgd = 2, kEpiGrad = 3, kEpiPartial = 4 };

// One input-side buffer of a (possibly channel-concatenated) conv input.
struct Seg {
  const float* x;   // NHWC [N][H][W][C] (fprop / wgrad operand)
  float* dx;        // NHWC gradient plane (dgrad output); nullptr = not materialised
  int C;            // channels of this buffer
  int cbase;        // channel offset inside the concatenated input
  int mask;         // dgrad: multiply dX by (x > 0) (fused ReLU backward)
};

// A 32-wide "virtual channel chunk" of the concatenated input (vector mode).
struct Chunk {
  int32_t seg, coff, valid, cbase;
};

struct ConvParams {
  int kind, epi;
  int relu;                   // fprop: fused ReLU on the output
  int N, H, W, C;             // input side
  int Ho, Wo, Cout;           // output side
  int kh, kw, stride, pad;
  int nseg;
  Seg seg[kMaxSegs];
  int nchunk;
  int chunk_arith;            // single segment: chunk i = channels [32i, 32i+32) computed, not tabled
  Chunk chunk[kMaxChunks];
  int vec_in;                 // every segment C % 4 == 0: 16-B gathers over input channels
  int vec_out;                // Cout % 4 == 0
  int tma_b_merged;           // dgrad/wgrad B loaded by one TMA per stage (C or Cout % 32 == 0)
  int wkw;                    // wgrad: pixels (K) per stage (32, or 64 on the TMA path)
  const float* w;             // weights KRSC
  float* w_mut;               // weights to update in place (SGD epilogue)
  const float* bias;          // FC bias for fprop (may be null)
  const float* dy;            // NHWC [N][Ho][Wo][Cout]
  float* y;                   // NHWC [N][Ho][Wo][Cout]
  float* out;                 // dW (kEpiGrad) or split-K partials (kEpiPartial)
  float lr;
  // GEMM geometry
  int M, Ncols, kblocks, kb_per_split;
  int splits;                 // split-K fprop: number of partial slabs
  int use_pair;               // wgrad: CTA-pair kernel (tc_conv_pair.cuh)
  int KK;                     // kh*kw*C: weight row length
  int sgd_tma;                // persistent FC wgrad: SGD epilogue through TMA boxes of W (map in tma_c)
};

// ------------------------------------------------------------------ PTX ----
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint32_t bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(count) : "memory");
}
__device__ __forceinline__ bool mbar_try_wait(uint32_t bar, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}\n"
      : "=r"(ok) : "r"(bar), "r"(parity) : "memory");
  return ok != 0;
}
__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t parity) {
  while (!mbar_try_wait(bar, parity)) {
  }
}
// Long waits (epilogue warps waiting for the whole main loop): let the
// hardware suspend the thread instead of spinning on issue slots.
__device__ __forceinline__ void mbar_wait_sleep(uint32_t bar, uint32_t parity) {
  uint32_t ok = 0;
  while (!ok) {
    asm volatile(
        "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2, %3;\n selp.u32 %0, 1, 0, p;\n}\n"
        : "=r"(ok)
        : "r"(bar), "r"(parity), "r"(1000000u)
        : "memory");
  }
}
__device__ __forceinline__ void tma_store_2d(const CUtensorMap* map, uint32_t src, int x, int y, bool add) {
  if (add)
    asm volatile("cp.reduce.async.bulk.tensor.2d.global.shared::cta.add.bulk_group [%0, {%2, %3}], [%1];" ::"l"(map),
                 "r"(src), "r"(x), "r"(y)
                 : "memory");
  else
    asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%2, %3}], [%1];" ::"l"(map), "r"(src),
                 "r"(x), "r"(y)
                 : "memory");
}
__device__ __forceinline__ void tma_store_3d(const CUtensorMap* map, uint32_t src, int x, int y, int z) {
  asm volatile("cp.async.bulk.tensor.3d.global.shared::cta.bulk_group [%0, {%2, %3, %4}], [%1];" ::"l"(map), "r"(src),
               "r"(x), "r"(y), "r"(z)
               : "memory");
}
// L2 prefetch of [src, src + bytes) in 16 KB bulk requests (bytes % 16 == 0):
// epilogue operands (the dgrad ReLU mask) warmed while the main loop runs.
__device__ __forceinline__ void prefetch_l2_bulk(const void* src, uint64_t bytes) {
  const char* s = static_cast<const char*>(src);
  for (uint64_t o = 0; o < bytes; o += 16384) {
    const uint32_t n = static_cast<uint32_t>(bytes - o < 16384 ? bytes - o : 16384);
    asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(s + o), "r"(n) : "memory");
  }
}
__device__ __forceinline__ void bulk_commit_and_drain() {
  asm volatile("cp.async.bulk.commit_group;" ::: "memory");
  asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
}
__device__ __forceinline__ void cp_async16(uint32_t dst, const void* src, uint32_t src_bytes) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(dst), "l"(src), "r"(src_bytes) : "memory");
}
__device__ __forceinline__ void cp_async4(uint32_t dst, const void* src, uint32_t src_bytes) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4, %2;" ::"r"(dst), "l"(src), "r"(src_bytes) : "memory");
}
__device__ __forceinline__ void cp_async_arrive_noinc(uint32_t bar) {
  asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];" ::"r"(bar) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint32_t bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes) : "memory");
}
__device__ __forceinline__ void tma_load_2d(uint32_t dst, const CUtensorMap* map, uint32_t bar, int x, int y) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];" ::"r"(dst),
      "l"(map), "r"(bar), "r"(x), "r"(y)
      : "memory");
}
__device__ __forceinline__ void tma_load_3d(uint32_t dst, const CUtensorMap* map, uint32_t bar, int x, int y, int z) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, %5}], "
      "[%2];" ::"r"(dst),
      "l"(map), "r"(bar), "r"(x), "r"(y), "r"(z)
      : "memory");
}
__device__ __forceinline__ void tma_load_4d(uint32_t dst, const CUtensorMap* map, uint32_t bar, int x, int y, int z,
                                            int w) {
  asm volatile(
      "cp.async.bulk.tensor.4d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, %5, "
      "%6}], [%2];" ::"r"(dst),
      "l"(map), "r"(bar), "r"(x), "r"(y), "r"(z), "r"(w)
      : "memory");
}
// im2col: coordinates (c, w, h, n) of the first window's top-left corner in
// input space (may be negative = padding), filter-tap offsets (w, h).
__device__ __forceinline__ void tma_load_im2col(uint32_t dst, const CUtensorMap* map, uint32_t bar, int c, int w,
                                                int h, int n, uint16_t ow, uint16_t oh) {
  asm volatile(
      "cp.async.bulk.tensor.4d.shared::cluster.global.im2col.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, %5, "
      "%6}], [%2], {%7, %8};" ::"r"(dst),
      "l"(map), "r"(bar), "r"(c), "r"(w), "r"(h), "r"(n), "h"(ow), "h"(oh)
      : "memory");
}

// One lane of the (fully converged) warp returns true.
__device__ __forceinline__ bool elect_one() {
  uint32_t pred = 0;
  asm volatile("{\n .reg .pred P;\n elect.sync _|P, 0xffffffff;\n selp.u32 %0, 1, 0, P;\n}\n" : "=r"(pred));
  return pred != 0;
}
__device__ __forceinline__ void fence_proxy_async() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
__device__ __forceinline__ void tc_fence_after() {
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void tc_fence_before() {
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void tc_commit(uint32_t bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(bar)
               : "memory");
}
__device__ __forceinline__ void tc_mma_tf32(uint32_t d_tmem, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                            uint32_t accumulate) {
  asm volatile(
      "{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n"
      " tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n}\n" ::"r"(d_tmem),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate)
      : "memory");
}

// 32 lanes x 32 columns of fp32 from TMEM (one column group per call).
__device__ __forceinline__ void tmem_ld32(uint32_t taddr, float (&v)[32]) {
  uint32_t r[32];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 "
      "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
      "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
        "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]),
        "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]),
        "=r"(r[22]), "=r"(r[23]), "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]),
        "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
  for (int i = 0; i < 32; ++i) v[i] = __uint_as_float(r[i]);
}

// UMMA shared-memory descriptor (sm100 version bits).
//   layout 2 = SWIZZLE_128B (K-major operands)
//   layout 1 = SWIZZLE_128B_BASE32B (MN-major tf32 operands: the only legal
//              MN-major smem layout for 32-bit types; 32-B swizzle granules,
//              4-row K atoms)
constexpr uint32_t kSw128 = 2, kSw128Base32 = 1;
__device__ __forceinline__ uint64_t make_sdesc(uint32_t saddr, uint32_t lbo, uint32_t sbo, uint32_t layout) {
  uint64_t d = 0;
  d |= static_cast<uint64_t>((saddr >> 4) & 0x3FFF);
  d |= static_cast<uint64_t>((lbo >> 4) & 0x3FFF) << 16;
  d |= static_cast<uint64_t>((sbo >> 4) & 0x3FFF) << 32;
  d |= static_cast<uint64_t>(1) << 46;  // version = 1 (Blackwell)
  d |= static_cast<uint64_t>(layout) << 61;
  return d;
}

// Instruction descriptor: kind::tf32, fp32 accumulate, M=128.
__host__ __device__ constexpr uint32_t make_idesc_tf32(int n, bool a_mn_major, bool b_mn_major) {
  return (1u << 4)                       // D format f32
         | (2u << 7)                     // A format tf32
         | (2u << 10)                    // B format tf32
         | ((a_mn_major ? 1u : 0u) << 15) | ((b_mn_major ? 1u : 0u) << 16) |
         (static_cast<uint32_t>(n >> 3) << 17) | (static_cast<uint32_t>(kBM >> 4) << 24);
}

// Swizzled byte address of 16-B chunk j of a 128-B operand row.
//   K-major tile (SWIZZLE_128B): row = M/N index; 16-B chunk j ^ (row % 8).
//   MN-major tile (SWIZZLE_128B_BASE32B): row = (k, mc): K index k in [0,32)
//     and 32-wide MN chunk mc (4096 B per chunk, K rows at 128 B); the 32-B
//     granule (j / 2) is XORed with (k % 4).
__device__ __forceinline__ uint32_t kmaj_addr(uint32_t base, int row, int j) {
  return base + (row >> 3) * 1024 + (row & 7) * 128 + (((j ^ (row & 7)) & 7) << 4);
}
__device__ __forceinline__ uint32_t mnmaj_addr(uint32_t base, int k, int mc, int j) {
  return base + mc * 4096 + k * 128 + (((((j >> 1) ^ (k & 3)) << 1) | (j & 1)) << 4);
}

__device__ __forceinline__ Chunk chunk_at(const ConvParams& p, int i) {
  if (p.chunk_arith) {
    Chunk c;
    c.seg = 0;
    c.coff = static_cast<int32_t>(i * 32);
    const int v = p.C - i * 32;
    c.valid = static_cast<int32_t>(v < 32 ? v : 32);
    c.cbase = c.coff;
    return c;
  }
  return p.chunk[i];
}

// ---------------------------------------------------------- gathers ------
// Segment lookup for a flat channel index (scalar mode).
__device__ __forceinline__ int seg_of(const ConvParams& p, int c) {
  int s = 0;
#pragma unroll 1
  for (int i = 1; i < p.nseg; ++i)
    if (c >= p.seg[i].cbase) s = i;
  return s;
}

struct Pix {
  int n, h, w;
};
__device__ __forceinline__ Pix decode_pix(int m, int Hg, int Wg) {
  Pix q;
  q.w = m % Wg;
  const int t = m / Wg;
  q.h = t % Hg;
  q.n = t / Hg;
  return q;
}

template <int BN>
struct Gather {
  // ---- FPROP ------------------------------------------------------------
  // A: im2col rows (output pixel) x 32 channels of tap (r,s) & chunk, K-major.
  // B: weight rows (co) x 32 channels, K-major.
  __device__ static void fprop(const ConvParams& p, int m0, int n0, int kb, uint32_t sa, uint32_t sb,
                               int tid) {
    if (p.vec_in) {
      const int tap = kb / p.nchunk, ck = kb - tap * p.nchunk;
      const int r = tap / p.kw, s = tap - r * p.kw;
      const Chunk c = chunk_at(p, ck);
      const Seg sg = p.seg[c.seg];
      const int j = tid & 7;
      const bool jv = (j * 4) < c.valid;
#pragma unroll 4
      for (int i = 0; i < kBM / 16; ++i) {
        const int row = (tid >> 3) + 16 * i;
        const int m = m0 + row;
        const float* src = sg.x;
        uint32_t bytes = 0;
        if (m < p.M && jv) {
          const Pix q = decode_pix(m, p.Ho, p.Wo);
          const int ih = q.h * p.stride - p.pad + r, iw = q.w * p.stride - p.pad + s;
          if (ih >= 0 && ih < p.H && iw >= 0 && iw < p.W) {
            src = sg.x + ((static_cast<int64_t>(q.n) * p.H + ih) * p.W + iw) * sg.C + c.coff + j * 4;
            bytes = 16;
          }
        }
        cp_async16(kmaj_addr(sa, row, j), src, bytes);
      }
#pragma unroll 4
      for (int i = 0; i < BN / 16; ++i) {
        const int row = (tid >> 3) + 16 * i;
        const int co = n0 + row;
        const float* src = p.w;
        uint32_t bytes = 0;
        if (co < p.Cout && jv) {
          src = p.w + static_cast<int64_t>(co) * p.KK + tap * p.C + c.cbase + j * 4;
          bytes = 16;
        }
        cp_async16(kmaj_addr(sb, row, j), src, bytes);
      }
    } else {
      // Flat K = (r, s, c) over the concatenated channels; one fp32 per lane.
      const int e = tid & 31;
      const int k = kb * kBK + e;
      const bool kv = k < p.KK;
      int r = 0, s = 0, c = 0, sgi = 0;
      if (kv) {
        const int tap = k / p.C;
        c = k - tap * p.C;
        r = tap / p.kw;
        s = tap - r * p.kw;
        sgi = seg_of(p, c);
      }
      const Seg sg = p.seg[sgi];
      const int cl = c - sg.cbase;
#pragma unroll 4
      for (int i = 0; i < kBM / 4; ++i) {
        const int row = (tid >> 5) + 4 * i;
        const int m = m0 + row;
        const float* src = sg.x;
        uint32_t bytes = 0;
        if (kv && m < p.M) {
          const Pix q = decode_pix(m, p.Ho, p.Wo);
          const int ih = q.h * p.stride - p.pad + r, iw = q.w * p.stride - p.pad + s;
          if (ih >= 0 && ih < p.H && iw >= 0 && iw < p.W) {
            src = sg.x + ((static_cast<int64_t>(q.n) * p.H + ih) * p.W + iw) * sg.C + cl;
            bytes = 4;
          }
        }
        cp_async4(kmaj_addr(sa, row, e >> 2) + (e & 3) * 4, src, bytes);
      }
#pragma unroll 4
      for (int i = 0; i < BN / 4; ++i) {
        const int row = (tid >> 5) + 4 * i;
        const int co = n0 + row;
        const float* src = p.w;
        uint32_t bytes = 0;
        if (kv && co < p.Cout) {
          src = p.w + static_cast<int64_t>(co) * p.KK + k;
          bytes = 4;
        }
        cp_async4(kmaj_addr(sb, row, e >> 2) + (e & 3) * 4, src, bytes);
      }
    }
  }

  // ---- DGRAD (stride 1) --------------------------------------------------
  // A: im2col of dY (grid = input pixels, pad' = k-1-pad), K-major over co.
  // B: W^T, MN-major: K rows = co, MN = virtual input channel.
  __device__ static void dgrad(const ConvParams& p, int m0, int n0, int kb, uint32_t sa, uint32_t sb,
                               int tid) {
    const int padh = p.kh - 1 - p.pad, padw = p.kw - 1 - p.pad;
    // K decode: vec_out -> (tap, co-chunk of 32); else flat (tap, co).
    int tap, co0;
    if (p.vec_out) {
      const int nck = (p.Cout + 31) >> 5;
      tap = kb / nck;
      co0 = (kb - tap * nck) * 32;
    } else {
      tap = 0;
      co0 = 0;  // per-element decode below
    }
    if (p.vec_out) {
      const int r = tap / p.kw, s = tap - r * p.kw;
      const int j = tid & 7;
      const bool jv = (co0 + j * 4) < p.Cout;
#pragma unroll 4
      for (int i = 0; i < kBM / 16; ++i) {
        const int row = (tid >> 3) + 16 * i;
        const int m = m0 + row;
        const float* src = p.dy;
        uint32_t bytes = 0;
        if (m < p.M && jv) {
          const Pix q = decode_pix(m, p.H, p.W);
          const int oh = q.h - padh + r, ow = q.w - padw + s;
          if (oh >= 0 && oh < p.Ho && ow >= 0 && ow < p.Wo) {
            src = p.dy + ((static_cast<int64_t>(q.n) * p.Ho + oh) * p.Wo + ow) * p.Cout + co0 + j * 4;
            bytes = 16;
          }
        }
        cp_async16(kmaj_addr(sa, row, j), src, bytes);
      }
    } else {
      const int e = tid & 31;
      const int k = kb * kBK + e;
      const int KD = p.kh * p.kw * p.Cout;
      const bool kv = k < KD;
      int r = 0, s = 0, co = 0;
      if (kv) {
        const int t = k / p.Cout;
        co = k - t * p.Cout;
        r = t / p.kw;
        s = t - r * p.kw;
      }
#pragma unroll 4
      for (int i = 0; i < kBM / 4; ++i) {
        const int row = (tid >> 5) + 4 * i;
        const int m = m0 + row;
        const float* src = p.dy;
        uint32_t bytes = 0;
        if (kv && m < p.M) {
          const Pix q = decode_pix(m, p.H, p.W);
          const int oh = q.h - padh + r, ow = q.w - padw + s;
          if (oh >= 0 && oh < p.Ho && ow >= 0 && ow < p.Wo) {
            src = p.dy + ((static_cast<int64_t>(q.n) * p.Ho + oh) * p.Wo + ow) * p.Cout + co;
            bytes = 4;
          }
        }
        cp_async4(kmaj_addr(sa, row, e >> 2) + (e & 3) * 4, src, bytes);
      }
    }
    // B operand (MN-major): row (k, mc) holds W[co(k)][flip tap][virtual ci chunk mc]
    if (p.vec_in) {
      const int j = tid & 7;
#pragma unroll 2
      for (int i = 0; i < BN / 16; ++i) {
        const int q = (tid >> 3) + 16 * i;
        const int k = q & 31, mc = q >> 5;
        int co, rr, ss;
        bool kv;
        if (p.vec_out) {
          co = co0 + k;
          rr = tap / p.kw;
          ss = tap - rr * p.kw;
          kv = co < p.Cout;
        } else {
          const int kf = kb * kBK + k;
          kv = kf < p.kh * p.kw * p.Cout;
          const int t = kv ? kf / p.Cout : 0;
          co = kv ? kf - t * p.Cout : 0;
          rr = t / p.kw;
          ss = t - rr * p.kw;
        }
        const int vc = (n0 >> 5) + mc;
        const float* src = p.w;
        uint32_t bytes = 0;
        if (kv && vc < p.nchunk) {
          const Chunk c = chunk_at(p, vc);
          if (j * 4 < c.valid) {
            const int ftap = (p.kh - 1 - rr) * p.kw + (p.kw - 1 - ss);
            src = p.w + static_cast<int64_t>(co) * p.KK + ftap * p.C + c.cbase + j * 4;
            bytes = 16;
          }
        }
        cp_async16(mnmaj_addr(sb, k, mc, j), src, bytes);
      }
    } else {
      const int e = tid & 31;  // MN element within the chunk
#pragma unroll 2
      for (int i = 0; i < BN / 4; ++i) {
        const int q = (tid >> 5) + 4 * i;
        const int k = q & 31, mc = q >> 5;
        int co, rr, ss;
        bool kv;
        if (p.vec_out) {
          co = co0 + k;
          rr = tap / p.kw;
          ss = tap - rr * p.kw;
          kv = co < p.Cout;
        } else {
          const int kf = kb * kBK + k;
          kv = kf < p.kh * p.kw * p.Cout;
          const int t = kv ? kf / p.Cout : 0;
          co = kv ? kf - t * p.Cout : 0;
          rr = t / p.kw;
          ss = t - rr * p.kw;
        }
        const int ci = n0 + mc * 32 + e;
        const float* src = p.w;
        uint32_t bytes = 0;
        if (kv && ci < p.C) {
          const int ftap = (p.kh - 1 - rr) * p.kw + (p.kw - 1 - ss);
          src = p.w + static_cast<int64_t>(co) * p.KK + ftap * p.C + ci;
          bytes = 4;
        }
        cp_async4(mnmaj_addr(sb, k, mc, e >> 2) + (e & 3) * 4, src, bytes);
      }
    }
  }

  // ---- WGRAD ---------------------------------------------------------------
  // GEMM M = virtual (r,s,ci) columns of W, N = co, K = output pixels.
  // A: X_col^T, MN-major: K row = pixel, MN = virtual weight column.
  // B: dY^T,    MN-major: K row = pixel, MN = co.
  __device__ static void wgrad(const ConvParams& p, int m0, int n0, int kb, uint32_t sa, uint32_t sb,
                               int tid) {
    const int P = p.N * p.Ho * p.Wo;
    if (p.vec_in) {
      const int j = tid & 7;
#pragma unroll 2
      for (int i = 0; i < kBM / 16; ++i) {
        const int q = (tid >> 3) + 16 * i;
        const int k = q & 31, mc = q >> 5;
        const int pix = kb * kBK + k;
        const int vcol = (m0 >> 5) + mc;  // virtual chunk over (tap, chunk)
        const float* src = p.w;
        uint32_t bytes = 0;
        if (pix < P && vcol < p.kh * p.kw * p.nchunk) {
          const int tap = vcol / p.nchunk, ck = vcol - tap * p.nchunk;
          const Chunk c = chunk_at(p, ck);
          if (j * 4 < c.valid) {
            const int r = tap / p.kw, s = tap - r * p.kw;
            const Pix x = decode_pix(pix, p.Ho, p.Wo);
            const int ih = x.h * p.stride - p.pad + r, iw = x.w * p.stride - p.pad + s;
            if (ih >= 0 && ih < p.H && iw >= 0 && iw < p.W) {
              const Seg sg = p.seg[c.seg];
              src = sg.x + ((static_cast<int64_t>(x.n) * p.H + ih) * p.W + iw) * sg.C + c.coff + j * 4;
              bytes = 16;
            }
          }
        }
        cp_async16(mnmaj_addr(sa, k, mc, j), src, bytes);
      }
    } else {
      const int e = tid & 31;
#pragma unroll 2
      for (int i = 0; i < kBM / 4; ++i) {
        const int q = (tid >> 5) + 4 * i;
        const int k = q & 31, mc = q >> 5;
        const int pix = kb * kBK + k;
        const int col = m0 + mc * 32 + e;  // flat (r,s,c)
        const float* src = p.w;
        uint32_t bytes = 0;
        if (pix < P && col < p.KK) {
          const int tap = col / p.C, c = col - tap * p.C;
          const int r = tap / p.kw, s = tap - r * p.kw;
          const Pix x = decode_pix(pix, p.Ho, p.Wo);
          const int ih = x.h * p.stride - p.pad + r, iw = x.w * p.stride - p.pad + s;
          if (ih >= 0 && ih < p.H && iw >= 0 && iw < p.W) {
            const Seg sg = p.seg[seg_of(p, c)];
            src = sg.x + ((static_cast<int64_t>(x.n) * p.H + ih) * p.W + iw) * sg.C + (c - sg.cbase);
            bytes = 4;
          }
        }
        cp_async4(mnmaj_addr(sa, k, mc, e >> 2) + (e & 3) * 4, src, bytes);
      }
    }
    if (p.vec_out) {
      const int j = tid & 7;
#pragma unroll 2
      for (int i = 0; i < BN / 16; ++i) {
        const int q = (tid >> 3) + 16 * i;
        const int k = q & 31, mc = q >> 5;
        const int pix = kb * kBK + k;
        const int co = n0 + mc * 32 + j * 4;
        const float* src = p.dy;
        uint32_t bytes = 0;
        if (pix < P && co < p.Cout) {
          src = p.dy + static_cast<int64_t>(pix) * p.Cout + co;
          bytes = 16;
        }
        cp_async16(mnmaj_addr(sb, k, mc, j), src, bytes);
      }
    } else {
      const int e = tid & 31;
#pragma unroll 2
      for (int i = 0; i < BN / 4; ++i) {
        const int q = (tid >> 5) + 4 * i;
        const int k = q & 31, mc = q >> 5;
        const int pix = kb * kBK + k;
        const int co = n0 + mc * 32 + e;
        const float* src = p.dy;
        uint32_t bytes = 0;
        if (pix < P && co < p.Cout) {
          src = p.dy + static_cast<int64_t>(pix) * p.Cout + co;
          bytes = 4;
        }
        cp_async4(mnmaj_addr(sb, k, mc, e >> 2) + (e & 3) * 4, src, bytes);
      }
    }
  }
};

// Weight-row index of a wgrad GEMM row m (virtual (tap, chunk, lane) or flat).
__device__ __forceinline__ int wgrad_widx(const ConvParams& p, int m, bool& valid) {
  if (p.vec_in) {
    const int vcol = m >> 5, lane = m & 31;
    const int tap = vcol / p.nchunk, ck = vcol - tap * p.nchunk;
    if (tap >= p.kh * p.kw) {
      valid = false;
      return 0;
    }
    const Chunk c = chunk_at(p, ck);
    valid = lane < c.valid;
    return tap * p.C + c.cbase + lane;
  }
  valid = m < p.KK;
  return m;
}

// ------------------------------------------------------------ kernel ------
// PRECISE = 3xTF32: each operand x = hi + lo with hi = tf32(x) (what the
// tensor core reads from x itself: it truncates to 10 mantissa bits) and the
// exactly representable residual lo = x - hi kept in a second tile; the
// accumulator gets A*B + A*B_lo + A_lo*B, i.e. fp32-level products.
template <int BN, int STAGES, bool PRECISE, int BM = kBM, int KW = kBK>
struct TcSmem {
  static constexpr int kABytes = BM * KW * 4;
  static constexpr int kBBytes = BN * KW * 4;
  static constexpr int kHalf = kABytes + kBBytes;
  static constexpr int kStage = PRECISE ? 2 * kHalf : kHalf;
  static constexpr int kTotal = STAGES * kStage + 1024 /*align slack*/ + 256 /*barriers*/;
  static_assert(8 * (3 * STAGES + 2) <= 256, "barriers must fit their slot");
};

__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}
__device__ __forceinline__ void producers_sync() {  // named barrier over the 128 producer threads
  asm volatile("bar.sync 1, 128;" ::: "memory");
}
__device__ __forceinline__ void mbar_arrive(uint32_t bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(bar) : "memory");
}

// lo = x - tf32_trunc(x) for every fp32 of a stage's A|B tiles (layout-agnostic
// elementwise pass: the lo tiles mirror the hi tiles byte for byte).
template <int BYTES, int NT = 128>
__device__ __forceinline__ void split_lo(uint32_t hi, uint32_t lo, int tid) {
#pragma unroll 4
  for (int off = tid * 16; off < BYTES; off += NT * 16) {
    uint32_t a, b, c, d;
    asm volatile("ld.shared.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(a), "=r"(b), "=r"(c), "=r"(d) : "r"(hi + off));
    const float fa = __uint_as_float(a) - __uint_as_float(a & 0xFFFFE000u);
    const float fb = __uint_as_float(b) - __uint_as_float(b & 0xFFFFE000u);
    const float fc = __uint_as_float(c) - __uint_as_float(c & 0xFFFFE000u);
    const float fd = __uint_as_float(d) - __uint_as_float(d & 0xFFFFE000u);
    asm volatile("st.shared.v4.f32 [%0], {%1,%2,%3,%4};" ::"r"(lo + off), "f"(fa), "f"(fb), "f"(fc), "f"(fd)
                 : "memory");
  }
}

// TMA producer (single thread). A: im2col (fprop: X, dgrad: dY, 128-pixel
// columns, SWIZZLE_128B = K-major canonical; wgrad: X, KW-pixel columns per
// (tap, 32-channel) chunk, SWIZZLE_128B_ATOM_32B = MN-major canonical).
// B: tiled (fprop: W [Cout][KK] K-major; dgrad: W as (Cin, taps, Cout)
// MN-major chunks; wgrad: dY [P][Cout] MN-major chunks).
// Everything CTA-invariant (window origins of the tile, the wgrad tile's
// (tap, chunk) per MN chunk) is computed once and the per-stage coordinates
// advance incrementally: the issuing thread is serial, and per-stage integer
// divisions measurably throttled the small-box (wgrad) pipelines.
template <int BN, int BM, int KW>
struct TmaProducer {
  static constexpr int kH = BM / kBM;
  int kind;
  int qw[kH], qh[kH], qn[kH];  // fprop/dgrad: im2col window origin of each 128-row half
  int ck, nck, r, s;           // fprop/dgrad: current (tap, 32-channel chunk)
  int wch[BM / 32];            // wgrad: channel offset, tap of each MN chunk of A
  uint16_t wr[BM / 32], ws[BM / 32];
  int p0, pw, ph, pn;          // wgrad: first pixel of the stage

  __device__ __forceinline__ void init(const ConvParams& p, int m0, int kb) {
    kind = p.kind;
    if (kind != kWgrad) {
      nck = kind == kFprop ? p.nchunk : (p.Cout + 31) >> 5;
      const int tap = kb / nck;
      ck = kb - tap * nck;
      r = tap / p.kw;
      s = tap - r * p.kw;
#pragma unroll
      for (int h = 0; h < kH; ++h) {
        if (kind == kFprop) {
          const Pix q = decode_pix(m0 + h * kBM, p.Ho, p.Wo);
          qw[h] = q.w * p.stride - p.pad;
          qh[h] = q.h * p.stride - p.pad;
          qn[h] = q.n;
        } else {
          const Pix q = decode_pix(m0 + h * kBM, p.H, p.W);
          qw[h] = q.w - (p.kw - 1 - p.pad);
          qh[h] = q.h - (p.kh - 1 - p.pad);
          qn[h] = q.n;
        }
      }
    } else {
#pragma unroll
      for (int mc = 0; mc < BM / 32; ++mc) {
        const int vc = (m0 >> 5) + mc;
        const int tap = vc / p.nchunk, c = vc - tap * p.nchunk;
        const int rr = tap / p.kw;
        wch[mc] = c * 32;
        wr[mc] = static_cast<uint16_t>(rr);
        ws[mc] = static_cast<uint16_t>(tap - rr * p.kw);
      }
      p0 = kb * KW;
      const Pix q = decode_pix(p0, p.Ho, p.Wo);
      pw = q.w;
      ph = q.h;
      pn = q.n;
    }
  }

  __device__ __forceinline__ void issue(const ConvParams& p, const CUtensorMap* ta, const CUtensorMap* tb, int n0,
                                        uint32_t sa, uint32_t sb, uint32_t bar) const {
    if (kind == kFprop) {
#pragma unroll
      for (int h = 0; h < kH; ++h)
        tma_load_im2col(sa + h * 16384, ta, bar, ck * 32, qw[h], qh[h], qn[h], static_cast<uint16_t>(s),
                        static_cast<uint16_t>(r));
      tma_load_2d(sb, tb, bar, (r * p.kw + s) * p.C + ck * 32, n0);
    } else if (kind == kDgrad) {
#pragma unroll
      for (int h = 0; h < kH; ++h)
        tma_load_im2col(sa + h * 16384, ta, bar, ck * 32, qw[h], qh[h], qn[h], static_cast<uint16_t>(s),
                        static_cast<uint16_t>(r));
      const int ftap = (p.kh - 1 - r) * p.kw + (p.kw - 1 - s);
      if (p.tma_b_merged)
        tma_load_4d(sb, tb, bar, 0, ck * 32, n0 >> 5, ftap);
      else
        for (int mc = 0; mc < BN / 32; ++mc) tma_load_3d(sb + mc * 4096, tb, bar, n0 + mc * 32, ftap, ck * 32);
    } else {
      // KW pixels per stage: every MN chunk (32 channels / 32 output channels)
      // is KW K-rows of 128 B, chunks KW*128 B apart (the descriptors' LBO)
      const int iw = pw * p.stride - p.pad, ih = ph * p.stride - p.pad;
#pragma unroll
      for (int mc = 0; mc < BM / 32; ++mc)
        tma_load_im2col(sa + mc * (KW * 128), ta, bar, wch[mc], iw, ih, pn, ws[mc], wr[mc]);
      if (p.tma_b_merged)
        tma_load_3d(sb, tb, bar, 0, p0, n0 >> 5);
      else
        for (int mc = 0; mc < BN / 32; ++mc) tma_load_2d(sb + mc * (KW * 128), tb, bar, n0 + mc * 32, p0);
    }
  }

  __device__ __forceinline__ void next(const ConvParams& p) {
    if (kind != kWgrad) {
      if (++ck == nck) {
        ck = 0;
        if (++s == p.kw) {
          s = 0;
          ++r;
        }
      }
    } else {
      p0 += KW;
      pw += KW;
      while (pw >= p.Wo) {
        pw -= p.Wo;
        if (++ph == p.Ho) {
          ph = 0;
          ++pn;
        }
      }
    }
  }
};

// BM x BN output tile per CTA. BM = 256 (TMA path) issues two M=128 MMAs per
// K step against one B tile, into two TMEM accumulators: 43 (BN=128) or 64
// (BN=256) FLOP per staged byte instead of 32 / 43, the lever against the L2
// -> SM fill rate that bounds BM=128 tiles. Two CTAs per SM when the stage
// ring fits in half the shared memory, else one.
template <int BN, int STAGES, bool PRECISE, bool TMA, int BM = kBM, int KW = kBK>
__global__ void __launch_bounds__(160, (TcSmem<BN, STAGES, PRECISE, BM, KW>::kTotal <= 116 * 1024 ? 2 : 1))
    tc_conv_kernel(const __grid_constant__ ConvParams p,
                                                         const __grid_constant__ CUtensorMap tma_a,
                                                         const __grid_constant__ CUtensorMap tma_b,
                                                         const __grid_constant__ CUtensorMap tma_c) {
  extern __shared__ uint8_t smem_raw[];
  using L = TcSmem<BN, STAGES, PRECISE, BM, KW>;
  static_assert(KW == kBK || TMA, "wide K stages are TMA-wgrad only");
  constexpr int kHalves = BM / kBM;
  constexpr int kTmemCols = BN * kHalves;
  const uint32_t raw = smem_u32(smem_raw);
  const uint32_t base = (raw + 1023u) & ~1023u;
  const uint32_t bar_base = base + STAGES * L::kStage;
  auto full_bar = [&](int s) { return bar_base + 8u * s; };
  auto empty_bar = [&](int s) { return bar_base + 8u * (STAGES + s); };
  const uint32_t accum_bar = bar_base + 8u * (2 * STAGES);
  const uint32_t tmem_slot = bar_base + 8u * (2 * STAGES + 1);
  // PRECISE with TMA: warps 1-3 write each landed stage's lo tiles, then
  // arrive here; the MMA waits on split_bar instead of full_bar
  auto split_bar = [&](int s) { return bar_base + 8u * (2 * STAGES + 2 + s); };
  constexpr bool kSplitWarps = PRECISE && TMA;
  uint32_t* tmem_slot_ptr =
      reinterpret_cast<uint32_t*>(smem_raw + (tmem_slot - raw));

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  // linear tile index with the N tiles of one M tile adjacent, so the A
  // (activation) tile is read from DRAM once and re-hit in L2
  const int ntn = (p.Ncols + BN - 1) / BN;
  const int m0 = static_cast<int>(blockIdx.x / ntn) * BM;
  const int n0 = static_cast<int>(blockIdx.x % ntn) * BN;
  const int kb_begin = blockIdx.z * p.kb_per_split;
  int kb_end = kb_begin + p.kb_per_split;
  if (kb_end > p.kblocks) kb_end = p.kblocks;
  const int nkb = kb_end - kb_begin;

  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(full_bar(s), TMA ? 1 : 128);  // TMA: one expect_tx arrive; else 128 producer arrivals
      mbar_init(empty_bar(s), 1);
    }
    mbar_init(accum_bar, 1);
    if constexpr (kSplitWarps)
      for (int s = 0; s < STAGES; ++s) mbar_init(split_bar(s), 96);
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
  const uint32_t tmem = *reinterpret_cast<volatile uint32_t*>(tmem_slot_ptr);

  if (warp < 4) {
    // ---------------- producers ----------------
    const int tid = threadIdx.x;
    if constexpr (TMA) {
      if (tid == 0) {
        asm volatile("prefetch.tensormap [%0];" ::"l"(&tma_a) : "memory");
        asm volatile("prefetch.tensormap [%0];" ::"l"(&tma_b) : "memory");
        constexpr uint32_t kBytes = L::kABytes + L::kBBytes;
        TmaProducer<BN, BM, KW> tp;
        tp.init(p, m0, kb_begin);
        for (int it = 0; it < nkb; ++it) {
          const int s = it % STAGES;
          const uint32_t ph = (it / STAGES) & 1;
          if (it >= STAGES) mbar_wait(empty_bar(s), ph ^ 1);
          const uint32_t sa = base + s * L::kStage;
          mbar_expect_tx(full_bar(s), kBytes);
          tp.issue(p, &tma_a, &tma_b, n0, sa, sa + L::kABytes, full_bar(s));
          tp.next(p);
        }
      }
      if constexpr (kSplitWarps) {
        if (warp > 0) {
          // lo = x - tf32(x) of every landed stage (96 threads), then release it to the MMA
          for (int it = 0; it < nkb; ++it) {
            const int s = it % STAGES;
            mbar_wait(full_bar(s), (it / STAGES) & 1);
            const uint32_t sa = base + s * L::kStage;
            split_lo<L::kHalf, 96>(sa, sa + L::kHalf, tid - 32);
            fence_proxy_async();
            mbar_arrive(split_bar(s));
          }
        }
      }
      __syncwarp();
    }
    if constexpr (!TMA)
    for (int it = 0; it < nkb; ++it) {
      const int s = it % STAGES;
      const uint32_t ph = (it / STAGES) & 1;
      if (it >= STAGES) mbar_wait(empty_bar(s), ph ^ 1);
      const uint32_t sa = base + s * L::kStage;
      const uint32_t sb = sa + L::kABytes;
      const int kb = kb_begin + it;
      if (p.kind == kFprop)
        Gather<BN>::fprop(p, m0, n0, kb, sa, sb, tid);
      else if (p.kind == kDgrad)
        Gather<BN>::dgrad(p, m0, n0, kb, sa, sb, tid);
      else
        Gather<BN>::wgrad(p, m0, n0, kb, sa, sb, tid);
      if constexpr (!PRECISE || TMA) {
        cp_async_arrive_noinc(full_bar(s));
      } else {
        // one stage of lag: split the previous stage once every producer's copies landed
        cp_async_commit();
        cp_async_wait<1>();
        producers_sync();
        if (it > 0) {
          const int ps = (it - 1) % STAGES;
          const uint32_t pa = base + ps * L::kStage;
          split_lo<L::kHalf>(pa, pa + L::kHalf, tid);
          fence_proxy_async();
          mbar_arrive(full_bar(ps));
        }
      }
    }
    if constexpr (PRECISE && !TMA) {
      cp_async_wait<0>();
      producers_sync();
      if (nkb > 0) {
        const int ps = (nkb - 1) % STAGES;
        const uint32_t pa = base + ps * L::kStage;
        split_lo<L::kHalf>(pa, pa + L::kHalf, tid);
        fence_proxy_async();
        mbar_arrive(full_bar(ps));
      }
    }
    // ---------------- epilogue ----------------
    mbar_wait_sleep(accum_bar, 0);
    tc_fence_after();
    __syncwarp();
    const int row = warp * 32 + lane;
#pragma unroll 1
    for (int h = 0; h < kHalves; ++h) {
    const int m = m0 + h * kBM + row;
    const uint32_t taddr = tmem + h * BN + (static_cast<uint32_t>(warp * 32) << 16);
    if (TMA && p.kind != kWgrad) {
      // Stage the 128 x BN tile in the idle pipeline buffers as BN/32
      // SWIZZLE_128B boxes (128 rows x 128 B) and write it with TMA stores
      // (reduce-add for accumulation): fully coalesced, clipped at M / Cout.
#pragma unroll 1
      for (int cg = 0; cg < BN / 32; ++cg) {
        float v[32];
        tmem_ld32(taddr + cg * 32, v);
        const int nb = n0 + cg * 32;
        if (nkb <= 0) {
#pragma unroll
          for (int i = 0; i < 32; ++i) v[i] = 0.f;
        }
        const bool partial = p.epi == kEpiPartial;  // split-K fprop: raw partial sums
        if (p.kind == kFprop && p.bias && !partial) {
#pragma unroll
          for (int i = 0; i < 32; ++i) v[i] += (nb + i < p.Cout) ? p.bias[nb + i] : 0.f;
        }
        if (p.kind == kFprop && p.relu && !partial) {
#pragma unroll
          for (int i = 0; i < 32; ++i) v[i] = fmaxf(v[i], 0.f);
        }
        if (p.kind == kDgrad && p.seg[0].mask && !partial && m < p.M && nb < p.C) {
          // fused ReLU backward: the ReLU's output is this conv's input x
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
        const uint32_t rowaddr = base + cg * 16384 + row * 128;
#pragma unroll
        for (int j = 0; j < 8; ++j)
          asm volatile("st.shared.v4.f32 [%0], {%1, %2, %3, %4};" ::"r"(rowaddr + (((j ^ (row & 7)) & 7) << 4)),
                       "f"(v[4 * j]), "f"(v[4 * j + 1]), "f"(v[4 * j + 2]), "f"(v[4 * j + 3])
                       : "memory");
      }
      fence_proxy_async();
      asm volatile("bar.sync 2, 128;" ::: "memory");
      if (threadIdx.x == 0) {
        for (int cg = 0; cg < BN / 32; ++cg)
          if (n0 + cg * 32 < p.Ncols) {
            if (p.epi == kEpiPartial)  // split z's slab of the [splits][M][Cout] partials
              tma_store_3d(&tma_c, base + cg * 16384, n0 + cg * 32, m0 + h * kBM, static_cast<int>(blockIdx.z));
            else
              tma_store_2d(&tma_c, base + cg * 16384, n0 + cg * 32, m0 + h * kBM, p.epi == kEpiAccum);
          }
        bulk_commit_and_drain();
      }
      if (kHalves > 1) asm volatile("bar.sync 2, 128;" ::: "memory");  // staging read out before reuse
    } else {
#pragma unroll 1
    for (int cg = 0; cg < BN / 32; ++cg) {
      float v[32];
      tmem_ld32(taddr + cg * 32, v);
      if (nkb <= 0) {
#pragma unroll
        for (int i = 0; i < 32; ++i) v[i] = 0.f;
      }
      if (m >= p.M) continue;
      const int nb = n0 + cg * 32;
      if (p.kind == kFprop) {
        float* dst = p.y + static_cast<int64_t>(m) * p.Cout + nb;
        if (p.bias) {
#pragma unroll
          for (int i = 0; i < 32; ++i)
            if (nb + i < p.Cout) v[i] += p.bias[nb + i];
        }
        if (p.relu) {
#pragma unroll
          for (int i = 0; i < 32; ++i) v[i] = fmaxf(v[i], 0.f);
        }
        if (p.vec_out && nb + 32 <= p.Cout) {
          if (p.epi == kEpiAccum) {
            float4 a[8];  // loads in flight together, then the stores
#pragma unroll
            for (int i = 0; i < 8; ++i) a[i] = *reinterpret_cast<const float4*>(dst + 4 * i);
#pragma unroll
            for (int i = 0; i < 8; ++i) {
              v[4 * i] += a[i].x; v[4 * i + 1] += a[i].y; v[4 * i + 2] += a[i].z; v[4 * i + 3] += a[i].w;
            }
          }
#pragma unroll
          for (int i = 0; i < 32; i += 4)
            *reinterpret_cast<float4*>(dst + i) = make_float4(v[i], v[i + 1], v[i + 2], v[i + 3]);
        } else {
#pragma unroll
          for (int i = 0; i < 32; ++i)
            if (nb + i < p.Cout) dst[i] = (p.epi == kEpiAccum ? dst[i] : 0.f) + v[i];
        }
      } else if (p.kind == kDgrad) {
        if (p.vec_in) {
          const int vc = nb >> 5;
          if (vc >= p.nchunk) continue;
          const Chunk c = chunk_at(p, vc);
          const Seg sg = p.seg[c.seg];
          if (!sg.dx) continue;
          float* dst = sg.dx + static_cast<int64_t>(m) * sg.C + c.coff;
          if (sg.mask) {
            const float* xr = sg.x + static_cast<int64_t>(m) * sg.C + c.coff;
#pragma unroll
            for (int i = 0; i < 32; ++i)
              if (i < c.valid) v[i] = xr[i] > 0.f ? v[i] : 0.f;
          }
          if (c.valid == 32) {
            if (p.epi == kEpiAccum) {
              float4 a[8];
#pragma unroll
              for (int i = 0; i < 8; ++i) a[i] = *reinterpret_cast<const float4*>(dst + 4 * i);
#pragma unroll
              for (int i = 0; i < 8; ++i) {
                v[4 * i] += a[i].x; v[4 * i + 1] += a[i].y; v[4 * i + 2] += a[i].z; v[4 * i + 3] += a[i].w;
              }
            }
#pragma unroll
            for (int i = 0; i < 32; i += 4)
              *reinterpret_cast<float4*>(dst + i) = make_float4(v[i], v[i + 1], v[i + 2], v[i + 3]);
          } else {
#pragma unroll
            for (int i = 0; i < 32; ++i)
              if (i < c.valid) dst[i] = (p.epi == kEpiAccum ? dst[i] : 0.f) + v[i];
          }
        } else {
#pragma unroll
          for (int i = 0; i < 32; ++i) {
            const int ci = nb + i;
            if (ci < p.C) {
              const Seg sg = p.seg[seg_of(p, ci)];
              if (sg.dx) {
                float* dst = sg.dx + static_cast<int64_t>(m) * sg.C + (ci - sg.cbase);
                float val = v[i];
                if (sg.mask && sg.x[static_cast<int64_t>(m) * sg.C + (ci - sg.cbase)] <= 0.f) val = 0.f;
                *dst = (p.epi == kEpiAccum ? *dst : 0.f) + val;
              }
            }
          }
        }
      } else {
        // WGRAD: row m = weight column (virtual), columns = co.
        if (p.epi == kEpiPartial) {
          float* dst = p.out + static_cast<int64_t>(blockIdx.z) * p.Ncols * p.M;
#pragma unroll
          for (int i = 0; i < 32; ++i)
            if (nb + i < p.Cout) dst[static_cast<int64_t>(nb + i) * p.M + m] = v[i];
        } else {
          bool valid;
          const int widx = wgrad_widx(p, m, valid);
          if (!valid) continue;
          if (p.epi == kEpiSgd) {
            // all 32 loads in flight before the stores (the stores may alias
            // later loads as far as the compiler knows, which would serialise
            // 32 DRAM round trips per thread)
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
    }  // halves
  } else if (warp == 4) {
    // ---------------- MMA issuer ----------------
    // The whole warp runs the loop so the descriptors are warp-uniform
    // (uniform registers, no per-MMA waterfall loop); one elected lane
    // issues. Issued from lane 0 alone, each MMA cost ~10-20 instructions,
    // which bounded the N<=128 tiles.
    const bool a_mn = (p.kind == kWgrad);
    const bool b_mn = (p.kind != kFprop);
    const uint32_t idesc = make_idesc_tf32(BN, a_mn, b_mn);
    const bool leader = elect_one();
    for (int it = 0; it < nkb; ++it) {
      const int s = it % STAGES;
      const uint32_t ph = (it / STAGES) & 1;
      mbar_wait(kSplitWarps ? split_bar(s) : full_bar(s), ph);
      if constexpr (!TMA) fence_proxy_async();  // cp.async/st.shared writes -> async proxy
      tc_fence_after();
      const uint32_t sa = base + s * L::kStage;
      const uint32_t sb = sa + L::kABytes;
      if (leader) {
#pragma unroll
        for (int kk = 0; kk < KW / 8; ++kk) {
          // K-major: advance 32 B inside the swizzled row; MN-major: next 8 K
          // rows (MN chunks KW*128 B apart).
          const uint64_t ad = a_mn ? make_sdesc(sa + kk * 1024, KW * 128, 512, kSw128Base32)
                                   : make_sdesc(sa + kk * 32, 16, 1024, kSw128);
          const uint64_t bd = b_mn ? make_sdesc(sb + kk * 1024, KW * 128, 512, kSw128Base32)
                                   : make_sdesc(sb + kk * 32, 16, 1024, kSw128);
          if constexpr (PRECISE) {
            // lo tiles sit kHalf bytes above the hi tiles with identical layout:
            // descriptor start address += kHalf >> 4
            constexpr uint64_t kLo = static_cast<uint64_t>(L::kHalf >> 4);
            tc_mma_tf32(tmem, ad + kLo, bd, idesc, (it > 0 || kk > 0) ? 1u : 0u);
            tc_mma_tf32(tmem, ad, bd + kLo, idesc, 1u);
            tc_mma_tf32(tmem, ad, bd, idesc, 1u);
          } else {
#pragma unroll
            for (int h = 0; h < kHalves; ++h)  // second M half: A rows 128..255 sit 16 KB above
              tc_mma_tf32(tmem + h * BN, ad + static_cast<uint64_t>(h * ((kBM * KW * 4) >> 4)), bd, idesc,
                          (it > 0 || kk > 0) ? 1u : 0u);
          }
        }
        tc_commit(empty_bar(s));
      }
      __syncwarp();
    }
    if (leader) tc_commit(accum_bar);
    __syncwarp();
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 4) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(kTmemCols) : "memory");
  }
}

}  // namespace vdnnk
