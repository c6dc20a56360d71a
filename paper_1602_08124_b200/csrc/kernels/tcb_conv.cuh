// BF16-storage implicit-GEMM convolution engine (tcgen05 kind::f16, fp32
// accumulation in TMEM) for the reference's elem_size = 2 mode
// (/root/reference/proj/include/vdnnsim/cost_model.hpp:69, config.hpp:112):
// every feature map, gradient map and weight the planner sizes at 2 bytes per
// element is stored as bf16; products are exact in fp32 and accumulate in
// fp32; each result is rounded once (round-to-nearest-even) when it is stored.
//
// Same three contractions as the fp32 engine (tc_conv.cuh):
//   FPROP  Y[p][co]         = sum_{r,s,ci} X[p@(r,s)][ci] * W[co][r][s][ci]
//   DGRAD  dX[p][ci]        = sum_{r,s,co} dY[p@(r',s')][co] * W[co][k-1-r'][k-1-s'][ci]   (stride 1)
//   WGRAD  dW[(r,s,ci)][co] = sum_{p} X[p@(r,s)][ci] * dY[p][co]
//
// One 128 x BN output tile per CTA, split-K over grid.z. A 128-byte operand
// row holds 64 bf16, so one stage carries twice the K depth of an fp32 stage
// in the same bytes (4 MMAs of K = 16 per stage):
//   warps 0-3 : producers. K-major rows (im2col of X or dY, K-major W) and
//               MN-major rows (W^T for dgrad, X^T / dY^T for wgrad: K = 64
//               rows of 64 MN elements per 8 KB chunk) are gathered with
//               16-byte cp.async when every channel count is a multiple of 8,
//               else element by element (first layers, odd channel counts),
//               into the UMMA SWIZZLE_128B canonical layouts; after the main
//               loop the same warps run the epilogue (tcgen05.ld 32x32b).
//   warp 4    : TMEM allocator + single-thread tcgen05.mma issuer; stages are
//               released with tcgen05.commit -> EMPTY barrier.
#pragma once
#include <cuda_bf16.h>

#include "tc_conv.cuh"

namespace vdnnk {

using bf16 = __nv_bfloat16;

constexpr int kBKb = 64;         // bf16 per K block = one 128-B swizzle row
constexpr int kMaxChunksB = 96;

struct BSeg {
  const bf16* x;  // NHWC [N][H][W][C]
  bf16* dx;       // NHWC gradient plane (dgrad output); nullptr = not materialised
  int C, cbase, mask;
};

struct ConvParamsB {
  int kind, epi, relu;
  int N, H, W, C;
  int Ho, Wo, Cout;
  int kh, kw, stride, pad;
  int nseg;
  BSeg seg[kMaxSegs];
  int nchunk, chunk_arith;         // 64-wide virtual channel chunks (arith: single segment)
  Chunk chunk[kMaxChunksB];
  int vec_in, vec_out;             // every segment C % 8 == 0 / Cout % 8 == 0: 16-B gathers
  int tap_pack;                    // single segment with C == 8 (a padded first layer): one K block =
                                   // 8 taps x 8 channels, K = (tap, c) flat, 16-B gathers per tap
  const bf16* w;                   // KRSC
  bf16* w_mut;                     // SGD epilogue target
  const bf16* bias;                // FC bias (fprop)
  const bf16* dy;
  bf16* y;
  float* out;                      // fp32 dW (kEpiGrad) or split-K partials (kEpiPartial)
  float lr;
  int M, Ncols, kblocks, kb_per_split, KK;
};

__device__ __forceinline__ Chunk chunk_at_b(const ConvParamsB& p, int i) {
  if (p.chunk_arith) {
    Chunk c;
    c.seg = 0;
    c.coff = static_cast<int32_t>(i * 64);
    const int v = p.C - i * 64;
    c.valid = static_cast<int32_t>(v < 64 ? v : 64);
    c.cbase = c.coff;
    return c;
  }
  return p.chunk[i];
}

__device__ __forceinline__ int seg_of_b(const ConvParamsB& p, int c) {
  int s = 0;
#pragma unroll 1
  for (int i = 1; i < p.nseg; ++i)
    if (c >= p.seg[i].cbase) s = i;
  return s;
}

// MN-major SWIZZLE_128B tile: chunk mc = 64 MN elements x 64 K rows (8 KB),
// K row k at 128 B; the 16-B granule j is XORed with (k % 8).
__device__ __forceinline__ uint32_t mnb_addr(uint32_t base, int k, int mc, int j) {
  return base + mc * 8192 + k * 128 + (((j ^ (k & 7)) & 7) << 4);
}

__device__ __forceinline__ void st_shared_u16(uint32_t addr, uint16_t v) {
  asm volatile("st.shared.u16 [%0], %1;" ::"r"(addr), "h"(v) : "memory");
}
__device__ __forceinline__ uint16_t ld_bits(const bf16* p) { return __bfloat16_as_ushort(__ldg(p)); }

__device__ __forceinline__ void tc_mma_bf16(uint32_t d_tmem, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                            uint32_t accumulate) {
  asm volatile(
      "{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n"
      " tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}\n" ::"r"(d_tmem),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate)
      : "memory");
}

// kind::f16 instruction descriptor: bf16 A/B, fp32 D, M = 128.
__host__ __device__ constexpr uint32_t make_idesc_bf16(int n, bool a_mn_major, bool b_mn_major) {
  return (1u << 4)                       // D format f32
         | (1u << 7)                     // A format bf16
         | (1u << 10)                    // B format bf16
         | ((a_mn_major ? 1u : 0u) << 15) | ((b_mn_major ? 1u : 0u) << 16) |
         (static_cast<uint32_t>(n >> 3) << 17) | (static_cast<uint32_t>(kBM >> 4) << 24);
}

// Whether a stage's gathers include element-wise st.shared writes (then the
// producer fences them into the async proxy before arriving).
__device__ __forceinline__ bool scalar_gathers(const ConvParamsB& p) {
  if (p.kind == kFprop) return !p.vec_in;
  if (p.kind == kDgrad) return !p.vec_in || !p.vec_out;
  return !p.vec_in || !p.vec_out;
}

// 64 consecutive flat K elements (r, s, c) of one im2col row (output pixel
// q), single segment: one pixel decode, the (tap, channel) walk advanced
// incrementally, 2-byte loads packed into eight 16-B shared stores at
// dst(j) (j = 16-B granule). First layers (C = 3) and other channel counts
// that are not multiples of 8.
template <class Dst>
__device__ __forceinline__ void gather_row64(const ConvParamsB& p, const bf16* x, bool row_ok, int oh0, int ow0,
                                             int n, int k0, Dst dst) {
  int tap = k0 / p.C, c = k0 - tap * p.C;
  int r = tap / p.kw, s = tap - r * p.kw;
  const bf16* rowp = nullptr;
  auto locate = [&]() {
    const int ih = oh0 + r, iw = ow0 + s;
    rowp = (row_ok && r < p.kh && ih >= 0 && ih < p.H && iw >= 0 && iw < p.W)
               ? x + ((static_cast<int64_t>(n) * p.H + ih) * p.W + iw) * p.C
               : nullptr;
  };
  locate();
#pragma unroll
  for (int j = 0; j < 8; ++j) {
    uint32_t w[4];
#pragma unroll
    for (int h = 0; h < 4; ++h) {
      uint32_t pair = 0;
#pragma unroll
      for (int t = 0; t < 2; ++t) {
        const uint16_t v = rowp ? ld_bits(rowp + c) : static_cast<uint16_t>(0);
        pair |= static_cast<uint32_t>(v) << (16 * t);
        if (++c == p.C) {
          c = 0;
          if (++s == p.kw) {
            s = 0;
            ++r;
          }
          locate();
        }
      }
      w[h] = pair;
    }
    asm volatile("st.shared.v4.u32 [%0], {%1, %2, %3, %4};" ::"r"(dst(j)), "r"(w[0]), "r"(w[1]), "r"(w[2]),
                 "r"(w[3])
                 : "memory");
  }
}

template <int BN>
struct GatherB {
  // ---- FPROP: A = im2col rows (pixel) x 64 channels, B = W rows (co) x 64 channels (both K-major)
  __device__ static void fprop(const ConvParamsB& p, int m0, int n0, int kb, uint32_t sa, uint32_t sb, int tid) {
    if (p.tap_pack) {
      // 16-B granule j = the 8 channels of tap 8*kb + j
      const int j = tid & 7;
      const int tap = kb * 8 + j;
      const bool tv = tap < p.kh * p.kw;
      const int r = tv ? tap / p.kw : 0, s = tv ? tap - (tap / p.kw) * p.kw : 0;
      const bf16* x = p.seg[0].x;
#pragma unroll 4
      for (int i = 0; i < kBM / 16; ++i) {
        const int row = (tid >> 3) + 16 * i;
        const int m = m0 + row;
        const bf16* src = x;
        uint32_t bytes = 0;
        if (m < p.M && tv) {
          const Pix q = decode_pix(m, p.Ho, p.Wo);
          const int ih = q.h * p.stride - p.pad + r, iw = q.w * p.stride - p.pad + s;
          if (ih >= 0 && ih < p.H && iw >= 0 && iw < p.W) {
            src = x + ((static_cast<int64_t>(q.n) * p.H + ih) * p.W + iw) * 8;
            bytes = 16;
          }
        }
        cp_async16(kmaj_addr(sa, row, j), src, bytes);
      }
#pragma unroll 4
      for (int i = 0; i < BN / 16; ++i) {
        const int row = (tid >> 3) + 16 * i;
        const int co = n0 + row;
        const bool ok = co < p.Cout && tv;
        cp_async16(kmaj_addr(sb, row, j), ok ? p.w + static_cast<int64_t>(co) * p.KK + tap * 8 : p.w, ok ? 16 : 0);
      }
      return;
    }
    if (p.vec_in) {
      const int tap = kb / p.nchunk, ck = kb - tap * p.nchunk;
      const int r = tap / p.kw, s = tap - r * p.kw;
      const Chunk c = chunk_at_b(p, ck);
      const BSeg sg = p.seg[c.seg];
      const int j = tid & 7;
      const bool jv = (j * 8) < c.valid;
#pragma unroll 4
      for (int i = 0; i < kBM / 16; ++i) {
        const int row = (tid >> 3) + 16 * i;
        const int m = m0 + row;
        const bf16* src = sg.x;
        uint32_t bytes = 0;
        if (m < p.M && jv) {
          const Pix q = decode_pix(m, p.Ho, p.Wo);
          const int ih = q.h * p.stride - p.pad + r, iw = q.w * p.stride - p.pad + s;
          if (ih >= 0 && ih < p.H && iw >= 0 && iw < p.W) {
            src = sg.x + ((static_cast<int64_t>(q.n) * p.H + ih) * p.W + iw) * sg.C + c.coff + j * 8;
            bytes = 16;
          }
        }
        cp_async16(kmaj_addr(sa, row, j), src, bytes);
      }
#pragma unroll 4
      for (int i = 0; i < BN / 16; ++i) {
        const int row = (tid >> 3) + 16 * i;
        const int co = n0 + row;
        const bf16* src = p.w;
        uint32_t bytes = 0;
        if (co < p.Cout && jv) {
          src = p.w + static_cast<int64_t>(co) * p.KK + tap * p.C + c.cbase + j * 8;
          bytes = 16;
        }
        cp_async16(kmaj_addr(sb, row, j), src, bytes);
      }
    } else if (p.nseg == 1) {
      // flat K = (r, s, c), one im2col row per thread (kBM = 128 threads)
      const int m = m0 + tid;
      const bool ok = m < p.M;
      const Pix q = decode_pix(ok ? m : 0, p.Ho, p.Wo);
      gather_row64(p, p.seg[0].x, ok, q.h * p.stride - p.pad, q.w * p.stride - p.pad, q.n, kb * kBKb,
                   [&](int j) { return kmaj_addr(sa, tid, j); });
      // B: weight row co, 64 contiguous K elements (tpr threads per row)
      constexpr int kTpr = 128 / BN, kPer = 64 / kTpr;
      const int row = tid / kTpr, part = tid % kTpr;
      const int co = n0 + row;
      const int k0 = kb * kBKb + part * kPer;
#pragma unroll
      for (int j = 0; j < kPer / 8; ++j) {
        uint32_t w[4];
#pragma unroll
        for (int h = 0; h < 4; ++h) {
          const int k = k0 + 8 * j + 2 * h;
          const uint16_t lo = (co < p.Cout && k < p.KK) ? ld_bits(p.w + static_cast<int64_t>(co) * p.KK + k) : 0;
          const uint16_t hi =
              (co < p.Cout && k + 1 < p.KK) ? ld_bits(p.w + static_cast<int64_t>(co) * p.KK + k + 1) : 0;
          w[h] = static_cast<uint32_t>(lo) | (static_cast<uint32_t>(hi) << 16);
        }
        asm volatile("st.shared.v4.u32 [%0], {%1, %2, %3, %4};" ::"r"(kmaj_addr(sb, row, part * (kPer / 8) + j)),
                     "r"(w[0]), "r"(w[1]), "r"(w[2]), "r"(w[3])
                     : "memory");
      }
    } else {
      // flat K = (r, s, c) over the concatenated channels; one bf16 per lane
      const int e = tid & 63;
      const int k = kb * kBKb + e;
      const bool kv = k < p.KK;
      int r = 0, s = 0, c = 0, sgi = 0;
      if (kv) {
        const int tap = k / p.C;
        c = k - tap * p.C;
        r = tap / p.kw;
        s = tap - r * p.kw;
        sgi = seg_of_b(p, c);
      }
      const BSeg sg = p.seg[sgi];
      const int cl = c - sg.cbase;
      const uint32_t eoff = (e & 7) * 2;
#pragma unroll 4
      for (int i = 0; i < kBM / 2; ++i) {
        const int row = (tid >> 6) + 2 * i;
        const int m = m0 + row;
        uint16_t v = 0;
        if (kv && m < p.M) {
          const Pix q = decode_pix(m, p.Ho, p.Wo);
          const int ih = q.h * p.stride - p.pad + r, iw = q.w * p.stride - p.pad + s;
          if (ih >= 0 && ih < p.H && iw >= 0 && iw < p.W)
            v = ld_bits(sg.x + ((static_cast<int64_t>(q.n) * p.H + ih) * p.W + iw) * sg.C + cl);
        }
        st_shared_u16(kmaj_addr(sa, row, e >> 3) + eoff, v);
      }
#pragma unroll 4
      for (int i = 0; i < BN / 2; ++i) {
        const int row = (tid >> 6) + 2 * i;
        const int co = n0 + row;
        uint16_t v = 0;
        if (kv && co < p.Cout) v = ld_bits(p.w + static_cast<int64_t>(co) * p.KK + k);
        st_shared_u16(kmaj_addr(sb, row, e >> 3) + eoff, v);
      }
    }
  }

  // ---- DGRAD (stride 1): A = im2col of dY over the input grid (pad' = k-1-pad),
  // K-major over co; B = W^T, MN-major: K rows = co, MN = virtual input channel.
  __device__ static void dgrad(const ConvParamsB& p, int m0, int n0, int kb, uint32_t sa, uint32_t sb, int tid) {
    const int padh = p.kh - 1 - p.pad, padw = p.kw - 1 - p.pad;
    const int nck = (p.Cout + 63) >> 6;
    const int tap = p.vec_out ? kb / nck : 0;
    const int co0 = p.vec_out ? (kb - tap * nck) * 64 : 0;
    const int KD = p.kh * p.kw * p.Cout;
    if (p.vec_out) {
      const int r = tap / p.kw, s = tap - r * p.kw;
      const int j = tid & 7;
      const bool jv = (co0 + j * 8) < p.Cout;
#pragma unroll 4
      for (int i = 0; i < kBM / 16; ++i) {
        const int row = (tid >> 3) + 16 * i;
        const int m = m0 + row;
        const bf16* src = p.dy;
        uint32_t bytes = 0;
        if (m < p.M && jv) {
          const Pix q = decode_pix(m, p.H, p.W);
          const int oh = q.h - padh + r, ow = q.w - padw + s;
          if (oh >= 0 && oh < p.Ho && ow >= 0 && ow < p.Wo) {
            src = p.dy + ((static_cast<int64_t>(q.n) * p.Ho + oh) * p.Wo + ow) * p.Cout + co0 + j * 8;
            bytes = 16;
          }
        }
        cp_async16(kmaj_addr(sa, row, j), src, bytes);
      }
    } else {
      const int e = tid & 63;
      const int k = kb * kBKb + e;
      const bool kv = k < KD;
      int r = 0, s = 0, co = 0;
      if (kv) {
        const int t = k / p.Cout;
        co = k - t * p.Cout;
        r = t / p.kw;
        s = t - r * p.kw;
      }
      const uint32_t eoff = (e & 7) * 2;
#pragma unroll 4
      for (int i = 0; i < kBM / 2; ++i) {
        const int row = (tid >> 6) + 2 * i;
        const int m = m0 + row;
        uint16_t v = 0;
        if (kv && m < p.M) {
          const Pix q = decode_pix(m, p.H, p.W);
          const int oh = q.h - padh + r, ow = q.w - padw + s;
          if (oh >= 0 && oh < p.Ho && ow >= 0 && ow < p.Wo)
            v = ld_bits(p.dy + ((static_cast<int64_t>(q.n) * p.Ho + oh) * p.Wo + ow) * p.Cout + co);
        }
        st_shared_u16(kmaj_addr(sa, row, e >> 3) + eoff, v);
      }
    }
    // B: row (k, mc) holds W[co(k)][flipped tap][virtual ci chunk mc]
    auto kdecode = [&](int k, int& co, int& rr, int& ss) {
      if (p.vec_out) {
        co = co0 + k;
        rr = tap / p.kw;
        ss = tap - rr * p.kw;
        return co < p.Cout;
      }
      const int kf = kb * kBKb + k;
      const bool kv = kf < KD;
      const int t = kv ? kf / p.Cout : 0;
      co = kv ? kf - t * p.Cout : 0;
      rr = t / p.kw;
      ss = t - rr * p.kw;
      return kv;
    };
    if (p.vec_in) {
      const int j = tid & 7;
#pragma unroll 2
      for (int i = 0; i < BN / 16; ++i) {
        const int q = (tid >> 3) + 16 * i;
        const int k = q & 63, mc = q >> 6;
        int co, rr, ss;
        const bool kv = kdecode(k, co, rr, ss);
        const int vc = (n0 >> 6) + mc;
        const bf16* src = p.w;
        uint32_t bytes = 0;
        if (kv && vc < p.nchunk) {
          const Chunk c = chunk_at_b(p, vc);
          if (j * 8 < c.valid) {
            const int ftap = (p.kh - 1 - rr) * p.kw + (p.kw - 1 - ss);
            src = p.w + static_cast<int64_t>(co) * p.KK + ftap * p.C + c.cbase + j * 8;
            bytes = 16;
          }
        }
        cp_async16(mnb_addr(sb, k, mc, j), src, bytes);
      }
    } else {
      const int e = tid & 63;
      const uint32_t eoff = (e & 7) * 2;
#pragma unroll 2
      for (int i = 0; i < BN / 2; ++i) {
        const int q = (tid >> 6) + 2 * i;
        const int k = q & 63, mc = q >> 6;
        int co, rr, ss;
        const bool kv = kdecode(k, co, rr, ss);
        const int ci = n0 + mc * 64 + e;
        uint16_t v = 0;
        if (kv && ci < p.C) {
          const int ftap = (p.kh - 1 - rr) * p.kw + (p.kw - 1 - ss);
          v = ld_bits(p.w + static_cast<int64_t>(co) * p.KK + ftap * p.C + ci);
        }
        st_shared_u16(mnb_addr(sb, k, mc, e >> 3) + eoff, v);
      }
    }
  }

  // ---- WGRAD: GEMM M = virtual (r,s,ci) weight columns, N = co, K = output pixels.
  // A: X_col^T, MN-major (K row = pixel, MN = weight column); B: dY^T, MN-major.
  __device__ static void wgrad(const ConvParamsB& p, int m0, int n0, int kb, uint32_t sa, uint32_t sb, int tid) {
    const int P = p.N * p.Ho * p.Wo;
    if (p.tap_pack) {
      // MN col = tap * 8 + c: the 16-B granule j of MN chunk mc is tap (m0 + 64 mc) / 8 + j
      const int j = tid & 7;
#pragma unroll 2
      for (int i = 0; i < kBM / 16; ++i) {
        const int q = (tid >> 3) + 16 * i;
        const int k = q & 63, mc = q >> 6;
        const int pix = kb * kBKb + k;
        const int tap = (m0 + mc * 64) / 8 + j;
        const bf16* src = p.seg[0].x;
        uint32_t bytes = 0;
        if (pix < P && tap < p.kh * p.kw) {
          const int r = tap / p.kw, s = tap - r * p.kw;
          const Pix x = decode_pix(pix, p.Ho, p.Wo);
          const int ih = x.h * p.stride - p.pad + r, iw = x.w * p.stride - p.pad + s;
          if (ih >= 0 && ih < p.H && iw >= 0 && iw < p.W) {
            src = p.seg[0].x + ((static_cast<int64_t>(x.n) * p.H + ih) * p.W + iw) * 8;
            bytes = 16;
          }
        }
        cp_async16(mnb_addr(sa, k, mc, j), src, bytes);
      }
    } else if (p.vec_in) {
      const int j = tid & 7;
#pragma unroll 2
      for (int i = 0; i < kBM / 16; ++i) {
        const int q = (tid >> 3) + 16 * i;
        const int k = q & 63, mc = q >> 6;
        const int pix = kb * kBKb + k;
        const int vcol = (m0 >> 6) + mc;
        const bf16* src = p.w;
        uint32_t bytes = 0;
        if (pix < P && vcol < p.kh * p.kw * p.nchunk) {
          const int tap = vcol / p.nchunk, ck = vcol - tap * p.nchunk;
          const Chunk c = chunk_at_b(p, ck);
          if (j * 8 < c.valid) {
            const int r = tap / p.kw, s = tap - r * p.kw;
            const Pix x = decode_pix(pix, p.Ho, p.Wo);
            const int ih = x.h * p.stride - p.pad + r, iw = x.w * p.stride - p.pad + s;
            if (ih >= 0 && ih < p.H && iw >= 0 && iw < p.W) {
              const BSeg sg = p.seg[c.seg];
              src = sg.x + ((static_cast<int64_t>(x.n) * p.H + ih) * p.W + iw) * sg.C + c.coff + j * 8;
              bytes = 16;
            }
          }
        }
        cp_async16(mnb_addr(sa, k, mc, j), src, bytes);
      }
    } else if (p.nseg == 1) {
      // one pixel (K row) x 64 consecutive flat weight columns per thread
      const int k = tid & 63, mc = tid >> 6;
      const int pix = kb * kBKb + k;
      const bool ok = pix < P;
      const Pix x = decode_pix(ok ? pix : 0, p.Ho, p.Wo);
      gather_row64(p, p.seg[0].x, ok, x.h * p.stride - p.pad, x.w * p.stride - p.pad, x.n, m0 + mc * 64,
                   [&](int j) { return mnb_addr(sa, k, mc, j); });
    } else {
      const int e = tid & 63;
      const uint32_t eoff = (e & 7) * 2;
#pragma unroll 2
      for (int i = 0; i < kBM / 2; ++i) {
        const int q = (tid >> 6) + 2 * i;
        const int k = q & 63, mc = q >> 6;
        const int pix = kb * kBKb + k;
        const int col = m0 + mc * 64 + e;  // flat (r, s, c)
        uint16_t v = 0;
        if (pix < P && col < p.KK) {
          const int tap = col / p.C, c = col - tap * p.C;
          const int r = tap / p.kw, s = tap - r * p.kw;
          const Pix x = decode_pix(pix, p.Ho, p.Wo);
          const int ih = x.h * p.stride - p.pad + r, iw = x.w * p.stride - p.pad + s;
          if (ih >= 0 && ih < p.H && iw >= 0 && iw < p.W) {
            const BSeg sg = p.seg[seg_of_b(p, c)];
            v = ld_bits(sg.x + ((static_cast<int64_t>(x.n) * p.H + ih) * p.W + iw) * sg.C + (c - sg.cbase));
          }
        }
        st_shared_u16(mnb_addr(sa, k, mc, e >> 3) + eoff, v);
      }
    }
    if (p.vec_out) {
      const int j = tid & 7;
#pragma unroll 2
      for (int i = 0; i < BN / 16; ++i) {
        const int q = (tid >> 3) + 16 * i;
        const int k = q & 63, mc = q >> 6;
        const int pix = kb * kBKb + k;
        const int co = n0 + mc * 64 + j * 8;
        const bf16* src = p.dy;
        uint32_t bytes = 0;
        if (pix < P && co < p.Cout) {
          src = p.dy + static_cast<int64_t>(pix) * p.Cout + co;
          bytes = 16;
        }
        cp_async16(mnb_addr(sb, k, mc, j), src, bytes);
      }
    } else {
      const int e = tid & 63;
      const uint32_t eoff = (e & 7) * 2;
#pragma unroll 2
      for (int i = 0; i < BN / 2; ++i) {
        const int q = (tid >> 6) + 2 * i;
        const int k = q & 63, mc = q >> 6;
        const int pix = kb * kBKb + k;
        const int co = n0 + mc * 64 + e;
        uint16_t v = 0;
        if (pix < P && co < p.Cout) v = ld_bits(p.dy + static_cast<int64_t>(pix) * p.Cout + co);
        st_shared_u16(mnb_addr(sb, k, mc, e >> 3) + eoff, v);
      }
    }
  }
};

// Weight-row index of a wgrad GEMM row m (virtual (tap, 64-chunk, lane) or flat).
__device__ __forceinline__ int wgrad_widx_b(const ConvParamsB& p, int m, bool& valid) {
  if (p.vec_in && !p.tap_pack) {
    const int vcol = m >> 6, lane = m & 63;
    const int tap = vcol / p.nchunk, ck = vcol - tap * p.nchunk;
    if (tap >= p.kh * p.kw) {
      valid = false;
      return 0;
    }
    const Chunk c = chunk_at_b(p, ck);
    valid = lane < c.valid;
    return tap * p.C + c.cbase + lane;
  }
  valid = m < p.KK;
  return m;
}

__device__ __forceinline__ uint32_t pack_bf16x2(float a, float b) {
  const __nv_bfloat162 h = __floats2bfloat162_rn(a, b);
  return *reinterpret_cast<const uint32_t*>(&h);
}
__device__ __forceinline__ void unpack_bf16x8(const uint4& u, float* f) {
  const uint32_t w[4] = {u.x, u.y, u.z, u.w};
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    f[2 * i] = __uint_as_float(w[i] << 16);
    f[2 * i + 1] = __uint_as_float(w[i] & 0xFFFF0000u);
  }
}
__device__ __forceinline__ float bf2f(bf16 v) { return __bfloat162float(v); }

// 32 consecutive outputs of one row (fp32 v[]) -> bf16 at dst (n valid,
// accumulate adds the stored values first). 16-B stores when all 32 are valid
// and dst is 16-B aligned.
__device__ __forceinline__ void store_row32(bf16* dst, float (&v)[32], int n, bool accumulate) {
  if (n >= 32 && (reinterpret_cast<uintptr_t>(dst) & 15) == 0) {
    uint4* d4 = reinterpret_cast<uint4*>(dst);
    if (accumulate) {
      uint4 a[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) a[i] = d4[i];
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        float f[8];
        unpack_bf16x8(a[i], f);
#pragma unroll
        for (int t = 0; t < 8; ++t) v[8 * i + t] += f[t];
      }
    }
#pragma unroll
    for (int i = 0; i < 4; ++i)
      d4[i] = make_uint4(pack_bf16x2(v[8 * i], v[8 * i + 1]), pack_bf16x2(v[8 * i + 2], v[8 * i + 3]),
                         pack_bf16x2(v[8 * i + 4], v[8 * i + 5]), pack_bf16x2(v[8 * i + 6], v[8 * i + 7]));
    return;
  }
#pragma unroll
  for (int i = 0; i < 32; ++i)
    if (i < n) dst[i] = __float2bfloat16_rn((accumulate ? bf2f(dst[i]) : 0.f) + v[i]);
}

// Warp-cooperative store of a 32-row x 32-column bf16 block whose row r sits
// in lane r (the TMEM lane layout) through a 2 KB per-warp shared-memory
// transpose. Stored straight from the lanes, every 16-B st.global of the warp
// touches 32 rows (32 half-sectors on as many lines); transposed, it covers 8
// rows x 64 B (16 full sectors), a quarter of the L1 / L2 store requests.
// Each lane passes its own row's destination (null: row not stored) and,
// for the fused ReLU-backward select, its row of x (null: no mask); the
// reader of a chunk fetches both from the row's lane. The 16-B chunk index is
// XOR-swizzled with (row >> 1) & 3, so the row writes and the chunk reads are
// bank-conflict free. The mask is applied per element after the transpose:
// rounding then zeroing equals zeroing then rounding, so the stored values
// are bit-identical to store_row32's.
__device__ __forceinline__ void store_tile32_t(uint32_t scratch, const float (&v)[32], bf16* dst, const bf16* mask) {
  const int lane = threadIdx.x & 31;
  const int q = lane & 3;
  // the rows this lane stores (8i + lane / 4, chunk q) and their ReLU-mask
  // chunks: the mask loads are issued first so they fly during the transpose
  bf16* d[4];
  uint4 x[4];
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int r = 8 * i + (lane >> 2);
    d[i] = reinterpret_cast<bf16*>(__shfl_sync(0xffffffffu, reinterpret_cast<uintptr_t>(dst), r));
    const bf16* mk = reinterpret_cast<const bf16*>(__shfl_sync(0xffffffffu, reinterpret_cast<uintptr_t>(mask), r));
    x[i] = make_uint4(0x3f803f80u, 0x3f803f80u, 0x3f803f80u, 0x3f803f80u);  // 1.0: keep
    if (mk && d[i]) x[i] = __ldg(reinterpret_cast<const uint4*>(mk) + q);
  }
  __syncwarp();  // the previous block's chunk reads are done
#pragma unroll
  for (int c = 0; c < 4; ++c)
    asm volatile("st.shared.v4.u32 [%0], {%1, %2, %3, %4};" ::"r"(scratch + lane * 64 + ((c ^ ((lane >> 1) & 3)) << 4)),
                 "r"(pack_bf16x2(v[8 * c], v[8 * c + 1])), "r"(pack_bf16x2(v[8 * c + 2], v[8 * c + 3])),
                 "r"(pack_bf16x2(v[8 * c + 4], v[8 * c + 5])), "r"(pack_bf16x2(v[8 * c + 6], v[8 * c + 7]))
                 : "memory");
  __syncwarp();
  // bf16 bits b: x > 0 <=> 0 < b <= 0x7f80 (+inf) -- sign clear, nonzero, not NaN
  auto keep = [](uint32_t b) {
    return (((b & 0xffffu) - 1u) < 0x7f80u ? 0xffffu : 0u) | (((b >> 16) - 1u) < 0x7f80u ? 0xffff0000u : 0u);
  };
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int r = 8 * i + (lane >> 2);
    uint4 w;
    asm volatile("ld.shared.v4.u32 {%0, %1, %2, %3}, [%4];"
                 : "=r"(w.x), "=r"(w.y), "=r"(w.z), "=r"(w.w)
                 : "r"(scratch + r * 64 + ((q ^ ((r >> 1) & 3)) << 4))
                 : "memory");
    if (d[i])
      reinterpret_cast<uint4*>(d[i])[q] =
          make_uint4(w.x & keep(x[i].x), w.y & keep(x[i].y), w.z & keep(x[i].z), w.w & keep(x[i].w));
  }
}

// TMA producer (one thread; single-segment layers with 8-multiple channel
// counts). A: im2col boxes of 128 B channel chunks (fprop: X, dgrad: dY, 128
// pixels = the K-major A tile; wgrad: X, 64 pixels = one MN-major chunk of 64
// weight columns). B: tiled boxes (fprop: W as (C, tap, Cout) -> BN K-major
// rows; dgrad: the same map, 64 ci x 64 co per MN chunk; wgrad: dY [P][Cout],
// 64 co x 64 pixels per MN chunk). Channels past C and pixels past P read as
// zeros (TMA out-of-bounds fill). Coordinates advance incrementally: the
// issuing thread is serial.
template <int BN>
struct TmaProducerB {
  int kind;
  int qw, qh, qn;       // fprop / dgrad: im2col window origin of the tile's first row
  int ck, nck, r, s;    // fprop / dgrad: current (tap, 64-channel chunk)
  int wch[2], wr[2], ws[2];  // wgrad: channel offset and tap of each MN chunk of A
  int p0, pw, ph, pn;   // wgrad: first pixel of the stage

  __device__ __forceinline__ void init(const ConvParamsB& p, int m0, int kb) {
    kind = p.kind;
    if (kind != kWgrad) {
      nck = kind == kFprop ? p.nchunk : (p.Cout + 63) >> 6;
      const int tap = kb / nck;
      ck = kb - tap * nck;
      r = tap / p.kw;
      s = tap - r * p.kw;
      if (kind == kFprop) {
        const Pix q = decode_pix(m0, p.Ho, p.Wo);
        qw = q.w * p.stride - p.pad;
        qh = q.h * p.stride - p.pad;
        qn = q.n;
      } else {
        const Pix q = decode_pix(m0, p.H, p.W);
        qw = q.w - (p.kw - 1 - p.pad);
        qh = q.h - (p.kh - 1 - p.pad);
        qn = q.n;
      }
    } else {
#pragma unroll
      for (int mc = 0; mc < 2; ++mc) {
        const int vc = (m0 >> 6) + mc;
        const int tap = vc / p.nchunk, c = vc - tap * p.nchunk;
        wr[mc] = tap / p.kw;
        ws[mc] = tap - wr[mc] * p.kw;
        wch[mc] = c * 64;
        if (tap >= p.kh * p.kw) wch[mc] = -1;  // past the last tap: left zero
      }
      p0 = kb * kBKb;
      const Pix q = decode_pix(p0, p.Ho, p.Wo);
      pw = q.w;
      ph = q.h;
      pn = q.n;
    }
  }

  __device__ __forceinline__ void issue(const ConvParamsB& p, const CUtensorMap* ta, const CUtensorMap* tb, int n0,
                                        uint32_t sa, uint32_t sb, uint32_t bar) const {
    if (kind == kFprop) {
      tma_load_im2col(sa, ta, bar, ck * 64, qw, qh, qn, static_cast<uint16_t>(s), static_cast<uint16_t>(r));
      tma_load_3d(sb, tb, bar, ck * 64, r * p.kw + s, n0);
    } else if (kind == kDgrad) {
      tma_load_im2col(sa, ta, bar, ck * 64, qw, qh, qn, static_cast<uint16_t>(s), static_cast<uint16_t>(r));
      const int ftap = (p.kh - 1 - r) * p.kw + (p.kw - 1 - s);
#pragma unroll
      for (int mc = 0; mc < BN / 64; ++mc) tma_load_3d(sb + mc * 8192, tb, bar, n0 + mc * 64, ftap, ck * 64);
    } else {
      const int iw = pw * p.stride - p.pad, ih = ph * p.stride - p.pad;
#pragma unroll
      for (int mc = 0; mc < 2; ++mc)
        if (wch[mc] >= 0)
          tma_load_im2col(sa + mc * 8192, ta, bar, wch[mc], iw, ih, pn, static_cast<uint16_t>(ws[mc]),
                          static_cast<uint16_t>(wr[mc]));
#pragma unroll
      for (int mc = 0; mc < BN / 64; ++mc) tma_load_2d(sb + mc * 8192, tb, bar, n0 + mc * 64, p0);
    }
  }

  // bytes one stage's loads deliver (the expect_tx count)
  __device__ __forceinline__ uint32_t bytes() const {
    if (kind == kWgrad) return (wch[0] >= 0 ? 8192u : 0u) + (wch[1] >= 0 ? 8192u : 0u) + BN * 128u;
    return kBM * 128u + BN * 128u;
  }

  __device__ __forceinline__ void next(const ConvParamsB& p) {
    if (kind != kWgrad) {
      if (++ck == nck) {
        ck = 0;
        if (++s == p.kw) {
          s = 0;
          ++r;
        }
      }
    } else {
      p0 += kBKb;
      pw += kBKb;
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

// Epilogue of one 128 x BN tile (warp w drains TMEM lanes 32w..32w+31; `row`
// = 32w + lane): split-K partials, or fused bias / ReLU / ReLU-backward mask /
// accumulation with bf16 stores, or the wgrad SGD update / fp32 dW.
// `drained()` runs right after the tile's last TMEM read (a persistent
// kernel releases the accumulator there). zero: the tile had no K blocks.
template <int BN, class Drained>
__device__ __forceinline__ void tcb_epilogue(const ConvParamsB& p, uint32_t taddr, int m0, int n0, int z, int row,
                                             bool zero, Drained drained, int cg_lo = 0, int cg_hi = BN / 32,
                                             uint32_t scratch = 0) {
  const int m = m0 + row;
#pragma unroll 1
  for (int cg = cg_lo; cg < cg_hi; ++cg) {
    float v[32];
    tmem_ld32(taddr + cg * 32, v);
    if (cg == cg_hi - 1) drained();
    if (zero) {
#pragma unroll
      for (int i = 0; i < 32; ++i) v[i] = 0.f;
    }
    const int nb = n0 + cg * 32;
    if (scratch && p.epi == kEpiStore) {
      // full 32-column blocks of a plain bf16 store: transposed through the
      // warp's scratch (every condition here is warp-uniform)
      if (p.kind == kFprop && (p.Cout & 7) == 0 && nb + 32 <= p.Cout) {
        if (p.bias) {
#pragma unroll
          for (int i = 0; i < 32; ++i) v[i] += bf2f(p.bias[nb + i]);
        }
        if (p.relu) {
#pragma unroll
          for (int i = 0; i < 32; ++i) v[i] = fmaxf(v[i], 0.f);
        }
        store_tile32_t(scratch, v, m < p.M ? p.y + static_cast<int64_t>(m) * p.Cout + nb : nullptr, nullptr);
        continue;
      }
      if (p.kind == kDgrad && p.vec_in && (nb >> 6) < p.nchunk) {
        const Chunk c = chunk_at_b(p, nb >> 6);
        const BSeg sg = p.seg[c.seg];
        const int co = c.coff + (nb & 63);
        if (sg.dx && c.valid - (nb & 63) >= 32 && (sg.C & 7) == 0 && (co & 7) == 0) {
          const int64_t at = static_cast<int64_t>(m) * sg.C + co;
          store_tile32_t(scratch, v, m < p.M ? sg.dx + at : nullptr, sg.mask ? sg.x + at : nullptr);
          continue;
        }
      }
    }
    if (m >= p.M) continue;
    if (p.epi == kEpiPartial && p.kind != kWgrad) {
      // split-K fprop / dgrad: fp32 partial slab z of [splits][M][Ncols]
      if (nb >= p.Ncols) continue;
      float* dst = p.out + (static_cast<int64_t>(z) * p.M + m) * p.Ncols + nb;
      if (nb + 32 <= p.Ncols && (p.Ncols & 3) == 0) {
#pragma unroll
        for (int i = 0; i < 32; i += 4) *reinterpret_cast<float4*>(dst + i) = make_float4(v[i], v[i + 1], v[i + 2], v[i + 3]);
      } else {
#pragma unroll
        for (int i = 0; i < 32; ++i)
          if (nb + i < p.Ncols) dst[i] = v[i];
      }
      continue;
    }
    if (p.kind == kFprop) {
      if (nb >= p.Cout) continue;
      if (p.bias) {
#pragma unroll
        for (int i = 0; i < 32; ++i)
          if (nb + i < p.Cout) v[i] += bf2f(p.bias[nb + i]);
      }
      if (p.relu) {
#pragma unroll
        for (int i = 0; i < 32; ++i) v[i] = fmaxf(v[i], 0.f);
      }
      store_row32(p.y + static_cast<int64_t>(m) * p.Cout + nb, v, p.Cout - nb, p.epi == kEpiAccum);
    } else if (p.kind == kDgrad) {
      if (p.vec_in) {
        const int vc = nb >> 6, off = nb & 63;
        if (vc >= p.nchunk) continue;
        const Chunk c = chunk_at_b(p, vc);
        const BSeg sg = p.seg[c.seg];
        const int valid = c.valid - off;
        if (!sg.dx || valid <= 0) continue;
        const int64_t at = static_cast<int64_t>(m) * sg.C + c.coff + off;
        if (sg.mask) {
          // fused ReLU backward: the ReLU's output is this conv's input x
          const bf16* xr = sg.x + at;
          if (valid >= 32 && (reinterpret_cast<uintptr_t>(xr) & 15) == 0) {
            uint4 xa[4];  // 4 x 16-B loads in flight, then the selects
#pragma unroll
            for (int i = 0; i < 4; ++i) xa[i] = __ldg(reinterpret_cast<const uint4*>(xr) + i);
#pragma unroll
            for (int i = 0; i < 4; ++i) {
              float f[8];
              unpack_bf16x8(xa[i], f);
#pragma unroll
              for (int t = 0; t < 8; ++t) v[8 * i + t] = f[t] > 0.f ? v[8 * i + t] : 0.f;
            }
          } else {
#pragma unroll
            for (int i = 0; i < 32; ++i)
              if (i < valid && !(bf2f(xr[i]) > 0.f)) v[i] = 0.f;
          }
        }
        store_row32(sg.dx + at, v, valid, p.epi == kEpiAccum);
      } else {
#pragma unroll 4
        for (int i = 0; i < 32; ++i) {
          const int ci = nb + i;
          if (ci >= p.C) break;
          const BSeg sg = p.seg[seg_of_b(p, ci)];
          if (!sg.dx) continue;
          const int64_t at = static_cast<int64_t>(m) * sg.C + (ci - sg.cbase);
          float val = v[i];
          if (sg.mask && !(bf2f(sg.x[at]) > 0.f)) val = 0.f;
          sg.dx[at] = __float2bfloat16_rn((p.epi == kEpiAccum ? bf2f(sg.dx[at]) : 0.f) + val);
        }
      }
    } else {
      // WGRAD: row m = weight column (virtual), columns = co
      if (p.epi == kEpiPartial) {
        float* dst = p.out + static_cast<int64_t>(z) * p.Ncols * p.M;
#pragma unroll
        for (int i = 0; i < 32; ++i)
          if (nb + i < p.Cout) dst[static_cast<int64_t>(nb + i) * p.M + m] = v[i];
        continue;
      }
      bool valid;
      const int widx = wgrad_widx_b(p, m, valid);
      if (!valid) continue;
      if (p.epi == kEpiSgd) {
        bf16* wcol = p.w_mut + static_cast<int64_t>(nb) * p.KK + widx;
        float wv[32];
#pragma unroll
        for (int i = 0; i < 32; ++i) wv[i] = (nb + i < p.Cout) ? bf2f(wcol[static_cast<int64_t>(i) * p.KK]) : 0.f;
#pragma unroll
        for (int i = 0; i < 32; ++i)
          if (nb + i < p.Cout) wcol[static_cast<int64_t>(i) * p.KK] = __float2bfloat16_rn(wv[i] - p.lr * v[i]);
      } else {
#pragma unroll
        for (int i = 0; i < 32; ++i)
          if (nb + i < p.Cout) p.out[static_cast<int64_t>(nb + i) * p.KK + widx] = v[i];
      }
    }
  }
}

template <int BN, int STAGES>
struct TcbSmem {
  static constexpr int kABytes = kBM * 128;
  static constexpr int kBBytes = BN * 128;
  static constexpr int kStage = kABytes + kBBytes;
  static constexpr int kTotal = STAGES * kStage + 1024 /*align slack*/ + 256 /*barriers*/;
};

template <int BN, int STAGES, bool TMA>
__global__ void __launch_bounds__(160, (TcbSmem<BN, STAGES>::kTotal <= 116 * 1024 ? 2 : 1))
    tcb_conv_kernel(const __grid_constant__ ConvParamsB p, const __grid_constant__ CUtensorMap tma_a,
                    const __grid_constant__ CUtensorMap tma_b) {
  extern __shared__ uint8_t smem_raw[];
  using L = TcbSmem<BN, STAGES>;
  const uint32_t raw = smem_u32(smem_raw);
  const uint32_t base = (raw + 1023u) & ~1023u;
  const uint32_t bar_base = base + STAGES * L::kStage;
  auto full_bar = [&](int s) { return bar_base + 8u * s; };
  auto empty_bar = [&](int s) { return bar_base + 8u * (STAGES + s); };
  const uint32_t accum_bar = bar_base + 8u * (2 * STAGES);
  const uint32_t tmem_slot = bar_base + 8u * (2 * STAGES + 1);
  uint32_t* tmem_slot_ptr = reinterpret_cast<uint32_t*>(smem_raw + (tmem_slot - raw));

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const int ntn = (p.Ncols + BN - 1) / BN;
  const int m0 = static_cast<int>(blockIdx.x / ntn) * kBM;
  const int n0 = static_cast<int>(blockIdx.x % ntn) * BN;
  const int kb_begin = blockIdx.z * p.kb_per_split;
  int kb_end = kb_begin + p.kb_per_split;
  if (kb_end > p.kblocks) kb_end = p.kblocks;
  const int nkb = kb_end - kb_begin;

  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(full_bar(s), TMA ? 1 : 128);  // TMA: one expect_tx arrival; else one per producer thread
      mbar_init(empty_bar(s), 1);
    }
    mbar_init(accum_bar, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 4) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(tmem_slot), "r"(BN)
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
        TmaProducerB<BN> tp;
        tp.init(p, m0, kb_begin);
        const uint32_t nbytes = tp.bytes();
        for (int it = 0; it < nkb; ++it) {
          const int s = it % STAGES;
          const uint32_t ph = (it / STAGES) & 1;
          if (it >= STAGES) mbar_wait(empty_bar(s), ph ^ 1);
          const uint32_t sa = base + s * L::kStage;
          mbar_expect_tx(full_bar(s), nbytes);
          tp.issue(p, &tma_a, &tma_b, n0, sa, sa + L::kABytes, full_bar(s));
          tp.next(p);
        }
      }
      __syncwarp();
    }
    const bool scalar = scalar_gathers(p);
    if constexpr (!TMA)
    for (int it = 0; it < nkb; ++it) {
      const int s = it % STAGES;
      const uint32_t ph = (it / STAGES) & 1;
      if (it >= STAGES) mbar_wait(empty_bar(s), ph ^ 1);
      const uint32_t sa = base + s * L::kStage;
      const uint32_t sb = sa + L::kABytes;
      const int kb = kb_begin + it;
      if (p.kind == kFprop)
        GatherB<BN>::fprop(p, m0, n0, kb, sa, sb, tid);
      else if (p.kind == kDgrad)
        GatherB<BN>::dgrad(p, m0, n0, kb, sa, sb, tid);
      else
        GatherB<BN>::wgrad(p, m0, n0, kb, sa, sb, tid);
      if (scalar) {
        // element-wise st.shared in this stage: one stage of lag -- once this
        // thread's copies of the PREVIOUS stage landed (its cp.async group),
        // make that stage's writes visible to the tensor core's (async) proxy
        // and arrive, so each thread keeps two stages of loads in flight
        cp_async_commit();
        cp_async_wait<1>();
        if (it > 0) {
          fence_proxy_async();
          mbar_arrive(full_bar((it - 1) % STAGES));
        }
      } else {
        cp_async_arrive_noinc(full_bar(s));
      }
    }
    if (scalar && nkb > 0) {
      cp_async_wait<0>();
      fence_proxy_async();
      mbar_arrive(full_bar((nkb - 1) % STAGES));
    }
    // ---------------- epilogue ----------------
    mbar_wait_sleep(accum_bar, 0);
    tc_fence_after();
    __syncwarp();
    tcb_epilogue<BN>(p, tmem + (static_cast<uint32_t>(warp * 32) << 16), m0, n0, static_cast<int>(blockIdx.z),
                     warp * 32 + lane, nkb <= 0, [] {});
  } else if (warp == 4) {
    // ---------------- MMA issuer ----------------
    const bool a_mn = (p.kind == kWgrad);
    const bool b_mn = (p.kind != kFprop);
    const uint32_t idesc = make_idesc_bf16(BN, a_mn, b_mn);
    const bool leader = elect_one();
    for (int it = 0; it < nkb; ++it) {
      const int s = it % STAGES;
      const uint32_t ph = (it / STAGES) & 1;
      mbar_wait(full_bar(s), ph);
      fence_proxy_async();
      tc_fence_after();
      const uint32_t sa = base + s * L::kStage;
      const uint32_t sb = sa + L::kABytes;
      if (leader) {
#pragma unroll
        for (int kk = 0; kk < kBKb / 16; ++kk) {
          // K-major: next 32 B inside the swizzled row; MN-major: next 16 K
          // rows (two 8-row swizzle atoms, 2 KB), MN chunks 8 KB apart.
          const uint64_t ad = a_mn ? make_sdesc(sa + kk * 2048, 8192, 1024, kSw128)
                                   : make_sdesc(sa + kk * 32, 16, 1024, kSw128);
          const uint64_t bd = b_mn ? make_sdesc(sb + kk * 2048, 8192, 1024, kSw128)
                                   : make_sdesc(sb + kk * 32, 16, 1024, kSw128);
          tc_mma_bf16(tmem, ad, bd, idesc, (it > 0 || kk > 0) ? 1u : 0u);
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
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(BN) : "memory");
  }
}

// Persistent variant (TMA producers only): one CTA per SM walks a static
// round-robin of (split, M tile, N tile) with a continuous stage ring and two
// TMEM accumulator sets, so tile t's epilogue overlaps tile t+1's loads and
// MMAs, and the per-tile launch / pipeline fill / TMEM setup of the
// one-tile-per-CTA kernel is paid once per SM. BN = 256 tiles (N = 256 MMAs:
// half the A bytes per FLOP of BN = 128) fit with two accumulator sets.
//   warps 0-3 : epilogue        warp 4 : TMEM owner + MMA issuer
//   warp 5    : TMA producer (TmaProducerB, per-tile init)
template <int BN, int STAGES>
struct TcbPersistSmem {
  static constexpr int kABytes = kBM * 128;
  static constexpr int kBBytes = BN * 128;
  static constexpr int kStage = kABytes + kBBytes;
  static constexpr int kTotal = STAGES * kStage + 1024 + 256;
  static_assert(2 * BN <= 512, "two accumulator sets must fit TMEM");
};

// GATHER = true: the producers are four warps gathering with cp.async /
// element-wise stores (GatherB: concatenated inputs, channel counts that are
// not multiples of 8 -- first layers), one stage of lag per thread; the
// epilogue moves to warps 5-8 (TMEM lane quarter = warp % 4).
template <int BN, int STAGES, bool GATHER = false>
__global__ void __launch_bounds__(GATHER ? 288 : 192, 1)
    tcb_persist_kernel(const __grid_constant__ ConvParamsB p, const __grid_constant__ CUtensorMap tma_a,
                       const __grid_constant__ CUtensorMap tma_b, int splits) {
  extern __shared__ uint8_t smem_raw[];
  using L = TcbPersistSmem<BN, STAGES>;
  const uint32_t base = (smem_u32(smem_raw) + 1023u) & ~1023u;
  const uint32_t bars = base + STAGES * L::kStage;
  auto full_bar = [&](int s) { return bars + 8u * s; };
  auto empty_bar = [&](int s) { return bars + 8u * (STAGES + s); };
  auto tfull = [&](int a) { return bars + 8u * (2 * STAGES + a); };
  auto tempty = [&](int a) { return bars + 8u * (2 * STAGES + 2 + a); };
  const uint32_t tmem_slot = bars + 8u * (2 * STAGES + 4);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int ntn = (p.Ncols + BN - 1) / BN;
  const int mt = (p.M + kBM - 1) / kBM;
  const int ntiles = mt * ntn * splits;
  // tile -> (split z, m0, n0, K-block range); the N tiles of one M tile are
  // adjacent (the A tile is re-hit in L2)
  auto decode = [&](int t, int& z, int& m0, int& n0, int& kb0, int& nkb) {
    z = t / (mt * ntn);
    const int r = t - z * mt * ntn;
    m0 = (r / ntn) * kBM;
    n0 = (r % ntn) * BN;
    kb0 = z * p.kb_per_split;
    nkb = min(p.kblocks, kb0 + p.kb_per_split) - kb0;
  };

  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(full_bar(s), GATHER ? 128 : 1);
      mbar_init(empty_bar(s), 1);
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(tfull(a), 1);
      mbar_init(tempty(a), 128);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 4) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(tmem_slot), "r"(2 * BN)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  uint32_t tmem;
  asm volatile("ld.shared.u32 %0, [%1];" : "=r"(tmem) : "r"(tmem_slot) : "memory");

  const bool producer = GATHER ? warp < 4 : warp == 5;
  if (producer) {
   if constexpr (GATHER) {
    // ---------------- gather producers (128 threads) ----------------
    const int tid = threadIdx.x;
    const bool scalar = scalar_gathers(p);
    int s = 0, it_all = 0;
    uint32_t ph = 1;
    for (int t = blockIdx.x; t < ntiles; t += gridDim.x) {
      int z, m0, n0, kb0, nkb;
      decode(t, z, m0, n0, kb0, nkb);
      for (int it = 0; it < nkb; ++it, ++it_all) {
        mbar_wait(empty_bar(s), ph);
        const uint32_t sa = base + s * L::kStage;
        const uint32_t sb = sa + L::kABytes;
        if (p.kind == kFprop)
          GatherB<BN>::fprop(p, m0, n0, kb0 + it, sa, sb, tid);
        else if (p.kind == kDgrad)
          GatherB<BN>::dgrad(p, m0, n0, kb0 + it, sa, sb, tid);
        else
          GatherB<BN>::wgrad(p, m0, n0, kb0 + it, sa, sb, tid);
        if (scalar) {
          // one stage of lag: the previous stage is complete once its
          // cp.async group landed; fence its st.shared writes, arrive
          cp_async_commit();
          cp_async_wait<1>();
          if (it_all > 0) {
            fence_proxy_async();
            mbar_arrive(full_bar(s == 0 ? STAGES - 1 : s - 1));
          }
        } else {
          cp_async_arrive_noinc(full_bar(s));
        }
        if (++s == STAGES) {
          s = 0;
          ph ^= 1;
        }
      }
    }
    if (scalar && it_all > 0) {
      cp_async_wait<0>();
      fence_proxy_async();
      mbar_arrive(full_bar(s == 0 ? STAGES - 1 : s - 1));
    }
   } else {
    // ---------------- TMA producer ----------------
    if (lane == 0) {
      asm volatile("prefetch.tensormap [%0];" ::"l"(&tma_a) : "memory");
      asm volatile("prefetch.tensormap [%0];" ::"l"(&tma_b) : "memory");
      int s = 0;
      uint32_t ph = 1;  // the first pass over the ring does not wait
      for (int t = blockIdx.x; t < ntiles; t += gridDim.x) {
        int z, m0, n0, kb0, nkb;
        decode(t, z, m0, n0, kb0, nkb);
        TmaProducerB<BN> tp;
        tp.init(p, m0, kb0);
        const uint32_t nbytes = tp.bytes();
        for (int it = 0; it < nkb; ++it) {
          mbar_wait(empty_bar(s), ph);
          const uint32_t sa = base + s * L::kStage;
          mbar_expect_tx(full_bar(s), nbytes);
          tp.issue(p, &tma_a, &tma_b, n0, sa, sa + L::kABytes, full_bar(s));
          tp.next(p);
          if (++s == STAGES) {
            s = 0;
            ph ^= 1;
          }
        }
      }
    }
    __syncwarp();
   }
  } else if (warp == 4) {
    // ---------------- MMA issuer ----------------
    const bool a_mn = (p.kind == kWgrad);
    const bool b_mn = (p.kind != kFprop);
    const uint32_t idesc = make_idesc_bf16(BN, a_mn, b_mn);
    const bool leader = elect_one();
    int s = 0, lt = 0;
    uint32_t ph = 0;
    for (int t = blockIdx.x; t < ntiles; t += gridDim.x, ++lt) {
      int z, m0, n0, kb0, nkb;
      decode(t, z, m0, n0, kb0, nkb);
      const int acc = lt & 1;
      if (lt >= 2) mbar_wait(tempty(acc), ((lt >> 1) & 1) ^ 1);
      tc_fence_after();
      const uint32_t d = tmem + acc * BN;
      for (int it = 0; it < nkb; ++it) {
        mbar_wait(full_bar(s), ph);
        if constexpr (GATHER) fence_proxy_async();  // cp.async writes -> async proxy
        tc_fence_after();
        const uint32_t sa = base + s * L::kStage;
        const uint32_t sb = sa + L::kABytes;
        if (leader) {
#pragma unroll
          for (int kk = 0; kk < kBKb / 16; ++kk) {
            const uint64_t ad = a_mn ? make_sdesc(sa + kk * 2048, 8192, 1024, kSw128)
                                     : make_sdesc(sa + kk * 32, 16, 1024, kSw128);
            const uint64_t bd = b_mn ? make_sdesc(sb + kk * 2048, 8192, 1024, kSw128)
                                     : make_sdesc(sb + kk * 32, 16, 1024, kSw128);
            tc_mma_bf16(d, ad, bd, idesc, (it > 0 || kk > 0) ? 1u : 0u);
          }
          tc_commit(empty_bar(s));
        }
        __syncwarp();
        if (++s == STAGES) {
          s = 0;
          ph ^= 1;
        }
      }
      if (leader) tc_commit(tfull(acc));
      __syncwarp();
    }
  } else if (GATHER ? warp >= 5 : warp < 4) {
    // ---------------- epilogue ----------------
    const int q = warp & 3;  // TMEM lane quarter this warp may access
    int lt = 0;
    for (int t = blockIdx.x; t < ntiles; t += gridDim.x, ++lt) {
      int z, m0, n0, kb0, nkb;
      decode(t, z, m0, n0, kb0, nkb);
      const int acc = lt & 1;
      mbar_wait_sleep(tfull(acc), (lt >> 1) & 1);
      tc_fence_after();
      const uint32_t ta = tmem + acc * BN + (static_cast<uint32_t>(q * 32) << 16);
      const uint32_t release = tempty(acc);
      tcb_epilogue<BN>(p, ta, m0, n0, z, q * 32 + lane, nkb <= 0, [&] {
        tc_fence_before();
        mbar_arrive(release);
      });
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 4) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(2 * BN) : "memory");
  }
}

}  // namespace vdnnk
