// Launchers for the BF16-storage conv engine (tcb_conv.cuh): fprop / dgrad /
// wgrad of every CONV and FC layer when the plan stores 2-byte elements
// (cost_model.hpp:69). Split-K partials are fp32 and reduced in a fixed order
// (deterministic, independent of where the partials live), as in conv.cu.
#include <algorithm>
#include <cstdlib>
#include <cstring>

#include "kernels.h"
#include "tcb_conv.cuh"
#include "tcb_halo.cuh"
#include "tc_conv_pair.cuh"
#include "tcb_pair.cuh"
#include "tma_maps.h"

namespace vdnnk {

// first-layer kernels (conv_c3tcb.cu)
bool c3b_fprop_eligible(const ConvArgs& a);
bool c3b_wgrad_eligible(const ConvArgs& a);
size_t c3b_wgrad_ws_bytes(const ConvArgs& a);
cudaError_t c3b_fprop(const ConvArgs& a, const void* w, void* y, cudaStream_t st);
cudaError_t c3b_wgrad(const ConvArgs& a, const void* dy, void* w, float lr, float* dw_out, float* ws, size_t ws_bytes,
                      cudaStream_t st);

namespace {
constexpr int kNumSmsB = 148;
constexpr int kStagesB = 3;  // 3 x 32 KB (BN = 128) or 4 x 24 KB (BN = 64): two CTAs per SM

bool build_common_b(const ConvArgs& a, ConvParamsB& p) {
  std::memset(&p, 0, sizeof(p));
  if (a.nseg < 1 || a.nseg > kMaxSegs) return false;
  p.N = a.n;
  p.H = a.h;
  p.W = a.w;
  p.Ho = a.ho();
  p.Wo = a.wo();
  p.Cout = a.cout;
  p.kh = a.kh;
  p.kw = a.kw;
  p.stride = a.stride;
  p.pad = a.pad;
  p.nseg = a.nseg;
  int cb = 0;
  bool vec = true;
  for (int i = 0; i < a.nseg; ++i) {
    p.seg[i].x = reinterpret_cast<const bf16*>(a.x[i]);
    p.seg[i].dx = reinterpret_cast<bf16*>(a.dx[i]);
    p.seg[i].C = a.c[i];
    p.seg[i].cbase = cb;
    p.seg[i].mask = a.mask_in[i];
    cb += a.c[i];
    if (a.c[i] % 8 != 0) vec = false;
  }
  p.C = cb;
  p.KK = a.kh * a.kw * cb;
  int nch = 0;
  if (vec && a.nseg == 1) {
    p.chunk_arith = 1;
    nch = (cb + 63) / 64;
  } else if (vec) {
    for (int i = 0; i < a.nseg && vec; ++i)
      for (int c0 = 0; c0 < a.c[i]; c0 += 64) {
        if (nch >= kMaxChunksB) {
          vec = false;
          break;
        }
        Chunk& c = p.chunk[nch++];
        c.seg = i;
        c.coff = c0;
        c.valid = std::min(64, a.c[i] - c0);
        c.cbase = p.seg[i].cbase + c0;
      }
  }
  p.vec_in = vec ? 1 : 0;
  p.nchunk = vec ? nch : 0;
  p.vec_out = (a.cout % 8 == 0) ? 1 : 0;
  p.tap_pack = (a.nseg == 1 && cb == 8 && a.kh * a.kw > 1) ? 1 : 0;
  return true;
}

template <int BN, int STAGES, bool TMA>
cudaError_t launch_b(const ConvParamsB& p, int splits, const CUtensorMap& ta, const CUtensorMap& tb,
                     cudaStream_t st) {
  using L = TcbSmem<BN, STAGES>;
  static bool attr = false;
  if (!attr) {
    const cudaError_t e = cudaFuncSetAttribute(tcb_conv_kernel<BN, STAGES, TMA>,
                                               cudaFuncAttributeMaxDynamicSharedMemorySize, L::kTotal);
    if (e != cudaSuccess) return e;
    attr = true;
  }
  const int tiles = ((p.M + kBM - 1) / kBM) * ((p.Ncols + BN - 1) / BN);
  const dim3 grid(static_cast<unsigned>(tiles), 1, static_cast<unsigned>(splits));
  tcb_conv_kernel<BN, STAGES, TMA><<<grid, 160, L::kTotal, st>>>(p, ta, tb);
  count_launch();
  return cudaGetLastError();
}

thread_local bool g_no_tma_b = false;
// VDNN_BF16_C3=0: first layers on the generic engine (A/B switch)
const bool g_no_c3b = [] {
  const char* e = std::getenv("VDNN_BF16_C3");
  return e && std::atoi(e) == 0;
}();

// Layers the TMA producers can feed (one segment, 8-multiple channel counts,
// square windows, stride-1 dgrad): they run the persistent kernel.
bool tma_ok_b(const ConvParamsB& p) {
  return !g_no_tma_b && !p.tap_pack && p.nseg == 1 && p.vec_in && p.vec_out && p.kh == p.kw && (p.kind != kDgrad || p.stride == 1);
}

// N tile width: persistent kernel 64 / 128 / 256, one-tile kernel 64 / 128.
int tile_n(const ConvParamsB& p) {
  if (p.Ncols <= 64) return 64;
  return (tma_ok_b(p) && p.Ncols >= 256) ? 256 : 128;
}
// CTAs that run concurrently: one persistent CTA per SM, or two one-tile CTAs.
bool gather_persist();
int slots_b(const ConvParamsB& p) { return (tma_ok_b(p) || gather_persist()) ? kNumSmsB : 2 * kNumSmsB; }

template <int BN, int STAGES, bool GATHER = false>
cudaError_t launch_persist_b(const ConvParamsB& p, int splits, const CUtensorMap& ta, const CUtensorMap& tb,
                             cudaStream_t st) {
  using L = TcbPersistSmem<BN, STAGES>;
  static bool attr = false;
  if (!attr) {
    const cudaError_t e = cudaFuncSetAttribute(tcb_persist_kernel<BN, STAGES, GATHER>,
                                               cudaFuncAttributeMaxDynamicSharedMemorySize, L::kTotal);
    if (e != cudaSuccess) return e;
    attr = true;
  }
  const int64_t tiles = static_cast<int64_t>((p.M + kBM - 1) / kBM) * ((p.Ncols + BN - 1) / BN) * splits;
  const int grid = static_cast<int>(std::min<int64_t>(tiles, kNumSmsB));
  tcb_persist_kernel<BN, STAGES, GATHER><<<grid, GATHER ? 288 : 192, L::kTotal, st>>>(p, ta, tb, splits);
  count_launch();
  return cudaGetLastError();
}

// VDNN_BF16_GATHER_PERSIST=0: the one-tile-per-CTA gather kernel (A/B switch)
bool gather_persist() {
  static const bool on = [] {
    const char* e = std::getenv("VDNN_BF16_GATHER_PERSIST");
    return !e || std::atoi(e) != 0;
  }();
  return on;
}

// Tensor maps of the TMA producer (tcb_conv.cuh TmaProducerB); false = the
// cp.async gathers (concatenated inputs, channel counts not 8-multiples,
// non-square windows).
bool make_maps_b(const ConvParamsB& p, int bn, CUtensorMap* ta, CUtensorMap* tb) {
  if (g_no_tma_b || p.nseg != 1 || !p.vec_in || !p.vec_out || p.kh != p.kw) return false;
  const cuuint64_t taps = static_cast<cuuint64_t>(p.kh) * p.kw;
  const cuuint64_t C = static_cast<cuuint64_t>(p.C), Co = static_cast<cuuint64_t>(p.Cout);
  constexpr CUtensorMapDataType kBf = CU_TENSOR_MAP_DATA_TYPE_BFLOAT16;
  if (p.kind == kFprop || p.kind == kDgrad) {
    const bool f = p.kind == kFprop;
    if (f ? !encode_im2col(ta, p.seg[0].x, p.N, p.H, p.W, p.C, p.kh, p.stride, p.pad, kBM,
                           CU_TENSOR_MAP_SWIZZLE_128B, 2)
          : (p.stride != 1 || !encode_im2col(ta, p.dy, p.N, p.Ho, p.Wo, p.Cout, p.kh, 1, p.kh - 1 - p.pad, kBM,
                                             CU_TENSOR_MAP_SWIZZLE_128B, 2)))
      return false;
    // W as (C, tap, Cout): fprop boxes of 64 ci x BN co (K-major rows = co);
    // dgrad boxes of 64 ci x 64 co (MN-major chunk: K rows = co)
    const cuuint64_t dims[3] = {C, taps, Co};
    const cuuint64_t strides[2] = {C * 2, taps * C * 2};
    const cuuint32_t box[3] = {64, 1, static_cast<cuuint32_t>(f ? bn : 64)};
    return encode_tiled(tb, p.w, 3, dims, strides, box, CU_TENSOR_MAP_SWIZZLE_128B, kBf);
  }
  if (!encode_im2col(ta, p.seg[0].x, p.N, p.H, p.W, p.C, p.kh, p.stride, p.pad, kBKb, CU_TENSOR_MAP_SWIZZLE_128B, 2))
    return false;
  const cuuint64_t P = static_cast<cuuint64_t>(p.N) * p.Ho * p.Wo;
  const cuuint64_t dims[2] = {Co, P};
  const cuuint64_t strides[1] = {Co * 2};
  const cuuint32_t box[2] = {64, static_cast<cuuint32_t>(kBKb)};
  return encode_tiled(tb, p.dy, 2, dims, strides, box, CU_TENSOR_MAP_SWIZZLE_128B, kBf);
}

// Halo-reuse kernel (tcb_halo.cuh) for stride-1 k x k FPROP / DGRAD over one
// NHWC tensor: 64-multiple channel counts, <= 128 output columns, a padded
// input row that fits one TMA box (<= 256 pixels) and >= 75% of a tile's 256
// virtual rows real outputs (VGG: 224x224x64, 112x112x{64,128}).
// VDNN_BF16_HALO=0 disables (A/B switch).
bool halo_params_b(const ConvParamsB& p, HaloParamsB& h) {
  static const bool on = [] {
    const char* e = std::getenv("VDNN_BF16_HALO");
    return !e || std::atoi(e) != 0;
  }();
  if (!on || g_no_tma_b || (p.kind != kFprop && p.kind != kDgrad)) return false;
  if (p.nseg != 1 || !p.vec_in || p.tap_pack || p.stride != 1 || p.kh != p.kw || p.kh != 3) return false;
  if (p.C % 64 != 0 || p.Cout % 64 != 0 || p.bias) return false;
  std::memset(&h, 0, sizeof(h));
  h.kind = p.kind;
  h.N = p.N;
  h.kh = p.kh;
  h.kw = p.kw;
  if (p.kind == kFprop) {
    h.Hin = p.H, h.Win = p.W, h.Cin = p.C, h.pad = p.pad;
    h.Hout = p.Ho, h.Wout = p.Wo, h.Cout = p.Cout;
    h.out = p.y;
    h.relu = p.relu;
  } else {
    if (p.seg[0].dx == nullptr || p.pad > p.kh - 1) return false;
    h.Hin = p.Ho, h.Win = p.Wo, h.Cin = p.Cout, h.pad = p.kh - 1 - p.pad;
    h.Hout = p.H, h.Wout = p.W, h.Cout = p.C;
    h.out = p.seg[0].dx;
    h.mask_x = p.seg[0].mask ? p.seg[0].x : nullptr;
  }
  if (h.Cout > 128) return false;
  h.accum = p.epi == kEpiAccum;
  static const int epi_t = [] {  // VDNN_BF16_EPI_T=0: lanes store their rows directly (A/B switch)
    const char* e = std::getenv("VDNN_BF16_EPI_T");
    return !e || std::atoi(e) != 0 ? 1 : 0;
  }();
  h.epi_t = epi_t;
  h.P = h.Win + 2 * h.pad;
  if (h.P > 256 || h.Wout + h.kw - 1 != h.P) return false;
  h.TH = 256 / h.P;
  if (4 * h.TH * h.Wout < 3 * 256) return false;
  h.nck = h.Cin / 64;
  h.tiles_h = (h.Hout + h.TH - 1) / h.TH;
  return true;
}

template <int BN, int AS, int BS, bool RESB = false>
cudaError_t launch_halo_b(HaloParamsB& h, const ConvParamsB& p, cudaStream_t st) {
  using L = HaloSmemB<BN, AS, BS>;
  alignas(64) CUtensorMap ta, tb;
  std::memset(&ta, 0, sizeof(ta));
  std::memset(&tb, 0, sizeof(tb));
  const bf16* src = p.kind == kFprop ? p.seg[0].x : p.dy;
  {
    const cuuint64_t dims[4] = {static_cast<cuuint64_t>(h.Cin), static_cast<cuuint64_t>(h.Win),
                                static_cast<cuuint64_t>(h.Hin), static_cast<cuuint64_t>(h.N)};
    const cuuint64_t strides[3] = {static_cast<cuuint64_t>(h.Cin) * 2, static_cast<cuuint64_t>(h.Win) * h.Cin * 2,
                                   static_cast<cuuint64_t>(h.Hin) * h.Win * h.Cin * 2};
    const cuuint32_t box[4] = {64, static_cast<cuuint32_t>(h.P), static_cast<cuuint32_t>(h.TH), 1};
    if (!encode_tiled(&ta, src, 4, dims, strides, box, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16))
      return cudaErrorNotSupported;
  }
  const int taps = p.kh * p.kw;
  if (p.kind == kFprop) {
    // W [Cout][KK] (KRSC): 64-channel x BN-row K-major boxes
    const cuuint64_t dims[2] = {static_cast<cuuint64_t>(p.KK), static_cast<cuuint64_t>(p.Cout)};
    const cuuint64_t strides[1] = {static_cast<cuuint64_t>(p.KK) * 2};
    const cuuint32_t box[2] = {64, static_cast<cuuint32_t>(BN)};
    if (!encode_tiled(&tb, p.w, 2, dims, strides, box, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16))
      return cudaErrorNotSupported;
  } else {
    // W [co][tap][ci] as (ci, tap, co): a 64 ci x 64 co box of one tap is an
    // MN-major SWIZZLE_128B chunk (K = co rows of 64 ci)
    const cuuint64_t dims[3] = {static_cast<cuuint64_t>(p.C), static_cast<cuuint64_t>(taps),
                                static_cast<cuuint64_t>(p.Cout)};
    const cuuint64_t strides[2] = {static_cast<cuuint64_t>(p.C) * 2, static_cast<cuuint64_t>(taps) * p.C * 2};
    const cuuint32_t box[3] = {64, 1, 64};
    if (!encode_tiled(&tb, p.w, 3, dims, strides, box, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16))
      return cudaErrorNotSupported;
  }
  h.ntn = (h.Cout + BN - 1) / BN;
  h.ntiles = h.N * h.tiles_h * h.ntn;
  if (RESB && (h.ntn != 1 || h.nck * h.kh * 3 != BS)) return cudaErrorNotSupported;
  static bool attr_set = false;
  if (!attr_set) {
    cudaError_t e = cudaFuncSetAttribute(tcb_halo_kernel<BN, AS, BS, 3, RESB>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, L::kTotal);
    if (e != cudaSuccess) return e;
    attr_set = true;
  }
  tcb_halo_kernel<BN, AS, BS, 3, RESB><<<std::min(h.ntiles, kNumSmsB), kHaloBThreads, L::kTotal, st>>>(h, ta, tb);
  count_launch();
  return cudaGetLastError();
}

// CTA-pair kernel (tcb_pair.cuh) for TMA-fed layers with 256-column tiles;
// wgrad only when every
// 128-row half holds real weight rows (M % 256 == 0: constant stage bytes).
// VDNN_BF16_PAIR=0 disables (A/B switch).
bool pair_ok_b(const ConvParamsB& p, int splits) {
  static const bool on = [] {
    const char* e = std::getenv("VDNN_BF16_PAIR");
    return !e || std::atoi(e) != 0;
  }();
  if (!on || !tma_ok_b(p) || tile_n(p) != 256) return false;
  if (p.kind == kWgrad && p.M % 256 != 0) return false;
  (void)splits;  // an item is two single-CTA tiles: the pair grid keeps as many SMs busy
  return true;
}

template <int STAGES>
cudaError_t launch_pair_b(const ConvParamsB& p, int splits, const CUtensorMap& ta, const CUtensorMap& tb,
                          cudaStream_t st) {
  using L = TcbPairSmem<STAGES>;
  static bool attr = false;
  if (!attr) {
    const cudaError_t e =
        cudaFuncSetAttribute(tcb_pair_kernel<STAGES>, cudaFuncAttributeMaxDynamicSharedMemorySize, L::kTotal);
    if (e != cudaSuccess) return e;
    attr = true;
  }
  const int64_t items = static_cast<int64_t>((p.M + 255) / 256) * ((p.Ncols + 255) / 256) * splits;
  const int grid = 2 * static_cast<int>(std::min<int64_t>(items, kNumSmsB / 2));
  static const int epi_t = [] {  // VDNN_BF16_EPI_T=0: lanes store their rows directly (A/B switch)
    const char* e = std::getenv("VDNN_BF16_EPI_T");
    return !e || std::atoi(e) != 0 ? 1 : 0;
  }();
  tcb_pair_kernel<STAGES><<<grid, kTcbPairThreads, L::kTotal, st>>>(p, ta, tb, splits, epi_t);
  count_launch();
  return cudaGetLastError();
}

cudaError_t launch_any(const ConvParamsB& p, int splits, cudaStream_t st) {
  if (splits == 1) {
    HaloParamsB h;
    if (halo_params_b(p, h)) {
      static const bool resb = [] {  // VDNN_BF16_HALO_RESB=0: stream the filter per tile (A/B switch)
        const char* e = std::getenv("VDNN_BF16_HALO_RESB");
        return !e || std::atoi(e) != 0;
      }();
      cudaError_t e = cudaErrorNotSupported;
      if (resb && h.Cout == 64 && h.nck == 1) e = launch_halo_b<64, 4, 9, true>(h, p, st);  // 64 -> 64: 72 KB filter
      if (e == cudaErrorNotSupported)
        e = h.Cout <= 64 ? launch_halo_b<64, 4, 8>(h, p, st) : launch_halo_b<128, 4, 4>(h, p, st);
      if (e != cudaErrorNotSupported) return e;
    }
  }
  if (p.M <= 0 || p.Ncols <= 0) return cudaSuccess;
  const int bn = tile_n(p);
  alignas(64) CUtensorMap ta, tb;
  std::memset(&ta, 0, sizeof(ta));
  std::memset(&tb, 0, sizeof(tb));
  if (pair_ok_b(p, splits) && make_maps_b(p, 128, &ta, &tb)) return launch_pair_b<6>(p, splits, ta, tb, st);
  if (tma_ok_b(p) && make_maps_b(p, bn, &ta, &tb)) {
    if (bn == 256) return launch_persist_b<256, 4>(p, splits, ta, tb, st);
    if (bn == 128) return launch_persist_b<128, 6>(p, splits, ta, tb, st);
    return launch_persist_b<64, 8>(p, splits, ta, tb, st);
  }
  if (gather_persist())
    return bn == 64 ? launch_persist_b<64, 8, true>(p, splits, ta, tb, st)
                    : launch_persist_b<128, 6, true>(p, splits, ta, tb, st);
  return bn == 64 ? launch_b<64, 4, false>(p, splits, ta, tb, st) : launch_b<128, kStagesB, false>(p, splits, ta, tb, st);
}

// Split-K factor (same time model as conv.cu's pick_splits): waves of
// ceil(kblocks / s) K blocks against the partial slabs' write + re-read.
int pick_splits_b(int tiles, int kblocks, int bn, int64_t outputs, int slots) {
  int best = 1;
  double best_t = 1e30;
  const int smax = std::max(1, std::min(1024, kblocks / 4));
  for (int s = 1; s <= smax; ++s) {
    const double waves = static_cast<double>((static_cast<int64_t>(tiles) * s + slots - 1) / slots);
    const double kbps = static_cast<double>((kblocks + s - 1) / s);
    const double t_main = waves * kbps * 4.0 * bn / 1.9e9;
    const double t_part = s > 1 ? static_cast<double>(s) * static_cast<double>(outputs) * 8.0 / 5e12 : 0.0;
    const double t = t_main + t_part;
    if (t < best_t * (1 - 1e-6)) {
      best_t = t;
      best = s;
    }
  }
  return best;
}

int clamp_splits(ConvParamsB& p, int splits, size_t per, size_t ws_bytes) {
  if (splits > 1) splits = static_cast<int>(std::min<size_t>(splits, per ? ws_bytes / per : 1));
  if (splits < 1) splits = 1;
  p.kb_per_split = (p.kblocks + splits - 1) / splits;
  return (p.kblocks + p.kb_per_split - 1) / p.kb_per_split;
}

// ----------------------------------------------------------------- FPROP ---
bool fprop_params_b(const ConvArgs& a, const void* w, const void* bias, void* y, bool accumulate, ConvParamsB& p) {
  if (!build_common_b(a, p)) return false;
  p.kind = kFprop;
  p.relu = a.relu_out;
  p.epi = accumulate ? kEpiAccum : kEpiStore;
  p.w = static_cast<const bf16*>(w);
  p.bias = static_cast<const bf16*>(bias);
  p.y = static_cast<bf16*>(y);
  p.M = a.n * p.Ho * p.Wo;
  p.Ncols = a.cout;
  p.kblocks = p.tap_pack ? (a.kh * a.kw + 7) / 8 : p.vec_in ? a.kh * a.kw * p.nchunk : (p.KK + kBKb - 1) / kBKb;
  p.kb_per_split = p.kblocks;
  return true;
}

// FC layers at small batch: fewer output tiles than SMs over a long reduction.
int fprop_splits_b(const ConvParamsB& p) {
  if (p.epi != kEpiStore || p.nseg != 1 || !p.vec_in || !p.vec_out) return 1;
  const int tiles = ((p.M + kBM - 1) / kBM) * ((p.Ncols + tile_n(p) - 1) / tile_n(p));
  if (tiles >= kNumSmsB || p.kblocks < 32) return 1;
  return pick_splits_b(tiles, p.kblocks, tile_n(p), static_cast<int64_t>(p.M) * p.Cout, slots_b(p));
}

__global__ void fprop_reduce_b_kernel(const float* __restrict__ part, int splits, int64_t m, int cout,
                                      const bf16* __restrict__ bias, int relu, bf16* __restrict__ y) {
  const int64_t total = m * cout;
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < total;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    float s = part[i];
    for (int z = 1; z < splits; ++z) s += part[z * total + i];  // fixed order: deterministic
    if (bias) s += __bfloat162float(bias[i % cout]);
    if (relu) s = fmaxf(s, 0.f);
    y[i] = __float2bfloat16_rn(s);
  }
}

// ----------------------------------------------------------------- DGRAD ---
bool dgrad_params_b(const ConvArgs& a, const void* w, const void* dy, bool accumulate, ConvParamsB& p) {
  if (!build_common_b(a, p)) return false;
  p.kind = kDgrad;
  p.tap_pack = 0;  // dgrad keeps the 64-channel chunks
  p.epi = accumulate ? kEpiAccum : kEpiStore;
  p.w = static_cast<const bf16*>(w);
  p.dy = static_cast<const bf16*>(dy);
  p.M = a.n * a.h * a.w;
  p.Ncols = p.vec_in ? p.nchunk * 64 : p.C;
  p.kblocks = p.vec_out ? a.kh * a.kw * ((a.cout + 63) / 64) : (a.kh * a.kw * a.cout + kBKb - 1) / kBKb;
  p.kb_per_split = p.kblocks;
  return true;
}

int dgrad_splits_b(const ConvParamsB& p) {
  if (p.nseg != 1 || !p.vec_in || !p.vec_out || p.kh != 1 || p.kw != 1 || p.H != 1 || p.W != 1 || p.C % 64 != 0)
    return 1;
  const int tiles = ((p.M + kBM - 1) / kBM) * ((p.Ncols + tile_n(p) - 1) / tile_n(p));
  if (tiles >= kNumSmsB || p.kblocks < 32) return 1;
  return pick_splits_b(tiles, p.kblocks, tile_n(p), static_cast<int64_t>(p.M) * p.C, slots_b(p));
}

__global__ void dgrad_reduce_b_kernel(const float* __restrict__ part, int splits, int64_t m, int c,
                                      const bf16* __restrict__ mask_x, int accumulate, bf16* __restrict__ dx) {
  const int64_t total = m * c;
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < total;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    float s = part[i];
    for (int z = 1; z < splits; ++z) s += part[z * total + i];
    if (mask_x && !(__bfloat162float(mask_x[i]) > 0.f)) s = 0.f;
    if (accumulate) s += __bfloat162float(dx[i]);
    dx[i] = __float2bfloat16_rn(s);
  }
}

// ----------------------------------------------------------------- WGRAD ---
int wgrad_rows_b(const ConvParamsB& p) {
  return (p.vec_in && !p.tap_pack) ? p.kh * p.kw * p.nchunk * 64 : p.KK;
}

int wgrad_splits_b(const ConvParamsB& p, int M, int64_t P) {
  ConvParamsB q = p;  // tile shape of the launch (kind and Ncols as conv_wgrad_bf16 sets them)
  q.kind = kWgrad;
  q.Ncols = p.Cout;
  const int bn = tile_n(q);
  const int tiles = ((M + kBM - 1) / kBM) * ((p.Cout + bn - 1) / bn);
  const int kblocks = static_cast<int>((P + kBKb - 1) / kBKb);
  return pick_splits_b(tiles, kblocks, bn, static_cast<int64_t>(M) * p.Cout, slots_b(q));
}

__global__ void wgrad_reduce_b_kernel(const __grid_constant__ ConvParamsB p, int splits, float* __restrict__ dw) {
  const int64_t total = static_cast<int64_t>(p.Cout) * p.M;
  for (int64_t idx = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; idx < total;
       idx += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int m = static_cast<int>(idx % p.M);
    const int co = static_cast<int>(idx / p.M);
    bool valid;
    const int widx = wgrad_widx_b(p, m, valid);
    if (!valid) continue;
    float s = 0.f;
    for (int k = 0; k < splits; ++k) s += p.out[static_cast<int64_t>(k) * total + idx];
    const int64_t at = static_cast<int64_t>(co) * p.KK + widx;
    if (dw)
      dw[at] = s;
    else
      p.w_mut[at] = __float2bfloat16_rn(__bfloat162float(p.w_mut[at]) - p.lr * s);
  }
}

int reduce_blocks(int64_t total) { return static_cast<int>(std::min<int64_t>((total + 255) / 256, 8 * kNumSmsB)); }
}  // namespace

bool conv_bf16_c3_native(const ConvArgs& a) { return !g_no_c3b && c3b_fprop_eligible(a) && c3b_wgrad_eligible(a); }

void set_tma_bf16(bool on) { g_no_tma_b = !on; }

size_t conv_fprop_ws_bytes_bf16(const ConvArgs& a) {
  if (c3b_fprop_eligible(a)) return 0;
  ConvParamsB p;
  if (!fprop_params_b(a, nullptr, nullptr, nullptr, false, p)) return 0;
  const int s = fprop_splits_b(p);
  return s > 1 ? static_cast<size_t>(s) * p.M * p.Cout * sizeof(float) : 0;
}

cudaError_t conv_fprop_bf16(const ConvArgs& a, const void* w, const void* bias, void* y, bool accumulate,
                            cudaStream_t st, float* ws, size_t ws_bytes) {
  if (!accumulate && bias == nullptr && !g_no_c3b && c3b_fprop_eligible(a)) return c3b_fprop(a, w, y, st);
  ConvParamsB p;
  if (!fprop_params_b(a, w, bias, y, accumulate, p)) return cudaErrorInvalidValue;
  const size_t per = static_cast<size_t>(p.M) * p.Cout * sizeof(float);
  const int splits = clamp_splits(p, ws ? fprop_splits_b(p) : 1, per, ws_bytes);
  if (splits <= 1) {
    p.kb_per_split = p.kblocks;
    return launch_any(p, 1, st);
  }
  p.epi = kEpiPartial;
  p.out = ws;
  cudaError_t e = launch_any(p, splits, st);
  if (e != cudaSuccess) return e;
  const int64_t total = static_cast<int64_t>(p.M) * p.Cout;
  fprop_reduce_b_kernel<<<reduce_blocks(total), 256, 0, st>>>(ws, splits, p.M, p.Cout, p.bias, p.relu, p.y);
  count_launch();
  return cudaGetLastError();
}

size_t conv_dgrad_ws_bytes_bf16(const ConvArgs& a) {
  ConvParamsB p;
  if (a.stride != 1 || !dgrad_params_b(a, nullptr, nullptr, false, p)) return 0;
  const int s = dgrad_splits_b(p);
  return s > 1 ? static_cast<size_t>(s) * p.M * p.C * sizeof(float) : 0;
}

cudaError_t conv_dgrad_bf16(const ConvArgs& a, const void* w, const void* dy, bool accumulate, cudaStream_t st,
                            float* ws, size_t ws_bytes) {
  ConvParamsB p;
  if (!dgrad_params_b(a, w, dy, accumulate, p)) return cudaErrorInvalidValue;
  if (a.stride != 1) return cudaErrorNotSupported;
  const size_t per = static_cast<size_t>(p.M) * p.C * sizeof(float);
  const int splits = clamp_splits(p, (ws && p.seg[0].dx) ? dgrad_splits_b(p) : 1, per, ws_bytes);
  if (splits <= 1) {
    p.kb_per_split = p.kblocks;
    return launch_any(p, 1, st);
  }
  const bool accum = p.epi == kEpiAccum;
  p.epi = kEpiPartial;
  p.out = ws;
  cudaError_t e = launch_any(p, splits, st);
  if (e != cudaSuccess) return e;
  const int64_t total = static_cast<int64_t>(p.M) * p.C;
  dgrad_reduce_b_kernel<<<reduce_blocks(total), 256, 0, st>>>(ws, splits, p.M, p.C,
                                                               p.seg[0].mask ? p.seg[0].x : nullptr, accum ? 1 : 0,
                                                               p.seg[0].dx);
  count_launch();
  return cudaGetLastError();
}

// Halo WGRAD (tcb_halo.cuh) for stride-1 3x3 layers with 64-multiple input
// channels and 64 / 128 output channels whose padded input row fits a box.
// VDNN_BF16_HALO_WGRAD=0 disables (A/B switch).
constexpr size_t kSmemLimitB = 227 * 1024;
bool halo_wgb_params(const ConvParamsB& p, HaloWgParamsB& h) {
  static const bool on = [] {
    const char* e = std::getenv("VDNN_BF16_HALO_WGRAD");
    return !e || std::atoi(e) != 0;
  }();
  if (!on || g_no_tma_b) return false;
  if (p.nseg != 1 || !p.vec_in || p.tap_pack || p.stride != 1 || p.kh != p.kw || p.kh != 3) return false;
  if (p.C % 64 != 0 || (p.Cout != 64 && p.Cout != 128) || p.pad > p.kh - 1) return false;
  std::memset(&h, 0, sizeof(h));
  h.N = p.N, h.H = p.H, h.W = p.W, h.C = p.C, h.Cout = p.Cout, h.kh = p.kh, h.kw = p.kw, h.pad = p.pad;
  h.P = p.W + 2 * p.pad;
  h.Hout = p.Ho, h.Wout = p.Wo;
  if (h.Wout + h.kw - 1 != h.P || h.P > 240) return false;
  h.Kp = (h.P + 15) / 16 * 16;
  h.nck = p.C / 64;
  const int nblk = h.kh * h.nck, gmax = 512 / (2 * p.Cout);
  // G = the largest divisor of the block count that fits TMEM: every group
  // of CTAs carries the same number of blocks (64 -> 128 channels: 3 blocks,
  // G = 2 left half the CTAs idle for a third of the time)
  h.G = 1;
  for (int gd = std::min(gmax, nblk); gd >= 1; --gd)
    if (nblk % gd == 0) {
      h.G = gd;
      break;
    }
  h.ngroups = nblk / h.G;
  h.nrows = h.N * h.Hout;
  const int splits = std::max(1, kNumSmsB / h.ngroups);
  h.rows_per = (h.nrows + splits - 1) / splits;
  h.M = p.kh * p.kw * h.nck * 64;
  h.a_slot = halo_wgb_a_slot(h.Kp);
  h.b_slot = halo_wgb_b_slot(h.Kp, p.Cout);
  h.BS = 2;
  const size_t fixed = 1024 + 256 + static_cast<size_t>(h.BS) * h.b_slot;
  if (fixed + 2 * static_cast<size_t>(h.a_slot) > kSmemLimitB) return false;
  h.AS = static_cast<int>(std::min<size_t>(kHwbMaxAS, (kSmemLimitB - fixed) / h.a_slot));
  return true;
}
int halo_wgb_splits(const HaloWgParamsB& h) { return (h.nrows + h.rows_per - 1) / h.rows_per; }
size_t halo_wgb_smem(const HaloWgParamsB& h) {
  return 1024 + 256 + static_cast<size_t>(h.BS) * h.b_slot + static_cast<size_t>(h.AS) * h.a_slot;
}

template <int BN>
cudaError_t launch_halo_wgrad_b(HaloWgParamsB& h, const ConvParamsB& p, cudaStream_t st) {
  alignas(64) CUtensorMap tx, tdy;
  std::memset(&tx, 0, sizeof(tx));
  std::memset(&tdy, 0, sizeof(tdy));
  {
    // X as (c, w, h, n): one padded input row of 64 channels per box (zero fill = padding)
    const cuuint64_t dims[4] = {static_cast<cuuint64_t>(h.C), static_cast<cuuint64_t>(h.W),
                                static_cast<cuuint64_t>(h.H), static_cast<cuuint64_t>(h.N)};
    const cuuint64_t strides[3] = {static_cast<cuuint64_t>(h.C) * 2, static_cast<cuuint64_t>(h.W) * h.C * 2,
                                   static_cast<cuuint64_t>(h.H) * h.W * h.C * 2};
    const cuuint32_t box[4] = {64, static_cast<cuuint32_t>(h.P), 1, 1};
    if (!encode_tiled(&tx, p.seg[0].x, 4, dims, strides, box, CU_TENSOR_MAP_SWIZZLE_128B,
                      CU_TENSOR_MAP_DATA_TYPE_BFLOAT16))
      return cudaErrorNotSupported;
  }
  {
    // dY as (co, x, y, n): one output row of 64 channels, P pixels (x >= Wout zero-filled)
    const cuuint64_t dims[4] = {static_cast<cuuint64_t>(h.Cout), static_cast<cuuint64_t>(h.Wout),
                                static_cast<cuuint64_t>(h.Hout), static_cast<cuuint64_t>(h.N)};
    const cuuint64_t strides[3] = {static_cast<cuuint64_t>(h.Cout) * 2, static_cast<cuuint64_t>(h.Wout) * h.Cout * 2,
                                   static_cast<cuuint64_t>(h.Hout) * h.Wout * h.Cout * 2};
    const cuuint32_t box[4] = {64, static_cast<cuuint32_t>(h.P), 1, 1};
    if (!encode_tiled(&tdy, p.dy, 4, dims, strides, box, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16))
      return cudaErrorNotSupported;
  }
  const size_t smem = halo_wgb_smem(h);
  static size_t attr = 0;
  if (smem > attr) {
    cudaError_t e = cudaFuncSetAttribute(tcb_wgrad_halo_kernel<BN>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         static_cast<int>(smem));
    if (e != cudaSuccess) return e;
    attr = smem;
  }
  tcb_wgrad_halo_kernel<BN><<<halo_wgb_splits(h) * h.ngroups, 192, smem, st>>>(h, tx, tdy);
  count_launch();
  return cudaGetLastError();
}

size_t conv_wgrad_ws_bytes_bf16(const ConvArgs& a) {
  ConvParamsB p;
  if (!build_common_b(a, p)) return 0;
  const int M = wgrad_rows_b(p);
  const int64_t P = static_cast<int64_t>(a.n) * p.Ho * p.Wo;
  const int s = wgrad_splits_b(p, M, P);
  size_t b = s > 1 ? static_cast<size_t>(s) * M * a.cout * sizeof(float) : 0;
  ConvParamsB q = p;
  q.kind = kWgrad;
  HaloWgParamsB h;
  if (halo_wgb_params(q, h)) b = std::max(b, static_cast<size_t>(halo_wgb_splits(h)) * h.M * a.cout * sizeof(float));
  return c3b_wgrad_eligible(a) ? std::max(b, c3b_wgrad_ws_bytes(a)) : b;
}

cudaError_t conv_wgrad_bf16(const ConvArgs& a, const void* dy, void* w_mut, float lr, float* dw_out, float* ws,
                            size_t ws_bytes, cudaStream_t st) {
  if (!g_no_c3b && c3b_wgrad_eligible(a) && ws != nullptr && ws_bytes >= c3b_wgrad_ws_bytes(a))
    return c3b_wgrad(a, dy, w_mut, lr, dw_out, ws, ws_bytes, st);
  ConvParamsB p;
  if (!build_common_b(a, p)) return cudaErrorInvalidValue;
  p.kind = kWgrad;
  p.dy = static_cast<const bf16*>(dy);
  p.w = static_cast<const bf16*>(w_mut);
  p.w_mut = static_cast<bf16*>(w_mut);
  p.lr = lr;
  p.M = wgrad_rows_b(p);
  p.Ncols = a.cout;
  const int64_t P = static_cast<int64_t>(a.n) * p.Ho * p.Wo;
  p.kblocks = static_cast<int>((P + kBKb - 1) / kBKb);
  {
    HaloWgParamsB h;
    if (ws != nullptr && halo_wgb_params(p, h) &&
        ws_bytes >= static_cast<size_t>(halo_wgb_splits(h)) * h.M * a.cout * sizeof(float)) {
      h.part = ws;
      cudaError_t e = p.Cout == 64 ? launch_halo_wgrad_b<64>(h, p, st) : launch_halo_wgrad_b<128>(h, p, st);
      if (e == cudaSuccess) {
        p.out = ws;
        wgrad_reduce_b_kernel<<<reduce_blocks(static_cast<int64_t>(p.Cout) * p.M), 256, 0, st>>>(
            p, halo_wgb_splits(h), dw_out);
        count_launch();
        return cudaGetLastError();
      }
      if (e != cudaErrorNotSupported) return e;
    }
  }
  const size_t per = static_cast<size_t>(p.M) * a.cout * sizeof(float);
  const int splits = clamp_splits(p, ws ? wgrad_splits_b(p, p.M, P) : 1, per, ws_bytes);
  if (splits <= 1) {
    p.epi = dw_out ? kEpiGrad : kEpiSgd;
    p.out = dw_out;
    p.kb_per_split = p.kblocks;
    return launch_any(p, 1, st);
  }
  p.epi = kEpiPartial;
  p.out = ws;
  cudaError_t e = launch_any(p, splits, st);
  if (e != cudaSuccess) return e;
  const int64_t total = static_cast<int64_t>(p.Cout) * p.M;
  wgrad_reduce_b_kernel<<<reduce_blocks(total), 256, 0, st>>>(p, splits, dw_out);
  count_launch();
  return cudaGetLastError();
}

}  // namespace vdnnk
