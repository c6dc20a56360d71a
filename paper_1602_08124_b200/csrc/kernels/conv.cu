// Launchers for the tcgen05 implicit-GEMM conv engine (tc_conv.cuh).
#include <cuda.h>

#include <algorithm>
#include <atomic>
#include <cstdlib>
#include <cstring>

#include "kernels.h"
#include "tc_conv.cuh"
#include "tc_conv_persist.cuh"
#include "tc_conv_halo.cuh"
#include "tc_conv_pair.cuh"
#include "tc_conv_halo_pair.cuh"
#include "tma_maps.h"

namespace vdnnk {

bool smallc_eligible(const ConvArgs& a);
cudaError_t smallc_fprop(const ConvArgs& a, const float* w, float* y, cudaStream_t st);
size_t smallc_wgrad_ws_bytes(const ConvArgs& a, int* nblocks_out);
cudaError_t smallc_wgrad(const ConvArgs& a, const float* dy, float* w, float lr, float* dw_out, float* ws,
                         size_t ws_bytes, cudaStream_t st);
bool c3tc_fprop_eligible(const ConvArgs& a);
bool c3tc_wgrad_eligible(const ConvArgs& a);
size_t c3tc_wgrad_ws_bytes(const ConvArgs& a);
cudaError_t c3tc_fprop(const ConvArgs& a, const float* w, float* y, cudaStream_t st);
cudaError_t c3tc_wgrad(const ConvArgs& a, const float* dy, float* w, float lr, float* dw_out, float* ws,
                       size_t ws_bytes, cudaStream_t st);

namespace {
std::atomic<uint64_t> g_launches{0};
constexpr int kStages = 3;         // 3 x 32 KB (BN=128): two CTAs per SM overlap mainloop and epilogue
constexpr int kStagesPrecise = 3;
constexpr int kNumSms = 148;
constexpr int kStagesWide = 4;     // 4 x 48 KB (BN=256): one CTA per SM
thread_local int g_sm_reserve = -1;  // SMs the persistent conv kernels leave free (compressed transfers)

// CTAs (one per SM) of the persistent conv kernels: all 148 SMs, minus an
// even reserve for concurrent SM-driven transfers (zvc.cu kernels cannot
// co-reside with a ~200 KB-smem conv CTA; without a reserve they wait for a
// whole persistent conv kernel, or hold SMs a persistent kernel's
// statically scheduled CTAs need).
int persist_sms() {
  int r = g_sm_reserve;
  if (r < 0) {
    const char* e = std::getenv("VDNN_SM_RESERVE");
    r = e ? std::atoi(e) : 0;
  }
  r = std::max(0, std::min(r, 64)) & ~1;
  return kNumSms - r;
}

bool build_common(const ConvArgs& a, ConvParams& p) {
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
    p.seg[i].x = a.x[i];
    p.seg[i].dx = a.dx[i];
    p.seg[i].C = a.c[i];
    p.seg[i].cbase = cb;
    p.seg[i].mask = a.mask_in[i];
    cb += a.c[i];
    if (a.c[i] % 4 != 0) vec = false;
  }
  p.C = cb;
  p.KK = a.kh * a.kw * cb;
  // virtual 32-channel chunks per segment
  int nch = 0;
  if (vec && a.nseg == 1) {
    p.chunk_arith = 1;
    nch = (cb + 31) / 32;
  } else if (vec) {
    for (int i = 0; i < a.nseg && vec; ++i) {
      for (int c0 = 0; c0 < a.c[i]; c0 += 32) {
        if (nch >= kMaxChunks) {
          vec = false;
          break;
        }
        Chunk& c = p.chunk[nch++];
        c.seg = static_cast<int32_t>(i);
        c.coff = static_cast<int32_t>(c0);
        c.valid = static_cast<int32_t>(std::min(32, a.c[i] - c0));
        c.cbase = static_cast<int32_t>(p.seg[i].cbase + c0);
      }
    }
  }
  p.vec_in = vec ? 1 : 0;
  p.nchunk = vec ? nch : 0;
  p.vec_out = (a.cout % 4 == 0) ? 1 : 0;
  return true;
}

}  // namespace

// ---------------------------------------------------------- tensor maps ---
using PfnTiled = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                              const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                              CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
using PfnIm2col = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                               const cuuint64_t*, const int*, const int*, cuuint32_t, cuuint32_t, const cuuint32_t*,
                               CUtensorMapInterleave, CUtensorMapSwizzle, CUtensorMapL2promotion,
                               CUtensorMapFloatOOBfill);

void* driver_fn(const char* name) {
  void* f = nullptr;
  cudaDriverEntryPointQueryResult q;
  if (cudaGetDriverEntryPoint(name, &f, cudaEnableDefault, &q) != cudaSuccess || q != cudaDriverEntryPointSuccess)
    return nullptr;
  return f;
}

bool encode_tiled(CUtensorMap* m, const void* base, int rank, const cuuint64_t* dims, const cuuint64_t* strides,
                  const cuuint32_t* box, CUtensorMapSwizzle sw, CUtensorMapDataType dt) {
  static PfnTiled fn = reinterpret_cast<PfnTiled>(driver_fn("cuTensorMapEncodeTiled"));
  if (!fn) return false;
  const cuuint32_t es[5] = {1, 1, 1, 1, 1};
  return fn(m, dt, static_cast<cuuint32_t>(rank), const_cast<void*>(base), dims,
            strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE, sw, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

// NHWC [n][h][w][c] as an im2col source: windows of k x k with padding `pad`
// and stride `stride`; `pixels` rows of one 128-byte channel chunk per load
// (32 fp32 or, esz = 2, 64 bf16 channels).
bool encode_im2col(CUtensorMap* m, const void* base, int n, int h, int w, int c, int k, int stride, int pad,
                   int pixels, CUtensorMapSwizzle sw, int esz) {
  static PfnIm2col fn = reinterpret_cast<PfnIm2col>(driver_fn("cuTensorMapEncodeIm2col"));
  if (!fn) return false;
  const cuuint64_t dims[4] = {static_cast<cuuint64_t>(c), static_cast<cuuint64_t>(w), static_cast<cuuint64_t>(h),
                              static_cast<cuuint64_t>(n)};
  const cuuint64_t e = static_cast<cuuint64_t>(esz);
  const cuuint64_t strides[3] = {static_cast<cuuint64_t>(c) * e, static_cast<cuuint64_t>(w) * c * e,
                                 static_cast<cuuint64_t>(h) * w * c * e};
  const int lower[2] = {-pad, -pad};
  const int upper[2] = {pad - (k - 1), pad - (k - 1)};
  const cuuint32_t es[4] = {1, static_cast<cuuint32_t>(stride), static_cast<cuuint32_t>(stride), 1};
  return fn(m, esz == 2 ? CU_TENSOR_MAP_DATA_TYPE_BFLOAT16 : CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4,
            const_cast<void*>(base), dims, strides, lower, upper, static_cast<cuuint32_t>(128 / esz),
            static_cast<cuuint32_t>(pixels), es, CU_TENSOR_MAP_INTERLEAVE_NONE, sw, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

// 2D output map [rows][cols] for the TMA-store epilogue (128-row x 32-col boxes).
bool encode_out(CUtensorMap* m, const void* base, int64_t rows, int cols) {
  const cuuint64_t dims[2] = {static_cast<cuuint64_t>(cols), static_cast<cuuint64_t>(rows)};
  const cuuint64_t strides[1] = {static_cast<cuuint64_t>(cols) * 4};
  const cuuint32_t box[2] = {32, static_cast<cuuint32_t>(kBM)};
  return encode_tiled(m, base, 2, dims, strides, box, CU_TENSOR_MAP_SWIZZLE_128B);
}

// 3D [splits][rows][cols] fp32 partial-sum slabs (split-K fprop), 128 x 32 boxes.
bool encode_out3(CUtensorMap* m, const void* base, int splits, int64_t rows, int cols) {
  const cuuint64_t dims[3] = {static_cast<cuuint64_t>(cols), static_cast<cuuint64_t>(rows),
                              static_cast<cuuint64_t>(splits)};
  const cuuint64_t strides[2] = {static_cast<cuuint64_t>(cols) * 4, static_cast<cuuint64_t>(rows) * cols * 4};
  const cuuint32_t box[3] = {32, static_cast<cuuint32_t>(kBM), 1};
  return encode_tiled(m, base, 3, dims, strides, box, CU_TENSOR_MAP_SWIZZLE_128B);
}

namespace {

// Build the maps of the TMA producer (and output); false = cp.async gathers.
template <int BN, int KW = kBK>
bool make_maps(ConvParams& p, CUtensorMap* ta, CUtensorMap* tb, CUtensorMap* tc) {
  if (p.nseg != 1 || !p.vec_in || !p.vec_out || p.kh != p.kw) return false;
  const float* x = p.seg[0].x;
  if (p.kind == kFprop) {
    if (p.epi == kEpiPartial) {
      if (!encode_out3(tc, p.out, p.splits, p.M, p.Cout)) return false;
    } else if (!encode_out(tc, p.y, p.M, p.Cout)) {
      return false;
    }
    if (!encode_im2col(ta, x, p.N, p.H, p.W, p.C, p.kh, p.stride, p.pad, kBM, CU_TENSOR_MAP_SWIZZLE_128B))
      return false;
    const cuuint64_t dims[2] = {static_cast<cuuint64_t>(p.KK), static_cast<cuuint64_t>(p.Cout)};
    const cuuint64_t strides[1] = {static_cast<cuuint64_t>(p.KK) * 4};
    const cuuint32_t box[2] = {32, static_cast<cuuint32_t>(BN)};
    return encode_tiled(tb, p.w, 2, dims, strides, box, CU_TENSOR_MAP_SWIZZLE_128B);
  }
  if (p.kind == kDgrad) {
    if (p.stride != 1 || p.seg[0].dx == nullptr) return false;
    if (p.epi == kEpiPartial) {
      if (!encode_out3(tc, p.out, p.splits, p.M, p.C)) return false;
    } else if (!encode_out(tc, p.seg[0].dx, p.M, p.C)) {
      return false;
    }
    if (!encode_im2col(ta, p.dy, p.N, p.Ho, p.Wo, p.Cout, p.kh, 1, p.kh - 1 - p.pad, kBM,
                       CU_TENSOR_MAP_SWIZZLE_128B))
      return false;
    const int taps = p.kh * p.kw;
    if (p.C % 32 == 0) {
      // one load per stage: (32 ci, co, ci-chunk, tap) -> smem [chunk][32 co][32 ci]
      const cuuint64_t d4[4] = {32, static_cast<cuuint64_t>(p.Cout), static_cast<cuuint64_t>(p.C / 32),
                                static_cast<cuuint64_t>(taps)};
      const cuuint64_t s4[3] = {static_cast<cuuint64_t>(taps) * p.C * 4, 128, static_cast<cuuint64_t>(p.C) * 4};
      const cuuint32_t b4[4] = {32, 32, static_cast<cuuint32_t>(BN / 32), 1};
      p.tma_b_merged = 1;
      return encode_tiled(tb, p.w, 4, d4, s4, b4, CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B);
    }
    const cuuint64_t dims[3] = {static_cast<cuuint64_t>(p.C), static_cast<cuuint64_t>(taps),
                                static_cast<cuuint64_t>(p.Cout)};
    const cuuint64_t strides[2] = {static_cast<cuuint64_t>(p.C) * 4, static_cast<cuuint64_t>(taps) * p.C * 4};
    const cuuint32_t box[3] = {32, 1, 32};
    return encode_tiled(tb, p.w, 3, dims, strides, box, CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B);
  }
  if (!encode_im2col(ta, x, p.N, p.H, p.W, p.C, p.kh, p.stride, p.pad, KW, CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B))
    return false;
  const int64_t P = static_cast<int64_t>(p.N) * p.Ho * p.Wo;
  if (p.Cout % 32 == 0) {
    // one load per stage: (32 co, pixel, co-chunk) -> smem [chunk][32 pixels][32 co]
    const cuuint64_t d3[3] = {32, static_cast<cuuint64_t>(P), static_cast<cuuint64_t>(p.Cout / 32)};
    const cuuint64_t s3[2] = {static_cast<cuuint64_t>(p.Cout) * 4, 128};
    const cuuint32_t b3[3] = {32, KW, static_cast<cuuint32_t>(BN / 32)};
    p.tma_b_merged = 1;
    return encode_tiled(tb, p.dy, 3, d3, s3, b3, CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B);
  }
  const cuuint64_t dims[2] = {static_cast<cuuint64_t>(p.Cout), static_cast<cuuint64_t>(P)};
  const cuuint64_t strides[1] = {static_cast<cuuint64_t>(p.Cout) * 4};
  const cuuint32_t box[2] = {32, KW};
  return encode_tiled(tb, p.dy, 2, dims, strides, box, CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B);
}

// Which kinds use BN=256 tiles when the layer is wide enough (bit per kind;
// VDNN_WIDE_TILES overrides for experiments).
int wide_mask() {
  static const int m = [] {
    const char* e = std::getenv("VDNN_WIDE_TILES");
    return e ? std::atoi(e) : 7;
  }();
  return m;
}
bool use_wide(int kind) { return (wide_mask() >> kind) & 1; }
// wgrad: any layer with >= 256 output channels (split-K keeps the SMs busy);
// fprop/dgrad: only >= 256 columns (measured +12..16% at 256) with >= 4 waves of wide tiles, so halving
// the resident CTAs per SM neither starves the grid nor exposes epilogues.
bool wide_ok(const ConvParams& p) {
  if (p.Ncols < 256 || !use_wide(p.kind)) return false;
  if (p.kind == kWgrad) return static_cast<int64_t>(p.kblocks) * p.wkw >= 2048;  // mirrors wgrad_cfg
  const int64_t tiles = static_cast<int64_t>((p.M + kBM - 1) / kBM) * ((p.Ncols + 255) / 256);
  static const int min_cols = [] {
    const char* e = std::getenv("VDNN_WIDE_MIN");
    return e ? std::atoi(e) : 256;
  }();
  return p.Ncols >= min_cols && tiles >= 4 * kNumSms;
}

// BM = 256 tiles (two M=128 MMAs per K step): bit per kind; VDNN_TALL overrides.
int tall_mask() {
  static const int m = [] {
    const char* e = std::getenv("VDNN_TALL");
    return e ? std::atoi(e) : 7;
  }();
  return m;
}
bool tall_deep() {
  static const bool d = [] {
    const char* e = std::getenv("VDNN_TALL_DEEP");
    return e && std::atoi(e) != 0;
  }();
  return d;
}
// enough tall tiles for at least two waves of one CTA per SM
bool tall_ok(const ConvParams& p, int bn, int splits) {
  if (!((tall_mask() >> p.kind) & 1)) return false;
  if (p.kind == kWgrad && (bn != 256 || static_cast<int64_t>(p.kblocks) * kBK < 100000)) return false;
  const int64_t tiles = static_cast<int64_t>((p.M + 255) / 256) * ((p.Ncols + bn - 1) / bn) * splits;
  return tiles >= 2 * kNumSms;
}

thread_local bool g_precise = false;
thread_local bool g_no_tma = false;

template <int BN, int STAGES, bool PRECISE, bool TMA, int BM = kBM, int KW = kBK>
cudaError_t launch_bn(const ConvParams& p, const CUtensorMap& ta, const CUtensorMap& tb, const CUtensorMap& tc,
                      int splits, cudaStream_t st) {
  using L = TcSmem<BN, STAGES, PRECISE, BM, KW>;
  static bool attr_set = false;
  if (!attr_set) {
    cudaError_t e = cudaFuncSetAttribute(tc_conv_kernel<BN, STAGES, PRECISE, TMA, BM, KW>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, L::kTotal);
    if (e != cudaSuccess) return e;
    attr_set = true;
  }
  const unsigned tiles = static_cast<unsigned>((p.M + BM - 1) / BM) * static_cast<unsigned>((p.Ncols + BN - 1) / BN);
  dim3 grid(tiles, 1, splits);
  tc_conv_kernel<BN, STAGES, PRECISE, TMA, BM, KW><<<grid, 160, L::kTotal, st>>>(p, ta, tb, tc);
  count_launch();
  return cudaGetLastError();
}

template <int BN, int BM, int STAGES, bool WG = false>
cudaError_t launch_persist(const ConvParams& p, const CUtensorMap& ta, const CUtensorMap& tb, const CUtensorMap& tc,
                           cudaStream_t st) {
  using L = PersistSmem<BN, BM, STAGES, WG ? 4 : 2>;
  static bool attr_set = false;
  if (!attr_set) {
    cudaError_t e = cudaFuncSetAttribute(tc_conv_persist_kernel<BN, BM, STAGES, WG>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, L::kTotal);
    if (e != cudaSuccess) return e;
    attr_set = true;
  }
  const int tiles = ((p.M + BM - 1) / BM) * ((p.Ncols + BN - 1) / BN);
  tc_conv_persist_kernel<BN, BM, STAGES, WG><<<std::min(tiles, persist_sms()), 192, L::kTotal, st>>>(p, ta, tb, tc);
  count_launch();
  return cudaGetLastError();
}

// Persistent kernel selection. Measured (VGG-16 b256 shapes) against the
// one-tile-per-CTA tall/wide kernels: fprop with 128 output columns +8..11%
// (L2-bound at ~43 FLOP/B either way; the persistent ring removes per-tile
// fills), 64 columns +2%, dgrad 64 columns -16%, >= 256 columns -4..-10%
// (its BN=256 tile is BM=128 to keep two TMEM accumulator sets).
// VDNN_PERSIST=0 disables, =2 forces it for every fprop/dgrad.
bool use_persist(const ConvParams& p) {
  static const int mode = [] {
    const char* e = std::getenv("VDNN_PERSIST");
    return e ? std::atoi(e) : 1;
  }();
  if (mode == 0) return false;
  if (mode == 2) return true;
  return p.kind == kFprop && p.Ncols > 64 && p.Ncols <= 128;
}

// Persistent WGRAD (tc_conv_persist.cuh, WG) for short reductions: at most
// 32 K blocks (FC layers: K = batch) over at least two waves of 256 x 128
// tiles. VDNN_PERSIST_WGRAD=0 disables.
bool persist_wgrad(const ConvParams& p) {
  static const bool on = [] {
    const char* e = std::getenv("VDNN_PERSIST_WGRAD");
    return !e || std::atoi(e) != 0;
  }();
  if (!on || g_precise || g_no_tma || p.Ncols < 128 || p.kblocks > 32) return false;
  const int64_t tiles = static_cast<int64_t>((p.M + 255) / 256) * ((p.Ncols + 127) / 128);
  return tiles >= 2 * kNumSms;
}

// Halo-reuse kernel (tc_conv_halo.cuh) for stride-1 k x k (k >= 3) FPROP /
// DGRAD over one NHWC tensor with 32-multiple channels, when the padded input
// row fits a TMA box (<= 256 pixels) and >= 75% of the 256 virtual rows of a
// tile are real outputs. VDNN_HALO=0 disables.
bool halo_enabled() {
  static const bool on = [] {
    const char* e = std::getenv("VDNN_HALO");
    return !e || std::atoi(e) != 0;
  }();
  return on;
}

bool halo_params(const ConvParams& p, HaloParams& h) {
  if (!halo_enabled() || (p.kind != kFprop && p.kind != kDgrad)) return false;
  if (p.nseg != 1 || !p.vec_in || p.stride != 1 || p.kh != p.kw || p.kh < 3) return false;
  if (p.C % 32 != 0 || p.Cout % 32 != 0) return false;
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
  // Where it wins (measured, VGG-16 b256 shapes): <= 128 output columns over
  // >= 128 input channels, or 64 output columns (224x224x64 fprop/dgrad
  // 356 -> 416 TFLOP/s, 112x112x128 599 -> 627, 112x112 dgrad 128 -> 64
  // 243 -> 344). With 256+ columns the im2col BN=256 tiles are faster: the
  // tensor core's shared-memory operand reads (64 wavefronts per
  // M128xN128xK8, measured 87% busy) bound N=128 tiles, and N=256 MMAs read A
  // once per 256 columns.
  if (h.Cout > 128 || (h.Cout > 64 && h.Cin < 128)) return false;
  h.accum = p.epi == kEpiAccum;
  static const int epi_t = [] {  // VDNN_HALO_EPI_T=0: lanes store their rows directly (A/B switch)
    const char* e = std::getenv("VDNN_HALO_EPI_T");
    return !e || std::atoi(e) != 0 ? 1 : 0;
  }();
  h.epi_t = epi_t;
  h.P = h.Win + 2 * h.pad;
  if (h.P > 256 || h.Wout + h.kw - 1 != h.P) return false;
  h.TH = 256 / h.P;
  if (4 * h.TH * h.Wout < 3 * 256) return false;
  h.nck = h.Cin / 32;
  h.tiles_h = (h.Hout + h.TH - 1) / h.TH;
  return true;
}

template <int BN, int AS, int BS, int KW>
cudaError_t launch_halo(HaloParams& h, const ConvParams& p, cudaStream_t st) {
  using L = HaloSmem<BN, AS, BS>;
  alignas(64) CUtensorMap ta, tb;
  std::memset(&ta, 0, sizeof(ta));
  std::memset(&tb, 0, sizeof(tb));
  const float* src = p.kind == kFprop ? p.seg[0].x : p.dy;
  {
    const cuuint64_t dims[4] = {static_cast<cuuint64_t>(h.Cin), static_cast<cuuint64_t>(h.Win),
                                static_cast<cuuint64_t>(h.Hin), static_cast<cuuint64_t>(h.N)};
    const cuuint64_t strides[3] = {static_cast<cuuint64_t>(h.Cin) * 4, static_cast<cuuint64_t>(h.Win) * h.Cin * 4,
                                   static_cast<cuuint64_t>(h.Hin) * h.Win * h.Cin * 4};
    const cuuint32_t box[4] = {32, static_cast<cuuint32_t>(h.P), static_cast<cuuint32_t>(h.TH), 1};
    if (!encode_tiled(&ta, src, 4, dims, strides, box, CU_TENSOR_MAP_SWIZZLE_128B)) return cudaErrorNotSupported;
  }
  if (p.kind == kFprop) {
    const cuuint64_t dims[2] = {static_cast<cuuint64_t>(p.KK), static_cast<cuuint64_t>(p.Cout)};
    const cuuint64_t strides[1] = {static_cast<cuuint64_t>(p.KK) * 4};
    const cuuint32_t box[2] = {32, static_cast<cuuint32_t>(BN)};
    if (!encode_tiled(&tb, p.w, 2, dims, strides, box, CU_TENSOR_MAP_SWIZZLE_128B)) return cudaErrorNotSupported;
  } else {
    const int taps = p.kh * p.kw;
    const cuuint64_t d4[4] = {32, static_cast<cuuint64_t>(p.Cout), static_cast<cuuint64_t>(p.C / 32),
                              static_cast<cuuint64_t>(taps)};
    const cuuint64_t s4[3] = {static_cast<cuuint64_t>(taps) * p.C * 4, 128, static_cast<cuuint64_t>(p.C) * 4};
    const cuuint32_t b4[4] = {32, 32, static_cast<cuuint32_t>(BN / 32), 1};
    if (!encode_tiled(&tb, p.w, 4, d4, s4, b4, CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B)) return cudaErrorNotSupported;
  }
  h.ntn = (h.Cout + BN - 1) / BN;
  h.ntiles = h.N * h.tiles_h * h.ntn;
  static bool attr_set = false;
  if (!attr_set) {
    cudaError_t e = cudaFuncSetAttribute(tc_conv_halo_kernel<BN, AS, BS, KW>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         L::kTotal);
    if (e != cudaSuccess) return e;
    attr_set = true;
  }
  tc_conv_halo_kernel<BN, AS, BS, KW><<<std::min(h.ntiles, persist_sms()), 192, L::kTotal, st>>>(h, ta, tb);
  count_launch();
  return cudaGetLastError();
}

// Halo kernel on a CTA pair (tc_conv_halo_pair.cuh): same maps, B boxes of
// BN/2 rows per CTA. VDNN_HALO_PAIR=0 selects the single-CTA halo kernel.
bool halo_pair_enabled() {
  static const bool on = [] {
    const char* e = std::getenv("VDNN_HALO_PAIR");
    return !e || std::atoi(e) != 0;
  }();
  return on;
}

template <int BN, int AS, int BS, int KW, bool RESB = false>
cudaError_t launch_halo_pair(HaloParams& h, const ConvParams& p, cudaStream_t st) {
  using L = HaloPairSmem<BN, AS, BS>;
  const int smem = RESB ? L::total(h.nck * h.kh * KW) : L::kTotal;
  if (smem > 227 * 1024 || (RESB && h.Cout != BN)) return cudaErrorNotSupported;
  alignas(64) CUtensorMap ta, tb;
  std::memset(&ta, 0, sizeof(ta));
  std::memset(&tb, 0, sizeof(tb));
  const float* src = p.kind == kFprop ? p.seg[0].x : p.dy;
  {
    const cuuint64_t dims[4] = {static_cast<cuuint64_t>(h.Cin), static_cast<cuuint64_t>(h.Win),
                                static_cast<cuuint64_t>(h.Hin), static_cast<cuuint64_t>(h.N)};
    const cuuint64_t strides[3] = {static_cast<cuuint64_t>(h.Cin) * 4, static_cast<cuuint64_t>(h.Win) * h.Cin * 4,
                                   static_cast<cuuint64_t>(h.Hin) * h.Win * h.Cin * 4};
    const cuuint32_t box[4] = {32, static_cast<cuuint32_t>(h.P), static_cast<cuuint32_t>(h.TH), 1};
    if (!encode_tiled(&ta, src, 4, dims, strides, box, CU_TENSOR_MAP_SWIZZLE_128B)) return cudaErrorNotSupported;
  }
  if (p.kind == kFprop) {
    const cuuint64_t dims[2] = {static_cast<cuuint64_t>(p.KK), static_cast<cuuint64_t>(p.Cout)};
    const cuuint64_t strides[1] = {static_cast<cuuint64_t>(p.KK) * 4};
    const cuuint32_t box[2] = {32, static_cast<cuuint32_t>(BN / 2)};
    if (!encode_tiled(&tb, p.w, 2, dims, strides, box, CU_TENSOR_MAP_SWIZZLE_128B)) return cudaErrorNotSupported;
  } else {
    const int taps = p.kh * p.kw;
    const cuuint64_t d4[4] = {32, static_cast<cuuint64_t>(p.Cout), static_cast<cuuint64_t>(p.C / 32),
                              static_cast<cuuint64_t>(taps)};
    const cuuint64_t s4[3] = {static_cast<cuuint64_t>(taps) * p.C * 4, 128, static_cast<cuuint64_t>(p.C) * 4};
    const cuuint32_t b4[4] = {32, 32, static_cast<cuuint32_t>(BN / 64), 1};
    if (!encode_tiled(&tb, p.w, 4, d4, s4, b4, CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B)) return cudaErrorNotSupported;
  }
  if (h.Cout % BN != 0) return cudaErrorNotSupported;  // each CTA stages BN/2 whole B rows
  h.ntn = h.Cout / BN;
  const int ntiles = h.N * ((h.tiles_h + 1) / 2) * h.ntn;
  h.ntiles = ntiles;
  static int attr_smem = 0;
  if (smem > attr_smem) {
    cudaError_t e = cudaFuncSetAttribute(tc_conv_halo_pair_kernel<BN, AS, BS, KW, RESB>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (e != cudaSuccess) return e;
    attr_smem = smem;
  }
  const int grid = 2 * std::min(ntiles, persist_sms() / 2);
  tc_conv_halo_pair_kernel<BN, AS, BS, KW, RESB><<<grid, kHaloPairThreads, smem, st>>>(h, ta, tb);
  count_launch();
  return cudaGetLastError();
}

// CTA-pair kernel (tc_conv_pair.cuh) for FPROP / DGRAD with >= 256 output
// columns and at least two tiles of 256 x 256 per pair. VDNN_PAIR=0 disables.
// 64-column wgrad: 4-stage rings (2 CTAs / SM still fit) -- the short
// per-stage MMA work (4 x M128N64K8) leaves 3-stage rings latency-bound
bool wgrad_deep64() {
  static const bool on = [] {
    const char* e = std::getenv("VDNN_WGRAD_DEEP64");
    return !e || std::atoi(e) != 0;
  }();
  return on;
}

bool pair_enabled() {
  static const bool on = [] {
    const char* e = std::getenv("VDNN_PAIR");
    return !e || std::atoi(e) != 0;
  }();
  return on;
}

template <int STAGES, int KB, int NOUT = 2>
cudaError_t launch_pair(ConvParams& p, cudaStream_t st) {
  using L = PairSmem<STAGES, KB, NOUT>;
  alignas(64) CUtensorMap ta, tb, tc;
  std::memset(&ta, 0, sizeof(ta));
  std::memset(&tb, 0, sizeof(tb));
  std::memset(&tc, 0, sizeof(tc));
  // per-CTA halves: 128 A rows, 128 B rows (fprop) / 4 MN chunks (dgrad)
  if (!make_maps<128>(p, &ta, &tb, &tc)) return cudaErrorNotSupported;
  if (p.kind == kDgrad && !p.tma_b_merged) return cudaErrorNotSupported;
  static bool attr_set = false;
  if (!attr_set) {
    cudaError_t e =
        cudaFuncSetAttribute(tc_conv_pair_kernel<STAGES, KB, NOUT>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             L::kTotal);
    if (e != cudaSuccess) return e;
    attr_set = true;
  }
  const int tiles = ((p.M + 255) / 256) * ((p.Ncols + 255) / 256);
  const int grid = 2 * std::min(tiles, persist_sms() / 2);
  tc_conv_pair_kernel<STAGES, KB, NOUT><<<grid, 192, L::kTotal, st>>>(p, ta, tb, tc);
  count_launch();
  return cudaGetLastError();
}

template <int STAGES, int KW, int PN>
cudaError_t launch_wgrad_pair(ConvParams& p, int splits, cudaStream_t st) {
  using L = WgradPairSmem<STAGES, KW, PN>;
  alignas(64) CUtensorMap ta, tb, tc;
  std::memset(&ta, 0, sizeof(ta));
  std::memset(&tb, 0, sizeof(tb));
  std::memset(&tc, 0, sizeof(tc));
  if (!make_maps<PN / 2, KW>(p, &ta, &tb, &tc)) return cudaErrorNotSupported;
  static bool attr_set = false;
  if (!attr_set) {
    cudaError_t e = cudaFuncSetAttribute(tc_wgrad_pair_kernel<STAGES, KW, PN>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, L::kTotal);
    if (e != cudaSuccess) return e;
    attr_set = true;
  }
  const int work = ((p.M + 255) / 256) * ((p.Ncols + PN - 1) / PN) * splits;
  const int grid = 2 * std::min(work, persist_sms() / 2);
  tc_wgrad_pair_kernel<STAGES, KW, PN><<<grid, 192, L::kTotal, st>>>(p, ta, tb, splits);
  count_launch();
  return cudaGetLastError();
}

cudaError_t launch(ConvParams& p, int splits, cudaStream_t st) {
  if (p.M <= 0 || p.Ncols <= 0) return cudaSuccess;
  if (p.kind == kWgrad && p.use_pair && !g_precise && !g_no_tma) {
    cudaError_t e = cudaErrorNotSupported;
    if (p.Ncols >= 256)
      e = p.wkw == 64 ? launch_wgrad_pair<3, 64, 256>(p, splits, st) : launch_wgrad_pair<6, kBK, 256>(p, splits, st);
    else if (p.Ncols >= 128)
      e = launch_wgrad_pair<4, 64, 128>(p, splits, st);
    else
      e = launch_wgrad_pair<5, 64, 64>(p, splits, st);
    if (e != cudaErrorNotSupported) return e;
    p.tma_b_merged = 0;
  }
  if (!g_precise && !g_no_tma && splits == 1 && pair_enabled() && (p.kind == kFprop || p.kind == kDgrad) &&
      p.epi != kEpiPartial && p.Ncols >= 256 && p.Ncols % 128 == 0 &&
      static_cast<int64_t>((p.M + 255) / 256) * (p.Ncols / 256) >= kNumSms) {
    static const int stages = [] {
      const char* e = std::getenv("VDNN_PAIR_STAGES");
      return e ? std::atoi(e) : 5;
    }();
    cudaError_t e;
    if (stages == 3 && p.kblocks % 2 == 0)
      e = launch_pair<3, 2>(p, st);  // 64-channel (2 k-block) stages
    else if (stages == 6)
      e = launch_pair<6, 1>(p, st);
    else  // default: 5 stages, four TMA-store staging boxes (3 stores in flight: the 56x56x256
          // tiles' epilogue is as long as their 72-k-block main loop; measured -6% there)
      e = launch_pair<5, 1, 4>(p, st);
    if (e != cudaErrorNotSupported) return e;
    p.tma_b_merged = 0;
  }
  if (!g_precise && !g_no_tma && splits == 1) {
    HaloParams h;
    if (halo_params(p, h)) {
      cudaError_t e = cudaErrorNotSupported;
      static const bool resb = [] {
        const char* e = std::getenv("VDNN_HALO_RESB");
        return !e || std::atoi(e) != 0;
      }();
      if (h.kw == 3 && halo_pair_enabled() && resb && h.Cout == 64)  // filter half resident (<= 2 chunks)
        e = launch_halo_pair<64, 4, 1, 3, true>(h, p, st);
      if (e == cudaErrorNotSupported && h.kw == 3 && halo_pair_enabled())
        e = h.Cout <= 64 ? launch_halo_pair<64, 5, 8, 3>(h, p, st) : launch_halo_pair<128, 4, 7, 3>(h, p, st);
      if (e != cudaErrorNotSupported) return e;
      if (h.kw == 3)
        e = p.Ncols <= 64 ? launch_halo<64, 4, 8, 3>(h, p, st) : launch_halo<128, 3, 7, 3>(h, p, st);
      else if (h.kw == 5)
        e = p.Ncols <= 64 ? launch_halo<64, 4, 8, 5>(h, p, st) : launch_halo<128, 3, 7, 5>(h, p, st);
      if (e != cudaErrorNotSupported) return e;
    }
  }
  alignas(64) CUtensorMap ta, tb, tc;
  std::memset(&ta, 0, sizeof(ta));
  std::memset(&tb, 0, sizeof(tb));
  std::memset(&tc, 0, sizeof(tc));
  if (g_precise) {
    // TMA producer + split warps (the lo tiles computed from the landed hi
    // tiles); the cp.async gathers when the maps do not apply
    static const bool tma_precise = [] {
      const char* e = std::getenv("VDNN_PRECISE_TMA");
      return !e || std::atoi(e) != 0;
    }();
    if (tma_precise && !g_no_tma && (p.kind != kWgrad || p.wkw == kBK)) {
      if (p.Ncols <= 64 && make_maps<64>(p, &ta, &tb, &tc))
        return launch_bn<64, kStagesPrecise, true, true>(p, ta, tb, tc, splits, st);
      if (p.Ncols > 64 && make_maps<128>(p, &ta, &tb, &tc))
        return launch_bn<128, kStagesPrecise, true, true>(p, ta, tb, tc, splits, st);
    }
    if (p.Ncols <= 64) return launch_bn<64, kStagesPrecise, true, false>(p, ta, tb, tc, splits, st);
    return launch_bn<128, kStagesPrecise, true, false>(p, ta, tb, tc, splits, st);
  }
  if ((p.kind == kFprop || p.kind == kDgrad) && p.epi == kEpiPartial) {
    // split-K fprop (FC layers: few output tiles, long K): BN=128 TMA tiles,
    // partial slabs through the 3-D output map
    if (make_maps<128>(p, &ta, &tb, &tc)) return launch_bn<128, kStages, false, true>(p, ta, tb, tc, splits, st);
    return cudaErrorNotSupported;
  }
  if (p.kind == kWgrad && p.wkw == 64) {
    // 64-pixel stages: half the im2col TMA ops per FLOP (their issue rate,
    // not bytes, bounds the 32-pixel wgrad pipeline); one CTA per SM
    if (p.Ncols > 128 && make_maps<256, 64>(p, &ta, &tb, &tc))
      return launch_bn<256, 2, false, true, kBM, 64>(p, ta, tb, tc, splits, st);
    if (p.Ncols > 64 && p.Ncols <= 128 && make_maps<128, 64>(p, &ta, &tb, &tc))
      return launch_bn<128, 3, false, true, kBM, 64>(p, ta, tb, tc, splits, st);
    if (p.Ncols <= 64 && make_maps<64, 64>(p, &ta, &tb, &tc))
      return launch_bn<64, 4, false, true, kBM, 64>(p, ta, tb, tc, splits, st);
    // maps failed: fall back to 32-pixel K blocks
    p.wkw = kBK;
    p.kblocks *= 2;
    p.kb_per_split *= 2;
  }
  if (p.kind == kWgrad && splits == 1 && persist_wgrad(p) && p.wkw == kBK && p.epi != kEpiPartial) {
    // short-reduction wgrad (FC layers): persistent, SGD epilogue overlapped;
    // for FC layers the SGD goes through TMA boxes of W (tma_c)
    if (make_maps<128>(p, &ta, &tb, &tc)) {
      p.sgd_tma = 0;
      static const bool sgd_tma = [] {
        const char* e = std::getenv("VDNN_SGD_TMA");
        return !e || std::atoi(e) != 0;
      }();
      if (sgd_tma && p.epi == kEpiSgd && p.kh == 1 && p.kw == 1 && p.H == 1 && p.W == 1 && p.nseg == 1 &&
          p.C % 32 == 0 && p.KK % 4 == 0) {
        const cuuint64_t dims[2] = {static_cast<cuuint64_t>(p.KK), static_cast<cuuint64_t>(p.Cout)};
        const cuuint64_t strides[1] = {static_cast<cuuint64_t>(p.KK) * 4};
        const cuuint32_t box[2] = {128, 32};
        if (encode_tiled(&tc, p.w_mut, 2, dims, strides, box, CU_TENSOR_MAP_SWIZZLE_NONE)) p.sgd_tma = 1;
      }
      return launch_persist<128, 256, 3, true>(p, ta, tb, tc, st);
    }
    std::memset(&ta, 0, sizeof(ta));
    std::memset(&tb, 0, sizeof(tb));
    std::memset(&tc, 0, sizeof(tc));
    p.tma_b_merged = 0;
  }
  if (p.kind != kWgrad && splits == 1 && use_persist(p) && !g_no_tma) {
    if (p.Ncols <= 64) {
      if (make_maps<64>(p, &ta, &tb, &tc)) return launch_persist<64, 256, 4>(p, ta, tb, tc, st);
    } else if (p.Ncols <= 128) {
      if (make_maps<128>(p, &ta, &tb, &tc)) return launch_persist<128, 256, 4>(p, ta, tb, tc, st);
    } else if (make_maps<256>(p, &ta, &tb, &tc)) {
      return launch_persist<256, 128, 4>(p, ta, tb, tc, st);
    }
    std::memset(&ta, 0, sizeof(ta));
    std::memset(&tb, 0, sizeof(tb));
    std::memset(&tc, 0, sizeof(tc));
    p.tma_b_merged = 0;
  }
  const bool deep = tall_deep();
  if (p.Ncols <= 64) {
    if (!g_no_tma && make_maps<64>(p, &ta, &tb, &tc)) {
      if (tall_ok(p, 64, splits))
        return deep ? launch_bn<64, 5, false, true, 256>(p, ta, tb, tc, splits, st)
                    : launch_bn<64, 2, false, true, 256>(p, ta, tb, tc, splits, st);
      if (p.kind == kWgrad && wgrad_deep64()) return launch_bn<64, 4, false, true>(p, ta, tb, tc, splits, st);
      return launch_bn<64, kStages, false, true>(p, ta, tb, tc, splits, st);
    }
    return launch_bn<64, kStages, false, false>(p, ta, tb, tc, splits, st);
  }
  if (wide_ok(p) && !g_no_tma && make_maps<256>(p, &ta, &tb, &tc)) {
    if (tall_ok(p, 256, splits)) return launch_bn<256, 3, false, true, 256>(p, ta, tb, tc, splits, st);
    return launch_bn<256, kStagesWide, false, true>(p, ta, tb, tc, splits, st);
  }
  if (!g_no_tma && make_maps<128>(p, &ta, &tb, &tc)) {
    if (tall_ok(p, 128, splits))
      return deep ? launch_bn<128, 4, false, true, 256>(p, ta, tb, tc, splits, st)
                  : launch_bn<128, 2, false, true, 256>(p, ta, tb, tc, splits, st);
    return launch_bn<128, kStages, false, true>(p, ta, tb, tc, splits, st);
  }
  return launch_bn<128, kStages, false, false>(p, ta, tb, tc, splits, st);
}

bool wgrad_wide_k() {
  static const bool on = [] {
    const char* e = std::getenv("VDNN_WGRAD_KW");
    return e && std::atoi(e) == 64;
  }();
  return on;
}

// Tile shape and resident CTAs the wgrad launch will use (mirrors launch()).
struct WCfg {
  int bn, bm, slots, kw;
  bool pair;
};
// Tall wgrad tiles pay off only with wide (BN=256) tiles over many pixels
// (measured: +37% at 56x56x256, neutral at 28x28x512, -5..-20% at 14x14 or
// with 64/128-wide tiles, where the extra im2col boxes per stage dominate).
int wgrad_rows(const ConvParams& p) { return p.vec_in ? p.kh * p.kw * p.nchunk * 32 : p.KK; }

WCfg wgrad_cfg(const ConvParams& p, int64_t pixels) {
  WCfg c;
  const int ncols = p.Cout;
  const bool tma = !g_precise && !g_no_tma && p.nseg == 1 && p.vec_in && p.vec_out && p.kh == p.kw;
  // A short reduction (FC layers: K = batch) makes every tile mostly
  // epilogue (the SGD read-modify-write of its weights); BN=128 tiles run two
  // CTAs per SM so one CTA's epilogue overlaps the other's loads and MMAs.
  c.bn = (ncols >= 256 && use_wide(kWgrad) && tma && pixels >= 2048) ? 256 : (ncols <= 64 ? 64 : 128);
  c.bm = (tma && ((tall_mask() >> kWgrad) & 1) && c.bn == 256 && pixels >= 100000) ? 256 : kBM;
  const bool one_per_sm = c.bn > 128 || (c.bm > kBM && tall_deep());
  c.slots = one_per_sm ? kNumSms : 2 * kNumSms;
  c.kw = kBK;
  c.pair = false;
  // CTA pair (M = 256 weight rows x N = 256 output channels per pair)
  static const int pair_min = [] {  // narrowest layer that takes the pair wgrad (VDNN_PAIR_WGRAD_MIN)
    const char* e = std::getenv("VDNN_PAIR_WGRAD_MIN");
    return e ? std::atoi(e) : 256;
  }();
  if (tma && pair_enabled() && ncols >= pair_min && pixels >= 2048 && wgrad_rows(p) >= 256) {
    c.pair = true;
    c.bn = ncols >= 256 ? 256 : (ncols >= 128 ? 128 : 64);
    c.bm = 256;
    c.slots = kNumSms / 2;
    static const int kw = [] {
      const char* e = std::getenv("VDNN_PAIR_WGRAD_KW");
      return e ? std::atoi(e) : 64;
    }();
    c.kw = (kw == 32 && c.bn == 256) ? kBK : 64;
    return c;
  }
  // 64-pixel stages (opt-in, VDNN_WGRAD_KW=64): they halve the im2col boxes
  // per FLOP, which paid +18..42% while the producer thread recomputed every
  // box coordinate with integer divisions; with the incremental producer the
  // 32-pixel ring with two CTAs per SM is as fast or faster (56x56x256: 714 vs
  // 527 TFLOP/s)
  if (tma && c.bn == 256 && wgrad_wide_k()) {
    c.kw = 64;
    c.bm = kBM;
    c.slots = kNumSms;
  }
  return c;
}


// Split-K factor for WGRAD from a small time model: the main loop runs in
// ceil(tiles*s / slots) waves of ceil(kblocks/s) K blocks (~4*BN cycles each
// at the observed tensor-pipe duty), and every split adds a partial tile
// written and re-read by the reduce (8 B per output element at HBM speed).
int pick_splits(int tiles, int kblocks, int slots, int work, int64_t outputs) {
  int best = 1;
  double best_t = 1e30;
  const int smax = std::max(1, std::min(1024, kblocks / 4));
  for (int s = 1; s <= smax; ++s) {
    const double waves = static_cast<double>((static_cast<int64_t>(tiles) * s + slots - 1) / slots);
    const double kbps = static_cast<double>((kblocks + s - 1) / s);
    const double t_main = waves * kbps * 4.0 * work / 1.9e9;
    const double t_part = s > 1 ? static_cast<double>(s) * static_cast<double>(outputs) * 8.0 / 5e12 : 0.0;
    const double t = t_main + t_part;
    if (t < best_t * (1 - 1e-6)) {
      best_t = t;
      best = s;
    }
  }
  return best;
}

}  // namespace

uint64_t launch_count() { return g_launches.load(); }
void set_precise(bool on) { g_precise = on; }
void set_tma(bool on) { g_no_tma = !on; }
bool precise() { return g_precise; }
void count_launch(uint64_t k) { g_launches.fetch_add(k); }

namespace {
bool fprop_params(const ConvArgs& a, const float* w, const float* bias, float* y, bool accumulate, ConvParams& p) {
  if (!build_common(a, p)) return false;
  p.kind = kFprop;
  p.relu = a.relu_out;
  p.epi = accumulate ? kEpiAccum : kEpiStore;
  p.w = w;
  p.bias = bias;
  p.y = y;
  p.M = a.n * p.Ho * p.Wo;
  p.Ncols = a.cout;
  p.kblocks = p.vec_in ? a.kh * a.kw * p.nchunk : (p.KK + kBK - 1) / kBK;
  p.kb_per_split = p.kblocks;
  return true;
}

// Split-K factor for FPROP: only when the output has fewer BN=128 tiles than
// SMs (FC layers at small batch: FC6 of VGG-16 b256 is 2 x 32 tiles over a
// 25,088-long reduction) and the operands take the TMA path. Same time model
// as WGRAD, two CTAs per SM.
int fprop_splits(const ConvParams& p) {
  if (g_precise || g_no_tma || p.epi != kEpiStore || p.nseg != 1 || !p.vec_in || !p.vec_out || p.kh != p.kw)
    return 1;
  const int tiles = ((p.M + kBM - 1) / kBM) * ((p.Ncols + 127) / 128);
  if (tiles >= kNumSms || p.kblocks < 64) return 1;
  return pick_splits(tiles, p.kblocks, 2 * kNumSms, 128, static_cast<int64_t>(p.M) * p.Cout);
}

__global__ void fprop_reduce_kernel(const float* __restrict__ part, int splits, int64_t m, int cout,
                                    const float* __restrict__ bias, int relu, float* __restrict__ y) {
  const int64_t total4 = m * cout / 4;
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < total4;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    float4 s = reinterpret_cast<const float4*>(part)[i];
    for (int z = 1; z < splits; ++z) {  // fixed order: deterministic
      const float4 q = reinterpret_cast<const float4*>(part + z * m * cout)[i];
      s.x += q.x;
      s.y += q.y;
      s.z += q.z;
      s.w += q.w;
    }
    if (bias) {
      const int o = static_cast<int>((i * 4) % cout);
      s.x += bias[o];
      s.y += bias[o + 1];
      s.z += bias[o + 2];
      s.w += bias[o + 3];
    }
    if (relu) {
      s.x = fmaxf(s.x, 0.f);
      s.y = fmaxf(s.y, 0.f);
      s.z = fmaxf(s.z, 0.f);
      s.w = fmaxf(s.w, 0.f);
    }
    reinterpret_cast<float4*>(y)[i] = s;
  }
}
}  // namespace

size_t conv_fprop_ws_bytes(const ConvArgs& a) {
  if (c3tc_fprop_eligible(a) || smallc_eligible(a)) return 0;
  ConvParams p;
  if (!fprop_params(a, nullptr, nullptr, nullptr, false, p)) return 0;
  const int s = fprop_splits(p);
  return s > 1 ? static_cast<size_t>(s) * p.M * p.Cout * sizeof(float) : 0;
}

cudaError_t conv_fprop(const ConvArgs& a, const float* w, const float* bias, float* y, bool accumulate,
                       cudaStream_t st, float* ws, size_t ws_bytes) {
  if (!accumulate && bias == nullptr && c3tc_fprop_eligible(a)) return c3tc_fprop(a, w, y, st);
  // SIMT first layer only in the exact-fp32 mode: in TF32 mode the windows
  // c3tc does not take (AlexNet / OverFeat 11x11x3, K = 363) run on the
  // tensor-core engine with cp.async gathers (measured 8.8 TFLOP/s SIMT)
  if (!accumulate && bias == nullptr && smallc_eligible(a) && g_precise) return smallc_fprop(a, w, y, st);
  ConvParams p;
  if (!fprop_params(a, w, bias, y, accumulate, p)) return cudaErrorInvalidValue;
  int splits = ws ? fprop_splits(p) : 1;
  const size_t per = static_cast<size_t>(p.M) * p.Cout * sizeof(float);
  if (splits > 1) splits = static_cast<int>(std::min<size_t>(splits, ws_bytes / per));
  if (splits > 1) {
    p.kb_per_split = (p.kblocks + splits - 1) / splits;
    splits = (p.kblocks + p.kb_per_split - 1) / p.kb_per_split;
  }
  if (splits <= 1) {
    p.kb_per_split = p.kblocks;
    return launch(p, 1, st);
  }
  p.epi = kEpiPartial;
  p.out = ws;
  p.splits = splits;
  cudaError_t e = launch(p, splits, st);
  if (e != cudaSuccess) return e;
  const int64_t total4 = static_cast<int64_t>(p.M) * p.Cout / 4;
  const int blocks = static_cast<int>(std::min<int64_t>((total4 + 255) / 256, 4 * kNumSms));
  fprop_reduce_kernel<<<blocks, 256, 0, st>>>(ws, splits, p.M, p.Cout, bias, p.relu, y);
  count_launch();
  return cudaGetLastError();
}

namespace {
bool dgrad_params(const ConvArgs& a, const float* w, const float* dy, bool accumulate, ConvParams& p) {
  if (!build_common(a, p)) return false;
  p.kind = kDgrad;
  p.epi = accumulate ? kEpiAccum : kEpiStore;
  p.w = w;
  p.dy = dy;
  p.M = a.n * a.h * a.w;
  p.Ncols = p.vec_in ? p.nchunk * 32 : p.C;
  p.kblocks = p.vec_out ? a.kh * a.kw * ((a.cout + 31) / 32) : (a.kh * a.kw * a.cout + kBK - 1) / kBK;
  p.kb_per_split = p.kblocks;
  return true;
}

// Split-K for DGRAD of FC layers (1x1 over a 1x1 image) with fewer BN=128
// output tiles than SMs: AlexNet FC6 dX is 128 x 9,216 = 72 tiles over a
// 4,096-long reduction. Partials + ordered reduce (mask, accumulation).
int dgrad_splits(const ConvParams& p) {
  if (g_precise || g_no_tma || p.nseg != 1 || !p.vec_in || !p.vec_out || p.kh != 1 || p.kw != 1 || p.H != 1 ||
      p.W != 1 || p.C % 32 != 0)
    return 1;
  static const bool off = std::getenv("VDNN_NO_DGRAD_SPLIT") != nullptr;  // A/B switch
  const int tiles = ((p.M + kBM - 1) / kBM) * ((p.Ncols + 127) / 128);
  if (off || tiles >= kNumSms || p.kblocks < 64) return 1;
  return pick_splits(tiles, p.kblocks, 2 * kNumSms, 128, static_cast<int64_t>(p.M) * p.C);
}

__global__ void dgrad_reduce_kernel(const float* __restrict__ part, int splits, int64_t m, int c,
                                    const float* __restrict__ mask_x, int accumulate, float* __restrict__ dx) {
  const int64_t total4 = m * c / 4;
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < total4;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    float4 s = reinterpret_cast<const float4*>(part)[i];
    for (int z = 1; z < splits; ++z) {  // fixed order: deterministic
      const float4 q = reinterpret_cast<const float4*>(part + z * m * c)[i];
      s.x += q.x;
      s.y += q.y;
      s.z += q.z;
      s.w += q.w;
    }
    if (mask_x) {
      const float4 xv = reinterpret_cast<const float4*>(mask_x)[i];
      s.x = xv.x > 0.f ? s.x : 0.f;
      s.y = xv.y > 0.f ? s.y : 0.f;
      s.z = xv.z > 0.f ? s.z : 0.f;
      s.w = xv.w > 0.f ? s.w : 0.f;
    }
    if (accumulate) {
      const float4 o = reinterpret_cast<const float4*>(dx)[i];
      s.x += o.x;
      s.y += o.y;
      s.z += o.z;
      s.w += o.w;
    }
    reinterpret_cast<float4*>(dx)[i] = s;
  }
}
}  // namespace

void set_sm_reserve(int sms) { g_sm_reserve = sms; }

size_t conv_dgrad_ws_bytes(const ConvArgs& a) {
  ConvParams p;
  if (a.stride != 1 || !dgrad_params(a, nullptr, nullptr, false, p)) return 0;
  const int s = dgrad_splits(p);
  return s > 1 ? static_cast<size_t>(s) * p.M * p.C * sizeof(float) : 0;
}

cudaError_t conv_dgrad(const ConvArgs& a, const float* w, const float* dy, bool accumulate, cudaStream_t st,
                       float* ws, size_t ws_bytes) {
  ConvParams p;
  if (!dgrad_params(a, w, dy, accumulate, p)) return cudaErrorInvalidValue;
  if (a.stride != 1) return cudaErrorNotSupported;
  int splits = (ws && p.seg[0].dx) ? dgrad_splits(p) : 1;
  const size_t per = static_cast<size_t>(p.M) * p.C * sizeof(float);
  if (splits > 1) splits = static_cast<int>(std::min<size_t>(splits, ws_bytes / per));
  if (splits > 1) {
    p.kb_per_split = (p.kblocks + splits - 1) / splits;
    splits = (p.kblocks + p.kb_per_split - 1) / p.kb_per_split;
  }
  if (splits <= 1) {
    p.kb_per_split = p.kblocks;
    return launch(p, 1, st);
  }
  const bool accum = p.epi == kEpiAccum;
  p.epi = kEpiPartial;
  p.out = ws;
  p.splits = splits;
  cudaError_t e = launch(p, splits, st);
  if (e != cudaSuccess) return e;
  const int64_t total4 = static_cast<int64_t>(p.M) * p.C / 4;
  const int blocks = static_cast<int>(std::min<int64_t>((total4 + 255) / 256, 4 * kNumSms));
  dgrad_reduce_kernel<<<blocks, 256, 0, st>>>(ws, splits, p.M, p.C, p.seg[0].mask ? p.seg[0].x : nullptr,
                                              accum ? 1 : 0, p.seg[0].dx);
  count_launch();
  return cudaGetLastError();
}

namespace {
// Halo WGRAD (tc_conv_halo.cuh) for narrow stride-1 layers: <= 64 output
// channels over 32-multiple input channels, padded row <= 248 pixels.
// VDNN_HALO_WGRAD=0 disables.
bool halo_wgrad_enabled() {
  static const bool on = [] {
    const char* e = std::getenv("VDNN_HALO_WGRAD");
    return !e || std::atoi(e) != 0;
  }();
  return on;
}
constexpr size_t kSmemLimit = 227 * 1024;

bool halo_wg_params(const ConvParams& p, HaloWgParams& h, int& bn, size_t& smem) {
  if (!halo_enabled() || !halo_wgrad_enabled() || g_precise || g_no_tma) return false;
  if (p.nseg != 1 || !p.vec_in || p.stride != 1 || p.kh != p.kw || p.kh < 2 || p.kw > 4) return false;
  // measured (best-of-3 A/B): 224x224 64->64 2.83 -> 2.50 ms; with 128 output
  // channels the im2col kernel stays faster (112x112 128->128 1.61 vs 2.03)
  if (p.C % 32 != 0 || p.Cout % 32 != 0 || p.Cout > 64 || p.pad > p.kh - 1) return false;
  std::memset(&h, 0, sizeof(h));
  h.N = p.N, h.H = p.H, h.W = p.W, h.C = p.C, h.Cout = p.Cout, h.kh = p.kh, h.kw = p.kw, h.pad = p.pad;
  h.P = p.W + 2 * p.pad;
  h.Hout = p.Ho, h.Wout = p.Wo;
  if (h.Wout + h.kw - 1 != h.P || h.P > 248) return false;
  h.Kp = (h.P + 7) / 8 * 8;
  h.nck = p.C / 32;
  bn = p.Cout <= 64 ? 64 : 128;
  const int nblk = h.kh * h.nck, gmax = 512 / bn;
  h.ngroups = (nblk + gmax - 1) / gmax;
  h.G = (nblk + h.ngroups - 1) / h.ngroups;
  h.nrows = h.N * h.Hout;
  int splits = std::max(1, kNumSms / h.ngroups);
  // CTA pair (tc_conv_halo_pair.cuh): 64 channels, the blocks split evenly
  // between the two CTAs, one row range per pair
  static const bool pair_wg = [] {
    const char* e = std::getenv("VDNN_HALO_PAIR_WGRAD");
    return !e || std::atoi(e) != 0;
  }();
  h.pair = (pair_wg && halo_pair_enabled() && p.Cout == 64 && nblk % 2 == 0 && nblk / 2 * 64 <= 512) ? 1 : 0;
  if (h.pair) {
    // a fixed item count (4 per pair of a full grid): partials and reduce
    // order do not depend on the grid an SM reserve leaves
    h.ngroups = 1;
    h.G = nblk / 2;
    splits = 4 * (kNumSms / 2);
  }
  h.rows_per = (h.nrows + splits - 1) / splits;
  h.M = p.kh * p.kw * h.nck * 32;
  h.a_slot = halo_wg_a_slot(h.Kp);
  h.b_slot = halo_wg_b_slot(h.Kp, h.pair ? 32 : bn);
  h.BS = 2;
  const size_t fixed = 1024 + 256 + static_cast<size_t>(h.BS) * h.b_slot;
  if (fixed + 2 * static_cast<size_t>(h.a_slot) > kSmemLimit) return false;
  h.AS = static_cast<int>(std::min<size_t>(kHwMaxAS, (kSmemLimit - fixed) / h.a_slot));
  smem = fixed + static_cast<size_t>(h.AS) * h.a_slot;
  return true;
}
int halo_wg_splits(const HaloWgParams& h) { return (h.nrows + h.rows_per - 1) / h.rows_per; }

template <int BN>
cudaError_t launch_halo_wgrad(HaloWgParams& h, size_t smem, const ConvParams& p, cudaStream_t st) {
  alignas(64) CUtensorMap tx, tdy;
  std::memset(&tx, 0, sizeof(tx));
  std::memset(&tdy, 0, sizeof(tdy));
  {
    const cuuint64_t dims[4] = {static_cast<cuuint64_t>(h.C), static_cast<cuuint64_t>(h.W),
                                static_cast<cuuint64_t>(h.H), static_cast<cuuint64_t>(h.N)};
    const cuuint64_t strides[3] = {static_cast<cuuint64_t>(h.C) * 4, static_cast<cuuint64_t>(h.W) * h.C * 4,
                                   static_cast<cuuint64_t>(h.H) * h.W * h.C * 4};
    const cuuint32_t box[4] = {32, static_cast<cuuint32_t>(h.P), 1, 1};
    if (!encode_tiled(&tx, p.seg[0].x, 4, dims, strides, box, CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B))
      return cudaErrorNotSupported;
  }
  {
    const cuuint64_t dims[4] = {static_cast<cuuint64_t>(h.Cout), static_cast<cuuint64_t>(h.Wout),
                                static_cast<cuuint64_t>(h.Hout), static_cast<cuuint64_t>(h.N)};
    const cuuint64_t strides[3] = {static_cast<cuuint64_t>(h.Cout) * 4, static_cast<cuuint64_t>(h.Wout) * h.Cout * 4,
                                   static_cast<cuuint64_t>(h.Hout) * h.Wout * h.Cout * 4};
    const cuuint32_t box[4] = {32, static_cast<cuuint32_t>(h.P), 1, 1};
    if (!encode_tiled(&tdy, p.dy, 4, dims, strides, box, CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B))
      return cudaErrorNotSupported;
  }
  if (h.pair) {
    static bool pattr = false;
    if (!pattr) {
      cudaError_t e = cudaFuncSetAttribute(tc_wgrad_halo_pair_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                           static_cast<int>(kSmemLimit));
      if (e != cudaSuccess) return e;
      pattr = true;
    }
    const int items = halo_wg_splits(h);
    tc_wgrad_halo_pair_kernel<<<2 * std::min(items, persist_sms() / 2), 192, smem, st>>>(h, tx, tdy, items);
    count_launch();
    return cudaGetLastError();
  }
  static size_t attr = 0;
  if (smem > attr) {
    cudaError_t e = cudaFuncSetAttribute(tc_wgrad_halo_kernel<BN>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         static_cast<int>(kSmemLimit));
    if (e != cudaSuccess) return e;
    attr = kSmemLimit;
  }
  const int grid = halo_wg_splits(h) * h.ngroups;
  tc_wgrad_halo_kernel<BN><<<grid, 192, smem, st>>>(h, tx, tdy);
  count_launch();
  return cudaGetLastError();
}
}  // namespace

size_t conv_wgrad_ws_bytes(const ConvArgs& a) {
  if (smallc_eligible(a)) {
    // either kernel may run (the TF32 / exact-fp32 mode can change per call)
    size_t b = smallc_wgrad_ws_bytes(a, nullptr);
    const bool was = g_precise;
    g_precise = false;
    if (c3tc_wgrad_eligible(a)) b = std::max(b, c3tc_wgrad_ws_bytes(a));
    g_precise = was;
    return b;
  }
  const size_t first = 0;
  ConvParams p;
  if (!build_common(a, p)) return first;
  {
    ConvParams q = p;
    q.kind = kWgrad;
    HaloWgParams h;
    int bn;
    size_t smem;
    if (halo_wg_params(q, h, bn, smem))
      return static_cast<size_t>(halo_wg_splits(h)) * h.M * a.cout * sizeof(float);
  }
  const int M = wgrad_rows(p);
  const int64_t P = static_cast<int64_t>(a.n) * p.Ho * p.Wo;
  const WCfg c = wgrad_cfg(p, P);
  const int tiles = ((M + c.bm - 1) / c.bm) * ((a.cout + c.bn - 1) / c.bn);
  const int kblocks = static_cast<int>((P + c.kw - 1) / c.kw);
  const int splits = pick_splits(tiles, kblocks, c.slots, c.bn * c.bm / kBM * c.kw / kBK,
                                 static_cast<int64_t>(M) * a.cout);
  if (splits <= 1) return first;
  return std::max(first, static_cast<size_t>(splits) * M * a.cout * sizeof(float));
}

__global__ void wgrad_reduce_kernel(const __grid_constant__ ConvParams p, int splits) {
  const int64_t total = static_cast<int64_t>(p.Cout) * p.M;
  for (int64_t idx = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; idx < total;
       idx += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int m = static_cast<int>(idx % p.M);
    const int co = static_cast<int>(idx / p.M);
    bool valid;
    const int widx = wgrad_widx(p, m, valid);
    if (!valid) continue;
    float s = 0.f;
    for (int k = 0; k < splits; ++k) s += p.out[static_cast<int64_t>(k) * total + idx];
    if (p.w_mut && p.epi == kEpiSgd)
      p.w_mut[static_cast<int64_t>(co) * p.KK + widx] -= p.lr * s;
    else
      p.y[static_cast<int64_t>(co) * p.KK + widx] = s;  // y aliases dw_out here
  }
}

cudaError_t conv_wgrad(const ConvArgs& a, const float* dy, float* w_mut, float lr, float* dw_out, float* ws,
                       size_t ws_bytes, cudaStream_t st) {
  if (c3tc_wgrad_eligible(a) && ws != nullptr &&
      ws_bytes >= static_cast<size_t>(a.cout) * a.kh * a.kw * a.c[0] * sizeof(float))
    return c3tc_wgrad(a, dy, w_mut, lr, dw_out, ws, ws_bytes, st);
  // first-layer wgrad outside c3tc: the SIMT kernel (smem-resident weights,
  // hoisted window decode) beats the engine's scalar 4-byte gathers there
  // (AlexNet 11x11x3: 1.03 vs 1.71 ms)
  if (smallc_eligible(a) && ws != nullptr &&
      ws_bytes >= static_cast<size_t>(a.cout) * a.kh * a.kw * a.c[0] * sizeof(float))
    return smallc_wgrad(a, dy, w_mut, lr, dw_out, ws, ws_bytes, st);
  ConvParams p;
  if (!build_common(a, p)) return cudaErrorInvalidValue;
  p.kind = kWgrad;
  p.dy = dy;
  p.w = w_mut;
  p.w_mut = w_mut;
  p.lr = lr;
  p.M = wgrad_rows(p);
  p.Ncols = a.cout;
  {
    HaloWgParams h;
    int bn;
    size_t smem;
    if (ws != nullptr && halo_wg_params(p, h, bn, smem) &&
        ws_bytes >= static_cast<size_t>(halo_wg_splits(h)) * h.M * a.cout * sizeof(float)) {
      h.part = ws;
      const cudaError_t e = bn == 64 ? launch_halo_wgrad<64>(h, smem, p, st) : launch_halo_wgrad<128>(h, smem, p, st);
      if (e == cudaSuccess) {
        const int splits = halo_wg_splits(h);
        p.out = ws;
        p.epi = dw_out ? kEpiGrad : kEpiSgd;
        p.y = dw_out;
        if (dw_out) p.w_mut = nullptr;
        const int64_t total = static_cast<int64_t>(p.Cout) * p.M;
        const int blocks = static_cast<int>(std::min<int64_t>((total + 255) / 256, 4 * kNumSms));
        wgrad_reduce_kernel<<<blocks, 256, 0, st>>>(p, splits);
        count_launch();
        return cudaGetLastError();
      }
      if (e != cudaErrorNotSupported) return e;
    }
  }
  const int64_t P = static_cast<int64_t>(a.n) * p.Ho * p.Wo;
  const WCfg c = wgrad_cfg(p, P);
  p.wkw = c.kw;
  p.use_pair = c.pair ? 1 : 0;
  p.kblocks = static_cast<int>((P + c.kw - 1) / c.kw);
  const int tiles = ((p.M + c.bm - 1) / c.bm) * ((a.cout + c.bn - 1) / c.bn);
  int splits = pick_splits(tiles, p.kblocks, c.slots, c.bn * c.bm / kBM * c.kw / kBK,
                           static_cast<int64_t>(p.M) * a.cout);
  const size_t per = static_cast<size_t>(p.M) * a.cout * sizeof(float);
  if (ws == nullptr || per == 0) splits = 1;
  else splits = static_cast<int>(std::min<size_t>(splits, ws_bytes / per));
  if (splits < 1) splits = 1;
  p.kb_per_split = (p.kblocks + splits - 1) / splits;
  splits = (p.kblocks + p.kb_per_split - 1) / p.kb_per_split;
  if (splits <= 1) {
    p.epi = dw_out ? kEpiGrad : kEpiSgd;
    p.out = dw_out;
    p.kb_per_split = p.kblocks;
    return launch(p, 1, st);
  }
  p.epi = kEpiPartial;
  p.out = ws;
  cudaError_t e = launch(p, splits, st);
  if (e != cudaSuccess) return e;
  p.epi = dw_out ? kEpiGrad : kEpiSgd;
  p.y = dw_out;
  if (dw_out) p.w_mut = nullptr;
  const int64_t total = static_cast<int64_t>(p.Cout) * p.M;
  const int blocks = static_cast<int>(std::min<int64_t>((total + 255) / 256, 4 * kNumSms));
  wgrad_reduce_kernel<<<blocks, 256, 0, st>>>(p, splits);
  count_launch();
  return cudaGetLastError();
}

}  // namespace vdnnk
