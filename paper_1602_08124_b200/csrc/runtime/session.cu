// B200 executor for a vDNN plan.
//
// Layout:
//   * one cudaMalloc'd device arena spanning the planned pool offsets
//     [lo, hi); a buffer's pointer is base + its planned pool offset, so the
//     arena enforces the HBM budget the planner was given and the offsets are
//     byte-identical to the reference's (simulator.hpp:203-220);
//   * one cudaHostAlloc'd pinned arena with a slot per offloaded feature
//     buffer (HostLedger peak, memory_pool.hpp:225-256);
//   * two streams: compute (FWD/BWD kernels) and memory (OFFLOAD D2H /
//     PREFETCH H2D), gated by CUDA events exactly as the reference's sync
//     rules (simulator.hpp:315-322 forward, :400-441 backward; PAPER.md
//     Fig. 9): FWD(n+1) waits for layer n's offloads, BWD(m) waits for the
//     prefetches it reads, and the next BWD waits for every prefetch launched
//     during the current step. The memory stream waits for the compute
//     stream's "step start" event so a transfer never touches an extent
//     before every earlier user of it has finished.
//   * non-pool scratch (documented in DESIGN.md): softmax gradient / loss,
//     labels, split-K partials, and (data-parallel mode) the gradient arena.
#include <cstdlib>
#include <algorithm>
#include <cmath>
#include <cstring>
#include <map>
#include <set>
#include <stdexcept>

#include "session.h"

namespace vdnnrt {

using namespace vdnnp;

namespace {

struct CudaError : std::runtime_error {
  using std::runtime_error::runtime_error;
};
}  // namespace

void Session::check(cudaError_t e, const char* what) const {
  if (e != cudaSuccess) throw CudaError(std::string(what) + ": " + cudaGetErrorString(e));
}

// fp32 -> bf16 bit pattern, round to nearest even (NaN stays NaN)
uint16_t to_bf16_bits(float f) {
  uint32_t u;
  std::memcpy(&u, &f, 4);
  if ((u & 0x7FFFFFFFu) > 0x7F800000u) return static_cast<uint16_t>((u >> 16) | 0x40u);
  u += 0x7FFFu + ((u >> 16) & 1u);
  return static_cast<uint16_t>(u >> 16);
}

// count elements of pool storage at dev -> fp32 host values
void Session::read_device(float* host, const void* dev, size_t count) const {
  if (!bf_) {
    check(cudaMemcpy(host, dev, count * 4, cudaMemcpyDeviceToHost), "D2H");
    return;
  }
  std::vector<uint16_t> b(count);
  check(cudaMemcpy(b.data(), dev, count * 2, cudaMemcpyDeviceToHost), "D2H");
  for (size_t i = 0; i < count; ++i) {
    const uint32_t u = static_cast<uint32_t>(b[i]) << 16;
    std::memcpy(host + i, &u, 4);
  }
}

Session::Session(const Net& g, const Decision& d, const Cost& c, u64 capacity, const Options& o)
    : g_(g), d_(d), c_(c), cap_(capacity), o_(o) {
  // everything that can be rejected is rejected before the first allocation
  if (c_.elem != 4 && c_.elem != 2)
    throw PlanError(Err::Config, "the CUDA executor stores fp32 (elem_size 4) or bf16 (elem_size 2)");
  bf_ = c_.elem == 2;
  es_ = c_.elem;
  if (bf_ && o_.precise) throw PlanError(Err::Config, "precise (3xTF32) contractions apply to fp32 storage");
  if (bf_ && o_.compress_offload == 2)
    throw PlanError(Err::Config, "TF32-exact transfers apply to fp32 storage (bf16 maps use the lossless format)");
  if (o_.offload_target != 0 && o_.compress_offload)
    throw PlanError(Err::Config, "compressed offload targets the pinned host arena only");
  plan_ = vdnnp::plan(g_, d_, c_, cap_, {}, &prog_);
  if (!plan_.pass) throw PlanError(Err::Generic, "plan does not fit the budget: " + plan_.verdict());
  df_ = vdnnp::derive_dataflow(g_, d_, c_);
  L_ = g_.size();
  // The reference vocabulary (net_graph.hpp:83,281-321): concat and
  // elementwise joins, strided convs, any number of INPUT and LOSS layers.
  loss_classes_.assign(static_cast<size_t>(L_), 0);
  loss_grad_at_.assign(static_cast<size_t>(L_), 0);
  for (const Node& l : g_.nodes()) {
    if (l.in.size() > static_cast<size_t>(vdnnk::kMaxConvSegs))
      throw PlanError(Err::Config, "UNSUPPORTED: more than 8 inputs to one layer");
    if (l.kind == Kind::Input) {
      if (input_id_ < 0) input_id_ = l.id;
      inputs_.push_back(l.id);
    }
    if (l.kind == Kind::Loss) {
      if (loss_id_ < 0) loss_id_ = l.id;  // the first head writes the loss, later heads add to it
      const Dims& ld = g_.dims(l.in[0]);
      const int k = static_cast<int>(ld.c * ld.h * ld.w);
      loss_classes_[static_cast<size_t>(l.id)] = k;
      loss_grad_at_[static_cast<size_t>(l.id)] = loss_grad_count_;
      loss_grad_count_ += g_.batch() * static_cast<u64>(k);
      classes_ = std::max(classes_, k);
    }
  }
  if (input_id_ < 0 || loss_id_ < 0) throw PlanError(Err::Config, "UNSUPPORTED: graph needs an INPUT and a LOSS layer");
  logits_owner_ = g_.owner(g_.at(loss_id_).in[0]);
  // pinned host slots: one per offloaded owner
  host_slot_.assign(static_cast<size_t>(L_), kNoOff);
  for (const vdnnp::Xfer& x : prog_.xfers)
    if (x.to_host && host_slot_[static_cast<size_t>(x.owner)] == kNoOff) {
      host_slot_[static_cast<size_t>(x.owner)] = host_bytes_;
      // compressed mode: a slot holds the worst case (every chunk dense + its mask)
      const u64 slot = bf_ ? vdnnk::zvc_slot_bytes_bf16(x.bytes) : vdnnk::zvc_slot_bytes(x.bytes);
      host_bytes_ += round_up(o_.compress_offload ? std::max<u64>(x.bytes, slot) : x.bytes, 4096);
    }
  if (host_bytes_ > 0 && o_.offload_target == 0 && !o_.host_arena)
    throw PlanError(Err::Config, "plan offloads but the host arena is disabled");

  try {
    acquire();
  } catch (...) {
    release();  // a partly built session frees what it got (the destructor will not run)
    throw;
  }
}

// All device / host resources of a session, in one place so a failing
// constructor can undo them.
void Session::acquire() {
  check(cudaSetDevice(o_.device), "cudaSetDevice");
  check(cudaStreamCreateWithFlags(&cs_, cudaStreamNonBlocking), "stream");
  check(cudaStreamCreateWithFlags(&ms_, cudaStreamNonBlocking), "stream");

  // device arena over the planned span [arena_lo, arena_hi), plus the
  // two-buffer overflow gradient slots (if the graph needs them) right after
  if (prog_.arena_hi <= prog_.arena_lo) throw PlanError(Err::Generic, "empty plan");
  arena_lo_ = prog_.arena_lo;
  arena_bytes_ = prog_.arena_hi - prog_.arena_lo;
  // beyond the planned span (reported as non-pool scratch): two-buffer
  // overflow gradient slots, then the private planes of ACTVs over shared
  // elementwise-join maps
  const u64 overflow = static_cast<u64>(prog_.overflow_slots) * prog_.overflow_slot_bytes + prog_.private_bytes;
  check(cudaMalloc(&arena_, arena_bytes_ + overflow), "cudaMalloc(device arena)");
  base_ = arena_ - arena_lo_;
  scratch_bytes_ += overflow;

  if (host_bytes_ > 0 && o_.offload_target == 0) {
    check(cudaHostAlloc(&host_, host_bytes_, o_.compress_offload ? cudaHostAllocMapped : cudaHostAllocDefault),
          "cudaHostAlloc(host arena)");
    host_owned_ = true;
    if (o_.compress_offload) {
      void* dv = nullptr;
      check(cudaHostGetDevicePointer(&dv, host_, 0), "cudaHostGetDevicePointer(host arena)");
      host_dev_ = static_cast<char*>(dv);
    }
  }
  check(cudaMalloc(&wire_, 2 * sizeof(unsigned long long)), "cudaMalloc(wire counters)");
  check(cudaMemsetAsync(wire_, 0, 2 * sizeof(unsigned long long), cs_), "memset wire counters");

  // non-pool scratch: softmax gradient + per-row loss + loss, two label slots
  const u64 n = g_.batch();
  check(cudaMalloc(&loss_grad_, loss_grad_count_ * es_), "cudaMalloc(loss grad)");
  check(cudaMalloc(&row_loss_, n * 4), "cudaMalloc(row loss)");
  check(cudaMalloc(&loss_, 4), "cudaMalloc(loss)");
  check(cudaMalloc(&labels_, 2 * n * 4), "cudaMalloc(labels)");
  labels_next_ = labels_ + n;
  check(cudaHostAlloc(&pinned_loss_, 4, cudaHostAllocDefault), "cudaHostAlloc(loss)");
  scratch_bytes_ += loss_grad_count_ * es_ + n * 12 + 4;
  check(cudaMemsetAsync(labels_, 0, 2 * n * 4, cs_), "memset labels");

  build_program();

  // split-K partials: in the step's free pool gap when it is wide enough
  // (inside the budget), else in one fallback buffer sized for the steps
  // whose gap is not
  size_t need = 0;
  for (const FwdStep& s : fwd_)
    if (s.scratch > s.gap_len) need = std::max(need, s.scratch);
  for (const BwdStep& s : bwd_)
    if (s.scratch > s.gap_len) need = std::max(need, s.scratch);
  splitk_bytes_ = need;
  if (splitk_bytes_ > 0) check(cudaMalloc(&splitk_, splitk_bytes_), "cudaMalloc(split-K)");
  scratch_bytes_ += splitk_bytes_;

  if (o_.external_grads) {
    grad_off_.assign(static_cast<size_t>(L_), kNoOff);
    for (int i = 0; i < L_; ++i) {
      const u64 wb = df_.at[static_cast<size_t>(i)].w_bytes;
      if (wb == 0) continue;
      grad_off_[static_cast<size_t>(i)] = grads_count_;
      grads_count_ += wb / es_;  // fp32 gradients
    }
    check(cudaMalloc(&grads_, std::max<size_t>(grads_count_, 1) * 4), "cudaMalloc(grad arena)");
    scratch_bytes_ += grads_count_ * 4;
  }

  // timing / gating events
  const size_t nsteps = fwd_.size() + bwd_.size();
  const size_t nxfer = prog_.xfers.size();
  step_ev_.resize(nsteps);
  for (auto& e : step_ev_) check(cudaEventCreateWithFlags(&e, cudaEventDisableTiming), "event");
  xfer_ev_.resize(std::max<size_t>(nxfer, 1));
  for (auto& e : xfer_ev_) check(cudaEventCreateWithFlags(&e, cudaEventDisableTiming), "event");
  if (o_.record_timeline) {
    ev_.resize(2 * (nsteps + nxfer));
    for (auto& e : ev_) check(cudaEventCreate(&e), "event");
    t0_ev_.resize(nsteps);
    for (auto& e : t0_ev_) check(cudaEventCreate(&e), "event");
    check(cudaEventCreate(&ev_iter_), "event");
    ev_prev_.resize(ev_.size());
    for (auto& e : ev_prev_) check(cudaEventCreate(&e), "event");
    t0_ev_prev_.resize(nsteps);
    for (auto& e : t0_ev_prev_) check(cudaEventCreate(&e), "event");
    check(cudaEventCreate(&ev_iter_prev_), "event");
  }
  check(cudaEventCreateWithFlags(&ev_sync_, cudaEventDisableTiming), "event");
  check(cudaEventCreateWithFlags(&input_idle_ev_, cudaEventDisableTiming), "event");

  init_weights();
  check(cudaStreamSynchronize(cs_), "init");
}

Session::~Session() { release(); }

void Session::release() noexcept {
  if (cs_) cudaStreamSynchronize(cs_);
  if (ms_) cudaStreamSynchronize(ms_);
  if (in_stream_) cudaStreamSynchronize(in_stream_);
  if (gexec_) cudaGraphExecDestroy(gexec_);  // before the events its nodes record
  gexec_ = nullptr;
  for (auto* v : {&ev_, &step_ev_, &t0_ev_, &ev_prev_, &t0_ev_prev_, &xfer_ev_}) {
    for (auto e : *v)
      if (e) cudaEventDestroy(e);
    v->clear();
  }
  for (cudaEvent_t* e : {&ev_iter_prev_, &ev_iter_, &ev_sync_, &staged_ready_, &input_idle_ev_})
    if (*e) cudaEventDestroy(*e), *e = nullptr;
  for (auto& e : loss_ev_)
    if (e) cudaEventDestroy(e), e = nullptr;
  if (loss_ring_) cudaFreeHost(loss_ring_), loss_ring_ = nullptr;
  if (in_stream_) cudaStreamDestroy(in_stream_), in_stream_ = nullptr;
  peer_detach();
  if (xs_) cudaStreamSynchronize(xs_);
  for (auto e : wg_ev_)
    if (e) cudaEventDestroy(e);
  wg_ev_.clear();
  if (xs_done_) cudaEventDestroy(xs_done_), xs_done_ = nullptr;
  if (xs_) cudaStreamDestroy(xs_), xs_ = nullptr;
  if (signal_) cudaFree(signal_), signal_ = nullptr;
  if (arena_) cudaFree(arena_), arena_ = nullptr;
  if (host_ && host_owned_) cudaFreeHost(host_);
  host_ = nullptr;
  if (spill_map_) cudaIpcCloseMemHandle(spill_map_), spill_map_ = nullptr;
  if (spill_) cudaFree(spill_), spill_ = nullptr;
  for (void** p : {reinterpret_cast<void**>(&loss_grad_), reinterpret_cast<void**>(&row_loss_),
                   reinterpret_cast<void**>(&loss_), reinterpret_cast<void**>(&wire_),
                   reinterpret_cast<void**>(&labels_), reinterpret_cast<void**>(&splitk_)})
    if (*p) cudaFree(*p), *p = nullptr;
  if (pinned_loss_) cudaFreeHost(pinned_loss_), pinned_loss_ = nullptr;
  if (grads_ && grads_owned_) cudaFree(grads_);
  grads_ = nullptr;
  if (cs_) cudaStreamDestroy(cs_), cs_ = nullptr;
  if (ms_) cudaStreamDestroy(ms_), ms_ = nullptr;
  cudaGetLastError();  // leave no stale error from the teardown calls for the next session
}

// ------------------------------------------------------------- program ----
// The planner's Program already binds every operand to its pool offset, lists
// each step's transfers and the transfers its kernel waits for; this turns it
// into the launch-ready step lists.
void Session::build_program() {
  vdnnk::set_precise(o_.precise);  // scratch sizes depend on the contraction mode
  w_off_.assign(static_cast<size_t>(L_), kNoOff);
  for (int i = 0; i < L_; ++i) w_off_[static_cast<size_t>(i)] = prog_.w_off[static_cast<size_t>(i)];
  x_off_ = prog_.input_off;
  input_idle_after_ = inputs_.size() == 1 ? prog_.input_idle_after : -1;
  for (int id : inputs_) {  // setup extents of every INPUT layer
    u64 off = kNoOff;
    for (const Event& e : plan_.events)
      if (e.kind == Ev::Alloc && e.buffer == id && e.tag == "X") {
        off = e.off;
        break;
      }
    input_off_.push_back(off);
  }
  auto transfer = [&](int xi) {
    const vdnnp::Xfer& x = prog_.xfers[static_cast<size_t>(xi)];
    Transfer t;
    t.owner = x.owner;
    t.bytes = x.bytes;
    t.dev_off = x.dev_off;
    t.host_off = host_slot_[static_cast<size_t>(x.owner)];
    t.ev = xi;
    t.zvc = compressible(x.owner) && vdnnk::zvc_eligible(base_ + t.dev_off, t.bytes);
    t.tf32 = t.zvc && o_.compress_offload == 2 && tf32_exact_ok(x.owner);
    return t;
  };
  auto or_none = [](u64 v) { return v == vdnnp::kNoLoc ? kNoOff : v; };
  for (size_t si = 0; si < prog_.steps.size(); ++si) {
    const vdnnp::Step& p = prog_.steps[si];
    const Node& l = g_.at(p.layer);
    const bool contraction = l.kind == Kind::Conv || l.kind == Kind::Fc;
    if (!p.bwd) {
      FwdStep s;
      s.layer = p.layer;
      s.ev = static_cast<int>(si);
      for (u64 v : p.x) s.in_off.push_back(or_none(v));
      s.out_off = or_none(p.y);
      s.w_off = or_none(p.w);
      if (p.ws_bytes > 0) s.ws_off = or_none(p.ws), s.ws_bytes = p.ws_bytes;
      for (int xi : p.issues) s.offloads.push_back(transfer(xi));
      s.gap_off = p.gap_off;
      s.gap_len = p.gap_len;
      const float* probe_x = summed(s.layer) ? F(s.in_off[0]) : nullptr;  // shapes only
      if (summed(s.layer)) s.sum_bytes = round_up(g_.dims(l.in[0]).count() * es_, 1024);
      size_t at = s.sum_bytes;
      s.pad_c = padded_channels(s.layer);
      if (s.pad_c) {  // [X padded | W padded]
        const Dims& x = g_.dims(l.in[0]);
        s.x8_off = at;
        s.w8_off = at + round_up(x.n * x.h * x.w * static_cast<u64>(s.pad_c) * 2, 1024);
        at = s.w8_off + round_up(l.out * l.k * l.k * static_cast<u64>(s.pad_c) * 2, 1024);
      }
      if (contraction) {
        vdnnk::ConvArgs a = conv_args(s.layer, s.in_off, nullptr, probe_x);
        if (s.pad_c) a.c[0] = s.pad_c;
        s.part_bytes = bf_ ? vdnnk::conv_fprop_ws_bytes_bf16(a) : vdnnk::conv_fprop_ws_bytes(a);
      }
      s.part_off = at;
      s.scratch = s.part_bytes ? s.part_off + s.part_bytes : at;
      fwd_.push_back(std::move(s));
    } else {
      BwdStep s;
      s.layer = p.layer;
      s.ev = static_cast<int>(si);
      for (int xi : p.issues) s.prefetches.push_back(transfer(xi));
      s.wait_prefetch = p.wait_before;
      for (u64 v : p.x) s.in_off.push_back(or_none(v));
      s.out_off = or_none(p.y);
      s.w_off = or_none(p.w);
      if (p.ws_bytes > 0) s.ws_off = or_none(p.ws), s.ws_bytes = p.ws_bytes;
      for (const vdnnp::PlaneRef& pl : p.dx) s.plane_off.push_back(or_none(pl.off));
      s.accumulate = p.dx_accumulate;
      for (const vdnnp::PlaneRef& pl : p.dy) s.dy_off.push_back(pl.off);
      s.mask_plane.assign(s.plane_off.size(), 0);
      s.gap_off = p.gap_off;
      s.gap_len = p.gap_len;
      s.stage_dy = p.stage_dy;
      if (p.stage_dy && l.kind == Kind::Actv) s.priv_out = p.dx.at(0).off;
      const bool sum = summed(s.layer) && l.kind != Kind::Actv;
      const float* probe_x = sum ? F(s.in_off[0]) : nullptr;
      size_t at = 0;
      if (sum) s.sum_bytes = round_up(g_.dims(l.in[0]).count() * es_, 1024), at = s.sum_bytes;
      if (s.stage_dy && l.kind != Kind::Actv) {
        s.stage_off = at;
        s.stage_bytes = round_up(g_.dims(s.layer).count() * es_, 1024);
        at += s.stage_bytes;
      }
      bool any_plane = false;
      for (u64 o : s.plane_off) any_plane = any_plane || o != kNoOff;
      if (l.kind == Kind::Conv && l.s > 1 && any_plane) {  // dgrad through a zero-inserted dY
        const Dims& y = g_.dims(s.layer);
        s.dil_off = at;
        s.dil_bytes = round_up(y.n * ((y.h - 1) * l.s + 1) * ((y.w - 1) * l.s + 1) * y.c * es_, 1024);
        at += s.dil_bytes;
      }
      s.pad_c = any_plane ? 0 : padded_channels(s.layer);
      if (s.pad_c) {  // [X padded | W padded | fp32 dW of the padded weights]
        const Dims& x = g_.dims(l.in[0]);
        const u64 wn = l.out * l.k * l.k * static_cast<u64>(s.pad_c);
        s.x8_off = at;
        s.w8_off = at + round_up(x.n * x.h * x.w * static_cast<u64>(s.pad_c) * 2, 1024);
        s.dw8_off = s.w8_off + round_up(wn * 2, 1024);
        at = s.dw8_off + (o_.external_grads ? round_up(wn * 4, 1024) : 0);
      }
      if (contraction) {
        vdnnk::ConvArgs w = conv_args(s.layer, s.in_off, nullptr, probe_x);
        if (s.pad_c) w.c[0] = s.pad_c;
        s.part_bytes = bf_ ? vdnnk::conv_wgrad_ws_bytes_bf16(w) : vdnnk::conv_wgrad_ws_bytes(w);
        if (any_plane) {
          vdnnk::ConvArgs a = conv_args(s.layer, s.in_off, &s.plane_off, probe_x);
          a.stride = 1;
          s.part_bytes = std::max(s.part_bytes, bf_ ? vdnnk::conv_dgrad_ws_bytes_bf16(a) : vdnnk::conv_dgrad_ws_bytes(a));
        }
      }
      s.part_off = at;
      s.scratch = s.part_bytes ? at + s.part_bytes : at;
      bwd_.push_back(std::move(s));
    }
  }
  fuse_relus();
}

float* Session::scratch_for(u64 gap_off, u64 gap_len, size_t need) const {
  if (need == 0) return nullptr;
  return need <= gap_len ? F(gap_off) : splitk_;
}

// Compressed mode moves a buffer through the SMs only when it holds ReLU
// outputs (its owner feeds an in-place ACTV), about half zeros; dense maps
// (raw images, max-pool outputs: ~94% nonzero) keep the copy engines, which
// move dense bytes ~10% faster than SM-driven PCIe stores/loads.
// ReLU outputs (~35% nonzero on VGG-16) and max-pool outputs (the max of
// ReLU windows: ~50% zeros, tools/zvc_stats.py) go through the compressing
// kernels; dense maps (the input images) keep the copy engines.
// Mode 2: a map may travel TF32-exact when everything that reads it in the
// backward pass consumes it only through a tcgen05 kind::tf32 contraction
// (conv / FC wgrad operand) or a ReLU mask (x > 0, preserved: zvc.cu keeps
// any chunk with a would-be-zero denormal lossless): its readers, through
// in-place ACTV aliases, are conv layers with > 4 input channels (C <= 4
// layers may run SIMT kernels) and FC layers. A max-pool's backward routes
// dY by the window maximum of its input X, so pool inputs stay lossless;
// pool outputs qualify (the pool backward recomputes the maximum from X and
// does not read Y, elementwise.cu).
bool Session::tf32_exact_ok(int owner) const {
  const Kind k = g_.at(owner).kind;
  if (o_.precise || (k != Kind::Conv && k != Kind::Fc && k != Kind::Pool)) return false;
  std::vector<int> todo(g_.users(owner).begin(), g_.users(owner).end());
  while (!todo.empty()) {
    const int u = todo.back();
    todo.pop_back();
    const Node& n = g_.at(u);
    if (summed(u)) return false;  // a join's sum of truncated maps is not the truncated sum
    if (n.kind == Kind::Actv) {
      todo.insert(todo.end(), g_.users(u).begin(), g_.users(u).end());
    } else if (n.kind == Kind::Conv) {
      if (g_.in_dims(u).c <= 4) return false;
    } else if (n.kind != Kind::Fc) {
      return false;
    }
  }
  return true;
}

bool Session::compressible(int owner) const {
  if (!o_.compress_offload) return false;
  if (g_.at(owner).kind == Kind::Pool) return true;
  for (int u : g_.users(owner))
    if (g_.at(u).kind == Kind::Actv) return true;
  return false;
}

// ReLU fusion (bit-identical to running the ACTV kernels):
//  * FWD: a conv/FC whose only consumer is an ACTV applies max(0, .) in its
//    epilogue; the ACTV's FWD launches nothing (nothing else reads the
//    pre-activation values, and the buffer is the same in-place alias).
//  * BWD: the planner names, for an ACTV whose incoming plane has exactly one
//    writer (a conv/FC dgrad or pool backward reading the ACTV's output as
//    that input, nothing folded or accumulated into the plane), that writer's
//    step (Step::mask_host); its epilogue applies the mask (x > 0) and the
//    ACTV's BWD launches nothing.
void Session::fuse_relus() {
  std::vector<int> fwd_at(static_cast<size_t>(L_), -1);
  for (size_t i = 0; i < fwd_.size(); ++i) fwd_at[static_cast<size_t>(fwd_[i].layer)] = static_cast<int>(i);
  for (FwdStep& s : fwd_) {
    const Node& l = g_.at(s.layer);
    if (l.kind != Kind::Conv && l.kind != Kind::Fc) continue;
    const auto& us = g_.users(s.layer);
    if (us.size() != 1 || g_.at(us[0]).kind != Kind::Actv) continue;
    const int fa = fwd_at[static_cast<size_t>(us[0])];
    if (fa < 0) continue;
    s.relu = true;
    fwd_[static_cast<size_t>(fa)].skip = true;
  }
  const size_t nf = fwd_.size();
  for (BwdStep& a : bwd_) {
    const vdnnp::Step& p = prog_.steps[static_cast<size_t>(a.ev)];
    if (p.mask_host < 0 || static_cast<size_t>(p.mask_host) < nf) continue;
    BwdStep& host = bwd_[static_cast<size_t>(p.mask_host) - nf];
    host.mask_plane[static_cast<size_t>(p.mask_slot)] = 1;
    a.skip = true;
  }
}

// ------------------------------------------------------------- helpers ----
bool Session::summed(int layer) const {
  const Node& l = g_.at(layer);
  return l.join == Join::Elementwise && l.in.size() > 1;
}

// BF16 conv over the raw input with a channel count that is not a multiple
// of 8 (C = 3 images): its rows (6 B per pixel) cannot feed TMA, so the step
// pads X and W to 8 channels (zeros) in its scratch and runs the padded
// contraction; zero channels add nothing to Y, and their weight gradients are
// zero, so the update of the real weights is unchanged.
int Session::padded_channels(int layer) const {
  const Node& l = g_.at(layer);
  static const bool on = [] {  // VDNN_BF16_PAD=0: the unpadded gather path (A/B switch)
    const char* e = std::getenv("VDNN_BF16_PAD");
    return !e || std::atoi(e) != 0;
  }();
  if (!on || !bf_ || l.kind != Kind::Conv || l.in.size() != 1 || g_.at(l.in[0]).kind != Kind::Input) return 0;
  const int c = static_cast<int>(g_.dims(l.in[0]).c);
  if (c % 8 == 0) return 0;
  const std::vector<u64> shape_only(l.in.size(), 0);  // shapes only, no pointer is dereferenced
  if (vdnnk::conv_bf16_c3_native(conv_args(layer, shape_only, nullptr, nullptr))) return 0;
  return (c + 7) / 8 * 8;
}

// GEMM_WS as the reference's algorithm (algo_kernels = 1): a single-input
// conv whose planned algorithm is GEMM_WS and whose planned workspace holds
// the im2col matrix (cost_model.hpp:163-168 sizes it exactly so).
bool Session::gemmws(int layer, u64 ws_off, u64 ws_bytes) const {
  if (o_.algo_kernels != 1 || ws_off == kNoOff || ws_bytes == 0) return false;
  const Node& l = g_.at(layer);
  if (l.kind != Kind::Conv || l.in.size() != 1 || summed(layer) || padded_channels(layer)) return false;
  const auto it = d_.algos.find(layer);
  if (it == d_.algos.end() || it->second != Algo::GemmWs) return false;
  const std::vector<u64> shape_only(1, 0);
  return vdnnk::gemmws_col_bytes(conv_args(layer, shape_only, nullptr, nullptr), static_cast<int>(es_)) <= ws_bytes;
}

// X and W of a padded step into the scratch; `a` then describes the padded X.
void Session::pad_operands(vdnnk::ConvArgs& a, int cp, char* x8, const float* w, char* w8) {
  const int c = a.c[0];
  check(vdnnk::pad_channels_bf16(x8, a.x[0], static_cast<size_t>(a.n) * a.h * a.w, c, cp, cs_), "pad X");
  check(vdnnk::pad_channels_bf16(w8, w, static_cast<size_t>(a.cout) * a.kh * a.kw, c, cp, cs_), "pad W");
  a.x[0] = reinterpret_cast<const float*>(x8);
  a.c[0] = cp;
}

// X of an elementwise join (net_graph.hpp:290-296: identical shapes) = the
// sum of its inputs, into the step's scratch.
void Session::sum_inputs(int layer, const std::vector<u64>& in_off, float* dst) {
  const Node& l = g_.at(layer);
  std::vector<const float*> src;
  for (size_t i = 0; i < l.in.size(); ++i) src.push_back(F(in_off[i]));
  k_combine(dst, src, nullptr, g_.dims(l.in[0]).count(), "join sum");
}

// ---------------------------------------------- storage-type dispatch ----
void Session::k_combine(void* dst, const std::vector<const float*>& src, const void* y, size_t n, const char* what) {
  if (bf_) {
    std::vector<const void*> v(src.begin(), src.end());
    check(vdnnk::combine_bf16(dst, v.data(), static_cast<int>(v.size()), y, n, cs_), what);
  } else {
    check(vdnnk::combine(static_cast<float*>(dst), src.data(), static_cast<int>(src.size()),
                         static_cast<const float*>(y), n, cs_),
          what);
  }
}

void Session::k_add_into(float* dst, const std::vector<const float*>& src, size_t n, const char* what) {
  if (bf_) {
    std::vector<const void*> v(src.begin(), src.end());
    check(vdnnk::add_into_bf16(dst, v.data(), static_cast<int>(v.size()), n, cs_), what);
  } else {
    check(vdnnk::add_into(dst, src.data(), static_cast<int>(src.size()), n, cs_), what);
  }
}

void Session::k_relu_bwd(float* g0, const std::vector<const float*>& extra, const float* y, size_t n) {
  if (bf_) {
    std::vector<const void*> v(extra.begin(), extra.end());
    check(vdnnk::relu_bwd_bf16(g0, v.data(), static_cast<int>(v.size()), y, n, cs_), "relu_bwd");
  } else {
    check(vdnnk::relu_bwd(g0, extra.data(), static_cast<int>(extra.size()), y, n, cs_), "relu_bwd");
  }
}

vdnnk::PoolArgs Session::pool_args(int layer, const std::vector<u64>& in_off, const std::vector<u64>* planes,
                                   const float* sum_x) const {
  const Node& l = g_.at(layer);
  vdnnk::PoolArgs p;
  const Dims& first = g_.dims(l.in[0]);
  p.n = static_cast<int>(first.n);
  p.h = static_cast<int>(first.h);
  p.w = static_cast<int>(first.w);
  p.window = static_cast<int>(l.k);
  p.stride = static_cast<int>(l.s);
  p.nseg = sum_x ? 1 : static_cast<int>(l.in.size());
  for (int i = 0; i < p.nseg; ++i) {
    p.x[i] = sum_x ? sum_x : F(in_off[static_cast<size_t>(i)]);
    p.c[i] = static_cast<int>(g_.dims(l.in[static_cast<size_t>(i)]).c);
    p.dx[i] = nullptr;
  }
  if (planes) {
    for (size_t i = 0; i < planes->size(); ++i) {
      if ((*planes)[i] == kNoOff) continue;
      const size_t slot = sum_x ? 0 : i;  // a join's one shared map
      p.dx[slot] = F((*planes)[i]);
    }
  }
  return p;
}

vdnnk::ConvArgs Session::conv_args(int layer, const std::vector<u64>& in_off,
                                   const std::vector<u64>* planes, const float* sum_x) const {
  const Node& l = g_.at(layer);
  vdnnk::ConvArgs a;
  if (sum_x) {  // elementwise join: one segment (the summed input), one shared gradient map
    const Dims& d = g_.dims(l.in[0]);
    const bool fc = l.kind == Kind::Fc;
    a.nseg = 1;
    a.n = static_cast<int>(d.n);
    a.h = fc ? 1 : static_cast<int>(d.h);
    a.w = fc ? 1 : static_cast<int>(d.w);
    a.c[0] = static_cast<int>(fc ? d.c * d.h * d.w : d.c);
    a.x[0] = sum_x;
    if (planes)
      for (u64 o : *planes)
        if (o != kNoOff && !a.dx[0]) a.dx[0] = F(o);
    a.cout = static_cast<int>(l.out);
    a.kh = a.kw = fc ? 1 : static_cast<int>(l.k);
    a.stride = fc ? 1 : static_cast<int>(l.s);
    a.pad = fc ? 0 : static_cast<int>(l.p);
    return a;
  }
  a.nseg = static_cast<int>(l.in.size());
  const Dims& first = g_.dims(l.in[0]);
  a.n = static_cast<int>(first.n);
  const bool fc = l.kind == Kind::Fc;
  a.h = fc ? 1 : static_cast<int>(first.h);
  a.w = fc ? 1 : static_cast<int>(first.w);
  for (int i = 0; i < a.nseg; ++i) {
    const Dims& d = g_.dims(l.in[static_cast<size_t>(i)]);
    a.c[i] = static_cast<int>(fc ? d.c * d.h * d.w : d.c);
    a.x[i] = F(in_off[static_cast<size_t>(i)]);
    a.dx[i] = nullptr;
    if (planes && (*planes)[static_cast<size_t>(i)] != kNoOff) a.dx[i] = F((*planes)[static_cast<size_t>(i)]);
  }
  a.cout = static_cast<int>(l.out);
  if (fc) {
    a.kh = a.kw = 1;
    a.stride = 1;
    a.pad = 0;
  } else {
    a.kh = a.kw = static_cast<int>(l.k);
    a.stride = static_cast<int>(l.s);
    a.pad = static_cast<int>(l.p);
  }
  return a;
}

void Session::init_weights() {
  for (const Node& l : g_.nodes()) {
    const size_t i = static_cast<size_t>(l.id);
    if (df_.at[i].w_bytes == 0) continue;
    const u64 seed = o_.weight_seed + static_cast<u64>(l.id);
    auto normal = [&](u64 off, u64 n, float sd) {
      check(bf_ ? vdnnk::fill_normal_bf16(F(off), n, sd, seed, cs_) : vdnnk::fill_normal(F(off), n, sd, seed, cs_),
            "init");
    };
    if (l.kind == Kind::Conv) {
      const u64 fan = l.k * l.k * g_.in_dims(l.id).c;
      normal(w_off_[i], df_.at[i].w_bytes / es_, std::sqrt(2.0f / static_cast<float>(fan)));
    } else {
      const u64 in = g_.fc_inputs(l.id);
      normal(w_off_[i], in * l.out, std::sqrt(2.0f / static_cast<float>(in)));
      const u64 b = w_off_[i] + in * l.out * es_;
      check(bf_ ? vdnnk::fill_const_bf16(F(b), l.out, 0.0f, cs_) : vdnnk::fill_const(F(b), l.out, 0.0f, cs_), "init");
    }
  }
}

// ------------------------------------------------------------- execution --
void Session::run_fwd(const FwdStep& s, float lr) {
  (void)lr;
  const Node& l = g_.at(s.layer);
  cudaEvent_t start = step_ev_[static_cast<size_t>(s.ev)];
  check(cudaEventRecord(start, cs_), "record");
  if (timed_) check(cudaEventRecord(t0_ev_[static_cast<size_t>(s.ev)], cs_), "record");
  if (!s.offloads.empty()) {
    // the offloaded inputs are complete once every earlier compute op is: gate on the step start
    check(cudaStreamWaitEvent(ms_, start, 0), "wait");
    for (const Transfer& t : s.offloads) {
      if (timed_) check(cudaEventRecord(ev_[2 * (fwd_.size() + bwd_.size() + t.ev)], ms_), "record");
      if (t.zvc)
        check(bf_ ? vdnnk::zvc_compress_bf16(F(t.dev_off), t.bytes / 2, host_dev_ + t.host_off, wire_, ms_)
                  : vdnnk::zvc_compress(F(t.dev_off), t.bytes / 4, host_dev_ + t.host_off, wire_, ms_, t.tf32),
              "zvc offload");
      else {
        check(cudaMemcpyAsync(host_ + t.host_off, base_ + t.dev_off, t.bytes, cudaMemcpyDefault, ms_), "offload copy");
        copy_off_ += t.bytes;
      }
      raw_off_ += t.bytes;
      if (timed_) check(cudaEventRecord(ev_[2 * (fwd_.size() + bwd_.size() + t.ev) + 1], ms_), "record");
      check(cudaEventRecord(xfer_ev_[static_cast<size_t>(t.ev)], ms_), "record");
    }
  }
  if (timed_) check(cudaEventRecord(ev_[2 * s.ev], cs_), "record");
  if (!probes_.empty()) probe_copy(s.ev, false);
  char* scr = reinterpret_cast<char*>(scratch_for(s.gap_off, s.gap_len, s.scratch));
  const float* sum_x = nullptr;
  if (s.sum_bytes) {
    sum_inputs(s.layer, s.in_off, reinterpret_cast<float*>(scr));
    sum_x = reinterpret_cast<const float*>(scr);
  }
  float* part = s.part_bytes ? reinterpret_cast<float*>(scr + s.part_off) : nullptr;
  switch (l.kind) {
    case Kind::Conv:
    case Kind::Fc: {
      vdnnk::ConvArgs a = conv_args(s.layer, s.in_off, nullptr, sum_x);
      a.relu_out = s.relu ? 1 : 0;
      const float* bias = l.kind == Kind::Fc ? F(s.w_off + g_.fc_inputs(s.layer) * l.out * es_) : nullptr;
      const float* w = F(s.w_off);
      if (gemmws(s.layer, s.ws_off, s.ws_bytes)) {
        // GEMM_WS: im2col into the planned workspace, then Y = col x W^T
        float* col = F(s.ws_off);
        check(vdnnk::im2col(a, static_cast<int>(es_), col, cs_), "im2col");
        const vdnnk::ConvArgs g1 = vdnnk::gemmws_args(a, col, nullptr);
        check(bf_ ? vdnnk::conv_fprop_bf16(g1, w, nullptr, F(s.out_off), false, cs_, nullptr, 0)
                  : vdnnk::conv_fprop(g1, w, nullptr, F(s.out_off), false, cs_, nullptr, 0),
              "conv_fprop (GEMM_WS)");
        break;
      }
      if (s.pad_c) {
        w = reinterpret_cast<float*>(scr + s.w8_off);
        pad_operands(a, s.pad_c, scr + s.x8_off, F(s.w_off), scr + s.w8_off);
      }
      check(bf_ ? vdnnk::conv_fprop_bf16(a, w, bias, F(s.out_off), false, cs_, part, s.part_bytes)
                : vdnnk::conv_fprop(a, w, bias, F(s.out_off), false, cs_, part, s.part_bytes),
            "conv_fprop");
      break;
    }
    case Kind::Actv:
      if (!s.skip)
        check(bf_ ? vdnnk::relu_fwd_bf16(F(s.out_off), g_.dims(s.layer).count(), cs_)
                  : vdnnk::relu_fwd(F(s.out_off), g_.dims(s.layer).count(), cs_),
              "relu_fwd");
      break;
    case Kind::Pool:
      check(bf_ ? vdnnk::maxpool_fwd_bf16(pool_args(s.layer, s.in_off, nullptr, sum_x), F(s.out_off), cs_)
                : vdnnk::maxpool_fwd(pool_args(s.layer, s.in_off, nullptr, sum_x), F(s.out_off), cs_),
            "maxpool_fwd");
      break;
    case Kind::Loss: {
      const size_t li = static_cast<size_t>(s.layer);
      const int n = static_cast<int>(g_.batch());
      check(bf_ ? vdnnk::softmax_xent_fwd_bf16(F(s.in_off[0]), labels_, n, loss_classes_[li], LG(loss_grad_at_[li]),
                                               row_loss_, loss_, cs_, s.layer != loss_id_)
                : vdnnk::softmax_xent_fwd(F(s.in_off[0]), labels_, n, loss_classes_[li],
                                          loss_grad_ + loss_grad_at_[li], row_loss_, loss_, cs_, s.layer != loss_id_),
            "softmax_xent");
      break;
    }
    default:
      break;
  }
  if (!probes_.empty()) probe_copy(s.ev, true);
  if (timed_) check(cudaEventRecord(ev_[2 * s.ev + 1], cs_), "record");
  if (!s.offloads.empty())  // sync rule: FWD(n+1) may not start before n's offloads drain
    check(cudaStreamWaitEvent(cs_, xfer_ev_[static_cast<size_t>(s.offloads.back().ev)], 0), "wait");
  if (s.ev == input_idle_after_) check(cudaEventRecord(input_idle_ev_, cs_), "record");
}

void Session::run_bwd(const BwdStep& s, float lr) {
  const Node& l = g_.at(s.layer);
  const size_t mi = static_cast<size_t>(s.layer);
  cudaEvent_t start = step_ev_[static_cast<size_t>(s.ev)];
  check(cudaEventRecord(start, cs_), "record");
  if (timed_) check(cudaEventRecord(t0_ev_[static_cast<size_t>(s.ev)], cs_), "record");
  if (!s.prefetches.empty()) {
    check(cudaStreamWaitEvent(ms_, start, 0), "wait");
    for (const Transfer& t : s.prefetches) {
      if (timed_) check(cudaEventRecord(ev_[2 * (fwd_.size() + bwd_.size() + t.ev)], ms_), "record");
      if (t.zvc)
        check(bf_ ? vdnnk::zvc_decompress_bf16(host_dev_ + t.host_off, t.bytes / 2, F(t.dev_off), wire_ + 1, ms_)
                  : vdnnk::zvc_decompress(host_dev_ + t.host_off, t.bytes / 4, F(t.dev_off), wire_ + 1, ms_),
              "zvc prefetch");
      else {
        check(cudaMemcpyAsync(base_ + t.dev_off, host_ + t.host_off, t.bytes, cudaMemcpyDefault, ms_), "prefetch copy");
        copy_pre_ += t.bytes;
      }
      raw_pre_ += t.bytes;
      if (timed_) check(cudaEventRecord(ev_[2 * (fwd_.size() + bwd_.size() + t.ev) + 1], ms_), "record");
      check(cudaEventRecord(xfer_ev_[static_cast<size_t>(t.ev)], ms_), "record");
    }
  }
  for (int ev : s.wait_prefetch) check(cudaStreamWaitEvent(cs_, xfer_ev_[static_cast<size_t>(ev)], 0), "wait");
  if (timed_) check(cudaEventRecord(ev_[2 * s.ev], cs_), "record");

  char* scr = reinterpret_cast<char*>(scratch_for(s.gap_off, s.gap_len, s.scratch));
  float* part = s.part_bytes ? reinterpret_cast<float*>(scr + s.part_off) : nullptr;
  const size_t ycount = g_.dims(s.layer).count();
  float* dy = s.dy_off.empty() ? nullptr : F(s.dy_off[0]);
  std::vector<const float*> extra;
  for (size_t k = 1; k < s.dy_off.size(); ++k) extra.push_back(F(s.dy_off[k]));
  if (l.kind != Kind::Actv && s.stage_dy) {  // shared planes are read-only: sum into scratch
    std::vector<const float*> all{dy};
    all.insert(all.end(), extra.begin(), extra.end());
    dy = reinterpret_cast<float*>(scr + s.stage_off);
    k_combine(dy, all, nullptr, ycount, "fold (staged)");
  } else if (l.kind != Kind::Actv && !extra.empty()) {
    k_add_into(dy, extra, ycount, "fold");
  }
  const float* sum_x = nullptr;
  if (s.sum_bytes) {
    sum_inputs(s.layer, s.in_off, reinterpret_cast<float*>(scr));
    sum_x = reinterpret_cast<const float*>(scr);
  }
  if (!probes_.empty()) probe_copy(s.ev, false);

  switch (l.kind) {
    case Kind::Conv:
    case Kind::Fc: {
      const bool fc = l.kind == Kind::Fc;
      bool any_plane = false;
      for (u64 o : s.plane_off) any_plane = any_plane || o != kNoOff;
      if (gemmws(s.layer, s.ws_off, s.ws_bytes)) {
        // GEMM_WS: dcol = dY x W into the planned workspace, col2im into dX
        // (fused ReLU-backward mask / accumulation); then col = im2col(X) in
        // the same workspace and dW = dY^T x col (fused SGD / fp32 dW)
        float* col = F(s.ws_off);
        float* dw = grads_ ? grads_ + grad_off_[mi] : nullptr;
        if (any_plane) {
          vdnnk::ConvArgs ad = conv_args(s.layer, s.in_off, &s.plane_off, nullptr);
          ad.mask_in[0] = s.mask_plane.empty() ? 0 : s.mask_plane[0];
          vdnnk::ConvArgs g1 = vdnnk::gemmws_args(ad, col, col);
          check(bf_ ? vdnnk::conv_dgrad_bf16(g1, F(s.w_off), dy, false, cs_, nullptr, 0)
                    : vdnnk::conv_dgrad(g1, F(s.w_off), dy, false, cs_, nullptr, 0),
                "conv_dgrad (GEMM_WS)");
          check(vdnnk::col2im(ad, static_cast<int>(es_), col, s.accumulate, cs_), "col2im");
        }
        const vdnnk::ConvArgs a = conv_args(s.layer, s.in_off, nullptr, nullptr);
        check(vdnnk::im2col(a, static_cast<int>(es_), col, cs_), "im2col");
        const vdnnk::ConvArgs g2 = vdnnk::gemmws_args(a, col, nullptr);
        check(bf_ ? vdnnk::conv_wgrad_bf16(g2, dy, F(s.w_off), lr, dw, part, s.part_bytes, cs_)
                  : vdnnk::conv_wgrad(g2, dy, F(s.w_off), lr, dw, part, s.part_bytes, cs_),
              "conv_wgrad (GEMM_WS)");
        if (peer_inline_ && grads_) peer_layer(s.layer, lr);
        break;
      }
      if (any_plane) {
        vdnnk::ConvArgs a = conv_args(s.layer, s.in_off, &s.plane_off, sum_x);
        for (int i = 0; i < a.nseg; ++i) a.mask_in[i] = sum_x ? 0 : s.mask_plane[static_cast<size_t>(i)];
        const float* dyd = dy;
        if (s.dil_bytes) {  // strided conv: stride-1 dgrad over the zero-inserted dY
          const Dims& y = g_.dims(s.layer);
          float* d = reinterpret_cast<float*>(scr + s.dil_off);
          const int yn = static_cast<int>(y.n), yh = static_cast<int>(y.h), yw = static_cast<int>(y.w),
                    yc = static_cast<int>(y.c);
          check(bf_ ? vdnnk::dilate_bf16(d, dy, yn, yh, yw, yc, a.stride, cs_)
                    : vdnnk::dilate(d, dy, yn, yh, yw, yc, a.stride, cs_),
                "dilate dY");
          a.stride = 1;
          dyd = d;
        }
        check(bf_ ? vdnnk::conv_dgrad_bf16(a, F(s.w_off), dyd, s.accumulate, cs_, part, s.part_bytes)
                  : vdnnk::conv_dgrad(a, F(s.w_off), dyd, s.accumulate, cs_, part, s.part_bytes),
              "conv_dgrad");
      }
      vdnnk::ConvArgs a = conv_args(s.layer, s.in_off, nullptr, sum_x);
      // split-K partials: the split count depends only on the layer shape
      // (the launch always gets the bytes it asks for), so the reduction
      // order -- and every bit of the update -- is independent of the offload
      // policy and of where the partials live
      float* dw = grads_ ? grads_ + grad_off_[mi] : nullptr;
      if (s.pad_c) {
        // padded weights: the update (or fp32 dW) lands in the padded copy,
        // then the real channels are copied back
        const size_t rows = l.out * l.k * l.k;
        const int c = a.c[0];
        char* w8 = scr + s.w8_off;
        float* dw8 = dw ? reinterpret_cast<float*>(scr + s.dw8_off) : nullptr;
        pad_operands(a, s.pad_c, scr + s.x8_off, F(s.w_off), w8);
        check(vdnnk::conv_wgrad_bf16(a, dy, w8, lr, dw8, part, s.part_bytes, cs_), "conv_wgrad (padded)");
        check(dw ? vdnnk::unpad_channels_f32(dw, dw8, rows, c, s.pad_c, cs_)
                 : vdnnk::unpad_channels_bf16(F(s.w_off), w8, rows, c, s.pad_c, cs_),
              "unpad weights");
      } else {
        check(bf_ ? vdnnk::conv_wgrad_bf16(a, dy, F(s.w_off), lr, dw, part, s.part_bytes, cs_)
                  : vdnnk::conv_wgrad(a, dy, F(s.w_off), lr, dw, part, s.part_bytes, cs_),
              "conv_wgrad");
      }
      if (fc) {
        const u64 in = g_.fc_inputs(s.layer);
        float* bias = F(s.w_off + in * l.out * es_);
        float* db = grads_ ? grads_ + grad_off_[mi] + in * l.out : nullptr;
        const int n = static_cast<int>(g_.batch()), o = static_cast<int>(l.out);
        check(bf_ ? vdnnk::bias_grad_bf16(dy, n, o, bias, lr, db, cs_) : vdnnk::bias_grad(dy, n, o, bias, lr, db, cs_),
              "bias_grad");
      }
      if (peer_inline_ && grads_) peer_layer(s.layer, lr);
      break;
    }
    case Kind::Pool: {
      vdnnk::PoolArgs p = pool_args(s.layer, s.in_off, &s.plane_off, sum_x);
      bool any_plane = false;
      for (int i = 0; i < p.nseg; ++i) {
        p.mask_in[i] = (sum_x || s.mask_plane.empty()) ? 0 : s.mask_plane[static_cast<size_t>(i)];
        any_plane = any_plane || p.dx[i] != nullptr;
      }
      if (any_plane)
        check(bf_ ? vdnnk::maxpool_bwd_bf16(p, dy, cs_) : vdnnk::maxpool_bwd(p, F(s.out_off), dy, cs_), "maxpool_bwd");
      break;
    }
    case Kind::Actv:
      if (dy && s.priv_out != kNoOff) {  // shared incoming planes: masked sum into the private plane
        std::vector<const float*> all{dy};
        all.insert(all.end(), extra.begin(), extra.end());
        k_combine(F(s.priv_out), all, F(s.out_off), ycount, "relu_bwd (private plane)");
      } else if (dy && !s.skip) {
        k_relu_bwd(dy, extra, F(s.out_off), ycount);
      }
      break;
    case Kind::Loss: {
      const size_t li = static_cast<size_t>(s.layer);
      if (!s.plane_off.empty() && s.plane_off[0] != kNoOff)
        check(cudaMemcpyAsync(F(s.plane_off[0]), LG(loss_grad_at_[li]),
                              g_.batch() * static_cast<u64>(loss_classes_[li]) * es_, cudaMemcpyDeviceToDevice, cs_),
              "loss grad copy");
      break;
    }
    default:
      break;
  }
  if (!probes_.empty()) probe_copy(s.ev, true);
  if (timed_) check(cudaEventRecord(ev_[2 * s.ev + 1], cs_), "record");
  if (!s.prefetches.empty())  // prefetches launched here land before the next BWD
    check(cudaStreamWaitEvent(cs_, xfer_ev_[static_cast<size_t>(s.prefetches.back().ev)], 0), "wait");
  if (s.ev == input_idle_after_) check(cudaEventRecord(input_idle_ev_, cs_), "record");
}

void Session::step(float lr, float* loss_host) {
  if (host_bytes_ > 0 && !host_)
    throw PlanError(Err::Config, "the plan offloads but no offload buffer is set (set_offload_buffer / spill_attach)");
  timed_ = o_.record_timeline && !timeline_paused_;
  vdnnk::set_precise(o_.precise);
  if (sm_reserve_ < 0) {
    // Compressed transfers run on the SMs concurrently with the persistent
    // conv kernels: leave them 16 SMs (VGG-16 b256 dyn, interleaved A/B of
    // 0/8/16/24: dynt 1,468 -> 1,697 img/s, dynz 1,013 -> 1,118 at 16).
    // Same tiles, same accumulation order: results are unchanged.
    bool zvc = false;
    for (const FwdStep& f : fwd_)
      for (const Transfer& t : f.offloads) zvc = zvc || t.zvc;
    sm_reserve_ = std::getenv("VDNN_SM_RESERVE") ? 0 : (zvc ? 16 : 0);
  }
  vdnnk::set_sm_reserve(std::getenv("VDNN_SM_RESERVE") ? -1 : sm_reserve_);
  if (timed_ && !o_.cuda_graph) {  // this step records into the set the step before last used (see session.h)
    std::swap(ev_, ev_prev_);
    std::swap(t0_ev_, t0_ev_prev_);
    std::swap(ev_iter_, ev_iter_prev_);
  }
  if (has_staged_) {  // the batch prefetch_batch_host put in the INPUT extent (+ its labels) has landed
    check(cudaStreamWaitEvent(cs_, staged_ready_, 0), "wait");
    check(cudaMemcpyAsync(labels_, labels_next_, static_cast<u64>(g_.batch()) * 4, cudaMemcpyDeviceToDevice, cs_),
          "labels D2D");
    has_staged_ = false;
  }
  if (!o_.cuda_graph || eager_steps_ < 1) {
    try {
      enqueue_step(lr);
    } catch (...) {
      probes_.clear();
      throw;
    }
    probes_.clear();  // one-shot
    ++eager_steps_;
  } else {
    bool captured_now = false;
    if (!gexec_ || lr != graph_lr_) {
      captured_now = true;
      if (gexec_) cudaGraphExecDestroy(gexec_);
      gexec_ = nullptr;
      const u64 c0 = copy_off_, c1 = copy_pre_, r0 = raw_off_, r1 = raw_pre_, l0 = vdnnk::launch_count();
      cudaGraph_t graph = nullptr;
      check(cudaStreamBeginCapture(cs_, cudaStreamCaptureModeThreadLocal), "begin capture");
      try {
        enqueue_step(lr);
      } catch (...) {
        cudaStreamEndCapture(cs_, &graph);
        if (graph) cudaGraphDestroy(graph);
        throw;
      }
      check(cudaStreamEndCapture(cs_, &graph), "end capture");
      const cudaError_t e = cudaGraphInstantiate(&gexec_, graph, 0);
      cudaGraphDestroy(graph);
      check(e, "graph instantiate");
      graph_lr_ = lr;
      g_copy_off_ = copy_off_ - c0;
      g_copy_pre_ = copy_pre_ - c1;
      g_raw_off_ = raw_off_ - r0;
      g_raw_pre_ = raw_pre_ - r1;
      g_launches_ = vdnnk::launch_count() - l0;
      copy_off_ = c0, copy_pre_ = c1, raw_off_ = r0, raw_pre_ = r1;  // re-added per launch below
    }
    check(cudaGraphLaunch(gexec_, cs_), "graph launch");
    copy_off_ += g_copy_off_;
    copy_pre_ += g_copy_pre_;
    raw_off_ += g_raw_off_;
    raw_pre_ += g_raw_pre_;
    // the captured kernels were counted while capturing; every later replay launches them again
    if (captured_now) captured_now = false;
    else vdnnk::count_launch(g_launches_);
  }
  if (loss_host) {
    check(cudaMemcpyAsync(pinned_loss_, loss_, 4, cudaMemcpyDeviceToHost, cs_), "loss D2H");
    check(cudaStreamSynchronize(cs_), "sync");
    *loss_host = *pinned_loss_;
  }
}

void Session::transfer_stats(u64* offload_wire, u64* prefetch_wire, u64* offload_raw, u64* prefetch_raw) {
  synchronize();
  unsigned long long w[2] = {0, 0};
  check(cudaMemcpy(w, wire_, sizeof(w), cudaMemcpyDeviceToHost), "wire counters");
  if (offload_wire) *offload_wire = w[0] + copy_off_;
  if (prefetch_wire) *prefetch_wire = w[1] + copy_pre_;
  if (offload_raw) *offload_raw = raw_off_;
  if (prefetch_raw) *prefetch_raw = raw_pre_;
}

void Session::synchronize() {
  check(cudaStreamSynchronize(ms_), "sync");
  check(cudaStreamSynchronize(cs_), "sync");
}

void Session::set_batch_host(const float* images, const int32_t* labels) {
  const u64 bytes = df_.at[static_cast<size_t>(input_id_)].bytes;
  if (images) check(cudaMemcpyAsync(F(x_off_), images, bytes, cudaMemcpyHostToDevice, cs_), "images H2D");
  if (labels) check(cudaMemcpyAsync(labels_, labels, g_.batch() * 4, cudaMemcpyHostToDevice, cs_), "labels H2D");
}

void Session::set_batch_device(const float* images, const int32_t* labels) {
  const u64 bytes = df_.at[static_cast<size_t>(input_id_)].bytes;
  if (images) check(cudaMemcpyAsync(F(x_off_), images, bytes, cudaMemcpyDeviceToDevice, cs_), "images D2D");
  if (labels) check(cudaMemcpyAsync(labels_, labels, g_.batch() * 4, cudaMemcpyDeviceToDevice, cs_), "labels D2D");
}

void Session::prefetch_batch_host(const float* images, const int32_t* labels) {
  const u64 bytes = df_.at[static_cast<size_t>(input_id_)].bytes;
  const u64 lbytes = static_cast<u64>(g_.batch()) * 4;
  if (has_staged_) throw PlanError(Err::Generic, "a prefetched batch is already waiting for the next step");
  if (inputs_.size() != 1) throw PlanError(Err::Config, "prefetch_batch_host needs a graph with one INPUT layer");
  if (!in_stream_) {
    check(cudaStreamCreateWithFlags(&in_stream_, cudaStreamNonBlocking), "stream");
    check(cudaEventCreateWithFlags(&staged_ready_, cudaEventDisableTiming), "event");
  }
  // the last enqueued step records input_idle_ev_ once nothing it runs
  // touches the INPUT extent any more (or at its end); the previous staged
  // labels were consumed at that step's start
  check(cudaStreamWaitEvent(in_stream_, input_idle_ev_, 0), "wait");
  if (images) check(cudaMemcpyAsync(F(x_off_), images, bytes, cudaMemcpyHostToDevice, in_stream_), "images H2D");
  if (labels) {
    check(cudaMemcpyAsync(labels_next_, labels, lbytes, cudaMemcpyHostToDevice, in_stream_), "labels H2D");
  } else {
    check(cudaMemcpyAsync(labels_next_, labels_, lbytes, cudaMemcpyDeviceToDevice, in_stream_), "labels keep");
  }
  check(cudaEventRecord(staged_ready_, in_stream_), "record");
  has_staged_ = true;
}

int64_t Session::queue_loss() {
  if (!loss_ring_) {
    check(cudaHostAlloc(&loss_ring_, kLossRing * sizeof(float), cudaHostAllocDefault), "cudaHostAlloc(loss ring)");
    for (auto& e : loss_ev_) check(cudaEventCreateWithFlags(&e, cudaEventDisableTiming), "event");
  }
  const int64_t t = loss_tickets_++;
  const int slot = static_cast<int>(t % kLossRing);
  check(cudaMemcpyAsync(loss_ring_ + slot, loss_, 4, cudaMemcpyDeviceToHost, cs_), "loss D2H");
  check(cudaEventRecord(loss_ev_[slot], cs_), "record");
  return t;
}

float Session::wait_loss(int64_t ticket) {
  if (ticket < 0 || ticket >= loss_tickets_ || ticket < loss_tickets_ - kLossRing)
    throw PlanError(Err::Generic, "loss ticket out of range (at most 4 outstanding)");
  const int slot = static_cast<int>(ticket % kLossRing);
  check(cudaEventSynchronize(loss_ev_[slot]), "sync");
  return loss_ring_[slot];
}

// One iteration's stream work (both streams; in graph mode this is what gets captured).
void Session::enqueue_step(float lr) {
  if (timed_) check(cudaEventRecord(ev_iter_, cs_), "record");
  // the memory stream never runs ahead into a new iteration
  check(cudaEventRecord(ev_sync_, cs_), "record");
  check(cudaStreamWaitEvent(ms_, ev_sync_, 0), "wait");
  for (const FwdStep& s : fwd_) run_fwd(s, lr);
  for (const BwdStep& s : bwd_) run_bwd(s, lr);
  if (peer_inline_) peer_finish();
  if (input_idle_after_ < 0) check(cudaEventRecord(input_idle_ev_, cs_), "record");
}

float Session::read_loss() {
  check(cudaMemcpyAsync(pinned_loss_, loss_, 4, cudaMemcpyDeviceToHost, cs_), "loss D2H");
  check(cudaStreamSynchronize(cs_), "sync");
  return *pinned_loss_;
}

void Session::synthetic_batch(u64 seed) {
  for (size_t i = 0; i < inputs_.size(); ++i) {
    const u64 count = df_.at[static_cast<size_t>(inputs_[i])].bytes / es_;
    const u64 sd = seed + 7919 * i;
    check(bf_ ? vdnnk::fill_uniform_bf16(F(input_off_[i]), count, -1.0f, 1.0f, sd, cs_)
              : vdnnk::fill_uniform(F(input_off_[i]), count, -1.0f, 1.0f, sd, cs_),
          "images");
  }
  check(vdnnk::fill_labels(labels_, g_.batch(), classes_, seed + 1, cs_), "labels");
}

void Session::set_input(int layer, const float* images, bool device) {
  for (size_t i = 0; i < inputs_.size(); ++i) {
    if (inputs_[i] != layer) continue;
    const u64 bytes = df_.at[static_cast<size_t>(layer)].bytes;
    check(cudaMemcpyAsync(F(input_off_[i]), images, bytes, device ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice,
                          cs_),
          "images");
    return;
  }
  throw PlanError(Err::Generic, "set_input: not an INPUT layer");
}

void Session::get_weights(int layer, float* host, size_t count) {
  if (layer < 0 || layer >= L_ || w_off_[static_cast<size_t>(layer)] == kNoOff)
    throw PlanError(Err::Generic, "layer has no weights");
  if (count * es_ != df_.at[static_cast<size_t>(layer)].w_bytes) throw PlanError(Err::Generic, "weight count mismatch");
  synchronize();
  read_device(host, F(w_off_[static_cast<size_t>(layer)]), count);
}

void Session::set_weights(int layer, const float* host, size_t count) {
  if (layer < 0 || layer >= L_ || w_off_[static_cast<size_t>(layer)] == kNoOff)
    throw PlanError(Err::Generic, "layer has no weights");
  if (count * es_ != df_.at[static_cast<size_t>(layer)].w_bytes) throw PlanError(Err::Generic, "weight count mismatch");
  synchronize();
  if (!bf_) {
    check(cudaMemcpy(F(w_off_[static_cast<size_t>(layer)]), host, count * 4, cudaMemcpyHostToDevice), "H2D");
    return;
  }
  std::vector<uint16_t> b(count);
  for (size_t i = 0; i < count; ++i) b[i] = to_bf16_bits(host[i]);
  check(cudaMemcpy(F(w_off_[static_cast<size_t>(layer)]), b.data(), count * 2, cudaMemcpyHostToDevice), "H2D");
}

void Session::read_feature(int owner, float* host, size_t count) {
  // valid only for buffers still device-resident at the end of the step
  // (e.g. the INPUT extent or any buffer in the baseline scheme)
  synchronize();
  u64 off = kNoOff;
  for (const Event& e : plan_.events)
    if (e.kind == Ev::Alloc && e.buffer == owner && (e.tag == "X" || e.tag == "Y")) off = e.off;
  if (off == kNoOff) throw PlanError(Err::Generic, "owner has no feature buffer");
  if (count * es_ > df_.at[static_cast<size_t>(owner)].bytes) throw PlanError(Err::Generic, "count too large");
  read_device(host, F(off), count);
}

Session::ProbeLayout Session::probe_layout(int layer, bool bwd) const {
  if (layer < 0 || layer >= L_) throw PlanError(Err::Generic, "probe: layer out of range");
  ProbeLayout p;
  const Node& l = g_.at(layer);
  const size_t li = static_cast<size_t>(layer);
  auto add = [&](int what, int index, u64 bytes, int src, u64 src_off, bool after) {
    if (bytes == 0) return;
    ProbeSeg s;
    s.what = what, s.index = index, s.dst = p.total, s.bytes = bytes, s.src = src, s.src_off = src_off, s.after = after;
    p.segs.push_back(s);
    p.total += round_up(bytes, 256);
  };
  auto in_bytes = [&](size_t i) { return g_.dims(l.in[i]).count() * es_; };
  const u64 y_bytes = g_.dims(layer).count() * es_;
  const bool contraction = l.kind == Kind::Conv || l.kind == Kind::Fc;
  if (!bwd) {
    const FwdStep* s = nullptr;
    for (const FwdStep& f : fwd_)
      if (f.layer == layer) s = &f;
    if (!s) throw PlanError(Err::Generic, "probe: layer has no FWD step");
    p.relu = s->relu ? 1 : 0;
    p.skip = s->skip ? 1 : 0;
    for (size_t i = 0; i < s->in_off.size(); ++i)
      if (l.kind != Kind::Actv) add(kPX, static_cast<int>(i), in_bytes(i), 0, s->in_off[i], false);
    if (contraction) add(kPW, 0, df_.at[li].w_bytes, 0, s->w_off, false);
    if (l.kind == Kind::Actv) add(kPX, 0, y_bytes, 0, s->out_off, false);
    if (l.kind == Kind::Loss) {
      add(kPLossGrad, 0, g_.batch() * static_cast<u64>(loss_classes_[li]) * es_, 2, loss_grad_at_[li], true);
      add(kPLoss, 0, 4, 3, 0, true);
    } else {
      add(kPY, 0, y_bytes, 0, s->out_off, true);
    }
    return p;
  }
  const BwdStep* s = nullptr;
  for (const BwdStep& b : bwd_)
    if (b.layer == layer) s = &b;
  if (!s) throw PlanError(Err::Generic, "probe: layer has no BWD step");
  p.accumulate = s->accumulate ? 1 : 0;
  p.skip = s->skip ? 1 : 0;
  for (size_t i = 0; i < s->mask_plane.size(); ++i)
    if (s->mask_plane[i]) p.mask |= 1u << i;
  if (l.kind == Kind::Actv) {
    add(kPY, 0, y_bytes, 0, s->out_off, false);
    for (size_t k = 0; k < s->dy_off.size(); ++k) add(kPDY, static_cast<int>(k), y_bytes, 0, s->dy_off[k], false);
    if (!s->dy_off.empty()) add(kPDX, 0, y_bytes, 0, s->priv_out != kNoOff ? s->priv_out : s->dy_off[0], true);
    return p;
  }
  if (l.kind == Kind::Conv || l.kind == Kind::Fc || l.kind == Kind::Pool)
    for (size_t i = 0; i < s->in_off.size(); ++i) add(kPX, static_cast<int>(i), in_bytes(i), 0, s->in_off[i], false);
  if (contraction) add(kPW, 0, df_.at[li].w_bytes, 0, s->w_off, false);
  if (s->stage_dy) {  // shared planes stay as they are: every incoming plane (the kernels read their sum)
    for (size_t k = 0; k < s->dy_off.size(); ++k) add(kPDY, static_cast<int>(k), y_bytes, 0, s->dy_off[k], false);
  } else if (!s->dy_off.empty()) {
    add(kPDY, 0, y_bytes, 0, s->dy_off[0], false);  // after the fold of the other planes
  }
  for (size_t i = 0; i < s->plane_off.size(); ++i) {
    if (s->plane_off[i] == kNoOff) continue;
    const u64 b = l.kind == Kind::Loss ? g_.dims(l.in[0]).count() * es_ : in_bytes(i);
    if (s->accumulate) add(kPDXBefore, static_cast<int>(i), b, 0, s->plane_off[i], false);
    add(kPDX, static_cast<int>(i), b, 0, s->plane_off[i], true);
  }
  if (contraction && grads_) add(kPDW, 0, df_.at[li].w_bytes / es_ * 4, 1, grad_off_[li], true);  // fp32
  if (contraction && !grads_) add(kPW, 1, df_.at[li].w_bytes, 0, s->w_off, true);  // updated weights
  return p;
}

void Session::arm_probe(int layer, bool bwd, void* dst, u64 bytes) {
  if (o_.cuda_graph) throw PlanError(Err::Config, "probes are not available in cuda_graph mode");
  ArmedProbe a;
  a.lay = probe_layout(layer, bwd);
  if (!dst || bytes < a.lay.total) throw PlanError(Err::Generic, "probe: destination buffer too small");
  a.dst = static_cast<char*>(dst);
  if (!bwd) {
    for (const FwdStep& f : fwd_)
      if (f.layer == layer) a.ev = f.ev;
  } else {
    for (const BwdStep& b : bwd_)
      if (b.layer == layer) a.ev = b.ev;
  }
  probes_.push_back(std::move(a));
}

void Session::probe_copy(int ev, bool after) {
  for (const ArmedProbe& a : probes_) {
    if (a.ev != ev) continue;
    for (const ProbeSeg& s : a.lay.segs) {
      if (s.after != after) continue;
      const char* src = nullptr;
      switch (s.src) {
        case 0: src = base_ + s.src_off; break;
        case 1: src = reinterpret_cast<const char*>(grads_ + s.src_off); break;
        case 2: src = static_cast<const char*>(LG(s.src_off)); break;
        default: src = reinterpret_cast<const char*>(loss_); break;
      }
      check(cudaMemcpyAsync(a.dst + s.dst, src, s.bytes, cudaMemcpyDefault, cs_), "probe copy");
    }
  }
}

void Session::grad_buffer(int layer, void** ptr, size_t* count) {
  if (!grads_ || layer < 0 || layer >= L_ || grad_off_[static_cast<size_t>(layer)] == kNoOff) {
    *ptr = nullptr;
    *count = 0;
    return;
  }
  *ptr = grads_ + grad_off_[static_cast<size_t>(layer)];
  *count = df_.at[static_cast<size_t>(layer)].w_bytes / es_;
}

void Session::grad_arena(void** ptr, size_t* count) {
  *ptr = grads_;
  *count = grads_count_;
}

void Session::set_grad_arena(float* ptr, size_t count) {
  if (!o_.external_grads) throw PlanError(Err::Generic, "session was created without external_grads");
  if (!ptr || count < grads_count_) throw PlanError(Err::Generic, "gradient arena too small");
  synchronize();
  drop_graph();
  if (grads_ && grads_owned_) cudaFree(grads_);
  grads_ = ptr;
  grads_owned_ = false;
}

void Session::apply_grads(float lr, float scale) {
  if (!grads_) throw PlanError(Err::Generic, "session was created without external_grads");
  for (int i = 0; i < L_; ++i) {
    const size_t k = static_cast<size_t>(i);
    if (grad_off_[k] == kNoOff) continue;
    const size_t n = df_.at[k].w_bytes / es_;
    check(bf_ ? vdnnk::sgd_update_bf16(F(w_off_[k]), grads_ + grad_off_[k], lr * scale, n, cs_)
              : vdnnk::sgd_update(F(w_off_[k]), grads_ + grad_off_[k], lr * scale, n, cs_),
          "sgd");
  }
}

// ------------------------------------------------------ measured report ----
// Re-times the plan's event log with the CUDA-event measurements of the last
// step. Per step: T0 = compute stream reaches the step (after the previous
// step's sync waits), KS/KE = kernel group start/end, XS/XE = transfer
// start/end. The non-timed rows take the simulator's anchors
// (simulator.hpp:279-350 forward, :364-468 backward, :513-545 cleanup) on
// these measured times, so the result can be replay-checked like a plan.
vdnnp::Report Session::measured_report() const {
  if (ev_.empty()) throw PlanError(Err::Generic, "session was created without record_timeline");
  auto ns = [&](cudaEvent_t e) -> i64 {
    float ms = 0.f;
    if (cudaEventElapsedTime(&ms, ev_iter_, e) != cudaSuccess) {
      cudaGetLastError();  // do not leave a stale error for the next launch check
      return 0;
    }
    return std::max<i64>(0, static_cast<i64>(std::llround(static_cast<double>(ms) * 1e6)));
  };
  const size_t nst = fwd_.size() + bwd_.size();
  const size_t nx = ev_.size() / 2 - nst;
  std::vector<i64> t0(nst), ks(nst), ke(nst), xs(nx), xe(nx);
  for (size_t i = 0; i < nst; ++i) {
    t0[i] = ns(t0_ev_[i]);
    ks[i] = std::max(t0[i], ns(ev_[2 * i]));
    ke[i] = std::max(ks[i], ns(ev_[2 * i + 1]));
  }
  for (size_t i = 0; i < nx; ++i) {
    xs[i] = ns(ev_[2 * (nst + i)]);
    xe[i] = std::max(xs[i], ns(ev_[2 * (nst + i) + 1]));
  }
  vdnnp::Report r;
  r.pass = true;
  size_t fi = 0, bi = 0;
  size_t xi = 0;
  int cur = -1;          // step index of the current FWD/BWD group
  bool bwd = false;
  i64 horizon = 0;
  std::map<int, i64> off_end;
  // the step an event belongs to is the next FWD/BWD row at or after it for
  // ALLOC/PREFETCH (they precede their kernel), the last one for the rest
  auto next_step = [&]() -> int {
    if (!bwd && fi < fwd_.size()) return fwd_[fi].ev;
    if (bi < bwd_.size()) return bwd_[bi].ev;
    return cur;
  };
  // SYNC rows are measured, not copied from the plan (the planner's model
  // stalls at other steps than the B200 does): the compute stream's waits
  // under the reference's sync rules (simulator.hpp:315-322 forward: FWD(n+1)
  // after n's offloads; :400-441 backward: BWD(m) after the prefetches it
  // reads, and after the prefetches launched during BWD(m)), i.e. the gaps
  // kernel end -> next step start and step start -> kernel start.
  auto sync_row = [&](int layer, i64 a, i64 b, bool backward) {
    if (b <= a) return;
    Event e;
    e.kind = Ev::Sync;
    e.lane = Lane::Compute;
    e.layer = layer;
    e.t0 = a;
    e.t1 = b;
    (backward ? r.stall_bwd : r.stall_fwd) += b - a;
    horizon = std::max(horizon, b);
    r.events.push_back(e);
  };
  const int nsteps = static_cast<int>(nst);
  auto next_t0 = [&](int st) { return st + 1 < nsteps ? t0[static_cast<size_t>(st + 1)] : ke[static_cast<size_t>(st)]; };
  int fwd_sync_step = -1;   // forward step with offloads whose post-kernel wait is not emitted yet
  int bwd_tail_step = -1;   // backward step with prefetches: same, after its BWD row
  int bwd_pre_done = -1;    // backward step whose pre-kernel wait was emitted
  for (size_t k = 0; k < plan_.events.size(); ++k) {
    const Event& pe = plan_.events[k];
    Event e = pe;
    if (!bwd && pe.kind == Ev::Prefetch) bwd = true;
    if (!bwd && pe.kind == Ev::Bwd) bwd = true;
    if (!bwd && pe.kind == Ev::Alloc && pe.lane == Lane::Memory) bwd = true;
    if (pe.kind == Ev::Sync) continue;
    if (fwd_sync_step >= 0 && pe.kind != Ev::Offload) {
      const size_t st = static_cast<size_t>(fwd_sync_step);
      sync_row(prog_.steps[st].layer, ke[st], next_t0(fwd_sync_step), false);
      fwd_sync_step = -1;
    }
    if (bwd_tail_step >= 0 && pe.kind != Ev::Bwd) {
      const size_t st = static_cast<size_t>(bwd_tail_step);
      sync_row(prog_.steps[st].layer, ke[st], next_t0(bwd_tail_step), true);
      bwd_tail_step = -1;
    }
    if (bwd && bi < bwd_.size() && (pe.kind == Ev::Bwd || (pe.kind == Ev::Alloc && pe.lane == Lane::Compute)) &&
        bwd_pre_done != bwd_[bi].ev) {
      const BwdStep& b = bwd_[bi];
      bwd_pre_done = b.ev;
      if (!b.wait_prefetch.empty())
        sync_row(b.layer, t0[static_cast<size_t>(b.ev)], ks[static_cast<size_t>(b.ev)], true);
    }
    switch (pe.kind) {
      case Ev::Fwd:
        if (!fwd_[fi].offloads.empty()) fwd_sync_step = fwd_[fi].ev;
        cur = fwd_[fi++].ev;
        e.t0 = ks[static_cast<size_t>(cur)];
        e.t1 = ke[static_cast<size_t>(cur)];
        break;
      case Ev::Bwd:
        if (!bwd_[bi].prefetches.empty()) bwd_tail_step = bwd_[bi].ev;
        cur = bwd_[bi++].ev;
        e.t0 = ks[static_cast<size_t>(cur)];
        e.t1 = ke[static_cast<size_t>(cur)];
        break;
      case Ev::Offload:
      case Ev::Prefetch:
        e.t0 = xs[xi];
        e.t1 = xe[xi];
        ++xi;
        if (pe.kind == Ev::Offload) off_end[pe.buffer] = e.t1;
        break;
      case Ev::Alloc: {
        if (pe.t0 == 0 && fi == 0 && !bwd) {
          e.t0 = e.t1 = 0;  // setup
        } else {
          const int st = next_step();
          // forward / prefetch allocations at the step's T0; backward dX/WS/dW at kernel start
          const bool at_ready = bwd && pe.lane == Lane::Compute;
          e.t0 = e.t1 = at_ready ? ks[static_cast<size_t>(st)] : t0[static_cast<size_t>(st)];
        }
        break;
      }
      case Ev::Release: {
        if (pe.layer < 0) {
          e.t0 = e.t1 = horizon;  // cleanup
        } else if (pe.lane == Lane::Memory) {
          const i64 oe = off_end.count(pe.buffer) ? off_end[pe.buffer] : 0;
          e.t0 = e.t1 = std::max(ke[static_cast<size_t>(cur)], oe);
        } else {
          e.t0 = e.t1 = ke[static_cast<size_t>(cur)];
        }
        break;
      }
      case Ev::Sync:
        break;
    }
    if (pe.kind != Ev::Release || pe.layer >= 0) horizon = std::max(horizon, e.t1);
    r.events.push_back(e);
  }
  r.total = horizon;
  // pool high water / time-weighted average reconstructed from the re-timed log
  u64 live = 0, peak = 0;
  vdnnp::u128 area = 0;
  i64 last = 0;
  for (const Event& e : r.events) {
    if (e.kind != Ev::Alloc && e.kind != Ev::Release) continue;
    area += static_cast<vdnnp::u128>(live) * static_cast<vdnnp::u128>(std::max<i64>(0, e.t0 - last));
    last = std::max(last, e.t0);
    if (e.kind == Ev::Alloc) {
      live += round_up(e.bytes, kAlign);
      peak = std::max(peak, live);
    } else {
      live -= round_up(e.bytes, kAlign);
    }
  }
  if (r.total > last) area += static_cast<vdnnp::u128>(live) * static_cast<vdnnp::u128>(r.total - last);
  r.max_mem = peak;
  r.avg_mem = r.total > 0 ? static_cast<u64>(area / static_cast<vdnnp::u128>(r.total)) : 0;
  r.offload_bytes = plan_.offload_bytes;
  r.prefetch_bytes = plan_.prefetch_bytes;
  r.host_peak = plan_.host_peak;
  r.interference = plan_.interference;
  r.reuse.assign(static_cast<size_t>(L_), -1);
  std::vector<i64> fe(static_cast<size_t>(L_), -1), bs(static_cast<size_t>(L_), -1);
  for (const Event& e : r.events) {
    if (e.kind == Ev::Fwd) fe[static_cast<size_t>(e.layer)] = e.t1;
    if (e.kind == Ev::Bwd) bs[static_cast<size_t>(e.layer)] = e.t0;
  }
  for (size_t i = 0; i < static_cast<size_t>(L_); ++i)
    if (fe[i] >= 0 && bs[i] >= 0) r.reuse[i] = bs[i] - fe[i];
  return r;
}

void Session::layer_times(int n, double* fwd_ms, double* bwd_ms) const {
  if (ev_.empty()) throw PlanError(Err::Generic, "session was created without record_timeline");
  for (int i = 0; i < n; ++i) {
    if (fwd_ms) fwd_ms[i] = 0;
    if (bwd_ms) bwd_ms[i] = 0;
  }
  auto el = [&](size_t k) {
    float ms = 0.f;
    if (cudaEventElapsedTime(&ms, ev_[2 * k], ev_[2 * k + 1]) != cudaSuccess) {
      cudaGetLastError();
      return 0.0;
    }
    return static_cast<double>(ms);
  };
  for (const FwdStep& s : fwd_)
    if (s.layer < n && fwd_ms) fwd_ms[s.layer] = el(static_cast<size_t>(s.ev));
  for (const BwdStep& s : bwd_)
    if (s.layer < n && bwd_ms) bwd_ms[s.layer] = el(static_cast<size_t>(s.ev));
}

}  // namespace vdnnrt
