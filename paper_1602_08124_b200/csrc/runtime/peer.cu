// Data-parallel gradient exchange over peer memory (see kernels/peer.cu).
//
// Every rank runs the identical plan (deterministic planner,
// per-rank batch), so every weight sits at the same pool offset in every
// rank's arena and every gradient at the same index of every rank's gradient
// arena. The flat gradient index space is cut into chunks (per layer, at most
// kChunk floats, boundaries on 4-float multiples) dealt round-robin to the
// ranks; rank r reduces its chunks from all N gradient arenas, updates the
// weights and writes them into all N arenas.
#include <cstring>
#include <string>

#include "session.h"

namespace vdnnrt {

using vdnnp::Err;
using vdnnp::PlanError;

namespace {
constexpr uint32_t kChunk = 16384;  // floats per work item (64 KB of gradient)
}

Session::PeerHandle Session::peer_export() {
  if (!o_.external_grads || !grads_ || !grads_owned_)
    throw PlanError(Err::Generic, "peer exchange needs external_grads with the session-owned gradient arena");
  if (!signal_) {
    check(cudaMalloc(&signal_, 2 * vdnnk::kPeerMaxRanks * sizeof(unsigned long long)), "cudaMalloc(peer signal)");
    check(cudaMemset(signal_, 0, 2 * vdnnk::kPeerMaxRanks * sizeof(unsigned long long)), "memset(peer signal)");
  }
  PeerHandle h{};
  check(cudaIpcGetMemHandle(&h.arena, arena_), "cudaIpcGetMemHandle(arena)");
  check(cudaIpcGetMemHandle(&h.grads, grads_), "cudaIpcGetMemHandle(grads)");
  check(cudaIpcGetMemHandle(&h.signal, signal_), "cudaIpcGetMemHandle(signal)");
  h.arena_lo = arena_lo_;
  h.arena_bytes = arena_bytes_;
  h.grads_count = grads_count_;
  return h;
}

void Session::peer_attach(int rank, int world, const PeerHandle* all) {
  if (world < 1 || world > vdnnk::kPeerMaxRanks || rank < 0 || rank >= world)
    throw PlanError(Err::Generic, "peer_attach: rank/world out of range (1..8 ranks)");
  if (!signal_) peer_export();  // allocates the signal words
  peer_detach();
  synchronize();
  for (int p = 0; p < world; ++p) {
    const PeerHandle& h = all[p];
    if (h.arena_lo != arena_lo_ || h.arena_bytes != arena_bytes_ || h.grads_count != grads_count_)
      throw PlanError(Err::Generic, "peer_attach: rank " + std::to_string(p) +
                                        " runs a different plan (arena/gradient layout differs)");
  }
  vdnnk::PeerArgs a{};
  a.world = world;
  a.rank = rank;
  a.bf16 = bf_ ? 1 : 0;
  try {
    for (int p = 0; p < world; ++p) {
      if (p == rank) {
        a.arena[p] = base_;
        a.grads[p] = grads_;
        a.signal[p] = signal_;
        continue;
      }
      void* m = nullptr;
      check(cudaIpcOpenMemHandle(&m, all[p].arena, cudaIpcMemLazyEnablePeerAccess), "cudaIpcOpenMemHandle(arena)");
      peer_maps_.push_back(m);
      a.arena[p] = static_cast<char*>(m) - arena_lo_;
      check(cudaIpcOpenMemHandle(&m, all[p].grads, cudaIpcMemLazyEnablePeerAccess), "cudaIpcOpenMemHandle(grads)");
      peer_maps_.push_back(m);
      a.grads[p] = static_cast<const float*>(m);
      check(cudaIpcOpenMemHandle(&m, all[p].signal, cudaIpcMemLazyEnablePeerAccess),
            "cudaIpcOpenMemHandle(signal)");
      peer_maps_.push_back(m);
      a.signal[p] = static_cast<unsigned long long*>(m);
    }
  } catch (...) {
    peer_detach();
    throw;
  }

  // this rank's share of the chunks (contiguous per layer)
  std::vector<vdnnk::PeerChunk> mine;
  peer_first_.assign(static_cast<size_t>(L_), 0);
  peer_count_.assign(static_cast<size_t>(L_), 0);
  uint64_t j = 0;
  for (int i = 0; i < L_; ++i) {
    const size_t k = static_cast<size_t>(i);
    peer_first_[k] = static_cast<int>(mine.size());
    if (grad_off_[k] == kNoOff) continue;
    const uint64_t n = df_.at[k].w_bytes / es_;
    for (uint64_t s = 0; s < n; s += kChunk, ++j) {
      if (static_cast<int>(j % static_cast<uint64_t>(world)) != rank) continue;
      vdnnk::PeerChunk c{};
      c.w_off = w_off_[k] + es_ * s;
      c.g_off = grad_off_[k] + s;
      c.count = static_cast<uint32_t>(std::min<uint64_t>(kChunk, n - s));
      mine.push_back(c);
    }
    peer_count_[k] = static_cast<int>(mine.size()) - peer_first_[k];
  }
  if (!mine.empty()) {
    check(cudaMalloc(&peer_chunks_, mine.size() * sizeof(vdnnk::PeerChunk)), "cudaMalloc(peer chunks)");
    check(cudaMemcpy(peer_chunks_, mine.data(), mine.size() * sizeof(vdnnk::PeerChunk), cudaMemcpyHostToDevice),
          "H2D(peer chunks)");
  }
  a.chunks = peer_chunks_;
  a.nchunks = static_cast<int>(mine.size());
  peer_ = a;
  peer_world_ = world;
}

void Session::peer_exchange(float lr, float scale) {
  if (peer_world_ == 0) throw PlanError(Err::Generic, "peer_exchange: call peer_attach first");
  ++peer_epoch_;
  peer_.step = lr * scale;
  check(vdnnk::peer_barrier(peer_, peer_epoch_, 0, cs_), "peer barrier (pre)");
  check(vdnnk::peer_reduce_sgd(peer_, cs_), "peer reduce+sgd");
  check(vdnnk::peer_barrier(peer_, peer_epoch_, 1, cs_), "peer barrier (post)");
}

void Session::peer_overlap(bool on, float scale) {
  if (on && peer_world_ == 0) throw PlanError(Err::Generic, "peer_overlap: call peer_attach first");
  if (on && o_.cuda_graph)
    throw PlanError(Err::Config, "peer_overlap: the in-step exchange's barrier epochs are per step (no CUDA graph)");
  synchronize();
  if (on && !xs_) {
    check(cudaStreamCreateWithFlags(&xs_, cudaStreamNonBlocking), "stream");
    check(cudaEventCreateWithFlags(&xs_done_, cudaEventDisableTiming), "event");
    wg_ev_.assign(static_cast<size_t>(L_), nullptr);
    for (int i = 0; i < L_; ++i)
      if (grad_off_[static_cast<size_t>(i)] != kNoOff)
        check(cudaEventCreateWithFlags(&wg_ev_[static_cast<size_t>(i)], cudaEventDisableTiming), "event");
  }
  peer_inline_ = on;
  peer_scale_ = scale;
}

// One layer's share: every rank's dW(layer) is complete (pre barrier), then
// reduce + SGD + broadcast of this rank's chunks of that layer. Every rank
// enqueues the same layers in the same (backward) order, so the barrier
// epochs match.
void Session::peer_layer(int layer, float lr) {
  const size_t k = static_cast<size_t>(layer);
  check(cudaEventRecord(wg_ev_[k], cs_), "record");
  check(cudaStreamWaitEvent(xs_, wg_ev_[k], 0), "wait");
  vdnnk::PeerArgs a = peer_;
  a.step = lr * peer_scale_;
  a.chunks = peer_chunks_ ? peer_chunks_ + peer_first_[k] : nullptr;
  a.nchunks = peer_count_[k];
  check(vdnnk::peer_barrier(a, ++peer_epoch_, 0, xs_), "peer barrier (layer)");
  check(vdnnk::peer_reduce_sgd(a, xs_), "peer reduce+sgd (layer)");
}

// Every rank finished every layer (its weights are written everywhere, its
// gradients read by everyone) before any rank's next step; the compute stream
// joins the exchange stream.
void Session::peer_finish() {
  check(vdnnk::peer_barrier(peer_, ++peer_epoch_, 1, xs_), "peer barrier (post)");
  check(cudaEventRecord(xs_done_, xs_), "record");
  check(cudaStreamWaitEvent(cs_, xs_done_, 0), "wait");
}

void Session::peer_detach() {
  if (peer_world_ == 0 && peer_maps_.empty() && !peer_chunks_) return;
  if (cs_) cudaStreamSynchronize(cs_);
  if (xs_) cudaStreamSynchronize(xs_);  // in-step exchanges still reading the mappings
  drop_graph();
  for (void* m : peer_maps_) cudaIpcCloseMemHandle(m);
  peer_maps_.clear();
  if (peer_chunks_) cudaFree(peer_chunks_);
  peer_chunks_ = nullptr;
  peer_ = vdnnk::PeerArgs{};
  peer_world_ = 0;
  peer_inline_ = false;
}

// ------------------------------------------------ device offload target ----
void Session::set_offload_buffer(void* dev_ptr, u64 bytes) {
  if (o_.offload_target == 0) throw PlanError(Err::Config, "session offloads to the pinned host arena");
  if (!dev_ptr || bytes < host_bytes_) throw PlanError(Err::Generic, "offload buffer missing or too small");
  synchronize();
  drop_graph();
  host_ = static_cast<char*>(dev_ptr);
}

cudaIpcMemHandle_t Session::spill_export() {
  if (!spill_) {
    check(cudaMalloc(&spill_, std::max<u64>(host_bytes_, 4096)), "cudaMalloc(spill buffer)");
    scratch_bytes_ += std::max<u64>(host_bytes_, 4096);
  }
  cudaIpcMemHandle_t h;
  check(cudaIpcGetMemHandle(&h, spill_), "cudaIpcGetMemHandle(spill)");
  return h;
}

void Session::spill_attach(const cudaIpcMemHandle_t& h) {
  if (o_.offload_target == 0) throw PlanError(Err::Config, "session offloads to the pinned host arena");
  synchronize();
  drop_graph();
  if (spill_map_) cudaIpcCloseMemHandle(spill_map_);
  spill_map_ = nullptr;
  check(cudaIpcOpenMemHandle(&spill_map_, h, cudaIpcMemLazyEnablePeerAccess), "cudaIpcOpenMemHandle(spill)");
  host_ = static_cast<char*>(spill_map_);
}

}  // namespace vdnnrt
