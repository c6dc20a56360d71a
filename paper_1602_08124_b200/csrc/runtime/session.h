// B200 executor: replays a planner schedule on one device arena, a pinned
// host arena, a compute stream and a dedicated memcpy stream.
#pragma once
#include <cuda_runtime.h>

#include <cstdint>
#include <string>
#include <vector>

#include "../kernels/kernels.h"
#include "../planner/planner.hpp"

namespace vdnnrt {

using vdnnp::i64;
using vdnnp::u64;

constexpr u64 kNoOff = ~u64{0};  // "no buffer" offset
uint16_t to_bf16_bits(float f);  // round to nearest even

struct Options {
  int device = 0;
  u64 weight_seed = 5000;
  bool external_grads = false;
  bool record_timeline = false;
  bool host_arena = true;
  bool precise = false;  // 3xTF32 contractions
  // Offload / prefetch through the SMs in zero-value-compressed form
  // (kernels/zvc.cu) instead of cudaMemcpyAsync; same schedule, fewer bytes
  // on the host link. 1: lossless (every byte restored). 2: additionally,
  // maps whose only backward readers are TF32 contractions (conv/FC wgrad
  // operands) and ReLU masks travel TF32-exact (the 13 mantissa bits the
  // tensor core ignores are dropped): the training step stays bit-identical.
  int compress_offload = 0;
  // Where offloaded feature maps go: 0 = the pinned host arena (PCIe, the
  // reference's model); 1 = a device buffer set later with
  // set_offload_buffer / spill_attach (e.g. a peer GPU's spare HBM over
  // NVLink). Same schedule, same slots, same sync rules.
  int offload_target = 0;
  // Replay each training step as one CUDA graph (captured on the second
  // step, re-captured when lr changes): both streams' work, the transfers and
  // their event gating become graph nodes; one launch per step.
  bool cuda_graph = false;
  // 0: implicit GEMM for every planned conv algorithm (workspace reserved);
  // 1: GEMM_WS layers run im2col into the planned workspace + a 1x1 GEMM
  // (kernels/conv_gemmws.cu); FFT layers stay implicit
  int algo_kernels = 0;
};

struct Transfer {
  int owner = -1;
  u64 bytes = 0;
  u64 dev_off = 0;  // pool offset of the device extent
  u64 host_off = 0;
  int ev = -1;      // timing event pair index
  bool zvc = false; // compressed mode and the buffer holds ReLU outputs (sparse)
  bool tf32 = false; // compressed mode 2 and only TF32 consumers read it in backward
};

// Runtime form of one planned compute step (vdnnp::Step), with the pieces
// the launch code needs resolved.
struct FwdStep {
  int layer = -1;
  std::vector<u64> in_off;   // feature offsets of the layer's inputs (in input order, via owners)
  u64 out_off = 0;           // own feature buffer (or owner's for ACTV)
  u64 w_off = 0;
  u64 ws_off = 0, ws_bytes = 0;
  std::vector<Transfer> offloads;
  int ev = -1;
  bool relu = false;  // conv/FC: ReLU of the following ACTV fused into the epilogue
  bool skip = false;  // ACTV whose ReLU was fused into its producer
  u64 gap_off = 0, gap_len = 0;  // free pool segment while the kernel runs
  // step scratch (the free gap when it is wide enough, else the fallback
  // buffer): [summed elementwise-join input | split-K partials]
  size_t scratch = 0;
  size_t sum_bytes = 0;          // elementwise join: the summed input X
  size_t part_off = 0, part_bytes = 0;
  // BF16 first layer (raw input, C % 8 != 0): channel-padded copies of X and
  // W in the step's scratch feed the TMA producers
  int pad_c = 0;                 // padded channel count (0 = not padded)
  size_t x8_off = 0, w8_off = 0;
};

struct BwdStep {
  int layer = -1;
  std::vector<Transfer> prefetches;     // issued at this step (opportunistic + on demand)
  std::vector<int> wait_prefetch;       // owners whose prefetch must land before the kernels
  std::vector<u64> in_off;              // features of inputs (X), in input order
  u64 out_off = 0;                      // own feature buffer (POOL Y / ACTV owner)
  u64 w_off = 0;
  u64 ws_off = 0, ws_bytes = 0;
  std::vector<u64> plane_off;           // dX planes written by this step (per input; ~0 = none)
  bool accumulate = false;              // two-buffer fork accumulation
  std::vector<u64> dy_off;              // distinct incoming gradient locations (first = canonical)
  int ev = -1;
  std::vector<char> mask_plane;         // per input: ReLU backward of that input fused here
  bool skip = false;                    // ACTV whose backward was fused into its gradient's producer
  u64 gap_off = 0, gap_len = 0;         // free pool segment while the kernel runs
  // incoming planes all shared (elementwise join map, read-only): ACTV
  // writes the masked sum to its private plane priv_out, other layers read
  // the sum from scratch
  bool stage_dy = false;
  u64 priv_out = kNoOff;
  // step scratch: [summed join input | staged dY | zero-inserted dY (strided
  // conv dgrad) | split-K partials]
  size_t scratch = 0;
  size_t sum_bytes = 0, stage_off = 0, stage_bytes = 0, dil_off = 0, dil_bytes = 0, part_off = 0, part_bytes = 0;
  int pad_c = 0;                 // as FwdStep; plus the fp32 dW of the padded weights (external grads)
  size_t x8_off = 0, w8_off = 0, dw8_off = 0;
};

class Session {
 public:
  Session(const vdnnp::Net& g, const vdnnp::Decision& d, const vdnnp::Cost& c, u64 capacity, const Options& o);
  ~Session();
  Session(const Session&) = delete;
  Session& operator=(const Session&) = delete;

  void set_batch_host(const float* images, const int32_t* labels);
  void set_batch_device(const float* images, const int32_t* labels);
  // Graphs with several INPUT layers: images of one of them (layer id).
  void set_input(int layer, const float* images, bool device);
  // Input pipeline: copy the NEXT batch from pinned host memory straight into
  // the INPUT extent on a separate stream, as soon as the running step no
  // longer touches that extent (planned, Program::input_idle_after); the next
  // step() waits for it. No staging buffer outside the pool.
  void prefetch_batch_host(const float* images, const int32_t* labels);
  // Loss of the last step (D2H + sync), for callers that issue step()
  // without reading the loss and prefetch the next batch first.
  float read_loss();
  // Pipelined loss readback: queue the D2H of the last step's loss into a
  // pinned ring slot (returns a ticket) and wait for it later, so the host
  // can enqueue the next step before the previous loss arrives.
  int64_t queue_loss();
  float wait_loss(int64_t ticket);
  void synthetic_batch(u64 seed);
  void get_weights(int layer, float* host, size_t count);
  void set_weights(int layer, const float* host, size_t count);
  void step(float lr, float* loss_host);
  void synchronize();
  void read_feature(int owner, float* host, size_t count);
  vdnnp::Report measured_report() const;
  void layer_times(int n, double* fwd_ms, double* bwd_ms) const;
  void grad_buffer(int layer, void** ptr, size_t* count);
  void grad_arena(void** ptr, size_t* count);
  void apply_grads(float lr, float scale);
  void set_grad_arena(float* ptr, size_t count);
  // Data-parallel exchange over peer memory (runtime/peer.cu): export this
  // session's arena / gradient arena / signal words as CUDA IPC handles, map
  // every peer's, then run the fused reduce + SGD + broadcast each step.
  struct PeerHandle {
    cudaIpcMemHandle_t arena, grads, signal;
    u64 arena_lo, arena_bytes, grads_count;
  };
  PeerHandle peer_export();
  void peer_attach(int rank, int world, const PeerHandle* all);
  void peer_exchange(float lr, float scale);
  // In-step exchange (SURVEY §8(e) placement): each layer's share is reduced,
  // updated and broadcast on a side stream right after that layer's wgrad in
  // BWD, overlapping the rest of the backward pass; the step ends with one
  // barrier and the compute stream joins the side stream. Same chunks, same
  // summation order: bit-identical to peer_exchange after the step.
  void peer_overlap(bool on, float scale);
  void peer_detach();
  int peer_world() const { return peer_world_; }
  // Device offload target (Options::offload_target = 1): bytes the slots need,
  // a caller-provided device buffer, or a peer's spill buffer through IPC.
  u64 offload_bytes() const { return host_bytes_; }
  void set_offload_buffer(void* dev_ptr, u64 bytes);
  cudaIpcMemHandle_t spill_export();       // allocates this rank's spill buffer (offload_bytes) for a peer
  void spill_attach(const cudaIpcMemHandle_t& h);  // offload into a peer's spill buffer

  const vdnnp::Report& plan() const { return plan_; }
  u64 arena_bytes() const { return arena_bytes_; }
  u64 arena_lo() const { return arena_lo_; }
  u64 host_bytes() const { return host_bytes_; }
  // cumulative bytes that crossed the host link (compressed mode: the wire
  // form; copy mode: the planned bytes)
  void transfer_stats(u64* offload_wire, u64* prefetch_wire, u64* offload_raw, u64* prefetch_raw);
  u64 scratch_bytes() const { return scratch_bytes_; }
  cudaStream_t stream() const { return cs_; }

 private:
  float* F(u64 off) const { return reinterpret_cast<float*>(base_ + off); }
  // Storage format of every pool tensor: fp32 (elem_size 4) or bf16
  // (elem_size 2, cost_model.hpp:69); the kernel calls below dispatch on it.
  bool bf_ = false;
  u64 es_ = 4;
  void* LG(u64 elem) const { return reinterpret_cast<char*>(loss_grad_) + elem * es_; }  // softmax gradient
  void k_combine(void* dst, const std::vector<const float*>& src, const void* y, size_t n, const char* what);
  void k_add_into(float* dst, const std::vector<const float*>& src, size_t n, const char* what);
  void k_relu_bwd(float* g0, const std::vector<const float*>& extra, const float* y, size_t n);
  void read_device(float* host, const void* dev, size_t count) const;  // storage -> fp32 host
  void acquire();
  void release() noexcept;
  void build_program();
  void fuse_relus();
  float* scratch_for(u64 gap_off, u64 gap_len, size_t need) const;
  bool compressible(int owner) const;
  int sm_reserve_ = -1;  // SMs left to the compressed-transfer kernels (set on the first step)
  bool tf32_exact_ok(int owner) const;
  void init_weights();
  void run_fwd(const FwdStep& s, float lr);
  void run_bwd(const BwdStep& s, float lr);
  // sum_x: the summed input of an elementwise join (one segment, shared plane)
  vdnnk::ConvArgs conv_args(int layer, const std::vector<u64>& in_off, const std::vector<u64>* planes,
                            const float* sum_x = nullptr) const;
  vdnnk::PoolArgs pool_args(int layer, const std::vector<u64>& in_off, const std::vector<u64>* planes,
                            const float* sum_x) const;
  bool summed(int layer) const;  // elementwise join over >= 2 inputs
  int padded_channels(int layer) const;  // BF16 first layer: padded C (0 = none)
  // algo_kernels = 1 and the layer's planned algorithm is GEMM_WS with its workspace extent at ws_off
  bool gemmws(int layer, u64 ws_off, u64 ws_bytes) const;
  void pad_operands(vdnnk::ConvArgs& a, int cp, char* x8, const float* w, char* w8);
  void sum_inputs(int layer, const std::vector<u64>& in_off, float* dst);
  void check(cudaError_t e, const char* what) const;

  vdnnp::Net g_;
  vdnnp::Decision d_;
  vdnnp::Cost c_;
  u64 cap_;
  Options o_;
  vdnnp::Report plan_;
  vdnnp::Program prog_;   // the plan's executable form (bound offsets, transfers, waits)
  vdnnp::Dataflow df_;
  int L_ = 0;
  int input_id_ = -1, loss_id_ = -1, logits_owner_ = -1;
  int classes_ = 0;                 // max over LOSS heads (synthetic labels)
  std::vector<int> inputs_;         // INPUT layers (ids ascending) and their setup extents
  std::vector<u64> input_off_;
  std::vector<int> loss_classes_;   // per layer (LOSS heads only)
  std::vector<u64> loss_grad_at_;   // per layer: float offset of its softmax gradient in loss_grad_
  u64 loss_grad_count_ = 0;

  cudaStream_t cs_ = nullptr, ms_ = nullptr;
  char* arena_ = nullptr;
  char* base_ = nullptr;
  u64 arena_lo_ = 0, arena_bytes_ = 0;
  char* host_ = nullptr;
  char* host_dev_ = nullptr;  // device view of the mapped host arena (compressed mode)
  u64 host_bytes_ = 0;
  unsigned long long* wire_ = nullptr;  // [0] offload, [1] prefetch wire bytes (device counters)
  u64 raw_off_ = 0, raw_pre_ = 0;       // planned bytes issued so far
  u64 copy_off_ = 0, copy_pre_ = 0;     // of which moved by cudaMemcpyAsync
  std::vector<u64> host_slot_;  // per owner
  u64 scratch_bytes_ = 0;
  float* loss_grad_ = nullptr;
  float* row_loss_ = nullptr;
  float* loss_ = nullptr;
  int32_t* labels_ = nullptr;
  float* splitk_ = nullptr;      // split-K partials for steps whose free pool gap is too small
  size_t splitk_bytes_ = 0;
  size_t splitk_in_pool_ = 0;    // steps whose partials live in the pool's free gap
  float* grads_ = nullptr;       // external gradient arena
  bool grads_owned_ = true;
  std::vector<u64> grad_off_;    // per layer float offset into grads_
  size_t grads_count_ = 0;
  float* pinned_loss_ = nullptr;
  // input pipeline (prefetch_batch_host): the next batch lands directly in
  // the INPUT extent once the running step no longer touches it
  // (Program::input_idle_after); labels alternate between two slots
  cudaStream_t in_stream_ = nullptr;
  cudaEvent_t input_idle_ev_ = nullptr;   // recorded by every step after its idle point
  cudaEvent_t staged_ready_ = nullptr;
  int32_t* labels_next_ = nullptr;        // the other label slot
  bool has_staged_ = false;
  static constexpr int kLossRing = 4;
  float* loss_ring_ = nullptr;            // pinned, kLossRing slots
  cudaEvent_t loss_ev_[kLossRing] = {};
  int64_t loss_tickets_ = 0;
  unsigned long long* signal_ = nullptr;  // peer barrier flags [2][kPeerMaxRanks]
  vdnnk::PeerArgs peer_{};
  vdnnk::PeerChunk* peer_chunks_ = nullptr;
  std::vector<void*> peer_maps_;          // IPC-opened pointers (closed on detach)
  bool host_owned_ = false;               // host_ is our cudaHostAlloc (else a device target)
  // CUDA graph mode
  cudaGraphExec_t gexec_ = nullptr;
  float graph_lr_ = 0.f;
  int eager_steps_ = 0;
  u64 g_copy_off_ = 0, g_copy_pre_ = 0, g_raw_off_ = 0, g_raw_pre_ = 0, g_launches_ = 0;  // per-step deltas
  void enqueue_step(float lr);
  // A pointer the captured step reads or writes changed: re-capture (after
  // one eager step) instead of replaying into the old buffer.
  void drop_graph() noexcept {
    if (gexec_) cudaGraphExecDestroy(gexec_);
    gexec_ = nullptr;
    eager_steps_ = 0;
  }
  void* spill_ = nullptr;                 // buffer this rank hosts for a peer's offloads
  void* spill_map_ = nullptr;             // IPC mapping of the peer's spill buffer (our target)
  int peer_world_ = 0;
  unsigned long long peer_epoch_ = 0;
  bool peer_inline_ = false;              // peer_overlap: exchange inside the step
  float peer_scale_ = 1.f;
  cudaStream_t xs_ = nullptr;             // exchange stream
  cudaEvent_t xs_done_ = nullptr;
  std::vector<cudaEvent_t> wg_ev_;        // per layer: its wgrad finished (compute stream)
  std::vector<int> peer_first_, peer_count_;  // per layer: this rank's chunk range
  void peer_layer(int layer, float lr);   // enqueue one layer's exchange (after its wgrad)
  void peer_finish();                     // end of step: barrier, join

  u64 x_off_ = 0;                // INPUT feature extent (setup allocation)
  int input_idle_after_ = -1;    // step after which the INPUT extent may take the next batch
  std::vector<u64> w_off_;       // per layer weight offset
  std::vector<FwdStep> fwd_;
  std::vector<BwdStep> bwd_;

  // timing
  std::vector<cudaEvent_t> ev_;  // pairs: [2i] start, [2i+1] end
  cudaEvent_t ev_iter_ = nullptr;
  // the previous step's timing events: steps alternate between two sets so
  // the host can enqueue step k+1 while step k's events are still pending
  // (re-recording in-flight timing events stalled the host ~1 step)
  std::vector<cudaEvent_t> ev_prev_, t0_ev_prev_;
  cudaEvent_t ev_iter_prev_ = nullptr;
  cudaEvent_t ev_sync_ = nullptr;
  std::vector<cudaEvent_t> step_ev_;  // compute-side step-start events (cross-stream gating)
  std::vector<cudaEvent_t> t0_ev_;    // timed step-start events (record_timeline)
  std::vector<cudaEvent_t> xfer_ev_;  // per transfer completion
  bool timed_ = false;
  bool timeline_paused_ = false;  // record_timeline sessions: skip the per-op events (timed benchmark loops)

 public:
  // Pause / resume the per-op CUDA events of a record_timeline session; the
  // measured report and layer times then describe the last step run with
  // them on.
  void pause_timeline(bool paused) { timeline_paused_ = paused; }

  // Layer-local probe (parity tests): during the next step, copy the
  // operands of one compute step (FWD or BWD of one layer) into a
  // caller-provided device buffer -- what the kernels read, right before they
  // run, and what they wrote, right after -- so every kernel can be checked
  // against the oracle op evaluated on the very inputs it saw. The copies are
  // stream-ordered on the compute stream; probes are one-shot.
  enum ProbeWhat { kPX = 0, kPW = 1, kPY = 2, kPDY = 3, kPDXBefore = 4, kPDX = 5, kPDW = 6, kPLossGrad = 7,
                   kPLoss = 8 };
  struct ProbeSeg {
    int what = 0, index = 0;  // index: input slot (X, DX) or incoming plane (DY)
    u64 dst = 0, bytes = 0;   // byte range in the destination buffer
    int src = 0;              // 0 pool offset, 1 gradient arena (float offset), 2 loss gradient, 3 loss
    u64 src_off = 0;
    bool after = false;       // copied after the step's kernels (else before)
  };
  struct ProbeLayout {
    std::vector<ProbeSeg> segs;
    u64 total = 0;
    int relu = 0;        // FWD: the following ACTV's ReLU is applied in the epilogue
    int accumulate = 0;  // BWD: dX added into a plane that already holds a fork gradient
    unsigned mask = 0;   // BWD: bit i = ReLU-backward mask of input i (x_i > 0) applied in the epilogue
    int skip = 0;        // ACTV step fused into its neighbour (launches nothing)
  };
  ProbeLayout probe_layout(int layer, bool bwd) const;
  void arm_probe(int layer, bool bwd, void* dst, u64 bytes);

 private:
  struct ArmedProbe {
    int ev = -1;
    ProbeLayout lay;
    char* dst = nullptr;
  };
  std::vector<ArmedProbe> probes_;
  void probe_copy(int ev, bool after);
};

}  // namespace vdnnrt
