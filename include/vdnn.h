/*
 * vdnn.h — C ABI of the B200-native vDNN runtime (libvdnn.so).
 *
 * Drop-in boundary for the reference's layer-wise training path. The
 * reference (vdnnsim, /root/reference/proj/include/vdnnsim) is a header-only
 * C++20 library with no FFI; its path sits behind these free functions, each
 * of which has a C entry point here:
 *
 *   NetworkGraph::add_X, finalize   net_graph.hpp:101-229   -> vdnn_graph_add_X, _finalize
 *   build_preset / extend_vgg        presets.hpp:123-140     -> vdnn_preset, vdnn_extend_vgg
 *   CostModel (profiles, formulas)   cost_model.hpp:15-213   -> vdnn_cost_model, vdnn_cost_*
 *   baseline_footprint               footprint.hpp:81-104    -> vdnn_baseline_footprint
 *   static_decision                  decision.hpp:68-95      -> vdnn_decision_static
 *   PolicyDecision (+validate)       decision.hpp:30-57      -> vdnn_decision_create / _set_* / _validate
 *   find_prefetch_layer              prefetch.hpp:16-23      -> (inside vdnn_simulate)
 *   simulate / simulate_with_trace   simulator.hpp:568-584   -> vdnn_simulate
 *   per_layer_event_peaks            policy.hpp:45-56        -> vdnn_report_layer_peaks
 *   greedy_downgrade                 policy.hpp:65-109       -> vdnn_greedy_downgrade
 *   dynamic_select                   policy.hpp:115-148      -> vdnn_dynamic_select
 *   simulate_oracle                  policy.hpp:152-156      -> vdnn_simulate_oracle
 *   replay_check                     replay.hpp:95-304       -> vdnn_replay_check
 *
 * and the B200 training executor that *runs* a plan (vdnn_session_*), plus
 * kernel-level entry points (vdnn_kernel_*) used by the parity tests. The
 * executor's extensions have no reference counterpart (the reference only
 * times the schedule): the data-parallel exchange (vdnn_session_peer_*:
 * the reference is single-GPU), the device / peer-HBM offload
 * target (vdnn_session_set_offload_buffer, _spill_*: a LinkProfile other than
 * PCIe, cost_model.hpp:22-30), compressed offload (compress_offload) and the
 * input pipeline (vdnn_session_prefetch_batch_host).
 *
 * Conventions: every call returns vdnn_status; the message of the last
 * failure on the calling thread is vdnn_last_error(). OOM is not an error:
 * it is report data (pass = 0 + OOM info), exactly as in the reference
 * (simulator.hpp:203-212). Handles are opaque and caller-owned; destroy them
 * with the matching *_destroy. Independent handles may be used from different
 * threads concurrently; one handle is single-threaded.
 */
#ifndef VDNN_H_
#define VDNN_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum vdnn_status {
  VDNN_OK = 0,
  VDNN_ERROR = 1,            /* vdnnsim::Error (generic config/usage) */
  VDNN_SHAPE_MISMATCH = 2,   /* vdnnsim::ShapeMismatch   core.hpp:26 */
  VDNN_UNKNOWN_PRESET = 3,   /* vdnnsim::UnknownPreset   core.hpp:27 */
  VDNN_INVALID_DEPTH = 4,    /* vdnnsim::InvalidDepth    core.hpp:28 */
  VDNN_OVERFLOW = 5,         /* vdnnsim::OverflowError   core.hpp:29 */
  VDNN_WRONG_LAYER_KIND = 6, /* vdnnsim::WrongLayerKind  core.hpp:30 */
  VDNN_POOL_MISUSE = 7,      /* vdnnsim::PoolUseError    core.hpp:31 */
  VDNN_INVALID_DECISION = 8, /* vdnnsim::InvalidDecision core.hpp:32 */
  VDNN_CONFIG_ERROR = 9,     /* vdnnsim::ConfigError     core.hpp:33 */
  VDNN_CUDA_ERROR = 10,
  VDNN_NCCL_ERROR = 11,
  VDNN_UNSUPPORTED = 12,     /* graph valid for the planner but not runnable by the executor */
  VDNN_INVALID_ARGUMENT = 13
} vdnn_status;

const char* vdnn_last_error(void);
const char* vdnn_version(void);

/* ------------------------------------------------------------ graph ---- */
typedef struct vdnn_graph vdnn_graph;
typedef enum { VDNN_INPUT = 0, VDNN_CONV = 1, VDNN_ACTV = 2, VDNN_POOL = 3, VDNN_FC = 4, VDNN_LOSS = 5 } vdnn_layer_kind;
typedef enum { VDNN_JOIN_CONCAT = 0, VDNN_JOIN_ELEMENTWISE = 1 } vdnn_join_rule;

typedef struct vdnn_layer_info {
  int32_t id;
  int32_t kind;      /* vdnn_layer_kind */
  int32_t join;      /* vdnn_join_rule */
  int32_t n_inputs;
  int32_t inputs[16];
  uint64_t p0, p1, p2, p3; /* conv: kernel,stride,pad,out_channels; pool: window,stride; fc: out; input: c,h,w */
  uint64_t n, c, h, w;     /* inferred output shape (NCHW) */
  int32_t refcnt;
} vdnn_layer_info;

vdnn_status vdnn_graph_create(uint64_t batch, vdnn_graph** out);
vdnn_status vdnn_graph_clone(const vdnn_graph* g, vdnn_graph** out);
void vdnn_graph_destroy(vdnn_graph* g);
vdnn_status vdnn_graph_add_input(vdnn_graph* g, uint64_t c, uint64_t h, uint64_t w, int32_t* id);
vdnn_status vdnn_graph_add_conv(vdnn_graph* g, const int32_t* inputs, int32_t n_inputs, uint64_t out_channels,
                                uint64_t kernel, uint64_t stride, uint64_t pad, int32_t join, int32_t* id);
/* Generic NetworkGraph::add_layer (net_graph.hpp:109-113) as used by the INI inline-layer front-end
   (config.hpp:194-235): kind 0..5 = input, conv, actv, pool, fc, loss; params per kind as
   conv (kernel, stride, pad, out), pool (window, stride), fc (out), input (c, h, w). Arity and
   parameter checks happen at finalize, as in the reference. */
vdnn_status vdnn_graph_add_layer(vdnn_graph* g, int32_t kind, const int32_t* inputs, int32_t n_inputs, uint64_t p0,
                                 uint64_t p1, uint64_t p2, uint64_t p3, int32_t join, int32_t* id);
vdnn_status vdnn_graph_add_actv(vdnn_graph* g, int32_t input, int32_t* id);
vdnn_status vdnn_graph_add_pool(vdnn_graph* g, const int32_t* inputs, int32_t n_inputs, uint64_t window,
                                uint64_t stride, int32_t join, int32_t* id);
vdnn_status vdnn_graph_add_fc(vdnn_graph* g, const int32_t* inputs, int32_t n_inputs, uint64_t out_features,
                              int32_t join, int32_t* id);
vdnn_status vdnn_graph_add_loss(vdnn_graph* g, int32_t input, int32_t* id);
vdnn_status vdnn_graph_finalize(vdnn_graph* g); /* validate + infer shapes + refcounts */
vdnn_status vdnn_graph_size(const vdnn_graph* g, int32_t* n);
vdnn_status vdnn_graph_batch(const vdnn_graph* g, uint64_t* batch);
vdnn_status vdnn_graph_layer(const vdnn_graph* g, int32_t id, vdnn_layer_info* out);
vdnn_status vdnn_preset(const char* name, uint64_t batch, vdnn_graph** out);
vdnn_status vdnn_extend_vgg(int32_t extra_conv_layers, uint64_t batch, vdnn_graph** out);

/* ------------------------------------------------------- cost model ---- */
/* Field-for-field the reference CostModel/DeviceProfile/LinkProfile
 * (cost_model.hpp:15-26,65-75) with its defaults (Titan X / PCIe 3). */
typedef struct vdnn_cost_model {
  double peak_flops, dram_bw;
  uint64_t mem_capacity;
  double compute_efficiency;
  double link_effective_bw, link_nominal_bw, link_launch_overhead;
  uint64_t elem_size;
  double bwd_fwd_ratio;
  double speed_factor_implicit_gemm, speed_factor_gemm_ws, speed_factor_fft;
  int32_t n_overrides;          /* latency_overrides (cost_model.hpp:74-75) */
  const int32_t* override_layer;
  const double* override_fwd_s;
  const double* override_bwd_s;
} vdnn_cost_model;

void vdnn_cost_model_default(vdnn_cost_model* cm);
typedef enum { VDNN_ALGO_IMPLICIT_GEMM = 0, VDNN_ALGO_GEMM_WS = 1, VDNN_ALGO_FFT = 2 } vdnn_algo;
vdnn_status vdnn_cost_tensor_bytes(const vdnn_cost_model* cm, const vdnn_graph* g, int32_t id, uint64_t* bytes);
vdnn_status vdnn_cost_weight_bytes(const vdnn_cost_model* cm, const vdnn_graph* g, int32_t id, uint64_t* bytes);
vdnn_status vdnn_cost_conv_workspace(const vdnn_cost_model* cm, const vdnn_graph* g, int32_t id, int32_t algo,
                                     uint64_t* bytes);
vdnn_status vdnn_cost_layer_latency(const vdnn_cost_model* cm, const vdnn_graph* g, int32_t id, int32_t bwd,
                                    int32_t algo, double* seconds);
vdnn_status vdnn_cost_flops(const vdnn_cost_model* cm, const vdnn_graph* g, int32_t id, int32_t bwd, double* flops);
vdnn_status vdnn_cost_transfer_latency(const vdnn_cost_model* cm, uint64_t bytes, double* seconds);
vdnn_status vdnn_cost_fastest_algo(const vdnn_cost_model* cm, const vdnn_graph* g, int32_t id, int32_t* algo);
vdnn_status vdnn_gradient_map_bytes(const vdnn_cost_model* cm, const vdnn_graph* g, int32_t id, uint64_t* bytes);

typedef struct vdnn_footprint {
  uint64_t weights_bytes, feature_maps_bytes, gradient_buffers_bytes, workspace_bytes, total_bytes,
      classifier_bytes;
} vdnn_footprint;

/* ---------------------------------------------------------- decisions -- */
typedef struct vdnn_decision vdnn_decision;
typedef enum { VDNN_POLICY_BASELINE = 0, VDNN_POLICY_VDNN_ALL = 1, VDNN_POLICY_VDNN_CONV = 2 } vdnn_policy_kind;
typedef enum { VDNN_MODE_MEMORY_OPTIMAL = 0, VDNN_MODE_PERF_OPTIMAL = 1 } vdnn_algo_mode;
typedef enum { VDNN_GRAD_TWO_BUFFER_REUSE = 0, VDNN_GRAD_PER_LAYER = 1 } vdnn_gradient_scheme;

vdnn_status vdnn_decision_static(const vdnn_graph* g, int32_t kind, int32_t mode, const vdnn_cost_model* cm,
                                 vdnn_decision** out);
/* Empty decision (no offload, no algos, per_layer): fill with the setters. */
vdnn_status vdnn_decision_create(const vdnn_graph* g, vdnn_decision** out);
vdnn_status vdnn_decision_clone(const vdnn_decision* d, vdnn_decision** out);
void vdnn_decision_destroy(vdnn_decision* d);
vdnn_status vdnn_decision_set_offload(vdnn_decision* d, int32_t layer, int32_t flag);
vdnn_status vdnn_decision_set_algo(vdnn_decision* d, int32_t layer, int32_t algo); /* algo < 0 erases */
vdnn_status vdnn_decision_set_scheme(vdnn_decision* d, int32_t scheme);
vdnn_status vdnn_decision_set_label(vdnn_decision* d, const char* label);
vdnn_status vdnn_decision_get(const vdnn_decision* d, int32_t* n_layers, char* offload_flags /*n_layers*/,
                              int32_t* algos /*n_layers, -1 = none*/, int32_t* scheme, char* label,
                              size_t label_cap);
vdnn_status vdnn_decision_validate(const vdnn_decision* d, const vdnn_graph* g);
vdnn_status vdnn_baseline_footprint(const vdnn_graph* g, const vdnn_decision* algos_from, const vdnn_cost_model* cm,
                                    int32_t include_weight_grads, vdnn_footprint* out);

/* ---------------------------------------------------------- simulate --- */
typedef struct vdnn_report vdnn_report;
typedef enum { VDNN_STREAM_COMPUTE = 0, VDNN_STREAM_MEMORY = 1 } vdnn_stream;
typedef enum {
  VDNN_EV_FWD = 0, VDNN_EV_BWD = 1, VDNN_EV_OFFLOAD = 2, VDNN_EV_PREFETCH = 3,
  VDNN_EV_ALLOC = 4, VDNN_EV_RELEASE = 5, VDNN_EV_SYNC = 6
} vdnn_event_kind;
typedef enum { VDNN_PHASE_SETUP = 0, VDNN_PHASE_FORWARD = 1, VDNN_PHASE_BACKWARD = 2 } vdnn_phase;

typedef struct vdnn_event {  /* StreamEvent, sim_types.hpp:30-42 */
  int32_t stream, kind, layer, buffer;
  int64_t start_ns, end_ns;
  uint64_t bytes, offset;
  char tag[4];               /* "", "W", "dW", "X", "Y", "dX", "WS", "G2" */
} vdnn_event;

typedef struct vdnn_report_summary { /* RunReport, sim_types.hpp:63-90 */
  int32_t pass, has_oom;
  int32_t oom_layer, oom_phase, oom_fragmented;
  uint64_t oom_requested;
  char oom_tag[4];
  uint64_t max_mem_bytes, avg_mem_bytes, offload_traffic_bytes, prefetch_traffic_bytes, host_peak_bytes;
  int64_t stall_fwd_offload_ns, stall_bwd_prefetch_ns, total_ns;
  double interference_bound;
  uint64_t n_events;
  char verdict[96];
} vdnn_report_summary;

typedef struct vdnn_pool_trace_row { /* PoolTraceRow, memory_pool.hpp:22-30 */
  int64_t time_ns;
  char op;  /* 'a' / 'f' */
  char tag[4];
  uint64_t offset, bytes, current, high_water;
} vdnn_pool_trace_row;

#define VDNN_SIM_KEEP_POOL_TRACE 1
#define VDNN_SIM_INCLUDE_WEIGHT_GRADS 2

vdnn_status vdnn_simulate(const vdnn_graph* g, const vdnn_decision* d, const vdnn_cost_model* cm,
                          uint64_t capacity, uint32_t flags, vdnn_report** out);
vdnn_status vdnn_simulate_oracle(const vdnn_graph* g, const vdnn_cost_model* cm, vdnn_report** out);
void vdnn_report_destroy(vdnn_report* r);
vdnn_status vdnn_report_summary_get(const vdnn_report* r, vdnn_report_summary* out);
vdnn_status vdnn_report_events(const vdnn_report* r, vdnn_event* out, size_t cap, size_t* n);
vdnn_status vdnn_report_reuse_distance(const vdnn_report* r, int64_t* out, size_t cap, size_t* n);
vdnn_status vdnn_report_pool_trace(const vdnn_report* r, vdnn_pool_trace_row* out, size_t cap, size_t* n);
vdnn_status vdnn_report_layer_peaks(const vdnn_report* r, int32_t n_layers, uint64_t* fwd_peak, uint64_t* bwd_peak);
/* Schedule signature: FNV-1a-64 over "<stream>,<KIND>,<layer>,<bytes>,<tag>,<buffer>,<offset>;" of every
 * event whose kind is not FWD/BWD/SYNC. */
vdnn_status vdnn_report_signature(const vdnn_report* r, uint64_t* sig);
/* Build a report from an external event log (e.g. measured GPU timestamps). */
vdnn_status vdnn_report_from_events(const vdnn_event* ev, size_t n, const vdnn_report_summary* s,
                                    vdnn_report** out);

/* --------------------------------------------------- policy (vDNN_dyn) -- */
typedef struct vdnn_dyn vdnn_dyn;
typedef struct vdnn_pass_info {
  char phase[16];
  char label[64];
  int32_t pass, has_oom, oom_layer, oom_phase;
  int64_t total_ns;
  uint64_t max_mem_bytes;
} vdnn_pass_info;

vdnn_status vdnn_dynamic_select(const vdnn_graph* g, uint64_t capacity, const vdnn_cost_model* cm, vdnn_dyn** out);
void vdnn_dyn_destroy(vdnn_dyn* s);
vdnn_status vdnn_dyn_untrainable(const vdnn_dyn* s, int32_t* untrainable);
vdnn_status vdnn_dyn_decision(const vdnn_dyn* s, vdnn_decision** out); /* copy; VDNN_ERROR if untrainable */
vdnn_status vdnn_dyn_passes(const vdnn_dyn* s, vdnn_pass_info* out, size_t cap, size_t* n);
vdnn_status vdnn_dyn_pass_decision(const vdnn_dyn* s, size_t index, vdnn_decision** out);
/* greedy_downgrade: *found = 0 when no assignment fits (reference returns nullopt). */
vdnn_status vdnn_greedy_downgrade(const vdnn_graph* g, uint64_t capacity, int32_t offload_kind,
                                  const vdnn_cost_model* cm, int32_t* found, vdnn_decision** out);

/* ------------------------------------------------------------ replay --- */
typedef struct vdnn_violation {
  char kind[32];
  char detail[160];
} vdnn_violation;
vdnn_status vdnn_replay_check(const vdnn_report* r, const vdnn_graph* g, const vdnn_decision* d, uint64_t capacity,
                              vdnn_violation* out, size_t cap, size_t* n);
/* The executable program the session runs (operands bound to pool offsets,
 * per-step scratch gaps, transfers) checked against the plan's own event log:
 * every binding inside the extent live for that buffer at that step. Not a
 * reference entry point: the parity gate for the executor's view of a plan. */
vdnn_status vdnn_program_check(const vdnn_graph* g, const vdnn_decision* d, const vdnn_cost_model* cm,
                               uint64_t capacity, vdnn_violation* out, size_t cap, size_t* n);

/* ------------------------------------------------- B200 training session -- */
typedef struct vdnn_session vdnn_session;
typedef struct vdnn_session_options {
  int32_t device;            /* CUDA ordinal */
  uint64_t weight_seed;      /* He-normal init seed base (layer seed = base + id) */
  int32_t external_grads;    /* 1: wgrad writes dW to a non-pool gradient arena (for allreduce) */
  int32_t record_timeline;   /* 1: record CUDA events per op for a measured report */
  int32_t host_arena;        /* 1: pinned host arena for offloads (required when the plan offloads) */
  int32_t precise_fp32;      /* 1: conv/FC contractions as 3xTF32 (fp32-accurate); 0: TF32 */
  int32_t compress_offload;  /* 1: offload/prefetch through the SMs in lossless zero-value-compressed form;
                                2: as 1, and maps read in backward only by TF32 contractions and ReLU masks
                                travel TF32-exact (bit-identical training step; not with precise_fp32) */
  int32_t offload_target;    /* 0: pinned host arena (PCIe); 1: a device buffer set with
                                vdnn_session_set_offload_buffer / _spill_attach (e.g. a peer GPU's HBM) */
  int32_t cuda_graph;        /* 1: replay each step as one CUDA graph (captured on the 2nd step, re-captured
                                when lr changes) */
  int32_t algo_kernels;      /* 0: the implicit-GEMM kernels for every planned conv algorithm (fastest on the
                                B200; the planned workspace is reserved); 1: GEMM_WS layers run the
                                reference's algorithm -- im2col into the planned workspace + a 1x1 GEMM
                                (cost_model.hpp:163-168); FFT layers stay implicit (no FFT kernel) */
} vdnn_session_options;
void vdnn_session_options_default(vdnn_session_options* o);

vdnn_status vdnn_session_create(const vdnn_graph* g, const vdnn_decision* d, const vdnn_cost_model* cm,
                                uint64_t capacity, const vdnn_session_options* opt, vdnn_session** out);
void vdnn_session_destroy(vdnn_session* s);
/* The plan (simulate report) the session replays. Borrowed pointer. */
const vdnn_report* vdnn_session_plan(const vdnn_session* s);
vdnn_status vdnn_session_arena_info(const vdnn_session* s, uint64_t* arena_bytes, uint64_t* arena_base_offset,
                                    uint64_t* host_arena_bytes, uint64_t* scratch_bytes);
/* Inputs: host (pinned or pageable) or device pointers; NHWC fp32 images, int32 labels. */
vdnn_status vdnn_session_set_batch_host(vdnn_session* s, const float* images, const int32_t* labels);
vdnn_status vdnn_session_set_batch_device(vdnn_session* s, const float* images, const int32_t* labels);
vdnn_status vdnn_session_synthetic_batch(vdnn_session* s, uint64_t seed);
/* Graphs with several INPUT layers (net_graph.hpp allows any number): images of INPUT layer `layer`
 * (set_batch_* fills the first INPUT layer; labels are shared by every LOSS head, taken modulo its
 * class count; the step's loss is the sum over heads). */
vdnn_status vdnn_session_set_input(vdnn_session* s, int32_t layer, const float* images, int32_t on_device);
/* Input pipeline: stage the NEXT batch (pinned host pointers) on a separate stream while the current
 * step runs; the next vdnn_session_step consumes it. Pair with vdnn_session_step(s, lr, NULL) +
 * vdnn_session_read_loss so the host does not wait on the loss before staging the next batch. */
vdnn_status vdnn_session_prefetch_batch_host(vdnn_session* s, const float* images, const int32_t* labels);
vdnn_status vdnn_session_read_loss(vdnn_session* s, float* loss);
/* Pipelined loss readback: queue the last step's loss (ticket), wait for it later (<= 4 outstanding). */
vdnn_status vdnn_session_queue_loss(vdnn_session* s, int64_t* ticket);
vdnn_status vdnn_session_wait_loss(vdnn_session* s, int64_t ticket, float* loss);
/* Weights: per layer, KRSC conv / [out][in]+bias FC; float count = weight_bytes/4. */
vdnn_status vdnn_session_get_weights(vdnn_session* s, int32_t layer, float* host, size_t count);
vdnn_status vdnn_session_set_weights(vdnn_session* s, int32_t layer, const float* host, size_t count);
/* One forward + backward + SGD iteration. loss_host may be NULL (no D2H). */
vdnn_status vdnn_session_step(vdnn_session* s, float lr, float* loss_host);
/* Forward only (for tests); leaves logits readable via vdnn_session_read_buffer. */
vdnn_status vdnn_session_synchronize(vdnn_session* s);
/* record_timeline sessions: 1 = skip the per-op timing events on the following steps (benchmark loops:
   they cost ~10% on small nets), 0 = record again; reports describe the last step recorded. */
vdnn_status vdnn_session_pause_timeline(vdnn_session* s, int32_t paused);
/* Copy a feature buffer (owner layer) or gradient buffer to host as of the last step (debug/tests). */
vdnn_status vdnn_session_read_feature(vdnn_session* s, int32_t owner, float* host, size_t count);
/* Measured report of the last step: plan events with CUDA-event timestamps. */
vdnn_status vdnn_session_measured_report(vdnn_session* s, vdnn_report** out);
/* Per-layer measured FWD/BWD milliseconds of the last step (needs record_timeline). */
vdnn_status vdnn_session_layer_times(vdnn_session* s, int32_t n_layers, double* fwd_ms, double* bwd_ms);
/* Cumulative host-link bytes since creation: wire (what crossed PCIe) and planned (raw) per direction. Syncs. */
vdnn_status vdnn_session_transfer_stats(vdnn_session* s, uint64_t* offload_wire, uint64_t* prefetch_wire,
                                        uint64_t* offload_planned, uint64_t* prefetch_planned);
/* Gradient arena (external_grads=1): device pointer and float count of layer's dW (or 0). */
vdnn_status vdnn_session_grad_buffer(vdnn_session* s, int32_t layer, void** dev_ptr, size_t* count);
/* Copy layer's dW (+bias grad for FC) from the gradient arena to host (external_grads=1). */
vdnn_status vdnn_session_get_grads(vdnn_session* s, int32_t layer, float* host, size_t count);
/* Apply SGD from the gradient arena (after an external allreduce). */
vdnn_status vdnn_session_apply_grads(vdnn_session* s, float lr, float grad_scale);
/* Use a caller-owned device buffer (>= grad_arena count floats) as the gradient arena. */
vdnn_status vdnn_session_set_grad_arena(vdnn_session* s, void* dev_ptr, size_t count);
/* Whole-gradient-arena pointer for a single bucketed allreduce. */
vdnn_status vdnn_session_grad_arena(vdnn_session* s, void** dev_ptr, size_t* count);
/* Data-parallel exchange over peer memory (NVLink P2P through CUDA IPC), the
 * fused replacement of "NCCL all-reduce of the gradient arena + apply_grads":
 * each rank exports a handle (needs external_grads=1 and the session-owned
 * gradient arena), the caller all-gathers the handles by any means, every
 * rank attaches with the full array (index = rank), then after each
 * vdnn_session_step every rank calls vdnn_session_peer_exchange, which on the
 * compute stream waits for all ranks, reduces 1/N of the gradients from all
 * ranks in rank order, applies w -= lr*scale*sum and writes the new weights
 * into every rank's arena, then waits for all ranks again. All ranks must run
 * the same plan (checked) and call exchange the same number of times. */
typedef struct vdnn_peer_handle {
  uint8_t arena[64], grads[64], signal[64]; /* cudaIpcMemHandle_t */
  uint64_t arena_lo, arena_bytes, grads_count;
} vdnn_peer_handle;
vdnn_status vdnn_session_peer_export(vdnn_session* s, vdnn_peer_handle* out);
vdnn_status vdnn_session_peer_attach(vdnn_session* s, int32_t rank, int32_t world, const vdnn_peer_handle* all);
vdnn_status vdnn_session_peer_exchange(vdnn_session* s, float lr, float grad_scale);
/* on = 1: instead of vdnn_session_peer_exchange after the step, every layer's
 * exchange runs inside vdnn_session_step on a side stream right after that
 * layer's weight gradient (overlapping the rest of the backward pass), with
 * grad_scale applied; the step ends with one barrier. Same chunks and
 * summation order: bit-identical weights. Not with cuda_graph sessions. */
vdnn_status vdnn_session_peer_overlap(vdnn_session* s, int32_t on, float grad_scale);
vdnn_status vdnn_session_peer_detach(vdnn_session* s);
/* Device offload target (offload_target = 1): the bytes the offload slots need; use a caller-provided
 * device buffer, or host a spill buffer for a peer (export its CUDA IPC handle) and offload into a
 * peer's spill buffer (attach its handle) -- offloads then travel over NVLink instead of PCIe. */
vdnn_status vdnn_session_offload_bytes(vdnn_session* s, uint64_t* bytes);
vdnn_status vdnn_session_set_offload_buffer(vdnn_session* s, void* dev_ptr, uint64_t bytes);
vdnn_status vdnn_session_spill_export(vdnn_session* s, uint8_t ipc_handle[64]);
vdnn_status vdnn_session_spill_attach(vdnn_session* s, const uint8_t ipc_handle[64]);
/* Compute stream (cudaStream_t) for interop. */
vdnn_status vdnn_session_stream(vdnn_session* s, void** stream);
/* Layer-local probe (parity tests; not a reference entry point). During the next vdnn_session_step,
 * the operands of one compute step -- FWD (bwd = 0) or BWD (bwd = 1) of `layer` -- are copied into a
 * caller-provided device buffer: what its kernels read, right before they run, and what they wrote,
 * right after (stream-ordered on the compute stream; one-shot; not in cuda_graph mode). The layout
 * lists the segments (offset/bytes in the destination) and the fusions the step applies:
 *   X[i]: input i (NHWC fp32); W: weights (index 1 = after an in-step SGD); Y: output;
 *   DY: incoming gradient (after the fold of the other planes); DX_BEFORE[i] / DX[i]: gradient plane of
 *   input i before (two-buffer accumulation) / after; DW: dW (+bias grad) in the gradient arena;
 *   LOSS_GRAD (N x classes softmax gradient), LOSS (scalar). */
enum { VDNN_PROBE_X = 0, VDNN_PROBE_W = 1, VDNN_PROBE_Y = 2, VDNN_PROBE_DY = 3, VDNN_PROBE_DX_BEFORE = 4,
       VDNN_PROBE_DX = 5, VDNN_PROBE_DW = 6, VDNN_PROBE_LOSS_GRAD = 7, VDNN_PROBE_LOSS = 8 };
#define VDNN_PROBE_MAX_SEGS 40
typedef struct vdnn_probe_seg {
  int32_t what, index, after, pad_;
  uint64_t offset, bytes;
} vdnn_probe_seg;
typedef struct vdnn_probe_layout {
  int32_t nseg;
  int32_t relu_fused;    /* FWD: the next ACTV's ReLU applied in the epilogue */
  int32_t accumulate;    /* BWD: dX added into a plane holding a fork gradient */
  int32_t skip;          /* ACTV fused into a neighbour: launches nothing */
  uint32_t mask_planes;  /* BWD: bit i = dX[i] masked by (X[i] > 0) in the epilogue */
  uint32_t pad_;
  uint64_t total_bytes;
  vdnn_probe_seg seg[VDNN_PROBE_MAX_SEGS];
} vdnn_probe_layout;
vdnn_status vdnn_session_probe_layout(vdnn_session* s, int32_t layer, int32_t bwd, vdnn_probe_layout* out);
vdnn_status vdnn_session_arm_probe(vdnn_session* s, int32_t layer, int32_t bwd, void* dst_dev, uint64_t dst_bytes);
uint64_t vdnn_kernel_launch_count(void);

/* ------------------------------------------ kernel-level entry points ---- */
/* conv over NHWC fp32 segments (channel concat), KRSC weights, tf32 tensor cores. */
typedef struct vdnn_conv_desc {
  int32_t n, h, w;
  int32_t nseg;
  const float* x[8];
  float* dx[8];
  int32_t c[8];
  int32_t cout, kh, kw, stride, pad;
} vdnn_conv_desc;
vdnn_status vdnn_kernel_conv_fprop(const vdnn_conv_desc* d, const float* w, const float* bias, float* y,
                                   void* stream);
vdnn_status vdnn_kernel_conv_dgrad(const vdnn_conv_desc* d, const float* w, const float* dy, int32_t accumulate,
                                   void* stream);
vdnn_status vdnn_kernel_conv_wgrad(const vdnn_conv_desc* d, const float* dy, float* w, float lr, float* dw_out,
                                   float* ws, size_t ws_bytes, void* stream);
size_t vdnn_kernel_conv_wgrad_ws_bytes(const vdnn_conv_desc* d);
/* fprop with a workspace: outputs with fewer tiles than SMs (FC layers) run a deterministic split-K
   (partial slabs + ordered reduce with the bias/ReLU epilogue). ws_bytes >= vdnn_kernel_conv_fprop_ws_bytes
   uses the full split (0 when the shape does not split). */
vdnn_status vdnn_kernel_conv_fprop_ws(const vdnn_conv_desc* d, const float* w, const float* bias, float* y, float* ws,
                                      size_t ws_bytes, void* stream);
size_t vdnn_kernel_conv_fprop_ws_bytes(const vdnn_conv_desc* d);
/* dgrad with a workspace: FC layers (1x1 filter over a 1x1 image) with fewer dX tiles than SMs run the same
   deterministic split-K (partial slabs + ordered reduce with the ReLU mask and accumulation). */
vdnn_status vdnn_kernel_conv_dgrad_ws(const vdnn_conv_desc* d, const float* w, const float* dy, int32_t accumulate,
                                      float* ws, size_t ws_bytes, void* stream);
size_t vdnn_kernel_conv_dgrad_ws_bytes(const vdnn_conv_desc* d);
/* Calling-thread switch for the kernel-level conv entry points: 1 = 3xTF32 (fp32-accurate), 0 = TF32. */
void vdnn_kernel_set_precise(int32_t on);
/* Calling-thread switch: 1 = TMA producers where eligible (default), 0 = cp.async gathers everywhere. */
void vdnn_kernel_set_tma(int32_t on);
/* Lossless zero-value-compressed copy between a device buffer and a mapped pinned host buffer
   (device-accessible pointer, >= vdnn_kernel_zvc_slot_bytes(4*count) bytes); count % 4 == 0, 16-B aligned.
   wire (device u64 counter, may be NULL for decompress) accumulates the bytes moved. */
uint64_t vdnn_kernel_zvc_slot_bytes(uint64_t bytes);
vdnn_status vdnn_kernel_zvc_compress(const float* src, uint64_t count, void* host_dst, uint64_t* wire, void* stream);
/* As vdnn_kernel_zvc_compress, but nonzeros may travel TF32-exact (sign, exponent, top 10 mantissa bits;
   the low 13 bits -- ignored by tcgen05 kind::tf32 -- are dropped). Chunks holding a nonzero that would
   truncate to +-0 or an Inf/NaN stay lossless. */
vdnn_status vdnn_kernel_zvc_compress_tf32(const float* src, uint64_t count, void* host_dst, uint64_t* wire,
                                          void* stream);
vdnn_status vdnn_kernel_zvc_decompress(const void* host_src, uint64_t count, float* dst, uint64_t* wire,
                                       void* stream);
/* BF16 maps (elem_size = 2): lossless zero-value-compressed copy of `count` bf16 (count % 8 == 0, 16-B
   aligned) into a mapped pinned slot of >= vdnn_kernel_zvc_slot_bytes_bf16(2*count) bytes and back.
   Replaces nothing in the reference (a transfer format under its schedule). */
uint64_t vdnn_kernel_zvc_slot_bytes_bf16(uint64_t bytes);
vdnn_status vdnn_kernel_zvc_compress_bf16(const void* src, uint64_t count, void* host_dst, uint64_t* wire,
                                          void* stream);
vdnn_status vdnn_kernel_zvc_decompress_bf16(const void* host_src, uint64_t count, void* dst, uint64_t* wire,
                                            void* stream);
/* Measured tcgen05 kind::tf32 ceiling of the current device in TFLOP/s (roofline denominator). */
vdnn_status vdnn_kernel_tf32_peak(double* tflops);
vdnn_status vdnn_kernel_maxpool_fwd(const vdnn_conv_desc* d, int32_t window, int32_t stride, float* y, void* stream);
vdnn_status vdnn_kernel_maxpool_bwd(const vdnn_conv_desc* d, int32_t window, int32_t stride, const float* y,
                                    const float* dy, void* stream);
vdnn_status vdnn_kernel_relu_fwd(float* y, size_t n, void* stream);
vdnn_status vdnn_kernel_relu_bwd(float* g, const float* y, size_t n, void* stream);
vdnn_status vdnn_kernel_softmax_xent(const float* logits, const int32_t* labels, int32_t n, int32_t k, float* grad,
                                     float* row_loss, float* loss, void* stream);
vdnn_status vdnn_kernel_bias_grad(const float* dy, int32_t n, int32_t o, float* bias, float lr, float* db_out,
                                  void* stream);

#ifdef __cplusplus
}
#endif
#endif /* VDNN_H_ */
