// Host planner: a from-scratch, bit-exact restatement of the vdnnsim
// layer-wise training path (network graph, presets, cost/footprint byte
// formulas, the double-ended pool, host ledger, static and dynamic offload
// decisions, the offload/prefetch schedule generator and the event-log
// validator). Its output -- the ordered event log with pool offsets -- is what
// the CUDA executor replays on the device arena.
//
// Reference correspondence (all /root/reference/proj/include/vdnnsim/):
//   Graph / shape inference ........ net_graph.hpp:16-401
//   Presets ......................... presets.hpp:16-140
//   CostModel ....................... cost_model.hpp:15-219
//   Footprint ....................... footprint.hpp:48-104
//   Pool / HostLedger ............... memory_pool.hpp:41-256
//   Decisions ....................... decision.hpp:12-95
//   Prefetch-layer search ........... prefetch.hpp:16-23
//   Schedule generator (simulate) ... simulator.hpp:30-584
//   Dynamic policy (vDNN_dyn) ....... policy.hpp:13-156
//   Event-log validator ............. replay.hpp:15-304
#pragma once

#include <cstdint>
#include <map>
#include <optional>
#include <stdexcept>
#include <string>
#include <vector>

namespace vdnnp {

using u64 = std::uint64_t;
using i64 = std::int64_t;
using u128 = unsigned __int128;

constexpr int kNone = -1;
constexpr u64 kUnlimited = u64{1} << 62;  // core.hpp:17
constexpr u64 kAlign = 512;               // memory_pool.hpp:43

// Error classes map 1:1 onto the reference's exception hierarchy
// (core.hpp:21-32) and onto vdnn_status codes of the C ABI.
enum class Err { Generic = 1, Shape = 2, Preset = 3, Depth = 4, Overflow = 5, LayerKind = 6, Pool = 7,
                 Decision = 8, Config = 9 };
struct PlanError : std::runtime_error {
  Err code;
  PlanError(Err c, const std::string& m) : std::runtime_error(m), code(c) {}
};

u64 mul_checked(u64 a, u64 b, const char* what);
inline u64 round_up(u64 v, u64 a) { return (v + a - 1) / a * a; }
i64 seconds_to_ns(double s);

// ------------------------------------------------------------------ graph --
enum class Kind : int { Input = 0, Conv = 1, Actv = 2, Pool = 3, Fc = 4, Loss = 5 };
enum class Join : int { Concat = 0, Elementwise = 1 };
const char* kind_name(Kind k);

struct Dims {  // NCHW
  u64 n = 1, c = 1, h = 1, w = 1;
  u64 count() const;
  bool operator==(const Dims& o) const { return n == o.n && c == o.c && h == o.h && w == o.w; }
};

struct Node {
  int id = 0;
  Kind kind = Kind::Input;
  std::vector<int> in;
  Join join = Join::Concat;
  // conv: kernel, stride, pad, out_channels | pool: window, stride | fc: out | input: c, h, w
  u64 k = 1, s = 1, p = 0, out = 1;
  u64 ic = 1, ih = 1, iw = 1;
};

class Net {
 public:
  explicit Net(u64 batch = 1) : batch_(batch) {}
  u64 batch() const { return batch_; }
  int add(Node n);
  int input(u64 c, u64 h, u64 w);
  int conv(std::vector<int> in, u64 out, u64 kernel, u64 stride, u64 pad, Join j = Join::Concat);
  int actv(int in);
  int pool(std::vector<int> in, u64 window, u64 stride, Join j = Join::Concat);
  int fc(std::vector<int> in, u64 out, Join j = Join::Concat);
  int loss(int in);
  void finalize();  // validate + shapes + consumers
  bool finalized() const { return shapes_.size() == nodes_.size(); }

  int size() const { return static_cast<int>(nodes_.size()); }
  const Node& at(int id) const { return nodes_.at(static_cast<size_t>(id)); }
  const std::vector<Node>& nodes() const { return nodes_; }
  const Dims& dims(int id) const { return shapes_.at(static_cast<size_t>(id)); }
  const std::vector<int>& users(int id) const { return users_.at(static_cast<size_t>(id)); }
  int refs(int id) const { return static_cast<int>(users(id).size()); }

  // feature_owner (net_graph.hpp:386-389): nearest non-ACTV ancestor.
  int owner(int id) const;
  // input_shape_of (net_graph.hpp:393-401): joined X shape (no validation).
  Dims in_dims(int id) const;
  // fc_in_features (net_graph.hpp:371-382)
  u64 fc_inputs(int id) const;

 private:
  void check() const;
  Dims joined(const Node& n) const;
  u64 batch_;
  std::vector<Node> nodes_;
  std::vector<Dims> shapes_;
  std::vector<std::vector<int>> users_;
};

Net make_preset(const std::string& name, u64 batch);  // presets.hpp:123-130
Net make_deep_vgg(int extra_convs, u64 batch);        // presets.hpp:135-140

// ------------------------------------------------------------- cost model --
enum class Algo : int { Implicit = 0, GemmWs = 1, Fft = 2 };
const char* algo_name(Algo a);
std::optional<Algo> step_down(Algo a);  // cost_model.hpp:52-59

struct Cost {
  double peak_flops = 7e12, dram_bw = 336e9;
  u64 mem_capacity = 12884901888ull;
  double compute_efficiency = 0.5;
  double link_bw = 12.8e9, link_nominal_bw = 16e9, link_overhead = 0.0;
  u64 elem = 4;
  double bwd_ratio = 2.0;
  double sf_implicit = 1.0, sf_gemm_ws = 0.8, sf_fft = 0.6;
  std::map<int, std::pair<double, double>> pinned;  // latency_overrides

  double speed(Algo a) const;
  bool fft_ok(const Net& g, int id) const;
  Algo fastest(const Net& g, int id) const;
  double flop_count(const Net& g, int id, bool bwd) const;
  u64 traffic_bytes(const Net& g, int id) const;
  double latency(const Net& g, int id, bool bwd, Algo a = Algo::Implicit) const;
  u64 workspace(const Net& g, int id, Algo a) const;
  double transfer(u64 bytes) const { return link_overhead + static_cast<double>(bytes) / link_bw; }
  double interference() const { return link_nominal_bw / dram_bw; }
  u64 bytes_of(const Dims& d) const { return mul_checked(d.count(), elem, "tensor_bytes"); }
  u64 weights(const Net& g, int id) const;
};

// footprint.hpp:48-104
bool counted_feature(const Net& g, int owner);
u64 grad_map_bytes(const Net& g, int m, const Cost& c);
u64 max_grad_map_bytes(const Net& g, const Cost& c);
struct Footprint {
  u64 weights = 0, features = 0, gradients = 0, workspace = 0, total = 0, classifier = 0;
};
Footprint footprint(const Net& g, const std::map<int, Algo>& algos, const Cost& c, bool with_dw);

// ---------------------------------------------------------------- pool -----
struct TraceRow {
  i64 t = 0;
  char op = 'a';
  std::string tag;
  u64 off = 0, len = 0, cur = 0, hw = 0;
};

// The device arena's address map: an ordered list of segments that tiles
// [0, capacity) exactly, each either holding one allocation or free (no two
// free segments are ever adjacent). An allocation is named by its start
// offset, which is unique among live allocations. Placement policy
// (memory_pool.hpp:32-86): requests of at most capacity/8 bytes, and pinned
// requests, take the top of the highest-addressed free segment that fits;
// larger requests take the bottom of the smallest free segment that fits
// (lowest address on ties). Sizes are rounded up to 512 B.
class Arena {
 public:
  explicit Arena(u64 capacity, bool trace = false);
  std::optional<u64> place(u64 bytes, const std::string& tag, i64 t, bool pinned);
  void free_at(u64 off, i64 t);
  u64 requested_at(u64 off) const;
  u64 live_bytes() const { return live_; }
  u64 high_water() const { return hw_; }
  // (offset, length) of the largest free segment; lowest address on ties
  std::pair<u64, u64> widest_gap() const;
  u64 free_total() const;
  // a request that total free space could hold but no single gap can
  bool would_fragment(u64 bytes) const;
  void audit() const;  // tiling / coalescing / conservation invariants
  u128 byte_ns_until(i64 t);
  const std::vector<TraceRow>& trace() const { return rows_; }
  u64 capacity() const { return cap_; }

 private:
  // trivially copyable (the segment vector is spliced on every place / free;
  // a std::string member made that a string move per shifted segment):
  // the tag is an index into tags_, recorded only when tracing
  struct Seg {
    u64 off = 0, len = 0;
    bool used = false;
    u64 req = 0;
    int32_t tag = -1;
  };
  std::vector<std::string> tags_;
  void clock_to(i64 t);
  size_t seg_at(u64 off) const;  // index of the segment starting at off
  u64 cap_;
  bool trace_;
  std::vector<Seg> segs_;
  u64 live_ = 0, hw_ = 0;
  i64 now_ = 0;
  u128 area_ = 0;
  std::vector<TraceRow> rows_;
};

// ----------------------------------------------------------- decisions ----
enum class Policy : int { Baseline = 0, All = 1, ConvOnly = 2 };
enum class Mode : int { Memory = 0, Perf = 1 };
enum class Scheme : int { TwoBuffer = 0, PerLayer = 1 };
bool may_offload(Kind k);  // decision.hpp:26-28

struct Decision {
  std::vector<char> offload;
  std::map<int, Algo> algos;
  Scheme scheme = Scheme::PerLayer;
  std::string label;
  bool offloads(int id) const { return offload.at(static_cast<size_t>(id)) != 0; }
  void check(const Net& g) const;  // PolicyDecision::validate
};
std::map<int, Algo> pick_algos(const Net& g, Mode m, const Cost& c);
Decision make_static(Policy k, Mode m, const Net& g, const Cost& c);

// --------------------------------------------------------------- events ---
enum class Lane : int { Compute = 0, Memory = 1 };
enum class Ev : int { Fwd = 0, Bwd = 1, Offload = 2, Prefetch = 3, Alloc = 4, Release = 5, Sync = 6 };
enum class Stage : int { Setup = 0, Forward = 1, Backward = 2 };
const char* ev_name(Ev e);
const char* stage_name(Stage s);

struct Event {
  Lane lane = Lane::Compute;
  Ev kind = Ev::Fwd;
  int layer = kNone;
  i64 t0 = 0, t1 = 0;
  u64 bytes = 0;
  std::string tag;
  int buffer = kNone;
  u64 off = 0;
};

struct Oom {
  int layer = kNone;
  Stage stage = Stage::Setup;
  bool fragmented = false;
  u64 requested = 0;
  std::string tag;
};

struct Report {
  std::vector<Event> events;
  u64 max_mem = 0, avg_mem = 0, offload_bytes = 0, prefetch_bytes = 0, host_peak = 0;
  i64 stall_fwd = 0, stall_bwd = 0, total = 0;
  bool pass = false;
  std::optional<Oom> oom;
  std::vector<i64> reuse;
  double interference = 0.0;
  std::vector<TraceRow> pool_trace;
  std::string verdict() const;
};

struct SimFlags {
  bool trace = false;
  bool with_dw = false;
};

// ------------------------------------------------------------- dataflow ---
// What (graph, decision) fix before any timing (simulator.hpp:30-155): one
// record per layer id. Feature fields describe the buffer the layer owns
// (bytes == 0: it owns none -- ACTV aliases its producer's, LOSS has none).
struct LayerFlow {
  // own feature buffer
  u64 bytes = 0;
  i64 copy_ns = 0;              // one-way host-link time of the buffer
  int fwd_readers = 0;          // forward steps that read it
  int last_fwd_reader = kNone;
  std::vector<int> bwd_readers; // backward steps that read it (ascending)
  // the layer's own steps
  std::vector<int> x_owners;    // distinct owners of its inputs (ascending)
  std::vector<int> bwd_operands;// feature buffers its BWD reads (ascending)
  std::vector<int> drains;      // buffers its FWD offloads (ascending)
  u64 w_bytes = 0, ws_bytes = 0;
  i64 fwd_ns = 0, bwd_ns = 0;
  // gradients
  u64 dx_bytes = 0;             // its dX map (0: none)
  std::vector<int> dx_readers;  // BWD steps that take its dX as dY (ascending)
  std::vector<int> dy_sources;  // dX maps its BWD takes as dY (ascending)
};
struct Dataflow {
  std::vector<LayerFlow> at;
  u64 g2_bytes = 0, ws2_bytes = 0;  // two-buffer scheme: each G2 buffer, the shared WS
};
Dataflow derive_dataflow(const Net& g, const Decision& d, const Cost& c);

// --------------------------------------------------------------- program ---
// The executable form of a plan: every compute step (FWD/BWD of one layer)
// with its operands bound to pool offsets, the transfers it issues on the
// memory stream and the transfers it must wait for. The reference-format
// event log (Report::events) is rendered from the same walk, so the executor
// and the schedule parity tests consume one object.
constexpr u64 kNoLoc = ~u64{0};

struct PlaneRef {     // the gradient plane of `producer`'s dX w.r.t. its input slot `slot`
  int producer = kNone;
  int slot = 0;       // concat: input index; elementwise: 0 (one shared plane)
  u64 off = kNoLoc;   // pool offset (or overflow slot, see Program::overflow_base)
  bool operator==(const PlaneRef& o) const { return producer == o.producer && slot == o.slot; }
};

struct Xfer {         // one OFFLOAD (D2H) or PREFETCH (H2D) of a whole feature buffer
  bool to_host = true;
  int owner = kNone;
  u64 bytes = 0;
  u64 dev_off = 0;    // device extent (offload: source; prefetch: freshly placed destination)
  int step = -1;      // compute step in which it is issued (it starts after that step begins)
  i64 t0 = 0, t1 = 0; // planned memory-lane window
};

struct Step {
  bool bwd = false;
  int layer = kNone;
  i64 t_enter = 0, t0 = 0, t1 = 0, t_leave = 0;  // planned: lane reaches the step, kernel, lane moves on
  std::vector<int> issues;        // Program::xfers issued here (in issue order)
  std::vector<int> wait_before;   // xfers the kernel must see landed (BWD operands in flight)
  bool wait_after = false;        // the next step waits for every xfer issued here (sync rule)
  std::vector<u64> x;             // per input: feature extent of its owner (FWD, BWD of CONV/FC/POOL)
  u64 y = kNoLoc;                 // FWD: output extent; BWD: POOL output / ACTV alias
  u64 w = kNoLoc;
  u64 ws = kNoLoc, ws_bytes = 0;
  std::vector<PlaneRef> dx;       // BWD: per input, the plane it writes (off = kNoLoc: none)
  bool dx_accumulate = false;     // two-buffer: add into a fork gradient already in the slot
  std::vector<PlaneRef> dy;       // BWD: distinct incoming planes; [0] receives the fold of the rest
  u64 gap_off = 0, gap_len = 0;   // widest free pool segment while the kernel runs (scratch space)
  // BWD of an ACTV: the step whose epilogue may apply this ReLU's mask to
  // input slot mask_slot (the only writer of its incoming plane), or -1
  int mask_host = -1, mask_slot = -1;
  // Shared planes (the one gradient map of an elementwise join, read by every
  // input's chain: footprint.hpp:67) are read-only. A step whose incoming
  // planes are all shared does not fold in place: an ACTV writes its masked
  // sum to a private plane (dx[0], placed after the arena: the reference's
  // plan has no extent for it), any other layer sums into its scratch gap.
  bool stage_dy = false;
};

struct Program {
  std::vector<Step> steps;
  std::vector<Xfer> xfers;
  std::vector<u64> w_off;         // per layer weight extent (kNoLoc: none)
  int input = kNone;              // the INPUT layer whose setup extent takes each batch
  u64 input_off = kNoLoc;
  // the step after whose kernel nothing touches the INPUT extent again this
  // iteration (the next batch may land there), or -1 = only after the last step
  int input_idle_after = -1;
  u64 arena_lo = 0, arena_hi = 0; // span of every planned extent
  // two-buffer scheme: gradient slots beyond the plan's two G2 buffers (a
  // graph that needs more live maps than two), placed after arena_hi
  u64 overflow_base = 0, overflow_slot_bytes = 0;
  int overflow_slots = 0;
  // private planes of ACTVs over shared planes (Step::stage_dy), after the
  // overflow slots: [private_base, private_base + private_bytes)
  u64 private_base = 0, private_bytes = 0;
};

// One pass of the schedule: the report (always) and the program (when
// `prog` is non-null and the plan passes).
Report plan(const Net& g, const Decision& d, const Cost& c, u64 capacity, const SimFlags& f = {},
            Program* prog = nullptr);
Report plan_oracle(const Net& g, const Cost& c);

// policy.hpp
void layer_peaks(const Report& r, std::vector<u64>& fwd, std::vector<u64>& bwd, int layers);
struct PassRecord {
  std::string phase;
  Decision decision;
  bool pass = false;
  std::optional<Oom> oom;
  i64 total = 0;
  u64 max_mem = 0;
};
struct DynResult {
  std::optional<Decision> decision;
  std::vector<PassRecord> passes;
};
std::optional<Decision> greedy(const Net& g, u64 capacity, Policy kind, const Cost& c,
                               std::vector<PassRecord>* transcript = nullptr);
DynResult choose_dynamic(const Net& g, u64 capacity, const Cost& c);

// replay.hpp
struct Finding {
  std::string kind, detail;
};
std::vector<Finding> validate_log(const Report& r, const Net& g, const Decision& d, u64 capacity);

u64 schedule_signature(const Report& r);
// Bindings of a compiled Program against the event log of the same pass.
std::vector<Finding> check_program(const Program& P, const Report& r, const Net& g, const Decision& d);

}  // namespace vdnnp
