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

// Fixed-capacity, 512-B aligned suballocator with size-segregated
// double-ended placement (memory_pool.hpp:32-86): requests above capacity/8
// are best-fit bottom-up, smaller or pinned requests go to the top of the
// highest fitting extent.
class Arena {
 public:
  explicit Arena(u64 capacity, bool trace = false);
  std::optional<u64> alloc(u64 bytes, const std::string& tag, i64 t, bool pin_high);
  void release(u64 handle, i64 t);
  u64 offset(u64 handle) const;
  u64 requested(u64 handle) const;
  u64 in_use() const { return used_; }
  u64 peak() const { return peak_; }
  u64 largest_hole() const;
  u64 total_free() const;
  bool fragmented(u64 bytes) const;
  void verify() const;  // self_check
  u128 integral_until(i64 t);
  const std::vector<TraceRow>& trace() const { return rows_; }
  u64 capacity() const { return cap_; }

 private:
  struct Live {
    u64 off, len, req;
    std::string tag;
  };
  void tick(i64 t);
  void give_back(u64 off, u64 len);
  u64 cap_;
  bool trace_;
  std::map<u64, u64> holes_;  // offset -> length, coalesced
  std::map<u64, Live> live_;
  u64 used_ = 0, peak_ = 0, next_ = 1;
  i64 last_t_ = 0;
  u128 area_ = 0;
  std::vector<TraceRow> rows_;
};

class PinnedLedger {  // HostLedger, memory_pool.hpp:225-256
 public:
  void add(int owner, u64 bytes, i64 t);
  void remove(int owner, i64 t);
  u64 peak() const { return peak_; }
  u64 current() const { return cur_; }

 private:
  std::map<int, u64> held_;
  u64 cur_ = 0, peak_ = 0;
  i64 last_t_ = 0;
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

// Residency of a feature buffer (sim_types.hpp:93-100).
enum class Where : int { None = 0, Device, Draining, Host, Filling, Gone };

// Static per-(graph, decision) dataflow (simulator.hpp:30-155); also the
// executor's map of who reads what.
struct Liveness {
  int L = 0;
  std::vector<u64> feat;                       // owner -> bytes (0 = no buffer)
  std::vector<std::vector<int>> fwd_users;     // owner -> forward readers
  std::vector<std::vector<int>> bwd_users;     // owner -> backward readers
  std::vector<std::vector<int>> owners_in;     // layer -> distinct owners of X
  std::vector<std::vector<int>> bwd_reads;     // layer -> feature buffers BWD reads
  std::vector<u64> grad;                       // layer -> dX bytes
  std::vector<std::vector<int>> grad_users;    // grad buffer -> backward readers
  std::vector<std::vector<int>> grads_read;    // layer -> grad buffers its BWD reads
  std::vector<std::vector<int>> offloads_at;   // layer -> buffers it offloads
  std::vector<u64> wbytes, wsbytes;
  std::vector<i64> fwd_ns, bwd_ns, xfer_ns;
  u64 g2_bytes = 0, ws2_bytes = 0;
};
Liveness analyze(const Net& g, const Decision& d, const Cost& c);

// First layer below `current` with a host-resident offloaded buffer; the
// scan stops after the first CONV (prefetch.hpp:16-23).
std::optional<int> prefetch_candidate(int current, const std::vector<Where>& where,
                                      const std::vector<std::vector<int>>& offloads_at, const Net& g);

Report plan(const Net& g, const Decision& d, const Cost& c, u64 capacity, const SimFlags& f = {});
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

}  // namespace vdnnp
