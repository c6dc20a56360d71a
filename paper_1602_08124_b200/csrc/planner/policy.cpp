// Offload decisions: the static policies (vDNN_all / vDNN_conv / baseline)
// and vDNN_dyn, the profiling search over them (decision.hpp:12-95,
// policy.hpp:13-156). Every candidate is judged by one planner pass.
#include <algorithm>

#include "planner.hpp"

namespace vdnnp {

bool may_offload(Kind k) { return k == Kind::Conv || k == Kind::Pool || k == Kind::Input; }

void Decision::check(const Net& g) const {  // decision.hpp:38-56
  if (offload.size() != static_cast<size_t>(g.size()))
    throw PlanError(Err::Decision, "decision has " + std::to_string(offload.size()) + " offload flags for a " +
                                       std::to_string(g.size()) + "-layer graph");
  for (const Node& l : g.nodes()) {
    const bool on = offload[static_cast<size_t>(l.id)] != 0;
    if (on && !may_offload(l.kind))
      throw PlanError(Err::Decision, std::string("layer ") + std::to_string(l.id) + " (" + kind_name(l.kind) +
                                         ") cannot offload its input");
    if ((l.kind == Kind::Conv) != (algos.count(l.id) > 0))
      throw PlanError(Err::Decision, "layer " + std::to_string(l.id) +
                                         ": an algorithm must be chosen for every CONV layer and only for those");
    if (on && scheme == Scheme::TwoBuffer)
      throw PlanError(Err::Decision, "the two-buffer gradient scheme belongs to the no-offload baseline");
  }
  for (const auto& kv : algos)
    if (kv.first < 0 || kv.first >= g.size())
      throw PlanError(Err::Decision, "algorithm chosen for layer " + std::to_string(kv.first) + " outside the graph");
}

std::map<int, Algo> pick_algos(const Net& g, Mode m, const Cost& c) {
  std::map<int, Algo> a;
  for (const Node& l : g.nodes())
    if (l.kind == Kind::Conv) a.emplace(l.id, m == Mode::Perf ? c.fastest(g, l.id) : Algo::Implicit);
  return a;
}

Decision make_static(Policy k, Mode m, const Net& g, const Cost& c) {
  static const char* const names[] = {"baseline", "vdnn-all", "vdnn-conv"};
  Decision d;
  d.algos = pick_algos(g, m, c);
  d.scheme = k == Policy::Baseline ? Scheme::TwoBuffer : Scheme::PerLayer;
  d.offload.resize(static_cast<size_t>(g.size()));
  for (const Node& l : g.nodes()) {
    const bool on = k == Policy::All ? may_offload(l.kind) : (k == Policy::ConvOnly && l.kind == Kind::Conv);
    d.offload[static_cast<size_t>(l.id)] = on ? 1 : 0;
  }
  d.label = std::string(names[static_cast<int>(k)]) + (m == Mode::Perf ? "(p)" : "(m)");
  return d;
}

// Pool occupancy (512-B rounded) at each layer's FWD and BWD event, in log
// order (policy.hpp:45-56).
void layer_peaks(const Report& r, std::vector<u64>& fwd, std::vector<u64>& bwd, int layers) {
  fwd.assign(static_cast<size_t>(layers), 0);
  bwd.assign(static_cast<size_t>(layers), 0);
  u64 live = 0;
  for (const Event& e : r.events) {
    switch (e.kind) {
      case Ev::Alloc: live += round_up(e.bytes, kAlign); break;
      case Ev::Release: live -= round_up(e.bytes, kAlign); break;
      case Ev::Fwd: fwd[static_cast<size_t>(e.layer)] = live; break;
      case Ev::Bwd: bwd[static_cast<size_t>(e.layer)] = live; break;
      default: break;
    }
  }
}

namespace {

PassRecord judge(const char* phase, const Decision& d, const Net& g, const Cost& c, u64 capacity) {
  const Report r = plan(g, d, c, capacity);
  return PassRecord{phase, d, r.pass, r.oom, r.total, r.max_mem};
}

bool all_implicit(const Decision& d) {
  return std::all_of(d.algos.begin(), d.algos.end(), [](const auto& kv) { return kv.second == Algo::Implicit; });
}

}  // namespace

// Per-layer algorithm downgrade under one offload policy (policy.hpp:65-109):
// price every CONV layer's workspace headroom from a workspace-free pass on
// an unlimited pool, step each layer down FFT -> GEMM_WS -> IMPLICIT until its
// workspace fits that headroom, and confirm with one pass; if placement
// still fails, confirm once more with every layer at IMPLICIT.
std::optional<Decision> greedy(const Net& g, u64 capacity, Policy kind, const Cost& c,
                               std::vector<PassRecord>* transcript) {
  Decision d = make_static(kind, Mode::Perf, g, c);
  d.label = kind == Policy::ConvOnly ? "vdnn-conv+greedy" : "vdnn-all+greedy";

  Decision floor = d;
  for (auto& kv : floor.algos) kv.second = Algo::Implicit;
  std::vector<u64> at_fwd, at_bwd;
  layer_peaks(plan(g, floor, c, kUnlimited), at_fwd, at_bwd, g.size());

  for (auto& [id, algo] : d.algos) {
    const size_t i = static_cast<size_t>(id);
    const u64 used = std::max(at_fwd[i], at_bwd[i]);
    const u64 room = capacity > used ? capacity - used : 0;
    for (std::optional<Algo> a = algo; a; a = step_down(*a)) {
      algo = *a;
      if (round_up(c.workspace(g, id, algo), kAlign) <= room) break;
    }
  }
  std::vector<PassRecord> local;
  std::vector<PassRecord>& log = transcript ? *transcript : local;
  log.push_back(judge("P3", d, g, c, capacity));
  if (log.back().pass) return d;
  if (all_implicit(d)) return std::nullopt;
  for (auto& kv : d.algos) kv.second = Algo::Implicit;
  log.push_back(judge("P3", d, g, c, capacity));
  if (log.back().pass) return d;
  return std::nullopt;
}

// vDNN_dyn (policy.hpp:115-148): the memory floor (vDNN_all, implicit GEMM)
// decides trainability; then the fastest static configurations in order of
// increasing offload effort; then the greedy downgrades; else the floor.
DynResult choose_dynamic(const Net& g, u64 capacity, const Cost& c) {
  DynResult out;
  const Decision floor = make_static(Policy::All, Mode::Memory, g, c);
  out.passes.push_back(judge("P1", floor, g, c, capacity));
  if (!out.passes.back().pass) return out;  // untrainable under this budget

  for (Policy k : {Policy::Baseline, Policy::ConvOnly, Policy::All}) {
    out.passes.push_back(judge("P2", make_static(k, Mode::Perf, g, c), g, c, capacity));
    if (out.passes.back().pass) {
      out.decision = out.passes.back().decision;
      return out;
    }
  }
  for (Policy k : {Policy::ConvOnly, Policy::All})
    if (std::optional<Decision> d = greedy(g, capacity, k, c, &out.passes)) {
      out.decision = std::move(d);
      return out;
    }
  PassRecord fb = out.passes.front();
  fb.phase = "fallback";
  out.passes.push_back(fb);
  out.decision = floor;
  return out;
}

Report plan_oracle(const Net& g, const Cost& c) {  // policy.hpp:152-156
  Decision d = make_static(Policy::Baseline, Mode::Perf, g, c);
  d.label = "oracle";
  return plan(g, d, c, kUnlimited);
}

}  // namespace vdnnp
