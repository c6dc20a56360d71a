// Device-arena allocator, pinned-host ledger and offload decisions.
#include <algorithm>

#include "planner.hpp"

namespace vdnnp {

// ---------------------------------------------------------------- Arena ---
Arena::Arena(u64 capacity, bool trace) : cap_(capacity), trace_(trace) {
  if (capacity > 0) holes_.emplace(0, capacity);
}

void Arena::tick(i64 t) {  // memory_pool.hpp:174-180
  if (t < last_t_) throw PlanError(Err::Pool, "pool timestamps must be non-decreasing");
  area_ += static_cast<u128>(used_) * static_cast<u128>(t - last_t_);
  last_t_ = t;
}

// memory_pool.hpp:55-86
std::optional<u64> Arena::alloc(u64 bytes, const std::string& tag, i64 t, bool pin_high) {
  if (bytes == 0) throw PlanError(Err::Pool, "zero-byte allocation");
  tick(t);
  const u64 need = round_up(bytes, kAlign);
  const bool top = pin_high || need <= cap_ / 8;
  auto pick = holes_.end();
  if (top) {
    // highest-addressed hole that fits; the block sits at its upper end
    for (auto it = holes_.begin(); it != holes_.end(); ++it)
      if (it->second >= need) pick = it;
  } else {
    // smallest hole that fits (first in address order on ties), lower end
    for (auto it = holes_.begin(); it != holes_.end(); ++it)
      if (it->second >= need && (pick == holes_.end() || it->second < pick->second)) pick = it;
  }
  if (pick == holes_.end()) return std::nullopt;
  const u64 hole_off = pick->first;
  const u64 rest = pick->second - need;
  const u64 off = top ? hole_off + rest : hole_off;
  holes_.erase(pick);
  if (rest > 0) holes_.emplace(top ? hole_off : hole_off + need, rest);
  const u64 h = next_++;
  live_.emplace(h, Live{off, need, bytes, tag});
  used_ += need;
  peak_ = std::max(peak_, used_);
  if (trace_) rows_.push_back(TraceRow{t, 'a', tag, off, need, used_, peak_});
  return h;
}

void Arena::release(u64 handle, i64 t) {  // memory_pool.hpp:88-97
  tick(t);
  auto it = live_.find(handle);
  if (it == live_.end()) throw PlanError(Err::Pool, "free of unknown or already-freed allocation id");
  const Live e = it->second;
  live_.erase(it);
  used_ -= e.len;
  give_back(e.off, e.len);
  if (trace_) rows_.push_back(TraceRow{t, 'f', e.tag, e.off, e.len, used_, peak_});
}

void Arena::give_back(u64 off, u64 len) {  // memory_pool.hpp:194-209
  auto nxt = holes_.lower_bound(off);
  if (nxt != holes_.begin()) {
    auto prv = std::prev(nxt);
    if (prv->first + prv->second == off) {
      off = prv->first;
      len += prv->second;
      holes_.erase(prv);
    }
  }
  if (nxt != holes_.end() && off + len == nxt->first) {
    len += nxt->second;
    holes_.erase(nxt);
  }
  holes_.emplace(off, len);
}

u64 Arena::offset(u64 h) const {
  auto it = live_.find(h);
  if (it == live_.end()) throw PlanError(Err::Pool, "offset_of: unknown allocation id");
  return it->second.off;
}
u64 Arena::requested(u64 h) const {
  auto it = live_.find(h);
  if (it == live_.end()) throw PlanError(Err::Pool, "requested_of: unknown allocation id");
  return it->second.req;
}
u64 Arena::largest_hole() const {
  u64 m = 0;
  for (const auto& [o, l] : holes_) m = std::max(m, l);
  return m;
}
u64 Arena::total_free() const {
  u64 t = 0;
  for (const auto& [o, l] : holes_) t += l;
  return t;
}
bool Arena::fragmented(u64 bytes) const {
  const u64 need = round_up(bytes, kAlign);
  return need <= total_free() && need > largest_hole();
}
u128 Arena::integral_until(i64 t) {
  tick(t);
  return area_;
}

void Arena::verify() const {  // memory_pool.hpp:145-169
  std::map<u64, std::pair<u64, bool>> spans;
  for (const auto& [o, l] : holes_) spans.emplace(o, std::make_pair(l, false));
  for (const auto& [h, e] : live_)
    if (!spans.emplace(e.off, std::make_pair(e.len, true)).second)
      throw PlanError(Err::Pool, "pool self-check: duplicate extent offset");
  u64 cursor = 0, total = 0;
  bool prev_free = false, first = true;
  for (const auto& [o, sp] : spans) {
    if (o < cursor) throw PlanError(Err::Pool, "pool self-check: overlapping extents");
    if (o != cursor) throw PlanError(Err::Pool, "pool self-check: gap in extent coverage");
    if (!first && prev_free && !sp.second)
      throw PlanError(Err::Pool, "pool self-check: adjacent free extents not coalesced");
    prev_free = !sp.second;
    cursor = o + sp.first;
    total += sp.first;
    first = false;
  }
  if (total != cap_) throw PlanError(Err::Pool, "pool self-check: live + free != capacity");
}

// --------------------------------------------------------- PinnedLedger ---
void PinnedLedger::add(int owner, u64 bytes, i64 t) {
  if (t < last_t_) throw PlanError(Err::Pool, "host ledger timestamps must be non-decreasing");
  last_t_ = t;
  held_[owner] += bytes;
  cur_ += bytes;
  peak_ = std::max(peak_, cur_);
}
void PinnedLedger::remove(int owner, i64 t) {
  if (t < last_t_) throw PlanError(Err::Pool, "host ledger timestamps must be non-decreasing");
  last_t_ = t;
  auto it = held_.find(owner);
  if (it == held_.end()) throw PlanError(Err::Pool, "host ledger: unknown buffer");
  cur_ -= it->second;
  held_.erase(it);
}

// ------------------------------------------------------------ decisions ---
bool may_offload(Kind k) { return k == Kind::Conv || k == Kind::Pool || k == Kind::Input; }

void Decision::check(const Net& g) const {  // decision.hpp:38-56
  if (offload.size() != static_cast<size_t>(g.size()))
    throw PlanError(Err::Decision, "offload flags do not cover the graph");
  for (const Node& l : g.nodes()) {
    const bool flagged = offload[static_cast<size_t>(l.id)] != 0;
    if (flagged && !may_offload(l.kind))
      throw PlanError(Err::Decision, "layer " + std::to_string(l.id) + " is not offload-eligible");
    if ((l.kind == Kind::Conv) != (algos.count(l.id) > 0))
      throw PlanError(Err::Decision, "algorithm assignment must cover exactly the CONV layers");
    if (flagged && scheme == Scheme::TwoBuffer)
      throw PlanError(Err::Decision, "two-buffer gradient reuse implies the network-wide baseline: no offloading");
  }
  for (const auto& [id, a] : algos)
    if (id < 0 || id >= g.size()) throw PlanError(Err::Decision, "algorithm assignment references unknown layer");
}

std::map<int, Algo> pick_algos(const Net& g, Mode m, const Cost& c) {
  std::map<int, Algo> a;
  for (const Node& l : g.nodes())
    if (l.kind == Kind::Conv) a[l.id] = m == Mode::Memory ? Algo::Implicit : c.fastest(g, l.id);
  return a;
}

Decision make_static(Policy k, Mode m, const Net& g, const Cost& c) {  // decision.hpp:68-95
  Decision d;
  d.offload.assign(static_cast<size_t>(g.size()), 0);
  d.algos = pick_algos(g, m, c);
  if (k == Policy::Baseline) {
    d.scheme = Scheme::TwoBuffer;
    d.label = "baseline";
  } else {
    d.scheme = Scheme::PerLayer;
    d.label = k == Policy::All ? "vdnn-all" : "vdnn-conv";
    for (const Node& l : g.nodes()) {
      const bool on = k == Policy::All ? may_offload(l.kind) : l.kind == Kind::Conv;
      if (on) d.offload[static_cast<size_t>(l.id)] = 1;
    }
  }
  d.label += m == Mode::Memory ? "(m)" : "(p)";
  return d;
}

// ---------------------------------------------------- vDNN_dyn (policy) ---
void layer_peaks(const Report& r, std::vector<u64>& fwd, std::vector<u64>& bwd, int layers) {  // policy.hpp:45-56
  fwd.assign(static_cast<size_t>(layers), 0);
  bwd.assign(static_cast<size_t>(layers), 0);
  u64 cur = 0;
  for (const Event& e : r.events) {
    if (e.kind == Ev::Alloc) cur += round_up(e.bytes, kAlign);
    if (e.kind == Ev::Release) cur -= round_up(e.bytes, kAlign);
    if (e.kind == Ev::Fwd) fwd[static_cast<size_t>(e.layer)] = cur;
    if (e.kind == Ev::Bwd) bwd[static_cast<size_t>(e.layer)] = cur;
  }
}

namespace {
PassRecord record(const std::string& phase, const Decision& d, const Report& r) {
  PassRecord p;
  p.phase = phase;
  p.decision = d;
  p.pass = r.pass;
  p.oom = r.oom;
  p.total = r.total;
  p.max_mem = r.max_mem;
  return p;
}
}  // namespace

std::optional<Decision> greedy(const Net& g, u64 capacity, Policy kind, const Cost& c,
                               std::vector<PassRecord>* transcript) {  // policy.hpp:65-109
  Decision d = make_static(kind, Mode::Perf, g, c);
  d.label = std::string(kind == Policy::ConvOnly ? "vdnn-conv" : "vdnn-all") + "+greedy";
  Decision probe = d;
  for (auto& [id, a] : probe.algos) a = Algo::Implicit;
  const Report base = plan(g, probe, c, kUnlimited);
  std::vector<u64> fp, bp;
  layer_peaks(base, fp, bp, g.size());
  for (const Node& l : g.nodes()) {
    if (l.kind != Kind::Conv) continue;
    const size_t i = static_cast<size_t>(l.id);
    const u64 hf = capacity > fp[i] ? capacity - fp[i] : 0;
    const u64 hb = capacity > bp[i] ? capacity - bp[i] : 0;
    const u64 room = std::min(hf, hb);
    Algo a = d.algos.at(l.id);
    while (round_up(c.workspace(g, l.id, a), kAlign) > room) {
      auto lower = step_down(a);
      if (!lower) break;
      a = *lower;
    }
    d.algos[l.id] = a;
  }
  const Report chk = plan(g, d, c, capacity);
  if (transcript) transcript->push_back(record("P3", d, chk));
  if (chk.pass) return d;
  bool floor = true;
  for (const auto& [id, a] : d.algos) floor = floor && a == Algo::Implicit;
  if (floor) return std::nullopt;
  for (auto& [id, a] : d.algos) a = Algo::Implicit;
  const Report chk2 = plan(g, d, c, capacity);
  if (transcript) transcript->push_back(record("P3", d, chk2));
  if (!chk2.pass) return std::nullopt;
  return d;
}

DynResult choose_dynamic(const Net& g, u64 capacity, const Cost& c) {  // policy.hpp:115-148
  DynResult out;
  const Decision floor = make_static(Policy::All, Mode::Memory, g, c);
  const Report r1 = plan(g, floor, c, capacity);
  out.passes.push_back(record("P1", floor, r1));
  if (!r1.pass) return out;
  for (Policy k : {Policy::Baseline, Policy::ConvOnly, Policy::All}) {
    Decision d = make_static(k, Mode::Perf, g, c);
    const Report r = plan(g, d, c, capacity);
    out.passes.push_back(record("P2", d, r));
    if (r.pass) {
      out.decision = std::move(d);
      return out;
    }
  }
  for (Policy k : {Policy::ConvOnly, Policy::All}) {
    if (auto d = greedy(g, capacity, k, c, &out.passes)) {
      out.decision = std::move(d);
      return out;
    }
  }
  out.passes.push_back(record("fallback", floor, r1));
  out.decision = floor;
  return out;
}

Report plan_oracle(const Net& g, const Cost& c) {  // policy.hpp:152-156
  Decision d = make_static(Policy::Baseline, Mode::Perf, g, c);
  d.label = "oracle";
  return plan(g, d, c, kUnlimited);
}

}  // namespace vdnnp
