// Offload/prefetch schedule generator: the two-clock (compute stream, memory
// stream) event loop of the reference simulator, producing the ordered event
// log with pool offsets that the CUDA executor replays.
// Reference: /root/reference/proj/include/vdnnsim/simulator.hpp:30-584.
#include <algorithm>

#include "planner.hpp"

namespace vdnnp {

const char* ev_name(Ev e) {
  switch (e) {
    case Ev::Fwd: return "FWD";
    case Ev::Bwd: return "BWD";
    case Ev::Offload: return "OFFLOAD";
    case Ev::Prefetch: return "PREFETCH";
    case Ev::Alloc: return "ALLOC";
    case Ev::Release: return "RELEASE";
    case Ev::Sync: return "SYNC";
  }
  return "?";
}

const char* stage_name(Stage s) {
  switch (s) {
    case Stage::Setup: return "setup";
    case Stage::Forward: return "forward";
    case Stage::Backward: return "backward";
  }
  return "?";
}

std::string Report::verdict() const {  // sim_types.hpp:80-89
  if (pass) return "PASS";
  if (!oom) return "FAIL";
  std::string v = "OOM(layer=" + std::to_string(oom->layer) + ", phase=" + stage_name(oom->stage);
  if (oom->fragmented) v += ", fragmented";
  return v + ")";
}

namespace {
void uniq(std::vector<int>& v) {
  std::sort(v.begin(), v.end());
  v.erase(std::unique(v.begin(), v.end()), v.end());
}
}  // namespace

// simulator.hpp:55-155
Liveness analyze(const Net& g, const Decision& d, const Cost& c) {
  Liveness p;
  const int L = g.size();
  const size_t n = static_cast<size_t>(L);
  p.L = L;
  p.feat.assign(n, 0);
  p.fwd_users.assign(n, {});
  p.bwd_users.assign(n, {});
  p.owners_in.assign(n, {});
  p.bwd_reads.assign(n, {});
  p.grad.assign(n, 0);
  p.grad_users.assign(n, {});
  p.grads_read.assign(n, {});
  p.offloads_at.assign(n, {});
  p.wbytes.assign(n, 0);
  p.wsbytes.assign(n, 0);
  p.fwd_ns.assign(n, 0);
  p.bwd_ns.assign(n, 0);
  p.xfer_ns.assign(n, 0);

  for (const Node& l : g.nodes()) {
    const size_t i = static_cast<size_t>(l.id);
    if (l.kind != Kind::Actv && l.kind != Kind::Loss) {
      p.feat[i] = c.bytes_of(g.dims(l.id));
      p.xfer_ns[i] = seconds_to_ns(c.transfer(p.feat[i]));
    }
    p.wbytes[i] = c.weights(g, l.id);
    const Algo a = l.kind == Kind::Conv ? d.algos.at(l.id) : Algo::Implicit;
    if (l.kind == Kind::Conv) p.wsbytes[i] = c.workspace(g, l.id, a);
    p.fwd_ns[i] = seconds_to_ns(c.latency(g, l.id, false, a));
    p.bwd_ns[i] = seconds_to_ns(c.latency(g, l.id, true, a));

    for (int q : l.in) p.owners_in[i].push_back(g.owner(q));
    uniq(p.owners_in[i]);
    for (int o : p.owners_in[i]) p.fwd_users[static_cast<size_t>(o)].push_back(l.id);

    switch (l.kind) {  // backward feature operands
      case Kind::Conv:
      case Kind::Fc:
        p.bwd_reads[i] = p.owners_in[i];
        break;
      case Kind::Pool:
        p.bwd_reads[i] = p.owners_in[i];
        p.bwd_reads[i].push_back(l.id);
        uniq(p.bwd_reads[i]);
        break;
      case Kind::Actv:
        p.bwd_reads[i] = {g.owner(l.id)};
        break;
      default:
        break;
    }
    for (int o : p.bwd_reads[i]) p.bwd_users[static_cast<size_t>(o)].push_back(l.id);

    p.grad[i] = grad_map_bytes(g, l.id, c);
    if (p.grad[i] > 0) {
      for (int q : l.in) {
        for (int cur = q;;) {
          const Kind k = g.at(cur).kind;
          if (k == Kind::Input) break;
          p.grad_users[i].push_back(cur);
          if (k != Kind::Actv) break;
          cur = g.at(cur).in[0];
        }
      }
      uniq(p.grad_users[i]);
      for (int r : p.grad_users[i]) p.grads_read[static_cast<size_t>(r)].push_back(l.id);
    }
  }
  for (auto& v : p.bwd_users) uniq(v);
  for (auto& v : p.grads_read) uniq(v);

  for (const Node& l : g.nodes()) {
    const size_t i = static_cast<size_t>(l.id);
    if (!d.offloads(l.id)) continue;
    if (l.kind != Kind::Conv && l.kind != Kind::Pool) continue;
    for (int o : p.owners_in[i]) {
      const auto& rd = p.fwd_users[static_cast<size_t>(o)];
      if (rd.empty() || rd.back() != l.id) continue;
      if (p.bwd_users[static_cast<size_t>(o)].empty()) continue;
      p.offloads_at[i].push_back(o);
    }
  }
  if (d.scheme == Scheme::TwoBuffer) {
    p.g2_bytes = max_grad_map_bytes(g, c);
    for (size_t i = 0; i < n; ++i) p.ws2_bytes = std::max(p.ws2_bytes, p.wsbytes[i]);
  }
  return p;
}

std::optional<int> prefetch_candidate(int current, const std::vector<Where>& where,
                                      const std::vector<std::vector<int>>& offloads_at, const Net& g) {
  for (int i = current - 1; i >= 0; --i) {
    for (int o : offloads_at[static_cast<size_t>(i)])
      if (where[static_cast<size_t>(o)] == Where::Host) return i;
    if (g.at(i).kind == Kind::Conv) break;
  }
  return std::nullopt;
}

namespace {

class Planner {
 public:
  Planner(const Net& g, const Decision& d, const Cost& c, u64 capacity, const SimFlags& f)
      : g_(g), d_(d), c_(c), f_(f), lv_(analyze(g, d, c)), arena_(capacity, f.trace) {
    const size_t n = static_cast<size_t>(lv_.L);
    where_.assign(n, Where::None);
    fwd_left_.assign(n, 0);
    bwd_left_.assign(n, 0);
    grad_left_.assign(n, 0);
    for (size_t i = 0; i < n; ++i) {
      fwd_left_[i] = static_cast<int>(lv_.fwd_users[i].size());
      bwd_left_[i] = static_cast<int>(lv_.bwd_users[i].size());
      grad_left_[i] = static_cast<int>(lv_.grad_users[i].size());
    }
    feat_h_.assign(n, 0);
    grad_h_.assign(n, 0);
    w_h_.assign(n, 0);
    dw_h_.assign(n, 0);
    off_end_.assign(n, 0);
    pre_end_.assign(n, 0);
    fwd_end_.assign(n, -1);
    bwd_start_.assign(n, -1);
  }

  Report run() {
    if (setup() && forward() && backward()) {
      rep_.pass = true;
      teardown();
    }
    finish();
    if (f_.trace) rep_.pool_trace = arena_.trace();
    return std::move(rep_);
  }

 private:
  bool two_buf() const { return d_.scheme == Scheme::TwoBuffer; }

  void emit(Lane s, Ev k, int layer, i64 a, i64 b, u64 bytes, const char* tag = "", int buf = kNone, u64 off = 0) {
    rep_.events.push_back(Event{s, k, layer, a, b, bytes, tag, buf, off});
  }

  // simulator.hpp:203-212
  std::optional<u64> take(u64 bytes, const char* tag, int buf, int layer, Stage st, i64 t, Lane s,
                          bool pin = false) {
    auto h = arena_.alloc(bytes, tag, t, pin);
    if (!h) {
      rep_.oom = Oom{layer, st, arena_.fragmented(bytes), bytes, tag};
      return std::nullopt;
    }
    emit(s, Ev::Alloc, layer, t, t, bytes, tag, buf, arena_.offset(*h));
    return h;
  }

  // simulator.hpp:214-220
  void give(u64 h, const char* tag, int buf, int layer, i64 t, Lane s) {
    const u64 off = arena_.offset(h), bytes = arena_.requested(h);
    emit(s, Ev::Release, layer, t, t, bytes, tag, buf, off);
    arena_.release(h, t);
  }

  bool setup() {  // simulator.hpp:222-273
    for (const Node& l : g_.nodes()) {
      const size_t i = static_cast<size_t>(l.id);
      if (lv_.wbytes[i] > 0) {
        auto h = take(lv_.wbytes[i], "W", l.id, l.id, Stage::Setup, 0, Lane::Compute, true);
        if (!h) return false;
        w_h_[i] = *h;
      }
      if (f_.with_dw && lv_.wbytes[i] > 0 && two_buf()) {
        auto h = take(lv_.wbytes[i], "dW", l.id, l.id, Stage::Setup, 0, Lane::Compute, true);
        if (!h) return false;
        dw_h_[i] = *h;
      }
      if (l.kind == Kind::Input) {
        auto h = take(lv_.feat[i], "X", l.id, l.id, Stage::Setup, 0, Lane::Compute, true);
        if (!h) return false;
        feat_h_[i] = *h;
        where_[i] = Where::Device;
      }
    }
    if (!two_buf()) return true;
    for (const Node& l : g_.nodes()) {
      const size_t i = static_cast<size_t>(l.id);
      if (l.kind == Kind::Input || lv_.feat[i] == 0) continue;
      auto h = take(lv_.feat[i], "Y", l.id, l.id, Stage::Setup, 0, Lane::Compute, true);
      if (!h) return false;
      feat_h_[i] = *h;
      where_[i] = Where::Device;
    }
    for (int k = 0; k < 2 && lv_.g2_bytes > 0; ++k) {
      auto h = take(lv_.g2_bytes, "G2", kNone, kNone, Stage::Setup, 0, Lane::Compute, true);
      if (!h) return false;
      g2_h_.push_back(*h);
    }
    if (lv_.ws2_bytes > 0) {
      auto h = take(lv_.ws2_bytes, "WS", kNone, kNone, Stage::Setup, 0, Lane::Compute, true);
      if (!h) return false;
      ws2_h_ = *h;
    }
    return true;
  }

  bool forward() {  // simulator.hpp:275-356
    for (const Node& l : g_.nodes()) {
      if (l.kind == Kind::Input) continue;
      const size_t i = static_cast<size_t>(l.id);
      const i64 t0 = compute_t_;
      std::optional<u64> ws;
      if (!two_buf()) {
        if (lv_.feat[i] > 0) {
          auto h = take(lv_.feat[i], "Y", l.id, l.id, Stage::Forward, t0, Lane::Compute);
          if (!h) return false;
          feat_h_[i] = *h;
          where_[i] = Where::Device;
        }
        if (lv_.wsbytes[i] > 0) {
          ws = take(lv_.wsbytes[i], "WS", l.id, l.id, Stage::Forward, t0, Lane::Compute);
          if (!ws) return false;
        }
      }
      const i64 t1 = t0 + lv_.fwd_ns[i];
      emit(Lane::Compute, Ev::Fwd, l.id, t0, t1, 0);
      fwd_end_[i] = t1;

      i64 drained = 0;
      for (int o : lv_.offloads_at[i]) {
        const size_t oi = static_cast<size_t>(o);
        const i64 a = std::max(t0, memory_t_);
        const i64 b = a + lv_.xfer_ns[oi];
        emit(Lane::Memory, Ev::Offload, l.id, a, b, lv_.feat[oi], "X", o);
        memory_t_ = b;
        where_[oi] = Where::Draining;
        off_end_[oi] = b;
        rep_.offload_bytes += lv_.feat[oi];
        host_.add(o, lv_.feat[oi], b);
        drained = b;
      }
      const i64 next = std::max(t1, drained);
      if (next > t1) {
        emit(Lane::Compute, Ev::Sync, l.id, t1, next, 0);
        rep_.stall_fwd += next - t1;
      }
      compute_t_ = next;

      if (two_buf()) {
        for (int o : lv_.owners_in[i]) --fwd_left_[static_cast<size_t>(o)];
        continue;
      }
      if (ws) give(*ws, "WS", l.id, l.id, t1, Lane::Compute);
      struct Rel {
        i64 t;
        int o;
        bool drained;
      };
      std::vector<Rel> rel;
      for (int o : lv_.owners_in[i]) {
        const size_t oi = static_cast<size_t>(o);
        if (--fwd_left_[oi] > 0) continue;
        if (where_[oi] == Where::Draining)
          rel.push_back({std::max(t1, off_end_[oi]), o, true});
        else if (bwd_left_[oi] == 0)
          rel.push_back({t1, o, false});
      }
      std::stable_sort(rel.begin(), rel.end(), [](const Rel& a, const Rel& b) { return a.t < b.t; });
      for (const Rel& r : rel) {
        const size_t oi = static_cast<size_t>(r.o);
        give(feat_h_[oi], "X", r.o, l.id, r.t, r.drained ? Lane::Memory : Lane::Compute);
        where_[oi] = r.drained ? Where::Host : Where::Gone;
      }
    }
    return true;
  }

  // simulator.hpp:475-483
  bool fits(int p, u64 step_need) const {
    u64 fetch = 0;
    for (int o : lv_.offloads_at[static_cast<size_t>(p)])
      if (where_[static_cast<size_t>(o)] == Where::Host) fetch += round_up(lv_.feat[static_cast<size_t>(o)], kAlign);
    return fetch + step_need <= arena_.largest_hole();
  }

  // simulator.hpp:485-511
  bool fetch(int o, int at, i64 t0, i64& end_out, bool opportunistic) {
    const size_t oi = static_cast<size_t>(o);
    auto h = arena_.alloc(lv_.feat[oi], "X", t0, false);
    if (!h && opportunistic) return true;
    if (!h) {
      rep_.oom = Oom{at, Stage::Backward, arena_.fragmented(lv_.feat[oi]), lv_.feat[oi], "X"};
      return false;
    }
    emit(Lane::Memory, Ev::Alloc, at, t0, t0, lv_.feat[oi], "X", o, arena_.offset(*h));
    feat_h_[oi] = *h;
    const i64 a = std::max(t0, memory_t_);
    const i64 b = a + lv_.xfer_ns[oi];
    emit(Lane::Memory, Ev::Prefetch, at, a, b, lv_.feat[oi], "X", o);
    memory_t_ = b;
    where_[oi] = Where::Filling;
    pre_end_[oi] = b;
    host_.remove(o, b);
    rep_.prefetch_bytes += lv_.feat[oi];
    end_out = std::max(end_out, b);
    return true;
  }

  bool backward() {  // simulator.hpp:358-471
    for (int m = lv_.L - 1; m >= 0; --m) {
      const Node& l = g_.at(m);
      if (l.kind == Kind::Input) continue;
      const size_t i = static_cast<size_t>(m);
      const i64 t0 = compute_t_;

      i64 queued = 0;
      if (auto p = prefetch_candidate(m, where_, lv_.offloads_at, g_)) {
        u64 need = 0;
        if (!two_buf()) {
          if (lv_.grad[i] > 0) need += round_up(lv_.grad[i], kAlign);
          if (lv_.wsbytes[i] > 0) need += round_up(lv_.wsbytes[i], kAlign);
          if (f_.with_dw) need += round_up(lv_.wbytes[i], kAlign);
        }
        if (fits(*p, need)) {
          for (int o : lv_.offloads_at[static_cast<size_t>(*p)]) {
            if (where_[static_cast<size_t>(o)] != Where::Host) continue;
            if (!fetch(o, *p, t0, queued, true)) return false;
          }
        }
      }

      i64 ready = t0;
      for (int o : lv_.bwd_reads[i]) {
        const size_t oi = static_cast<size_t>(o);
        if (where_[oi] == Where::Host) {
          i64 e = 0;
          if (!fetch(o, m, t0, e, false)) return false;
          ready = std::max(ready, e);
        } else if (where_[oi] == Where::Filling) {
          ready = std::max(ready, pre_end_[oi]);
        }
      }
      for (int o : lv_.bwd_reads[i]) {
        const size_t oi = static_cast<size_t>(o);
        if (where_[oi] == Where::Filling && pre_end_[oi] <= ready) where_[oi] = Where::Device;
      }
      if (ready > t0) {
        emit(Lane::Compute, Ev::Sync, m, t0, ready, 0);
        rep_.stall_bwd += ready - t0;
      }

      std::optional<u64> ws, dw;
      if (!two_buf()) {
        if (lv_.grad[i] > 0) {
          auto h = take(lv_.grad[i], "dX", m, m, Stage::Backward, ready, Lane::Compute);
          if (!h) return false;
          grad_h_[i] = *h;
        }
        if (lv_.wsbytes[i] > 0) {
          ws = take(lv_.wsbytes[i], "WS", m, m, Stage::Backward, ready, Lane::Compute);
          if (!ws) return false;
        }
        if (f_.with_dw && lv_.wbytes[i] > 0) {
          dw = take(lv_.wbytes[i], "dW", m, m, Stage::Backward, ready, Lane::Compute);
          if (!dw) return false;
        }
      }

      const i64 t1 = ready + lv_.bwd_ns[i];
      emit(Lane::Compute, Ev::Bwd, m, ready, t1, 0);
      bwd_start_[i] = ready;
      const i64 next = std::max(t1, queued);
      if (next > t1) {
        emit(Lane::Compute, Ev::Sync, m, t1, next, 0);
        rep_.stall_bwd += next - t1;
      }
      compute_t_ = next;
      for (size_t oi = 0; oi < static_cast<size_t>(lv_.L); ++oi)
        if (where_[oi] == Where::Filling && pre_end_[oi] <= next) where_[oi] = Where::Device;

      if (two_buf()) continue;
      if (ws) give(*ws, "WS", m, m, t1, Lane::Compute);
      if (dw) give(*dw, "dW", m, m, t1, Lane::Compute);
      for (int o : lv_.bwd_reads[i]) {
        const size_t oi = static_cast<size_t>(o);
        if (--bwd_left_[oi] > 0) continue;
        if (fwd_left_[oi] == 0 && where_[oi] == Where::Device) {
          give(feat_h_[oi], "Y", o, m, t1, Lane::Compute);
          where_[oi] = Where::Gone;
        }
      }
      for (int gb : lv_.grads_read[i]) {
        const size_t gi = static_cast<size_t>(gb);
        if (--grad_left_[gi] == 0) give(grad_h_[gi], "dX", gb, m, t1, Lane::Compute);
      }
      if (lv_.grad[i] > 0 && lv_.grad_users[i].empty()) give(grad_h_[i], "dX", m, m, t1, Lane::Compute);
    }
    return true;
  }

  void teardown() {  // simulator.hpp:513-527
    const i64 t = std::max(compute_t_, memory_t_);
    for (int id = 0; id < lv_.L; ++id) {
      const size_t i = static_cast<size_t>(id);
      if (where_[i] == Where::Device || where_[i] == Where::Draining || where_[i] == Where::Filling) {
        give(feat_h_[i], "Y", id, kNone, t, Lane::Compute);
        where_[i] = Where::Gone;
      }
      if (w_h_[i] != 0) give(w_h_[i], "W", id, kNone, t, Lane::Compute);
      if (dw_h_[i] != 0) give(dw_h_[i], "dW", id, kNone, t, Lane::Compute);
    }
    for (u64 h : g2_h_) give(h, "G2", kNone, kNone, t, Lane::Compute);
    if (ws2_h_ != 0) give(ws2_h_, "WS", kNone, kNone, t, Lane::Compute);
  }

  void finish() {  // simulator.hpp:529-545
    const i64 total = std::max(compute_t_, memory_t_);
    rep_.total = total;
    rep_.max_mem = arena_.peak();
    if (total > 0) rep_.avg_mem = static_cast<u64>(arena_.integral_until(total) / static_cast<u128>(total));
    rep_.host_peak = host_.peak();
    rep_.interference = c_.interference();
    rep_.reuse.assign(static_cast<size_t>(lv_.L), -1);
    for (size_t i = 0; i < static_cast<size_t>(lv_.L); ++i)
      if (fwd_end_[i] >= 0 && bwd_start_[i] >= 0) rep_.reuse[i] = bwd_start_[i] - fwd_end_[i];
  }

  const Net& g_;
  const Decision& d_;
  const Cost& c_;
  SimFlags f_;
  Liveness lv_;
  Arena arena_;
  PinnedLedger host_;
  Report rep_;
  i64 compute_t_ = 0, memory_t_ = 0;
  std::vector<Where> where_;
  std::vector<int> fwd_left_, bwd_left_, grad_left_;
  std::vector<u64> feat_h_, grad_h_, w_h_, dw_h_, g2_h_;
  u64 ws2_h_ = 0;
  std::vector<i64> off_end_, pre_end_, fwd_end_, bwd_start_;
};

}  // namespace

Report plan(const Net& g, const Decision& d, const Cost& c, u64 capacity, const SimFlags& f) {
  if (!g.finalized()) throw PlanError(Err::Generic, "graph is not finalized");
  d.check(g);
  Planner p(g, d, c, capacity, f);
  return p.run();
}

// FNV-1a-64 over "<stream>,<KIND>,<layer>,<bytes>,<tag>,<buffer>,<offset>;" of
// every non-FWD/BWD/SYNC event (SURVEY.md §8c schedule signature).
u64 schedule_signature(const Report& r) {
  u64 h = 1469598103934665603ull;
  auto feed = [&h](const std::string& s) {
    for (unsigned char ch : s) {
      h ^= ch;
      h *= 1099511628211ull;
    }
  };
  for (const Event& e : r.events) {
    if (e.kind == Ev::Fwd || e.kind == Ev::Bwd || e.kind == Ev::Sync) continue;
    feed(std::to_string(static_cast<int>(e.lane)) + "," + ev_name(e.kind) + "," + std::to_string(e.layer) + "," +
         std::to_string(e.bytes) + "," + e.tag + "," + std::to_string(e.buffer) + "," + std::to_string(e.off) + ";");
  }
  return h;
}

}  // namespace vdnnp
