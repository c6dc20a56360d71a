// Schedule compiler: turns (graph, decision, cost, capacity) into the
// executable Program (steps with bound operands, transfers, waits) and the
// reference-format event log of the same walk.
//
// Semantics are those of the reference simulator (simulator.hpp:30-584),
// restated here in terms of a per-buffer state machine driven by a two-lane
// clock:
//   * compute lane: FWD(n) in id order, then BWD(m) in reverse id order;
//   * memory lane: one OFFLOAD per buffer whose last forward reader flags
//     offloading, one PREFETCH per offloaded buffer in backward, serialized;
//   * sync rules: FWD(n+1) starts after n's offloads end (:315-322); BWD(m)
//     starts after the prefetches of its operands end (:400-413); the step
//     after BWD(m) starts after every prefetch issued during BWD(m) (:434-441);
//   * pool traffic on the double-ended arena (memory_pool.hpp:55-86) with the
//     reference's event order, so offsets and the log are bit-identical.
#include <algorithm>
#include <tuple>

#include "planner.hpp"

namespace vdnnp {

const char* ev_name(Ev e) {
  static const char* const names[] = {"FWD", "BWD", "OFFLOAD", "PREFETCH", "ALLOC", "RELEASE", "SYNC"};
  const int i = static_cast<int>(e);
  return i >= 0 && i < 7 ? names[i] : "?";
}

const char* stage_name(Stage s) {
  static const char* const names[] = {"setup", "forward", "backward"};
  const int i = static_cast<int>(s);
  return i >= 0 && i < 3 ? names[i] : "?";
}

std::string Report::verdict() const {  // sim_types.hpp:80-89
  if (pass) return "PASS";
  if (!oom) return "FAIL";
  return "OOM(layer=" + std::to_string(oom->layer) + ", phase=" + stage_name(oom->stage) +
         (oom->fragmented ? ", fragmented)" : ")");
}

// ----------------------------------------------------------- dataflow ----
namespace {

void sort_dedup(std::vector<int>& v) {
  std::sort(v.begin(), v.end());
  v.erase(std::unique(v.begin(), v.end()), v.end());
}

// The layers whose BWD consumes the gradient w.r.t. input q of a layer:
// q itself and, through in-place ACTVs, the chain down to the first layer
// that owns its output (simulator.hpp:113-130). Raw INPUT stops the walk.
void gradient_consumers(const Net& g, int q, std::vector<int>& out) {
  for (int cur = q; g.at(cur).kind != Kind::Input; cur = g.at(cur).in[0]) {
    out.push_back(cur);
    if (g.at(cur).kind != Kind::Actv) break;
  }
}

}  // namespace

Dataflow derive_dataflow(const Net& g, const Decision& d, const Cost& c) {
  Dataflow df;
  df.at.resize(static_cast<size_t>(g.size()));
  auto F = [&](int id) -> LayerFlow& { return df.at[static_cast<size_t>(id)]; };

  for (const Node& l : g.nodes()) {
    LayerFlow& f = F(l.id);
    const Algo algo = l.kind == Kind::Conv ? d.algos.at(l.id) : Algo::Implicit;
    if (l.kind != Kind::Actv && l.kind != Kind::Loss) {
      f.bytes = c.bytes_of(g.dims(l.id));
      f.copy_ns = seconds_to_ns(c.transfer(f.bytes));
    }
    f.w_bytes = c.weights(g, l.id);
    if (l.kind == Kind::Conv) f.ws_bytes = c.workspace(g, l.id, algo);
    f.fwd_ns = seconds_to_ns(c.latency(g, l.id, false, algo));
    f.bwd_ns = seconds_to_ns(c.latency(g, l.id, true, algo));

    for (int q : l.in) f.x_owners.push_back(g.owner(q));
    sort_dedup(f.x_owners);
    for (int o : f.x_owners) {
      ++F(o).fwd_readers;
      F(o).last_fwd_reader = l.id;  // ids ascend, so the last write is the last reader
    }
    // backward feature operands: CONV/FC read X, POOL reads X and its Y,
    // an in-place ACTV reads the map it aliases, LOSS reads nothing
    if (l.kind == Kind::Conv || l.kind == Kind::Fc || l.kind == Kind::Pool) f.bwd_operands = f.x_owners;
    if (l.kind == Kind::Pool) f.bwd_operands.push_back(l.id);
    if (l.kind == Kind::Actv) f.bwd_operands.push_back(g.owner(l.id));
    sort_dedup(f.bwd_operands);
    for (int o : f.bwd_operands) F(o).bwd_readers.push_back(l.id);

    f.dx_bytes = grad_map_bytes(g, l.id, c);
    if (f.dx_bytes > 0) {
      for (int q : l.in) gradient_consumers(g, q, f.dx_readers);
      sort_dedup(f.dx_readers);
      for (int r : f.dx_readers) F(r).dy_sources.push_back(l.id);
    }
  }
  for (LayerFlow& f : df.at) {
    sort_dedup(f.bwd_readers);
    sort_dedup(f.dy_sources);
  }
  // a flagged CONV/POOL drains each input buffer it is the last forward
  // reader of, when the backward pass reads that buffer again
  for (const Node& l : g.nodes()) {
    if (!d.offloads(l.id) || (l.kind != Kind::Conv && l.kind != Kind::Pool)) continue;
    for (int o : F(l.id).x_owners)
      if (F(o).last_fwd_reader == l.id && !F(o).bwd_readers.empty()) F(l.id).drains.push_back(o);
  }
  if (d.scheme == Scheme::TwoBuffer) {
    df.g2_bytes = max_grad_map_bytes(g, c);
    for (const LayerFlow& f : df.at) df.ws2_bytes = std::max(df.ws2_bytes, f.ws_bytes);
  }
  return df;
}

// ------------------------------------------------------------ compiler ----
namespace {

// Where a feature buffer's bytes are (sim_types.hpp:93-100).
enum class Res : unsigned char { Absent, OnDevice, GoingOut, OnHost, ComingIn, Retired };

struct BufState {
  Res res = Res::Absent;
  std::optional<u64> at;     // device extent while allocated
  int fwd_left = 0, bwd_left = 0;
  i64 out_done = 0, in_done = 0;  // planned end of its offload / prefetch
};

class Compiler {
 public:
  Compiler(const Net& g, const Decision& d, const Cost& c, u64 capacity, const SimFlags& f, Program* prog)
      : g_(g), d_(d), c_(c), f_(f), prog_(prog), df_(derive_dataflow(g, d, c)), pool_(capacity, f.trace),
        L_(static_cast<size_t>(g.size())), buf_(L_), dx_at_(L_), w_at_(L_), dw_at_(L_), dx_left_(L_, 0),
        fwd_end_(L_, -1), bwd_start_(L_, -1) {
    per_layer_ = d.scheme == Scheme::PerLayer;
    for (size_t i = 0; i < L_; ++i) {
      buf_[i].fwd_left = df_.at[i].fwd_readers;
      buf_[i].bwd_left = static_cast<int>(df_.at[i].bwd_readers.size());
      dx_left_[i] = static_cast<int>(df_.at[i].dx_readers.size());
    }
    if (prog_) *prog_ = Program{};
  }

  Report run() {
    const bool ok = provision() && forward_pass() && backward_pass();
    if (ok) {
      rep_.pass = true;
      teardown();
    }
    summarize();
    if (f_.trace) rep_.pool_trace = pool_.trace();
    if (prog_ && ok) finish_program();
    return std::move(rep_);
  }

 private:
  const LayerFlow& at(int id) const { return df_.at[static_cast<size_t>(id)]; }
  BufState& B(int id) { return buf_[static_cast<size_t>(id)]; }

  void log(Lane lane, Ev k, int layer, i64 a, i64 b, u64 bytes = 0, const std::string& tag = {}, int buffer = kNone,
           u64 off = 0) {
    rep_.events.push_back(Event{lane, k, layer, a, b, bytes, tag, buffer, off});
  }

  // Pool request logged as ALLOC; a failure records the OOM and stops the run.
  std::optional<u64> reserve(u64 bytes, const char* tag, int buffer, int layer, Stage stage, i64 t, Lane lane,
                             bool pinned = false) {
    std::optional<u64> off = pool_.place(bytes, tag, t, pinned);
    if (!off) {
      rep_.oom = Oom{layer, stage, pool_.would_fragment(bytes), bytes, tag};
      return std::nullopt;
    }
    log(lane, Ev::Alloc, layer, t, t, bytes, tag, buffer, *off);
    return off;
  }

  void unreserve(u64 off, const char* tag, int buffer, int layer, i64 t, Lane lane) {
    log(lane, Ev::Release, layer, t, t, pool_.requested_at(off), tag, buffer, off);
    pool_.free_at(off, t);
  }

  // ---------------------------------------------------------- provision --
  // Everything that lives for the whole iteration, pinned to the top of the
  // pool at t = 0 (simulator.hpp:222-273): per layer W, the two-buffer dW
  // mirror (with weight gradients on), the raw input; the two-buffer scheme
  // adds every feature map, two network-max gradient buffers and the
  // network-max workspace.
  bool provision() {
    struct Want {
      u64 bytes;
      const char* tag;
      int id;
      std::optional<u64>* slot;
    };
    std::vector<Want> wants;
    for (const Node& l : g_.nodes()) {
      const size_t i = static_cast<size_t>(l.id);
      if (at(l.id).w_bytes > 0) wants.push_back({at(l.id).w_bytes, "W", l.id, &w_at_[i]});
      if (at(l.id).w_bytes > 0 && f_.with_dw && !per_layer_) wants.push_back({at(l.id).w_bytes, "dW", l.id, &dw_at_[i]});
      if (l.kind == Kind::Input) wants.push_back({at(l.id).bytes, "X", l.id, &buf_[i].at});
    }
    if (!per_layer_) {
      for (const Node& l : g_.nodes())
        if (l.kind != Kind::Input && at(l.id).bytes > 0)
          wants.push_back({at(l.id).bytes, "Y", l.id, &buf_[static_cast<size_t>(l.id)].at});
      g2_.assign(df_.g2_bytes > 0 ? 2 : 0, std::nullopt);
      for (auto& s : g2_) wants.push_back({df_.g2_bytes, "G2", kNone, &s});
      if (df_.ws2_bytes > 0) wants.push_back({df_.ws2_bytes, "WS", kNone, &ws2_});
    }
    for (const Want& w : wants) {
      *w.slot = reserve(w.bytes, w.tag, w.id, w.id, Stage::Setup, 0, Lane::Compute, true);
      if (!*w.slot) return false;
      if (w.id != kNone && (std::string(w.tag) == "X" || std::string(w.tag) == "Y")) B(w.id).res = Res::OnDevice;
    }
    return true;
  }

  // ------------------------------------------------------------ forward --
  bool forward_pass() {
    for (const Node& l : g_.nodes()) {
      if (l.kind == Kind::Input) continue;
      const int n = l.id;
      const LayerFlow& f = at(n);
      const i64 t0 = clock_;
      std::optional<u64> ws;
      if (per_layer_) {
        if (f.bytes > 0) {
          B(n).at = reserve(f.bytes, "Y", n, n, Stage::Forward, t0, Lane::Compute);
          if (!B(n).at) return false;
          B(n).res = Res::OnDevice;
        }
        if (f.ws_bytes > 0 && !(ws = reserve(f.ws_bytes, "WS", n, n, Stage::Forward, t0, Lane::Compute))) return false;
      }
      const i64 t1 = t0 + f.fwd_ns;
      log(Lane::Compute, Ev::Fwd, n, t0, t1);
      fwd_end_[static_cast<size_t>(n)] = t1;
      Step* st = open_step(false, n, t0, t0, t1, ws);

      // drain the buffers this layer reads for the last time
      i64 drained = 0;
      for (int o : f.drains) {
        const i64 a = std::max(t0, lane_mem_), b = a + at(o).copy_ns;
        log(Lane::Memory, Ev::Offload, n, a, b, at(o).bytes, "X", o);
        lane_mem_ = b;
        B(o).res = Res::GoingOut;
        B(o).out_done = b;
        rep_.offload_bytes += at(o).bytes;
        ledger_add(o, at(o).bytes, b);
        note_xfer(st, true, o, a, b);
        drained = b;
      }
      clock_ = std::max(t1, drained);
      if (clock_ > t1) {
        log(Lane::Compute, Ev::Sync, n, t1, clock_);
        rep_.stall_fwd += clock_ - t1;
      }
      if (st) {
        st->wait_after = !f.drains.empty();
        st->t_leave = clock_;
      }

      for (int o : f.x_owners) --B(o).fwd_left;
      if (!per_layer_) continue;
      if (ws) unreserve(*ws, "WS", n, n, t1, Lane::Compute);
      // inputs read for the last time leave the pool: a drained one once its
      // offload is done (memory lane), one never read again at once
      std::vector<std::tuple<i64, int, bool>> out;  // (time, owner, drained)
      for (int o : f.x_owners) {
        if (B(o).fwd_left > 0) continue;
        if (B(o).res == Res::GoingOut) out.emplace_back(std::max(t1, B(o).out_done), o, true);
        else if (B(o).bwd_left == 0) out.emplace_back(t1, o, false);
      }
      std::sort(out.begin(), out.end());  // by time; x_owners ascend, so ties keep owner order
      for (const auto& [t, o, was_drained] : out) {
        unreserve(*B(o).at, "X", o, n, t, was_drained ? Lane::Memory : Lane::Compute);
        B(o).at.reset();
        B(o).res = was_drained ? Res::OnHost : Res::Retired;
      }
    }
    return true;
  }

  // ----------------------------------------------------------- backward --
  // The layer whose drained inputs the step below `m` should bring back:
  // the first one under m with a buffer still on the host, searching no
  // further than the first CONV (prefetch.hpp:16-23).
  std::optional<int> refill_target(int m) {
    for (int i = m - 1; i >= 0; --i) {
      for (int o : at(i).drains)
        if (B(o).res == Res::OnHost) return i;
      if (g_.at(i).kind == Kind::Conv) return std::nullopt;
    }
    return std::nullopt;
  }

  // H2D of buffer o into a fresh extent (simulator.hpp:485-511). An
  // opportunistic fetch that does not fit is skipped; a demanded one is OOM.
  bool refill(int o, int tagged_layer, i64 t0, Step* st, i64& landed, bool optional_fetch) {
    const u64 bytes = at(o).bytes;
    std::optional<u64> off = pool_.place(bytes, "X", t0, false);
    if (!off) {
      if (optional_fetch) return true;
      rep_.oom = Oom{tagged_layer, Stage::Backward, pool_.would_fragment(bytes), bytes, "X"};
      return false;
    }
    log(Lane::Memory, Ev::Alloc, tagged_layer, t0, t0, bytes, "X", o, *off);
    B(o).at = off;
    const i64 a = std::max(t0, lane_mem_), b = a + at(o).copy_ns;
    log(Lane::Memory, Ev::Prefetch, tagged_layer, a, b, bytes, "X", o);
    lane_mem_ = b;
    B(o).res = Res::ComingIn;
    B(o).in_done = b;
    ledger_remove(o, b);
    rep_.prefetch_bytes += bytes;
    note_xfer(st, false, o, a, b);
    landed = std::max(landed, b);
    return true;
  }

  bool backward_pass() {
    for (int m = g_.size() - 1; m >= 0; --m) {
      if (g_.at(m).kind == Kind::Input) continue;
      const LayerFlow& f = at(m);
      const i64 t0 = clock_;
      Step* st = open_step(true, m, t0, 0, 0, std::nullopt);

      // (1) opportunistic prefetch of the next drained layer's buffers, if
      // they and this step's own transients fit in the widest free gap
      i64 issued_end = 0;
      if (const std::optional<int> p = refill_target(m)) {
        u64 need = 0, fetch = 0;
        if (per_layer_) need = round_up(f.dx_bytes, kAlign) + round_up(f.ws_bytes, kAlign) +
                               (f_.with_dw ? round_up(f.w_bytes, kAlign) : 0);
        for (int o : at(*p).drains)
          if (B(o).res == Res::OnHost) fetch += round_up(at(o).bytes, kAlign);
        if (fetch + need <= pool_.widest_gap().second)
          for (int o : at(*p).drains)
            if (B(o).res == Res::OnHost && !refill(o, *p, t0, st, issued_end, true)) return false;
      }
      // (2) operands still on the host come back now; (3) wait for operands in flight
      i64 ready = t0;
      for (int o : f.bwd_operands) {
        if (B(o).res == Res::OnHost) {
          i64 e = 0;
          if (!refill(o, m, t0, st, e, false)) return false;
          ready = std::max(ready, e);
        } else if (B(o).res == Res::ComingIn) {
          ready = std::max(ready, B(o).in_done);
        }
      }
      for (int o : f.bwd_operands)
        if (B(o).res == Res::ComingIn) {
          if (st) st->wait_before.push_back(xfer_of_(o));
          if (B(o).in_done <= ready) B(o).res = Res::OnDevice;
        }
      if (ready > t0) {
        log(Lane::Compute, Ev::Sync, m, t0, ready);
        rep_.stall_bwd += ready - t0;
      }
      // (4) this step's transients, then the kernel
      std::optional<u64> ws, dw;
      if (per_layer_) {
        if (f.dx_bytes > 0) {
          dx_at_[static_cast<size_t>(m)] = reserve(f.dx_bytes, "dX", m, m, Stage::Backward, ready, Lane::Compute);
          if (!dx_at_[static_cast<size_t>(m)]) return false;
        }
        if (f.ws_bytes > 0 && !(ws = reserve(f.ws_bytes, "WS", m, m, Stage::Backward, ready, Lane::Compute))) return false;
        if (f_.with_dw && f.w_bytes > 0 && !(dw = reserve(f.w_bytes, "dW", m, m, Stage::Backward, ready, Lane::Compute)))
          return false;
      }
      const i64 t1 = ready + f.bwd_ns;
      log(Lane::Compute, Ev::Bwd, m, ready, t1);
      bwd_start_[static_cast<size_t>(m)] = ready;
      if (st) {
        st->t0 = ready;
        st->t1 = t1;
        bind_bwd(*st, ws);
      }
      // (5) the prefetches issued here land before the next step
      clock_ = std::max(t1, issued_end);
      if (clock_ > t1) {
        log(Lane::Compute, Ev::Sync, m, t1, clock_);
        rep_.stall_bwd += clock_ - t1;
      }
      if (st) {
        st->wait_after = !st->issues.empty();
        st->t_leave = clock_;
      }
      for (BufState& b : buf_)
        if (b.res == Res::ComingIn && b.in_done <= clock_) b.res = Res::OnDevice;

      if (!per_layer_) continue;
      // (6) retire what this step was the last user of
      if (ws) unreserve(*ws, "WS", m, m, t1, Lane::Compute);
      if (dw) unreserve(*dw, "dW", m, m, t1, Lane::Compute);
      for (int o : f.bwd_operands)
        if (--B(o).bwd_left == 0 && B(o).fwd_left == 0 && B(o).res == Res::OnDevice) {
          unreserve(*B(o).at, "Y", o, m, t1, Lane::Compute);
          B(o).at.reset();
          B(o).res = Res::Retired;
        }
      for (int src : f.dy_sources)
        if (--dx_left_[static_cast<size_t>(src)] == 0) retire_dx(src, m, t1);
      if (f.dx_bytes > 0 && f.dx_readers.empty()) retire_dx(m, m, t1);
    }
    return true;
  }

  void retire_dx(int producer, int layer, i64 t) {
    std::optional<u64>& a = dx_at_[static_cast<size_t>(producer)];
    unreserve(*a, "dX", producer, layer, t, Lane::Compute);
    a.reset();
  }

  // ------------------------------------------------------------ teardown --
  void teardown() {  // simulator.hpp:513-527
    const i64 t = std::max(clock_, lane_mem_);
    for (int id = 0; id < g_.size(); ++id) {
      const size_t i = static_cast<size_t>(id);
      const Res r = buf_[i].res;
      if (r == Res::OnDevice || r == Res::GoingOut || r == Res::ComingIn) {
        unreserve(*buf_[i].at, "Y", id, kNone, t, Lane::Compute);
        buf_[i].res = Res::Retired;
      }
      if (w_at_[i]) unreserve(*w_at_[i], "W", id, kNone, t, Lane::Compute);
      if (dw_at_[i]) unreserve(*dw_at_[i], "dW", id, kNone, t, Lane::Compute);
    }
    for (const auto& s : g2_) unreserve(*s, "G2", kNone, kNone, t, Lane::Compute);
    if (ws2_) unreserve(*ws2_, "WS", kNone, kNone, t, Lane::Compute);
  }

  void summarize() {  // simulator.hpp:529-545
    const i64 total = std::max(clock_, lane_mem_);
    rep_.total = total;
    rep_.max_mem = pool_.high_water();
    if (total > 0) rep_.avg_mem = static_cast<u64>(pool_.byte_ns_until(total) / static_cast<u128>(total));
    rep_.host_peak = host_peak_;
    rep_.interference = c_.interference();
    rep_.reuse.assign(L_, -1);
    for (size_t i = 0; i < L_; ++i)
      if (fwd_end_[i] >= 0 && bwd_start_[i] >= 0) rep_.reuse[i] = bwd_start_[i] - fwd_end_[i];
  }

  // pinned-host ledger (memory_pool.hpp:225-256): bytes held from offload
  // end to prefetch end
  void ledger_add(int o, u64 bytes, i64 t) {
    if (t < ledger_t_) throw PlanError(Err::Pool, "host ledger clock moved backwards");
    ledger_t_ = t;
    host_held_[o] += bytes;
    host_now_ += bytes;
    host_peak_ = std::max(host_peak_, host_now_);
  }
  void ledger_remove(int o, i64 t) {
    if (t < ledger_t_) throw PlanError(Err::Pool, "host ledger clock moved backwards");
    ledger_t_ = t;
    auto it = host_held_.find(o);
    if (it == host_held_.end()) throw PlanError(Err::Pool, "host ledger: buffer " + std::to_string(o) + " is not held");
    host_now_ -= it->second;
    host_held_.erase(it);
  }

  // -------------------------------------------------------- program side --
  Step* open_step(bool bwd, int layer, i64 enter, i64 t0, i64 t1, const std::optional<u64>& ws) {
    if (!prog_) return nullptr;
    prog_->steps.emplace_back();
    Step& s = prog_->steps.back();
    s.bwd = bwd;
    s.layer = layer;
    s.t_enter = enter;
    s.t0 = t0;
    s.t1 = t1;
    if (!bwd) bind_fwd(s, ws);
    return &s;
  }

  void note_xfer(Step* st, bool to_host, int owner, i64 a, i64 b) {
    if (!prog_) return;
    Xfer x;
    x.to_host = to_host;
    x.owner = owner;
    x.bytes = at(owner).bytes;
    x.dev_off = *B(owner).at;
    x.step = static_cast<int>(prog_->steps.size()) - 1;
    x.t0 = a;
    x.t1 = b;
    prog_->xfers.push_back(x);
    const int id = static_cast<int>(prog_->xfers.size()) - 1;
    if (!to_host) last_in_[owner] = id;
    if (st) st->issues.push_back(id);
  }
  int xfer_of_(int owner) const { return last_in_.at(owner); }

  u64 loc(const std::optional<u64>& o) const { return o ? *o : kNoLoc; }

  void bind_common(Step& s, const std::optional<u64>& ws) {
    const Node& l = g_.at(s.layer);
    for (int q : l.in) s.x.push_back(loc(B(g_.owner(q)).at));
    s.w = loc(w_at_[static_cast<size_t>(s.layer)]);
    const u64 wsb = at(s.layer).ws_bytes;
    if (wsb > 0) {
      s.ws = per_layer_ ? loc(ws) : loc(ws2_);
      s.ws_bytes = wsb;
    }
    const auto gap = pool_.widest_gap();
    s.gap_off = gap.first;
    s.gap_len = gap.second;
  }

  void bind_fwd(Step& s, const std::optional<u64>& ws) {
    bind_common(s, ws);
    const Node& l = g_.at(s.layer);
    if (l.kind == Kind::Actv) s.y = loc(B(g_.owner(s.layer)).at);
    else if (l.kind != Kind::Loss) s.y = loc(B(s.layer).at);
  }

  // offset of the plane of `producer`'s dX that holds input slot j
  u64 plane_rel(int producer, size_t j) const {
    const Node& l = g_.at(producer);
    if (l.join == Join::Elementwise) return 0;  // one shared plane (footprint.hpp:67)
    u64 rel = 0;
    for (size_t k = 0; k < j; ++k) {
      const int q = l.in[k];
      if (g_.at(g_.owner(q)).kind != Kind::Input) rel += c_.bytes_of(g_.dims(q));
    }
    return rel;
  }
  int plane_slot(int producer, size_t j) const {
    return g_.at(producer).join == Join::Elementwise ? 0 : static_cast<int>(j);
  }
  // A fold is recorded per chain (the buffer owner its steps lead to): a
  // shared plane folded into one chain's plane stays itself for the others.
  PlaneRef canon(PlaneRef p, int chain) const {
    for (auto it = folded_.find({p.producer, p.slot, chain}); it != folded_.end();
         it = folded_.find({p.producer, p.slot, chain}))
      p.producer = it->second.first, p.slot = it->second.second;
    return p;
  }
  // the one gradient map of an elementwise join over >= 2 non-INPUT inputs
  bool shared(const PlaneRef& p) const {
    const Node& l = g_.at(p.producer);
    if (l.kind == Kind::Actv || l.join != Join::Elementwise) return false;
    int n = 0;
    for (int q : l.in) n += g_.at(g_.owner(q)).kind != Kind::Input;
    return n >= 2;
  }
  u64 dx_base(int producer) const {
    if (auto it = private_plane_.find(producer); it != private_plane_.end()) return it->second;
    if (per_layer_) return loc(dx_at_[static_cast<size_t>(producer)]);
    return g2_slot_.at(static_cast<size_t>(producer));
  }

  void bind_bwd(Step& s, const std::optional<u64>& ws) {
    bind_common(s, ws);
    const int m = s.layer;
    const Node& l = g_.at(m);
    if (l.kind == Kind::Actv) s.y = loc(B(g_.owner(m)).at);
    else if (l.kind == Kind::Pool) s.y = loc(B(m).at);
    if (!per_layer_ && g2_slot_.empty()) assign_gradient_slots();
    if (at(m).dx_bytes > 0) {
      const u64 base = dx_base(m);
      for (size_t j = 0; j < l.in.size(); ++j) {
        PlaneRef p{m, plane_slot(m, j), kNoLoc};
        if (g_.at(g_.owner(l.in[j])).kind != Kind::Input) p.off = base + plane_rel(m, j);
        s.dx.push_back(p);
      }
      if (!per_layer_) s.dx_accumulate = g2_accum_[static_cast<size_t>(m)] != 0;
    }
    // incoming planes: of every dX map m reads, the planes whose input chain
    // passes through m; already-folded planes resolve to their fold target
    const int owner_m = g_.owner(m);
    for (int src : at(m).dy_sources) {
      const Node& sl = g_.at(src);
      for (size_t j = 0; j < sl.in.size(); ++j) {
        if (g_.at(g_.owner(sl.in[j])).kind == Kind::Input) continue;
        std::vector<int> chain;
        gradient_consumers(g_, sl.in[j], chain);
        if (std::find(chain.begin(), chain.end(), m) == chain.end()) continue;
        PlaneRef p = canon(PlaneRef{src, plane_slot(src, j), kNoLoc}, owner_m);
        if (!per_layer_) {  // two-buffer fork accumulation shares one slot
          auto it = g2_alias_.find(p.producer);
          if (it != g2_alias_.end()) p = canon(PlaneRef{it->second.first, it->second.second, kNoLoc}, owner_m);
        }
        if (std::find(s.dy.begin(), s.dy.end(), p) != s.dy.end()) continue;
        p.off = dx_base(p.producer) + plane_rel(p.producer, static_cast<size_t>(slot_input(p)));
        s.dy.push_back(p);
      }
    }
    // the fold goes into a plane of this chain's own when there is one
    std::stable_partition(s.dy.begin(), s.dy.end(), [&](const PlaneRef& p) { return !shared(p); });
    if (!s.dy.empty() && shared(s.dy[0])) {
      if (l.kind == Kind::Actv) {  // masked sum -> a private plane the rest of the chain reads
        const u64 bytes = c_.bytes_of(g_.dims(m));
        private_plane_[m] = private_mark_ + private_bytes_;
        private_bytes_ += round_up(bytes, kAlign);
        s.dx = {PlaneRef{m, 0, private_plane_[m]}};
        s.stage_dy = true;
        for (const PlaneRef& p : s.dy) folded_[{p.producer, p.slot, owner_m}] = {m, 0};
      } else {
        s.stage_dy = s.dy.size() > 1;  // the kernels read the sum from the step's scratch
      }
    } else {
      for (size_t k = 1; k < s.dy.size(); ++k)
        folded_[{s.dy[k].producer, s.dy[k].slot, owner_m}] = {s.dy[0].producer, s.dy[0].slot};
    }
    bwd_step_of_[m] = static_cast<int>(prog_->steps.size()) - 1;
    if (l.kind == Kind::Actv && s.dy.size() == 1 && !s.stage_dy) find_mask_host(s);
  }

  // An ACTV's backward (dY *= (y > 0)) can run in the epilogue of the one
  // step that writes its incoming plane when that plane has no other
  // contributor (nothing folded or accumulated into it), the writer is a
  // CONV/FC dgrad or POOL backward reading the ACTV's output as that input,
  // and the plane is not shared by an elementwise join.
  void find_mask_host(Step& s) {
    const PlaneRef p = s.dy[0];
    for (const auto& [from, to] : folded_)
      if (to == std::make_pair(p.producer, p.slot)) return;
    if (shared(p)) return;
    for (const auto& [acc, to] : g2_alias_)
      if (to.first == p.producer) return;
    const Node& pl = g_.at(p.producer);
    if (pl.kind != Kind::Conv && pl.kind != Kind::Fc && pl.kind != Kind::Pool) return;
    if (pl.join == Join::Elementwise && pl.in.size() > 1) return;
    if (pl.in[static_cast<size_t>(p.slot)] != s.layer) return;
    auto it = bwd_step_of_.find(p.producer);
    if (it == bwd_step_of_.end()) return;
    if (prog_->steps[static_cast<size_t>(it->second)].dx_accumulate) return;
    s.mask_host = it->second;
    s.mask_slot = p.slot;
  }
  int slot_input(const PlaneRef& p) const {
    if (g_.at(p.producer).join != Join::Elementwise) return p.slot;
    const Node& l = g_.at(p.producer);  // shared plane: first non-INPUT input
    for (size_t j = 0; j < l.in.size(); ++j)
      if (g_.at(g_.owner(l.in[j])).kind != Kind::Input) return static_cast<int>(j);
    return 0;
  }

  // Two-buffer scheme: the plan provisions two network-max gradient buffers
  // (simulator.hpp:259-264) and no per-layer dX. Producers take a slot in
  // backward order; a single-plane producer whose gradient is w.r.t. the same
  // tensor as a live one accumulates into that slot (the fork sum). Should
  // more than two maps be live at once, extra slots follow the arena
  // (Program::overflow_*).
  void assign_gradient_slots() {
    g2_slot_.assign(L_, kNoLoc);
    g2_accum_.assign(L_, 0);
    std::vector<u64> base;
    for (const auto& s : g2_) base.push_back(*s);
    const u64 slot_bytes = round_up(df_.g2_bytes, kAlign);
    // input index of a producer's only gradient plane (kNone: several / none)
    auto single_plane = [&](int p) -> int {
      int j1 = kNone, count = 0;
      const Node& l = g_.at(p);
      for (size_t j = 0; j < l.in.size(); ++j)
        if (g_.at(g_.owner(l.in[j])).kind != Kind::Input) j1 = static_cast<int>(j), ++count;
      return count == 1 ? j1 : kNone;
    };
    auto plane_tensor = [&](int p) {
      const int j = single_plane(p);
      return j == kNone ? kNone : g_.at(p).in[static_cast<size_t>(j)];
    };
    std::vector<std::vector<int>> holders;  // per slot: live producers
    std::vector<int> slot_of(L_, -1), left(L_, 0);
    for (int m = g_.size() - 1; m >= 0; --m) {
      const size_t i = static_cast<size_t>(m);
      if (g_.at(m).kind == Kind::Input) continue;
      if (at(m).dx_bytes > 0) {
        const int q = plane_tensor(m);
        int host = kNone;
        for (size_t sl = 0; sl < holders.size() && host == kNone && q != kNone; ++sl)
          for (int p : holders[sl])
            if (plane_tensor(p) == q) {
              host = p;
              break;
            }
        if (host != kNone) {
          slot_of[i] = slot_of[static_cast<size_t>(host)];
          g2_accum_[i] = 1;
          const int h = canon_host(host);
          g2_alias_[m] = {h, plane_slot(h, static_cast<size_t>(single_plane(h)))};
        } else {
          int sl = 0;
          while (sl < static_cast<int>(holders.size()) && !holders[static_cast<size_t>(sl)].empty()) ++sl;
          if (sl == static_cast<int>(holders.size())) holders.emplace_back();
          slot_of[i] = sl;
        }
        holders[static_cast<size_t>(slot_of[i])].push_back(m);
        left[i] = static_cast<int>(at(m).dx_readers.size());
        const int sl = slot_of[i];
        if (sl < static_cast<int>(base.size())) {
          g2_slot_[i] = base[static_cast<size_t>(sl)];
        } else {
          const int extra = sl - static_cast<int>(base.size());
          overflow_slots_ = std::max(overflow_slots_, extra + 1);
          g2_slot_[i] = overflow_mark_ + static_cast<u64>(extra) * slot_bytes;
        }
      }
      auto drop = [&](int p) {
        auto& h = holders[static_cast<size_t>(slot_of[static_cast<size_t>(p)])];
        h.erase(std::remove(h.begin(), h.end(), p), h.end());
      };
      for (int src : at(m).dy_sources)
        if (--left[static_cast<size_t>(src)] == 0) drop(src);
      if (at(m).dx_bytes > 0 && at(m).dx_readers.empty()) drop(m);
    }
  }
  int canon_host(int p) const {
    auto it = g2_alias_.find(p);
    return it == g2_alias_.end() ? p : it->second.first;
  }

  void finish_program() {
    Program& P = *prog_;
    P.w_off.assign(L_, kNoLoc);
    for (size_t i = 0; i < L_; ++i) P.w_off[i] = loc(w_at_[i]);
    u64 lo = ~u64{0}, hi = 0;
    for (const Event& e : rep_.events)
      if (e.kind == Ev::Alloc) {
        lo = std::min(lo, e.off);
        hi = std::max(hi, e.off + round_up(e.bytes, kAlign));
      }
    P.arena_lo = hi > lo ? lo : 0;
    P.arena_hi = hi;
    // a step's scratch gap is only usable inside the span the executor maps
    for (Step& st : P.steps) {
      const u64 g0 = std::max(st.gap_off, P.arena_lo), g1 = std::min(st.gap_off + st.gap_len, P.arena_hi);
      st.gap_off = g1 > g0 ? g0 : 0;
      st.gap_len = g1 > g0 ? g1 - g0 : 0;
    }
    // overflow gradient slots sit right after the planned span; rebase the
    // placeholder offsets handed out during binding
    P.overflow_slots = overflow_slots_;
    P.overflow_slot_bytes = round_up(df_.g2_bytes, kAlign);
    P.overflow_base = hi;
    if (overflow_slots_ > 0) {
      auto fix = [&](u64& off) {
        if (off != kNoLoc && off >= overflow_mark_) off = off - overflow_mark_ + hi;
      };
      for (Step& s : P.steps) {
        for (PlaneRef& p : s.dx) fix(p.off);
        for (PlaneRef& p : s.dy) fix(p.off);
      }
    }
    P.private_base = hi + static_cast<u64>(overflow_slots_) * P.overflow_slot_bytes;
    P.private_bytes = private_bytes_;
    if (private_bytes_ > 0) {
      auto fix = [&](u64& off) {
        if (off != kNoLoc && off >= private_mark_ && off < overflow_mark_) off = off - private_mark_ + P.private_base;
      };
      for (Step& s : P.steps) {
        for (PlaneRef& p : s.dx) fix(p.off);
        for (PlaneRef& p : s.dy) fix(p.off);
      }
    }
    // the INPUT layer's setup extent and the last step that touches it
    for (const Node& l : g_.nodes())
      if (l.kind == Kind::Input && P.input == kNone) P.input = l.id;
    if (P.input != kNone) {
      for (const Event& e : rep_.events)
        if (e.kind == Ev::Alloc && e.buffer == P.input && e.tag == "X") {
          P.input_off = e.off;
          break;
        }
      idle_after_input(P);
      // once the next batch may be landing in the INPUT extent, a step's
      // scratch gap must stay clear of it: keep the wider side
      if (P.input_idle_after >= 0) {
        const u64 a0 = P.input_off, a1 = a0 + round_up(at(P.input).bytes, kAlign);
        for (size_t k = static_cast<size_t>(P.input_idle_after) + 1; k < P.steps.size(); ++k) {
          Step& st = P.steps[k];
          const u64 g0 = st.gap_off, g1 = st.gap_off + st.gap_len;
          if (g1 <= a0 || a1 <= g0) continue;
          const u64 left = a0 > g0 ? a0 - g0 : 0, right = g1 > a1 ? g1 - a1 : 0;
          if (left >= right) st.gap_len = left;
          else st.gap_off = a1, st.gap_len = right;
        }
      }
    }
  }

  // Walk the log with a step counter: every ALLOC whose extent overlaps the
  // INPUT extent, and the release of such an allocation, marks the step it
  // belongs to as touching the extent (a RELEASE on the memory lane closes a
  // drained buffer only after its offload; it belongs to the step whose
  // kernel it follows). The INPUT itself stays touched while any later
  // step reads it.
  void idle_after_input(Program& P) {
    const u64 a0 = P.input_off, a1 = a0 + round_up(at(P.input).bytes, kAlign);
    int step = -1, last = -1;
    std::map<u64, u64> live;  // overlapping live extents: off -> end
    for (const Event& e : rep_.events) {
      if (e.kind == Ev::Fwd || e.kind == Ev::Bwd) {
        ++step;
        if (!live.empty()) last = step;
        continue;
      }
      if (e.layer == kNone && e.kind == Ev::Release) continue;  // teardown
      if (e.kind == Ev::Alloc) {
        const u64 b = e.off + round_up(e.bytes, kAlign);
        if (e.off < a1 && a0 < b) {
          live[e.off] = b;
          last = std::max(last, step + 1);  // the extent is written by the next kernel (or a prefetch in it)
        }
      } else if (e.kind == Ev::Release) {
        if (live.erase(e.off)) last = std::max(last, step);
      }
    }
    const int nsteps = static_cast<int>(P.steps.size());
    P.input_idle_after = (!live.empty() || last >= nsteps - 1) ? -1 : std::max(last, 0);
  }

  const Net& g_;
  const Decision& d_;
  const Cost& c_;
  SimFlags f_;
  Program* prog_;
  Dataflow df_;
  Arena pool_;
  size_t L_;
  bool per_layer_ = true;
  Report rep_;
  i64 clock_ = 0, lane_mem_ = 0;
  std::vector<BufState> buf_;
  std::vector<std::optional<u64>> dx_at_, w_at_, dw_at_, g2_;
  std::optional<u64> ws2_;
  std::vector<int> dx_left_;
  std::vector<i64> fwd_end_, bwd_start_;
  std::map<int, u64> host_held_;
  u64 host_now_ = 0, host_peak_ = 0;
  i64 ledger_t_ = 0;
  // program binding state
  std::map<int, int> last_in_;                               // owner -> its prefetch xfer
  std::map<std::tuple<int, int, int>, std::pair<int, int>> folded_;  // (plane, chain) -> plane it was folded into
  std::map<int, u64> private_plane_;                         // ACTV -> its private plane (marker offset)
  u64 private_bytes_ = 0;
  static constexpr u64 private_mark_ = u64{1} << 62;
  std::vector<u64> g2_slot_;
  std::vector<char> g2_accum_;
  std::map<int, std::pair<int, int>> g2_alias_;
  std::map<int, int> bwd_step_of_;                           // layer -> its BWD step index
  int overflow_slots_ = 0;
  static constexpr u64 overflow_mark_ = u64{1} << 63;
};

}  // namespace

Report plan(const Net& g, const Decision& d, const Cost& c, u64 capacity, const SimFlags& f, Program* prog) {
  if (!g.finalized()) throw PlanError(Err::Generic, "graph is not finalized");
  d.check(g);
  return Compiler(g, d, c, capacity, f, prog).run();
}

// FNV-1a-64 over "<stream>,<KIND>,<layer>,<bytes>,<tag>,<buffer>,<offset>;" of
// every event that is not FWD/BWD/SYNC (SURVEY.md §8c schedule signature).
u64 schedule_signature(const Report& r) {
  u64 h = 1469598103934665603ull;
  for (const Event& e : r.events) {
    if (e.kind == Ev::Fwd || e.kind == Ev::Bwd || e.kind == Ev::Sync) continue;
    const std::string row = std::to_string(static_cast<int>(e.lane)) + "," + ev_name(e.kind) + "," +
                            std::to_string(e.layer) + "," + std::to_string(e.bytes) + "," + e.tag + "," +
                            std::to_string(e.buffer) + "," + std::to_string(e.off) + ";";
    for (unsigned char ch : row) h = (h ^ ch) * 1099511628211ull;
  }
  return h;
}

}  // namespace vdnnp
