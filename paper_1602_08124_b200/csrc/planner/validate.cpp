// Event-log validator (the contract of replay.hpp:95-304): checks any log --
// planned, or re-timed from CUDA events by the executor -- against its own
// reading of the graph's dataflow and a lifetime table of pool extents.
// Finding kinds are the reference's; the checks are grouped as
//   lanes      -- every timed event is well formed and a lane runs one
//                 transfer / kernel at a time;
//   pool       -- extents stay inside the capacity, never overlap while live,
//                 are opened / closed in pairs; high water and the
//                 time-weighted average equal the report's;
//   transfers  -- at most one offload / prefetch per buffer, only by flagged
//                 layers, every offload comes back (passing runs), and an
//                 offloaded extent is not released before its offload ends;
//   operands   -- every FWD/BWD finds its feature maps (and, per-layer
//                 scheme, its gradient maps) resident, prefetched data landed.
#include <algorithm>
#include <map>
#include <set>

#include "planner.hpp"

namespace vdnnp {

namespace {

struct Lifetime {  // one residency of a (class, buffer) in the pool
  i64 open = 0, close = -1;  // close = -1: still resident at the end of the log
};
using BufKey = std::pair<char, int>;  // class ('F' feature, 'G' dX, 'W', 'D' dW, 'S' WS) and buffer

char class_of(const std::string& tag) {
  if (tag == "X" || tag == "Y") return 'F';
  if (tag == "dX") return 'G';
  if (tag == "W") return 'W';
  if (tag == "dW") return 'D';
  if (tag == "WS") return 'S';
  return '?';
}

struct Checker {
  const Report& r;
  const Net& g;
  const Decision& d;
  u64 cap;
  std::vector<Finding> found;
  std::map<BufKey, std::vector<Lifetime>> lives;
  std::map<int, const Event*> first_out, first_in;  // buffer -> its first offload / prefetch
  int g2_seen = 0;

  void flag(const char* kind, std::string detail) { found.push_back({kind, std::move(detail)}); }

  // ------------------------------------------------------------- lanes --
  void lanes() {
    i64 busy_until[2] = {0, 0};
    for (const Event& e : r.events) {
      if (e.t1 < e.t0) flag("event-order", std::string(ev_name(e.kind)) + " finishes before it starts");
      const bool timed = e.kind == Ev::Fwd || e.kind == Ev::Bwd || e.kind == Ev::Offload || e.kind == Ev::Prefetch;
      if (!timed) continue;
      i64& b = busy_until[e.lane == Lane::Compute ? 0 : 1];
      if (e.t0 < b)
        flag("stream-overlap", std::string(ev_name(e.kind)) + "(" + std::to_string(e.layer) +
                                   ") starts while its lane is still busy");
      b = std::max(b, e.t1);
    }
  }

  // -------------------------------------------------------------- pool --
  void pool() {
    std::multimap<u64, u64> live;  // start -> end of live extents
    std::map<BufKey, i64> opened;
    u64 in_use = 0, high = 0;
    u128 area = 0;
    i64 now = 0;
    for (const Event& e : r.events) {
      if (e.kind != Ev::Alloc && e.kind != Ev::Release) continue;
      if (e.t0 < now) flag("pool-order", "pool event at " + std::to_string(e.t0) + " after one at " + std::to_string(now));
      area += static_cast<u128>(in_use) * static_cast<u128>(e.t0 - now);
      now = e.t0;
      const bool g2 = e.tag == "G2";
      const BufKey key{class_of(e.tag), e.buffer};
      if (e.kind == Ev::Alloc) {
        const u64 a = e.off, b = e.off + round_up(e.bytes, kAlign);
        if (b > cap) flag("capacity-breach", e.tag + "/" + std::to_string(e.buffer) + " ends past the pool");
        for (auto it = live.begin(); it != live.end() && it->first < b; ++it)
          if (it->second > a) {
            flag("pool-overlap", e.tag + "/" + std::to_string(e.buffer) + " at " + std::to_string(a) +
                                     " overlaps a live extent");
            break;
          }
        live.emplace(a, b);
        in_use += b - a;
        high = std::max(high, in_use);
        if (g2) {
          ++g2_seen;
          continue;
        }
        if (opened.count(key)) flag("double-alloc", e.tag + "/" + std::to_string(e.buffer) + " opened twice");
        opened[key] = e.t0;
      } else {
        auto it = live.find(e.off);
        if (it == live.end()) {
          flag("negative-count", "no live extent at " + std::to_string(e.off) + " to release");
        } else {
          in_use -= it->second - it->first;
          live.erase(it);
        }
        if (g2) continue;
        auto o = opened.find(key);
        if (o == opened.end()) {
          flag("negative-count", e.tag + "/" + std::to_string(e.buffer) + " released but not open");
          continue;
        }
        lives[key].push_back(Lifetime{o->second, e.t0});
        opened.erase(o);
      }
    }
    for (const auto& [key, t] : opened) lives[key].push_back(Lifetime{t, -1});
    if (high != r.max_mem) flag("report-mismatch", "high water " + std::to_string(high) + " vs reported " +
                                                     std::to_string(r.max_mem));
    if (r.total > 0) {
      area += static_cast<u128>(in_use) * static_cast<u128>(r.total - now);
      const u64 avg = static_cast<u64>(area / static_cast<u128>(r.total));
      if (avg != r.avg_mem) flag("report-mismatch", "average occupancy " + std::to_string(avg) + " vs reported " +
                                                      std::to_string(r.avg_mem));
    }
  }

  // --------------------------------------------------------- transfers --
  void transfers() {
    std::map<int, int> outs, ins;
    for (const Event& e : r.events) {
      if (e.kind == Ev::Offload && outs[e.buffer]++ == 0) first_out[e.buffer] = &e;
      if (e.kind == Ev::Prefetch && ins[e.buffer]++ == 0) first_in[e.buffer] = &e;
    }
    for (const auto& [b, n] : outs) {
      const std::string name = "buffer " + std::to_string(b);
      if (n > 1) flag("double-offload", name + " left the device " + std::to_string(n) + " times");
      if (!d.offloads(first_out[b]->layer))
        flag("unsanctioned-offload", name + " offloaded by unflagged layer " + std::to_string(first_out[b]->layer));
      if (r.pass && !ins.count(b)) flag("offload-not-prefetched", name + " never came back");
      // the device copy must outlive the offload that reads it
      auto lv = lives.find(BufKey{'F', b});
      if (lv == lives.end()) continue;
      const Event* off = first_out[b];
      for (const Lifetime& l : lv->second)
        if (l.open <= off->t0 && l.close >= 0 && l.close < off->t1)
          flag("release-before-offload-end", name + " released while its offload was in flight");
    }
    for (const auto& [b, n] : ins) {
      const std::string name = "buffer " + std::to_string(b);
      if (n > 1) flag("double-prefetch", name + " came back " + std::to_string(n) + " times");
      if (!outs.count(b)) flag("prefetch-without-offload", name + " prefetched but never offloaded");
    }
  }

  // ---------------------------------------------------------- operands --
  bool resident(char cls, int buffer, i64 a, i64 b) const {
    auto it = lives.find(BufKey{cls, buffer});
    if (it == lives.end()) return false;
    return std::any_of(it->second.begin(), it->second.end(),
                       [&](const Lifetime& l) { return l.open <= a && (l.close < 0 || l.close >= b); });
  }
  // a prefetched buffer is readable once its prefetch ended, or before its
  // offload began (the original copy)
  bool landed(int buffer, i64 a) const {
    auto in = first_in.find(buffer);
    if (in == first_in.end() || a >= in->second->t1) return true;
    auto out = first_out.find(buffer);
    return out != first_out.end() && a < out->second->t0;
  }

  int root(int id) const {
    for (int hop = 0; hop < (1 << 20) && g.at(id).kind == Kind::Actv; ++hop) id = g.at(id).in[0];
    return id;
  }
  std::set<int> feature_reads(int id, bool bwd) const {
    std::set<int> s;
    const Node& l = g.at(id);
    const bool reads_x = !bwd || l.kind == Kind::Conv || l.kind == Kind::Fc || l.kind == Kind::Pool;
    if (reads_x)
      for (int q : l.in) s.insert(root(q));
    if (bwd && l.kind == Kind::Pool) s.insert(id);
    if (bwd && l.kind == Kind::Actv) s.insert(root(id));
    return s;
  }
  bool owns_gradient(int id) const {
    const Node& l = g.at(id);
    if (l.kind == Kind::Actv || l.kind == Kind::Input) return false;
    return std::any_of(l.in.begin(), l.in.end(), [&](int q) { return g.at(root(q)).kind != Kind::Input; });
  }
  // dX maps BWD(m) takes as dY: its consumers', looking through in-place ACTVs
  void incoming(int m, std::set<int>& out) const {
    for (int c : g.users(m)) {
      if (g.at(c).kind == Kind::Actv) incoming(c, out);
      else if (owns_gradient(c)) out.insert(c);
    }
  }

  void operands() {
    const bool per_layer = d.scheme == Scheme::PerLayer;
    for (const Event& e : r.events) {
      if (e.kind != Ev::Fwd && e.kind != Ev::Bwd) continue;
      const bool bwd = e.kind == Ev::Bwd;
      const std::string step = std::string(bwd ? "BWD(" : "FWD(") + std::to_string(e.layer) + ")";
      for (int o : feature_reads(e.layer, bwd)) {
        if (!resident('F', o, e.t0, e.t1)) flag("use-after-release", step + " reads buffer " + std::to_string(o) +
                                                                         " while it is not resident");
        if (bwd && !landed(o, e.t0))
          flag("prefetch-before-use", step + " starts before buffer " + std::to_string(o) + " is back");
      }
      if (!bwd || !per_layer) continue;
      if (owns_gradient(e.layer) && !resident('G', e.layer, e.t0, e.t1))
        flag("use-after-release", step + " has no gradient map of its own");
      std::set<int> dy;
      incoming(e.layer, dy);
      for (int c : dy)
        if (!resident('G', c, e.t0, e.t1))
          flag("use-after-release", step + " reads the gradient of layer " + std::to_string(c) + " after release");
    }
    if (!per_layer && r.pass && max_grad_map_bytes(g, Cost{}) > 0 && g2_seen != 2)
      flag("missing-gradient-buffers", "two-buffer scheme provisioned " + std::to_string(g2_seen) +
                                           " gradient buffers instead of 2");
  }
};

}  // namespace

std::vector<Finding> validate_log(const Report& r, const Net& g, const Decision& d, u64 capacity) {
  Checker c{r, g, d, capacity, {}, {}, {}, {}, 0};
  c.lanes();
  c.pool();
  c.transfers();
  c.operands();
  return std::move(c.found);
}

}  // namespace vdnnp

namespace vdnnp {

// Consistency of a compiled Program with the event log of the same pass:
// walking the log with a step counter, every operand a step is bound to must
// lie inside the extent the log has live for that buffer at that moment, the
// scratch gap must not overlap any live extent, and every transfer must name
// the extent the log moved. This is what makes a stale binding (a gradient
// plane pointing at a recycled extent) a test failure on the CPU.
std::vector<Finding> check_program(const Program& P, const Report& r, const Net& g, const Decision& d) {
  std::vector<Finding> out;
  auto flag = [&](const std::string& k, const std::string& m) { out.push_back({k, m}); };
  struct Live {
    u64 end;
    std::string tag;
    int buffer;
  };
  std::map<u64, Live> live;
  auto inside = [&](u64 off, const char* tag_class, int buffer) {
    auto it = live.upper_bound(off);
    if (it == live.begin()) return false;
    --it;
    if (off >= it->second.end || it->second.buffer != buffer) return false;
    const std::string& t = it->second.tag;
    if (std::string(tag_class) == "F") return t == "X" || t == "Y";
    return t == tag_class;
  };
  const bool per_layer = d.scheme == Scheme::PerLayer;
  size_t si = 0;
  int xi = 0;
  for (const Event& e : r.events) {
    if (e.kind == Ev::Alloc) {
      live[e.off] = Live{e.off + round_up(e.bytes, kAlign), e.tag, e.buffer};
    } else if (e.kind == Ev::Release) {
      live.erase(e.off);
    } else if (e.kind == Ev::Offload || e.kind == Ev::Prefetch) {
      if (xi >= static_cast<int>(P.xfers.size())) {
        flag("program-xfer", "more transfers logged than compiled");
        continue;
      }
      const Xfer& x = P.xfers[static_cast<size_t>(xi++)];
      if (x.owner != e.buffer || x.bytes != e.bytes || x.to_host != (e.kind == Ev::Offload) ||
          !inside(x.dev_off, "F", x.owner) || x.step != static_cast<int>(si) - (e.kind == Ev::Offload ? 1 : 0))
        flag("program-xfer", std::string(ev_name(e.kind)) + " of buffer " + std::to_string(e.buffer) +
                                 " does not match compiled transfer " + std::to_string(xi - 1));
    } else if (e.kind == Ev::Fwd || e.kind == Ev::Bwd) {
      if (si >= P.steps.size()) {
        flag("program-step", "more steps logged than compiled");
        continue;
      }
      const Step& s = P.steps[si++];
      const std::string at = std::string(s.bwd ? "BWD(" : "FWD(") + std::to_string(s.layer) + ")";
      if (s.layer != e.layer || s.bwd != (e.kind == Ev::Bwd) || s.t0 != e.t0 || s.t1 != e.t1) {
        flag("program-step", at + " out of order with the log");
        continue;
      }
      const Node& l = g.at(s.layer);
      const bool reads_x = !s.bwd || l.kind == Kind::Conv || l.kind == Kind::Fc || l.kind == Kind::Pool;
      if (s.x.size() != l.in.size()) flag("program-operand", at + " input count");
      for (size_t j = 0; reads_x && j < s.x.size(); ++j)
        if (!inside(s.x[j], "F", g.owner(l.in[j]))) flag("program-operand", at + " input " + std::to_string(j));
      const bool has_y = s.bwd ? (l.kind == Kind::Pool || l.kind == Kind::Actv) : l.kind != Kind::Loss;
      if (has_y && !inside(s.y, "F", g.owner(s.layer))) flag("program-operand", at + " output map");
      if (l.kind == Kind::Conv || l.kind == Kind::Fc)
        if (!inside(s.w, "W", s.layer)) flag("program-operand", at + " weights");
      if (s.ws_bytes > 0 && per_layer && !inside(s.ws, "WS", s.layer)) flag("program-operand", at + " workspace");
      for (const auto& [off, lv] : live)
        if (s.gap_len > 0 && off < s.gap_off + s.gap_len && s.gap_off < lv.end)
          flag("program-gap", at + " scratch gap overlaps live " + lv.tag + "/" + std::to_string(lv.buffer));
      if (!s.bwd || !per_layer) continue;
      auto priv = [&](u64 off) { return off >= P.private_base && off < P.private_base + P.private_bytes; };
      for (const PlaneRef& p : s.dx)
        if (p.off != kNoLoc && (p.producer != s.layer || !(inside(p.off, "dX", s.layer) || priv(p.off))))
          flag("program-plane", at + " writes a plane outside its own dX");
      for (const PlaneRef& p : s.dy)
        if (!inside(p.off, "dX", p.producer) && !priv(p.off))
          flag("program-plane", at + " reads plane " + std::to_string(p.producer) + "/" + std::to_string(p.slot) +
                                    " outside the live dX of its producer");
    }
  }
  if (si != P.steps.size() || xi != static_cast<int>(P.xfers.size()))
    flag("program-step", "compiled steps/transfers not all in the log");
  return out;
}

}  // namespace vdnnp
