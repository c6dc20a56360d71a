// Graph, presets, byte/latency formulas and footprint accounting.
#include <algorithm>
#include <bit>
#include <cmath>

#include "planner.hpp"

namespace vdnnp {

u64 mul_checked(u64 a, u64 b, const char* what) {  // core.hpp:34-40
  u64 r = 0;
  if (__builtin_mul_overflow(a, b, &r))
    throw PlanError(Err::Overflow, std::string(what) + ": product exceeds 64-bit range");
  return r;
}

i64 seconds_to_ns(double s) { return static_cast<i64>(std::llround(s * 1e9)); }  // core.hpp:46-48

const char* kind_name(Kind k) {
  switch (k) {
    case Kind::Input: return "input";
    case Kind::Conv: return "conv";
    case Kind::Actv: return "actv";
    case Kind::Pool: return "pool";
    case Kind::Fc: return "fc";
    case Kind::Loss: return "loss";
  }
  return "?";
}

u64 Dims::count() const {
  u64 e = mul_checked(n, c, "TensorShape");
  e = mul_checked(e, h, "TensorShape");
  return mul_checked(e, w, "TensorShape");
}

// ------------------------------------------------------------------ Net ---
int Net::add(Node n) {
  n.id = static_cast<int>(nodes_.size());
  nodes_.push_back(std::move(n));
  shapes_.clear();
  users_.clear();
  return nodes_.back().id;
}
int Net::input(u64 c, u64 h, u64 w) {
  Node n;
  n.kind = Kind::Input;
  n.ic = c;
  n.ih = h;
  n.iw = w;
  return add(std::move(n));
}
int Net::conv(std::vector<int> in, u64 out, u64 kernel, u64 stride, u64 pad, Join j) {
  Node n;
  n.kind = Kind::Conv;
  n.in = std::move(in);
  n.join = j;
  n.k = kernel;
  n.s = stride;
  n.p = pad;
  n.out = out;
  return add(std::move(n));
}
int Net::actv(int in) {
  Node n;
  n.kind = Kind::Actv;
  n.in = {in};
  return add(std::move(n));
}
int Net::pool(std::vector<int> in, u64 window, u64 stride, Join j) {
  Node n;
  n.kind = Kind::Pool;
  n.in = std::move(in);
  n.join = j;
  n.k = window;
  n.s = stride;
  return add(std::move(n));
}
int Net::fc(std::vector<int> in, u64 out, Join j) {
  Node n;
  n.kind = Kind::Fc;
  n.in = std::move(in);
  n.join = j;
  n.out = out;
  return add(std::move(n));
}
int Net::loss(int in) {
  Node n;
  n.kind = Kind::Loss;
  n.in = {in};
  return add(std::move(n));
}

// Structural rules of a layer list (net_graph.hpp:231-279): ids are
// positions, inputs point strictly backwards and are distinct, each kind has
// its arity and positive parameters.
void Net::check() const {
  if (batch_ < 1) throw PlanError(Err::Generic, "a graph needs a batch of at least 1");
  auto bad = [](const Node& l, const std::string& why) {
    return PlanError(Err::Generic, std::string(kind_name(l.kind)) + " layer " + std::to_string(l.id) + ": " + why);
  };
  for (size_t i = 0; i < nodes_.size(); ++i) {
    const Node& l = nodes_[i];
    if (l.id != static_cast<int>(i)) throw bad(l, "stored at position " + std::to_string(i));
    std::vector<int> seen;
    for (int q : l.in) {
      if (q < 0 || q >= l.id) throw bad(l, "input " + std::to_string(q) + " is not an earlier layer");
      if (std::find(seen.begin(), seen.end(), q) != seen.end())
        throw bad(l, "input " + std::to_string(q) + " listed twice");
      seen.push_back(q);
    }
    const size_t arity = l.in.size();
    bool ok = true;
    switch (l.kind) {
      case Kind::Input: ok = arity == 0 && l.ic >= 1 && l.ih >= 1 && l.iw >= 1; break;
      case Kind::Actv: ok = arity == 1; break;
      case Kind::Conv: ok = arity >= 1 && l.k >= 1 && l.s >= 1 && l.out >= 1; break;
      case Kind::Pool: ok = arity >= 1 && l.k >= 1 && l.s >= 1; break;
      case Kind::Fc: ok = arity >= 1 && l.out >= 1; break;
      case Kind::Loss: ok = arity >= 1; break;
    }
    if (!ok) throw bad(l, "wrong number of inputs (" + std::to_string(arity) + ") or a non-positive parameter");
  }
}

// Shape of a layer's joined input (net_graph.hpp:281-297): a concat stacks
// channels of maps that agree on n/h/w; an elementwise join needs equal shapes.
Dims Net::joined(const Node& l) const {
  Dims s = shapes_.at(static_cast<size_t>(l.in[0]));
  for (size_t i = 1; i < l.in.size(); ++i) {
    const Dims& t = shapes_.at(static_cast<size_t>(l.in[i]));
    const bool fits = l.join == Join::Concat ? (t.n == s.n && t.h == s.h && t.w == s.w) : t == s;
    if (!fits)
      throw PlanError(Err::Shape, "layer " + std::to_string(l.id) + ": input " + std::to_string(l.in[i]) +
                                      (l.join == Join::Concat ? " cannot be concatenated (n/h/w differ)"
                                                              : " cannot be summed (shape differs)"));
    if (l.join == Join::Concat) s.c += t.c;
  }
  return s;
}

// Shapes in id order (net_graph.hpp:299-358): conv (h + 2p - k)/s + 1 with
// exact division, pool floor((h - k)/s) + 1, FC (n, out, 1, 1), LOSS
// (n, 1, 1, 1), ACTV keeps its input's shape; then the consumer lists.
void Net::finalize() {
  check();
  shapes_.assign(nodes_.size(), Dims{});
  for (const Node& l : nodes_) {
    const size_t i = static_cast<size_t>(l.id);
    if (l.kind == Kind::Input) {
      shapes_[i] = Dims{batch_, l.ic, l.ih, l.iw};
      continue;
    }
    if (l.kind == Kind::Actv) {
      shapes_[i] = shapes_[static_cast<size_t>(l.in[0])];
      continue;
    }
    const Dims x = joined(l);
    auto shape_error = [&](const char* why) {
      return PlanError(Err::Shape, "layer " + std::to_string(l.id) + ": " + why);
    };
    if (l.kind == Kind::Conv) {
      const u64 h = x.h + 2 * l.p, w = x.w + 2 * l.p;
      if (h < l.k || w < l.k) throw shape_error("the filter does not fit the padded input");
      if ((h - l.k) % l.s || (w - l.k) % l.s) throw shape_error("stride does not divide the padded span");
      shapes_[i] = Dims{x.n, l.out, (h - l.k) / l.s + 1, (w - l.k) / l.s + 1};
    } else if (l.kind == Kind::Pool) {
      if (x.h < l.k || x.w < l.k) throw shape_error("the pooling window does not fit the input");
      shapes_[i] = Dims{x.n, x.c, (x.h - l.k) / l.s + 1, (x.w - l.k) / l.s + 1};
    } else if (l.kind == Kind::Fc) {
      shapes_[i] = Dims{x.n, l.out, 1, 1};
    } else {
      shapes_[i] = Dims{x.n, 1, 1, 1};
    }
  }
  users_.assign(nodes_.size(), {});
  for (const Node& l : nodes_)
    for (int q : l.in) users_[static_cast<size_t>(q)].push_back(l.id);
}

int Net::owner(int id) const {
  while (at(id).kind == Kind::Actv) id = at(id).in[0];
  return id;
}

Dims Net::in_dims(int id) const {
  const Node& l = at(id);
  if (l.in.empty()) return Dims{batch_, 0, 0, 0};
  Dims s = dims(l.in[0]);
  for (size_t i = 1; i < l.in.size(); ++i)
    if (l.join == Join::Concat) s.c += dims(l.in[i]).c;
  return s;
}

u64 Net::fc_inputs(int id) const {
  const Node& l = at(id);
  const Dims& first = dims(l.in[0]);
  u64 c = 0;
  for (int q : l.in) {
    if (l.join == Join::Concat)
      c += dims(q).c;
    else
      c = dims(q).c;
  }
  return c * first.h * first.w;
}

// -------------------------------------------------------------- presets ---
namespace {
int vgg_groups(Net& g, int prev, const std::vector<std::pair<u64, int>>& groups) {
  for (const auto& [ch, reps] : groups) {
    for (int i = 0; i < reps; ++i) prev = g.actv(g.conv({prev}, ch, 3, 1, 1));
    prev = g.pool({prev}, 2, 2);
  }
  return prev;
}

Net vgg(int extra, u64 batch) {  // presets.hpp:28-44 ("VGG-16" = 16 conv, groups {2,2,4,4,4})
  Net g(batch);
  int x = g.input(3, 224, 224);
  const std::pair<u64, int> base[] = {{64, 2}, {128, 2}, {256, 4}, {512, 4}, {512, 4}};
  std::vector<std::pair<u64, int>> groups;
  for (const auto& [c, r] : base) groups.emplace_back(c, r + extra);
  x = vgg_groups(g, x, groups);
  x = g.actv(g.fc({x}, 4096));
  x = g.actv(g.fc({x}, 4096));
  x = g.fc({x}, 1000);
  g.loss(x);
  g.finalize();
  return g;
}

Net alexnet(u64 batch) {  // presets.hpp:48-70
  Net g(batch);
  int x = g.input(3, 227, 227);
  x = g.pool({g.actv(g.conv({x}, 64, 11, 4, 0))}, 3, 2);
  x = g.pool({g.actv(g.conv({x}, 192, 5, 1, 2))}, 3, 2);
  x = g.actv(g.conv({x}, 384, 3, 1, 1));
  x = g.actv(g.conv({x}, 256, 3, 1, 1));
  x = g.pool({g.actv(g.conv({x}, 256, 3, 1, 1))}, 3, 2);
  x = g.actv(g.fc({x}, 4096));
  x = g.fc({x}, 1000);
  g.loss(x);
  g.finalize();
  return g;
}

Net overfeat(u64 batch) {  // presets.hpp:73-97
  Net g(batch);
  int x = g.input(3, 231, 231);
  x = g.pool({g.actv(g.conv({x}, 96, 11, 4, 0))}, 2, 2);
  x = g.pool({g.actv(g.conv({x}, 256, 5, 1, 0))}, 2, 2);
  x = g.actv(g.conv({x}, 512, 3, 1, 1));
  x = g.actv(g.conv({x}, 1024, 3, 1, 1));
  x = g.pool({g.actv(g.conv({x}, 1024, 3, 1, 1))}, 2, 2);
  x = g.actv(g.fc({x}, 3072));
  x = g.actv(g.fc({x}, 4096));
  x = g.fc({x}, 1000);
  g.loss(x);
  g.finalize();
  return g;
}

Net inception_toy(u64 batch) {  // presets.hpp:101-119
  Net g(batch);
  int x = g.input(3, 32, 32);
  const int fork = g.actv(g.conv({x}, 64, 3, 1, 1));
  const int a = g.actv(g.conv({fork}, 32, 1, 1, 0));
  const int b = g.actv(g.conv({fork}, 32, 3, 1, 1));
  const int c = g.actv(g.conv({fork}, 16, 5, 1, 2));
  x = g.pool({g.actv(g.conv({a, b, c}, 64, 3, 1, 1, Join::Concat))}, 2, 2);
  x = g.fc({x}, 10);
  g.loss(x);
  g.finalize();
  return g;
}
}  // namespace

Net make_preset(const std::string& name, u64 batch) {
  if (batch < 1) throw PlanError(Err::Generic, "batch must be >= 1");
  if (name == "vgg16") return vgg(0, batch);
  if (name == "alexnet") return alexnet(batch);
  if (name == "overfeat") return overfeat(batch);
  if (name == "inception_toy") return inception_toy(batch);
  throw PlanError(Err::Preset, "unknown network preset: " + name);
}

Net make_deep_vgg(int extra, u64 batch) {
  if (extra < 0 || extra % 100 != 0)
    throw PlanError(Err::Depth, "extra conv layers must be a non-negative multiple of 100 (20 per group)");
  return vgg(extra / 5, batch);
}

// ------------------------------------------------------------ cost model --
const char* algo_name(Algo a) {
  switch (a) {
    case Algo::Implicit: return "implicit_gemm";
    case Algo::GemmWs: return "gemm_ws";
    case Algo::Fft: return "fft";
  }
  return "?";
}

std::optional<Algo> step_down(Algo a) {
  if (a == Algo::Fft) return Algo::GemmWs;
  if (a == Algo::GemmWs) return Algo::Implicit;
  return std::nullopt;
}

double Cost::speed(Algo a) const {
  switch (a) {
    case Algo::Implicit: return sf_implicit;
    case Algo::GemmWs: return sf_gemm_ws;
    case Algo::Fft: return sf_fft;
  }
  return 1.0;
}

bool Cost::fft_ok(const Net& g, int id) const { return g.at(id).kind == Kind::Conv && g.at(id).s == 1; }
Algo Cost::fastest(const Net& g, int id) const { return fft_ok(g, id) ? Algo::Fft : Algo::GemmWs; }

// cost_model.hpp:95-121 -- multiplication order kept for bit-identical doubles.
double Cost::flop_count(const Net& g, int id, bool bwd) const {
  const Node& l = g.at(id);
  const Dims& o = g.dims(id);
  double f = 0.0;
  switch (l.kind) {
    case Kind::Conv: {
      const Dims x = g.in_dims(id);
      f = 2.0 * double(l.k) * double(l.k) * double(x.c) * double(o.c) * double(o.h) * double(o.w) * double(o.n);
      break;
    }
    case Kind::Actv:
      f = double(o.count());
      break;
    case Kind::Pool:
      f = double(l.k) * double(l.k) * double(o.count());
      break;
    case Kind::Fc:
      f = 2.0 * double(g.fc_inputs(id)) * double(l.out) * double(o.n);
      break;
    case Kind::Input:
    case Kind::Loss:
      return 0.0;
  }
  return bwd ? bwd_ratio * f : f;
}

u64 Cost::traffic_bytes(const Net& g, int id) const {  // cost_model.hpp:123-137
  switch (g.at(id).kind) {
    case Kind::Actv: return 2 * bytes_of(g.dims(id));
    case Kind::Pool: return bytes_of(g.in_dims(id)) + bytes_of(g.dims(id));
    case Kind::Fc: return weights(g, id) + bytes_of(g.in_dims(id)) + bytes_of(g.dims(id));
    default: return 0;
  }
}

double Cost::latency(const Net& g, int id, bool bwd, Algo a) const {  // cost_model.hpp:141-154
  if (auto it = pinned.find(id); it != pinned.end()) return bwd ? it->second.second : it->second.first;
  const Kind k = g.at(id).kind;
  if (k == Kind::Input || k == Kind::Loss) return 0.0;
  const double eff = compute_efficiency * peak_flops;
  const double ft = flop_count(g, id, bwd) / eff;
  if (k == Kind::Conv) return ft * speed(a);
  double bt = double(traffic_bytes(g, id)) / dram_bw;
  if (bwd) bt *= bwd_ratio;
  return std::max(ft, bt);
}

u64 Cost::workspace(const Net& g, int id, Algo a) const {  // cost_model.hpp:156-181
  const Node& l = g.at(id);
  if (l.kind != Kind::Conv) throw PlanError(Err::LayerKind, "conv_workspace on non-CONV layer");
  const Dims x = g.in_dims(id);
  const Dims& o = g.dims(id);
  if (a == Algo::Implicit) return 0;
  if (a == Algo::GemmWs) {
    u64 b = mul_checked(l.k * l.k, x.c, "workspace");
    b = mul_checked(b, o.h * o.w, "workspace");
    b = mul_checked(b, o.n, "workspace");
    return mul_checked(b, elem, "workspace");
  }
  const u64 ph = std::bit_ceil(x.h), pw = std::bit_ceil(x.w);
  u64 b = mul_checked(u64{2} * std::max(x.c, o.c), ph * pw, "workspace");
  b = mul_checked(b, o.n, "workspace");
  return mul_checked(b, elem, "workspace");
}

u64 Cost::weights(const Net& g, int id) const {  // cost_model.hpp:196-212
  const Node& l = g.at(id);
  if (l.kind == Kind::Conv) {
    const Dims x = g.in_dims(id);
    u64 b = mul_checked(l.k * l.k, x.c, "weights");
    b = mul_checked(b, l.out, "weights");
    return mul_checked(b, elem, "weights");
  }
  if (l.kind == Kind::Fc) {
    const u64 b = mul_checked(g.fc_inputs(id) + 1, l.out, "weights");
    return mul_checked(b, elem, "weights");
  }
  return 0;
}

// ------------------------------------------------------------ footprint ---
namespace {
void alias_readers(const Net& g, int owner, std::vector<int>& out) {
  for (int c : g.users(owner)) {
    out.push_back(c);
    if (g.at(c).kind == Kind::Actv) alias_readers(g, c, out);
  }
}
}  // namespace

bool counted_feature(const Net& g, int owner) {  // footprint.hpp:48-56
  const Kind k = g.at(owner).kind;
  if (k == Kind::Actv || k == Kind::Loss) return false;
  std::vector<int> r;
  alias_readers(g, owner, r);
  for (int x : r)
    if (g.at(x).kind != Kind::Loss) return true;
  return false;
}

u64 grad_map_bytes(const Net& g, int m, const Cost& c) {  // footprint.hpp:60-71
  const Node& l = g.at(m);
  if (l.kind == Kind::Actv || l.kind == Kind::Input) return 0;
  u64 total = 0;
  for (int q : l.in) {
    if (g.at(g.owner(q)).kind == Kind::Input) continue;
    const u64 b = c.bytes_of(g.dims(q));
    if (l.join == Join::Elementwise) return b;
    total += b;
  }
  return total;
}

u64 max_grad_map_bytes(const Net& g, const Cost& c) {
  u64 m = 0;
  for (const Node& l : g.nodes()) m = std::max(m, grad_map_bytes(g, l.id, c));
  return m;
}

Footprint footprint(const Net& g, const std::map<int, Algo>& algos, const Cost& c, bool with_dw) {
  Footprint r;
  for (const Node& l : g.nodes()) {
    u64 w = c.weights(g, l.id);
    if (with_dw) w *= 2;
    r.weights += w;
    if (l.kind == Kind::Fc) r.classifier += w;
    if (counted_feature(g, l.id)) {
      const u64 b = c.bytes_of(g.dims(l.id));
      r.features += b;
      if (l.kind == Kind::Fc) r.classifier += b;
    }
    if (l.kind == Kind::Conv) {
      auto it = algos.find(l.id);
      const Algo a = it == algos.end() ? Algo::Implicit : it->second;
      r.workspace = std::max(r.workspace, c.workspace(g, l.id, a));
    }
  }
  r.gradients = 2 * max_grad_map_bytes(g, c);
  r.total = r.weights + r.features + r.gradients + r.workspace;
  return r;
}

}  // namespace vdnnp
