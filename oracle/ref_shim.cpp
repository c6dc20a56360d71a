// ORACLE / TEST INFRASTRUCTURE ONLY -- never linked into libvdnn.so.
//
// extern "C" shim over the *unmodified* reference simulator headers
// (/root/reference/proj/include/vdnnsim, compiled read-only by oracle/Makefile
// into oracle/_ref/libvdnnref.so). Used by tests/ (golden fixtures and
// differential fuzzing), by __graft_entry__.smoke() as the checker, and by
// bench.py's reference arm (timing the reference's own CPU path).
//
// Text interchange (kept trivial so the Python side can build it):
//   graph : "B=<batch>|<layer>|<layer>..."  layer = "<kind> <in0,in1,..> <p0> <p1> <p2> <p3> <join>"
//           kinds: input(p0..p2 = c,h,w) conv(k,s,p,out) actv pool(window,stride) fc(out) loss
//   cost  : "key=value,..." (pf,bw,cap,eff,lbw,lnom,lov,es,ratio,sfi,sfg,sff) + ";ov=id:f:b,id:f:b"
//   dec   : "static:<baseline|all|conv>:<m|p>" | "dyn" | "oracle" | "greedy:<conv|all>"
//           | "custom:<scheme 0|1>:<label>:<off ids ,>:<id=algo ,>"
// Results come back as a malloc'd JSON string (free with vref_free).
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <sstream>
#include <string>
#include <vector>

#include "vdnnsim/fuzz.hpp"
#include "vdnnsim/policy.hpp"
#include "vdnnsim/presets.hpp"
#include "vdnnsim/replay.hpp"
#include "vdnnsim/simulator.hpp"

using namespace vdnnsim;

namespace {

std::vector<std::string> split(const std::string& s, char sep) {
  std::vector<std::string> out;
  std::string cur;
  for (char c : s) {
    if (c == sep) {
      out.push_back(cur);
      cur.clear();
    } else {
      cur.push_back(c);
    }
  }
  out.push_back(cur);
  return out;
}

NetworkGraph parse_graph(const std::string& spec) {
  auto parts = split(spec, '|');
  NetworkGraph g(std::stoull(parts.at(0).substr(2)));
  for (size_t i = 1; i < parts.size(); ++i) {
    std::istringstream is(parts[i]);
    std::string kind, ins;
    unsigned long long p0, p1, p2, p3;
    int join;
    is >> kind >> ins >> p0 >> p1 >> p2 >> p3 >> join;
    std::vector<LayerId> in;
    if (ins != "-")
      for (auto& t : split(ins, ',')) in.push_back(std::stoi(t));
    const JoinRule j = join ? JoinRule::Elementwise : JoinRule::Concat;
    if (kind == "input") g.add_input(p0, p1, p2);
    else if (kind == "conv") g.add_conv(in, p3, p0, p1, p2, j);
    else if (kind == "actv") g.add_actv(in.at(0));
    else if (kind == "pool") g.add_pool(in, p0, p1, j);
    else if (kind == "fc") g.add_fc(in, p0, j);
    else if (kind == "loss") g.add_loss(in.at(0));
    else throw ConfigError("bad layer kind " + kind);
  }
  g.finalize();
  return g;
}

CostModel parse_cost(const std::string& spec) {
  CostModel cm;
  if (spec.empty()) return cm;
  auto halves = split(spec, ';');
  for (auto& kv : split(halves[0], ',')) {
    if (kv.empty()) continue;
    auto eq = kv.find('=');
    const std::string k = kv.substr(0, eq);
    const double v = std::strtod(kv.c_str() + eq + 1, nullptr);
    if (k == "pf") cm.device.peak_flops = v;
    else if (k == "bw") cm.device.dram_bw = v;
    else if (k == "cap") cm.device.mem_capacity = std::strtoull(kv.c_str() + eq + 1, nullptr, 10);
    else if (k == "eff") cm.device.compute_efficiency = v;
    else if (k == "lbw") cm.link.effective_bw = v;
    else if (k == "lnom") cm.link.nominal_bw = v;
    else if (k == "lov") cm.link.fixed_launch_overhead = v;
    else if (k == "es") cm.elem_size = std::strtoull(kv.c_str() + eq + 1, nullptr, 10);
    else if (k == "ratio") cm.bwd_fwd_ratio = v;
    else if (k == "sfi") cm.speed_factor_implicit_gemm = v;
    else if (k == "sfg") cm.speed_factor_gemm_ws = v;
    else if (k == "sff") cm.speed_factor_fft = v;
  }
  if (halves.size() > 1 && halves[1].rfind("ov=", 0) == 0) {
    for (auto& t : split(halves[1].substr(3), ',')) {
      if (t.empty()) continue;
      auto f = split(t, ':');
      cm.latency_overrides[std::stoi(f[0])] = {std::strtod(f[1].c_str(), nullptr), std::strtod(f[2].c_str(), nullptr)};
    }
  }
  return cm;
}

AlgoId algo_of(int a) { return a == 0 ? AlgoId::ImplicitGemm : (a == 1 ? AlgoId::GemmWs : AlgoId::Fft); }
int algo_int(AlgoId a) { return a == AlgoId::ImplicitGemm ? 0 : (a == AlgoId::GemmWs ? 1 : 2); }

std::string jstr(const std::string& s) {
  std::string o = "\"";
  for (char c : s) {
    if (c == '"' || c == '\\') o.push_back('\\');
    o.push_back(c);
  }
  return o + "\"";
}

std::string decision_json(const PolicyDecision& d) {
  std::ostringstream os;
  os << "{\"label\":" << jstr(d.label) << ",\"scheme\":" << (d.gradient_scheme == GradientScheme::PerLayer ? 1 : 0)
     << ",\"offload\":[";
  bool first = true;
  for (size_t i = 0; i < d.offload.size(); ++i)
    if (d.offload[i]) {
      os << (first ? "" : ",") << i;
      first = false;
    }
  os << "],\"algos\":{";
  first = true;
  for (const auto& [id, a] : d.algos) {
    os << (first ? "" : ",") << "\"" << id << "\":" << algo_int(a);
    first = false;
  }
  os << "}}";
  return os.str();
}

std::string oom_json(const std::optional<OomInfo>& o) {
  if (!o) return "null";
  std::ostringstream os;
  os << "{\"layer\":" << o->layer << ",\"phase\":" << int(o->phase) << ",\"fragmented\":" << (o->fragmented ? 1 : 0)
     << ",\"requested\":" << o->requested << ",\"tag\":" << jstr(o->tag) << "}";
  return os.str();
}

std::string signature(const RunReport& r) {
  std::uint64_t h = 1469598103934665603ull;
  for (const StreamEvent& e : r.events) {
    if (e.kind == EventKind::Fwd || e.kind == EventKind::Bwd || e.kind == EventKind::Sync) continue;
    const std::string s = std::to_string(int(e.stream)) + "," + to_string(e.kind) + "," + std::to_string(e.layer) +
                          "," + std::to_string(e.bytes) + "," + e.tag + "," + std::to_string(e.buffer) + "," +
                          std::to_string(e.offset) + ";";
    for (unsigned char c : s) {
      h ^= c;
      h *= 1099511628211ull;
    }
  }
  char buf[32];
  std::snprintf(buf, sizeof buf, "%016llx", static_cast<unsigned long long>(h));
  return buf;
}

std::string report_json(const RunReport& r, const NetworkGraph& g, const PolicyDecision& d, Bytes cap,
                        bool with_events) {
  std::ostringstream os;
  os << "{\"verdict\":" << jstr(r.verdict()) << ",\"pass\":" << (r.pass ? 1 : 0) << ",\"oom\":" << oom_json(r.oom)
     << ",\"max_mem_bytes\":" << r.max_mem_bytes << ",\"avg_mem_bytes\":" << r.avg_mem_bytes
     << ",\"offload_traffic_bytes\":" << r.offload_traffic_bytes
     << ",\"prefetch_traffic_bytes\":" << r.prefetch_traffic_bytes << ",\"host_peak_bytes\":" << r.host_peak_bytes
     << ",\"stall_fwd_offload_ns\":" << r.stall_fwd_offload_ns << ",\"stall_bwd_prefetch_ns\":"
     << r.stall_bwd_prefetch_ns << ",\"total_ns\":" << r.total_ns << ",\"n_events\":" << r.events.size()
     << ",\"signature\":\"" << signature(r) << "\",\"reuse_distance_ns\":[";
  for (size_t i = 0; i < r.reuse_distance_ns.size(); ++i) os << (i ? "," : "") << r.reuse_distance_ns[i];
  os << "]";
  std::vector<Bytes> fp, bp;
  detail::per_layer_event_peaks(r, fp, bp, g.size());
  os << ",\"fwd_peak\":[";
  for (size_t i = 0; i < fp.size(); ++i) os << (i ? "," : "") << fp[i];
  os << "],\"bwd_peak\":[";
  for (size_t i = 0; i < bp.size(); ++i) os << (i ? "," : "") << bp[i];
  os << "]";
  const auto viol = replay_check(r, g, d, cap);
  os << ",\"violations\":[";
  for (size_t i = 0; i < viol.size(); ++i) os << (i ? "," : "") << jstr(viol[i].kind);
  os << "]";
  if (with_events) {
    os << ",\"events\":[";
    for (size_t i = 0; i < r.events.size(); ++i) {
      const StreamEvent& e = r.events[i];
      os << (i ? "," : "") << "[" << int(e.stream) << "," << int(e.kind) << "," << e.layer << "," << e.start << ","
         << e.end << "," << e.bytes << "," << jstr(e.tag) << "," << e.buffer << "," << e.offset << "]";
    }
    os << "]";
  }
  os << "}";
  return os.str();
}

char* dup(const std::string& s) {
  char* p = static_cast<char*>(std::malloc(s.size() + 1));
  std::memcpy(p, s.c_str(), s.size() + 1);
  return p;
}

std::string run(const char* graph_spec, const char* cost_spec, const char* dec_spec, unsigned long long capacity,
                int flags) {
  const NetworkGraph g = parse_graph(graph_spec);
  const CostModel cm = parse_cost(cost_spec ? cost_spec : "");
  const std::string ds = dec_spec;
  SimOptions opt;
  opt.include_weight_grads = (flags & 2) != 0;
  const bool with_events = (flags & 1) != 0;
  std::ostringstream os;
  PolicyDecision d;
  std::string passes = "null";
  bool untrainable = false;
  if (ds == "dyn") {
    DynamicSelection sel = dynamic_select(g, capacity, cm);
    std::ostringstream ps;
    ps << "[";
    for (size_t i = 0; i < sel.passes.size(); ++i) {
      const auto& p = sel.passes[i];
      ps << (i ? "," : "") << "{\"phase\":" << jstr(p.phase) << ",\"label\":" << jstr(p.decision.label)
         << ",\"pass\":" << (p.pass ? 1 : 0) << ",\"oom\":" << oom_json(p.oom) << ",\"total_ns\":" << p.total_ns
         << ",\"max_mem_bytes\":" << p.max_mem_bytes << ",\"decision\":" << decision_json(p.decision) << "}";
    }
    ps << "]";
    passes = ps.str();
    if (sel.untrainable()) {
      untrainable = true;
    } else {
      d = *sel.decision;
    }
  } else if (ds == "oracle") {
    d = static_decision(PolicyKind::Baseline, AlgoMode::PerfOptimal, g, cm);
    d.label = "oracle";
    capacity = kUnlimitedBytes;
  } else if (ds.rfind("greedy:", 0) == 0) {
    const PolicyKind k = ds.substr(7) == "conv" ? PolicyKind::VdnnConv : PolicyKind::VdnnAll;
    std::vector<ProfilePassResult> tr;
    auto got = greedy_downgrade(g, capacity, k, cm, &tr);
    if (!got) untrainable = true;
    else d = *got;
  } else if (ds.rfind("static:", 0) == 0) {
    auto f = split(ds, ':');
    const PolicyKind k = f[1] == "baseline" ? PolicyKind::Baseline : (f[1] == "all" ? PolicyKind::VdnnAll : PolicyKind::VdnnConv);
    d = static_decision(k, f[2] == "m" ? AlgoMode::MemoryOptimal : AlgoMode::PerfOptimal, g, cm);
  } else if (ds.rfind("custom:", 0) == 0) {
    auto f = split(ds, ':');
    d.gradient_scheme = f[1] == "0" ? GradientScheme::TwoBufferReuse : GradientScheme::PerLayer;
    d.label = f[2];
    d.offload.assign(g.size(), 0);
    if (!f[3].empty())
      for (auto& t : split(f[3], ',')) d.offload.at(std::stoul(t)) = 1;
    if (!f[4].empty())
      for (auto& t : split(f[4], ',')) {
        auto kv = split(t, '=');
        d.algos[std::stoi(kv[0])] = algo_of(std::stoi(kv[1]));
      }
  } else {
    throw ConfigError("bad decision spec " + ds);
  }
  os << "{\"capacity\":" << capacity << ",\"untrainable\":" << (untrainable ? 1 : 0) << ",\"passes\":" << passes;
  if (!untrainable) {
    const RunReport r = simulate(g, d, cm, capacity, opt);
    os << ",\"decision\":" << decision_json(d) << ",\"report\":" << report_json(r, g, d, capacity, with_events);
  }
  os << "}";
  return os.str();
}

}  // namespace

extern "C" {

void vref_free(char* p) { std::free(p); }

// Returns JSON, or {"error": "..."} on exception.
char* vref_run(const char* graph_spec, const char* cost_spec, const char* dec_spec, unsigned long long capacity,
               int flags) {
  try {
    return dup(run(graph_spec, cost_spec, dec_spec, capacity, flags));
  } catch (const std::exception& e) {
    return dup(std::string("{\"error\":") + jstr(e.what()) + "}");
  }
}

static std::string graph_spec_of(const NetworkGraph& g);

char* vref_preset_spec(const char* name, unsigned long long batch, int extra) {
  try {
    NetworkGraph g = extra > 0 ? extend_vgg(extra, batch) : build_preset(name, batch);
    return dup(graph_spec_of(g));
  } catch (const std::exception& e) {
    return dup(std::string("ERROR:") + e.what());
  }
}

// The reference fuzz campaign's graph generator (fuzz.hpp:26-63) for one seed:
// the graphs its differential campaign plans, to be run on the GPU as well.
char* vref_fuzz_graph(unsigned long long seed, int max_layers) {
  try {
    std::mt19937_64 rng(seed);
    return dup(graph_spec_of(fuzzdetail::random_graph(rng, max_layers)));
  } catch (const std::exception& e) {
    return dup(std::string("ERROR:") + e.what());
  }
}

static std::string graph_spec_of(const NetworkGraph& g) {
  {
    std::ostringstream os;
    os << "B=" << g.batch();
    for (const LayerDescriptor& l : g.layers()) {
      os << "|" << to_string(l.kind) << " ";
      if (l.inputs.empty()) os << "-";
      for (size_t i = 0; i < l.inputs.size(); ++i) os << (i ? "," : "") << l.inputs[i];
      unsigned long long p[4] = {0, 0, 0, 0};
      if (l.conv) { p[0] = l.conv->kernel; p[1] = l.conv->stride; p[2] = l.conv->pad; p[3] = l.conv->out_channels; }
      if (l.pool) { p[0] = l.pool->window; p[1] = l.pool->stride; }
      if (l.fc) p[0] = l.fc->out_features;
      if (l.input) { p[0] = l.input->c; p[1] = l.input->h; p[2] = l.input->w; }
      os << " " << p[0] << " " << p[1] << " " << p[2] << " " << p[3] << " " << (l.join == JoinRule::Elementwise ? 1 : 0);
    }
    return os.str();
  }
}

// Replay-check an externally produced event log (e.g. measured on the GPU).
// events: n rows of 9 int64 (stream, kind, layer, start, end, bytes, tagcode, buffer, offset);
// tagcode 0..7 = "", W, dW, X, Y, dX, WS, G2. Returns JSON list of violation kinds.
char* vref_replay(const char* graph_spec, const char* dec_spec, unsigned long long capacity, const long long* ev,
                  long long n, unsigned long long max_mem, unsigned long long avg_mem, long long total_ns, int pass) {
  static const char* tags[] = {"", "W", "dW", "X", "Y", "dX", "WS", "G2"};
  try {
    const NetworkGraph g = parse_graph(graph_spec);
    PolicyDecision d;
    const std::string ds = dec_spec;
    auto f = split(ds, ':');
    d.gradient_scheme = f.at(1) == "0" ? GradientScheme::TwoBufferReuse : GradientScheme::PerLayer;
    d.offload.assign(g.size(), 0);
    if (!f[3].empty())
      for (auto& t : split(f[3], ',')) d.offload.at(std::stoul(t)) = 1;
    if (!f[4].empty())
      for (auto& t : split(f[4], ',')) {
        auto kv = split(t, '=');
        d.algos[std::stoi(kv[0])] = algo_of(std::stoi(kv[1]));
      }
    RunReport r;
    for (long long i = 0; i < n; ++i) {
      const long long* e = ev + 9 * i;
      StreamEvent s;
      s.stream = e[0] ? Stream::Memory : Stream::Compute;
      s.kind = static_cast<EventKind>(e[1]);
      s.layer = static_cast<LayerId>(e[2]);
      s.start = e[3];
      s.end = e[4];
      s.bytes = static_cast<Bytes>(e[5]);
      s.tag = tags[e[6]];
      s.buffer = static_cast<LayerId>(e[7]);
      s.offset = static_cast<Bytes>(e[8]);
      r.events.push_back(s);
    }
    r.max_mem_bytes = max_mem;
    r.avg_mem_bytes = avg_mem;
    r.total_ns = total_ns;
    r.pass = pass != 0;
    const auto v = replay_check(r, g, d, capacity);
    std::ostringstream os;
    os << "[";
    for (size_t i = 0; i < v.size(); ++i) os << (i ? "," : "") << "[" << jstr(v[i].kind) << "," << jstr(v[i].detail) << "]";
    os << "]";
    return dup(os.str());
  } catch (const std::exception& e) {
    return dup(std::string("{\"error\":") + jstr(e.what()) + "}");
  }
}

// Reference fuzz campaign (fuzz.hpp:89-158): returns trials and violations.
char* vref_fuzz(unsigned long long seed, int trials) {
  const FuzzResult r = run_fuzz_campaign(seed, trials);
  std::ostringstream os;
  os << "{\"trials\":" << r.trials << ",\"failed_trials\":" << r.failed_trials << ",\"violations\":" << r.violations << "}";
  return dup(os.str());
}

// Wall-clock seconds per call of the reference CPU path: dynamic_select (all
// profiling passes) + simulate of the chosen decision, averaged over iters.
double vref_time_plan(const char* graph_spec, unsigned long long capacity, int iters) {
  const NetworkGraph g = parse_graph(graph_spec);
  const CostModel cm;
  auto t0 = std::chrono::steady_clock::now();
  std::uint64_t sink = 0;
  for (int i = 0; i < iters; ++i) {
    DynamicSelection sel = dynamic_select(g, capacity, cm);
    if (sel.decision) sink += simulate(g, *sel.decision, cm, capacity).max_mem_bytes;
  }
  auto t1 = std::chrono::steady_clock::now();
  if (sink == 42) std::puts("");
  return std::chrono::duration<double>(t1 - t0).count() / iters;
}

}  // extern "C"
