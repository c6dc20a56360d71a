// ORACLE / TEST INFRASTRUCTURE ONLY -- never linked into libvdnn.so.
//
// extern "C" shim over the reference's front-end and artefact formats
// (vdnnsim/config.hpp INI reader + build_network, vdnnsim/report.hpp JSON
// writers), compiled from the unmodified headers in place by oracle/Makefile
// into oracle/_ref/libvdnnref_fmt.so. nlohmann/json is the copy vendored in
// the image (cudnn_frontend/thirdparty, v3.11.3), since the reference's own
// vendor/ directory is absent. Used only by tests/test_formats.py.
#include <cstdlib>
#include <cstring>
#include <sstream>
#include <string>

#include "vdnnsim/config.hpp"
#include "vdnnsim/policy.hpp"
#include "vdnnsim/report.hpp"
#include "vdnnsim/simulator.hpp"

using namespace vdnnsim;

namespace {

char* dup(const std::string& s) {
  char* p = static_cast<char*>(std::malloc(s.size() + 1));
  std::memcpy(p, s.c_str(), s.size() + 1);
  return p;
}

// graph -> the text spec of ref_shim.cpp ("B=<batch>|<kind> <ins> p0 p1 p2 p3 join|...")
std::string spec_of(const NetworkGraph& g) {
  std::ostringstream os;
  os << "B=" << g.batch();
  for (const LayerDescriptor& l : g.layers()) {
    os << "|" << to_string(l.kind) << " ";
    if (l.inputs.empty()) os << "-";
    for (size_t i = 0; i < l.inputs.size(); ++i) os << (i ? "," : "") << l.inputs[i];
    unsigned long long p[4] = {0, 0, 0, 0};
    if (l.conv) {
      p[0] = l.conv->kernel;
      p[1] = l.conv->stride;
      p[2] = l.conv->pad;
      p[3] = l.conv->out_channels;
    } else if (l.pool) {
      p[0] = l.pool->window;
      p[1] = l.pool->stride;
    } else if (l.fc) {
      p[0] = l.fc->out_features;
    } else if (l.input) {
      p[0] = l.input->c;
      p[1] = l.input->h;
      p[2] = l.input->w;
    }
    os << " " << p[0] << " " << p[1] << " " << p[2] << " " << p[3] << " "
       << (l.join == JoinRule::Elementwise ? 1 : 0);
  }
  return os.str();
}

NetworkGraph graph_of_spec(const std::string& spec);  // defined below (same format as ref_shim.cpp)

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

NetworkGraph graph_of_spec(const std::string& spec) {
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

std::string error_json(const std::exception& e) {
  json j;
  j["error"] = e.what();
  j["type"] = dynamic_cast<const ConfigError*>(&e)     ? "ConfigError"
              : dynamic_cast<const UnknownPreset*>(&e) ? "UnknownPreset"
              : dynamic_cast<const Error*>(&e)         ? "Error"
                                                       : "other";
  return j.dump();
}

}  // namespace

extern "C" {

void vref_fmt_free(char* p) { std::free(p); }

// load_config(path) + build_network(cfg): every field the front-end produces.
char* vref_fmt_config(const char* path) {
  try {
    const ExperimentConfig cfg = load_config(path);
    json j;
    j["network"] = cfg.network;
    j["batch"] = cfg.batch;
    j["policy"] = cfg.policy;
    j["algo_mode"] = cfg.algo_mode == AlgoMode::PerfOptimal ? "perf" : "memory";
    j["capacity"] = cfg.capacity ? json(*cfg.capacity) : json(nullptr);
    j["effective_capacity"] = cfg.effective_capacity();
    j["decision_file"] = cfg.decision_file;
    j["include_weight_grads"] = cfg.include_weight_grads;
    j["seed"] = cfg.seed;
    j["inline_layers"] = cfg.inline_layers;
    const CostModel& c = cfg.cost;
    j["cost"] = {{"peak_flops", c.device.peak_flops},
                 {"dram_bw", c.device.dram_bw},
                 {"mem_capacity", c.device.mem_capacity},
                 {"compute_efficiency", c.device.compute_efficiency},
                 {"elem_size", c.elem_size},
                 {"bwd_fwd_ratio", c.bwd_fwd_ratio},
                 {"link_effective_bw", c.link.effective_bw},
                 {"link_nominal_bw", c.link.nominal_bw},
                 {"link_launch_overhead", c.link.fixed_launch_overhead}};
    json ov = json::object();
    for (const auto& [id, fb] : c.latency_overrides) ov[std::to_string(id)] = {fb.first, fb.second};
    j["latency_overrides"] = ov;
    try {
      j["graph"] = spec_of(build_network(cfg));
    } catch (const std::exception& e) {
      j["graph_error"] = json::parse(error_json(e));
    }
    return dup(j.dump());
  } catch (const std::exception& e) {
    return dup(error_json(e));
  }
}

char* vref_fmt_graph_to_json(const char* spec) {
  try {
    return dup(graph_to_json(graph_of_spec(spec)).dump());
  } catch (const std::exception& e) {
    return dup(error_json(e));
  }
}

char* vref_fmt_graph_from_json(const char* text) {
  try {
    return dup(spec_of(graph_from_json(json::parse(text))));
  } catch (const std::exception& e) {
    return dup(error_json(e));
  }
}

// report_to_json + decision_to_json of a reference simulate() run (dyn decision)
char* vref_fmt_report(const char* spec, unsigned long long capacity) {
  try {
    const NetworkGraph g = graph_of_spec(spec);
    const CostModel cm;
    const DynamicSelection sel = dynamic_select(g, capacity, cm);
    json j;
    if (!sel.decision) {
      j["untrainable"] = true;
      return dup(j.dump());
    }
    const RunReport r = simulate(g, *sel.decision, cm, capacity);
    j["decision"] = decision_to_json(*sel.decision);
    j["report"] = report_to_json(r, true);
    return dup(j.dump());
  } catch (const std::exception& e) {
    return dup(error_json(e));
  }
}

}  // extern "C"
