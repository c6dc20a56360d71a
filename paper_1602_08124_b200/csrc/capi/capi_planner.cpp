// extern "C" planner entry points (graph, cost model, decisions, simulate,
// vDNN_dyn, replay). Every C++ exception is translated into a vdnn_status.
#include <cstring>
#include <new>
#include <string>

#include "../planner/planner.hpp"
#include "capi_common.h"
#include "handles.h"

using vdnncapi::fail;
using namespace vdnnp;

namespace {

template <class F>
vdnn_status guard(F&& f) {
  try {
    vdnncapi::clear_error();
    return f();
  } catch (const PlanError& e) {
    return fail(static_cast<vdnn_status>(static_cast<int>(e.code)), e.what());
  } catch (const std::bad_alloc&) {
    return fail(VDNN_ERROR, "out of host memory");
  } catch (const std::exception& e) {
    return fail(VDNN_ERROR, e.what());
  }
}

void copy_tag(char (&dst)[4], const std::string& s) {
  std::memset(dst, 0, sizeof dst);
  std::strncpy(dst, s.c_str(), sizeof dst - 1);
}

Policy policy_of(int32_t k) {
  if (k == VDNN_POLICY_BASELINE) return Policy::Baseline;
  if (k == VDNN_POLICY_VDNN_ALL) return Policy::All;
  if (k == VDNN_POLICY_VDNN_CONV) return Policy::ConvOnly;
  throw PlanError(Err::Config, "unknown policy kind " + std::to_string(k));
}

Algo algo_of(int32_t a) {
  if (a == VDNN_ALGO_IMPLICIT_GEMM) return Algo::Implicit;
  if (a == VDNN_ALGO_GEMM_WS) return Algo::GemmWs;
  if (a == VDNN_ALGO_FFT) return Algo::Fft;
  throw PlanError(Err::Config, "unknown convolution algorithm " + std::to_string(a));
}

std::vector<int> inputs_of(const int32_t* in, int32_t n) {
  if (n < 0 || (n > 0 && !in)) throw PlanError(Err::Generic, "bad input list");
  return std::vector<int>(in, in + n);
}

Join join_of(int32_t j) { return j == VDNN_JOIN_ELEMENTWISE ? Join::Elementwise : Join::Concat; }

const Net& net_of(const vdnn_graph* g) {
  if (!g) throw PlanError(Err::Generic, "null graph");
  return g->net;
}

const Net& final_net(const vdnn_graph* g) {
  const Net& n = net_of(g);
  if (!n.finalized()) throw PlanError(Err::Generic, "graph is not finalized");
  return n;
}

void check_layer(const Net& n, int32_t id) {
  if (id < 0 || id >= n.size()) throw PlanError(Err::Generic, "layer id out of range");
}

template <class T>
vdnn_status copy_out(const std::vector<T>& v, T* out, size_t cap, size_t* n) {
  if (n) *n = v.size();
  if (out) std::memcpy(out, v.data(), sizeof(T) * std::min(cap, v.size()));
  return VDNN_OK;
}

}  // namespace

namespace vdnncapi {
Cost cost_from(const vdnn_cost_model* cm) {
  Cost c;
  if (!cm) return c;
  c.peak_flops = cm->peak_flops;
  c.dram_bw = cm->dram_bw;
  c.mem_capacity = cm->mem_capacity;
  c.compute_efficiency = cm->compute_efficiency;
  c.link_bw = cm->link_effective_bw;
  c.link_nominal_bw = cm->link_nominal_bw;
  c.link_overhead = cm->link_launch_overhead;
  c.elem = cm->elem_size;
  c.bwd_ratio = cm->bwd_fwd_ratio;
  c.sf_implicit = cm->speed_factor_implicit_gemm;
  c.sf_gemm_ws = cm->speed_factor_gemm_ws;
  c.sf_fft = cm->speed_factor_fft;
  for (int32_t i = 0; i < cm->n_overrides; ++i)
    c.pinned[cm->override_layer[i]] = {cm->override_fwd_s[i], cm->override_bwd_s[i]};
  return c;
}
}  // namespace vdnncapi

using vdnncapi::cost_from;

extern "C" {

// ------------------------------------------------------------------ graph
vdnn_status vdnn_graph_create(uint64_t batch, vdnn_graph** out) {
  return guard([&] {
    if (!out) throw PlanError(Err::Generic, "null out");
    *out = new vdnn_graph{Net(batch)};
    return VDNN_OK;
  });
}
vdnn_status vdnn_graph_clone(const vdnn_graph* g, vdnn_graph** out) {
  return guard([&] {
    *out = new vdnn_graph{net_of(g)};
    return VDNN_OK;
  });
}
void vdnn_graph_destroy(vdnn_graph* g) { delete g; }

vdnn_status vdnn_graph_add_input(vdnn_graph* g, uint64_t c, uint64_t h, uint64_t w, int32_t* id) {
  return guard([&] {
    const int r = g->net.input(c, h, w);
    if (id) *id = r;
    return VDNN_OK;
  });
}
vdnn_status vdnn_graph_add_conv(vdnn_graph* g, const int32_t* in, int32_t n, uint64_t out, uint64_t k, uint64_t s,
                                uint64_t p, int32_t join, int32_t* id) {
  return guard([&] {
    const int r = g->net.conv(inputs_of(in, n), out, k, s, p, join_of(join));
    if (id) *id = r;
    return VDNN_OK;
  });
}
vdnn_status vdnn_graph_add_layer(vdnn_graph* g, int32_t kind, const int32_t* in, int32_t n, uint64_t p0, uint64_t p1,
                                 uint64_t p2, uint64_t p3, int32_t join, int32_t* id) {
  return guard([&] {
    if (kind < 0 || kind > 5) throw vdnnp::PlanError(vdnnp::Err::Config, "unknown layer kind");
    vdnnp::Node d;
    d.kind = static_cast<vdnnp::Kind>(kind);
    d.in = inputs_of(in, n);
    d.join = join_of(join);
    switch (d.kind) {
      case vdnnp::Kind::Conv:
        d.k = p0;
        d.s = p1;
        d.p = p2;
        d.out = p3;
        break;
      case vdnnp::Kind::Pool:
        d.k = p0;
        d.s = p1;
        break;
      case vdnnp::Kind::Fc:
        d.out = p0;
        break;
      case vdnnp::Kind::Input:
        d.ic = p0;
        d.ih = p1;
        d.iw = p2;
        break;
      default:
        break;
    }
    const int r = g->net.add(std::move(d));
    if (id) *id = r;
    return VDNN_OK;
  });
}
vdnn_status vdnn_graph_add_actv(vdnn_graph* g, int32_t input, int32_t* id) {
  return guard([&] {
    const int r = g->net.actv(input);
    if (id) *id = r;
    return VDNN_OK;
  });
}
vdnn_status vdnn_graph_add_pool(vdnn_graph* g, const int32_t* in, int32_t n, uint64_t window, uint64_t stride,
                                int32_t join, int32_t* id) {
  return guard([&] {
    const int r = g->net.pool(inputs_of(in, n), window, stride, join_of(join));
    if (id) *id = r;
    return VDNN_OK;
  });
}
vdnn_status vdnn_graph_add_fc(vdnn_graph* g, const int32_t* in, int32_t n, uint64_t out, int32_t join, int32_t* id) {
  return guard([&] {
    const int r = g->net.fc(inputs_of(in, n), out, join_of(join));
    if (id) *id = r;
    return VDNN_OK;
  });
}
vdnn_status vdnn_graph_add_loss(vdnn_graph* g, int32_t input, int32_t* id) {
  return guard([&] {
    const int r = g->net.loss(input);
    if (id) *id = r;
    return VDNN_OK;
  });
}
vdnn_status vdnn_graph_finalize(vdnn_graph* g) {
  return guard([&] {
    if (!g) throw PlanError(Err::Generic, "null graph");
    g->net.finalize();
    return VDNN_OK;
  });
}
vdnn_status vdnn_graph_size(const vdnn_graph* g, int32_t* n) {
  return guard([&] {
    *n = net_of(g).size();
    return VDNN_OK;
  });
}
vdnn_status vdnn_graph_batch(const vdnn_graph* g, uint64_t* b) {
  return guard([&] {
    *b = net_of(g).batch();
    return VDNN_OK;
  });
}
vdnn_status vdnn_graph_layer(const vdnn_graph* g, int32_t id, vdnn_layer_info* o) {
  return guard([&] {
    const Net& n = net_of(g);
    check_layer(n, id);
    const Node& l = n.at(id);
    std::memset(o, 0, sizeof(*o));
    o->id = l.id;
    o->kind = static_cast<int32_t>(l.kind);
    o->join = static_cast<int32_t>(l.join);
    o->n_inputs = static_cast<int32_t>(l.in.size());
    for (size_t i = 0; i < l.in.size() && i < 16; ++i) o->inputs[i] = l.in[i];
    switch (l.kind) {
      case Kind::Conv: o->p0 = l.k; o->p1 = l.s; o->p2 = l.p; o->p3 = l.out; break;
      case Kind::Pool: o->p0 = l.k; o->p1 = l.s; break;
      case Kind::Fc: o->p0 = l.out; break;
      case Kind::Input: o->p0 = l.ic; o->p1 = l.ih; o->p2 = l.iw; break;
      default: break;
    }
    if (n.finalized()) {
      const Dims& d = n.dims(id);
      o->n = d.n;
      o->c = d.c;
      o->h = d.h;
      o->w = d.w;
      o->refcnt = n.refs(id);
    }
    return VDNN_OK;
  });
}
vdnn_status vdnn_preset(const char* name, uint64_t batch, vdnn_graph** out) {
  return guard([&] {
    if (!name) throw PlanError(Err::Preset, "null preset name");
    *out = new vdnn_graph{make_preset(name, batch)};
    return VDNN_OK;
  });
}
vdnn_status vdnn_extend_vgg(int32_t extra, uint64_t batch, vdnn_graph** out) {
  return guard([&] {
    *out = new vdnn_graph{make_deep_vgg(extra, batch)};
    return VDNN_OK;
  });
}

// ------------------------------------------------------------- cost model
void vdnn_cost_model_default(vdnn_cost_model* cm) {
  const Cost c;
  std::memset(cm, 0, sizeof(*cm));
  cm->peak_flops = c.peak_flops;
  cm->dram_bw = c.dram_bw;
  cm->mem_capacity = c.mem_capacity;
  cm->compute_efficiency = c.compute_efficiency;
  cm->link_effective_bw = c.link_bw;
  cm->link_nominal_bw = c.link_nominal_bw;
  cm->link_launch_overhead = c.link_overhead;
  cm->elem_size = c.elem;
  cm->bwd_fwd_ratio = c.bwd_ratio;
  cm->speed_factor_implicit_gemm = c.sf_implicit;
  cm->speed_factor_gemm_ws = c.sf_gemm_ws;
  cm->speed_factor_fft = c.sf_fft;
}
vdnn_status vdnn_cost_tensor_bytes(const vdnn_cost_model* cm, const vdnn_graph* g, int32_t id, uint64_t* b) {
  return guard([&] {
    const Net& n = final_net(g);
    check_layer(n, id);
    *b = cost_from(cm).bytes_of(n.dims(id));
    return VDNN_OK;
  });
}
vdnn_status vdnn_cost_weight_bytes(const vdnn_cost_model* cm, const vdnn_graph* g, int32_t id, uint64_t* b) {
  return guard([&] {
    const Net& n = final_net(g);
    check_layer(n, id);
    *b = cost_from(cm).weights(n, id);
    return VDNN_OK;
  });
}
vdnn_status vdnn_cost_conv_workspace(const vdnn_cost_model* cm, const vdnn_graph* g, int32_t id, int32_t algo,
                                     uint64_t* b) {
  return guard([&] {
    const Net& n = final_net(g);
    check_layer(n, id);
    *b = cost_from(cm).workspace(n, id, algo_of(algo));
    return VDNN_OK;
  });
}
vdnn_status vdnn_cost_layer_latency(const vdnn_cost_model* cm, const vdnn_graph* g, int32_t id, int32_t bwd,
                                    int32_t algo, double* s) {
  return guard([&] {
    const Net& n = final_net(g);
    check_layer(n, id);
    *s = cost_from(cm).latency(n, id, bwd != 0, algo_of(algo));
    return VDNN_OK;
  });
}
vdnn_status vdnn_cost_flops(const vdnn_cost_model* cm, const vdnn_graph* g, int32_t id, int32_t bwd, double* f) {
  return guard([&] {
    const Net& n = final_net(g);
    check_layer(n, id);
    *f = cost_from(cm).flop_count(n, id, bwd != 0);
    return VDNN_OK;
  });
}
vdnn_status vdnn_cost_transfer_latency(const vdnn_cost_model* cm, uint64_t bytes, double* s) {
  return guard([&] {
    *s = cost_from(cm).transfer(bytes);
    return VDNN_OK;
  });
}
vdnn_status vdnn_cost_fastest_algo(const vdnn_cost_model* cm, const vdnn_graph* g, int32_t id, int32_t* a) {
  return guard([&] {
    const Net& n = final_net(g);
    check_layer(n, id);
    *a = static_cast<int32_t>(cost_from(cm).fastest(n, id));
    return VDNN_OK;
  });
}
vdnn_status vdnn_gradient_map_bytes(const vdnn_cost_model* cm, const vdnn_graph* g, int32_t id, uint64_t* b) {
  return guard([&] {
    const Net& n = final_net(g);
    check_layer(n, id);
    *b = grad_map_bytes(n, id, cost_from(cm));
    return VDNN_OK;
  });
}

// -------------------------------------------------------------- decisions
vdnn_status vdnn_decision_static(const vdnn_graph* g, int32_t kind, int32_t mode, const vdnn_cost_model* cm,
                                 vdnn_decision** out) {
  return guard([&] {
    const Net& n = final_net(g);
    *out = new vdnn_decision{make_static(policy_of(kind), mode == VDNN_MODE_PERF_OPTIMAL ? Mode::Perf : Mode::Memory,
                                         n, cost_from(cm))};
    return VDNN_OK;
  });
}
vdnn_status vdnn_decision_create(const vdnn_graph* g, vdnn_decision** out) {
  return guard([&] {
    Decision d;
    d.offload.assign(static_cast<size_t>(net_of(g).size()), 0);
    *out = new vdnn_decision{d};
    return VDNN_OK;
  });
}
vdnn_status vdnn_decision_clone(const vdnn_decision* d, vdnn_decision** out) {
  return guard([&] {
    *out = new vdnn_decision{d->d};
    return VDNN_OK;
  });
}
void vdnn_decision_destroy(vdnn_decision* d) { delete d; }
vdnn_status vdnn_decision_set_offload(vdnn_decision* d, int32_t layer, int32_t flag) {
  return guard([&] {
    if (layer < 0 || static_cast<size_t>(layer) >= d->d.offload.size())
      throw PlanError(Err::Decision, "decision file references unknown layer");
    d->d.offload[static_cast<size_t>(layer)] = flag ? 1 : 0;
    return VDNN_OK;
  });
}
vdnn_status vdnn_decision_set_algo(vdnn_decision* d, int32_t layer, int32_t algo) {
  return guard([&] {
    if (algo < 0)
      d->d.algos.erase(layer);
    else
      d->d.algos[layer] = algo_of(algo);
    return VDNN_OK;
  });
}
vdnn_status vdnn_decision_set_scheme(vdnn_decision* d, int32_t scheme) {
  return guard([&] {
    d->d.scheme = scheme == VDNN_GRAD_TWO_BUFFER_REUSE ? Scheme::TwoBuffer : Scheme::PerLayer;
    return VDNN_OK;
  });
}
vdnn_status vdnn_decision_set_label(vdnn_decision* d, const char* label) {
  return guard([&] {
    d->d.label = label ? label : "";
    return VDNN_OK;
  });
}
vdnn_status vdnn_decision_get(const vdnn_decision* d, int32_t* n_layers, char* flags, int32_t* algos, int32_t* scheme,
                              char* label, size_t label_cap) {
  return guard([&] {
    const int L = static_cast<int>(d->d.offload.size());
    if (n_layers) *n_layers = L;
    if (flags)
      for (int i = 0; i < L; ++i) flags[i] = d->d.offload[static_cast<size_t>(i)];
    if (algos) {
      for (int i = 0; i < L; ++i) algos[i] = -1;
      for (const auto& [id, a] : d->d.algos)
        if (id >= 0 && id < L) algos[id] = static_cast<int32_t>(a);
    }
    if (scheme) *scheme = static_cast<int32_t>(d->d.scheme);
    if (label && label_cap > 0) {
      std::strncpy(label, d->d.label.c_str(), label_cap - 1);
      label[label_cap - 1] = 0;
    }
    return VDNN_OK;
  });
}
vdnn_status vdnn_decision_validate(const vdnn_decision* d, const vdnn_graph* g) {
  return guard([&] {
    d->d.check(net_of(g));
    return VDNN_OK;
  });
}
vdnn_status vdnn_baseline_footprint(const vdnn_graph* g, const vdnn_decision* d, const vdnn_cost_model* cm,
                                    int32_t with_dw, vdnn_footprint* out) {
  return guard([&] {
    const std::map<int, Algo> none;
    const Footprint f = footprint(final_net(g), d ? d->d.algos : none, cost_from(cm), with_dw != 0);
    out->weights_bytes = f.weights;
    out->feature_maps_bytes = f.features;
    out->gradient_buffers_bytes = f.gradients;
    out->workspace_bytes = f.workspace;
    out->total_bytes = f.total;
    out->classifier_bytes = f.classifier;
    return VDNN_OK;
  });
}

// --------------------------------------------------------------- simulate
vdnn_status vdnn_simulate(const vdnn_graph* g, const vdnn_decision* d, const vdnn_cost_model* cm, uint64_t capacity,
                          uint32_t flags, vdnn_report** out) {
  return guard([&] {
    if (!d) throw PlanError(Err::Decision, "null decision");
    SimFlags f;
    f.trace = (flags & VDNN_SIM_KEEP_POOL_TRACE) != 0;
    f.with_dw = (flags & VDNN_SIM_INCLUDE_WEIGHT_GRADS) != 0;
    *out = new vdnn_report{plan(final_net(g), d->d, cost_from(cm), capacity, f)};
    return VDNN_OK;
  });
}
vdnn_status vdnn_simulate_oracle(const vdnn_graph* g, const vdnn_cost_model* cm, vdnn_report** out) {
  return guard([&] {
    *out = new vdnn_report{plan_oracle(final_net(g), cost_from(cm))};
    return VDNN_OK;
  });
}
void vdnn_report_destroy(vdnn_report* r) { delete r; }

vdnn_status vdnn_report_summary_get(const vdnn_report* rp, vdnn_report_summary* s) {
  return guard([&] {
    const Report& r = rp->r;
    std::memset(s, 0, sizeof(*s));
    s->pass = r.pass ? 1 : 0;
    s->has_oom = r.oom ? 1 : 0;
    if (r.oom) {
      s->oom_layer = r.oom->layer;
      s->oom_phase = static_cast<int32_t>(r.oom->stage);
      s->oom_fragmented = r.oom->fragmented ? 1 : 0;
      s->oom_requested = r.oom->requested;
      copy_tag(s->oom_tag, r.oom->tag);
    }
    s->max_mem_bytes = r.max_mem;
    s->avg_mem_bytes = r.avg_mem;
    s->offload_traffic_bytes = r.offload_bytes;
    s->prefetch_traffic_bytes = r.prefetch_bytes;
    s->host_peak_bytes = r.host_peak;
    s->stall_fwd_offload_ns = r.stall_fwd;
    s->stall_bwd_prefetch_ns = r.stall_bwd;
    s->total_ns = r.total;
    s->interference_bound = r.interference;
    s->n_events = r.events.size();
    std::strncpy(s->verdict, r.verdict().c_str(), sizeof(s->verdict) - 1);
    return VDNN_OK;
  });
}
vdnn_status vdnn_report_events(const vdnn_report* rp, vdnn_event* out, size_t cap, size_t* n) {
  return guard([&] {
    const auto& ev = rp->r.events;
    if (n) *n = ev.size();
    if (out) {
      for (size_t i = 0; i < ev.size() && i < cap; ++i) {
        const Event& e = ev[i];
        vdnn_event& o = out[i];
        o.stream = static_cast<int32_t>(e.lane);
        o.kind = static_cast<int32_t>(e.kind);
        o.layer = e.layer;
        o.buffer = e.buffer;
        o.start_ns = e.t0;
        o.end_ns = e.t1;
        o.bytes = e.bytes;
        o.offset = e.off;
        copy_tag(o.tag, e.tag);
      }
    }
    return VDNN_OK;
  });
}
vdnn_status vdnn_report_reuse_distance(const vdnn_report* rp, int64_t* out, size_t cap, size_t* n) {
  return guard([&] { return copy_out<int64_t>(rp->r.reuse, out, cap, n); });
}
vdnn_status vdnn_report_pool_trace(const vdnn_report* rp, vdnn_pool_trace_row* out, size_t cap, size_t* n) {
  return guard([&] {
    const auto& t = rp->r.pool_trace;
    if (n) *n = t.size();
    if (out)
      for (size_t i = 0; i < t.size() && i < cap; ++i) {
        out[i].time_ns = t[i].t;
        out[i].op = t[i].op;
        copy_tag(out[i].tag, t[i].tag);
        out[i].offset = t[i].off;
        out[i].bytes = t[i].len;
        out[i].current = t[i].cur;
        out[i].high_water = t[i].hw;
      }
    return VDNN_OK;
  });
}
vdnn_status vdnn_report_layer_peaks(const vdnn_report* rp, int32_t n_layers, uint64_t* fwd, uint64_t* bwd) {
  return guard([&] {
    for (const Event& e : rp->r.events)
      if ((e.kind == Ev::Fwd || e.kind == Ev::Bwd) && (e.layer < 0 || e.layer >= n_layers))
        throw PlanError(Err::Generic, "n_layers smaller than the report's layer ids");
    std::vector<u64> f, b;
    layer_peaks(rp->r, f, b, n_layers);
    for (int i = 0; i < n_layers; ++i) {
      if (fwd) fwd[i] = f[static_cast<size_t>(i)];
      if (bwd) bwd[i] = b[static_cast<size_t>(i)];
    }
    return VDNN_OK;
  });
}
vdnn_status vdnn_report_signature(const vdnn_report* rp, uint64_t* sig) {
  return guard([&] {
    *sig = schedule_signature(rp->r);
    return VDNN_OK;
  });
}
vdnn_status vdnn_report_from_events(const vdnn_event* ev, size_t n, const vdnn_report_summary* s, vdnn_report** out) {
  return guard([&] {
    Report r;
    r.events.reserve(n);
    for (size_t i = 0; i < n; ++i) {
      Event e;
      e.lane = ev[i].stream ? Lane::Memory : Lane::Compute;
      e.kind = static_cast<Ev>(ev[i].kind);
      e.layer = ev[i].layer;
      e.buffer = ev[i].buffer;
      e.t0 = ev[i].start_ns;
      e.t1 = ev[i].end_ns;
      e.bytes = ev[i].bytes;
      e.off = ev[i].offset;
      e.tag = std::string(ev[i].tag, strnlen(ev[i].tag, 4));
      r.events.push_back(e);
    }
    if (s) {
      r.pass = s->pass != 0;
      r.max_mem = s->max_mem_bytes;
      r.avg_mem = s->avg_mem_bytes;
      r.offload_bytes = s->offload_traffic_bytes;
      r.prefetch_bytes = s->prefetch_traffic_bytes;
      r.host_peak = s->host_peak_bytes;
      r.stall_fwd = s->stall_fwd_offload_ns;
      r.stall_bwd = s->stall_bwd_prefetch_ns;
      r.total = s->total_ns;
      r.interference = s->interference_bound;
    }
    *out = new vdnn_report{std::move(r)};
    return VDNN_OK;
  });
}

// ------------------------------------------------------------------- dyn
vdnn_status vdnn_dynamic_select(const vdnn_graph* g, uint64_t capacity, const vdnn_cost_model* cm, vdnn_dyn** out) {
  return guard([&] {
    *out = new vdnn_dyn{choose_dynamic(final_net(g), capacity, cost_from(cm))};
    return VDNN_OK;
  });
}
void vdnn_dyn_destroy(vdnn_dyn* s) { delete s; }
vdnn_status vdnn_dyn_untrainable(const vdnn_dyn* s, int32_t* u) {
  return guard([&] {
    *u = s->res.decision ? 0 : 1;
    return VDNN_OK;
  });
}
vdnn_status vdnn_dyn_decision(const vdnn_dyn* s, vdnn_decision** out) {
  return guard([&] {
    if (!s->res.decision) throw PlanError(Err::Generic, "network is untrainable under this budget");
    *out = new vdnn_decision{*s->res.decision};
    return VDNN_OK;
  });
}
vdnn_status vdnn_dyn_passes(const vdnn_dyn* s, vdnn_pass_info* out, size_t cap, size_t* n) {
  return guard([&] {
    const auto& p = s->res.passes;
    if (n) *n = p.size();
    if (out)
      for (size_t i = 0; i < p.size() && i < cap; ++i) {
        std::memset(&out[i], 0, sizeof(out[i]));
        std::strncpy(out[i].phase, p[i].phase.c_str(), sizeof(out[i].phase) - 1);
        std::strncpy(out[i].label, p[i].decision.label.c_str(), sizeof(out[i].label) - 1);
        out[i].pass = p[i].pass ? 1 : 0;
        out[i].has_oom = p[i].oom ? 1 : 0;
        if (p[i].oom) {
          out[i].oom_layer = p[i].oom->layer;
          out[i].oom_phase = static_cast<int32_t>(p[i].oom->stage);
        }
        out[i].total_ns = p[i].total;
        out[i].max_mem_bytes = p[i].max_mem;
      }
    return VDNN_OK;
  });
}
vdnn_status vdnn_dyn_pass_decision(const vdnn_dyn* s, size_t index, vdnn_decision** out) {
  return guard([&] {
    if (index >= s->res.passes.size()) throw PlanError(Err::Generic, "pass index out of range");
    *out = new vdnn_decision{s->res.passes[index].decision};
    return VDNN_OK;
  });
}
vdnn_status vdnn_greedy_downgrade(const vdnn_graph* g, uint64_t capacity, int32_t kind, const vdnn_cost_model* cm,
                                  int32_t* found, vdnn_decision** out) {
  return guard([&] {
    auto d = greedy(final_net(g), capacity, policy_of(kind), cost_from(cm));
    *found = d ? 1 : 0;
    *out = d ? new vdnn_decision{*d} : nullptr;
    return VDNN_OK;
  });
}

// ---------------------------------------------------------------- replay
vdnn_status vdnn_replay_check(const vdnn_report* r, const vdnn_graph* g, const vdnn_decision* d, uint64_t capacity,
                              vdnn_violation* out, size_t cap, size_t* n) {
  return guard([&] {
    const auto v = validate_log(r->r, final_net(g), d->d, capacity);
    if (n) *n = v.size();
    if (out)
      for (size_t i = 0; i < v.size() && i < cap; ++i) {
        std::memset(&out[i], 0, sizeof(out[i]));
        std::strncpy(out[i].kind, v[i].kind.c_str(), sizeof(out[i].kind) - 1);
        std::strncpy(out[i].detail, v[i].detail.c_str(), sizeof(out[i].detail) - 1);
      }
    return VDNN_OK;
  });
}

// Compile the executable program of a plan and check its operand bindings,
// scratch gaps and transfers against the plan's own event log.
vdnn_status vdnn_program_check(const vdnn_graph* g, const vdnn_decision* d, const vdnn_cost_model* cm,
                               uint64_t capacity, vdnn_violation* out, size_t cap, size_t* n) {
  return guard([&] {
    const Net& net = final_net(g);
    Program prog;
    const Report r = plan(net, d->d, cost_from(cm), capacity, {}, &prog);
    std::vector<Finding> v;
    if (r.pass) v = check_program(prog, r, net, d->d);
    if (n) *n = v.size();
    if (out)
      for (size_t i = 0; i < v.size() && i < cap; ++i) {
        std::memset(&out[i], 0, sizeof(out[i]));
        std::strncpy(out[i].kind, v[i].kind.c_str(), sizeof(out[i].kind) - 1);
        std::strncpy(out[i].detail, v[i].detail.c_str(), sizeof(out[i].detail) - 1);
      }
    return VDNN_OK;
  });
}

}  // extern "C"
