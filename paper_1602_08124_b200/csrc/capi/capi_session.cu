// extern "C" training-session entry points (the B200 executor).
#include <cstring>
#include <new>
#include <stdexcept>
#include <string>
#include <vector>

#include "../runtime/session.h"
#include "capi_common.h"
#include "handles.h"

using vdnncapi::fail;

struct vdnn_session {
  vdnnrt::Session* s;
  vdnn_report plan_view;
};

namespace {
template <class F>
vdnn_status guard(F&& f) {
  try {
    vdnncapi::clear_error();
    return f();
  } catch (const vdnnp::PlanError& e) {
    const std::string msg = e.what();
    if (msg.rfind("UNSUPPORTED", 0) == 0) return fail(VDNN_UNSUPPORTED, msg);
    return fail(static_cast<vdnn_status>(static_cast<int>(e.code)), msg);
  } catch (const std::bad_alloc&) {
    return fail(VDNN_ERROR, "out of host memory");
  } catch (const std::exception& e) {
    return fail(VDNN_CUDA_ERROR, e.what());
  }
}
vdnnrt::Session& S(vdnn_session* s) {
  if (!s || !s->s) throw std::runtime_error("null session");
  return *s->s;
}
}  // namespace

extern "C" {

void vdnn_session_options_default(vdnn_session_options* o) {
  std::memset(o, 0, sizeof(*o));
  o->device = 0;
  o->weight_seed = 5000;
  o->external_grads = 0;
  o->record_timeline = 0;
  o->host_arena = 1;
  o->precise_fp32 = 0;
  o->compress_offload = 0;
  o->offload_target = 0;
  o->cuda_graph = 0;
  o->algo_kernels = 0;
}

vdnn_status vdnn_session_create(const vdnn_graph* g, const vdnn_decision* d, const vdnn_cost_model* cm,
                                uint64_t capacity, const vdnn_session_options* opt, vdnn_session** out) {
  return guard([&] {
    if (!g || !d || !out) throw vdnnp::PlanError(vdnnp::Err::Generic, "null argument");
    vdnnrt::Options o;
    if (opt) {
      o.device = opt->device;
      o.weight_seed = opt->weight_seed;
      o.external_grads = opt->external_grads != 0;
      o.record_timeline = opt->record_timeline != 0;
      o.host_arena = opt->host_arena != 0;
      o.precise = opt->precise_fp32 != 0;
      if (opt->compress_offload < 0 || opt->compress_offload > 2)
        throw vdnnp::PlanError(vdnnp::Err::Config, "compress_offload must be 0, 1 or 2");
      o.compress_offload = opt->compress_offload;
      o.offload_target = opt->offload_target;
      o.cuda_graph = opt->cuda_graph != 0;
      o.algo_kernels = opt->algo_kernels;
    }
    if (!g->net.finalized()) throw vdnnp::PlanError(vdnnp::Err::Generic, "graph is not finalized");
    auto* s = new vdnnrt::Session(g->net, d->d, vdnncapi::cost_from(cm), capacity, o);
    *out = new vdnn_session{s, vdnn_report{s->plan()}};
    return VDNN_OK;
  });
}

void vdnn_session_destroy(vdnn_session* s) {
  if (!s) return;
  delete s->s;
  delete s;
}

const vdnn_report* vdnn_session_plan(const vdnn_session* s) { return s ? &s->plan_view : nullptr; }

vdnn_status vdnn_session_arena_info(const vdnn_session* s, uint64_t* arena_bytes, uint64_t* lo, uint64_t* host_bytes,
                                    uint64_t* scratch) {
  return guard([&] {
    const vdnnrt::Session& x = *s->s;
    if (arena_bytes) *arena_bytes = x.arena_bytes();
    if (lo) *lo = x.arena_lo();
    if (host_bytes) *host_bytes = x.host_bytes();
    if (scratch) *scratch = x.scratch_bytes();
    return VDNN_OK;
  });
}

vdnn_status vdnn_session_set_batch_host(vdnn_session* s, const float* images, const int32_t* labels) {
  return guard([&] {
    S(s).set_batch_host(images, labels);
    return VDNN_OK;
  });
}
vdnn_status vdnn_session_set_batch_device(vdnn_session* s, const float* images, const int32_t* labels) {
  return guard([&] {
    S(s).set_batch_device(images, labels);
    return VDNN_OK;
  });
}
vdnn_status vdnn_session_synthetic_batch(vdnn_session* s, uint64_t seed) {
  return guard([&] {
    S(s).synthetic_batch(seed);
    return VDNN_OK;
  });
}
vdnn_status vdnn_session_get_weights(vdnn_session* s, int32_t layer, float* host, size_t count) {
  return guard([&] {
    S(s).get_weights(layer, host, count);
    return VDNN_OK;
  });
}
vdnn_status vdnn_session_set_weights(vdnn_session* s, int32_t layer, const float* host, size_t count) {
  return guard([&] {
    S(s).set_weights(layer, host, count);
    return VDNN_OK;
  });
}
vdnn_status vdnn_session_step(vdnn_session* s, float lr, float* loss_host) {
  return guard([&] {
    S(s).step(lr, loss_host);
    return VDNN_OK;
  });
}
vdnn_status vdnn_session_pause_timeline(vdnn_session* s, int32_t paused) {
  return guard([&] {
    S(s).pause_timeline(paused != 0);
    return VDNN_OK;
  });
}
vdnn_status vdnn_session_synchronize(vdnn_session* s) {
  return guard([&] {
    S(s).synchronize();
    return VDNN_OK;
  });
}
vdnn_status vdnn_session_read_feature(vdnn_session* s, int32_t owner, float* host, size_t count) {
  return guard([&] {
    S(s).read_feature(owner, host, count);
    return VDNN_OK;
  });
}
vdnn_status vdnn_session_measured_report(vdnn_session* s, vdnn_report** out) {
  return guard([&] {
    S(s).synchronize();
    *out = new vdnn_report{S(s).measured_report()};
    return VDNN_OK;
  });
}
vdnn_status vdnn_session_layer_times(vdnn_session* s, int32_t n, double* fwd_ms, double* bwd_ms) {
  return guard([&] {
    S(s).synchronize();
    S(s).layer_times(n, fwd_ms, bwd_ms);
    return VDNN_OK;
  });
}
vdnn_status vdnn_session_transfer_stats(vdnn_session* s, uint64_t* offload_wire, uint64_t* prefetch_wire,
                                        uint64_t* offload_planned, uint64_t* prefetch_planned) {
  return guard([&] {
    S(s).transfer_stats(offload_wire, prefetch_wire, offload_planned, prefetch_planned);
    return VDNN_OK;
  });
}
vdnn_status vdnn_session_grad_buffer(vdnn_session* s, int32_t layer, void** ptr, size_t* count) {
  return guard([&] {
    S(s).grad_buffer(layer, ptr, count);
    return VDNN_OK;
  });
}
vdnn_status vdnn_session_grad_arena(vdnn_session* s, void** ptr, size_t* count) {
  return guard([&] {
    S(s).grad_arena(ptr, count);
    return VDNN_OK;
  });
}
vdnn_status vdnn_session_set_grad_arena(vdnn_session* s, void* ptr, size_t count) {
  return guard([&] {
    S(s).set_grad_arena(static_cast<float*>(ptr), count);
    return VDNN_OK;
  });
}
vdnn_status vdnn_session_get_grads(vdnn_session* s, int32_t layer, float* host, size_t count) {
  return guard([&] {
    void* p = nullptr;
    size_t n = 0;
    S(s).grad_buffer(layer, &p, &n);
    if (!p || n != count) throw vdnnp::PlanError(vdnnp::Err::Generic, "no gradient buffer / count mismatch");
    S(s).synchronize();
    if (cudaMemcpy(host, p, count * 4, cudaMemcpyDeviceToHost) != cudaSuccess)
      throw std::runtime_error("cudaMemcpy(grads)");
    return VDNN_OK;
  });
}
vdnn_status vdnn_session_apply_grads(vdnn_session* s, float lr, float scale) {
  return guard([&] {
    S(s).apply_grads(lr, scale);
    return VDNN_OK;
  });
}
static_assert(sizeof(cudaIpcMemHandle_t) == 64, "vdnn_peer_handle assumes 64-byte IPC handles");
vdnn_status vdnn_session_peer_export(vdnn_session* s, vdnn_peer_handle* out) {
  return guard([&] {
    const auto h = S(s).peer_export();
    std::memcpy(out->arena, &h.arena, 64);
    std::memcpy(out->grads, &h.grads, 64);
    std::memcpy(out->signal, &h.signal, 64);
    out->arena_lo = h.arena_lo;
    out->arena_bytes = h.arena_bytes;
    out->grads_count = h.grads_count;
    return VDNN_OK;
  });
}
vdnn_status vdnn_session_peer_attach(vdnn_session* s, int32_t rank, int32_t world, const vdnn_peer_handle* all) {
  return guard([&] {
    if (world < 1 || world > 8 || !all) throw vdnnp::PlanError(vdnnp::Err::Generic, "peer_attach: 1..8 ranks");
    std::vector<vdnnrt::Session::PeerHandle> v(static_cast<size_t>(world));
    for (int p = 0; p < world; ++p) {
      std::memcpy(&v[p].arena, all[p].arena, 64);
      std::memcpy(&v[p].grads, all[p].grads, 64);
      std::memcpy(&v[p].signal, all[p].signal, 64);
      v[p].arena_lo = all[p].arena_lo;
      v[p].arena_bytes = all[p].arena_bytes;
      v[p].grads_count = all[p].grads_count;
    }
    S(s).peer_attach(rank, world, v.data());
    return VDNN_OK;
  });
}
vdnn_status vdnn_session_peer_exchange(vdnn_session* s, float lr, float scale) {
  return guard([&] {
    S(s).peer_exchange(lr, scale);
    return VDNN_OK;
  });
}
vdnn_status vdnn_session_peer_overlap(vdnn_session* s, int32_t on, float scale) {
  return guard([&] {
    S(s).peer_overlap(on != 0, scale);
    return VDNN_OK;
  });
}
vdnn_status vdnn_session_peer_detach(vdnn_session* s) {
  return guard([&] {
    S(s).peer_detach();
    return VDNN_OK;
  });
}
vdnn_status vdnn_session_prefetch_batch_host(vdnn_session* s, const float* images, const int32_t* labels) {
  return guard([&] {
    S(s).prefetch_batch_host(images, labels);
    return VDNN_OK;
  });
}
vdnn_status vdnn_session_read_loss(vdnn_session* s, float* loss) {
  return guard([&] {
    if (!loss) throw vdnnp::PlanError(vdnnp::Err::Generic, "null loss pointer");
    *loss = S(s).read_loss();
    return VDNN_OK;
  });
}
vdnn_status vdnn_session_queue_loss(vdnn_session* s, int64_t* ticket) {
  return guard([&] {
    *ticket = S(s).queue_loss();
    return VDNN_OK;
  });
}
vdnn_status vdnn_session_wait_loss(vdnn_session* s, int64_t ticket, float* loss) {
  return guard([&] {
    *loss = S(s).wait_loss(ticket);
    return VDNN_OK;
  });
}
vdnn_status vdnn_session_offload_bytes(vdnn_session* s, uint64_t* bytes) {
  return guard([&] {
    *bytes = S(s).offload_bytes();
    return VDNN_OK;
  });
}
vdnn_status vdnn_session_set_offload_buffer(vdnn_session* s, void* dev_ptr, uint64_t bytes) {
  return guard([&] {
    S(s).set_offload_buffer(dev_ptr, bytes);
    return VDNN_OK;
  });
}
vdnn_status vdnn_session_spill_export(vdnn_session* s, uint8_t ipc_handle[64]) {
  return guard([&] {
    const cudaIpcMemHandle_t h = S(s).spill_export();
    std::memcpy(ipc_handle, &h, 64);
    return VDNN_OK;
  });
}
vdnn_status vdnn_session_spill_attach(vdnn_session* s, const uint8_t ipc_handle[64]) {
  return guard([&] {
    cudaIpcMemHandle_t h;
    std::memcpy(&h, ipc_handle, 64);
    S(s).spill_attach(h);
    return VDNN_OK;
  });
}
vdnn_status vdnn_session_stream(vdnn_session* s, void** stream) {
  return guard([&] {
    *stream = S(s).stream();
    return VDNN_OK;
  });
}

}  // extern "C"

vdnn_status vdnn_session_probe_layout(vdnn_session* s, int32_t layer, int32_t bwd, vdnn_probe_layout* out) {
  return guard([&] {
    const vdnnrt::Session::ProbeLayout p = S(s).probe_layout(layer, bwd != 0);
    if (p.segs.size() > VDNN_PROBE_MAX_SEGS) throw vdnnp::PlanError(vdnnp::Err::Generic, "probe: too many segments");
    std::memset(out, 0, sizeof(*out));
    out->nseg = static_cast<int32_t>(p.segs.size());
    out->relu_fused = p.relu;
    out->accumulate = p.accumulate;
    out->skip = p.skip;
    out->mask_planes = p.mask;
    out->total_bytes = p.total;
    for (size_t i = 0; i < p.segs.size(); ++i) {
      out->seg[i].what = p.segs[i].what;
      out->seg[i].index = p.segs[i].index;
      out->seg[i].after = p.segs[i].after ? 1 : 0;
      out->seg[i].offset = p.segs[i].dst;
      out->seg[i].bytes = p.segs[i].bytes;
    }
    return VDNN_OK;
  });
}
vdnn_status vdnn_session_arm_probe(vdnn_session* s, int32_t layer, int32_t bwd, void* dst, uint64_t bytes) {
  return guard([&] {
    S(s).arm_probe(layer, bwd != 0, dst, bytes);
    return VDNN_OK;
  });
}
vdnn_status vdnn_session_set_input(vdnn_session* s, int32_t layer, const float* images, int32_t on_device) {
  return guard([&] {
    S(s).set_input(layer, images, on_device != 0);
    return VDNN_OK;
  });
}
