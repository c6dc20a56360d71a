"""Python mirror of the reference's network-definition and offload-policy API.

Names, argument meaning and error behaviour follow vdnnsim
(/root/reference/proj/include/vdnnsim): ``NetworkGraph`` (net_graph.hpp:101),
``build_preset``/``extend_vgg`` (presets.hpp:123-140), ``CostModel``
(cost_model.hpp:65), ``static_decision`` (decision.hpp:68), ``simulate``
(simulator.hpp:568), ``dynamic_select`` (policy.hpp:115), ``greedy_downgrade``
(policy.hpp:65), ``simulate_oracle`` (policy.hpp:152), ``replay_check``
(replay.hpp:95), ``baseline_footprint`` (footprint.hpp:81). Everything runs in
libvdnn.so (C++ planner); this module only marshals.

Errors: the reference throws ``vdnnsim::Error`` subclasses; here the same
conditions raise the matching Python exception below (all subclasses of
``VdnnError``). OOM is never an exception: it is ``RunReport.pass_ = False``
with ``RunReport.oom`` set.
"""
from __future__ import annotations

import ctypes as C
import enum
from dataclasses import dataclass, field
from typing import Dict, List, Optional, Sequence, Tuple

from . import _lib as L
from ._lib import VdnnError

KUNLIMITED_BYTES = 1 << 62  # core.hpp:17


class ShapeMismatch(VdnnError):
    pass


class UnknownPreset(VdnnError):
    pass


class InvalidDepth(VdnnError):
    pass


class OverflowError_(VdnnError):
    pass


class WrongLayerKind(VdnnError):
    pass


class PoolUseError(VdnnError):
    pass


class InvalidDecision(VdnnError):
    pass


class ConfigError(VdnnError):
    pass


_ERRS = {
    L.SHAPE_MISMATCH: ShapeMismatch, L.UNKNOWN_PRESET: UnknownPreset, L.INVALID_DEPTH: InvalidDepth,
    L.OVERFLOW: OverflowError_, L.WRONG_LAYER_KIND: WrongLayerKind, L.POOL_MISUSE: PoolUseError,
    L.INVALID_DECISION: InvalidDecision, L.CONFIG_ERROR: ConfigError,
}


def _call(name: str, *args) -> None:
    st = getattr(L.lib(), name)(*args)
    if st != L.OK:
        msg = L.lib().vdnn_last_error().decode(errors="replace")
        raise _ERRS.get(st, VdnnError)(st, msg)


class LayerKind(enum.IntEnum):
    Input = 0
    Conv = 1
    Actv = 2
    Pool = 3
    Fc = 4
    Loss = 5


class JoinRule(enum.IntEnum):
    Concat = 0
    Elementwise = 1


class AlgoId(enum.IntEnum):
    ImplicitGemm = 0
    GemmWs = 1
    Fft = 2


class PolicyKind(enum.IntEnum):
    Baseline = 0
    VdnnAll = 1
    VdnnConv = 2


class AlgoMode(enum.IntEnum):
    MemoryOptimal = 0
    PerfOptimal = 1


class GradientScheme(enum.IntEnum):
    TwoBufferReuse = 0
    PerLayer = 1


class Stream(enum.IntEnum):
    Compute = 0
    Memory = 1


class EventKind(enum.IntEnum):
    Fwd = 0
    Bwd = 1
    Offload = 2
    Prefetch = 3
    Alloc = 4
    Release = 5
    Sync = 6


class Phase(enum.IntEnum):
    Setup = 0
    Forward = 1
    Backward = 2


_EV_NAMES = ["FWD", "BWD", "OFFLOAD", "PREFETCH", "ALLOC", "RELEASE", "SYNC"]
_PHASE_NAMES = ["setup", "forward", "backward"]


@dataclass(frozen=True)
class TensorShape:
    n: int
    c: int
    h: int
    w: int

    def elements(self) -> int:
        return self.n * self.c * self.h * self.w


@dataclass(frozen=True)
class LayerDescriptor:
    id: int
    kind: LayerKind
    inputs: Tuple[int, ...]
    join: JoinRule
    params: Tuple[int, int, int, int]


# ------------------------------------------------------------------ graph --
class NetworkGraph:
    """DAG of layers in topological id order (net_graph.hpp:101-229)."""

    def __init__(self, batch: int = 1, _handle=None):
        self._h = C.c_void_p()
        if _handle is not None:
            self._h = _handle
        else:
            _call("vdnn_graph_create", C.c_uint64(batch), C.byref(self._h))
        self._finalized = _handle is not None

    def __del__(self):
        h = getattr(self, "_h", None)
        if h is not None and h.value and L._lib is not None:
            L._lib.vdnn_graph_destroy(h)
            self._h = None

    @property
    def handle(self):
        return self._h

    @staticmethod
    def _ins(inputs: Sequence[int]):
        arr = (C.c_int32 * max(len(inputs), 1))(*inputs)
        return arr, len(inputs)

    def add_input(self, c: int, h: int, w: int) -> int:
        out = C.c_int32()
        _call("vdnn_graph_add_input", self._h, C.c_uint64(c), C.c_uint64(h), C.c_uint64(w), C.byref(out))
        return out.value

    def add_conv(self, inputs: Sequence[int], out_channels: int, kernel: int, stride: int, pad: int,
                 join: JoinRule = JoinRule.Concat) -> int:
        arr, n = self._ins(inputs)
        out = C.c_int32()
        _call("vdnn_graph_add_conv", self._h, arr, n, C.c_uint64(out_channels), C.c_uint64(kernel),
              C.c_uint64(stride), C.c_uint64(pad), int(join), C.byref(out))
        return out.value

    def add_layer(self, kind: "LayerKind", inputs: Sequence[int] = (), params: Sequence[int] = (),
                  join: "JoinRule" = None) -> int:
        """NetworkGraph::add_layer (net_graph.hpp:109-113): any kind with any
        input list; params per kind = conv (kernel, stride, pad, out), pool
        (window, stride), fc (out,), input (c, h, w). Checked at finalize."""
        arr, n = self._ins(inputs)
        p = list(params) + [0] * (4 - len(params))
        out = C.c_int32()
        _call("vdnn_graph_add_layer", self._h, int(kind), arr, n, *[C.c_uint64(int(v)) for v in p[:4]],
              int(join if join is not None else JoinRule.Concat), C.byref(out))
        return out.value

    def add_actv(self, inp: int) -> int:
        out = C.c_int32()
        _call("vdnn_graph_add_actv", self._h, int(inp), C.byref(out))
        return out.value

    def add_pool(self, inputs: Sequence[int], window: int, stride: int, join: JoinRule = JoinRule.Concat) -> int:
        arr, n = self._ins(inputs)
        out = C.c_int32()
        _call("vdnn_graph_add_pool", self._h, arr, n, C.c_uint64(window), C.c_uint64(stride), int(join), C.byref(out))
        return out.value

    def add_fc(self, inputs: Sequence[int], out_features: int, join: JoinRule = JoinRule.Concat) -> int:
        arr, n = self._ins(inputs)
        out = C.c_int32()
        _call("vdnn_graph_add_fc", self._h, arr, n, C.c_uint64(out_features), int(join), C.byref(out))
        return out.value

    def add_loss(self, inp: int) -> int:
        out = C.c_int32()
        _call("vdnn_graph_add_loss", self._h, int(inp), C.byref(out))
        return out.value

    def finalize(self) -> "NetworkGraph":
        _call("vdnn_graph_finalize", self._h)
        self._finalized = True
        return self

    def size(self) -> int:
        n = C.c_int32()
        _call("vdnn_graph_size", self._h, C.byref(n))
        return n.value

    def __len__(self) -> int:
        return self.size()

    @property
    def batch(self) -> int:
        b = C.c_uint64()
        _call("vdnn_graph_batch", self._h, C.byref(b))
        return b.value

    def _info(self, id: int) -> L.LayerInfo:
        info = L.LayerInfo()
        _call("vdnn_graph_layer", self._h, int(id), C.byref(info))
        return info

    def layer(self, id: int) -> LayerDescriptor:
        i = self._info(id)
        return LayerDescriptor(i.id, LayerKind(i.kind), tuple(i.inputs[: i.n_inputs]), JoinRule(i.join),
                               (i.p0, i.p1, i.p2, i.p3))

    def layers(self) -> List[LayerDescriptor]:
        return [self.layer(i) for i in range(self.size())]

    def shape(self, id: int) -> TensorShape:
        i = self._info(id)
        return TensorShape(i.n, i.c, i.h, i.w)

    def refcnt(self, id: int) -> int:
        return self._info(id).refcnt

    def count_kind(self, k: LayerKind) -> int:
        return sum(1 for l in self.layers() if l.kind == k)

    def spec(self) -> str:
        """Text form consumed by the oracle shim (oracle/ref_shim.cpp)."""
        parts = [f"B={self.batch}"]
        names = ["input", "conv", "actv", "pool", "fc", "loss"]
        for l in self.layers():
            ins = ",".join(str(q) for q in l.inputs) if l.inputs else "-"
            parts.append(f"{names[l.kind]} {ins} {l.params[0]} {l.params[1]} {l.params[2]} {l.params[3]} {int(l.join)}")
        return "|".join(parts)


def build_preset(name: str, batch: int) -> NetworkGraph:
    h = C.c_void_p()
    _call("vdnn_preset", name.encode(), C.c_uint64(batch), C.byref(h))
    return NetworkGraph(_handle=h)


def extend_vgg(extra_conv_layers: int, batch: int) -> NetworkGraph:
    h = C.c_void_p()
    _call("vdnn_extend_vgg", int(extra_conv_layers), C.c_uint64(batch), C.byref(h))
    return NetworkGraph(_handle=h)


# ------------------------------------------------------------- cost model --
@dataclass
class CostModel:
    """cost_model.hpp:15-26,65-75 (defaults: Titan X, PCIe 3)."""
    peak_flops: float = 7e12
    dram_bw: float = 336e9
    mem_capacity: int = 12884901888
    compute_efficiency: float = 0.5
    link_effective_bw: float = 12.8e9
    link_nominal_bw: float = 16e9
    link_fixed_launch_overhead: float = 0.0
    elem_size: int = 4
    bwd_fwd_ratio: float = 2.0
    speed_factor_implicit_gemm: float = 1.0
    speed_factor_gemm_ws: float = 0.8
    speed_factor_fft: float = 0.6
    latency_overrides: Dict[int, Tuple[float, float]] = field(default_factory=dict)

    def _c(self):
        cm = L.CostModelC()
        cm.peak_flops = self.peak_flops
        cm.dram_bw = self.dram_bw
        cm.mem_capacity = self.mem_capacity
        cm.compute_efficiency = self.compute_efficiency
        cm.link_effective_bw = self.link_effective_bw
        cm.link_nominal_bw = self.link_nominal_bw
        cm.link_launch_overhead = self.link_fixed_launch_overhead
        cm.elem_size = self.elem_size
        cm.bwd_fwd_ratio = self.bwd_fwd_ratio
        cm.speed_factor_implicit_gemm = self.speed_factor_implicit_gemm
        cm.speed_factor_gemm_ws = self.speed_factor_gemm_ws
        cm.speed_factor_fft = self.speed_factor_fft
        ids = sorted(self.latency_overrides)
        n = len(ids)
        keep = ((C.c_int32 * max(n, 1))(*ids), (C.c_double * max(n, 1))(*[self.latency_overrides[i][0] for i in ids]),
                (C.c_double * max(n, 1))(*[self.latency_overrides[i][1] for i in ids]))
        cm.n_overrides = n
        cm.override_layer = C.cast(keep[0], C.POINTER(C.c_int32))
        cm.override_fwd_s = C.cast(keep[1], C.POINTER(C.c_double))
        cm.override_bwd_s = C.cast(keep[2], C.POINTER(C.c_double))
        cm._keep = keep
        return cm

    def spec(self) -> str:
        """Text form consumed by the oracle shim."""
        kv = (f"pf={self.peak_flops!r},bw={self.dram_bw!r},cap={self.mem_capacity},eff={self.compute_efficiency!r},"
              f"lbw={self.link_effective_bw!r},lnom={self.link_nominal_bw!r},lov={self.link_fixed_launch_overhead!r},"
              f"es={self.elem_size},ratio={self.bwd_fwd_ratio!r},sfi={self.speed_factor_implicit_gemm!r},"
              f"sfg={self.speed_factor_gemm_ws!r},sff={self.speed_factor_fft!r}")
        if self.latency_overrides:
            kv += ";ov=" + ",".join(f"{i}:{f!r}:{b!r}" for i, (f, b) in sorted(self.latency_overrides.items()))
        return kv

    def _u64(self, fn, g, id, *extra):
        out = C.c_uint64()
        cm = self._c()
        _call(fn, C.byref(cm), g.handle, int(id), *extra, C.byref(out))
        return out.value

    def tensor_bytes_of_layer(self, g: NetworkGraph, id: int) -> int:
        return self._u64("vdnn_cost_tensor_bytes", g, id)

    def tensor_bytes_of(self, shape: TensorShape) -> int:
        return shape.elements() * self.elem_size

    def weight_bytes(self, g: NetworkGraph, id: int) -> int:
        return self._u64("vdnn_cost_weight_bytes", g, id)

    def conv_workspace(self, g: NetworkGraph, id: int, algo: AlgoId) -> int:
        return self._u64("vdnn_cost_conv_workspace", g, id, int(algo))

    def layer_latency(self, g: NetworkGraph, id: int, bwd: bool = False, algo: AlgoId = AlgoId.ImplicitGemm) -> float:
        out = C.c_double()
        cm = self._c()
        _call("vdnn_cost_layer_latency", C.byref(cm), g.handle, int(id), int(bool(bwd)), int(algo), C.byref(out))
        return out.value

    def flops(self, g: NetworkGraph, id: int, bwd: bool = False) -> float:
        out = C.c_double()
        cm = self._c()
        _call("vdnn_cost_flops", C.byref(cm), g.handle, int(id), int(bool(bwd)), C.byref(out))
        return out.value

    def transfer_latency(self, nbytes: int) -> float:
        out = C.c_double()
        cm = self._c()
        _call("vdnn_cost_transfer_latency", C.byref(cm), C.c_uint64(nbytes), C.byref(out))
        return out.value

    def fastest_algo(self, g: NetworkGraph, id: int) -> AlgoId:
        out = C.c_int32()
        cm = self._c()
        _call("vdnn_cost_fastest_algo", C.byref(cm), g.handle, int(id), C.byref(out))
        return AlgoId(out.value)

    def fft_applicable(self, g: NetworkGraph, id: int) -> bool:
        l = g.layer(id)
        return l.kind == LayerKind.Conv and l.params[1] == 1

    def offload_interference_bound(self) -> float:
        return self.link_nominal_bw / self.dram_bw


def gradient_map_bytes(g: NetworkGraph, m: int, cm: CostModel) -> int:
    return cm._u64("vdnn_gradient_map_bytes", g, m)


# -------------------------------------------------------------- decisions --
@dataclass
class PolicyDecision:
    """decision.hpp:30-57."""
    offload: List[int]
    algos: Dict[int, AlgoId]
    gradient_scheme: GradientScheme = GradientScheme.PerLayer
    label: str = ""

    def offloads(self, id: int) -> bool:
        return bool(self.offload[id])

    @classmethod
    def _from_handle(cls, h) -> "PolicyDecision":
        n = C.c_int32()
        _call("vdnn_decision_get", h, C.byref(n), None, None, None, None, C.c_size_t(0))
        flags = (C.c_char * max(n.value, 1))()
        algos = (C.c_int32 * max(n.value, 1))()
        scheme = C.c_int32()
        label = C.create_string_buffer(256)
        _call("vdnn_decision_get", h, C.byref(n), flags, algos, C.byref(scheme), label, C.c_size_t(256))
        return cls([1 if flags[i] != b"\x00" else 0 for i in range(n.value)],
                   {i: AlgoId(algos[i]) for i in range(n.value) if algos[i] >= 0},
                   GradientScheme(scheme.value), label.value.decode())

    def _handle(self, g: NetworkGraph):
        h = C.c_void_p()
        _call("vdnn_decision_create", g.handle, C.byref(h))
        try:
            # the C side sizes offload to the graph; re-create if sizes differ (validate reports it)
            if len(self.offload) != g.size():
                raise InvalidDecision(L.INVALID_DECISION, "offload flags do not cover the graph")
            for i, f in enumerate(self.offload):
                if f:
                    _call("vdnn_decision_set_offload", h, i, 1)
            for i, a in self.algos.items():
                _call("vdnn_decision_set_algo", h, int(i), int(a))
            _call("vdnn_decision_set_scheme", h, int(self.gradient_scheme))
            _call("vdnn_decision_set_label", h, self.label.encode())
        except Exception:
            L.lib().vdnn_decision_destroy(h)
            raise
        return _Owned(h, "vdnn_decision_destroy")

    def validate(self, g: NetworkGraph) -> None:
        d = self._handle(g)
        _call("vdnn_decision_validate", d.h, g.handle)

    def spec(self) -> str:
        """Oracle-shim form: custom:<scheme>:<label>:<offload ids>:<id=algo>."""
        off = ",".join(str(i) for i, f in enumerate(self.offload) if f)
        alg = ",".join(f"{i}={int(a)}" for i, a in sorted(self.algos.items()))
        return f"custom:{int(self.gradient_scheme)}:{self.label}:{off}:{alg}"


class _Owned:
    def __init__(self, h, destroy):
        self.h = h
        self._destroy = destroy

    def __del__(self):
        if self.h is not None and self.h.value and L._lib is not None:
            getattr(L._lib, self._destroy)(self.h)
            self.h = None


class _Borrowed:
    def __init__(self, h):
        self.h = h


def static_decision(kind: PolicyKind, mode: AlgoMode, g: NetworkGraph, cm: CostModel) -> PolicyDecision:
    h = C.c_void_p()
    c = cm._c()
    _call("vdnn_decision_static", g.handle, int(kind), int(mode), C.byref(c), C.byref(h))
    o = _Owned(h, "vdnn_decision_destroy")
    return PolicyDecision._from_handle(o.h)


# ---------------------------------------------------------------- reports --
@dataclass
class StreamEvent:
    stream: Stream
    kind: EventKind
    layer: int
    start: int
    end: int
    bytes: int
    tag: str = ""
    buffer: int = -1
    offset: int = 0


@dataclass
class OomInfo:
    layer: int
    phase: Phase
    fragmented: bool
    requested: int
    tag: str


@dataclass
class SimOptions:
    keep_pool_trace: bool = False
    include_weight_grads: bool = False


class RunReport:
    """sim_types.hpp:63-90; events are materialised lazily."""

    def __init__(self, handle, owned: bool = True):
        self._own = _Owned(handle, "vdnn_report_destroy") if owned else _Borrowed(handle)
        s = L.ReportSummary()
        _call("vdnn_report_summary_get", handle, C.byref(s))
        self.pass_ = bool(s.pass_)
        self.oom = (OomInfo(s.oom_layer, Phase(s.oom_phase), bool(s.oom_fragmented), s.oom_requested,
                            s.oom_tag.decode()) if s.has_oom else None)
        self.max_mem_bytes = s.max_mem_bytes
        self.avg_mem_bytes = s.avg_mem_bytes
        self.offload_traffic_bytes = s.offload_traffic_bytes
        self.prefetch_traffic_bytes = s.prefetch_traffic_bytes
        self.host_peak_bytes = s.host_peak_bytes
        self.stall_fwd_offload_ns = s.stall_fwd_offload_ns
        self.stall_bwd_prefetch_ns = s.stall_bwd_prefetch_ns
        self.total_ns = s.total_ns
        self.interference_bound = s.interference_bound
        self._verdict = s.verdict.decode()
        self._n = s.n_events
        self._events = None

    @property
    def handle(self):
        return self._own.h

    def verdict(self) -> str:
        return self._verdict

    def stall_ns(self) -> int:
        return self.stall_fwd_offload_ns + self.stall_bwd_prefetch_ns

    def raw_events(self):
        arr = (L.Event * max(self._n, 1))()
        n = C.c_size_t()
        _call("vdnn_report_events", self.handle, arr, C.c_size_t(self._n), C.byref(n))
        return arr, n.value

    @property
    def events(self) -> List[StreamEvent]:
        if self._events is None:
            arr, n = self.raw_events()
            self._events = [StreamEvent(Stream(e.stream), EventKind(e.kind), e.layer, e.start_ns, e.end_ns, e.bytes,
                                        e.tag.decode(), e.buffer, e.offset) for e in arr[:n]]
        return self._events

    @property
    def reuse_distance_ns(self) -> List[int]:
        n = C.c_size_t()
        _call("vdnn_report_reuse_distance", self.handle, None, C.c_size_t(0), C.byref(n))
        out = (C.c_int64 * max(n.value, 1))()
        _call("vdnn_report_reuse_distance", self.handle, out, n, C.byref(n))
        return list(out[: n.value])

    def pool_trace(self):
        n = C.c_size_t()
        _call("vdnn_report_pool_trace", self.handle, None, C.c_size_t(0), C.byref(n))
        out = (L.PoolTraceRow * max(n.value, 1))()
        _call("vdnn_report_pool_trace", self.handle, out, n, C.byref(n))
        return [(r.time_ns, r.op.decode(), r.tag.decode(), r.offset, r.bytes, r.current, r.high_water)
                for r in out[: n.value]]

    def signature(self) -> str:
        s = C.c_uint64()
        _call("vdnn_report_signature", self.handle, C.byref(s))
        return f"{s.value:016x}"

    def layer_peaks(self, layers: int) -> Tuple[List[int], List[int]]:
        f = (C.c_uint64 * max(layers, 1))()
        b = (C.c_uint64 * max(layers, 1))()
        _call("vdnn_report_layer_peaks", self.handle, int(layers), f, b)
        return list(f[:layers]), list(b[:layers])


def simulate(g: NetworkGraph, decision: PolicyDecision, cost: CostModel, capacity: int,
             options: Optional[SimOptions] = None) -> RunReport:
    options = options or SimOptions()
    d = decision._handle(g)
    c = cost._c()
    flags = (1 if options.keep_pool_trace else 0) | (2 if options.include_weight_grads else 0)
    h = C.c_void_p()
    _call("vdnn_simulate", g.handle, d.h, C.byref(c), C.c_uint64(capacity), C.c_uint32(flags), C.byref(h))
    return RunReport(h)


def simulate_with_trace(g, decision, cost, capacity, options: Optional[SimOptions] = None):
    opts = SimOptions(True, (options or SimOptions()).include_weight_grads)
    r = simulate(g, decision, cost, capacity, opts)
    return r, r.pool_trace()


def simulate_oracle(g: NetworkGraph, cost: CostModel) -> RunReport:
    c = cost._c()
    h = C.c_void_p()
    _call("vdnn_simulate_oracle", g.handle, C.byref(c), C.byref(h))
    return RunReport(h)


def per_layer_event_peaks(report: RunReport, layers: int) -> Tuple[List[int], List[int]]:
    return report.layer_peaks(layers)


@dataclass
class ProfilePassResult:
    phase: str
    decision: PolicyDecision
    pass_: bool
    oom: Optional[OomInfo]
    total_ns: int
    max_mem_bytes: int


@dataclass
class DynamicSelection:
    decision: Optional[PolicyDecision]
    passes: List[ProfilePassResult]

    def untrainable(self) -> bool:
        return self.decision is None


def dynamic_select(g: NetworkGraph, capacity: int, cost: CostModel) -> DynamicSelection:
    c = cost._c()
    h = C.c_void_p()
    _call("vdnn_dynamic_select", g.handle, C.c_uint64(capacity), C.byref(c), C.byref(h))
    own = _Owned(h, "vdnn_dyn_destroy")
    n = C.c_size_t()
    _call("vdnn_dyn_passes", own.h, None, C.c_size_t(0), C.byref(n))
    infos = (L.PassInfo * max(n.value, 1))()
    _call("vdnn_dyn_passes", own.h, infos, n, C.byref(n))
    passes = []
    for i, p in enumerate(infos[: n.value]):
        dh = C.c_void_p()
        _call("vdnn_dyn_pass_decision", own.h, C.c_size_t(i), C.byref(dh))
        down = _Owned(dh, "vdnn_decision_destroy")
        d = PolicyDecision._from_handle(down.h)
        oom = OomInfo(p.oom_layer, Phase(p.oom_phase), False, 0, "") if p.has_oom else None
        passes.append(ProfilePassResult(p.phase.decode(), d, bool(p.pass_), oom, p.total_ns, p.max_mem_bytes))
    u = C.c_int32()
    _call("vdnn_dyn_untrainable", own.h, C.byref(u))
    dec = None
    if not u.value:
        dh = C.c_void_p()
        _call("vdnn_dyn_decision", own.h, C.byref(dh))
        down = _Owned(dh, "vdnn_decision_destroy")
        dec = PolicyDecision._from_handle(down.h)
    return DynamicSelection(dec, passes)


def greedy_downgrade(g: NetworkGraph, capacity: int, offload_kind: PolicyKind, cost: CostModel
                     ) -> Optional[PolicyDecision]:
    c = cost._c()
    found = C.c_int32()
    h = C.c_void_p()
    _call("vdnn_greedy_downgrade", g.handle, C.c_uint64(capacity), int(offload_kind), C.byref(c), C.byref(found),
          C.byref(h))
    if not found.value:
        return None
    own = _Owned(h, "vdnn_decision_destroy")
    return PolicyDecision._from_handle(own.h)


@dataclass
class Violation:
    kind: str
    detail: str


def replay_check(report: RunReport, g: NetworkGraph, decision: PolicyDecision, capacity: int) -> List[Violation]:
    d = decision._handle(g)
    n = C.c_size_t()
    _call("vdnn_replay_check", report.handle, g.handle, d.h, C.c_uint64(capacity), None, C.c_size_t(0), C.byref(n))
    out = (L.Violation * max(n.value, 1))()
    _call("vdnn_replay_check", report.handle, g.handle, d.h, C.c_uint64(capacity), out, n, C.byref(n))
    return [Violation(v.kind.decode(), v.detail.decode()) for v in out[: n.value]]


def program_check(g: NetworkGraph, decision: PolicyDecision, cost: "CostModel", capacity: int) -> List[Violation]:
    """Compile the plan's executable program (the executor's operand bindings,
    scratch gaps, transfers) and check it against the plan's own event log."""
    d = decision._handle(g)
    cm = cost._c()
    n = C.c_size_t()
    _call("vdnn_program_check", g.handle, d.h, C.byref(cm), C.c_uint64(capacity), None, C.c_size_t(0), C.byref(n))
    out = (L.Violation * max(n.value, 1))()
    _call("vdnn_program_check", g.handle, d.h, C.byref(cm), C.c_uint64(capacity), out, n, C.byref(n))
    return [Violation(v.kind.decode(), v.detail.decode()) for v in out[: n.value]]


@dataclass
class FootprintReport:
    weights_bytes: int
    feature_maps_bytes: int
    gradient_buffers_bytes: int
    workspace_bytes: int
    total_bytes: int
    classifier_bytes: int

    def feature_map_fraction(self) -> float:
        return 0.0 if self.total_bytes == 0 else self.feature_maps_bytes / self.total_bytes


def baseline_footprint(g: NetworkGraph, algos: Dict[int, AlgoId], cost: CostModel,
                       include_weight_grads: bool = False) -> FootprintReport:
    dec = PolicyDecision([0] * g.size(), dict(algos), GradientScheme.PerLayer, "")
    d = dec._handle(g)
    c = cost._c()
    f = L.Footprint()
    _call("vdnn_baseline_footprint", g.handle, d.h, C.byref(c), int(bool(include_weight_grads)), C.byref(f))
    return FootprintReport(f.weights_bytes, f.feature_maps_bytes, f.gradient_buffers_bytes, f.workspace_bytes,
                           f.total_bytes, f.classifier_bytes)


def report_from_events(events, summary: Dict) -> RunReport:
    """Wrap an externally produced event log (e.g. measured) as a RunReport."""
    n = len(events)
    arr = (L.Event * max(n, 1))()
    for i, e in enumerate(events):
        arr[i].stream, arr[i].kind, arr[i].layer, arr[i].buffer = int(e.stream), int(e.kind), e.layer, e.buffer
        arr[i].start_ns, arr[i].end_ns, arr[i].bytes, arr[i].offset = e.start, e.end, e.bytes, e.offset
        arr[i].tag = e.tag.encode()
    s = L.ReportSummary()
    for k, v in summary.items():
        setattr(s, k, v)
    h = C.c_void_p()
    _call("vdnn_report_from_events", arr, C.c_size_t(n), C.byref(s), C.byref(h))
    return RunReport(h)


# ---------------------------------------------------------------- session --
class Session:
    """B200 training session: replays the plan of (graph, decision, capacity)
    on one device arena + pinned host arena with compute/memory streams.

    There is no CPU fallback: creating a session needs a CUDA device and the
    in-tree libvdnn.so; every failure raises.
    """

    def __init__(self, g: NetworkGraph, decision: PolicyDecision, cost: Optional[CostModel] = None,
                 capacity: int = 12884901888, device: int = 0, weight_seed: int = 5000,
                 external_grads: bool = False, record_timeline: bool = False, precise_fp32: bool = False,
                 compress_offload=False, offload_target: str = "host", cuda_graph: bool = False,
                 algo_kernels: str = "fastest"):
        """compress_offload: move offloads/prefetches through the SMs in a
        lossless zero-value-compressed form (same schedule, bit-identical
        restored buffers, fewer bytes on the host link). "tf32": the same,
        and maps whose backward readers are only TF32 contractions and ReLU
        masks travel TF32-exact (the 13 low mantissa bits the tensor core
        ignores are dropped; the training step stays bit-identical).
        offload_target: "host" (pinned host memory over PCIe, the reference's
        model) or "device" (a device buffer given to set_offload_buffer, or a
        peer GPU's spill buffer via spill_export / spill_attach: NVLink).
        cuda_graph: replay each step as one CUDA graph (captured on the second
        step; re-captured when lr changes).
        algo_kernels: "fastest" runs the implicit-GEMM kernels for every planned
        conv algorithm (the planned workspace is still reserved); "planned" runs
        GEMM_WS layers as the reference's algorithm -- im2col into the planned
        workspace + a 1x1 GEMM (cost_model.hpp:163-168); FFT layers stay
        implicit (no FFT kernel: slower than implicit GEMM on this part,
        profiles/r02s4_algo_probe.txt)."""
        if algo_kernels not in ("fastest", "planned"):
            raise ValueError(f"algo_kernels must be 'fastest' or 'planned', not {algo_kernels!r}")
        if offload_target not in ("host", "device"):
            raise ValueError(f"offload_target must be 'host' or 'device', not {offload_target!r}")
        self.graph = g
        self.decision = decision
        self.cost = cost or CostModel()
        self.capacity = capacity
        opt = L.SessionOptions()
        L.lib().vdnn_session_options_default(C.byref(opt))
        opt.device = device
        opt.weight_seed = weight_seed
        opt.external_grads = int(external_grads)
        opt.record_timeline = int(record_timeline)
        opt.precise_fp32 = int(precise_fp32)
        if compress_offload not in (False, True, 0, 1, "zvc", "tf32"):
            raise ValueError(f"compress_offload must be a bool, 'zvc' or 'tf32', not {compress_offload!r}")
        opt.compress_offload = 2 if compress_offload == "tf32" else int(bool(compress_offload))
        opt.offload_target = 0 if offload_target == "host" else 1
        opt.cuda_graph = int(cuda_graph)
        opt.algo_kernels = 1 if algo_kernels == "planned" else 0
        d = decision._handle(g)
        c = self.cost._c()
        h = C.c_void_p()
        _call("vdnn_session_create", g.handle, d.h, C.byref(c), C.c_uint64(capacity), C.byref(opt), C.byref(h))
        self._own = _Owned(h, "vdnn_session_destroy")
        self.plan = RunReport(C.c_void_p(L.lib().vdnn_session_plan(h)), owned=False)
        self._plan_keepalive = self._own
        self.batch = g.batch
        self._loss = C.c_float()
        # storage format of every pool tensor (cost_model.hpp:69): fp32, or bf16 at elem_size 2
        self.bf16 = self.cost.elem_size == 2
        self.elem_size = 2 if self.bf16 else 4

    def _storage(self, a):
        """Host array -> the session's storage format (fp32, or bf16 bit patterns)."""
        import numpy as np
        a = np.ascontiguousarray(a, dtype=np.float32)
        return to_bf16_bits(a) if self.bf16 else a

    @property
    def handle(self):
        return self._own.h

    def arena_info(self) -> Dict[str, int]:
        a, lo, hb, sb = C.c_uint64(), C.c_uint64(), C.c_uint64(), C.c_uint64()
        _call("vdnn_session_arena_info", self.handle, C.byref(a), C.byref(lo), C.byref(hb), C.byref(sb))
        return {"arena_bytes": a.value, "arena_base_offset": lo.value, "host_arena_bytes": hb.value,
                "scratch_bytes": sb.value}

    def transfer_stats(self) -> Dict[str, int]:
        """Cumulative host-link bytes since creation: what crossed PCIe (wire)
        and what the plan moved (planned), per direction."""
        v = [C.c_uint64() for _ in range(4)]
        _call("vdnn_session_transfer_stats", self.handle, *[C.byref(x) for x in v])
        return {"offload_wire": v[0].value, "prefetch_wire": v[1].value, "offload_planned": v[2].value,
                "prefetch_planned": v[3].value}

    def set_batch(self, images, labels) -> None:
        """Host arrays: images float32 NHWC [N,H,W,C] (C-contiguous; rounded to
        bf16 for an elem_size-2 session), labels int32 [N]."""
        import numpy as np
        im = self._storage(images)
        lb = np.ascontiguousarray(labels, dtype=np.int32)
        _call("vdnn_session_set_batch_host", self.handle, im.ctypes.data_as(C.c_void_p),
              lb.ctypes.data_as(C.c_void_p))
        self._keep = (im, lb)  # the copy is asynchronous: keep sources alive until the next call

    def set_input(self, layer: int, images) -> None:
        """Images (float32 NHWC host array) of one INPUT layer of a multi-input graph."""
        im = self._storage(images)
        _call("vdnn_session_set_input", self.handle, int(layer), im.ctypes.data_as(C.c_void_p), 0)
        self._keep_inputs = getattr(self, "_keep_inputs", {})
        self._keep_inputs[layer] = im  # asynchronous copy: keep the source alive

    def set_batch_ptr(self, images_ptr: int, labels_ptr: int, device: bool = False) -> None:
        fn = "vdnn_session_set_batch_device" if device else "vdnn_session_set_batch_host"
        _call(fn, self.handle, C.c_void_p(images_ptr), C.c_void_p(labels_ptr))

    def prefetch_batch_ptr(self, images_ptr: int, labels_ptr: int) -> None:
        """Stage the NEXT batch from pinned host memory on the input stream
        (overlapping the running step); the next step() consumes it."""
        _call("vdnn_session_prefetch_batch_host", self.handle, C.c_void_p(images_ptr), C.c_void_p(labels_ptr))

    def read_loss(self) -> float:
        """Loss of the last step (after step(want_loss=False))."""
        _call("vdnn_session_read_loss", self.handle, C.byref(self._loss))
        return float(self._loss.value)

    def queue_loss(self) -> int:
        """Queue the D2H of the last step's loss; returns a ticket for wait_loss."""
        t = C.c_int64()
        _call("vdnn_session_queue_loss", self.handle, C.byref(t))
        return t.value

    def wait_loss(self, ticket: int) -> float:
        v = C.c_float()
        _call("vdnn_session_wait_loss", self.handle, C.c_int64(ticket), C.byref(v))
        return float(v.value)

    def synthetic_batch(self, seed: int = 1234) -> None:
        _call("vdnn_session_synthetic_batch", self.handle, C.c_uint64(seed))

    def step(self, lr: float = 0.01, want_loss: bool = True) -> Optional[float]:
        if want_loss:
            _call("vdnn_session_step", self.handle, C.c_float(lr), C.byref(self._loss))
            return float(self._loss.value)
        _call("vdnn_session_step", self.handle, C.c_float(lr), None)
        return None

    def synchronize(self) -> None:
        _call("vdnn_session_synchronize", self.handle)

    def pause_timeline(self, paused: bool = True) -> None:
        """record_timeline sessions: skip (or resume) the per-op timing events;
        measured_report / layer_times describe the last step recorded."""
        _call("vdnn_session_pause_timeline", self.handle, C.c_int32(int(paused)))

    def weight_count(self, layer: int) -> int:
        return self.cost.weight_bytes(self.graph, layer) // self.elem_size

    def get_weights(self, layer: int):
        import numpy as np
        n = self.weight_count(layer)
        out = np.empty(n, dtype=np.float32)
        _call("vdnn_session_get_weights", self.handle, int(layer), out.ctypes.data_as(C.c_void_p), C.c_size_t(n))
        return out

    def set_weights(self, layer: int, values) -> None:
        import numpy as np
        v = np.ascontiguousarray(values, dtype=np.float32).ravel()
        _call("vdnn_session_set_weights", self.handle, int(layer), v.ctypes.data_as(C.c_void_p),
              C.c_size_t(v.size))

    def read_feature(self, owner: int, count: int):
        import numpy as np
        out = np.empty(count, dtype=np.float32)
        _call("vdnn_session_read_feature", self.handle, int(owner), out.ctypes.data_as(C.c_void_p),
              C.c_size_t(count))
        return out

    def measured_report(self) -> RunReport:
        h = C.c_void_p()
        _call("vdnn_session_measured_report", self.handle, C.byref(h))
        return RunReport(h)

    def layer_times(self):
        n = self.graph.size()
        f = (C.c_double * n)()
        b = (C.c_double * n)()
        _call("vdnn_session_layer_times", self.handle, n, f, b)
        return list(f), list(b)

    def grad_arena(self) -> Tuple[int, int]:
        p = C.c_void_p()
        n = C.c_size_t()
        _call("vdnn_session_grad_arena", self.handle, C.byref(p), C.byref(n))
        return (p.value or 0), n.value

    def get_grads(self, layer: int):
        """dW (and FC bias gradient) of the last step; needs external_grads=True."""
        import numpy as np
        n = self.weight_count(layer)
        out = np.empty(n, dtype=np.float32)
        _call("vdnn_session_get_grads", self.handle, int(layer), out.ctypes.data_as(C.c_void_p), C.c_size_t(n))
        return out

    def set_grad_arena(self, dev_ptr: int, count: int) -> None:
        _call("vdnn_session_set_grad_arena", self.handle, C.c_void_p(dev_ptr), C.c_size_t(count))

    def apply_grads(self, lr: float, scale: float = 1.0) -> None:
        _call("vdnn_session_apply_grads", self.handle, C.c_float(lr), C.c_float(scale))

    # -- device offload target (offload_target="device") --
    def offload_bytes(self) -> int:
        v = C.c_uint64()
        _call("vdnn_session_offload_bytes", self.handle, C.byref(v))
        return v.value

    def set_offload_buffer(self, dev_ptr: int, nbytes: int) -> None:
        _call("vdnn_session_set_offload_buffer", self.handle, C.c_void_p(dev_ptr), C.c_uint64(nbytes))

    def spill_export(self) -> bytes:
        """Allocate this rank's spill buffer (offload_bytes) and return its IPC handle."""
        h = (C.c_uint8 * 64)()
        _call("vdnn_session_spill_export", self.handle, h)
        return bytes(h)

    def spill_attach(self, handle: bytes) -> None:
        """Offload into the spill buffer a peer exported (NVLink instead of PCIe)."""
        h = (C.c_uint8 * 64).from_buffer_copy(handle)
        _call("vdnn_session_spill_attach", self.handle, h)

    # -- data-parallel exchange over peer memory (vdnn_session_peer_*) --
    def peer_export(self) -> bytes:
        """This rank's IPC handles (opaque bytes, to be all-gathered)."""
        h = L.PeerHandle()
        _call("vdnn_session_peer_export", self.handle, C.byref(h))
        return bytes(h)

    def peer_attach(self, rank: int, handles: List[bytes]) -> None:
        """Map every rank's arenas (handles[i] = rank i's peer_export())."""
        arr = (L.PeerHandle * len(handles))()
        for i, b in enumerate(handles):
            C.memmove(C.byref(arr[i]), b, C.sizeof(L.PeerHandle))
        _call("vdnn_session_peer_attach", self.handle, C.c_int32(rank), C.c_int32(len(handles)), arr)

    def peer_exchange(self, lr: float, scale: float = 1.0) -> None:
        """Fused all-reduce + SGD + weight broadcast on the compute stream."""
        _call("vdnn_session_peer_exchange", self.handle, C.c_float(lr), C.c_float(scale))

    def peer_overlap(self, on: bool = True, scale: float = 1.0) -> None:
        """Exchange each layer inside step(), on a side stream right after that
        layer's wgrad (overlapping the rest of backward); bit-identical to
        peer_exchange after the step."""
        _call("vdnn_session_peer_overlap", self.handle, C.c_int32(int(on)), C.c_float(scale))

    def peer_detach(self) -> None:
        _call("vdnn_session_peer_detach", self.handle)

    # -- layer-local probe (parity tests) --
    PROBE_NAMES = ("X", "W", "Y", "DY", "DX_BEFORE", "DX", "DW", "LOSS_GRAD", "LOSS")

    def probe_layout(self, layer: int, bwd: bool) -> Dict:
        """Segments the probe of FWD/BWD(layer) copies, and the fusions that step applies."""
        lay = L.ProbeLayout()
        _call("vdnn_session_probe_layout", self.handle, int(layer), int(bool(bwd)), C.byref(lay))
        segs = [(self.PROBE_NAMES[lay.seg[i].what], lay.seg[i].index, bool(lay.seg[i].after),
                 lay.seg[i].offset, lay.seg[i].bytes) for i in range(lay.nseg)]
        return {"segs": segs, "total_bytes": lay.total_bytes, "relu_fused": bool(lay.relu_fused),
                "accumulate": bool(lay.accumulate), "skip": bool(lay.skip), "mask_planes": lay.mask_planes}

    def probe_step(self, probes, lr: float = 0.01, device: int = 0):
        """Run one step with layer-local probes armed: probes = [(layer, bwd), ...].
        Returns (loss, {(layer, bwd): {(name, index[, "after"]): torch fp32 tensor on the device}}):
        each operand as the step's kernels read it (before) or wrote it (after). Pool tensors of a
        bf16 session are widened exactly to fp32; DW (the fp32 gradient arena) and LOSS are fp32."""
        import torch
        bufs, lays = {}, {}
        for layer, bwd in probes:
            lay = self.probe_layout(layer, bwd)
            buf = torch.empty(max(4, lay["total_bytes"]), dtype=torch.uint8, device=f"cuda:{device}")
            _call("vdnn_session_arm_probe", self.handle, int(layer), int(bool(bwd)), C.c_void_p(buf.data_ptr()),
                  C.c_uint64(buf.numel()))
            bufs[(layer, bwd)], lays[(layer, bwd)] = buf, lay
        loss = self.step(lr)
        self.synchronize()
        out = {}
        for key, lay in lays.items():
            d = {"_layout": lay}
            for name, idx, after, off, nb in lay["segs"]:
                raw = bufs[key][off: off + nb]
                if self.bf16 and name not in ("DW", "LOSS"):
                    t = raw.view(torch.bfloat16).float()
                else:
                    t = raw.view(torch.float32)
                d[(name, idx, "after") if (after and name == "W") else (name, idx)] = t
            out[key] = d
        return loss, out

    @property
    def stream(self) -> int:
        p = C.c_void_p()
        _call("vdnn_session_stream", self.handle, C.byref(p))
        return p.value or 0


def placements(r: "RunReport"):
    """(kind, layer, buffer, tag, bytes, offset) of every non-SYNC event in log
    order: what a schedule places where. SYNC rows (stalls) depend on timing
    -- a measured log and a re-planned one stall at other steps -- everything
    else is timing-independent (the schedule signature covers the same rows)."""
    return [(int(e.kind), e.layer, e.buffer, e.tag, e.bytes, e.offset) for e in r.events
            if e.kind != EventKind.Sync]


def to_bf16_bits(a):
    """float32 array -> uint16 bf16 bit patterns, round to nearest even (NaN kept NaN)."""
    import numpy as np
    u = np.ascontiguousarray(a, dtype=np.float32).view(np.uint32)
    r = ((u + np.uint32(0x7FFF) + ((u >> np.uint32(16)) & np.uint32(1))) >> np.uint32(16)).astype(np.uint16)
    nan = (u & np.uint32(0x7FFFFFFF)) > np.uint32(0x7F800000)
    if nan.any():
        r[nan] = ((u[nan] >> np.uint32(16)) | np.uint32(0x40)).astype(np.uint16)
    return r


def from_bf16_bits(b):
    """uint16 bf16 bit patterns -> float32 (exact)."""
    import numpy as np
    return (np.ascontiguousarray(b, dtype=np.uint16).astype(np.uint32) << np.uint32(16)).view(np.float32)


def kernel_launch_count() -> int:
    return int(L.lib().vdnn_kernel_launch_count())
