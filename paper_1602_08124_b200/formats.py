"""Artefact formats of the reference, produced from planned *or measured* runs.

Schemas follow /root/reference/proj/include/vdnnsim/report.hpp so the
reference's own tooling (and its replay_check) can consume B200 logs:

* graph_to_json / graph_from_json ......... report.hpp:44-111
* decision_to_json / decision_from_json ... report.hpp:115-148
* report_to_json (+events) ................ report.hpp:152-193
* events_csv (six-column timeline) ........ report.hpp:196-204
* pool_trace_csv .......................... report.hpp:206-214
* profile_passes_csv ...................... report.hpp:228-236
* pool_trace_from_report / write_artifacts: the same files for a measured step
"""
from __future__ import annotations

import json
from typing import Dict, List

from . import api as V

_KIND = ["input", "conv", "actv", "pool", "fc", "loss"]
_ALGO = ["implicit_gemm", "gemm_ws", "fft"]
_EV = ["FWD", "BWD", "OFFLOAD", "PREFETCH", "ALLOC", "RELEASE", "SYNC"]
_STREAM = ["compute", "memory"]
_PHASE = ["setup", "forward", "backward"]


def graph_to_json(g: V.NetworkGraph) -> Dict:
    layers = []
    for l in g.layers():
        e = {"id": l.id, "kind": _KIND[l.kind]}
        if l.inputs:
            e["inputs"] = list(l.inputs)
        if len(l.inputs) > 1:
            e["join"] = "concat" if l.join == V.JoinRule.Concat else "eltwise"
        k, s, p, out = l.params
        if l.kind == V.LayerKind.Conv:
            e.update(kernel=k, stride=s, pad=p, out_channels=out)
        elif l.kind == V.LayerKind.Pool:
            e.update(window=k, stride=s)
        elif l.kind == V.LayerKind.Fc:
            e["out_features"] = k
        elif l.kind == V.LayerKind.Input:
            e.update(c=k, h=s, w=p)
        sh = g.shape(l.id)
        e["shape"] = [sh.n, sh.c, sh.h, sh.w]
        layers.append(e)
    return {"batch": g.batch, "layers": layers}


def graph_from_json(j: Dict) -> V.NetworkGraph:
    """report.hpp:80-111: generic add_layer per entry, checked at finalize."""
    try:
        g = V.NetworkGraph(int(j["batch"]))
        for e in j["layers"]:
            kind = e["kind"]
            if kind not in _KIND:
                raise V.ConfigError(9, "unknown layer kind: " + str(kind))
            k = V.LayerKind(_KIND.index(kind))
            ins = [int(x) for x in e.get("inputs", [])]
            join = V.JoinRule.Elementwise if e.get("join") == "eltwise" else V.JoinRule.Concat
            if k == V.LayerKind.Conv:
                params = (e["kernel"], e["stride"], e["pad"], e["out_channels"])
            elif k == V.LayerKind.Pool:
                params = (e["window"], e["stride"])
            elif k == V.LayerKind.Fc:
                params = (e["out_features"],)
            elif k == V.LayerKind.Input:
                params = (e["c"], e["h"], e["w"])
            else:
                params = ()
            g.add_layer(k, ins, [int(x) for x in params], join)
    except KeyError as ex:
        raise V.ConfigError(9, f"graph json: missing key {ex}")
    return g.finalize()


def decision_to_json(d: V.PolicyDecision) -> Dict:
    return {"label": d.label,
            "gradient_scheme": "two_buffer_reuse" if d.gradient_scheme == V.GradientScheme.TwoBufferReuse
            else "per_layer",
            "offload_layers": [i for i, f in enumerate(d.offload) if f],
            "algorithms": {str(i): _ALGO[int(a)] for i, a in sorted(d.algos.items())},
            "layer_count": len(d.offload)}


def decision_from_json(j: Dict, g: V.NetworkGraph) -> V.PolicyDecision:
    n = g.size()
    off = [0] * n
    for i in j["offload_layers"]:
        if int(i) >= n:
            raise V.InvalidDecision(8, "decision file references unknown layer")
        off[int(i)] = 1
    algos = {int(k): V.AlgoId(_ALGO.index(v)) for k, v in j["algorithms"].items()}
    scheme = (V.GradientScheme.TwoBufferReuse if j.get("gradient_scheme", "per_layer") == "two_buffer_reuse"
              else V.GradientScheme.PerLayer)
    d = V.PolicyDecision(off, algos, scheme, j.get("label", "decision-file"))
    d.validate(g)
    return d


def _event_json(e: V.StreamEvent) -> Dict:
    j = {"stream": _STREAM[e.stream], "kind": _EV[e.kind], "layer": e.layer, "start_ns": e.start,
         "end_ns": e.end, "bytes": e.bytes}
    if e.tag:
        j["tag"] = e.tag
    if e.buffer != -1:
        j["buffer"] = e.buffer
    if e.kind in (V.EventKind.Alloc, V.EventKind.Release):
        j["offset"] = e.offset
    return j


def report_to_json(r: V.RunReport, with_events: bool = True) -> Dict:
    j = {"verdict": r.verdict(), "pass": r.pass_}
    if r.oom is not None:
        j["oom"] = {"layer": r.oom.layer, "phase": _PHASE[r.oom.phase], "fragmented": r.oom.fragmented,
                    "requested_bytes": r.oom.requested, "tag": r.oom.tag}
    j.update(max_mem_bytes=r.max_mem_bytes, avg_mem_bytes=r.avg_mem_bytes,
             offload_traffic_bytes=r.offload_traffic_bytes, prefetch_traffic_bytes=r.prefetch_traffic_bytes,
             host_peak_bytes=r.host_peak_bytes, stall_fwd_offload_ns=r.stall_fwd_offload_ns,
             stall_bwd_prefetch_ns=r.stall_bwd_prefetch_ns, total_ns=r.total_ns,
             interference_bound=r.interference_bound, reuse_distance_ns=r.reuse_distance_ns)
    if with_events:
        j["events"] = [_event_json(e) for e in r.events]
    return j


def events_csv(r: V.RunReport) -> str:
    rows = ["stream,kind,layer,start_ns,end_ns,bytes"]
    for e in r.events:
        rows.append(f"{_STREAM[e.stream]},{_EV[e.kind]},{e.layer},{e.start},{e.end},{e.bytes}")
    return "\n".join(rows) + "\n"


def pool_trace_csv(trace) -> str:
    rows = ["time_ns,op,tag,offset,bytes,current,high_water"]
    for t, op, tag, off, nbytes, cur, hw in trace:
        rows.append(f"{t},{'alloc' if op == 'a' else 'free'},{tag},{off},{nbytes},{cur},{hw}")
    return "\n".join(rows) + "\n"


def profile_passes_csv(passes: List[V.ProfilePassResult]) -> str:
    rows = ["phase,decision,verdict,total_ns,max_mem_bytes"]
    for p in passes:
        rows.append(f"{p.phase},{p.decision.label},{'PASS' if p.pass_ else 'OOM'},{p.total_ns},{p.max_mem_bytes}")
    return "\n".join(rows) + "\n"


def calibrated_cost_model(session: "V.Session", link_gbs: float = None) -> V.CostModel:
    """pin every layer's planner latency to its measured B200
    time (CostModel.latency_overrides, cost_model.hpp:74-75,143-145) and,
    optionally, the link to the measured host bandwidth. Schedules, offsets and
    decisions are timing-independent, so re-planning with this model keeps
    them bit-identical while the planned timestamps track the hardware."""
    fwd, bwd = session.layer_times()
    base = session.cost
    cm = V.CostModel(**{k: getattr(base, k) for k in base.__dataclass_fields__ if k != "latency_overrides"})
    for i in range(session.graph.size()):
        if session.graph.layer(i).kind == V.LayerKind.Input:
            continue
        cm.latency_overrides[i] = (fwd[i] * 1e-3, bwd[i] * 1e-3)
    if link_gbs:
        cm.link_effective_bw = link_gbs * 1e9
    return cm


def pool_trace_from_report(r: V.RunReport, alignment: int = 512) -> List:
    """Pool trace (report.hpp:206-214 rows: time, op, tag, offset, bytes,
    current, high_water) of a *measured* log: the ALLOC / RELEASE events in log
    order, which is the order the planner's pool saw them
    (memory_pool.hpp:84,96), with lengths rounded to the pool alignment
    (memory_pool.hpp:43,59), a free carrying its extent's allocation tag
    (memory_pool.hpp:96; a RELEASE event may name another tag,
    simulator.hpp:456,519), and the measured timestamps. Equal to the planned
    trace (simulate_with_trace) in every column except time."""
    rows, cur, hw, live = [], 0, 0, {}
    for e in r.events:
        if e.kind == V.EventKind.Alloc:
            need = (e.bytes + alignment - 1) // alignment * alignment
            cur += need
            hw = max(hw, cur)
            live[e.offset] = (need, e.tag)
            rows.append((e.start, "a", e.tag, e.offset, need, cur, hw))
        elif e.kind == V.EventKind.Release:
            need, tag = live.pop(e.offset)
            cur -= need
            rows.append((e.start, "f", tag, e.offset, need, cur, hw))
    return rows


def write_artifacts(out_dir: str, g: V.NetworkGraph, d: V.PolicyDecision, measured: V.RunReport,
                    passes: List = None) -> Dict[str, str]:
    """The reference's artefacts (report.hpp:44-236) for a measured B200 step:
    graph.json, decision.json, report.json (events with tag / buffer / offset),
    timeline.csv, pool_trace.csv and, for vDNN_dyn, profile_passes.csv."""
    import os
    os.makedirs(out_dir, exist_ok=True)
    files = {
        "graph.json": dumps(graph_to_json(g)),
        "decision.json": dumps(decision_to_json(d)),
        "report.json": dumps(report_to_json(measured)),
        "timeline.csv": events_csv(measured),
        "pool_trace.csv": pool_trace_csv(pool_trace_from_report(measured)),
    }
    if passes:
        files["profile_passes.csv"] = profile_passes_csv(passes)
    for name, text in files.items():
        with open(os.path.join(out_dir, name), "w") as f:
            f.write(text)
    return {k: os.path.join(out_dir, k) for k in files}


def dumps(obj) -> str:
    return json.dumps(obj, separators=(",", ":"))
