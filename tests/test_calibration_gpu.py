"""SURVEY §8(f)1-2 on hardware: the calibrated cost model and the
reference's artefact formats from a measured B200 step.

* calibrated cost model: every layer's planner latency pinned to its measured
  B200 time (CostModel.latency_overrides, cost_model.hpp:74-75,143-145) and the
  link to the measured host bandwidth. Schedules and decisions are
  timing-independent, so the re-plan keeps the signature and the dyn decision
  bit for bit, while the planned step time now tracks the measured one;
* artefacts (report.hpp:44-236) written for the measured step: report.json
  with every event's tag / buffer / offset, timeline.csv, pool_trace.csv,
  decision.json, graph.json, profile_passes.csv -- and read back: the
  reference's own replay_check (compiled, oracle/_ref) accepts the measured
  log, and the measured pool trace equals the planned one in every column
  but time.
"""
import json
import os

import numpy as np
import pytest

torch = pytest.importorskip("torch")

import paper_1602_08124_b200 as V
from paper_1602_08124_b200 import formats as F
from oracle import refsim

pytestmark = pytest.mark.gpu
CAP = 12884901888


def _need_gpu():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


def _measure(g, d, cm, steps=3):
    s = V.Session(g, d, cm, CAP, record_timeline=True)
    s.synthetic_batch(5)
    for _ in range(steps):
        s.step(0.01, want_loss=False)
    s.step(0.01)
    return s, s.measured_report()


def _link_gbs(m):
    """Measured host-link bandwidth of the step: planned bytes over the
    measured OFFLOAD / PREFETCH durations (both directions together)."""
    by = sum(e.bytes for e in m.events if e.kind in (V.EventKind.Offload, V.EventKind.Prefetch))
    ns = sum(e.end - e.start for e in m.events if e.kind in (V.EventKind.Offload, V.EventKind.Prefetch))
    return by / ns if ns else None


@pytest.mark.parametrize("es", [4, 2], ids=["fp32", "bf16"])
def test_vgg16_b256_dyn_calibrated_replan_tracks_the_measured_step(es, tmp_path):
    _need_gpu()
    g = V.build_preset("vgg16", 256)
    cm = V.CostModel()
    cm.elem_size = es
    sel = V.dynamic_select(g, CAP, cm)
    d = sel.decision
    s, m = _measure(g, d, cm)
    plan = s.plan
    gbs = _link_gbs(m)
    cal = F.calibrated_cost_model(s, link_gbs=gbs)
    # the default model plans for a Titan X + PCIe 3 (cost_model.hpp:15-30)
    r = V.simulate(g, d, cal, CAP)
    assert r.signature() == plan.signature()
    assert V.placements(r) == V.placements(plan)
    sel2 = V.dynamic_select(g, CAP, cal)
    assert sel2.decision.label == d.label
    assert sel2.decision.spec() == d.spec()
    err = abs(r.total_ns - m.total_ns) / m.total_ns
    err_default = abs(plan.total_ns - m.total_ns) / m.total_ns
    print(f"es={es} {d.label}: measured {m.total_ns / 1e6:.2f} ms, calibrated plan {r.total_ns / 1e6:.2f} ms "
          f"({err:.3%}), default model {plan.total_ns / 1e6:.2f} ms ({err_default:.1%}), link {gbs:.2f} GB/s")
    assert err <= 0.05
    # stall predictions: the calibrated plan's exposed transfer vs the measured SYNC stalls
    assert abs(r.stall_ns() - m.stall_ns()) <= 0.05 * m.total_ns
    # artefacts of the measured step, read back
    files = F.write_artifacts(str(tmp_path), g, d, m, sel.passes)
    rep = json.load(open(files["report.json"]))
    assert rep["verdict"] == "PASS" and len(rep["events"]) == len(m.events)
    assert [e.get("offset") for e in rep["events"] if e["kind"] != "SYNC"] == \
        [F._event_json(e).get("offset") for e in plan.events if e.kind != V.EventKind.Sync]
    rows = open(files["pool_trace.csv"]).read().splitlines()[1:]
    _, planned_trace = V.simulate_with_trace(g, d, cm, CAP)
    assert [r_.split(",")[1:] for r_ in rows] == [
        ["alloc" if t[1] == "a" else "free"] + [str(x) for x in t[2:]] for t in planned_trace]
    assert len(open(files["timeline.csv"]).read().splitlines()) == len(m.events) + 1
    d2 = F.decision_from_json(json.load(open(files["decision.json"])), g)
    assert d2.spec() == d.spec()
    if refsim.available():
        ev = [(int(e.stream), int(e.kind), e.layer, e.start, e.end, e.bytes, e.tag, e.buffer, e.offset)
              for e in m.events]
        assert refsim.replay(g.spec(), d.spec(), CAP, ev, m.max_mem_bytes, m.avg_mem_bytes, m.total_ns, True) == []
