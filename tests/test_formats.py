"""Reference artefact formats (report.hpp) from our planner: JSON round trips,
CSV schemas, and calibrated cost models that keep schedules bit-identical."""
import json
import os

import pytest

import paper_1602_08124_b200 as V
from paper_1602_08124_b200 import formats as F
from oracle import refsim
from planner_util import graph_from_spec

GIB12 = 12884901888


def test_graph_json_round_trip():  # test_config_report.cpp:124-152
    for name, b in (("alexnet", 8), ("inception_toy", 4), ("vgg16", 2)):
        g = V.build_preset(name, b)
        j = F.graph_to_json(g)
        g2 = F.graph_from_json(json.loads(json.dumps(j)))
        assert F.graph_to_json(g2) == j
        assert g2.spec() == g.spec()


def test_decision_json_round_trip():
    g = V.build_preset("vgg16", 256)
    sel = V.dynamic_select(g, GIB12, V.CostModel())
    j = F.decision_to_json(sel.decision)
    assert j["label"] == "vdnn-conv+greedy" and j["gradient_scheme"] == "per_layer"
    d2 = F.decision_from_json(json.loads(json.dumps(j)), g)
    assert d2 == sel.decision


def test_csv_schemas():  # test_config_report.cpp:154-197
    g = V.build_preset("alexnet", 8)
    d = V.static_decision(V.PolicyKind.VdnnAll, V.AlgoMode.MemoryOptimal, g, V.CostModel())
    r, trace = V.simulate_with_trace(g, d, V.CostModel(), GIB12)
    csv = F.events_csv(r).splitlines()
    assert csv[0] == "stream,kind,layer,start_ns,end_ns,bytes" and len(csv) == len(r.events) + 1
    assert F.pool_trace_csv(trace).splitlines()[0] == "time_ns,op,tag,offset,bytes,current,high_water"
    sel = V.dynamic_select(g, GIB12, V.CostModel())
    assert F.profile_passes_csv(sel.passes).splitlines()[0] == "phase,decision,verdict,total_ns,max_mem_bytes"
    j = F.report_to_json(r)
    assert j["verdict"] == "PASS" and len(j["events"]) == len(r.events)
    assert all("offset" in e for e in j["events"] if e["kind"] in ("ALLOC", "RELEASE"))


def test_latency_overrides_never_change_schedules():
    """SURVEY key finding 1: any cost model gives the same event sequence and
    offsets -- the basis of the calibrated-plan feature."""
    g = V.build_preset("vgg16", 32)
    cm = V.CostModel()
    d = V.static_decision(V.PolicyKind.VdnnAll, V.AlgoMode.MemoryOptimal, g, cm)
    base = V.simulate(g, d, cm, GIB12)
    fast = V.CostModel(peak_flops=2.25e15, dram_bw=8e12, link_effective_bw=55e9, link_nominal_bw=64e9,
                       latency_overrides={i: (1e-4 * (i % 7 + 1), 2e-4) for i in range(1, g.size())})
    r = V.simulate(g, d, fast, GIB12)
    assert r.signature() == base.signature() and r.total_ns != base.total_ns
    if refsim.available():
        ref = refsim.run(g.spec(), "static:all:m", GIB12, cost_spec=fast.spec(), events=False)["report"]
        assert ref["signature"] == r.signature() and ref["total_ns"] == r.total_ns


ART = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "profiles", "r02_artifacts")


@pytest.mark.parametrize("run", ["vgg16_b256_dyn", "vgg16_b256_dynb"])
def test_committed_measured_artifacts_replay_clean(run):
    """The artefact files of a measured B200 step (bench.py --artifacts,
    report.hpp:44-236 formats) are consumed as the reference's own tools
    would: graph and decision JSON round-trip into our API, the measured
    event log passes our replay_check and the compiled reference's, and the
    measured pool trace equals the planned one in every column but time."""
    import json
    import paper_1602_08124_b200 as V
    from paper_1602_08124_b200 import formats as F
    from oracle import refsim
    d = os.path.join(ART, run)
    g = F.graph_from_json(json.load(open(os.path.join(d, "graph.json"))))
    dec = F.decision_from_json(json.load(open(os.path.join(d, "decision.json"))), g)
    cal = json.load(open(os.path.join(d, "calibration.json")))
    cm = V.CostModel()
    cm.elem_size = cal["elem_size"]
    plan, trace = V.simulate_with_trace(g, dec, cm, cal["capacity"])
    assert plan.signature() == cal["signature_planned"] == cal["signature_calibrated"]
    rep = json.load(open(os.path.join(d, "report.json")))
    kinds = {"FWD": 0, "BWD": 1, "OFFLOAD": 2, "PREFETCH": 3, "ALLOC": 4, "RELEASE": 5, "SYNC": 6}
    ev = [(0 if e["stream"] == "compute" else 1, kinds[e["kind"]], e["layer"], e["start_ns"], e["end_ns"], e["bytes"],
           e.get("tag", ""), e.get("buffer", -1), e.get("offset", 0)) for e in rep["events"]]
    assert [x for x in ev if x[1] != 6 and x[1] in (4, 5)] != []
    placed = [(k, l, b, t, by, o) for (_, k, l, _, _, by, t, b, o) in ev if k != 6]
    assert placed == [tuple(p) for p in V.placements(plan)]
    assert abs(cal["calibrated_rel_err"]) < 0.05
    rows = open(os.path.join(d, "pool_trace.csv")).read().splitlines()[1:]
    assert [r.split(",")[1:] for r in rows] == [["alloc" if t[1] == "a" else "free"] + [str(x) for x in t[2:]]
                                                for t in trace]
    if refsim.available():
        out = refsim.replay(g.spec(), dec.spec(), cal["capacity"], ev, rep["max_mem_bytes"], rep["avg_mem_bytes"],
                            rep["total_ns"], True)
        assert out == [], out[:5]
