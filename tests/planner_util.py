"""Helpers shared by the planner parity tests (spec parsing, comparisons)."""
from __future__ import annotations

import paper_1602_08124_b200 as V

KIND = {"input": 0, "conv": 1, "actv": 2, "pool": 3, "fc": 4, "loss": 5}


def graph_from_spec(spec: str) -> V.NetworkGraph:
    parts = spec.split("|")
    g = V.NetworkGraph(int(parts[0][2:]))
    for p in parts[1:]:
        kind, ins, p0, p1, p2, p3, join = p.split()
        inputs = [] if ins == "-" else [int(x) for x in ins.split(",")]
        p0, p1, p2, p3, join = int(p0), int(p1), int(p2), int(p3), V.JoinRule(int(join))
        if kind == "input":
            g.add_input(p0, p1, p2)
        elif kind == "conv":
            g.add_conv(inputs, p3, p0, p1, p2, join)
        elif kind == "actv":
            g.add_actv(inputs[0])
        elif kind == "pool":
            g.add_pool(inputs, p0, p1, join)
        elif kind == "fc":
            g.add_fc(inputs, p0, join)
        elif kind == "loss":
            g.add_loss(inputs[0])
    return g.finalize()


def cost_from_spec(spec: str) -> V.CostModel:
    cm = V.CostModel()
    if not spec:
        return cm
    halves = spec.split(";")
    m = {"pf": "peak_flops", "bw": "dram_bw", "cap": "mem_capacity", "eff": "compute_efficiency",
         "lbw": "link_effective_bw", "lnom": "link_nominal_bw", "lov": "link_fixed_launch_overhead",
         "es": "elem_size", "ratio": "bwd_fwd_ratio", "sfi": "speed_factor_implicit_gemm",
         "sfg": "speed_factor_gemm_ws", "sff": "speed_factor_fft"}
    for kv in halves[0].split(","):
        k, v = kv.split("=")
        setattr(cm, m[k], int(v) if k in ("cap", "es") else float(v))
    if len(halves) > 1 and halves[1].startswith("ov="):
        for t in halves[1][3:].split(","):
            i, f, b = t.split(":")
            cm.latency_overrides[int(i)] = (float(f), float(b))
    return cm


def decision_for(spec: str, g: V.NetworkGraph, cm: V.CostModel, capacity: int):
    """Returns (decision or None, capacity actually simulated, dyn passes or None)."""
    if spec.startswith("static:"):
        _, k, m = spec.split(":")
        kind = {"baseline": V.PolicyKind.Baseline, "all": V.PolicyKind.VdnnAll, "conv": V.PolicyKind.VdnnConv}[k]
        mode = V.AlgoMode.MemoryOptimal if m == "m" else V.AlgoMode.PerfOptimal
        return V.static_decision(kind, mode, g, cm), capacity, None
    if spec == "dyn":
        sel = V.dynamic_select(g, capacity, cm)
        return sel.decision, capacity, sel.passes
    if spec == "oracle":
        d = V.static_decision(V.PolicyKind.Baseline, V.AlgoMode.PerfOptimal, g, cm)
        d.label = "oracle"
        return d, V.KUNLIMITED_BYTES, None
    if spec.startswith("greedy:"):
        kind = V.PolicyKind.VdnnConv if spec.endswith("conv") else V.PolicyKind.VdnnAll
        return V.greedy_downgrade(g, capacity, kind, cm), capacity, None
    raise ValueError(spec)


def decision_json(d: V.PolicyDecision) -> dict:
    return {"label": d.label, "scheme": int(d.gradient_scheme),
            "offload": [i for i, f in enumerate(d.offload) if f],
            "algos": {str(i): int(a) for i, a in sorted(d.algos.items())}}


def report_json(r: V.RunReport, layers: int, events: bool = True) -> dict:
    fp, bp = r.layer_peaks(layers)
    out = {
        "verdict": r.verdict(), "pass": int(r.pass_),
        "oom": None if r.oom is None else {"layer": r.oom.layer, "phase": int(r.oom.phase),
                                           "fragmented": int(r.oom.fragmented), "requested": r.oom.requested,
                                           "tag": r.oom.tag},
        "max_mem_bytes": r.max_mem_bytes, "avg_mem_bytes": r.avg_mem_bytes,
        "offload_traffic_bytes": r.offload_traffic_bytes, "prefetch_traffic_bytes": r.prefetch_traffic_bytes,
        "host_peak_bytes": r.host_peak_bytes, "stall_fwd_offload_ns": r.stall_fwd_offload_ns,
        "stall_bwd_prefetch_ns": r.stall_bwd_prefetch_ns, "total_ns": r.total_ns, "n_events": len(r.events),
        "signature": r.signature(), "reuse_distance_ns": r.reuse_distance_ns, "fwd_peak": fp, "bwd_peak": bp,
    }
    if events:
        out["events"] = [[int(e.stream), int(e.kind), e.layer, e.start, e.end, e.bytes, e.tag, e.buffer, e.offset]
                         for e in r.events]
    return out


def compare_case(spec_graph: str, case: dict, cost_spec: str = "") -> None:
    g = graph_from_spec(spec_graph)
    cm = cost_from_spec(cost_spec)
    ref = case["result"]
    d, cap, passes = decision_for(case["decision_spec"], g, cm, case["capacity"])
    assert bool(ref["untrainable"]) == (d is None), case["decision_spec"]
    if ref.get("passes") is not None:
        assert passes is not None
        got = [{"phase": p.phase, "label": p.decision.label, "pass": int(p.pass_), "total_ns": p.total_ns,
                "max_mem_bytes": p.max_mem_bytes, "decision": decision_json(p.decision)} for p in passes]
        want = [{k: p[k] for k in ("phase", "label", "pass", "total_ns", "max_mem_bytes", "decision")}
                for p in ref["passes"]]
        assert got == want
    if d is None:
        return
    assert decision_json(d) == ref["decision"]
    r = V.simulate(g, d, cm, cap)
    want = ref["report"]
    got = report_json(r, g.size(), events="events" in want)
    want = {k: v for k, v in want.items() if k != "violations"}
    assert got.keys() == want.keys()
    for k in want:
        assert got[k] == want[k], f"{case['decision_spec']} @ {case['capacity']}: field {k} differs"
    assert [v.kind for v in V.replay_check(r, g, d, cap)] == ref["report"]["violations"]


def vocab_spec(rng) -> str:
    """A random graph over the reference's whole vocabulary (net_graph.hpp:83,
    281-321): elementwise joins of ReLU branches (read-only shared gradient
    maps), concat joins, strided convs (exact divisibility), overlapping and
    non-overlapping pools, two INPUT layers, an auxiliary LOSS head, an FC over
    an elementwise join. Spec format of graph_from_spec."""
    batch = 2 + rng.randrange(3)
    h = rng.choice([9, 12, 15, 16])
    layers, shape = [], {}

    def add(s, sh=None):
        layers.append(s)
        shape[len(layers) - 1] = sh
        return len(layers) - 1

    c0 = rng.choice([3, 4, 8])
    inputs = [add(f"input - {c0} {h} {h} 0 0", (c0, h, h))]
    if rng.randrange(2):  # a second INPUT layer, concatenated with the first
        c1 = rng.choice([1, 4])
        inputs.append(add(f"input - {c1} {h} {h} 0 0", (c1, h, h)))
    c = rng.choice([8, 16, 32])
    prev = add(f"conv {','.join(map(str, inputs))} 3 1 1 {c} 0", (c, h, h))
    prev = add(f"actv {prev} 0 0 0 0 0", shape[prev])
    aux_done = False
    for _ in range(4 + rng.randrange(3)):
        c, hh, _w = shape[prev]
        r = rng.randrange(6)
        if r == 0:  # elementwise join of two branches, at least one a ReLU chain
            oc = rng.choice([4, 8, 32])
            a = add(f"conv {prev} 3 1 1 {oc} 0", (oc, hh, hh))
            a = add(f"actv {a} 0 0 0 0 0", shape[a])
            b = add(f"conv {prev} 1 1 0 {oc} 0", (oc, hh, hh))
            if rng.randrange(2):
                b = add(f"actv {b} 0 0 0 0 0", shape[b])
            k, oc2 = rng.choice([1, 3]), rng.choice([8, 16])
            prev = add(f"conv {a},{b} {k} 1 {k // 2} {oc2} 1", (oc2, hh, hh))
        elif r == 1 and hh >= 5:  # strided conv: (h + 2p - k) divisible by the stride
            k, p = rng.choice([(3, 1), (1, 0)]) if hh % 2 else rng.choice([(2, 0), (4, 1)])
            oc = rng.choice([8, 16, 32])
            ho = (hh + 2 * p - k) // 2 + 1
            prev = add(f"conv {prev} {k} 2 {p} {oc} 0", (oc, ho, ho))
            prev = add(f"actv {prev} 0 0 0 0 0", shape[prev])
        elif r == 2 and hh >= 4:
            win = rng.choice([2, 3])
            ho = (hh - win) // 2 + 1
            prev = add(f"pool {prev} {win} 2 0 0 0", (c, ho, ho))
        elif r == 3:  # concat fork/join
            oa = rng.choice([4, 8])
            a = add(f"conv {prev} 1 1 0 {oa} 0", (oa, hh, hh))
            b = add(f"actv {prev} 0 0 0 0 0", shape[prev])
            oc = rng.choice([8, 16])
            prev = add(f"conv {a},{b} 3 1 1 {oc} 0", (oc, hh, hh))
        elif r == 4 and not aux_done:  # auxiliary LOSS head
            f = add(f"fc {prev} {rng.choice([5, 10])} 0 0 0 0")
            add(f"loss {f} 0 0 0 0 0")
            aux_done = True
        else:
            oc = rng.choice([8, 16, 32, 64])
            prev = add(f"conv {prev} 3 1 1 {oc} 0", (oc, hh, hh))
            prev = add(f"actv {prev} 0 0 0 0 0", shape[prev])
    if rng.randrange(2):  # classifier over an elementwise join of two FC branches
        a = add(f"fc {prev} 16 0 0 0 0")
        a = add(f"actv {a} 0 0 0 0 0")
        b = add(f"fc {prev} 16 0 0 0 0")
        prev = add(f"fc {a},{b} 10 0 0 0 1")
    else:
        prev = add(f"fc {prev} 10 0 0 0 0")
    add(f"loss {prev} 0 0 0 0 0")
    return f"B={batch}|" + "|".join(layers)
