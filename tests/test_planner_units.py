"""The reference's unit tests restated against our planner (CPU only).

Each test cites the reference test it mirrors (/root/reference/proj/tests/).
"""
import pytest

import paper_1602_08124_b200 as V
from planner_util import graph_from_spec

cm0 = V.CostModel()
GIB12 = 12884901888


def single_conv(stride=1):  # test_cost_model.cpp:7-17
    g = V.NetworkGraph(64)
    i = g.add_input(64, 224, 224)
    if stride == 1:
        g.add_conv([i], 64, 3, 1, 1)
    else:
        g.add_conv([i], 64, 4, 2, 0)
    return g.finalize()


def small_linear(batch=2):  # test_simulator.cpp:27-37
    g = V.NetworkGraph(batch)
    p = g.add_input(4, 16, 16)
    p = g.add_conv([p], 8, 3, 1, 1)
    p = g.add_actv(p)
    p = g.add_pool([p], 2, 2)
    p = g.add_fc([p], 64)
    g.add_loss(p)
    return g.finalize()


# ----------------------------------------------------------- net_graph --
def test_shapes_conv_pool_fc():  # test_net_graph.cpp:24-97
    g = V.build_preset("alexnet", 128)
    assert g.shape(1) == V.TensorShape(128, 64, 55, 55)
    assert g.shape(3) == V.TensorShape(128, 64, 27, 27)
    assert g.shape(13) == V.TensorShape(128, 256, 6, 6)
    assert g.shape(14) == V.TensorShape(128, 4096, 1, 1)
    assert g.shape(17) == V.TensorShape(128, 1, 1, 1)


def test_preset_layer_counts():  # test_net_graph.cpp:131-172
    assert V.build_preset("alexnet", 1).size() == 18
    assert V.build_preset("overfeat", 1).size() == 20
    assert V.build_preset("inception_toy", 1).size() == 14
    g = V.build_preset("vgg16", 1)
    assert g.size() == 44 and g.count_kind(V.LayerKind.Conv) == 16 and g.count_kind(V.LayerKind.Pool) == 5
    assert g.count_kind(V.LayerKind.Fc) == 3


def test_vgg_deepening():  # test_net_graph.cpp:174-211
    g = V.extend_vgg(400, 32)
    assert g.count_kind(V.LayerKind.Conv) == 416
    assert g.size() == 844
    with pytest.raises(V.InvalidDepth):
        V.extend_vgg(150, 32)
    with pytest.raises(V.InvalidDepth):
        V.extend_vgg(-100, 32)


def test_unknown_preset_and_bad_batch():
    with pytest.raises(V.UnknownPreset):
        V.build_preset("googlenet", 8)
    with pytest.raises(V.VdnnError):
        V.build_preset("vgg16", 0)


def test_refcounts_and_consumers():  # test_net_graph.cpp:99-129
    g = V.build_preset("inception_toy", 2)
    assert g.refcnt(2) == 3  # the fork activation feeds three branches
    assert g.refcnt(0) == 1
    assert g.refcnt(13) == 0


def test_shape_errors():  # test_net_graph.cpp (validation)
    g = V.NetworkGraph(1)
    i = g.add_input(3, 10, 10)
    g.add_conv([i], 4, 3, 2, 0)  # (10 - 3) % 2 != 0
    with pytest.raises(V.ShapeMismatch):
        g.finalize()
    g = V.NetworkGraph(1)
    a = g.add_input(3, 8, 8)
    b = g.add_pool([a], 2, 2)
    g.add_conv([a, b], 4, 1, 1, 0)  # concat of 8x8 and 4x4
    with pytest.raises(V.ShapeMismatch):
        g.finalize()
    g = V.NetworkGraph(1)
    a = g.add_input(3, 8, 8)
    g.add_conv([], 4, 1, 1, 0)
    with pytest.raises(V.VdnnError):
        g.finalize()


def test_concat_channels_sum():
    g = V.build_preset("inception_toy", 2)
    assert g.shape(9) == V.TensorShape(2, 64, 32, 32)
    assert V.CostModel().weight_bytes(g, 9) == 3 * 3 * (32 + 32 + 16) * 64 * 4


# ---------------------------------------------------------- cost model --
def test_conv_latency_hand_value():  # test_cost_model.cpp:19-27
    g = single_conv()
    t = cm0.layer_latency(g, 1, False, V.AlgoId.ImplicitGemm)
    assert abs(t - 236760072192.0 / 3.5e12) < 1e-9
    assert abs(t - 0.06764573) < 1e-6


def test_speed_factors_exact():  # test_cost_model.cpp:29-35
    g = single_conv()
    base = cm0.layer_latency(g, 1, False, V.AlgoId.ImplicitGemm)
    assert cm0.layer_latency(g, 1, False, V.AlgoId.Fft) == 0.6 * base
    assert cm0.layer_latency(g, 1, False, V.AlgoId.GemmWs) == 0.8 * base


def test_backward_is_double_forward():  # test_cost_model.cpp:50-59
    g = V.build_preset("alexnet", 16)
    for l in g.layers():
        f = cm0.layer_latency(g, l.id, False, V.AlgoId.GemmWs)
        assert cm0.layer_latency(g, l.id, True, V.AlgoId.GemmWs) == 2.0 * f


def test_override_pins():  # test_cost_model.cpp:74-80
    g = single_conv()
    cm = V.CostModel(latency_overrides={1: (0.010, 0.025)})
    assert cm.layer_latency(g, 1, False, V.AlgoId.Fft) == 0.010
    assert cm.layer_latency(g, 1, True, V.AlgoId.Fft) == 0.025


def test_workspace_values():  # test_cost_model.cpp:82-105
    g = single_conv()
    assert cm0.conv_workspace(g, 1, V.AlgoId.ImplicitGemm) == 0
    assert cm0.conv_workspace(g, 1, V.AlgoId.Fft) == 2 * 64 * 256 * 256 * 64 * 4
    g2 = V.NetworkGraph(64)
    i = g2.add_input(3, 224, 224)
    g2.add_conv([i], 64, 3, 1, 1)
    g2.finalize()
    assert cm0.conv_workspace(g2, 1, V.AlgoId.GemmWs) == 346816512
    g3 = V.NetworkGraph(1)
    i = g3.add_input(1, 8, 8)
    g3.add_pool([i], 2, 2)
    g3.finalize()
    with pytest.raises(V.WrongLayerKind):
        cm0.conv_workspace(g3, 1, V.AlgoId.Fft)


def test_transfer_and_interference():  # test_cost_model.cpp:138-166
    assert abs(cm0.transfer_latency(822083584) - 0.06422528) < 1e-9
    assert cm0.transfer_latency(0) == 0.0
    page = V.CostModel(link_effective_bw=200e6, link_nominal_bw=200e6)
    assert abs(page.transfer_latency(4096) - 20.48e-6) < 1e-9
    assert abs(cm0.offload_interference_bound() - 16.0 / 336.0) < 1e-12


def test_fft_forbidden_for_stride():  # test_cost_model.cpp:168-175
    g = single_conv(stride=2)
    assert not cm0.fft_applicable(g, 1)
    assert cm0.fastest_algo(g, 1) == V.AlgoId.GemmWs
    assert cm0.fastest_algo(single_conv(), 1) == V.AlgoId.Fft


# ----------------------------------------------------------- footprint --
def test_footprint_hand_values():  # test_footprint.cpp:28-69
    assert V.CostModel().tensor_bytes_of(V.TensorShape(256, 64, 112, 112)) == 822083584
    g = V.build_preset("vgg16", 256)
    d = V.static_decision(V.PolicyKind.Baseline, V.AlgoMode.PerfOptimal, g, cm0)
    fp = V.baseline_footprint(g, d.algos, cm0)
    assert (fp.weights_bytes, fp.feature_maps_bytes, fp.gradient_buffers_bytes, fp.workspace_bytes,
            fp.total_bytes) == (574646944, 16938172416, 6576668672, 8589934592, 32679422624)
    assert 21e9 < fp.total_bytes < 35e9
    a = V.build_preset("alexnet", 128)
    da = V.static_decision(V.PolicyKind.Baseline, V.AlgoMode.PerfOptimal, a, cm0)
    assert 0.825e9 < V.baseline_footprint(a, da.algos, cm0).total_bytes < 1.375e9


def test_gradient_map_rules():  # footprint.hpp:60-71
    g = V.build_preset("alexnet", 2)
    assert V.gradient_map_bytes(g, 1, cm0) == 0       # conv on raw input
    assert V.gradient_map_bytes(g, 2, cm0) == 0       # ACTV owns none
    assert V.gradient_map_bytes(g, 4, cm0) == cm0.tensor_bytes_of(g.shape(3))
    t = V.build_preset("inception_toy", 2)
    assert V.gradient_map_bytes(t, 9, cm0) == sum(cm0.tensor_bytes_of(t.shape(q)) for q in (4, 6, 8))


# ------------------------------------------------------------ decisions --
def test_static_flags():  # test_policy.cpp:13-59
    g = V.build_preset("vgg16", 8)
    d = V.static_decision(V.PolicyKind.VdnnAll, V.AlgoMode.MemoryOptimal, g, cm0)
    for l in g.layers():
        assert d.offloads(l.id) == (l.kind in (V.LayerKind.Conv, V.LayerKind.Pool, V.LayerKind.Input))
    assert d.gradient_scheme == V.GradientScheme.PerLayer and d.label == "vdnn-all(m)"
    d = V.static_decision(V.PolicyKind.VdnnConv, V.AlgoMode.PerfOptimal, g, cm0)
    assert sum(d.offload) == 16 and d.label == "vdnn-conv(p)"
    a = V.build_preset("alexnet", 8)
    d = V.static_decision(V.PolicyKind.Baseline, V.AlgoMode.PerfOptimal, a, cm0)
    assert d.gradient_scheme == V.GradientScheme.TwoBufferReuse
    assert d.algos[1] == V.AlgoId.GemmWs and d.algos[4] == V.AlgoId.Fft


def test_invalid_decisions_rejected():  # test_simulator.cpp:286-292, decision.hpp:38-56
    g = small_linear()
    d = V.static_decision(V.PolicyKind.VdnnAll, V.AlgoMode.MemoryOptimal, g, cm0)
    d.offload[2] = 1  # ACTV
    with pytest.raises(V.InvalidDecision):
        V.simulate(g, d, cm0, V.KUNLIMITED_BYTES)
    d = V.static_decision(V.PolicyKind.Baseline, V.AlgoMode.MemoryOptimal, g, cm0)
    d.offload[1] = 1  # offload under two-buffer reuse
    with pytest.raises(V.InvalidDecision):
        V.simulate(g, d, cm0, V.KUNLIMITED_BYTES)
    d = V.static_decision(V.PolicyKind.VdnnAll, V.AlgoMode.MemoryOptimal, g, cm0)
    del d.algos[1]
    with pytest.raises(V.InvalidDecision):
        V.simulate(g, d, cm0, V.KUNLIMITED_BYTES)


# ----------------------------------------------------------- simulator --
def test_no_offload_total_is_sum_of_latencies():  # test_simulator.cpp:39-54
    g = small_linear()
    d = V.static_decision(V.PolicyKind.Baseline, V.AlgoMode.MemoryOptimal, g, cm0)
    r = V.simulate(g, d, cm0, V.KUNLIMITED_BYTES)
    assert r.pass_
    expect = 0
    for l in g.layers():
        expect += round(cm0.layer_latency(g, l.id, False) * 1e9) + round(cm0.layer_latency(g, l.id, True) * 1e9)
    assert r.total_ns == expect and r.stall_ns() == 0 and r.offload_traffic_bytes == 0


def test_baseline_peak_manual_enumeration():  # test_simulator.cpp:68-88
    g = small_linear()
    d = V.static_decision(V.PolicyKind.Baseline, V.AlgoMode.MemoryOptimal, g, cm0)
    r = V.simulate(g, d, cm0, V.KUNLIMITED_BYTES)

    def a(b):
        return (b + 511) // 512 * 512
    expect = (a(9 * 4 * 8 * 4) + a((8 * 8 * 8 + 1) * 64 * 4) + a(2 * 4 * 16 * 16 * 4) + a(2 * 8 * 16 * 16 * 4)
              + a(2 * 8 * 8 * 8 * 4) + a(2 * 64 * 4) + 2 * a(2 * 8 * 16 * 16 * 4))
    assert r.max_mem_bytes == expect
    assert r.max_mem_bytes == r.avg_mem_bytes


def test_fig8_offload_sync_exact_ns():  # test_simulator.cpp:93-133
    g = V.NetworkGraph(1)
    i = g.add_input(5, 1000, 1000)
    c1 = g.add_conv([i], 20, 1, 1, 0)
    c2 = g.add_conv([c1], 1, 1, 1, 0)
    c3 = g.add_conv([c2], 1, 1, 1, 0)
    g.add_loss(c3)
    g.finalize()
    cm = V.CostModel(link_effective_bw=4e9, latency_overrides={c1: (0.01, 0.01), c2: (0.01, 0.01),
                                                                c3: (0.01, 0.01)})
    d = V.static_decision(V.PolicyKind.VdnnAll, V.AlgoMode.MemoryOptimal, g, cm)
    r = V.simulate(g, d, cm, V.KUNLIMITED_BYTES)
    fwd = {e.layer: e for e in r.events if e.kind == V.EventKind.Fwd}
    off = {e.layer: e for e in r.events if e.kind == V.EventKind.Offload}
    ms = 1_000_000
    assert (fwd[c1].start, fwd[c1].end, off[c1].start, off[c1].end) == (0, 10 * ms, 0, 5 * ms)
    assert fwd[c2].start == 10 * ms and (off[c2].start, off[c2].end) == (10 * ms, 30 * ms)
    assert fwd[c3].start == 30 * ms and r.stall_fwd_offload_ns == 10 * ms
    assert V.replay_check(r, g, d, V.KUNLIMITED_BYTES) == []


def test_sync_rule_exactness_alexnet():  # test_simulator.cpp:160-182
    g = V.build_preset("alexnet", 16)
    d = V.static_decision(V.PolicyKind.VdnnAll, V.AlgoMode.PerfOptimal, g, cm0)
    r = V.simulate(g, d, cm0, V.KUNLIMITED_BYTES)
    fwds = [e for e in r.events if e.kind == V.EventKind.Fwd]
    last_off = {}
    for e in r.events:
        if e.kind == V.EventKind.Offload:
            last_off[e.layer] = max(last_off.get(e.layer, 0), e.end)
    for a, b in zip(fwds, fwds[1:]):
        assert b.start == max(a.end, last_off.get(a.layer, a.end))


def test_prefetch_conservation_and_replay():  # test_simulator.cpp:184-203
    for name in ("alexnet", "inception_toy"):
        g = V.build_preset(name, 8)
        for k in (V.PolicyKind.VdnnAll, V.PolicyKind.VdnnConv):
            d = V.static_decision(k, V.AlgoMode.MemoryOptimal, g, cm0)
            r = V.simulate(g, d, cm0, V.KUNLIMITED_BYTES)
            assert r.pass_ and V.replay_check(r, g, d, V.KUNLIMITED_BYTES) == []
            off = {e.buffer for e in r.events if e.kind == V.EventKind.Offload}
            pre = {e.buffer for e in r.events if e.kind == V.EventKind.Prefetch}
            assert off == pre and r.offload_traffic_bytes == r.prefetch_traffic_bytes


def test_vgg16_b256_fits_titanx_and_baseline_ooms():  # test_simulator.cpp:228-249
    g = V.build_preset("vgg16", 256)
    d = V.static_decision(V.PolicyKind.VdnnAll, V.AlgoMode.MemoryOptimal, g, cm0)
    r = V.simulate(g, d, cm0, GIB12)
    assert r.pass_ and r.max_mem_bytes <= GIB12 and 12e9 < r.offload_traffic_bytes < 20e9
    b = V.static_decision(V.PolicyKind.Baseline, V.AlgoMode.PerfOptimal, g, cm0)
    r = V.simulate(g, b, cm0, GIB12)
    assert not r.pass_ and r.oom.phase == V.Phase.Setup and r.verdict().startswith("OOM(layer=13, phase=setup")


def test_oom_verdict_and_corrupt_log_detected():  # test_simulator.cpp:294-331
    g = small_linear()
    d = V.static_decision(V.PolicyKind.VdnnAll, V.AlgoMode.MemoryOptimal, g, cm0)
    r = V.simulate(g, d, cm0, 4096)
    assert not r.pass_ and "OOM" in r.verdict()
    r = V.simulate(g, d, cm0, V.KUNLIMITED_BYTES)
    ev = list(r.events)
    for e in ev:
        if e.kind == V.EventKind.Release and e.buffer == 0 and e.tag in ("X", "Y"):
            e.start = e.end = 0
            break
    bad = V.report_from_events(ev, {"pass_": 1, "max_mem_bytes": r.max_mem_bytes, "avg_mem_bytes": r.avg_mem_bytes,
                                    "total_ns": r.total_ns})
    assert V.replay_check(bad, g, d, V.KUNLIMITED_BYTES) != []
    assert V.replay_check(r, g, d, 1024) != []  # capacity breach


def test_pool_trace_matches_events_and_host_peak():  # test_simulator.cpp:333-372
    g = small_linear()
    d = V.static_decision(V.PolicyKind.VdnnAll, V.AlgoMode.MemoryOptimal, g, cm0)
    r, trace = V.simulate_with_trace(g, d, cm0, V.KUNLIMITED_BYTES)
    n_pool = sum(1 for e in r.events if e.kind in (V.EventKind.Alloc, V.EventKind.Release))
    assert len(trace) == n_pool and max(t[6] for t in trace) == r.max_mem_bytes
    g = V.build_preset("vgg16", 32)
    d = V.static_decision(V.PolicyKind.VdnnAll, V.AlgoMode.MemoryOptimal, g, cm0)
    r = V.simulate(g, d, cm0, GIB12)
    assert r.host_peak_bytes == r.offload_traffic_bytes


def test_weight_grad_option_both_schemes():  # test_simulator.cpp:350-363
    g = small_linear()
    for k in (V.PolicyKind.Baseline, V.PolicyKind.VdnnAll):
        d = V.static_decision(k, V.AlgoMode.MemoryOptimal, g, cm0)
        w = V.simulate(g, d, cm0, V.KUNLIMITED_BYTES, V.SimOptions(include_weight_grads=True))
        wo = V.simulate(g, d, cm0, V.KUNLIMITED_BYTES)
        assert w.pass_ and w.max_mem_bytes > wo.max_mem_bytes
        assert V.replay_check(w, g, d, V.KUNLIMITED_BYTES) == []


def test_reuse_distance_shrinks_with_depth():  # test_simulator.cpp:251-266
    g = V.build_preset("vgg16", 32)
    d = V.static_decision(V.PolicyKind.Baseline, V.AlgoMode.PerfOptimal, g, cm0)
    r = V.simulate(g, d, cm0, V.KUNLIMITED_BYTES)
    convs = [l.id for l in g.layers() if l.kind == V.LayerKind.Conv]
    rd = r.reuse_distance_ns
    assert rd[convs[0]] > rd[convs[-1]]


# --------------------------------------------------------------- policy --
def test_dyn_slack_gives_baseline_and_oracle_time():  # test_policy.cpp:301-314
    g = V.build_preset("vgg16", 16)
    sel = V.dynamic_select(g, GIB12, cm0)
    assert sel.decision.label == "baseline(p)" and not any(sel.decision.offload)
    run = V.simulate(g, sel.decision, cm0, GIB12)
    assert run.total_ns == V.simulate_oracle(g, cm0).total_ns
    assert sel.passes[0].phase == "P1" and sel.passes[0].pass_


def test_dyn_vgg16_b256_recovers_via_later_phase():  # test_policy.cpp:316-330
    g = V.build_preset("vgg16", 256)
    sel = V.dynamic_select(g, GIB12, cm0)
    assert V.simulate(g, sel.decision, cm0, GIB12).pass_
    assert any(p.decision.label == "baseline(p)" and not p.pass_ for p in sel.passes)
    assert sel.decision.label == "vdnn-conv+greedy"


def test_dyn_tiny_pool_untrainable():  # test_policy.cpp:332-340
    g = V.build_preset("alexnet", 64)
    sel = V.dynamic_select(g, 1 << 20, cm0)
    assert sel.untrainable() and len(sel.passes) == 1 and sel.passes[0].phase == "P1"


SHRINK = ("B=4|input - 8 16 16 0 0|conv 0 3 1 1 8 0|actv 1 0 0 0 0 0|pool 2 2 2 0 0 0|conv 3 3 1 1 8 0|"
          "actv 4 0 0 0 0 0|pool 5 2 2 0 0 0|conv 6 3 1 1 8 0|actv 7 0 0 0 0 0|fc 8 10 0 0 0 0|loss 9 0 0 0 0 0")


def test_greedy_feasibility_matches_exhaustive_enumeration():  # test_policy.cpp:236-283
    g = graph_from_spec(SHRINK)
    convs = [l.id for l in g.layers() if l.kind == V.LayerKind.Conv]
    algos = list(V.AlgoId)
    for kind in (V.PolicyKind.VdnnConv, V.PolicyKind.VdnnAll):
        peaks = []
        for a0 in algos:
            for a1 in algos:
                for a2 in algos:
                    d = V.static_decision(kind, V.AlgoMode.MemoryOptimal, g, cm0)
                    d.algos.update({convs[0]: a0, convs[1]: a1, convs[2]: a2})
                    peaks.append(V.simulate(g, d, cm0, V.KUNLIMITED_BYTES).max_mem_bytes)
        caps = sorted({c for p in peaks for c in (p, p - 512, p + 512)} | {1024, 1 << 40})
        for cap in caps:
            feasible = False
            for a0 in algos:
                for a1 in algos:
                    for a2 in algos:
                        d = V.static_decision(kind, V.AlgoMode.MemoryOptimal, g, cm0)
                        d.algos.update({convs[0]: a0, convs[1]: a1, convs[2]: a2})
                        if V.simulate(g, d, cm0, cap).pass_:
                            feasible = True
            assert (V.greedy_downgrade(g, cap, kind, cm0) is not None) == feasible, cap


def test_greedy_no_downgrade_with_ample_capacity():  # test_policy.cpp:174-182
    g = graph_from_spec(SHRINK)
    d = V.greedy_downgrade(g, 1 << 40, V.PolicyKind.VdnnConv, cm0)
    for l in g.layers():
        if l.kind == V.LayerKind.Conv:
            assert d.algos[l.id] == cm0.fastest_algo(g, l.id)
    assert d.label == "vdnn-conv+greedy"
