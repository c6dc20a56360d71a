"""BF16 feature storage (the reference's elem_size = 2; cost_model.hpp:69,
config.hpp:112) on the B200 executor.

The planner sizes every feature map, gradient map and weight at 2 bytes; the
executor stores them as bf16 and runs the kind::f16 engine (tcb_conv.cuh) and
the bf16 memory-bound kernels. Checks:

* every BASELINE config at full size under its policy, layer-local against
  float64 on the operands the kernels read (tests/layer_parity.py, BF16
  bounds: one round-to-nearest-even per stored value, 2^-8 relative; fp32
  gradient arena 5e-4);
* the schedule is the reference's at es=2 (tests/golden/es2.json), the
  measured log replays clean, and offloading moves bytes only: every policy
  gives bit-identical losses and weights;
* the reference's whole graph vocabulary (random graphs, INI, graph JSON)
  layer-locally under every policy.
"""
import gc
import hashlib
import random

import numpy as np
import pytest

torch = pytest.importorskip("torch")

import paper_1602_08124_b200 as V
from oracle import numeric
from planner_util import graph_from_spec, vocab_spec

import layer_parity as LP
import test_layer_parity_gpu as TL
import test_vocab_gpu as TV

pytestmark = pytest.mark.gpu
CAP = 12884901888


def _need_gpu():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


def _cm():
    cm = V.CostModel()
    cm.elem_size = 2
    return cm


def test_vgg16_b256_dyn_every_layer_bf16():
    """BASELINE config 4 in BF16: dyn settles on vdnn-conv(p) (5.32 GB each way)."""
    _, ops = TL._run("vgg16_b256", "vgg16", 256, "dyn", False, expect_label="vdnn-conv(p)", es=2)
    assert {"fprop", "dgrad", "wgrad", "pool_fwd", "pool_bwd"} <= ops


def test_alexnet_b128_vdnn_all_every_layer_bf16():
    TL._run("alexnet_b128", "alexnet", 128, "all", False, es=2)


def test_overfeat_b128_vdnn_conv_every_layer_bf16():
    TL._run("overfeat_b128", "overfeat", 128, "conv", False, es=2)


def test_inception_toy_b128_dyn_every_layer_bf16():
    recs, _ = TL._run("inception_toy_b128", "inception_toy", 128, "dyn", False, expect_label="baseline(p)", es=2)
    assert any(r["tensor"].startswith("DX") for r in recs)


def test_vgg416_b32_dyn_sampled_layers_bf16():
    g = V.extend_vgg(400, 32)
    L = numeric.layers_of(g)
    convs = [l.id for l in L if l.kind == numeric.CONV]
    pools = [l.id for l in L if l.kind == numeric.POOL]
    fcs = [l.id for l in L if l.kind == numeric.FC]
    pick = sorted(set(convs[:3] + convs[len(convs) // 2: len(convs) // 2 + 2] + convs[-2:] + pools + fcs
                      + [L[-1].id]))
    TL._run("vgg416_b32", "vgg16", 32, "dyn", False, layers=pick, extra=400, expect_label="vdnn-conv(p)", es=2)


def test_vgg16_b256_bf16_plan_and_policy_invariance():
    """Full size, es=2: the dyn schedule is the reference's (golden es2.json),
    the measured log keeps every planned offset and replays clean, and a step
    under dyn, vDNN_all(m) and no offload gives the same loss and weights bit
    for bit."""
    _need_gpu()
    import json
    import os
    g = V.build_preset("vgg16", 256)
    cm = _cm()
    gold = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "es2.json")))
    want = [c for c in gold if c["spec"].startswith("B=256") and c["decision_spec"] == "dyn"][0]["result"]
    d = V.dynamic_select(g, CAP, cm).decision
    assert d.label == "vdnn-conv(p)"

    def run(decision, capacity, **kw):
        s = V.Session(g, decision, cm, capacity, **kw)
        s.synthetic_batch(7)
        loss = s.step(0.01)
        h = hashlib.sha256()
        for l in g.layers():
            if l.kind in (V.LayerKind.Conv, V.LayerKind.Fc):
                h.update(np.ascontiguousarray(s.get_weights(l.id)).tobytes())
        return s, loss, h.hexdigest()

    s, loss_dyn, w_dyn = run(d, CAP, record_timeline=True)
    assert s.plan.signature() == want["report"]["signature"]
    m = s.measured_report()
    assert m.offload_traffic_bytes == s.plan.offload_traffic_bytes == 5317853184
    assert V.placements(m) == V.placements(s.plan)  # every non-SYNC row, planned offsets
    assert V.replay_check(m, g, d, CAP) == []
    st = s.transfer_stats()
    assert st["offload_planned"] == 5317853184
    del s, m
    gc.collect()
    da = V.static_decision(V.PolicyKind.VdnnAll, V.AlgoMode.MemoryOptimal, g, cm)
    s, loss_a, w_a = run(da, CAP)
    del s
    gc.collect()
    free, _ = torch.cuda.mem_get_info()
    db = V.static_decision(V.PolicyKind.Baseline, V.AlgoMode.PerfOptimal, g, cm)
    s, loss_b, w_b = run(db, int(free - (6 << 30)))
    del s
    gc.collect()
    assert np.isfinite(loss_dyn)
    assert loss_dyn == loss_a == loss_b
    assert w_dyn == w_a == w_b


def test_small_net_bf16_tracks_float64_end_to_end():
    """inception_toy b8, vDNN_all, one step: the bf16 loss within 2e-2 of the
    float64 oracle (bf16-rounded weights and images) -- end-to-end storage
    noise, not a kernel bound (the kernel bounds are layer-local above)."""
    _need_gpu()
    g = V.build_preset("inception_toy", 8)
    cm = _cm()
    d = V.static_decision(V.PolicyKind.VdnnAll, V.AlgoMode.MemoryOptimal, g, cm)
    w = numeric.he_weights(g, cm, seed=11)
    wb = {k: V.from_bf16_bits(V.to_bf16_bits(v)) for k, v in w.items()}
    rng = np.random.default_rng(12)
    images = V.from_bf16_bits(V.to_bf16_bits(rng.uniform(-1, 1, size=(8, 32, 32, 3)).astype(np.float32)))
    labels = rng.integers(0, 10, size=8).astype(np.int32)
    s = V.Session(g, d, cm, 64 << 20, external_grads=True)
    for k, v in w.items():
        s.set_weights(k, v)
        assert np.array_equal(s.get_weights(k), wb[k])  # upload rounds to nearest even
    s.set_batch(images, labels)
    loss = s.step(0.01)
    cl, _, _ = numeric.train_step(g, wb, images.reshape(8, 32, 32, 3), labels, 0.01)
    assert abs(loss - cl) <= 2e-2 * max(1.0, abs(cl)), (loss, cl)


@pytest.mark.parametrize("seed", range(3))
def test_random_full_vocabulary_graphs_bf16(seed):
    """Elementwise joins (rounded summed input), shared read-only gradient
    maps, concat joins, strided convs, two INPUTs, two LOSS heads, odd channel
    counts (element-wise gathers): layer-local under every policy."""
    _need_gpu()
    rng = random.Random(2000 + seed)
    cm = _cm()
    for t in range(3):
        spec = vocab_spec(rng)
        g = graph_from_spec(spec)
        ims, labels = TV._inputs_and_labels(g, seed * 10 + t)
        for d in TV._decisions(g, cm):
            TV.run_and_compare(g, d, cm, ims, labels, False, f"bf16 {spec} {d.label}")


def test_graph_json_network_bf16():
    """The GoogLeNet-like graph-JSON module (concat of 1x1/3x3/5x5/pool
    branches, residual elementwise join, two heads) in BF16, layer-local."""
    _need_gpu()
    g = TV.json_graph()
    cm = _cm()
    ims, labels = TV._inputs_and_labels(g, 6)
    for d in TV._decisions(g, cm):
        TV.run_and_compare(g, d, cm, ims, labels, False, f"bf16 json {d.label}")


def test_bf16_rejects_fp32_only_modes():
    _need_gpu()
    g = V.build_preset("inception_toy", 4)
    cm = _cm()
    d = V.static_decision(V.PolicyKind.VdnnAll, V.AlgoMode.MemoryOptimal, g, cm)
    with pytest.raises(V.VdnnError, match="3xTF32"):
        V.Session(g, d, cm, 64 << 20, precise_fp32=True)
    # lossless compression applies to bf16 maps too (tests/test_zvc_gpu.py);
    # the TF32-exact format is fp32-only
    with pytest.raises(V.VdnnError, match="TF32-exact"):
        V.Session(g, d, cm, 64 << 20, compress_offload="tf32")


def test_cpasync_gathers_bf16():
    """The cp.async gather producers (taken for concatenated inputs and
    channel counts that are not 8-multiples) on layers that otherwise take
    the TMA producers: VGG-16 b16 and inception_toy b32, layer-local."""
    _need_gpu()
    from paper_1602_08124_b200 import _lib as L
    L.lib().vdnn_kernel_set_tma(0)
    try:
        TL._run("vgg16_b16_cpasync", "vgg16", 16, "all", False, es=2)
        TL._run("inception_toy_b32_cpasync", "inception_toy", 32, "all", False, es=2)
    finally:
        L.lib().vdnn_kernel_set_tma(1)


@pytest.mark.parametrize("net,batch", [("alexnet", 16), ("vgg16", 4)])
def test_bf16_fused_sgd_matches_external_gradients(net, batch):
    """The fused wgrad + SGD epilogues (pair / persistent / first-layer
    reduce kernels) apply w <- bf16(w - lr * dW) with the dW the same kernels
    write in external-gradient mode: one step with SGD equals the rounded
    update computed on the host (fused multiply-add, as the device rounds it)
    from an external-gradient step, to within one bf16 ulp and exactly for
    almost every weight."""
    _need_gpu()
    g = V.build_preset(net, batch)
    cm = _cm()
    d = V.static_decision(V.PolicyKind.Baseline, V.AlgoMode.PerfOptimal, g, cm)
    w = numeric.he_weights(g, cm, seed=21)
    rng = np.random.default_rng(22)
    sh = g.shape(0)
    images = rng.uniform(-1, 1, size=(batch, sh.h, sh.w, sh.c)).astype(np.float32)
    labels = rng.integers(0, 10, size=batch).astype(np.int32)
    lr = 0.05

    def session(ext):
        s = V.Session(g, d, cm, 8 << 30, external_grads=ext)
        for k, v in w.items():
            s.set_weights(k, v)
        s.set_batch(images, labels)
        s.step(lr)
        return s

    a = session(True)
    grads = {k: a.get_grads(k) for k in w}
    before = {k: a.get_weights(k) for k in w}  # bf16-rounded initial weights (external grads: no update)
    del a
    gc.collect()
    b = session(False)
    exact = total = 0
    for k in w:
        got = b.get_weights(k)
        # the device fuses the multiply-add (one fp32 rounding, then RNE to
        # bf16): at w ~ lr * dW a separately rounded product would differ by
        # many bf16 ulps of the tiny result
        fused = (before[k].astype(np.float64) - np.float64(np.float32(lr)) * grads[k].astype(np.float64))
        want = V.from_bf16_bits(V.to_bf16_bits(fused.astype(np.float32)))
        # got and want are bf16 values: compare their 16-bit patterns
        ulp = np.abs(V.to_bf16_bits(want).astype(np.int64) - V.to_bf16_bits(got).astype(np.int64))
        assert int(ulp.max()) <= 1, (k, int(ulp.max()))
        exact += int((ulp == 0).sum())
        total += ulp.size
    assert exact >= 0.99 * total, (exact, total)
