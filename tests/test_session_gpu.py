"""End-to-end parity of the B200 executor against the CPU numeric oracle.

One training iteration (forward, backward, SGD) of preset and hand-built
graphs under every offload policy; the planner's schedule is replayed on the
device arena with real offload/prefetch copies. Compared with
oracle/numeric.py (float64 CPU restatement of the same dataflow):

* loss: |gpu - cpu| <= LOSS_TOL * max(1, |cpu|)
* weight gradients (recovered as (W_before - W_after)/lr for every layer):
  max |gpu - cpu| <= GRAD_TOL * max |cpu| per layer.
The tensor-core path computes in TF32 (10-bit mantissa inputs, fp32
accumulate); GRAD_TOL covers TF32 rounding compounded through up to 8 layers.
Policies must not change the numbers: for a fork-free network every policy
yields bit-identical weights after the step.
"""
import numpy as np
import pytest

torch = pytest.importorskip("torch")

import paper_1602_08124_b200 as V
from oracle import numeric, refsim

pytestmark = pytest.mark.gpu
LOSS_TOL = 5e-3
GRAD_TOL = 3e-2
LR = 0.01


def _need_gpu():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


def _batch(g, seed=1234):
    s = g.shape(0)
    rng = np.random.default_rng(seed)
    images = rng.uniform(-1, 1, size=(s.n, s.h, s.w, s.c)).astype(np.float32)
    loss_in = g.layer(g.size() - 1).inputs[0]
    ls = g.shape(loss_in)
    labels = rng.integers(0, ls.c * ls.h * ls.w, size=s.n).astype(np.int32)
    return images, labels


def _run_gpu(g, d, weights, images, labels, capacity=2 << 30, record=False):
    s = V.Session(g, d, V.CostModel(), capacity, record_timeline=record)
    for k, w in weights.items():
        s.set_weights(k, w)
    s.set_batch(images, labels)
    loss = s.step(LR)
    after = {k: s.get_weights(k) for k in weights}
    return s, loss, after


def _check(g, weights, after, loss, images, labels, tag):
    cl, cw, cg = numeric.train_step(g, weights, images, labels, LR)
    assert abs(loss - cl) <= LOSS_TOL * max(1.0, abs(cl)), f"{tag}: loss {loss} vs {cl}"
    for k in weights:
        gg = (weights[k].astype(np.float64) - after[k].astype(np.float64)) / LR
        ref = cg[k]
        scale = max(np.abs(ref).max(), 1e-12)
        err = np.abs(gg - ref).max() / scale
        assert err <= GRAD_TOL, f"{tag}: layer {k} grad err {err:.3e}"


POLICIES = [
    ("baseline(p)", V.PolicyKind.Baseline, V.AlgoMode.PerfOptimal),
    ("vdnn-all(m)", V.PolicyKind.VdnnAll, V.AlgoMode.MemoryOptimal),
    ("vdnn-conv(m)", V.PolicyKind.VdnnConv, V.AlgoMode.MemoryOptimal),
    ("vdnn-all(p)", V.PolicyKind.VdnnAll, V.AlgoMode.PerfOptimal),
]


@pytest.mark.parametrize("name,kind,mode", POLICIES)
def test_alexnet_step_matches_oracle(name, kind, mode):
    _need_gpu()
    g = V.build_preset("alexnet", 8)
    cm = V.CostModel()
    w = numeric.he_weights(g, cm)
    images, labels = _batch(g)
    d = V.static_decision(kind, mode, g, cm)
    s, loss, after = _run_gpu(g, d, w, images, labels, capacity=4 << 30)
    _check(g, w, after, loss, images, labels, name)


def test_policies_do_not_change_numbers():
    """Offloading only moves bytes: every policy gives bit-identical results."""
    _need_gpu()
    g = V.build_preset("alexnet", 4)
    cm = V.CostModel()
    w = numeric.he_weights(g, cm, seed=7)
    images, labels = _batch(g, seed=8)
    outs = []
    for name, kind, mode in POLICIES:
        d = V.static_decision(kind, mode, g, cm)
        _, loss, after = _run_gpu(g, d, w, images, labels, capacity=4 << 30)
        outs.append((name, loss, after))
    for name, loss, after in outs[1:]:
        assert loss == outs[0][1], name
        for k in after:
            assert np.array_equal(after[k], outs[0][2][k]), f"{name} layer {k}"


@pytest.mark.parametrize("name,kind,mode", POLICIES)
def test_inception_fork_join_matches_oracle(name, kind, mode):
    _need_gpu()
    g = V.build_preset("inception_toy", 4)
    cm = V.CostModel()
    w = numeric.he_weights(g, cm, seed=3)
    images, labels = _batch(g, seed=4)
    d = V.static_decision(kind, mode, g, cm)
    s, loss, after = _run_gpu(g, d, w, images, labels)
    _check(g, w, after, loss, images, labels, name)


def _odd_graph():
    g = V.NetworkGraph(3)
    x = g.add_input(3, 12, 12)
    a = g.add_conv([x], 5, 3, 1, 1)
    a = g.add_actv(a)
    b = g.add_conv([a], 6, 1, 1, 0)
    c = g.add_actv(a)                      # second reader of a's buffer (in-place alias)
    j = g.add_conv([b, c], 7, 3, 1, 1)     # concat of odd channel counts
    j = g.add_actv(j)
    p = g.add_pool([j], 2, 2)
    f = g.add_fc([p], 9)
    f = g.add_actv(f)
    f = g.add_fc([f], 4)
    g.add_loss(f)
    return g.finalize()


@pytest.mark.parametrize("kind", [V.PolicyKind.VdnnAll, V.PolicyKind.VdnnConv, V.PolicyKind.Baseline])
def test_odd_shapes_concat_alias_matches_oracle(kind):
    _need_gpu()
    g = _odd_graph()
    cm = V.CostModel()
    w = numeric.he_weights(g, cm, seed=5)
    images, labels = _batch(g, seed=6)
    d = V.static_decision(kind, V.AlgoMode.MemoryOptimal, g, cm)
    s, loss, after = _run_gpu(g, d, w, images, labels, capacity=64 << 20)
    _check(g, w, after, loss, images, labels, str(kind))


def test_dyn_under_tight_budget_and_measured_log_replays_clean():
    """VGG-16 at b8 under a budget that forces vDNN_dyn to offload; the measured
    (CUDA-event timed) event log passes our replay_check and the reference's."""
    _need_gpu()
    g = V.build_preset("vgg16", 8)
    cm = V.CostModel()
    oracle_run = V.simulate_oracle(g, cm)
    cap = int(oracle_run.max_mem_bytes * 0.55)
    sel = V.dynamic_select(g, cap, cm)
    assert sel.decision is not None and sel.decision.label != "baseline(p)"
    s = V.Session(g, sel.decision, cm, cap, record_timeline=True)
    s.synthetic_batch(1)
    l0 = s.step(LR)
    l1 = s.step(LR)
    assert np.isfinite(l0) and np.isfinite(l1)
    info = s.arena_info()
    assert info["arena_bytes"] <= cap
    m = s.measured_report()
    assert m.offload_traffic_bytes == s.plan.offload_traffic_bytes > 0
    assert [e.offset for e in m.events] == [e.offset for e in s.plan.events]
    viol = V.replay_check(m, g, sel.decision, cap)
    assert viol == [], viol[:5]
    if refsim.available():
        ev = [(int(e.stream), int(e.kind), e.layer, e.start, e.end, e.bytes, e.tag, e.buffer, e.offset)
              for e in m.events]
        ref = refsim.replay(g.spec(), sel.decision.spec().replace("custom:", "custom:"), cap, ev, m.max_mem_bytes,
                            m.avg_mem_bytes, m.total_ns, True)
        assert ref == [], ref[:5]
