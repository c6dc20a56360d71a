"""End-to-end parity of the B200 executor against the CPU numeric oracle.

One training iteration (forward, backward, SGD) of preset and hand-built
graphs under every offload policy; the planner's schedule is replayed on the
device arena with real offload/prefetch copies. Compared with
oracle/numeric.py (float64 CPU restatement of the same dataflow):

* loss: |gpu - cpu| <= LOSS_TOL * max(1, |cpu|)
* weight gradients (read back from the gradient arena, external_grads=True):
  ||gpu - cpu||_2 <= TOL * ||cpu||_2 per layer (relative L2 norm: a ReLU mask
  or max-pool argmax that flips on a near-tie routes one entry differently,
  which a max-abs metric would amplify into a spurious failure).
The tensor-core path computes in TF32 (10-bit mantissa inputs, fp32
accumulate). Against the oracle that reads conv/FC operands the way kind::tf32
does, the tolerance is TF32_GRAD_TOL; against plain float64, GRAD_TOL.
Policies must not change the numbers: for a fork-free network every policy
yields bit-identical weights after the step.
"""
import numpy as np
import pytest

torch = pytest.importorskip("torch")

import paper_1602_08124_b200 as V
from oracle import numeric, refsim

pytestmark = pytest.mark.gpu
LR = 0.01
# fp32 mode (precise_fp32=True: 3xTF32 contractions) vs the float64 oracle.
# The tensor core's fp32 accumulation is not round-to-nearest: measured
# single-layer bias ~7e-9 * K relative (K = reduction length), so deep nets
# sit at ~1e-4 on the loss and <= ~6e-3 rel-L2 on early-layer dW (AlexNet).
FP32_LOSS_TOL = 2e-4
FP32_GRAD_TOL = 2e-2
# TF32 mode (default) vs the float64 oracle: TF32 operand truncation (2^-11
# relative per operand) compounds through the layers and flips near-tied
# ReLU masks / pool argmaxes, so per-layer weight gradients of deep nets
# differ by a few percent in relative L2 (measured: <= 8e-2 on AlexNet b8).
TF32_LOSS_TOL = 1e-2
TF32_GRAD_TOL = 1.5e-1


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


def _run_gpu(g, d, weights, images, labels, capacity=2 << 30, record=False, grads=False, precise=False):
    """grads=True: dW goes to the gradient arena (read back exactly) instead of
    the fused SGD epilogue; returns the gradients instead of updated weights."""
    s = V.Session(g, d, V.CostModel(), capacity, record_timeline=record, external_grads=grads,
                  precise_fp32=precise)
    for k, w in weights.items():
        s.set_weights(k, w)
    s.set_batch(images, labels)
    loss = s.step(LR)
    if grads:
        return s, loss, {k: s.get_grads(k) for k in weights}
    after = {k: s.get_weights(k) for k in weights}
    return s, loss, after


def _errs(g, weights, grads, loss, images, labels, tf32):
    cl, cw, cg = numeric.train_step(g, weights, images, labels, LR, tf32_operands=tf32)
    out = {}
    for k in weights:
        gg = grads[k].astype(np.float64)
        ref = cg[k]
        out[k] = np.linalg.norm(gg - ref) / max(np.linalg.norm(ref), 1e-30)
    return cl, out


def _check(g, weights, grads, loss, images, labels, tag, precise):
    cl, errs = _errs(g, weights, grads, loss, images, labels, False)
    lt, gt = (FP32_LOSS_TOL, FP32_GRAD_TOL) if precise else (TF32_LOSS_TOL, TF32_GRAD_TOL)
    print(tag, "precise" if precise else "tf32", "loss", loss, cl, {k: f"{v:.2e}" for k, v in errs.items()})
    assert abs(loss - cl) <= lt * max(1.0, abs(cl)), f"{tag}: loss {loss} vs {cl}"
    for k, e in errs.items():
        assert e <= gt, f"{tag}: layer {k} grad rel-L2 err {e:.3e} (tol {gt})"


POLICIES = [
    ("baseline(p)", V.PolicyKind.Baseline, V.AlgoMode.PerfOptimal),
    ("vdnn-all(m)", V.PolicyKind.VdnnAll, V.AlgoMode.MemoryOptimal),
    ("vdnn-conv(m)", V.PolicyKind.VdnnConv, V.AlgoMode.MemoryOptimal),
    ("vdnn-all(p)", V.PolicyKind.VdnnAll, V.AlgoMode.PerfOptimal),
]


@pytest.mark.parametrize("precise", [True, False], ids=["fp32", "tf32"])
@pytest.mark.parametrize("name,kind,mode", POLICIES)
def test_alexnet_step_matches_oracle(name, kind, mode, precise):
    _need_gpu()
    g = V.build_preset("alexnet", 8)
    cm = V.CostModel()
    w = numeric.he_weights(g, cm)
    images, labels = _batch(g)
    d = V.static_decision(kind, mode, g, cm)
    s, loss, grads = _run_gpu(g, d, w, images, labels, capacity=4 << 30, grads=True, precise=precise)
    _check(g, w, grads, loss, images, labels, name, precise)


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


@pytest.mark.parametrize("precise", [True, False], ids=["fp32", "tf32"])
@pytest.mark.parametrize("name,kind,mode", POLICIES)
def test_inception_fork_join_matches_oracle(name, kind, mode, precise):
    _need_gpu()
    g = V.build_preset("inception_toy", 4)
    cm = V.CostModel()
    w = numeric.he_weights(g, cm, seed=3)
    images, labels = _batch(g, seed=4)
    d = V.static_decision(kind, mode, g, cm)
    s, loss, grads = _run_gpu(g, d, w, images, labels, grads=True, precise=precise)
    _check(g, w, grads, loss, images, labels, name, precise)


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


@pytest.mark.parametrize("precise", [True, False], ids=["fp32", "tf32"])
@pytest.mark.parametrize("kind", [V.PolicyKind.VdnnAll, V.PolicyKind.VdnnConv, V.PolicyKind.Baseline])
def test_odd_shapes_concat_alias_matches_oracle(kind, precise):
    _need_gpu()
    g = _odd_graph()
    cm = V.CostModel()
    w = numeric.he_weights(g, cm, seed=5)
    images, labels = _batch(g, seed=6)
    d = V.static_decision(kind, V.AlgoMode.MemoryOptimal, g, cm)
    s, loss, grads = _run_gpu(g, d, w, images, labels, capacity=64 << 20, grads=True, precise=precise)
    _check(g, w, grads, loss, images, labels, str(kind), precise)



def test_fused_sgd_matches_external_grads():
    """The fused wgrad+SGD epilogue applies exactly lr * dW of the grad path."""
    _need_gpu()
    g = V.build_preset("inception_toy", 2)
    cm = V.CostModel()
    w = numeric.he_weights(g, cm, seed=9)
    images, labels = _batch(g, seed=10)
    d = V.static_decision(V.PolicyKind.VdnnAll, V.AlgoMode.MemoryOptimal, g, cm)
    _, l1, grads = _run_gpu(g, d, w, images, labels, grads=True)
    _, l2, after = _run_gpu(g, d, w, images, labels)
    assert l1 == l2
    for k in w:
        ref = w[k].astype(np.float32) - np.float32(LR) * grads[k]
        np.testing.assert_allclose(after[k], ref, rtol=0, atol=2e-7 * max(1.0, float(np.abs(w[k]).max())))


def test_dyn_under_tight_budget_and_measured_log_replays_clean():
    """VGG-16 at b8 under a budget that forces vDNN_dyn to offload; the measured
    (CUDA-event timed) event log passes our replay_check and the reference's."""
    _need_gpu()
    g = V.build_preset("vgg16", 8)
    cm = V.CostModel()
    floor = V.static_decision(V.PolicyKind.VdnnAll, V.AlgoMode.MemoryOptimal, g, cm)
    cap = int(V.simulate(g, floor, cm, V.KUNLIMITED_BYTES).max_mem_bytes * 1.05)
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
    assert V.placements(m) == V.placements(s.plan)  # every non-SYNC row, planned offsets
    viol = V.replay_check(m, g, sel.decision, cap)
    assert viol == [], viol[:5]
    if refsim.available():
        ev = [(int(e.stream), int(e.kind), e.layer, e.start, e.end, e.bytes, e.tag, e.buffer, e.offset)
              for e in m.events]
        ref = refsim.replay(g.spec(), sel.decision.spec().replace("custom:", "custom:"), cap, ev, m.max_mem_bytes,
                            m.avg_mem_bytes, m.total_ns, True)
        assert ref == [], ref[:5]


def test_vgg16_b32_production_kernels_match_oracle():
    """VGG-16 at batch 32 runs the production kernel variants end to end:
    halo-reuse fprop/dgrad (224x224x64, 112x112x128), CTA-pair fprop/dgrad
    (56x56x256, 28x28x512) and pair wgrad, split-K FC fprop, the 2x2 pool fast
    path and the tensor-core first layer -- under vDNN_conv with real
    offload/prefetch, against the float64 restatement evaluated on the GPU
    (same TF32 tolerances as the small nets), and bit-identical to the
    no-offload run."""
    _need_gpu()
    g = V.build_preset("vgg16", 32)
    cm = V.CostModel()
    w = numeric.he_weights(g, cm, seed=41)
    images, labels = _batch(g, seed=42)
    d = V.static_decision(V.PolicyKind.VdnnConv, V.AlgoMode.MemoryOptimal, g, cm)
    s, loss, grads = _run_gpu(g, d, w, images, labels, capacity=3 << 30, grads=True)
    assert s.plan.offload_traffic_bytes > 0
    cl, _, cg = numeric.train_step(g, w, images, labels, LR, device="cuda")
    errs = {k: np.linalg.norm(grads[k].astype(np.float64) - cg[k]) / max(np.linalg.norm(cg[k]), 1e-30) for k in w}
    print("vgg16 b32 loss", loss, cl, {k: f"{v:.2e}" for k, v in errs.items()})
    assert abs(loss - cl) <= TF32_LOSS_TOL * max(1.0, abs(cl))
    for k, e in errs.items():
        assert e <= TF32_GRAD_TOL, f"layer {k} grad rel-L2 err {e:.3e}"
    # against the oracle that reads every contraction operand the way kind::tf32 does
    cl2, _, cg2 = numeric.train_step(g, w, images, labels, LR, device="cuda", tf32_operands=True)
    errs2 = {k: np.linalg.norm(grads[k].astype(np.float64) - cg2[k]) / max(np.linalg.norm(cg2[k]), 1e-30) for k in w}
    print("vs tf32-operand oracle", loss, cl2, {k: f"{v:.2e}" for k, v in errs2.items()})
    # measured: loss 7e-5 relative; dW 1e-3 (last FC) .. 1.1e-1 (first conv) rel-L2,
    # the spread being ReLU-mask / pool-argmax flips compounding backwards
    assert abs(loss - cl2) <= 1e-3 * max(1.0, abs(cl2))
    for k, e in errs2.items():
        assert e <= TF32_GRAD_TOL, f"layer {k} grad rel-L2 err vs tf32 oracle {e:.3e}"
    del s
    db = V.static_decision(V.PolicyKind.Baseline, V.AlgoMode.PerfOptimal, g, cm)
    _, loss_b, grads_b = _run_gpu(g, db, w, images, labels, capacity=8 << 30, grads=True)
    assert loss_b == loss
    for k in w:
        assert np.array_equal(grads_b[k], grads[k]), f"layer {k}"


def test_device_offload_target_is_bit_identical():
    """offload_target="device": the same plan's offloads/prefetches go to a
    device buffer (the stand-in for a peer GPU's HBM) instead of pinned host
    memory -- same slots, same sync rules, so identical weights, and the
    measured log still replays clean."""
    _need_gpu()
    g = V.build_preset("alexnet", 8)
    cm = V.CostModel()
    w = numeric.he_weights(g, cm, seed=13)
    images, labels = _batch(g, seed=14)
    d = V.static_decision(V.PolicyKind.VdnnAll, V.AlgoMode.MemoryOptimal, g, cm)
    outs = []
    for target in ("host", "device"):
        s = V.Session(g, d, cm, 4 << 30, record_timeline=True, offload_target=target)
        spill = None
        if target == "device":
            n = s.offload_bytes()
            assert n > 0
            spill = torch.empty(n // 4 + 1, dtype=torch.float32, device="cuda")
            s.set_offload_buffer(spill.data_ptr(), spill.numel() * 4)
        for k, v in w.items():
            s.set_weights(k, v)
        s.set_batch(images, labels)
        loss = s.step(LR)
        loss2 = s.step(LR)
        outs.append((loss, loss2, {k: s.get_weights(k) for k in w}))
        assert V.replay_check(s.measured_report(), g, d, 4 << 30) == []
        del s, spill
    assert outs[0][0] == outs[1][0] and outs[0][1] == outs[1][1]
    for k in w:
        assert np.array_equal(outs[0][2][k], outs[1][2][k]), k


def test_device_offload_target_requires_a_buffer():
    _need_gpu()
    g = V.build_preset("alexnet", 4)
    cm = V.CostModel()
    d = V.static_decision(V.PolicyKind.VdnnAll, V.AlgoMode.MemoryOptimal, g, cm)
    s = V.Session(g, d, cm, 4 << 30, offload_target="device")
    s.synthetic_batch(3)
    with pytest.raises(V.VdnnError):
        s.step(LR)
    with pytest.raises(V.VdnnError):
        V.Session(g, d, cm, 4 << 30, offload_target="device", compress_offload=True)


def test_prefetched_batches_match_set_batch():
    """Input pipeline: batches staged with prefetch_batch_ptr (pinned host ->
    device on the input stream, overlapping the running step) give the same
    weights and losses as set_batch before every step."""
    _need_gpu()
    g = V.build_preset("alexnet", 4)
    cm = V.CostModel()
    w = numeric.he_weights(g, cm, seed=71)
    d = V.static_decision(V.PolicyKind.VdnnAll, V.AlgoMode.MemoryOptimal, g, cm)
    batches = [_batch(g, seed=72 + i) for i in range(3)]
    pinned = [(torch.from_numpy(im).pin_memory(), torch.from_numpy(lb).pin_memory()) for im, lb in batches]
    outs = []
    for mode in ("set", "prefetch", "pipelined"):
        s = V.Session(g, d, cm, 4 << 30)
        for k, v in w.items():
            s.set_weights(k, v)
        losses = []
        if mode == "set":
            for im, lb in batches:
                s.set_batch(im, lb)
                losses.append(s.step(LR))
        elif mode == "prefetch":
            s.prefetch_batch_ptr(pinned[0][0].data_ptr(), pinned[0][1].data_ptr())
            for i in range(3):
                s.step(LR, want_loss=False)
                if i + 1 < 3:
                    s.prefetch_batch_ptr(pinned[i + 1][0].data_ptr(), pinned[i + 1][1].data_ptr())
                losses.append(s.read_loss())
        else:  # loss readback pipelined one step behind (queue_loss / wait_loss)
            s.prefetch_batch_ptr(pinned[0][0].data_ptr(), pinned[0][1].data_ptr())
            tickets = []
            for i in range(3):
                s.step(LR, want_loss=False)
                tickets.append(s.queue_loss())
                if i + 1 < 3:
                    s.prefetch_batch_ptr(pinned[i + 1][0].data_ptr(), pinned[i + 1][1].data_ptr())
            losses = [s.wait_loss(t) for t in tickets]
        outs.append((losses, {k: s.get_weights(k) for k in w}))
        del s
    for o in outs[1:]:
        assert o[0] == outs[0][0]
        for k in w:
            assert np.array_equal(o[1][k], outs[0][1][k]), k


@pytest.mark.parametrize("compress", [False, True], ids=["copy-engines", "zvc"])
def test_cuda_graph_steps_are_bit_identical(compress):
    """cuda_graph=True: the step is captured once (second step) and replayed
    as one CUDA graph -- both streams, the offload/prefetch copies and their
    event gating -- and re-captured when lr changes. Weights, losses, transfer
    accounting and the measured log equal the eager run."""
    _need_gpu()
    g = V.build_preset("alexnet", 4)
    cm = V.CostModel()
    w = numeric.he_weights(g, cm, seed=81)
    images, labels = _batch(g, seed=82)
    d = V.static_decision(V.PolicyKind.VdnnAll, V.AlgoMode.MemoryOptimal, g, cm)
    outs = []
    for graph in (False, True):
        s = V.Session(g, d, cm, 4 << 30, record_timeline=True, compress_offload=compress, cuda_graph=graph)
        for k, v in w.items():
            s.set_weights(k, v)
        s.set_batch(images, labels)
        l0 = V.kernel_launch_count()
        losses = [s.step(LR) for _ in range(3)] + [s.step(LR / 2) for _ in range(2)]
        launches = V.kernel_launch_count() - l0
        stats = s.transfer_stats()
        assert V.replay_check(s.measured_report(), g, d, 4 << 30) == []
        outs.append((losses, {k: s.get_weights(k) for k in w}, stats, launches))
        del s
    assert outs[0][0] == outs[1][0]
    for k in w:
        assert np.array_equal(outs[0][1][k], outs[1][1][k]), k
    assert outs[0][2] == outs[1][2]
    assert outs[0][3] == outs[1][3]


def test_vgg16_b256_headline_plan_full_size():
    """BASELINE config 4 at full size: VGG-16 b256 under the 12 GiB budget.
    The dyn decision and schedule are the reference's (vdnn-conv+greedy,
    signature 2188dd2e41bf52e2 in tests/golden/vgg16_b256.json); the measured
    event log of the real run keeps every planned pool offset and replays
    clean; one training step with copy-engine transfers, with TF32-exact
    compressed transfers, and without offload (32.7 GB pool) gives the same
    loss and the same updated weights bit for bit (size-independent
    properties at the size the headline is quoted on)."""
    _need_gpu()
    import gc
    import hashlib
    import torch
    g = V.build_preset("vgg16", 256)
    cm = V.CostModel()
    cap = 12884901888
    sel = V.dynamic_select(g, cap, cm)
    d = sel.decision
    assert d.label == "vdnn-conv+greedy"

    def run(decision, capacity, **kw):
        s = V.Session(g, decision, cm, capacity, **kw)
        s.synthetic_batch(7)
        loss = s.step(LR)
        h = hashlib.sha256()
        for l in g.layers():
            if l.kind in (V.LayerKind.Conv, V.LayerKind.Fc):
                h.update(np.ascontiguousarray(s.get_weights(l.id)).tobytes())
        return s, loss, h.hexdigest()

    s, loss_dyn, w_dyn = run(d, cap, record_timeline=True)
    assert s.plan.signature() == "2188dd2e41bf52e2"
    assert s.arena_info()["arena_bytes"] <= cap
    m = s.measured_report()
    assert m.offload_traffic_bytes == s.plan.offload_traffic_bytes == 10635706368
    assert V.placements(m) == V.placements(s.plan)  # every non-SYNC row, planned offsets
    assert V.replay_check(m, g, d, cap) == []
    del s, m
    gc.collect()
    s, loss_t, w_t = run(d, cap, compress_offload="tf32")
    st = s.transfer_stats()
    assert st["offload_wire"] < 0.4 * st["offload_planned"]
    del s
    gc.collect()
    free, _ = torch.cuda.mem_get_info()
    db = V.static_decision(V.PolicyKind.Baseline, V.AlgoMode.PerfOptimal, g, cm)
    s, loss_b, w_b = run(db, int(free - (6 << 30)))
    del s
    gc.collect()
    assert np.isfinite(loss_dyn)
    assert loss_dyn == loss_t == loss_b
    assert w_dyn == w_t == w_b


def test_pause_timeline_keeps_numbers_and_reports_last_recorded_step():
    """pause_timeline skips the per-op events (benchmark loops) without
    changing results; after resuming, the measured report and layer times
    describe the last recorded step and still replay clean."""
    _need_gpu()
    g = V.build_preset("alexnet", 16)
    cm = V.CostModel()
    d = V.static_decision(V.PolicyKind.VdnnAll, V.AlgoMode.MemoryOptimal, g, cm)
    cap = 4 << 30
    losses = []
    for pause in (False, True):
        s = V.Session(g, d, cm, cap, record_timeline=True)
        s.synthetic_batch(5)
        s.step(LR)
        s.pause_timeline(pause)
        s.step(LR)
        s.step(LR)
        s.pause_timeline(False)
        losses.append(s.step(LR))
        f, b = s.layer_times()
        assert sum(f) > 0 and sum(b) > 0
        m = s.measured_report()
        assert V.replay_check(m, g, d, cap) == []
        del s
    assert losses[0] == losses[1]
