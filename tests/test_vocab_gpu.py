"""The reference's whole graph vocabulary on the B200 executor.

net_graph.hpp accepts concat and elementwise joins (:83, :281-297), strided
convs (:307-321), any number of INPUT and LOSS layers; the planner plans all
of them bit-exactly. These tests run such graphs end to end -- forward,
backward, SGD with real offload/prefetch under every policy -- against the
numeric oracle (oracle/numeric.train_step):

* random graphs from a generator that exercises every construct at once
  (elementwise joins whose inputs are ReLU chains -> read-only shared
  gradient maps and private planes; strided convs with and without a data
  gradient; two INPUT layers; an auxiliary LOSS head);
* the reference fuzz campaign's own graphs (fuzz.hpp:26-63, exported by the
  compiled reference, oracle/_ref);
* a network defined inline in an INI experiment file (config.hpp:183-269)
  and one defined as graph JSON (report.hpp:44-111).

Graphs are small, so the fp32 mode (3xTF32) is compared end to end with
float64 at a tight bound: loss within 1e-4 relative, every weight gradient
within 1e-3 relative L2. TF32 mode is compared layer by layer
(tests/layer_parity.py: every kernel on the operands it read, against the
oracle op that reads contraction operands as kind::tf32 does) -- end to end,
a TF32 operand truncation can flip a near-tied ReLU mask or pool argmax and
the difference compounds backwards.
"""
import json
import os
import random

import numpy as np
import pytest

torch = pytest.importorskip("torch")

import paper_1602_08124_b200 as V
from oracle import numeric, refsim
from planner_util import graph_from_spec, vocab_spec

import layer_parity as LP

pytestmark = pytest.mark.gpu
LR = 0.01
FP32_LOSS_TOL, FP32_GRAD_TOL = 1e-4, 1e-3


def _need_gpu():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


def _inputs_and_labels(g, seed):
    rng = np.random.default_rng(seed)
    ims = {}
    for l in g.layers():
        if l.kind == V.LayerKind.Input:
            s = g.shape(l.id)
            ims[l.id] = rng.uniform(-1, 1, size=(s.n, s.h, s.w, s.c)).astype(np.float32)
    labels = rng.integers(0, 1000, size=g.batch).astype(np.int32)
    return ims, labels


def _decisions(g, cm):
    out = [V.static_decision(k, m, g, cm) for k, m in
           ((V.PolicyKind.Baseline, V.AlgoMode.PerfOptimal), (V.PolicyKind.VdnnAll, V.AlgoMode.MemoryOptimal),
            (V.PolicyKind.VdnnConv, V.AlgoMode.MemoryOptimal))]
    floor = V.simulate(g, out[1], cm, V.KUNLIMITED_BYTES).max_mem_bytes
    sel = V.dynamic_select(g, int(floor * 1.02), cm).decision
    if sel is not None:
        out.append(sel)
    return out


def run_and_compare(g, d, cm, ims, labels, precise, tag, cap=1 << 30):
    w = numeric.he_weights(g, cm, seed=3)
    s = V.Session(g, d, cm, cap, external_grads=True, precise_fp32=precise, record_timeline=True)
    for k, v in w.items():
        s.set_weights(k, v)
    first = min(ims)
    s.set_batch(ims[first], labels)
    for k, im in ims.items():
        if k != first:
            s.set_input(k, im)
    loss = s.step(LR)
    assert V.replay_check(s.measured_report(), g, d, cap) == []
    if not precise:  # layer-local (same inputs and weights every step: external_grads)
        recs = LP.check_session(s, g, labels, precise=False)
        bad = LP.violations(recs, False, bf16=s.bf16)
        assert not bad, f"{tag}: " + "; ".join(bad[:6])
        return loss
    grads = {k: s.get_grads(k) for k in w}
    del s
    cl, _, cg = numeric.train_step(g, w, ims, labels, LR)
    assert abs(loss - cl) <= FP32_LOSS_TOL * max(1.0, abs(cl)), f"{tag}: loss {loss} vs {cl}"
    for k in w:
        err = np.linalg.norm(grads[k].astype(np.float64) - cg[k]) / max(np.linalg.norm(cg[k]), 1e-30)
        assert err <= FP32_GRAD_TOL, f"{tag}: layer {k} dW rel-L2 {err:.3e}"
    return loss


@pytest.mark.parametrize("seed", range(8))
def test_random_full_vocabulary_graphs(seed):
    _need_gpu()
    rng = random.Random(1000 + seed)
    cm = V.CostModel()
    for t in range(3):
        spec = vocab_spec(rng)
        g = graph_from_spec(spec)
        ims, labels = _inputs_and_labels(g, seed * 10 + t)
        for d in _decisions(g, cm):
            for precise in (True, False):
                run_and_compare(g, d, cm, ims, labels, precise, f"{spec} {d.label} precise={precise}")


@pytest.mark.skipif(not refsim.available(), reason="compiled reference (oracle/_ref) not built")
def test_reference_fuzz_graphs_on_gpu():
    """The reference fuzz generator's graphs (fuzz.hpp:26-63), every policy."""
    _need_gpu()
    cm = V.CostModel()
    for seed in range(40):
        spec = refsim.fuzz_graph(seed, 12 + seed % 10)
        g = graph_from_spec(spec)
        ims, labels = _inputs_and_labels(g, seed)
        for d in _decisions(g, cm):
            run_and_compare(g, d, cm, ims, labels, True, f"fuzz {seed} {spec} {d.label}")


INI = """
[network]
batch = 4
layer00 = input c=3 h=12 w=12
layer01 = conv inputs=0 k=3 s=1 p=1 out=16
layer02 = actv inputs=1
layer03 = conv inputs=2 k=3 s=1 p=1 out=16
layer04 = actv inputs=3
layer05 = conv inputs=2 k=1 s=1 p=0 out=16
layer06 = conv inputs=4,5 join=eltwise k=2 s=2 p=0 out=8
layer07 = actv inputs=6
layer08 = pool inputs=7 window=2 stride=2
layer09 = fc inputs=8 out=10
layer10 = loss inputs=9
[policy]
policy = vdnn_all
capacity = 1 GiB
"""


def test_ini_inline_network_runs_and_matches(tmp_path):
    """config.hpp:183-269 inline layers (ids follow the keys' sorted order, as
    std::map visits them): an elementwise join of a ReLU branch and a plain
    branch feeding a strided conv, under every policy."""
    _need_gpu()
    from paper_1602_08124_b200 import config
    p = tmp_path / "net.ini"
    p.write_text(INI)
    cfg = config.load_config(str(p))
    g = config.build_network(cfg)
    cm = V.CostModel()
    ims, labels = _inputs_and_labels(g, 5)
    for d in _decisions(g, cm):
        run_and_compare(g, d, cm, ims, labels, True, f"ini {d.label}")


def test_graph_json_network_runs_and_matches():
    """report.hpp:44-111 graph JSON: a GoogLeNet-like module (concat of 1x1,
    3x3, 5x5 and pool branches), a residual elementwise join and two heads."""
    _need_gpu()
    g = json_graph()
    cm = V.CostModel()
    ims, labels = _inputs_and_labels(g, 6)
    for d in _decisions(g, cm):
        for precise in (True, False):
            run_and_compare(g, d, cm, ims, labels, precise, f"json {d.label} precise={precise}")


def json_graph():
    from paper_1602_08124_b200 import formats
    L = []

    def lay(kind, inputs=(), **kw):
        e = {"id": len(L), "kind": kind}
        if inputs:
            e["inputs"] = list(inputs)
        e.update(kw)
        L.append(e)
        return e["id"]

    x = lay("input", c=3, h=16, w=16)
    s = lay("conv", [x], kernel=3, stride=1, pad=1, out_channels=32)
    s = lay("actv", [s])
    b1 = lay("conv", [s], kernel=1, stride=1, pad=0, out_channels=16)
    b1 = lay("actv", [b1])
    b2 = lay("conv", [s], kernel=3, stride=1, pad=1, out_channels=16)
    b2 = lay("actv", [b2])
    b3 = lay("conv", [s], kernel=5, stride=1, pad=2, out_channels=8)
    b3 = lay("actv", [b3])
    b4 = lay("pool", [s], window=3, stride=1)
    b4 = lay("conv", [b4], kernel=3, stride=1, pad=2, out_channels=8)
    cat = lay("conv", [b1, b2, b3, b4], join="concat", kernel=1, stride=1, pad=0, out_channels=32)
    cat = lay("actv", [cat])
    res = lay("conv", [cat, s], join="eltwise", kernel=4, stride=2, pad=1, out_channels=32)
    res = lay("actv", [res])
    aux = lay("fc", [cat], out_features=7)
    lay("loss", [aux])
    f = lay("fc", [res], out_features=10)
    lay("loss", [f])
    return formats.graph_from_json({"batch": 4, "layers": L})
