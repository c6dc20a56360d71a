"""The reference's GEMM_WS convolution algorithm as real kernels
(Session(algo_kernels="planned"), kernels/conv_gemmws.cu): for a layer whose
planned algorithm is GEMM_WS, im2col of X into the planned workspace
(cost_model.hpp:163-168 sizes it as the k*k*Cin*Ho*Wo*N im2col matrix), the
contraction as a 1x1 GEMM over it, col2im (with the fused ReLU-backward mask
and accumulation) for the data gradient.

Checked layer-locally (tests/layer_parity.py): every FWD / dgrad / wgrad
result against the float64 oracle op on the operands the step read, at the
same bounds as the implicit-GEMM kernels -- end-to-end comparisons of two
kernel families only measure how near-ties of ReLU / max-pool flip after one
different rounding. Covers a strided window (AlexNet conv1, 11x11 stride 4)
and BF16 storage; the plan (and every workspace extent) is unchanged."""
import numpy as np
import pytest

import paper_1602_08124_b200 as V

torch = pytest.importorskip("torch")

import layer_parity as LP

pytestmark = pytest.mark.gpu


def _gemmws_decision(g, cm):
    base = V.static_decision(V.PolicyKind.Baseline, V.AlgoMode.PerfOptimal, g, cm)
    algos = {i: (V.AlgoId.GemmWs if g.layer(i).kind == V.LayerKind.Conv else a) for i, a in base.algos.items()}
    return V.PolicyDecision(list(base.offload), algos, base.gradient_scheme, "baseline(gemm_ws)")


@pytest.mark.parametrize("net,batch,es", [("vgg16", 2, 4), ("alexnet", 4, 4), ("vgg16", 2, 2), ("alexnet", 4, 2)])
def test_gemmws_kernels_layer_local(net, batch, es):
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    g = V.build_preset(net, batch)
    cm = V.CostModel()
    cm.elem_size = es
    d = _gemmws_decision(g, cm)
    ref = V.Session(g, d, cm, 64 << 30, external_grads=True)
    s = V.Session(g, d, cm, 64 << 30, external_grads=True, algo_kernels="planned")
    assert s.plan.signature() == ref.plan.signature()  # same plan, same workspace extents
    del ref
    sh = g.shape(0)
    rng = np.random.default_rng(40 + batch)
    images = rng.uniform(-1, 1, size=(batch, sh.h, sh.w, sh.c)).astype(np.float32)
    ls = g.shape(g.layer(g.size() - 1).inputs[0])
    labels = rng.integers(0, ls.c * ls.h * ls.w, size=batch).astype(np.int32)
    s.set_batch(images, labels)
    s.step(0.01)
    recs = LP.check_session(s, g, labels, precise=False)
    ops = {r["op"] for r in recs}
    assert {"fprop", "dgrad", "wgrad"} <= ops
    if es == 2:
        # BF16 storage: the GEMM_WS data gradient is rounded twice -- the
        # column gradient is stored in the (bf16-sized) planned workspace, and
        # col2im's fp32 sum of up to k*k of those values is rounded again into
        # dX -- so its bound is two storage roundings; everything else keeps
        # the one-rounding bounds of the implicit kernels
        recs = [dict(r, err_plain=r["err_plain"] / 2) if r["op"] == "dgrad" else r for r in recs]
    bad = LP.violations(recs, False, bf16=es == 2)
    assert not bad, f"{net} es={es} GEMM_WS: {len(bad)} violations: " + "; ".join(bad[:8])


def test_gemmws_mode_validation():
    with pytest.raises(ValueError):
        V.Session(V.build_preset("inception_toy", 2), None, algo_kernels="fft")
