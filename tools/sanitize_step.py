"""One small training step per mode, for compute-sanitizer runs
(memcheck / racecheck / synccheck):

    compute-sanitizer --tool memcheck python tools/sanitize_step.py

Covers the executor (offload/prefetch copies under vDNN_all), the tcgen05
conv engines (TF32 with TMA and cp.async producers, 3xTF32, BF16 kind::f16
with TMA and gathers), the memory-bound kernels and the loss, on presets small
enough that the instrumented run finishes in minutes.
"""
import sys

sys.path.insert(0, ".")
import numpy as np

import paper_1602_08124_b200 as V
from paper_1602_08124_b200 import _lib as L

NETS = [("inception_toy", 4), ("alexnet", 2), ("vgg16", 2)]


def run(net, batch, es, precise, tma):
    g = V.build_preset(net, batch)
    cm = V.CostModel()
    cm.elem_size = es
    d = V.static_decision(V.PolicyKind.VdnnAll, V.AlgoMode.MemoryOptimal, g, cm)
    L.lib().vdnn_kernel_set_tma(int(tma))
    s = V.Session(g, d, cm, 4 << 30, precise_fp32=precise, external_grads=(es == 4 and not precise))
    s.synthetic_batch(3)
    loss = s.step(0.01)
    s.synchronize()
    assert np.isfinite(loss), (net, es, precise, tma, loss)
    print(f"{net} b{batch} es={es} precise={precise} tma={tma}: loss {loss:.6f}", flush=True)
    del s


def main():
    only = sys.argv[1] if len(sys.argv) > 1 else None
    for net, b in NETS:
        if only and net != only:
            continue
        for es, precise, tma in ((4, False, True), (4, False, False), (4, True, True), (2, False, True),
                                 (2, False, False)):
            run(net, b, es, precise, tma)
    print("sanitize_step: ok")


if __name__ == "__main__":
    main()
