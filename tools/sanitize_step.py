"""One small training step per mode, for compute-sanitizer runs
(memcheck / racecheck / synccheck):

    compute-sanitizer --tool memcheck python tools/sanitize_step.py

Covers the executor (offload/prefetch copies under vDNN_all, also through the
fp32 and BF16 zero-value-compressing kernels), the tcgen05 conv engines (TF32
with TMA and cp.async producers, 3xTF32 with TMA + split warps, BF16 kind::f16:
pair, halo, halo wgrad, persistent, first-layer c3b, gathers), the
memory-bound kernels and the loss, on presets small enough that the
instrumented run finishes in minutes.
"""
import sys

sys.path.insert(0, ".")
import numpy as np

import paper_1602_08124_b200 as V
from paper_1602_08124_b200 import _lib as L

NETS = [("inception_toy", 4), ("alexnet", 2), ("vgg16", 2)]


def run(net, batch, es, precise, tma, compress=False):
    g = V.build_preset(net, batch)
    cm = V.CostModel()
    cm.elem_size = es
    d = V.static_decision(V.PolicyKind.VdnnAll, V.AlgoMode.MemoryOptimal, g, cm)
    L.lib().vdnn_kernel_set_tma(int(tma))
    s = V.Session(g, d, cm, 4 << 30, precise_fp32=precise, external_grads=(es == 4 and not precise),
                  compress_offload=compress)
    s.synthetic_batch(3)
    loss = s.step(0.01)
    s.synchronize()
    assert np.isfinite(loss), (net, es, precise, tma, loss)
    print(f"{net} b{batch} es={es} precise={precise} tma={tma} compress={compress}: loss {loss:.6f}", flush=True)
    del s


def main():
    only = sys.argv[1] if len(sys.argv) > 1 else None
    for net, b in NETS:
        if only and net != only:
            continue
        for es, precise, tma, comp in ((4, False, True, False), (4, False, False, False), (4, True, True, False),
                                       (2, False, True, False), (2, False, False, False), (4, False, True, True),
                                       (2, False, True, True)):
            run(net, b, es, precise, tma, comp)
    print("sanitize_step: ok")


if __name__ == "__main__":
    main()
