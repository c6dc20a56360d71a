"""Per-layer timing of one VGG-16 (or other preset) training step on the GPU.

    python tools/prof_layers.py [net] [batch] [policy] [--no-tma] [--bf16] [--precise]
"""
import sys

sys.path.insert(0, ".")
import paper_1602_08124_b200 as V
from paper_1602_08124_b200 import _lib as L

net = sys.argv[1] if len(sys.argv) > 1 else "vgg16"
batch = int(sys.argv[2]) if len(sys.argv) > 2 else 256
policy = sys.argv[3] if len(sys.argv) > 3 else "none"
if "--no-tma" in sys.argv:
    L.lib().vdnn_kernel_set_tma(0)
g = V.build_preset(net, batch)
cm = V.CostModel()
if "--bf16" in sys.argv:
    cm.elem_size = 2
if policy == "none":
    d = V.static_decision(V.PolicyKind.Baseline, V.AlgoMode.PerfOptimal, g, cm)
    cap = 150 << 30
else:
    d = V.dynamic_select(g, 12884901888, cm).decision
    cap = 12884901888
s = V.Session(g, d, cm, cap, record_timeline=True, precise_fp32="--precise" in sys.argv)
s.synthetic_batch(1)
for _ in range(3):
    s.step(0.01, want_loss=False)
s.step(0.01)
f, b = s.layer_times()
tot_f = tot_b = 0.0
names = ["input", "conv", "actv", "pool", "fc", "loss"]
gem = 0.0
for l in g.layers():
    if l.kind == V.LayerKind.Input:
        continue
    fl = cm.flops(g, l.id, False) if l.kind in (V.LayerKind.Conv, V.LayerKind.Fc) else 0.0
    raw = all(g.layer(q).kind == V.LayerKind.Input for q in l.inputs)
    tf_f = fl / (f[l.id] * 1e-3) / 1e12 if f[l.id] > 0 and fl else 0
    tf_b = (fl * (1 if raw else 2)) / (b[l.id] * 1e-3) / 1e12 if b[l.id] > 0 and fl else 0
    sh = g.shape(l.id)
    print(f"{l.id:3d} {names[l.kind]:5s} {str((sh.c, sh.h, sh.w)):18s} fwd {f[l.id]:8.3f} ms {tf_f:6.1f} TF  "
          f"bwd {b[l.id]:8.3f} ms {tf_b:6.1f} TF")
    tot_f += f[l.id]
    tot_b += b[l.id]
print(f"total fwd {tot_f:.2f} ms bwd {tot_b:.2f} ms")
