"""One training step of a preset (for ncu launch lists): python tools/one_step.py [net] [batch] [policy] [--bf16]"""
import sys

sys.path.insert(0, ".")
import paper_1602_08124_b200 as V

net = sys.argv[1] if len(sys.argv) > 1 else "vgg16"
batch = int(sys.argv[2]) if len(sys.argv) > 2 else 256
policy = sys.argv[3] if len(sys.argv) > 3 else "none"
g = V.build_preset(net, batch)
cm = V.CostModel()
if "--bf16" in sys.argv:
    cm.elem_size = 2
if policy == "none":
    d, cap = V.static_decision(V.PolicyKind.Baseline, V.AlgoMode.PerfOptimal, g, cm), 150 << 30
else:
    d, cap = V.dynamic_select(g, 12884901888, cm).decision, 12884901888
s = V.Session(g, d, cm, cap)
s.synthetic_batch(1)
s.step(0.01, want_loss=False)
print("loss", s.step(0.01))
