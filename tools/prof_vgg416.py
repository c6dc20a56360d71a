import sys
sys.path.insert(0, ".")
import paper_1602_08124_b200 as V
from collections import defaultdict
g = V.extend_vgg(400, 32)
cm = V.CostModel()
d = V.static_decision(V.PolicyKind.Baseline, V.AlgoMode.PerfOptimal, g, cm)
s = V.Session(g, d, cm, 100 << 30, record_timeline=True)
s.synthetic_batch(1)
for _ in range(3):
    s.step(0.01, want_loss=False)
s.step(0.01)
f, b = s.layer_times()
agg = defaultdict(lambda: [0, 0.0, 0.0, 0.0])
for l in g.layers():
    if l.kind != V.LayerKind.Conv and l.kind != V.LayerKind.Pool:
        continue
    sh = g.shape(l.id)
    key = (l.kind.name, sh.c, sh.h)
    fl = cm.flops(g, l.id, False) if l.kind == V.LayerKind.Conv else 0
    a = agg[key]
    a[0] += 1; a[1] += f[l.id]; a[2] += b[l.id]; a[3] += fl
for k, (n, ff, bb, fl) in sorted(agg.items(), key=lambda x: -(x[1][1] + x[1][2])):
    tf = fl / (ff * 1e-3) / 1e12 if ff else 0
    print(f"{k}: n={n} fwd {ff:8.2f} ms ({tf:5.0f} TF) bwd {bb:8.2f} ms")
print("total", sum(f), sum(b))
