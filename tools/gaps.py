"""Where does GPU time go between layer kernels? Prints the measured
FWD/BWD event intervals of one no-offload step and the idle gaps between
consecutive compute events: python tools/gaps.py [net] [batch]"""
import sys

sys.path.insert(0, ".")
import paper_1602_08124_b200 as V

net = sys.argv[1] if len(sys.argv) > 1 else "vgg16"
batch = int(sys.argv[2]) if len(sys.argv) > 2 else 256
g = V.build_preset(net, batch)
cm = V.CostModel()
d = V.static_decision(V.PolicyKind.Baseline, V.AlgoMode.PerfOptimal, g, cm)
s = V.Session(g, d, cm, 150 << 30, record_timeline=True)
s.synthetic_batch(1)
for _ in range(4):
    s.step(0.01, want_loss=False)
s.step(0.01, want_loss=True)
m = s.measured_report()
ev = sorted([e for e in m.events if e.kind in (V.EventKind.Fwd, V.EventKind.Bwd)], key=lambda e: e.start)
busy = sum(e.end - e.start for e in ev)
print(f"total {m.total_ns / 1e6:.2f} ms, compute events {busy / 1e6:.2f} ms, first start {ev[0].start / 1e6:.3f} ms")
gaps = []
for a, b in zip(ev, ev[1:]):
    gaps.append((b.start - a.end, a, b))
print(f"sum of gaps {sum(x[0] for x in gaps) / 1e6:.2f} ms over {len(gaps)} boundaries")
for gap, a, b in sorted(gaps, key=lambda x: -x[0])[:12]:
    print(f"  gap {gap / 1e3:8.1f} us after {a.kind.name} {a.layer:3d} before {b.kind.name} {b.layer:3d}")
