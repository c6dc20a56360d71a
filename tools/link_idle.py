"""Where is the host link idle in a vDNN_dyn step? From the measured event
log of one VGG-16 b256 step under 12 GiB: the union of OFFLOAD/PREFETCH
intervals vs the step, and the compute events that run while no transfer
is in flight (the exposed compute):
python tools/link_idle.py [net] [batch] [capacity] [compress: 0 | zvc | tf32]"""
import sys

sys.path.insert(0, ".")
import paper_1602_08124_b200 as V

net = sys.argv[1] if len(sys.argv) > 1 else "vgg16"
batch = int(sys.argv[2]) if len(sys.argv) > 2 else 256
cap = int(sys.argv[3]) if len(sys.argv) > 3 else 12884901888
comp = sys.argv[4] if len(sys.argv) > 4 else "0"
comp = {"0": False, "zvc": True, "tf32": "tf32"}[comp]
g = V.build_preset(net, batch)
cm = V.CostModel()
d = V.dynamic_select(g, cap, cm).decision
s = V.Session(g, d, cm, cap, record_timeline=True, compress_offload=comp)
s.synthetic_batch(1)
for _ in range(3):
    s.step(0.01, want_loss=False)
s.step(0.01, want_loss=True)
m = s.measured_report()
xfer = sorted([(e.start, e.end) for e in m.events if e.kind in (V.EventKind.Offload, V.EventKind.Prefetch)])
comp = sorted([e for e in m.events if e.kind in (V.EventKind.Fwd, V.EventKind.Bwd)], key=lambda e: e.start)
busy = []
for a, b in xfer:
    if busy and a <= busy[-1][1]:
        busy[-1][1] = max(busy[-1][1], b)
    else:
        busy.append([a, b])
t_end = max(e.end for e in m.events)
link = sum(b - a for a, b in busy)
print(f"step {t_end / 1e6:.1f} ms, link busy {link / 1e6:.1f} ms, idle {(t_end - link) / 1e6:.1f} ms")
exposed = []
for e in comp:
    ov = sum(max(0, min(e.end, b) - max(e.start, a)) for a, b in busy)
    ex = (e.end - e.start) - ov
    if ex > 50_000:
        exposed.append((ex, e))
for ex, e in sorted(exposed, key=lambda t: -t[0])[:15]:
    print(f"  {str(e.kind).split('.')[-1]:4s} layer {e.layer:3d} {g.layer(e.layer).kind.name:5s} exposed {ex / 1e6:6.2f} ms of {(e.end - e.start) / 1e6:6.2f}")
print(f"exposed compute total {sum(x for x, _ in exposed) / 1e6:.1f} ms")
