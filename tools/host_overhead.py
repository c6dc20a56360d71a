"""Host enqueue cost of one training step vs its GPU time (is the executor
launch-bound?): python tools/host_overhead.py [net] [batch] [policy]"""
import sys
import time

sys.path.insert(0, ".")
import torch
import paper_1602_08124_b200 as V

net = sys.argv[1] if len(sys.argv) > 1 else "vgg16"
batch = int(sys.argv[2]) if len(sys.argv) > 2 else 256
policy = sys.argv[3] if len(sys.argv) > 3 else "none"
g = V.build_preset(net, batch)
cm = V.CostModel()
if policy == "none":
    d, cap = V.static_decision(V.PolicyKind.Baseline, V.AlgoMode.PerfOptimal, g, cm), 150 << 30
else:
    d, cap = V.dynamic_select(g, 12884901888, cm).decision, 12884901888
for rec in (False, True):
    s = V.Session(g, d, cm, cap, record_timeline=rec)
    s.synthetic_batch(1)
    for _ in range(3):
        s.step(0.01, want_loss=False)
    s.synchronize()
    host = []
    t0 = time.perf_counter()
    for _ in range(10):
        a = time.perf_counter()
        s.step(0.01, want_loss=False)
        host.append(time.perf_counter() - a)
    s.synchronize()
    wall = (time.perf_counter() - t0) / 10
    print(f"record_timeline={rec}: host enqueue per step {1e3 * sum(host) / len(host):.2f} ms "
          f"(max {1e3 * max(host):.2f}), wall per step {1e3 * wall:.2f} ms, launches/step "
          f"{V.kernel_launch_count()}")
    del s
