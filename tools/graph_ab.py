"""Step time of the small BASELINE nets (no-offload and vDNN_all) with and
without CUDA-graph replay and per-op timeline events:
python tools/graph_ab.py [net] [batch]"""
import sys

import torch

sys.path.insert(0, ".")
import paper_1602_08124_b200 as V

net = sys.argv[1] if len(sys.argv) > 1 else "inception_toy"
batch = int(sys.argv[2]) if len(sys.argv) > 2 else 128
g = V.build_preset(net, batch)
cm = V.CostModel()
for pol in ("none", "all"):
    if pol == "none":
        d = V.static_decision(V.PolicyKind.Baseline, V.AlgoMode.PerfOptimal, g, cm)
    else:
        d = V.static_decision(V.PolicyKind.VdnnAll, V.AlgoMode.MemoryOptimal, g, cm)
    for rep in range(2):
        for graph in (False, True):
            for timeline in (False, True):
                s = V.Session(g, d, cm, 12884901888, record_timeline=timeline, cuda_graph=graph)
                st = torch.cuda.ExternalStream(s.stream)
                s.synthetic_batch(3)
                for _ in range(5):
                    s.step(0.01, want_loss=False)
                s.synchronize()
                a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                a.record(st)
                n = 30
                for _ in range(n):
                    s.step(0.01, want_loss=False)
                b.record(st)
                b.synchronize()
                ms = a.elapsed_time(b) / n
                print(f"{net} b{batch} {pol:4s} graph={int(graph)} timeline={int(timeline)}: {ms:.3f} ms/step "
                      f"({batch / ms * 1e3:,.0f} img/s)")
                del s
