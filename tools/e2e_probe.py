"""Where does the e2e (input copy + loss readback) time go? AlexNet b128 by default.
    python tools/e2e_probe.py [net] [batch]"""
import sys
import time

sys.path.insert(0, ".")
import numpy as np
import torch
import paper_1602_08124_b200 as V

net = sys.argv[1] if len(sys.argv) > 1 else "alexnet"
batch = int(sys.argv[2]) if len(sys.argv) > 2 else 128
g = V.build_preset(net, batch)
cm = V.CostModel()
d = V.static_decision(V.PolicyKind.Baseline, V.AlgoMode.PerfOptimal, g, cm)
s = V.Session(g, d, cm, 8 << 30)
s.synthetic_batch(1)
sh = g.shape(0)
imgs = torch.from_numpy(np.random.default_rng(0).uniform(-1, 1, size=(sh.n, sh.h, sh.w, sh.c)).astype(np.float32)).pin_memory()
labs = torch.zeros(sh.n, dtype=torch.int32).pin_memory()


def run(name, fn, n=20):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(n):
        fn()
    s.synchronize()
    torch.cuda.synchronize()
    print(f"{name:40s} {1e3 * (time.perf_counter() - t0) / n:7.3f} ms/step")


run("step only (no input copy, no loss)", lambda: s.step(0.01, want_loss=False))
run("step + sync loss", lambda: s.step(0.01, want_loss=True))
run("set_batch + step + sync loss", lambda: (s.set_batch_ptr(imgs.data_ptr(), labs.data_ptr()), s.step(0.01, True)))
pend = []
s.prefetch_batch_ptr(imgs.data_ptr(), labs.data_ptr())


def piped():
    s.step(0.01, want_loss=False)
    pend.append(s.queue_loss())
    s.prefetch_batch_ptr(imgs.data_ptr(), labs.data_ptr())
    if len(pend) > 1:
        s.wait_loss(pend.pop(0))


run("prefetch + step + pipelined loss", piped)
