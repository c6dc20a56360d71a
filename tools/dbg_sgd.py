import sys
sys.path.insert(0, ".")
import numpy as np
import paper_1602_08124_b200 as V
from oracle import numeric
net, batch = (sys.argv[1], int(sys.argv[2])) if len(sys.argv) > 2 else ("alexnet", 16)
g = V.build_preset(net, batch)
cm = V.CostModel(); cm.elem_size = 2
d = V.static_decision(V.PolicyKind.Baseline, V.AlgoMode.PerfOptimal, g, cm)
w = numeric.he_weights(g, cm, seed=21)
rng = np.random.default_rng(22)
sh = g.shape(0)
images = rng.uniform(-1, 1, size=(batch, sh.h, sh.w, sh.c)).astype(np.float32)
labels = rng.integers(0, 10, size=batch).astype(np.int32)
lr = 0.05
def session(ext):
    s = V.Session(g, d, cm, 8 << 30, external_grads=ext)
    for k, v in w.items(): s.set_weights(k, v)
    s.set_batch(images, labels); s.step(lr); return s
a = session(True); grads = {k: a.get_grads(k) for k in w}; before = {k: a.get_weights(k) for k in w}; del a
b = session(False)
for k in w:
    got = b.get_weights(k)
    want = V.from_bf16_bits(V.to_bf16_bits(before[k] - np.float32(lr) * grads[k]))
    u = np.abs(V.to_bf16_bits(want).astype(np.int64) - V.to_bf16_bits(got).astype(np.int64))
    bad = np.nonzero(u > 1)[0]
    impl = (before[k] - got) / lr
    print(k, g.layer(k).kind, w[k].size, "max ulp", u.max(), "n>1", bad.size, "n>0", int((u > 0).sum()),
          "| dW rel err (implied vs ext)", float(np.linalg.norm(impl - grads[k]) / max(np.linalg.norm(grads[k]), 1e-30)))
    if bad.size:
        i = bad[:5]
        print("   idx", i, "before", before[k][i], "grad", grads[k][i], "got", got[i], "want", want[i])
