"""Debug: compare every forward feature buffer of a baseline(p) run with the oracle."""
import sys, numpy as np, torch
sys.path.insert(0, ".")
import paper_1602_08124_b200 as V
from oracle import numeric
name = sys.argv[1] if len(sys.argv) > 1 else "alexnet"
g = V.build_preset(name, 8 if name == "alexnet" else 4)
cm = V.CostModel()
w = numeric.he_weights(g, cm)
s0 = g.shape(0)
rng = np.random.default_rng(1234)
images = rng.uniform(-1, 1, size=(s0.n, s0.h, s0.w, s0.c)).astype(np.float32)
li = g.layer(g.size() - 1).inputs[0]
labels = rng.integers(0, g.shape(li).c, size=s0.n).astype(np.int32)
d = V.static_decision(V.PolicyKind.Baseline, V.AlgoMode.PerfOptimal, g, cm)
s = V.Session(g, d, cm, 8 << 30, external_grads=True)
for k, v in w.items():
    s.set_weights(k, v)
s.set_batch(images, labels)
loss = s.step(0.01)
# oracle forward buffers
L = numeric.layers_of(g)
q = numeric.tf32
buf = {}
import torch.nn.functional as Fn
for l in L:
    if l.kind == 0:
        buf[l.id] = torch.tensor(images, dtype=torch.float64)
    elif l.kind == 1:
        k, st, p, co = l.params
        x = torch.cat([buf[numeric.owner(L, qq)] for qq in l.inputs], 3).permute(0, 3, 1, 2)
        ww = torch.tensor(w[l.id], dtype=torch.float64).reshape(co, k, k, x.shape[1]).permute(0, 3, 1, 2)
        buf[l.id] = Fn.conv2d(q(x), q(ww), stride=st, padding=p).permute(0, 2, 3, 1).contiguous()
    elif l.kind == 2:
        o = numeric.owner(L, l.id); buf[o] = torch.relu(buf[o])
    elif l.kind == 3:
        k, st = l.params[0], l.params[1]
        x = torch.cat([buf[numeric.owner(L, qq)] for qq in l.inputs], 3).permute(0, 3, 1, 2)
        buf[l.id] = Fn.max_pool2d(x, k, st).permute(0, 2, 3, 1).contiguous()
    elif l.kind == 4:
        out = l.params[0]
        x = torch.cat([buf[numeric.owner(L, qq)].reshape(s0.n, -1) for qq in l.inputs], 1)
        ww = torch.tensor(w[l.id], dtype=torch.float64)
        fin = x.shape[1]
        buf[l.id] = (q(x) @ q(ww[:out * fin].reshape(out, fin)).t() + ww[out * fin:]).reshape(s0.n, 1, 1, out)
for o, t in buf.items():
    gpu = s.read_feature(o, t.numel()).astype(np.float64)
    ref = t.reshape(-1).numpy()
    err = np.linalg.norm(gpu - ref) / max(np.linalg.norm(ref), 1e-30)
    mx = np.abs(gpu - ref).max()
    print(f"layer {o:3d} kind {L[o].kind} rel-L2 {err:.3e} max-abs {mx:.3e} |ref|max {np.abs(ref).max():.3e}")
print("loss", loss)
