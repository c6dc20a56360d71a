"""Statistics of the feature maps vDNN_dyn offloads (VGG-16, batch 32): zero
fraction and, for nonzeros, how many distinct top bytes (sign + 7 exponent
bits) a 1024-value chunk holds -- what a denser lossless format could gain."""
import sys

sys.path.insert(0, ".")
import numpy as np
import paper_1602_08124_b200 as V

g = V.build_preset("vgg16", 32)
cm = V.CostModel()
d = V.static_decision(V.PolicyKind.Baseline, V.AlgoMode.PerfOptimal, g, cm)
s = V.Session(g, d, cm, 16 << 30)
s.synthetic_batch(3)
for _ in range(3):
    s.step(0.01)
s.step(0.01)
tot_raw = tot_zvc = tot_nib = 0
for l in g.layers():
    if l.kind not in (V.LayerKind.Conv, V.LayerKind.Pool):
        continue
    sh = g.shape(l.id)
    n = sh.n * sh.c * sh.h * sh.w
    x = s.read_feature(l.id, n)
    u = x.view(np.uint32)
    nz = u != 0
    chunks = u[: n // 1024 * 1024].reshape(-1, 1024)
    nzc = chunks != 0
    top = (chunks >> 24).astype(np.int32)
    rng = np.where(nzc, top, 255).min(axis=1), np.where(nzc, top, -1).max(axis=1)
    span = np.maximum(rng[1] - rng[0], 0)
    nnz = nzc.sum(axis=1)
    zvc = 128 + 4 * nnz
    nib = np.where(span <= 15, 128 + 4 + (3.5 * nnz), zvc)
    tot_raw += 4 * chunks.size
    tot_zvc += zvc.sum()
    tot_nib += nib.sum()
    print(f"L{l.id:2d} {'pool' if l.kind == V.LayerKind.Pool else 'conv'} {sh.c:4d}x{sh.h:3d}: zeros {1 - nz.mean():.3f}  chunks with top-byte span<=15: "
          f"{(span <= 15).mean():.3f}  zvc {zvc.sum() / (4 * chunks.size):.3f}  +nibble {nib.sum() / (4 * chunks.size):.3f}")
print(f"all conv outputs: zvc {tot_zvc / tot_raw:.3f}  zvc+nibble {tot_nib / tot_raw:.3f}")
