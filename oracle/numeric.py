"""ORACLE ONLY: CPU restatement of one training iteration as the executor runs it.

The reference (vdnnsim) computes no values -- "numerical gradient computation
is OUT of scope" -- so numeric parity is
*unpinned by the reference*; this module restates the dataflow the reference
fixes (simulator.hpp:90-131, footprint.hpp:58-71, net_graph.hpp:384-389) with
standard definitions, in float64 on the CPU:

* buffers are per feature-buffer owner; ACTV (ReLU) is applied *in place* on
  the owner's buffer, and its backward masks the incoming gradient by
  (owner buffer > 0) -- the same aliasing the reference's buffer model has;
* CONV has no bias; FC has a bias stored after its [out][in] weights;
  activations are NHWC, conv weights KRSC, FC input features are flattened
  per input segment in (h, w, c) order and concatenated in input order;
* no gradient w.r.t. the raw INPUT; concat-join gradients are split into
  per-input planes; gradients arriving at a fork are summed;
* max-pool is floor mode, no padding, first maximum wins ties;
* LOSS = mean softmax cross-entropy; plain SGD w -= lr * dW.

Only tests/, __graft_entry__.smoke() and bench.py's reference arm use this.
"""
from __future__ import annotations

from typing import Dict, List, Tuple

import numpy as np
import torch
import torch.nn.functional as Fn

INPUT, CONV, ACTV, POOL, FC, LOSS = range(6)


class Layer:
    def __init__(self, id, kind, inputs, params, shape, join=0):
        self.id, self.kind, self.inputs, self.params, self.shape = id, kind, list(inputs), params, shape
        self.join = join  # 0 = concat, 1 = elementwise sum


def layers_of(g) -> List[Layer]:
    """From a paper_1602_08124_b200.NetworkGraph (finalized), a graph spec
    string ("B=<batch>|<kind> <inputs> p0 p1 p2 p3 <join>|...", the format of
    oracle/refsim.preset_spec), or an already converted layer list."""
    if isinstance(g, str):
        return layers_from_spec(g)
    if isinstance(g, list):
        return g
    out = []
    for l in g.layers():
        s = g.shape(l.id)
        out.append(Layer(l.id, int(l.kind), l.inputs, l.params, (s.n, s.c, s.h, s.w), int(l.join)))
    return out


_KINDS = {"input": INPUT, "conv": CONV, "actv": ACTV, "pool": POOL, "fc": FC, "loss": LOSS}


def layers_from_spec(spec: str) -> List[Layer]:
    """Graph spec -> layers with inferred NCHW shapes (net_graph.hpp:299-358:
    conv (h + 2p - k)/s + 1, pool floor without padding, concat sums C,
    elementwise keeps the shape, FC -> (n, out, 1, 1), LOSS -> (n, 1, 1, 1)).
    Lets the reference arm build its graphs without the product library."""
    parts = spec.split("|")
    batch = int(parts[0].split("=")[1])
    out: List[Layer] = []
    for i, p in enumerate(parts[1:]):
        kind_s, ins_s, a, b, c, d, j = p.split()
        kind = _KINDS[kind_s]
        ins = [] if ins_s == "-" else [int(x) for x in ins_s.split(",")]
        prm = (int(a), int(b), int(c), int(d))
        join = int(j)
        if kind == INPUT:
            shape = (batch, prm[0], prm[1], prm[2])
        else:
            n, ch, h, w = out[ins[0]].shape
            for q in ins[1:]:
                if join == 0:
                    ch += out[q].shape[1]
            if kind == CONV:
                k, s, pad, cout = prm
                shape = (n, cout, (h + 2 * pad - k) // s + 1, (w + 2 * pad - k) // s + 1)
            elif kind == POOL:
                k, s = prm[0], prm[1]
                shape = (n, ch, (h - k) // s + 1, (w - k) // s + 1)
            elif kind == FC:
                shape = (n, prm[0], 1, 1)
            elif kind == LOSS:
                shape = (n, 1, 1, 1)
            else:
                shape = out[ins[0]].shape
        out.append(Layer(i, kind, ins, prm, shape, join))
    return out


def owner(L: List[Layer], i: int) -> int:
    while L[i].kind == ACTV:
        i = L[i].inputs[0]
    return i


def _nhwc(shape):
    n, c, h, w = shape
    return (n, h, w, c)


def tf32(t: torch.Tensor) -> torch.Tensor:
    """Emulate the tensor core's kind::tf32 operand read: keep the top 19 bits
    (sign, 8-bit exponent, 10-bit mantissa) of each fp32 value (truncation)."""
    i = t.to(torch.float32).contiguous().view(torch.int32)
    return (i & ~0x1FFF).view(torch.float32).to(t.dtype)


def train_step(g, weights: Dict[int, np.ndarray], images: np.ndarray, labels: np.ndarray, lr: float,
               dtype=torch.float64, tf32_operands: bool = False, device: str = "cpu"
               ) -> Tuple[float, Dict[int, np.ndarray], Dict[int, np.ndarray]]:
    """Returns (loss, updated weights, weight gradients).

    device="cuda" evaluates the same float64 restatement with torch on the GPU
    (test infrastructure for network sizes the CPU cannot finish quickly).

    tf32_operands=True rounds both operands of every conv/FC contraction the
    way kind::tf32 reads them (fp32 values stay fp32 between layers); this is
    the tight-tolerance oracle for the tensor-core path."""
    q = tf32 if tf32_operands else (lambda t: t)
    L = layers_of(g)
    N = len(L)
    buf: Dict[int, torch.Tensor] = {}
    W = {k: torch.tensor(v, dtype=dtype, device=device) for k, v in weights.items()}
    grads: Dict[int, torch.Tensor] = {}

    def cat_in(l: Layer, flatten: bool = False):
        parts = []
        for q in l.inputs:
            t = buf[owner(L, q)]
            parts.append(t.reshape(t.shape[0], -1) if flatten else t)
        if l.join == 1 and len(parts) > 1:  # elementwise join: sum (net_graph.hpp:290-296)
            out = parts[0]
            for t in parts[1:]:
                out = out + t
            return out
        return torch.cat(parts, dim=1 if flatten else 3)

    def in_channels(l: Layer, flatten: bool = False):
        cs = []
        for q in l.inputs:
            n, c, h, w = L[q].shape
            cs.append(c * h * w if flatten else c)
        return cs

    # ---------------- forward
    gscratch = None
    loss = 0.0
    for l in L:
        if l.kind == INPUT:  # several INPUT layers: images = {layer id: array}
            im = images[l.id] if isinstance(images, dict) else images
            buf[l.id] = torch.tensor(im, dtype=dtype, device=device).reshape(_nhwc(l.shape))
        elif l.kind == CONV:
            k, s, p, cout = l.params
            x = cat_in(l).permute(0, 3, 1, 2)
            cin = x.shape[1]
            w = W[l.id].reshape(cout, k, k, cin).permute(0, 3, 1, 2)
            buf[l.id] = Fn.conv2d(q(x), q(w), stride=s, padding=p).permute(0, 2, 3, 1).contiguous()
        elif l.kind == ACTV:
            o = owner(L, l.id)
            buf[o] = torch.relu(buf[o])
        elif l.kind == POOL:
            k, s = l.params[0], l.params[1]
            x = cat_in(l).permute(0, 3, 1, 2)
            buf[l.id] = Fn.max_pool2d(x, k, s).permute(0, 2, 3, 1).contiguous()
        elif l.kind == FC:
            out = l.params[0]
            x = cat_in(l, flatten=True)
            fin = x.shape[1]
            w = W[l.id][: out * fin].reshape(out, fin)
            b = W[l.id][out * fin:]
            buf[l.id] = (q(x) @ q(w).t() + b).reshape(_nhwc(l.shape))
        elif l.kind == LOSS:
            # several LOSS heads: the loss is their sum; each head reads the
            # shared label vector modulo its class count
            z = buf[owner(L, l.inputs[0])].reshape(l.shape[0], -1)
            lab = torch.tensor(labels, dtype=torch.long, device=device) % z.shape[1]
            lse = torch.logsumexp(z, dim=1)
            loss += float((lse - z[torch.arange(z.shape[0], device=z.device), lab]).mean())
            pr = torch.softmax(z, dim=1)
            oh = torch.zeros_like(pr)
            oh[torch.arange(z.shape[0], device=z.device), lab] = 1.0
            if gscratch is None:
                gscratch = {}
            gscratch[l.id] = (pr - oh) / z.shape[0]

    # ---------------- backward
    def produces(l: Layer) -> bool:
        if l.kind in (ACTV, INPUT):
            return False
        return any(L[owner(L, q)].kind != INPUT for q in l.inputs)

    planes: Dict[Tuple[int, int], torch.Tensor] = {}
    merged: Dict[Tuple[int, int], Tuple[int, int]] = {}

    def canon(key):
        while key in merged:
            key = merged[key]
        return key

    def readers_of(gid: int):
        # grads_read: gradient buffers whose input chains pass through m
        return gid

    def incoming(m: int):
        keys = []
        for gid in range(N):
            gl = L[gid]
            if not produces(gl):
                continue
            for j, q in enumerate(gl.inputs):
                if L[owner(L, q)].kind == INPUT:
                    continue
                cur = q
                hit = False
                while True:
                    if cur == m:
                        hit = True
                        break
                    if L[cur].kind != ACTV:
                        break
                    cur = L[cur].inputs[0]
                if hit:
                    c = canon((gid, j))
                    if c not in keys:
                        keys.append(c)
        return keys

    def set_planes(l: Layer, full: torch.Tensor, flatten: bool):
        """Split a gradient w.r.t. the concatenated input into per-input planes
        (elementwise join: every input receives the whole gradient)."""
        off = 0
        cs = in_channels(l, flatten)
        for j, q in enumerate(l.inputs):
            c = cs[j]
            if l.join == 1 and len(l.inputs) > 1:
                if L[owner(L, q)].kind != INPUT:
                    planes[(l.id, j)] = full.reshape(_nhwc(L[q].shape)).contiguous()
                continue
            if L[owner(L, q)].kind != INPUT:
                part = full[:, off:off + c] if flatten else full[..., off:off + c]
                planes[(l.id, j)] = part.reshape(_nhwc(L[q].shape)).contiguous()
            off += c

    for m in range(N - 1, -1, -1):
        l = L[m]
        if l.kind == INPUT:
            continue
        keys = incoming(m)
        dy = None
        if keys:
            dy = planes[keys[0]]
            if len(keys) > 1:
                for k2 in keys[1:]:
                    dy = dy + planes[k2]
                    merged[k2] = keys[0]
                planes[keys[0]] = dy
        if l.kind == LOSS:
            if produces(l):
                planes[(m, 0)] = gscratch[m].reshape(_nhwc(L[l.inputs[0]].shape)).clone()
        elif l.kind == ACTV:
            if dy is None:  # nothing downstream needs this map's gradient
                continue
            y = buf[owner(L, m)]
            planes[keys[0]] = torch.where(y > 0, dy, torch.zeros_like(dy))
        elif l.kind == CONV:
            k, s, p, cout = l.params
            x = cat_in(l).permute(0, 3, 1, 2)
            cin = x.shape[1]
            w4 = W[m].reshape(cout, k, k, cin).permute(0, 3, 1, 2)
            dyn = dy.permute(0, 3, 1, 2)
            if produces(l):
                dx = torch.nn.grad.conv2d_input(x.shape, q(w4), q(dyn), stride=s, padding=p)
                set_planes(l, dx.permute(0, 2, 3, 1), False)
            dw = torch.nn.grad.conv2d_weight(q(x), w4.shape, q(dyn), stride=s, padding=p)
            gk = dw.permute(0, 2, 3, 1).reshape(-1)
            grads[m] = gk
            W[m] = W[m] - lr * gk
        elif l.kind == FC:
            out = l.params[0]
            x = cat_in(l, flatten=True)
            fin = x.shape[1]
            w = W[m][: out * fin].reshape(out, fin)
            d2 = dy.reshape(dy.shape[0], -1)
            if produces(l):
                set_planes(l, q(d2) @ q(w), True)
            dw = q(d2).t() @ q(x)
            db = d2.sum(0)
            gk = torch.cat([dw.reshape(-1), db])
            grads[m] = gk
            W[m] = W[m] - lr * gk
        elif l.kind == POOL:
            k, s = l.params[0], l.params[1]
            x = cat_in(l).permute(0, 3, 1, 2).detach().requires_grad_(True)
            y = Fn.max_pool2d(x, k, s)
            y.backward(dy.permute(0, 3, 1, 2))
            if produces(l):
                set_planes(l, x.grad.permute(0, 2, 3, 1), False)
    return (loss, {k: v.cpu().numpy().astype(np.float32) for k, v in W.items()},
            {k: v.cpu().numpy() for k, v in grads.items()})


def he_weights(g, cost=None, seed: int = 5000) -> Dict[int, np.ndarray]:
    """Host-side He-normal init (numpy), for tests that upload weights."""
    rng = np.random.default_rng(seed)
    L = layers_of(g)
    out = {}
    for l in L:
        if l.kind == CONV:
            k, s, p, cout = l.params
            cs = [L[q].shape[1] for q in l.inputs]
            cin = cs[0] if l.join == 1 else sum(cs)
            fan = k * k * cin
            out[l.id] = (rng.standard_normal(cout * k * k * cin) * np.sqrt(2.0 / fan)).astype(np.float32)
        elif l.kind == FC:
            outf = l.params[0]
            fs = [int(np.prod(L[q].shape[1:])) for q in l.inputs]
            fin = fs[0] if l.join == 1 else sum(fs)
            w = (rng.standard_normal(outf * fin) * np.sqrt(2.0 / fin)).astype(np.float32)
            out[l.id] = np.concatenate([w, np.zeros(outf, np.float32)])
    return out


# ------------------------------------------------------------------------------
# Layer-local ops (ORACLE ONLY): one layer's FWD or BWD evaluated on the very
# operands a B200 step's kernels read (Session.probe_step), so every kernel is
# checked at the single-contraction bound instead of through a whole network.
# Same definitions as train_step above; the dataflow of each op follows
# simulator.hpp:90-131 (operands: CONV/FC read X, POOL reads X (+Y), ACTV its
# aliased Y) and footprint.hpp:60-71 (one gradient plane per non-INPUT input;
# an elementwise join shares one plane).
# ------------------------------------------------------------------------------

def _join(l: Layer, xs: List[torch.Tensor], flatten: bool) -> torch.Tensor:
    parts = [x.reshape(x.shape[0], -1) if flatten else x for x in xs]
    if l.join == 1 and len(parts) > 1:  # elementwise: sum
        out = parts[0]
        for p in parts[1:]:
            out = out + p
        return out
    return torch.cat(parts, dim=1 if flatten else 3)


def _split(l: Layer, L: List[Layer], full: torch.Tensor, flatten: bool) -> List[torch.Tensor]:
    """Gradient w.r.t. the joined input -> per-input planes (elementwise: the
    same gradient for every input)."""
    out, off = [], 0
    for q in l.inputs:
        n, c, h, w = L[q].shape
        shape = (full.shape[0], h, w, c)  # the batch may be a leading sample
        if l.join == 1 and len(l.inputs) > 1:
            out.append(full.reshape(shape))
            continue
        cc = c * h * w if flatten else c
        part = full[:, off:off + cc] if flatten else full[..., off:off + cc]
        out.append(part.reshape(shape))
        off += cc
    return out


def layer_forward(g, layer: int, xs: List[torch.Tensor], w: torch.Tensor = None, relu: bool = False,
                  labels=None, tf32_operands: bool = False, batch: int = None, dtype=torch.float64):
    """FWD of one layer. xs: its inputs as NHWC tensors (any float dtype, any
    device); w: flat weights (KRSC conv, [out][in]+bias FC). relu: the next
    ACTV's ReLU fused into the epilogue. batch: evaluate only the first
    `batch` images (every FWD op is separable per image). Returns
    {"Y": NHWC} or, for LOSS, {"LOSS": scalar, "LOSS_GRAD": [N, classes]}."""
    L = layers_of(g)
    l = L[layer]
    q = tf32 if tf32_operands else (lambda t: t)
    xs = [x.to(dtype) for x in xs]
    if batch is not None:
        xs = [x[:batch] for x in xs]
    if l.kind == CONV:
        k, s, p, cout = l.params
        x = _join(l, xs, False).permute(0, 3, 1, 2)
        w4 = w.to(dtype).reshape(cout, k, k, x.shape[1]).permute(0, 3, 1, 2)
        y = Fn.conv2d(q(x), q(w4), stride=s, padding=p).permute(0, 2, 3, 1)
    elif l.kind == FC:
        out = l.params[0]
        x = _join(l, xs, True)
        fin = x.shape[1]
        wd = w.to(dtype)
        y = (q(x) @ q(wd[: out * fin].reshape(out, fin)).t() + wd[out * fin:]).reshape(x.shape[0], 1, 1, out)
    elif l.kind == POOL:
        k, s = l.params[0], l.params[1]
        y = Fn.max_pool2d(_join(l, xs, False).permute(0, 3, 1, 2), k, s).permute(0, 2, 3, 1)
    elif l.kind == ACTV:
        y = xs[0]
    elif l.kind == LOSS:
        z = xs[0].reshape(xs[0].shape[0], -1)
        lab = torch.as_tensor(labels, dtype=torch.long, device=z.device)[: z.shape[0]] % z.shape[1]
        idx = torch.arange(z.shape[0], device=z.device)
        loss = (torch.logsumexp(z, dim=1) - z[idx, lab]).mean()
        pr = torch.softmax(z, dim=1)
        pr[idx, lab] -= 1.0
        return {"LOSS": loss, "LOSS_GRAD": pr / z.shape[0]}
    else:
        raise ValueError("layer has no FWD op")
    if relu or l.kind == ACTV:
        y = torch.relu(y)
    return {"Y": y.contiguous()}


def layer_backward(g, layer: int, xs: List[torch.Tensor], dy: torch.Tensor, w: torch.Tensor = None,
                   mask: int = 0, dx_before: Dict[int, torch.Tensor] = None, planes=None,
                   tf32_operands: bool = False, batch: int = None, out_channels=None,
                   want_dw: bool = True, dtype=torch.float64):
    """BWD of one layer on the operands its kernels read. dy: incoming gradient
    (NHWC, the fold of every incoming plane); mask bit i: dX[i] *= (X[i] > 0)
    (the producer's ReLU backward fused into this epilogue); dx_before[i]:
    plane contents before an accumulating (two-buffer) write; planes: input
    slots that have a plane (default: every input). batch: dX of the first
    `batch` images only (separable per image); out_channels: dW rows to
    evaluate (dW[co] reads only dY[..., co] -- over the whole batch).
    Returns {"DX": {i: NHWC}, "DW": flat KRSC / [out][in]+bias rows}."""
    L = layers_of(g)
    l = L[layer]
    q = tf32 if tf32_operands else (lambda t: t)
    xs = [x.to(dtype) for x in xs]
    dy = dy.to(dtype)
    planes = list(range(len(l.inputs))) if planes is None else planes
    out = {"DX": {}}
    xb = [x[:batch] for x in xs] if batch is not None else xs
    dyb = dy[:batch] if batch is not None else dy
    if l.kind == CONV:
        k, s, p, cout = l.params
        x = _join(l, xb, False).permute(0, 3, 1, 2)
        cin = x.shape[1]
        w4 = w.to(dtype).reshape(cout, k, k, cin).permute(0, 3, 1, 2)
        if planes:
            full = torch.nn.grad.conv2d_input(x.shape, q(w4), q(dyb.permute(0, 3, 1, 2)), stride=s, padding=p)
            split = _split(l, L, full.permute(0, 2, 3, 1), False)
            for i in planes:
                out["DX"][i] = split[i]
        if want_dw:
            co = list(range(cout)) if out_channels is None else list(out_channels)
            xa = _join(l, xs, False).permute(0, 3, 1, 2)
            dya = dy.permute(0, 3, 1, 2)[:, co]
            dw = torch.nn.grad.conv2d_weight(q(xa), (len(co), cin, k, k), q(dya), stride=s, padding=p)
            out["DW"] = dw.permute(0, 2, 3, 1).reshape(len(co), -1)  # rows = selected output channels
            out["DW_rows"] = co
    elif l.kind == FC:
        o = l.params[0]
        d2 = dyb.reshape(dyb.shape[0], -1)
        xa = _join(l, xs, True)
        fin = xa.shape[1]
        wd = w.to(dtype)[: o * fin].reshape(o, fin)
        if planes:
            split = _split(l, L, q(d2) @ q(wd), True)
            for i in planes:
                out["DX"][i] = split[i]
        if want_dw:
            co = list(range(o)) if out_channels is None else list(out_channels)
            dfull = dy.reshape(dy.shape[0], -1)[:, co]
            out["DW"] = q(dfull).t() @ q(xa)
            out["DB"] = dfull.sum(0)
            out["DW_rows"] = co
    elif l.kind == POOL:
        k, s = l.params[0], l.params[1]
        x = _join(l, xb, False).permute(0, 3, 1, 2).detach().requires_grad_(True)
        Fn.max_pool2d(x, k, s).backward(dyb.permute(0, 3, 1, 2))
        split = _split(l, L, x.grad.permute(0, 2, 3, 1), False)
        for i in planes:
            out["DX"][i] = split[i]
    else:
        raise ValueError("layer has no BWD contraction/pool op")
    for i in list(out["DX"].keys()):
        d = out["DX"][i]
        if mask >> i & 1:
            d = torch.where(xb[i] > 0, d, torch.zeros_like(d))
        if dx_before is not None and i in dx_before:
            b = dx_before[i].to(dtype)
            d = d + (b[:batch] if batch is not None else b)
        out["DX"][i] = d.contiguous()
    return out


def max_rel(gpu: torch.Tensor, ref: torch.Tensor) -> float:
    """max |gpu - ref| / max |ref| (0 when both are all zero)."""
    ref = ref.to(torch.float64)
    d = (gpu.to(torch.float64).reshape(ref.shape) - ref).abs().max().item()
    m = ref.abs().max().item()
    return d / m if m > 0 else d
