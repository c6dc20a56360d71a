"""Layer-local parity harness (test infrastructure).

Runs training steps of a Session with layer probes armed
(Session.probe_step): every compute step's kernels are checked against the
oracle op (oracle/numeric.layer_forward / layer_backward) evaluated in float64
on the very operands those kernels read, so each FWD / dgrad / wgrad / pool /
loss launch of a full-size BASELINE config is held to a single-contraction
bound instead of a whole-network one.

Ops are sampled only where the float64 oracle would be slow: FWD and dX are
separable per image (the first `nb` images are compared), dW[co] reads only
dY[..., co] (a spread of output channels is compared, each over the whole
batch). The sample sizes come from a FLOP budget per op.
"""
from __future__ import annotations

import math
import os
from typing import Dict, List, Tuple

import numpy as np
import torch

import paper_1602_08124_b200 as V
from oracle import numeric

GFLOP_BUDGET = float(os.environ.get("VDNN_PARITY_GFLOP", "15"))
CAPTURE_BYTES = int(float(os.environ.get("VDNN_PARITY_CAPTURE_GB", "24")) * (1 << 30))


def _reduction(l, L, op: str) -> int:
    """Reduction length K of one output element (cost_model.hpp:100-115 shapes)."""
    n, c_out, ho, wo = l.shape
    cin = sum(L[q].shape[1] for q in l.inputs) if l.join == 0 else L[l.inputs[0]].shape[1]
    if l.kind == numeric.CONV:
        k = l.params[0]
        return {"fprop": k * k * cin, "dgrad": k * k * c_out, "wgrad": n * ho * wo}[op]
    if l.kind == numeric.FC:
        fin = sum(int(np.prod(L[q].shape[1:])) for q in l.inputs) if l.join == 0 else int(np.prod(L[l.inputs[0]].shape[1:]))
        return {"fprop": fin, "dgrad": l.params[0], "wgrad": n}[op]
    return 1


def _sample_batch(l, L) -> int:
    n = l.shape[0]
    per_img = 2.0 * _reduction(l, L, "fprop") * l.shape[1] * l.shape[2] * l.shape[3]
    return max(1, min(n, int(GFLOP_BUDGET * 1e9 // max(per_img, 1.0))))


def _sample_channels(l, L) -> List[int]:
    cout = l.shape[1]
    per_ch = 2.0 * _reduction(l, L, "wgrad") * _reduction(l, L, "fprop")
    m = max(1, min(cout, int(GFLOP_BUDGET * 1e9 // max(per_ch, 1.0))))
    if m >= cout:
        return list(range(cout))
    return sorted(set([0, cout - 1] + [int(round(i * (cout - 1) / max(1, m - 1))) for i in range(m)]))[:max(m, 2)]


def probe_bytes(s: V.Session, layer: int) -> int:
    return sum(s.probe_layout(layer, b)["total_bytes"] for b in (False, True) if _has(s, layer, b))


def _has(s, layer, bwd) -> bool:
    try:
        s.probe_layout(layer, bwd)
        return True
    except V.VdnnError:
        return False


def check_session(s: V.Session, g, labels: np.ndarray, layers: List[int] = None, lr: float = 0.01,
                  precise: bool = False) -> List[Dict]:
    """Probe every (or the listed) layer's FWD and BWD over as many steps as
    the capture budget needs; returns one record per compared tensor:
    {layer, kind, op, tensor, K, err_emu, err_plain}. err_emu compares with the
    oracle that reads contraction operands the way kind::tf32 does (TF32
    mode; equal to err_plain in fp32 mode), err_plain with plain float64.
    bf16 sessions (elem_size 2): the probed operands are exact bf16 values
    and kind::f16 reads them unrounded, so plain float64 is the emulating
    oracle too."""
    L = numeric.layers_of(g)
    todo = [l.id for l in L if l.kind in (numeric.CONV, numeric.FC, numeric.POOL, numeric.LOSS, numeric.ACTV)]
    if layers is not None:
        todo = [i for i in todo if i in layers]
    groups, cur, cur_b = [], [], 0
    for i in todo:
        b = probe_bytes(s, i)
        if cur and cur_b + b > CAPTURE_BYTES:
            groups.append(cur)
            cur, cur_b = [], 0
        cur.append(i)
        cur_b += b
    if cur:
        groups.append(cur)
    recs: List[Dict] = []
    for grp in groups:
        probes = [(i, b) for i in grp for b in (False, True) if _has(s, i, b)]
        _, cap = s.probe_step(probes, lr)
        for (i, bwd), d in cap.items():
            lay = d["_layout"]
            fused = [f for f, on in (("relu", lay["relu_fused"]), ("accumulate", lay["accumulate"]),
                                     ("mask", lay["mask_planes"] != 0)) if on]
            for r in _compare(g, L, i, bwd, d, labels, precise or s.bf16, s.bf16):
                r["fused"] = fused
                recs.append(r)
        del cap
        torch.cuda.empty_cache()
    return recs


def _rec(l, op, tensor, K, e_emu, e_plain):
    kind = {numeric.CONV: "conv", numeric.FC: "fc", numeric.POOL: "pool", numeric.LOSS: "loss",
            numeric.ACTV: "actv"}[l.kind]
    return {"layer": l.id, "kind": kind, "op": op, "tensor": tensor, "K": int(K), "err_emu": float(e_emu),
            "err_plain": float(e_plain)}


def _bf16(t: torch.Tensor) -> torch.Tensor:
    return t.to(torch.float32).to(torch.bfloat16).to(torch.float64)


def _summed_inputs(l, xs, bf16):
    """bf16 sessions store an elementwise join's summed input (rounded once)
    before the kernels read it: hand the oracle that stored sum (the join of
    [sum, 0, ...] is the sum itself)."""
    if not (bf16 and l.join == 1 and len(xs) > 1):
        return xs
    tot = _bf16(sum(x.to(torch.float64) for x in xs))
    return [tot] + [torch.zeros_like(tot) for _ in xs[1:]]


def _compare(g, L, i, bwd, d, labels, precise, bf16=False) -> List[Dict]:
    l = L[i]
    lay = d["_layout"]
    out: List[Dict] = []
    shapes = [L[q].shape for q in l.inputs]
    emu = not precise
    if lay["skip"]:
        return out
    if not bwd:
        if l.kind == numeric.ACTV:
            x = d[("X", 0)]
            y = d[("Y", 0)]
            ref = torch.relu(x.to(torch.float64))
            e = numeric.max_rel(y, ref)
            return [_rec(l, "fwd", "Y", 1, e, e)]
        xs = _summed_inputs(l, [d[("X", j)].reshape(numeric._nhwc(sh)) for j, sh in enumerate(shapes)], bf16)
        w = d.get(("W", 0))
        if l.kind == numeric.LOSS:
            r = numeric.layer_forward(g, i, xs, labels=labels)
            n = xs[0].shape[0]
            e2 = numeric.max_rel(d[("LOSS_GRAD", 0)].reshape(n, -1), r["LOSS_GRAD"])
            out = [_rec(l, "fwd", "LOSS_GRAD", 1, e2, e2)]
            if i == min(x.id for x in L if x.kind == numeric.LOSS):  # later heads add to the loss
                e1 = abs(float(d[("LOSS", 0)][0]) - float(r["LOSS"])) / max(1.0, abs(float(r["LOSS"])))
                out.append(_rec(l, "fwd", "LOSS", 1, e1, e1))
            return out
        nb = _sample_batch(l, L)
        y = d[("Y", 0)].reshape(numeric._nhwc(l.shape))[:nb]
        r_plain = numeric.layer_forward(g, i, xs, w, relu=lay["relu_fused"], batch=nb)["Y"]
        r_emu = numeric.layer_forward(g, i, xs, w, relu=lay["relu_fused"], batch=nb, tf32_operands=True)["Y"] \
            if emu and l.kind in (numeric.CONV, numeric.FC) else r_plain
        K = _reduction(l, L, "fprop")
        out.append(_rec(l, "fprop" if l.kind != numeric.POOL else "pool_fwd", "Y", K,
                        numeric.max_rel(y, r_emu), numeric.max_rel(y, r_plain)))
        return out
    # ---- backward
    if l.kind == numeric.ACTV:
        y = d[("Y", 0)]
        dys = [d[("DY", k)] for k in range(sum(1 for sg in lay["segs"] if sg[0] == "DY"))]
        tot = sum(t.to(torch.float64) for t in dys)
        ref = torch.where(y.to(torch.float64) > 0, tot, torch.zeros_like(tot))
        e = numeric.max_rel(d[("DX", 0)], ref)
        return [_rec(l, "relu_bwd", "DX", len(dys), e, e)]
    if l.kind == numeric.LOSS:
        return out  # copies the FWD's gradient (checked there)
    xs = _summed_inputs(l, [d[("X", j)].reshape(numeric._nhwc(sh)) for j, sh in enumerate(shapes)], bf16)
    ndy = sum(1 for sg in lay["segs"] if sg[0] == "DY")  # > 1: shared planes the kernels read the sum of
    dy = sum(d[("DY", k)].to(torch.float64) for k in range(ndy)).reshape(numeric._nhwc(l.shape))
    if bf16 and ndy > 1:  # the staged sum is stored (rounded once) before the kernels read it
        dy = _bf16(dy)
    w = d.get(("W", 0))
    planes = sorted(k[1] for k in d if isinstance(k, tuple) and k[0] == "DX")
    if l.join == 1 and len(l.inputs) > 1:  # one shared map: every probed DX segment is the same extent
        planes = planes[:1]
    before = {j: d[("DX_BEFORE", j)].reshape(numeric._nhwc(shapes[j])) for j in planes if ("DX_BEFORE", j) in d}
    contraction = l.kind in (numeric.CONV, numeric.FC)
    nb = _sample_batch(l, L)
    co = _sample_channels(l, L) if contraction else None
    want_dw = contraction and ("DW", 0) in d
    r_plain = numeric.layer_backward(g, i, xs, dy, w, mask=lay["mask_planes"], dx_before=before or None,
                                     planes=planes, batch=nb, out_channels=co, want_dw=want_dw)
    r_emu = numeric.layer_backward(g, i, xs, dy, w, mask=lay["mask_planes"], dx_before=before or None,
                                   planes=planes, batch=nb, out_channels=co, want_dw=want_dw,
                                   tf32_operands=True) if emu and contraction else r_plain
    for j in planes:
        gx = d[("DX", j)].reshape(numeric._nhwc(shapes[j]))[:nb]
        op = "dgrad" if contraction else "pool_bwd"
        K = _reduction(l, L, "dgrad") if contraction else 1
        out.append(_rec(l, op, f"DX[{j}]", K, numeric.max_rel(gx, r_emu["DX"][j]),
                        numeric.max_rel(gx, r_plain["DX"][j])))
    if want_dw:
        flat = d[("DW", 0)]
        o = l.shape[1]
        K = _reduction(l, L, "wgrad")
        if l.kind == numeric.CONV:
            gw = flat.reshape(o, -1)[co]
            out.append(_rec(l, "wgrad", "DW", K, numeric.max_rel(gw, r_emu["DW"]), numeric.max_rel(gw, r_plain["DW"])))
        else:
            fin = r_plain["DW"].shape[1]
            gw = flat[: o * fin].reshape(o, fin)[co]
            gb = flat[o * fin:][co]
            out.append(_rec(l, "wgrad", "DW", K, numeric.max_rel(gw, r_emu["DW"]), numeric.max_rel(gw, r_plain["DW"])))
            eb = numeric.max_rel(gb, r_plain["DB"])
            out.append(_rec(l, "bias_grad", "DB", K, eb, eb))
    return out


# Bounds (max |gpu - ref| / max |ref| of each compared tensor).
# TF32 mode (kind::tf32 tensor cores, fp32 accumulation):
#   * against the oracle that reads contraction operands as kind::tf32 does
#     (truncation to 10 mantissa bits), only the fp32 accumulation order
#     differs:                                          TF32_EMU_TOL
#   * against plain float64 (the operand rounding itself): TF32_PLAIN_TOL
# fp32 mode (3xTF32): against plain float64, a bound growing with the
# reduction length K:                                   FP32_TOL(K)
#   (the tensor core's fp32 accumulation is not round-to-nearest and 3xTF32
#   issues three MMAs per K step into one accumulator: measured fprop 2.9e-4
#   at K = 36,864, wgrad 1.0e-3 at K = 802,816 -- about what TF32 mode shows
#   against float64, so 3xTF32 removes the operand rounding, not the
#   accumulation error)
# Memory-bound ops (max-pool, ReLU, loss) compute in fp32 exactly as the
# oracle defines them:                                  EXACT_TOL
# Measured on B200 at the BASELINE sizes (profiles/r02_parity_*.json):
# fprop/dgrad <= 1.5e-5, wgrad <= 2.3e-4 (K = N*Ho*Wo up to 12.8 M, split-K
# partials) against the emulating oracle; <= 1.3e-3 against float64.
TF32_EMU_TOL = {"fprop": 1e-4, "dgrad": 1e-4, "wgrad": 5e-4}
# BF16 storage (elem_size 2): exact products, fp32 accumulation, one
# round-to-nearest-even per stored bf16 value (unit roundoff 2^-8 of the
# element, so at most 2^-8 of max |ref|) -- Y, dX (including overlapping-window
# pool sums), the softmax gradient and summed ReLU-backward planes:
# BF16_STORE_TOL; the fp32 gradient arena (dW, db) is not rounded: BF16_DW_TOL
# (fp32 accumulation over K up to 12.8 M); max-pool forward, a single-plane
# ReLU and the fp32 loss value are exact.
BF16_STORE_TOL = 2.0 ** -8 + 1e-4
BF16_DW_TOL = 5e-4
TF32_PLAIN_TOL = 4e-3
EXACT_TOL = 1e-6


def fp32_tol(K: int) -> float:
    return 4e-6 + 1.2e-8 * K


def violations(recs: List[Dict], precise: bool, bf16: bool = False) -> List[str]:
    bad = []
    if bf16:
        for r in recs:
            if r["tensor"] in ("DW", "DB"):
                tol = BF16_DW_TOL
            elif (r["op"] in ("fprop", "dgrad", "pool_bwd") or r["tensor"] == "LOSS_GRAD"
                  or (r["op"] == "relu_bwd" and r["K"] > 1)):
                tol = BF16_STORE_TOL
            elif r["tensor"] == "LOSS":
                tol = 1e-5
            else:
                tol = EXACT_TOL
            if r["err_plain"] > tol:
                bad.append(f"L{r['layer']} {r['op']} {r['tensor']} K={r['K']}: {r['err_plain']:.3e} > {tol:.2e}")
        return bad
    for r in recs:
        contraction = r["op"] in ("fprop", "dgrad", "wgrad")
        if not contraction:
            tol = EXACT_TOL if r["op"] != "bias_grad" else 1e-5
            if r["err_plain"] > tol:
                bad.append(f"L{r['layer']} {r['op']} {r['tensor']}: {r['err_plain']:.3e} > {tol:.1e}")
            continue
        if precise:
            tol = fp32_tol(r["K"])
            if r["err_plain"] > tol:
                bad.append(f"L{r['layer']} {r['op']} {r['tensor']} K={r['K']}: {r['err_plain']:.3e} > {tol:.2e}")
        else:
            # small contractions may run on fp32-exact SIMT / rounding paths
            # (first layers with C <= 4, tiny wgrad): more accurate than TF32
            # truncation, so they meet the fp32 bound against float64 instead
            if r["err_emu"] > TF32_EMU_TOL[r["op"]] and r["err_plain"] > fp32_tol(r["K"]):
                bad.append(f"L{r['layer']} {r['op']} {r['tensor']} K={r['K']}: vs tf32-operand oracle "
                           f"{r['err_emu']:.3e} > {TF32_EMU_TOL[r['op']]:.1e}")
            if r["err_plain"] > TF32_PLAIN_TOL:
                bad.append(f"L{r['layer']} {r['op']} {r['tensor']} K={r['K']}: vs float64 "
                           f"{r['err_plain']:.3e} > {TF32_PLAIN_TOL:.1e}")
    return bad


def summarize(recs: List[Dict]) -> Dict[str, float]:
    out: Dict[str, float] = {}
    for r in recs:
        k = r["op"]
        out[k + "_emu_max"] = max(out.get(k + "_emu_max", 0.0), r["err_emu"])
        out[k + "_plain_max"] = max(out.get(k + "_plain_max", 0.0), r["err_plain"])
    return out
