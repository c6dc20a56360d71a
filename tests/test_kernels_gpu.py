"""Kernel-level parity: tcgen05 conv/FC contractions and memory-bound kernels
versus a float64 CPU reference of the same op (torch functional ops).

Tolerance: the tensor-core path is kind::tf32 (10-bit mantissa inputs, fp32
accumulate): max abs error <= 4e-3 * max |reference| of the output. In
precise mode (3xTF32, fp32-accurate products) the bound is
(4e-6 + 1.2e-8 * K) * max |reference|, K the reduction length. Memory-bound
kernels are exact (bit-equal) except softmax (1e-4 relative on the gradient).
"""
import ctypes as C

import numpy as np
import pytest

torch = pytest.importorskip("torch")

from paper_1602_08124_b200 import _lib as L

pytestmark = pytest.mark.gpu
TF32_TOL = 4e-3


def _dev():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    return torch.device("cuda:0")


def _desc(n, h, w, xs, cs, cout, k, stride, pad, dxs=None):
    d = L.ConvDesc()
    d.n, d.h, d.w, d.nseg = n, h, w, len(cs)
    for i, c in enumerate(cs):
        d.x[i] = xs[i].data_ptr() if xs is not None and xs[i] is not None else None
        d.dx[i] = dxs[i].data_ptr() if dxs is not None and dxs[i] is not None else None
        d.c[i] = c
    d.cout, d.kh, d.kw, d.stride, d.pad = cout, k, k, stride, pad
    return d


def _ref_conv(x_nhwc_list, w_krsc, stride, pad):
    x = torch.cat([t.double().cpu() for t in x_nhwc_list], dim=3).permute(0, 3, 1, 2)
    w = w_krsc.double().cpu().permute(0, 3, 1, 2)
    x.requires_grad_(True)
    w.requires_grad_(True)
    y = torch.nn.functional.conv2d(x, w, stride=stride, padding=pad)
    return x, w, y


def _close(a, b, tol=None):
    tol = TF32_TOL if tol is None else tol
    a = a.double().cpu()
    b = b.double().cpu()
    scale = max(b.abs().max().item(), 1e-30)
    err = (a - b).abs().max().item() / scale
    print(f"  rel err {err:.3e}")
    assert err < tol, f"max rel err {err:.3e} (scale {scale:.3e})"


CASES = [
    # n, h, w, segs, cout, k, stride, pad
    (2, 14, 14, [64], 128, 3, 1, 1),
    (2, 9, 9, [32, 32, 16], 64, 3, 1, 1),     # concat join, partial chunk
    (3, 35, 35, [3], 64, 11, 4, 0),           # AlexNet-style first layer (scalar K)
    (2, 8, 8, [5, 3], 7, 3, 1, 1),            # odd channels everywhere (scalar paths)
    (4, 7, 7, [256], 96, 1, 1, 0),            # 1x1
    (5, 1, 1, [300], 40, 1, 1, 0),            # FC as 1x1 over a 1x1 image
    (2, 12, 12, [8], 300, 5, 1, 2),           # Cout > tile N
    (8, 1, 1, [9216], 4096, 1, 1, 0),         # AlexNet FC6 as 1x1
    (8, 1, 1, [4096], 1000, 1, 1, 0),         # AlexNet FC8 as 1x1
    (2, 27, 27, [64], 192, 5, 1, 2),          # AlexNet conv2
    (2, 13, 13, [384], 256, 3, 1, 1),         # AlexNet conv4
    (3, 17, 17, [64], 96, 3, 2, 1),           # strided (fprop/wgrad only)
    (2, 10, 10, [48], 36, 5, 1, 2),           # channels not multiples of 32
    (300, 1, 1, [64], 20, 1, 1, 0),           # M spans several tiles of a 1x1 "image"
    (3, 20, 20, [3], 64, 3, 1, 1),            # VGG-style first layer (small-C SIMT path)
    (2, 23, 23, [3], 96, 11, 4, 0),           # OverFeat-style first layer, Cout 96
    (2, 9, 9, [4], 40, 3, 2, 1),              # C = 4, strided, Cout not a multiple of 32
    (4, 14, 14, [256], 512, 3, 1, 1),         # wide (BN=256) tiles, several M and N tiles
    (2, 6, 6, [128], 288, 3, 1, 1),           # wide tiles with a partial second N tile
    (2, 30, 30, [3], 128, 3, 1, 1),           # first layer on the tensor cores (K = 27 in one block)
    (4, 17, 17, [2], 32, 3, 2, 1),            # C = 2, strided, Cout 32 (tensor-core first layer)
    (2, 16, 16, [1], 64, 5, 1, 2),            # C = 1, 5x5 (K = 25)
]


@pytest.fixture(params=["tf32-tma", "tf32-cpasync", "fp32"])
def precise(request):
    L.lib().vdnn_kernel_set_precise(int(request.param == "fp32"))
    L.lib().vdnn_kernel_set_tma(int(request.param != "tf32-cpasync"))
    yield request.param == "fp32"
    L.lib().vdnn_kernel_set_precise(0)
    L.lib().vdnn_kernel_set_tma(1)


@pytest.mark.parametrize("case", CASES)
def test_conv_fprop_dgrad_wgrad(case, precise):
    global TF32_TOL
    tol_saved = TF32_TOL
    # fp32 mode: products are fp32-accurate; the tensor core's accumulation
    # carries a small bias (~7e-9 per reduction term, measured), so the
    # bound scales with the reduction length K.
    n, h, w, segs, cout, k, stride, pad = case
    kred = max(k * k * sum(segs), k * k * cout, n * h * w)
    TF32_TOL = 4e-6 + 1.2e-8 * kred if precise else tol_saved
    try:
        _conv_case(case)
    finally:
        TF32_TOL = tol_saved


def _conv_case(case):
    dev = _dev()
    n, h, w, segs, cout, k, stride, pad = case
    g = torch.Generator().manual_seed(CASES.index(case) + 1)
    xs = [torch.randn(n, h, w, c, generator=g).to(dev) for c in segs]
    cin = sum(segs)
    wt = (torch.randn(cout, k, k, cin, generator=g) * (2.0 / (k * k * cin)) ** 0.5).to(dev)
    ho = (h + 2 * pad - k) // stride + 1
    wo = (w + 2 * pad - k) // stride + 1
    y = torch.empty(n, ho, wo, cout, device=dev)
    d = _desc(n, h, w, xs, segs, cout, k, stride, pad)
    L.call("vdnn_kernel_conv_fprop", C.byref(d), C.c_void_p(wt.data_ptr()), None, C.c_void_p(y.data_ptr()), None)
    torch.cuda.synchronize()
    xr, wr, yr = _ref_conv(xs, wt, stride, pad)
    _close(y, yr.permute(0, 2, 3, 1))
    fws = L.lib().vdnn_kernel_conv_fprop_ws_bytes(C.byref(d))
    if fws > 0:  # split-K fprop (few output tiles, long reduction)
        ws = torch.empty(fws // 4, device=dev)
        y2 = torch.full_like(y, float("nan"))
        L.call("vdnn_kernel_conv_fprop_ws", C.byref(d), C.c_void_p(wt.data_ptr()), None, C.c_void_p(y2.data_ptr()),
               C.c_void_p(ws.data_ptr()), C.c_size_t(fws), None)
        torch.cuda.synchronize()
        _close(y2, yr.permute(0, 2, 3, 1))

    dy = torch.randn(n, ho, wo, cout, generator=g).to(dev)
    yr.backward(dy.double().cpu().permute(0, 3, 1, 2))
    if stride == 1:
        dxs = [torch.full_like(t, float("nan")) for t in xs]
        d2 = _desc(n, h, w, xs, segs, cout, k, stride, pad, dxs)
        L.call("vdnn_kernel_conv_dgrad", C.byref(d2), C.c_void_p(wt.data_ptr()), C.c_void_p(dy.data_ptr()),
               0, None)
        torch.cuda.synchronize()
        gx = xr.grad.permute(0, 2, 3, 1)
        off = 0
        for t, c in zip(dxs, segs):
            _close(t, gx[..., off:off + c])
            off += c
        dws = L.lib().vdnn_kernel_conv_dgrad_ws_bytes(C.byref(d2))
        if dws > 0:  # split-K dgrad (few dX tiles, long reduction)
            wsd = torch.empty(dws // 4, device=dev)
            dx2 = [torch.full_like(t, float("nan")) for t in xs]
            d3 = _desc(n, h, w, xs, segs, cout, k, stride, pad, dx2)
            L.call("vdnn_kernel_conv_dgrad_ws", C.byref(d3), C.c_void_p(wt.data_ptr()), C.c_void_p(dy.data_ptr()),
                   0, C.c_void_p(wsd.data_ptr()), C.c_size_t(dws), None)
            torch.cuda.synchronize()
            _close(dx2[0], gx)
    # wgrad with dW output (no SGD), with and without split-K workspace
    for use_ws in (False, True):
        dw = torch.full_like(wt, float("nan"))
        ws_bytes = L.lib().vdnn_kernel_conv_wgrad_ws_bytes(C.byref(d)) if use_ws else 0
        ws = torch.empty(max(ws_bytes // 4, 1), device=dev)
        L.call("vdnn_kernel_conv_wgrad", C.byref(d), C.c_void_p(dy.data_ptr()), C.c_void_p(wt.data_ptr()),
               C.c_float(0.0), C.c_void_p(dw.data_ptr()), C.c_void_p(ws.data_ptr() if use_ws else 0),
               C.c_size_t(ws_bytes), None)
        torch.cuda.synchronize()
        _close(dw, wr.grad.permute(0, 2, 3, 1))
    # fused SGD epilogue
    w2 = wt.clone()
    lr = 0.01
    L.call("vdnn_kernel_conv_wgrad", C.byref(d), C.c_void_p(dy.data_ptr()), C.c_void_p(w2.data_ptr()),
           C.c_float(lr), None, None, C.c_size_t(0), None)
    torch.cuda.synchronize()
    ref = wt.double().cpu() - lr * wr.grad.permute(0, 2, 3, 1)
    diff = (w2.double().cpu() - ref).abs().max().item()
    assert diff < TF32_TOL * lr * max(wr.grad.abs().max().item(), 1e-30) + 2e-7 * max(1.0, wt.abs().max().item())


def test_wgrad_split_k_large_reduction():
    """K = N*Ho*Wo large enough that split-K partials + reduce kernel run."""
    dev = _dev()
    n, h, w, c, cout = 8, 56, 56, 64, 64
    g = torch.Generator().manual_seed(7)
    x = torch.randn(n, h, w, c, generator=g).to(dev)
    dy = torch.randn(n, h, w, cout, generator=g).to(dev)
    wt = torch.zeros(cout, 3, 3, c, device=dev)
    d = _desc(n, h, w, [x], [c], cout, 3, 1, 1)
    ws_bytes = L.lib().vdnn_kernel_conv_wgrad_ws_bytes(C.byref(d))
    assert ws_bytes > 0
    ws = torch.empty(ws_bytes // 4, device=dev)
    dw = torch.empty_like(wt)
    L.call("vdnn_kernel_conv_wgrad", C.byref(d), C.c_void_p(dy.data_ptr()), C.c_void_p(wt.data_ptr()),
           C.c_float(0.0), C.c_void_p(dw.data_ptr()), C.c_void_p(ws.data_ptr()), C.c_size_t(ws_bytes), None)
    torch.cuda.synchronize()
    xr, wr, yr = _ref_conv([x], wt, 1, 1)
    yr.backward(dy.double().cpu().permute(0, 3, 1, 2))
    _close(dw, wr.grad.permute(0, 2, 3, 1))


@pytest.mark.parametrize("window,stride,segs,h", [(3, 2, [64], 13), (3, 2, [16, 8], 13), (3, 2, [3], 13),
                                                 (2, 2, [16, 8], 13), (2, 2, [3], 13), (2, 2, [64], 13),
                                                 (2, 2, [64], 14), (3, 3, [8], 12)])
def test_maxpool(window, stride, segs, h):
    """Forward and backward against torch (ties from ReLU zeros on purpose).
    The backward gets a NaN-filled Y: the kernels recompute each window's
    maximum from X and must not read it."""
    dev = _dev()
    n, w = 2, h
    g = torch.Generator().manual_seed(3)
    # ties on purpose: relu'd inputs have many zeros
    xs = [torch.relu(torch.randn(n, h, w, c, generator=g)).to(dev) for c in segs]
    ho, wo = (h - window) // stride + 1, (w - window) // stride + 1
    ct = sum(segs)
    y = torch.empty(n, ho, wo, ct, device=dev)
    d = _desc(n, h, w, xs, segs, 0, 1, 1, 0)
    L.call("vdnn_kernel_maxpool_fwd", C.byref(d), window, stride, C.c_void_p(y.data_ptr()), None)
    torch.cuda.synchronize()
    xc = torch.cat([t.cpu() for t in xs], dim=3).permute(0, 3, 1, 2).double().requires_grad_(True)
    yr = torch.nn.functional.max_pool2d(xc, window, stride)
    assert torch.equal(y.cpu().double(), yr.detach().permute(0, 2, 3, 1))
    dy = torch.randn(n, ho, wo, ct, generator=g).to(dev)
    dxs = [torch.full_like(t, float("nan")) for t in xs]
    d2 = _desc(n, h, w, xs, segs, 0, 1, 1, 0, dxs)
    y.fill_(float("nan"))
    L.call("vdnn_kernel_maxpool_bwd", C.byref(d2), window, stride, C.c_void_p(y.data_ptr()),
           C.c_void_p(dy.data_ptr()), None)
    torch.cuda.synchronize()
    yr.backward(dy.cpu().double().permute(0, 3, 1, 2))
    gx = xc.grad.permute(0, 2, 3, 1)
    off = 0
    for t, c in zip(dxs, segs):
        torch.testing.assert_close(t.cpu().double(), gx[..., off:off + c], rtol=1e-6, atol=1e-6)
        off += c


def test_relu_and_softmax():
    dev = _dev()
    g = torch.Generator().manual_seed(11)
    x = torch.randn(1000003, generator=g).to(dev)
    y = x.clone()
    L.call("vdnn_kernel_relu_fwd", C.c_void_p(y.data_ptr()), C.c_size_t(y.numel()), None)
    gr = torch.randn(1000003, generator=g).to(dev)
    g2 = gr.clone()
    L.call("vdnn_kernel_relu_bwd", C.c_void_p(g2.data_ptr()), C.c_void_p(y.data_ptr()), C.c_size_t(y.numel()), None)
    torch.cuda.synchronize()
    assert torch.equal(y, torch.relu(x))
    assert torch.equal(g2, torch.where(y > 0, gr, torch.zeros_like(gr)))
    n, k = 37, 1000
    z = torch.randn(n, k, generator=g).to(dev) * 3
    lab = torch.randint(0, k, (n,), generator=g, dtype=torch.int32).to(dev)
    grad = torch.empty(n, k, device=dev)
    rl = torch.empty(n, device=dev)
    loss = torch.empty(1, device=dev)
    L.call("vdnn_kernel_softmax_xent", C.c_void_p(z.data_ptr()), C.c_void_p(lab.data_ptr()), n, k,
           C.c_void_p(grad.data_ptr()), C.c_void_p(rl.data_ptr()), C.c_void_p(loss.data_ptr()), None)
    torch.cuda.synchronize()
    zr = z.double().cpu().requires_grad_(True)
    lr_ = torch.nn.functional.cross_entropy(zr, lab.long().cpu())
    lr_.backward()
    assert abs(loss.item() - lr_.item()) < 1e-5 * max(1.0, abs(lr_.item()))
    torch.testing.assert_close(grad.double().cpu(), zr.grad, rtol=1e-4, atol=1e-7)


def test_fc_fprop_split_k_with_bias():
    """VGG-16 FC6 at batch 256 (2 x 32 output tiles over K = 25,088): the
    split-K partial slabs + ordered reduce with the fused bias, against the
    unsplit kernel and a float64 reference; deterministic across calls."""
    dev = _dev()
    n, k, o = 256, 25088, 4096
    g = torch.Generator(device=dev).manual_seed(7)
    x = torch.randn(n, 1, 1, k, device=dev, generator=g)
    wt = torch.randn(o, 1, 1, k, device=dev, generator=g) * (2.0 / k) ** 0.5
    b = torch.randn(o, device=dev, generator=g)
    d = _desc(n, 1, 1, [x], [k], o, 1, 1, 0)
    fws = L.lib().vdnn_kernel_conv_fprop_ws_bytes(C.byref(d))
    assert fws > 0
    ws = torch.empty(fws // 4, device=dev)
    outs = []
    for _ in range(2):
        y = torch.full((n, 1, 1, o), float("nan"), device=dev)
        L.call("vdnn_kernel_conv_fprop_ws", C.byref(d), C.c_void_p(wt.data_ptr()), C.c_void_p(b.data_ptr()),
               C.c_void_p(y.data_ptr()), C.c_void_p(ws.data_ptr()), C.c_size_t(fws), None)
        outs.append(y)
    y1 = torch.empty_like(outs[0])
    L.call("vdnn_kernel_conv_fprop", C.byref(d), C.c_void_p(wt.data_ptr()), C.c_void_p(b.data_ptr()),
           C.c_void_p(y1.data_ptr()), None)
    torch.cuda.synchronize()
    ref = (x.double().reshape(n, k) @ wt.double().reshape(o, k).T + b.double()).reshape(n, 1, 1, o)
    assert torch.equal(outs[0], outs[1])
    _close(outs[0], ref)
    _close(y1, ref)


@pytest.mark.parametrize("accumulate", [False, True])
def test_fc_dgrad_split_k(accumulate):
    """AlexNet FC6 dX at batch 128 (1 x 72 tiles over K = 4,096): split-K
    partial slabs + ordered reduce, plain and accumulating (branch-join)
    mode, against the unsplit kernel and a float64 reference; deterministic
    across calls. (The fused ReLU mask is a session-level flag: covered by
    the VGG-16 session parity test, whose FC7 dX splits.)"""
    dev = _dev()
    n, k, o = 128, 9216, 4096
    g = torch.Generator(device=dev).manual_seed(11)
    x = torch.randn(n, 1, 1, k, device=dev, generator=g)
    wt = torch.randn(o, 1, 1, k, device=dev, generator=g) * (2.0 / k) ** 0.5
    dy = torch.randn(n, 1, 1, o, device=dev, generator=g)
    base = torch.randn(n, 1, 1, k, device=dev, generator=g)
    d = _desc(n, 1, 1, [x], [k], o, 1, 1, 0)
    ws_bytes = L.lib().vdnn_kernel_conv_dgrad_ws_bytes(C.byref(d))
    assert ws_bytes > 0
    ws = torch.empty(ws_bytes // 4, device=dev)
    outs = []
    for use_ws in (True, True, False):
        dx = base.clone() if accumulate else torch.full_like(x, float("nan"))
        dd = _desc(n, 1, 1, [x], [k], o, 1, 1, 0, [dx])
        if use_ws:
            L.call("vdnn_kernel_conv_dgrad_ws", C.byref(dd), C.c_void_p(wt.data_ptr()), C.c_void_p(dy.data_ptr()),
                   1 if accumulate else 0, C.c_void_p(ws.data_ptr()), C.c_size_t(ws_bytes), None)
        else:
            L.call("vdnn_kernel_conv_dgrad", C.byref(dd), C.c_void_p(wt.data_ptr()), C.c_void_p(dy.data_ptr()),
                   1 if accumulate else 0, None)
        outs.append(dx)
    torch.cuda.synchronize()
    ref = (dy.double().reshape(n, o) @ wt.double().reshape(o, k)).reshape(n, 1, 1, k)
    if accumulate:
        ref = ref + base.double()
    assert torch.equal(outs[0], outs[1])
    _close(outs[0], ref)
    _close(outs[2], ref)


# Shapes large enough to select the production tile variants: tall (BM=256)
# 128/64-wide tiles, wide (BN=256) tall tiles, 64-pixel wgrad stages, split-K
# over hundreds of CTAs. Reference: torch float64 on the GPU (same op).
LARGE = [
    (32, 56, 56, 64, 128),    # fprop tall BN=128, dgrad tall BN=64, wgrad BN=128
    (64, 56, 56, 256, 256),   # fprop/dgrad wide+tall (BN=256, BM=256), wgrad BN=256 KW=64
    # halo-reuse fprop/dgrad (tc_conv_halo.cuh): one padded row per tile (P = 226),
    # two rows (P = 114), eight rows (P = 30)
    (2, 224, 224, 64, 64),
    (4, 112, 112, 128, 128),
    (8, 28, 28, 512, 512),
    # halo on a CTA pair (tc_conv_halo_pair.cuh) with an odd number of row
    # tiles (P = 26, TH = 9: 3 per image), so a rank-1 CTA computes past the
    # last row tile and must store nothing
    (3, 24, 24, 128, 128),
    (3, 24, 24, 64, 64),
    # CTA-pair (cta_group::2) fprop/dgrad: 256 x 256 tiles over >= 148 tiles,
    # and a 384-column layer whose second tile leaves the peer's B half empty
    (32, 28, 28, 512, 512),
    (64, 28, 28, 384, 384),
]


@pytest.mark.parametrize("shape", LARGE)
def test_conv_production_tiles(shape):
    dev = _dev()
    n, h, w, c, cout = shape
    g = torch.Generator(device=dev).manual_seed(n + c)
    x = torch.randn(n, h, w, c, device=dev, generator=g)
    wt = torch.randn(cout, 3, 3, c, device=dev, generator=g) * (2.0 / (9 * c)) ** 0.5
    dy = torch.randn(n, h, w, cout, device=dev, generator=g)
    xr = x.double().permute(0, 3, 1, 2).requires_grad_(True)
    wr = wt.double().permute(0, 3, 1, 2).requires_grad_(True)
    yr = torch.nn.functional.conv2d(xr, wr, padding=1)
    yr.backward(dy.double().permute(0, 3, 1, 2))
    y = torch.empty(n, h, w, cout, device=dev)
    dx = torch.full_like(x, float("nan"))
    d = _desc(n, h, w, [x], [c], cout, 3, 1, 1, [dx])
    L.call("vdnn_kernel_conv_fprop", C.byref(d), C.c_void_p(wt.data_ptr()), None, C.c_void_p(y.data_ptr()), None)
    L.call("vdnn_kernel_conv_dgrad", C.byref(d), C.c_void_p(wt.data_ptr()), C.c_void_p(dy.data_ptr()), 0, None)
    ws_bytes = L.lib().vdnn_kernel_conv_wgrad_ws_bytes(C.byref(d))
    ws = torch.empty(max(ws_bytes // 4, 1), device=dev)
    dw = torch.full_like(wt, float("nan"))
    L.call("vdnn_kernel_conv_wgrad", C.byref(d), C.c_void_p(dy.data_ptr()), C.c_void_p(wt.data_ptr()),
           C.c_float(0.0), C.c_void_p(dw.data_ptr()), C.c_void_p(ws.data_ptr()), C.c_size_t(ws_bytes), None)
    torch.cuda.synchronize()
    for got, ref in ((y, yr.detach().permute(0, 2, 3, 1)), (dx, xr.grad.permute(0, 2, 3, 1)),
                     (dw, wr.grad.permute(0, 2, 3, 1))):
        err = (got.double() - ref).abs().max().item() / ref.abs().max().item()
        assert err < TF32_TOL, err
    # accumulating dgrad (two-buffer fork accumulation): dx_acc = base + dX
    base = torch.randn_like(x)
    dxa = base.clone()
    da = _desc(n, h, w, [x], [c], cout, 3, 1, 1, [dxa])
    L.call("vdnn_kernel_conv_dgrad", C.byref(da), C.c_void_p(wt.data_ptr()), C.c_void_p(dy.data_ptr()), 1, None)
    torch.cuda.synchronize()
    refa = base.double() + xr.grad.permute(0, 2, 3, 1)
    err = (dxa.double() - refa).abs().max().item() / refa.abs().max().item()
    assert err < TF32_TOL, err
    # fused SGD epilogue (w -= lr * dW), same split-K workspace
    lr = 1e-3
    w2 = wt.clone()
    L.call("vdnn_kernel_conv_wgrad", C.byref(d), C.c_void_p(dy.data_ptr()), C.c_void_p(w2.data_ptr()),
           C.c_float(lr), None, C.c_void_p(ws.data_ptr()), C.c_size_t(ws_bytes), None)
    torch.cuda.synchronize()
    gref = wr.grad.permute(0, 2, 3, 1)
    diff = (w2.double() - (wt.double() - lr * gref)).abs().max().item()
    assert diff < TF32_TOL * lr * gref.abs().max().item() + 2e-7 * wt.abs().max().item(), diff


_HALO_SNIPPET = r"""
import ctypes as C, sys, torch
sys.path.insert(0, {root!r})
from paper_1602_08124_b200 import _lib as L
n, h, c, cout = {shape!r}
g = torch.Generator(device="cuda").manual_seed(3)
x = torch.randn(n, h, h, c, device="cuda", generator=g)
wt = torch.randn(cout, 3, 3, c, device="cuda", generator=g) * (2.0 / (9 * c)) ** 0.5
dy = torch.randn(n, h, h, cout, device="cuda", generator=g)
y = torch.empty(n, h, h, cout, device="cuda")
dx = torch.empty_like(x)
d = L.ConvDesc(); d.n, d.h, d.w, d.nseg = n, h, h, 1
d.x[0] = x.data_ptr(); d.dx[0] = dx.data_ptr(); d.c[0] = c
d.cout, d.kh, d.kw, d.stride, d.pad = cout, 3, 3, 1, 1
L.call("vdnn_kernel_conv_fprop", C.byref(d), C.c_void_p(wt.data_ptr()), None, C.c_void_p(y.data_ptr()), None)
L.call("vdnn_kernel_conv_dgrad", C.byref(d), C.c_void_p(wt.data_ptr()), C.c_void_p(dy.data_ptr()), 0, None)
torch.cuda.synchronize()
torch.save({{"y": y.cpu(), "dx": dx.cpu()}}, {out!r})
"""


@pytest.mark.parametrize("shape", [(2, 224, 64, 64), (3, 24, 128, 128), (4, 56, 128, 64)])
def test_halo_pair_bit_identical_to_single_cta(shape, tmp_path):
    """The CTA-pair halo kernel accumulates every output in the same K order
    as the single-CTA halo kernel: fprop and dgrad outputs are bit-identical
    (VDNN_HALO_PAIR=0 selects the single-CTA kernel in a child process)."""
    import os
    import subprocess
    import sys
    _dev()
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    outs = []
    for flag in ("1", "0"):
        out = str(tmp_path / f"halo{flag}.pt")
        env = dict(os.environ, VDNN_HALO_PAIR=flag)
        subprocess.run([sys.executable, "-c", _HALO_SNIPPET.format(root=root, shape=shape, out=out)], env=env,
                       check=True, timeout=300)
        outs.append(torch.load(out))
    assert torch.equal(outs[0]["y"], outs[1]["y"])
    assert torch.equal(outs[0]["dx"], outs[1]["dx"])


@pytest.mark.parametrize("n,h,cout", [(16, 227, 64), (8, 231, 96)])
def test_first_layer_big_window_tensor_cores(n, h, cout):
    """AlexNet / OverFeat conv1 (11x11x3, stride 4, K = 363 = 12 K blocks) on
    the multi-K-block first-layer tensor-core kernels (fprop + wgrad with the
    ordered partial reduce), against float64 torch on the GPU."""
    dev = _dev()
    g = torch.Generator(device=dev).manual_seed(h)
    x = torch.randn(n, h, h, 3, device=dev, generator=g)
    wt = torch.randn(cout, 11, 11, 3, device=dev, generator=g) * (2.0 / 363) ** 0.5
    ho = (h - 11) // 4 + 1
    dy = torch.randn(n, ho, ho, cout, device=dev, generator=g)
    xr = x.double().permute(0, 3, 1, 2)
    wr = wt.double().permute(0, 3, 1, 2).requires_grad_(True)
    yr = torch.nn.functional.conv2d(xr, wr, stride=4)
    yr.backward(dy.double().permute(0, 3, 1, 2))
    y = torch.full((n, ho, ho, cout), float("nan"), device=dev)
    d = _desc(n, h, h, [x], [3], cout, 11, 4, 0)
    L.call("vdnn_kernel_conv_fprop", C.byref(d), C.c_void_p(wt.data_ptr()), None, C.c_void_p(y.data_ptr()), None)
    ws_bytes = L.lib().vdnn_kernel_conv_wgrad_ws_bytes(C.byref(d))
    ws = torch.empty(max(ws_bytes // 4, 1), device=dev)
    dw = torch.full_like(wt, float("nan"))
    L.call("vdnn_kernel_conv_wgrad", C.byref(d), C.c_void_p(dy.data_ptr()), C.c_void_p(wt.data_ptr()),
           C.c_float(0.0), C.c_void_p(dw.data_ptr()), C.c_void_p(ws.data_ptr()), C.c_size_t(ws_bytes), None)
    torch.cuda.synchronize()
    for got, ref in ((y, yr.detach().permute(0, 2, 3, 1)), (dw, wr.grad.permute(0, 2, 3, 1))):
        err = (got.double() - ref).abs().max().item() / ref.abs().max().item()
        assert err < TF32_TOL, err
