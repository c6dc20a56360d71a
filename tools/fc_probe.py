"""FC layer kernels at VGG-16 b256 shapes: fprop (split-K), dgrad (split-K when
few tiles), wgrad with the fused SGD epilogue; ms and TFLOP/s."""
import ctypes as C
import sys

import torch

sys.path.insert(0, ".")
from paper_1602_08124_b200 import _lib as L

dev = torch.device("cuda")


def t(fn, n=20):
    fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(n):
        fn()
    b.record()
    b.synchronize()
    return a.elapsed_time(b) / n


for n, k, o in [(256, 25088, 4096), (256, 4096, 4096), (256, 4096, 1000), (128, 9216, 4096)]:
    x = torch.randn(n, 1, 1, k, device=dev)
    w = torch.randn(o, 1, 1, k, device=dev) * 0.01
    dy = torch.randn(n, 1, 1, o, device=dev)
    dx = torch.empty_like(x)
    y = torch.empty(n, 1, 1, o, device=dev)
    d = L.ConvDesc()
    d.n, d.h, d.w, d.nseg = n, 1, 1, 1
    d.x[0] = x.data_ptr()
    d.dx[0] = dx.data_ptr()
    d.c[0] = k
    d.cout, d.kh, d.kw, d.stride, d.pad = o, 1, 1, 1, 0
    fws = L.lib().vdnn_kernel_conv_fprop_ws_bytes(C.byref(d))
    dws = L.lib().vdnn_kernel_conv_dgrad_ws_bytes(C.byref(d))
    wws = L.lib().vdnn_kernel_conv_wgrad_ws_bytes(C.byref(d))
    ws = torch.empty(max(fws, dws, wws, 4) // 4, device=dev)
    fl = 2 * n * k * o
    tf = t(lambda: L.call("vdnn_kernel_conv_fprop_ws", C.byref(d), C.c_void_p(w.data_ptr()), None,
                          C.c_void_p(y.data_ptr()), C.c_void_p(ws.data_ptr()), C.c_size_t(ws.numel() * 4), None))
    td = t(lambda: L.call("vdnn_kernel_conv_dgrad_ws", C.byref(d), C.c_void_p(w.data_ptr()), C.c_void_p(dy.data_ptr()),
                          0, C.c_void_p(ws.data_ptr()), C.c_size_t(ws.numel() * 4), None))
    tw = t(lambda: L.call("vdnn_kernel_conv_wgrad", C.byref(d), C.c_void_p(dy.data_ptr()), C.c_void_p(w.data_ptr()),
                          C.c_float(1e-9), None, C.c_void_p(ws.data_ptr()), C.c_size_t(ws.numel() * 4), None))
    print(f"FC {n}x{k}->{o}: fprop {tf:.3f} ms {fl / tf / 1e9:.0f} TF (ws {fws >> 20} MB) | dgrad {td:.3f} ms "
          f"{fl / td / 1e9:.0f} TF (ws {dws >> 20} MB) | wgrad+SGD {tw:.3f} ms {fl / tw / 1e9:.0f} TF, "
          f"{2 * 4 * k * o / tw / 1e6:.0f} GB/s of weight r+w (ws {wws >> 20} MB)")
