"""Microbenchmark of the conv engine per VGG-16 b256 layer: fprop / dgrad / wgrad ms and TFLOP/s."""
import ctypes as C, sys
sys.path.insert(0, ".")
import torch
from paper_1602_08124_b200 import _lib as L
dev = torch.device("cuda")
shapes = [(256, 224, 224, 64, 64), (256, 112, 112, 128, 128), (256, 56, 56, 256, 256), (256, 28, 28, 512, 512),
          (256, 14, 14, 512, 512), (256, 112, 112, 64, 128)]
if "notma" in sys.argv[1:]:
    L.lib().vdnn_kernel_set_tma(0)
if "precise" in sys.argv[1:]:
    L.lib().vdnn_kernel_set_precise(1)
def t(fn, n=int(__import__("os").environ.get("REPS", "5"))):
    fn(); torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(n): fn()
    e.record(); e.synchronize()
    return s.elapsed_time(e) / n
for n, h, w, c, co in shapes:
    x = torch.randn(n, h, w, c, device=dev); wt = torch.randn(co, 3, 3, c, device=dev) * 0.01
    y = torch.empty(n, h, w, co, device=dev); dy = torch.randn(n, h, w, co, device=dev); dx = torch.empty_like(x)
    d = L.ConvDesc(); d.n, d.h, d.w, d.nseg = n, h, w, 1; d.x[0] = x.data_ptr(); d.dx[0] = dx.data_ptr(); d.c[0] = c
    d.cout, d.kh, d.kw, d.stride, d.pad = co, 3, 3, 1, 1
    ws_b = L.lib().vdnn_kernel_conv_wgrad_ws_bytes(C.byref(d)); ws = torch.empty(max(ws_b // 4, 1), device=dev)
    dw = torch.empty_like(wt)
    fl = 2 * 9 * c * co * h * w * n
    tf = t(lambda: L.call("vdnn_kernel_conv_fprop", C.byref(d), C.c_void_p(wt.data_ptr()), None, C.c_void_p(y.data_ptr()), None))
    td = t(lambda: L.call("vdnn_kernel_conv_dgrad", C.byref(d), C.c_void_p(wt.data_ptr()), C.c_void_p(dy.data_ptr()), 0, None))
    tw = t(lambda: L.call("vdnn_kernel_conv_wgrad", C.byref(d), C.c_void_p(dy.data_ptr()), C.c_void_p(wt.data_ptr()), C.c_float(0), C.c_void_p(dw.data_ptr()), C.c_void_p(ws.data_ptr()), C.c_size_t(ws_b), None))
    print(f"{n}x{h}x{w} {c}->{co}: fprop {tf:.3f} ms {fl/tf/1e9:.0f} TF | dgrad {td:.3f} ms {fl/td/1e9:.0f} TF | wgrad {tw:.3f} ms {fl/tw/1e9:.0f} TF (ws {ws_b/1e6:.1f} MB)")
    del x, y, dy, dx, ws
