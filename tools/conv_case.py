"""Run one conv shape's fprop/dgrad/wgrad a few times (for ncu / quick timing).

    python tools/conv_case.py N H W C COUT [K STRIDE PAD] [--reps R]
"""
import ctypes as C, sys
sys.path.insert(0, ".")
import torch
from paper_1602_08124_b200 import _lib as L

args = [a for a in sys.argv[1:] if not a.startswith("--")]
reps = int(sys.argv[sys.argv.index("--reps") + 1]) if "--reps" in sys.argv else 5
if "--reps" in sys.argv:
    args.remove(str(reps))
n, h, w, c, co = map(int, args[:5])
k, st, pad = (map(int, args[5:8]) if len(args) >= 8 else (3, 1, 1))
ho, wo = (h + 2 * pad - k) // st + 1, (w + 2 * pad - k) // st + 1
dev = torch.device("cuda")
x = torch.randn(n, h, w, c, device=dev)
wt = torch.randn(co, k, k, c, device=dev) * 0.01
y = torch.empty(n, ho, wo, co, device=dev)
dy = torch.randn(n, ho, wo, co, device=dev)
dx = torch.empty_like(x)
d = L.ConvDesc(); d.n, d.h, d.w, d.nseg = n, h, w, 1; d.x[0] = x.data_ptr(); d.dx[0] = dx.data_ptr(); d.c[0] = c
d.cout, d.kh, d.kw, d.stride, d.pad = co, k, k, st, pad
ws_b = L.lib().vdnn_kernel_conv_wgrad_ws_bytes(C.byref(d)); ws = torch.empty(max(ws_b // 4, 1), device=dev)
dw = torch.empty_like(wt)
fl = 2 * k * k * c * co * ho * wo * n
fns = {
    "fprop": lambda: L.call("vdnn_kernel_conv_fprop", C.byref(d), C.c_void_p(wt.data_ptr()), None, C.c_void_p(y.data_ptr()), None),
    "wgrad": lambda: L.call("vdnn_kernel_conv_wgrad", C.byref(d), C.c_void_p(dy.data_ptr()), C.c_void_p(wt.data_ptr()), C.c_float(0), C.c_void_p(dw.data_ptr()), C.c_void_p(ws.data_ptr()), C.c_size_t(ws_b), None),
}
if st == 1 and c > 4:
    fns["dgrad"] = lambda: L.call("vdnn_kernel_conv_dgrad", C.byref(d), C.c_void_p(wt.data_ptr()), C.c_void_p(dy.data_ptr()), 0, None)
for name, fn in fns.items():
    fn(); torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(reps): fn()
    e.record(); e.synchronize()
    t = s.elapsed_time(e) / reps
    print(f"{name}: {t:.3f} ms {fl / t / 1e9:.1f} TF")
