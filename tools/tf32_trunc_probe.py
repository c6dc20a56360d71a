"""Does tcgen05.mma kind::tf32 truncate or round its fp32 operands? Run the
conv engine (fprop, wgrad) on X, on X with the low 13 mantissa bits cleared
(truncation) and on X rounded to nearest tf32; compare outputs bitwise."""
import ctypes as C
import sys

import torch

sys.path.insert(0, ".")
from paper_1602_08124_b200 import _lib as L

dev = torch.device("cuda")
g = torch.Generator(device=dev).manual_seed(1)
for (n, h, c, co) in [(8, 56, 64, 64), (4, 28, 128, 256), (64, 1, 4096, 1000)]:
    x = torch.randn(n, h, h, c, device=dev, generator=g)
    x = torch.relu(x)
    wt = torch.randn(co, 3 if h > 1 else 1, 3 if h > 1 else 1, c, device=dev, generator=g) * 0.05
    k = 3 if h > 1 else 1
    dy = torch.randn(n, h, h, co, device=dev, generator=g)
    xi = x.view(torch.int32)
    xt = (xi & ~0x1FFF).view(torch.float32)
    xr = ((xi + 0x1000) & ~0x1FFF).view(torch.float32)  # round half away (magnitude) = RN except ties
    outs = {}
    for name, xx in (("orig", x), ("trunc", xt), ("round", xr)):
        d = L.ConvDesc(); d.n, d.h, d.w, d.nseg = n, h, h, 1
        d.x[0] = xx.data_ptr(); d.c[0] = c
        d.cout, d.kh, d.kw, d.stride, d.pad = co, k, k, 1, (1 if k == 3 else 0)
        y = torch.empty(n, h, h, co, device=dev)
        L.call("vdnn_kernel_conv_fprop", C.byref(d), C.c_void_p(wt.data_ptr()), None, C.c_void_p(y.data_ptr()), None)
        wsb = L.lib().vdnn_kernel_conv_wgrad_ws_bytes(C.byref(d)); ws = torch.empty(max(wsb // 4, 1), device=dev)
        dw = torch.empty_like(wt)
        L.call("vdnn_kernel_conv_wgrad", C.byref(d), C.c_void_p(dy.data_ptr()), C.c_void_p(wt.data_ptr()),
               C.c_float(0.0), C.c_void_p(dw.data_ptr()), C.c_void_p(ws.data_ptr()), C.c_size_t(wsb), None)
        torch.cuda.synchronize()
        outs[name] = (y, dw)
    for name in ("trunc", "round"):
        print((n, h, c, co), name, "fprop equal:", torch.equal(outs["orig"][0], outs[name][0]),
              "wgrad equal:", torch.equal(outs["orig"][1], outs[name][1]))
