import sys, ctypes as C, numpy as np, torch
sys.path.insert(0, ".")
from paper_1602_08124_b200 import _lib as L
def trunc(t):
    i = t.float().contiguous().view(torch.int32); return (i & ~0x1FFF).view(torch.float32).double()
def rne(t):
    i = t.float().contiguous().view(torch.int32).to(torch.int64)
    r = ((i + 0xFFF + ((i >> 13) & 1)) & ~0x1FFF)
    return r.to(torch.int32).view(torch.float32).double()
dev = torch.device("cuda")
for C_ in (64, 63, 32, 4, 3, 128):
    torch.manual_seed(0)
    n, h, w, co = 2, 8, 8, 64
    x = torch.randn(n, h, w, C_).to(dev); wt = torch.randn(co, 1, 1, C_).to(dev)
    y = torch.empty(n, h, w, co, device=dev)
    d = L.ConvDesc(); d.n, d.h, d.w, d.nseg = n, h, w, 1
    d.x[0] = x.data_ptr(); d.c[0] = C_; d.cout, d.kh, d.kw, d.stride, d.pad = co, 1, 1, 1, 0
    L.call("vdnn_kernel_conv_fprop", C.byref(d), C.c_void_p(wt.data_ptr()), None, C.c_void_p(y.data_ptr()), None)
    torch.cuda.synchronize()
    xc, wc = x.cpu().double().reshape(-1, C_), wt.cpu().double().reshape(co, C_)
    g = y.cpu().double().reshape(-1, co)
    for nm, f in (("fp64", lambda t: t), ("trunc", trunc), ("rne", rne)):
        ref = f(xc) @ f(wc).t()
        print(C_, nm, f"{(torch.linalg.norm(g - ref) / torch.linalg.norm(ref)).item():.3e}")
