import ctypes as C, sys
sys.path.insert(0, ".")
import torch
from paper_1602_08124_b200 import _lib as L
sys.path.insert(0, "tests")
from test_kernels_gpu import _desc
dev = torch.device("cuda")
for (n, h, cout, k, st) in [(2, 35, 64, 11, 4), (16, 227, 64, 11, 4), (2, 20, 64, 7, 1)]:
    g = torch.Generator(device=dev).manual_seed(h)
    x = torch.randn(n, h, h, 3, device=dev, generator=g)
    wt = torch.randn(cout, k, k, 3, device=dev, generator=g) * 0.1
    ho = (h - k) // st + 1
    y = torch.full((n, ho, ho, cout), float("nan"), device=dev)
    d = _desc(n, h, h, [x], [3], cout, k, st, 0)
    L.call("vdnn_kernel_conv_fprop", C.byref(d), C.c_void_p(wt.data_ptr()), None, C.c_void_p(y.data_ptr()), None)
    torch.cuda.synchronize()
    yr = torch.nn.functional.conv2d(x.double().permute(0, 3, 1, 2), wt.double().permute(0, 3, 1, 2), stride=st).permute(0, 2, 3, 1)
    diff = (y.double() - yr).abs()
    print(n, h, cout, k, "fprop err", (diff.max() / yr.abs().max()).item(), "nan", torch.isnan(y).sum().item(),
          "bad frac", (diff > 1e-2 * yr.abs().max()).float().mean().item())
    bad = (diff > 1e-2 * yr.abs().max()).nonzero()
    if len(bad): print("  first bad idx", bad[:5].tolist())
