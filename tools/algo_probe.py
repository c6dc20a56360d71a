"""Measured time per convolution algorithm on the B200: the
reference's cost model picks, per CONV layer, implicit GEMM (no workspace),
GEMM_WS (an im2col buffer, `cost_model.hpp:163-168`) or FFT (frequency planes
padded to powers of two, `:169-175`), with speed factors 1.0 / 0.8 / 0.6 of a
Titan X. The executor reserves each layer's planned workspace (memory
semantics unchanged) and always runs the tcgen05 implicit-GEMM kernel; this
probe measures why, forward pass of the VGG-16 layer shapes:

  implicit : vdnn_kernel_conv_fprop (tcgen05 implicit GEMM, TF32)
  gemm_ws  : im2col into the workspace (the buffer the reference sizes) +
             the same engine as a 1x1 GEMM over it (vdnn_kernel_conv_fprop,
             kh = kw = 1, C = k*k*Cin)
  fft      : rfft2 of the input planes padded to powers of two, the
             per-frequency complex channel contraction, irfft2 (torch.fft /
             torch.matmul -- cuFFT + cuBLAS, a probe only: nothing here runs
             on the product path)

    python tools/algo_probe.py [batch]
"""
import ctypes as C
import sys

sys.path.insert(0, ".")
import torch

from paper_1602_08124_b200 import _lib as L

dev = torch.device("cuda")
batch = int(sys.argv[1]) if len(sys.argv) > 1 else 32
shapes = [(224, 64, 64), (112, 128, 128), (56, 256, 256), (28, 512, 512), (14, 512, 512)]


def timeit(fn, n=5):
    fn()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(n):
        fn()
    e.record()
    e.synchronize()
    return s.elapsed_time(e) / n


def desc(n, h, w, c, co, k, pad, x, dx=None):
    d = L.ConvDesc()
    d.n, d.h, d.w, d.nseg = n, h, w, 1
    d.x[0] = x.data_ptr()
    d.dx[0] = dx.data_ptr() if dx is not None else 0
    d.c[0] = c
    d.cout, d.kh, d.kw, d.stride, d.pad = co, k, k, 1, pad
    return d


print(f"VGG-16 conv forward, batch {batch}, TF32 (ms; workspace GB as the reference sizes it at this batch)")
print(f"{'layer':>18} {'implicit':>9} {'gemm_ws':>9} {'(im2col':>8} {'gemm)':>7} {'ws GB':>6} {'fft':>9} {'ws GB':>6}")
for hw, c, co in shapes:
    n = batch
    x = torch.randn(n, hw, hw, c, device=dev)
    wt = torch.randn(co, 3, 3, c, device=dev) * 0.05
    y = torch.empty(n, hw, hw, co, device=dev)
    d = desc(n, hw, hw, c, co, 3, 1, x)
    t_imp = timeit(lambda: L.call("vdnn_kernel_conv_fprop", C.byref(d), C.c_void_p(wt.data_ptr()), None,
                                  C.c_void_p(y.data_ptr()), None))
    # GEMM_WS: im2col [n*hw*hw][9*c] (tap-major, channel-minor: the KRSC weight row order)
    col = torch.empty(n, hw, hw, 9, c, device=dev)
    xp = torch.nn.functional.pad(x, (0, 0, 1, 1, 1, 1))

    def im2col():
        for r in range(3):
            for s in range(3):
                col[:, :, :, r * 3 + s, :] = xp[:, r:r + hw, s:s + hw, :]

    d1 = desc(n * hw * hw, 1, 1, 9 * c, co, 1, 0, col)
    y1 = torch.empty_like(y)
    t_col = timeit(im2col)
    t_gemm = timeit(lambda: L.call("vdnn_kernel_conv_fprop", C.byref(d1), C.c_void_p(wt.data_ptr()), None,
                                   C.c_void_p(y1.data_ptr()), None))
    im2col()
    L.call("vdnn_kernel_conv_fprop", C.byref(d1), C.c_void_p(wt.data_ptr()), None, C.c_void_p(y1.data_ptr()), None)
    L.call("vdnn_kernel_conv_fprop", C.byref(d), C.c_void_p(wt.data_ptr()), None, C.c_void_p(y.data_ptr()), None)
    torch.cuda.synchronize()
    rel = ((y1 - y).norm() / y.norm()).item()
    ws_gemm = 9 * c * hw * hw * n * 4 / 1e9
    del col
    # FFT: planes padded to the next power of two (the reference's workspace model)
    ph = 1 << (hw - 1).bit_length()
    xn = x.permute(0, 3, 1, 2)
    wn = wt.permute(0, 3, 1, 2)

    def fft_conv():
        xf = torch.fft.rfft2(xn, s=(ph, ph))                       # [n, c, ph, ph/2+1]
        wf = torch.fft.rfft2(torch.flip(wn, (2, 3)), s=(ph, ph))   # [co, c, ph, ph/2+1]
        yf = torch.einsum("ncuv,kcuv->nkuv", xf, wf)               # per-frequency channel contraction
        return torch.fft.irfft2(yf, s=(ph, ph))

    try:
        t_fft = timeit(fft_conv, n=3)
    except torch.OutOfMemoryError:
        t_fft = float("nan")
    torch.cuda.empty_cache()
    ws_fft = 2 * max(c, co) * ph * ph * n * 4 / 1e9
    print(f"{hw:>3}x{hw:<3} {c:>4}->{co:<4} {t_imp:9.3f} {t_col + t_gemm:9.3f} {t_col:8.3f} {t_gemm:7.3f} "
          f"{ws_gemm:6.2f} {t_fft:9.3f} {ws_fft:6.2f}   (gemm_ws vs implicit rel {rel:.1e})")
