"""Throughput of the float64 oracle ops on the GPU (sizing the layer-parity samples)."""
import time
import torch
import torch.nn.functional as F


def t(fn, reps=3):
    fn(); torch.cuda.synchronize()
    s = time.time()
    for _ in range(reps):
        fn()
    torch.cuda.synchronize()
    return (time.time() - s) / reps


for (n, c, h, k, co) in [(8, 64, 224, 3, 64), (8, 256, 56, 3, 256), (8, 512, 28, 3, 512)]:
    x = torch.randn(n, c, h, h, dtype=torch.float64, device="cuda")
    w = torch.randn(co, c, k, k, dtype=torch.float64, device="cuda")
    fl = 2 * n * co * h * h * c * k * k
    a = t(lambda: F.conv2d(x, w, padding=1))
    dy = torch.randn(n, co, h, h, dtype=torch.float64, device="cuda")
    b = t(lambda: torch.nn.grad.conv2d_input(x.shape, w, dy, padding=1))
    c2 = t(lambda: torch.nn.grad.conv2d_weight(x, w.shape, dy, padding=1))
    print(f"n{n} c{c} h{h} co{co}: fprop {fl/a/1e12:.2f} TF/s  dgrad {fl/b/1e12:.2f}  wgrad {fl/c2/1e12:.2f}")
a = torch.randn(8192, 8192, dtype=torch.float64, device="cuda")
print("dgemm", 2 * 8192**3 / t(lambda: a @ a) / 1e12, "TF/s")
