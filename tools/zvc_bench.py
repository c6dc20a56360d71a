"""Throughput of the zero-value-compressed transfer kernels alone (1 GiB
ReLU-like buffer, ~50% zeros): raw-equivalent and wire GB/s per direction."""
import ctypes as C, sys
sys.path.insert(0, ".")
import torch
from paper_1602_08124_b200 import _lib as L

lib = L.lib()
n = 1 << 28
x = torch.relu(torch.randn(n, device="cuda"))
for dens in (0.5, 1.0):
    if dens == 1.0:
        x = torch.rand(n, device="cuda") + 1
    slot = lib.vdnn_kernel_zvc_slot_bytes(C.c_uint64(4 * n))
    host = torch.empty(slot // 4 + 4, dtype=torch.float32).pin_memory()
    wire = torch.zeros(2, dtype=torch.int64, device="cuda")
    y = torch.empty_like(x)
    def comp():
        lib.vdnn_kernel_zvc_compress(C.c_void_p(x.data_ptr()), C.c_uint64(n), C.c_void_p(host.data_ptr()), C.c_void_p(wire.data_ptr()), None)
    def dec():
        lib.vdnn_kernel_zvc_decompress(C.c_void_p(host.data_ptr()), C.c_uint64(n), C.c_void_p(y.data_ptr()), C.c_void_p(wire.data_ptr() + 8), None)
    for name, fn in (("compress", comp), ("decompress", dec)):
        fn(); torch.cuda.synchronize()
        wire.zero_()
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record(); fn(); e.record(); e.synchronize()
        ms = s.elapsed_time(e)
        w = int(wire[0 if name == "compress" else 1])
        print(f"density {dens:.1f} {name:10s} {ms:7.2f} ms  raw {4 * n / ms / 1e6:6.1f} GB/s  wire {w / ms / 1e6:5.1f} GB/s")
