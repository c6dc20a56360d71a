"""Zero-value-compressed offload (kernels/zvc.cu): lossless round trip of any
bit pattern through a pinned host slot, wire bytes = masks + nonzeros, and a
compressed-offload session that is bit-identical to the copy-engine one."""
import ctypes as C

import numpy as np
import pytest

import paper_1602_08124_b200 as V
from paper_1602_08124_b200 import _lib as L

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


def _pad16(b):
    return (b + 15) // 16 * 16


def _expected_wire(x):
    """Bytes the v2 format moves (zvc.cu): per 1024-value chunk the mask and a
    16-B header, then either the raw nonzeros or -- when the nonzeros' top
    bytes span <= 15 -- their low 3 bytes plus a 4-bit top-byte offset."""
    u = x.view(torch.int32).cpu().numpy().view(np.uint32)
    n = u.size
    u = np.concatenate([u, np.zeros((-n) % 1024, dtype=np.uint32)]).reshape(-1, 1024)
    total = 0
    for row in u:
        nzv = row[row != 0]
        nnz = nzv.size
        top = nzv >> 24
        if nnz and int(top.max()) - int(top.min()) <= 15:
            total += 144 + _pad16(3 * nnz) + _pad16((nnz + 1) // 2)
        else:
            total += 144 + _pad16(4 * nnz)
    return total


def _roundtrip(x):
    n = x.numel()
    lib = L.lib()
    slot = lib.vdnn_kernel_zvc_slot_bytes(C.c_uint64(4 * n))
    host = torch.empty(slot // 4 + 4, dtype=torch.float32).pin_memory()
    host.fill_(float("nan"))  # garbage the decompressor must not read as values
    wire = torch.zeros(2, dtype=torch.int64, device="cuda")
    y = torch.full_like(x, 7.0)
    assert lib.vdnn_kernel_zvc_compress(C.c_void_p(x.data_ptr()), C.c_uint64(n), C.c_void_p(host.data_ptr()),
                                        C.c_void_p(wire.data_ptr()), None) == 0, lib.vdnn_last_error()
    assert lib.vdnn_kernel_zvc_decompress(C.c_void_p(host.data_ptr()), C.c_uint64(n), C.c_void_p(y.data_ptr()),
                                          C.c_void_p(wire.data_ptr() + 8), None) == 0, lib.vdnn_last_error()
    torch.cuda.synchronize()
    assert torch.equal(x.view(torch.int32), y.view(torch.int32)), "round trip not bit-exact"
    w = wire.cpu().tolist()
    assert w[0] == w[1] == _expected_wire(x)
    return w[0]


@pytest.mark.parametrize("n", [4, 1024, 1028, 4096 * 3 + 8, 1 << 20])
def test_zvc_roundtrip_relu_like(n):
    g = torch.Generator(device="cuda").manual_seed(n)
    x = torch.relu(torch.randn(n, device="cuda", generator=g))
    _roundtrip(x)


def test_zvc_special_values():
    vals = torch.tensor([0.0, -0.0, float("nan"), float("inf"), -float("inf"), 1e-45, -1e-45, 3.0] * 512,
                        device="cuda")
    w = _roundtrip(vals)
    # only +0.0 is dropped (-0.0 is a value); mixed signs / exponents: raw mode
    assert w == 4 * 144 + 4 * (vals.numel() - 512)


def test_zvc_all_zero_and_dense():
    z = torch.zeros(1 << 16, device="cuda")
    assert _roundtrip(z) == 144 * 64
    d = torch.rand(1 << 16, device="cuda") + 1.0  # [1, 2): one top byte -> packed mode, 3.5 B per value
    assert _roundtrip(d) == 144 * 64 + 64 * (3072 + 512)


def test_zvc_packed_mode_edge_cases():
    """Top-byte span exactly 15 (packed) and 16 (raw), odd nonzero counts."""
    base = torch.tensor([1.0], device="cuda").view(torch.int32)
    rows = []
    for span, nnz in ((15, 1023), (16, 1001), (0, 1), (7, 3)):
        t = torch.zeros(1024, dtype=torch.int32, device="cuda")
        idx = torch.randperm(1024, device="cuda")[:nnz]
        tops = torch.arange(nnz, device="cuda") % (span + 1)
        vals = (base + (tops << 24) - (0 << 24)) | (torch.arange(nnz, device="cuda", dtype=torch.int32) & 0xFFFFFF)
        t[idx] = vals.to(torch.int32)
        rows.append(t)
    x = torch.cat(rows).view(torch.float32)
    _roundtrip(x)


def _train(g, d, cap, compress, steps=2):
    s = V.Session(g, d, V.CostModel(), cap, compress_offload=compress)
    s.synthetic_batch(7)
    losses = [s.step(0.01) for _ in range(steps)]
    ws = [s.get_weights(l.id) for l in g.layers() if l.kind in (V.LayerKind.Conv, V.LayerKind.Fc)]
    return losses, ws, s.transfer_stats(), s


@pytest.mark.parametrize("net,batch", [("alexnet", 16), ("inception_toy", 16)])
def test_compressed_session_bit_identical(net, batch):
    g = V.build_preset(net, batch)
    d = V.static_decision(V.PolicyKind.VdnnAll, V.AlgoMode.MemoryOptimal, g, V.CostModel())
    cap = 8 << 30
    l0, w0, t0, _ = _train(g, d, cap, False)
    l1, w1, t1, s1 = _train(g, d, cap, True)
    assert l0 == l1
    for a, b in zip(w0, w1):
        assert np.array_equal(a.view(np.int32), b.view(np.int32))
    planned = s1.plan.offload_traffic_bytes
    assert t1["offload_planned"] == t1["prefetch_planned"] == 2 * planned
    assert t0["offload_wire"] == t0["offload_planned"]          # copy engines move the planned bytes
    assert t1["offload_wire"] == t1["prefetch_wire"]             # what went out comes back
    assert t1["offload_wire"] < t1["offload_planned"]            # ReLU maps are sparse
