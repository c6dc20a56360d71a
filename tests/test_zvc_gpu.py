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


def _chunk_modes(x, tf32=False):
    """Per 1024-value chunk: (mode, nnz) as zvc.cu chooses them."""
    u = x.view(torch.int32).cpu().numpy().view(np.uint32)
    n = u.size
    u = np.concatenate([u, np.zeros((-n) % 1024, dtype=np.uint32)]).reshape(-1, 1024)
    out = []
    for row in u:
        nzv = row[row != 0]
        nnz = nzv.size
        top = nzv >> 24
        inexact = bool(np.any((nzv & 0x7FFFE000) == 0) or np.any((nzv & 0x7F800000) == 0x7F800000))
        if nnz and int(top.max()) - int(top.min()) <= 15:
            out.append((2 if tf32 and not inexact else 1, nnz))
        else:
            out.append((0, nnz))
    return out


def _expected_wire(x, tf32=False):
    """Bytes the v2 format moves (zvc.cu): per 1024-value chunk the mask and a
    16-B header, then either the raw nonzeros, or -- when the nonzeros' top
    bytes span <= 15 -- their low 3 bytes plus a 4-bit top-byte offset, or
    (TF32-exact transfers) one u16 per nonzero."""
    total = 0
    for mode, nnz in _chunk_modes(x, tf32):
        total += 144 + (_pad16(2 * nnz) if mode == 2 else
                        _pad16(3 * nnz) + _pad16((nnz + 1) // 2) if mode == 1 else _pad16(4 * nnz))
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


def _roundtrip_tf32(x):
    """TF32-exact transfer: mode-2 chunks come back with the low 13 mantissa
    bits cleared, every other chunk bit-exact; wire bytes per the model."""
    n = x.numel()
    lib = L.lib()
    slot = lib.vdnn_kernel_zvc_slot_bytes(C.c_uint64(4 * n))
    host = torch.empty(slot // 4 + 4, dtype=torch.float32).pin_memory()
    host.fill_(float("nan"))
    wire = torch.zeros(2, dtype=torch.int64, device="cuda")
    y = torch.full_like(x, 7.0)
    assert lib.vdnn_kernel_zvc_compress_tf32(C.c_void_p(x.data_ptr()), C.c_uint64(n), C.c_void_p(host.data_ptr()),
                                             C.c_void_p(wire.data_ptr()), None) == 0, lib.vdnn_last_error()
    assert lib.vdnn_kernel_zvc_decompress(C.c_void_p(host.data_ptr()), C.c_uint64(n), C.c_void_p(y.data_ptr()),
                                          C.c_void_p(wire.data_ptr() + 8), None) == 0, lib.vdnn_last_error()
    torch.cuda.synchronize()
    modes = _chunk_modes(x, tf32=True)
    xi = x.view(torch.int32).cpu()
    want = xi.clone()
    for c, (mode, _) in enumerate(modes):
        if mode == 2:
            want[c * 1024:(c + 1) * 1024] &= ~0x1FFF
    assert torch.equal(y.view(torch.int32).cpu(), want)
    w = wire.cpu().tolist()
    assert w[0] == w[1] == _expected_wire(x, tf32=True)
    return w[0], modes


@pytest.mark.parametrize("n", [1024, 4096 * 3 + 8, 1 << 20])
def test_zvc_tf32_exact_relu_like(n):
    g = torch.Generator(device="cuda").manual_seed(n + 1)
    x = torch.relu(torch.randn(n, device="cuda", generator=g))
    w, modes = _roundtrip_tf32(x)
    assert all(m == 2 for m, nnz in modes if nnz)
    assert w < _expected_wire(x)  # 2 B per nonzero instead of 3.5


def test_zvc_tf32_exact_keeps_denormals_and_specials_lossless():
    """Chunks whose top bytes span <= 15 but that hold a nonzero TF32
    truncation cannot represent stay in the lossless packed mode: a positive
    denormal next to tiny normals (truncation would zero it and flip the ReLU
    mask), +Inf / a NaN payload next to huge normals."""
    g = torch.Generator(device="cuda").manual_seed(3)
    r = torch.rand(4096, device="cuda", generator=g) + 1.0
    x = torch.cat([r[:1024] * 2.0 ** -120, r[1024:2048] * 2.0 ** 120, r[2048:3072] * 2.0 ** 120,
                   torch.relu(r[3072:] - 1.5)])
    xi = x.view(torch.int32)
    xi[5] = 1                   # positive denormal
    xi[1024 + 7] = 0x7F800000   # +Inf
    xi[2048 + 9] = 0x7FC00001   # NaN with a payload
    _, modes = _roundtrip_tf32(x)
    assert [m for m, _ in modes] == [1, 1, 1, 2]


def test_tf32_operands_truncate():
    """The premise of TF32-exact transfers: the tensor core ignores the 13 low
    mantissa bits of fp32 operands, so a conv on X and on X with those bits
    cleared gives bit-identical fprop and wgrad outputs."""
    dev = torch.device("cuda")
    g = torch.Generator(device=dev).manual_seed(2)
    n, h, c, co = 4, 28, 64, 128
    x = torch.relu(torch.randn(n, h, h, c, device=dev, generator=g))
    xt = (x.view(torch.int32) & ~0x1FFF).view(torch.float32)
    wt = torch.randn(co, 3, 3, c, device=dev, generator=g) * 0.05
    dy = torch.randn(n, h, h, co, device=dev, generator=g)
    outs = []
    for xx in (x, xt):
        d = L.ConvDesc()
        d.n, d.h, d.w, d.nseg = n, h, h, 1
        d.x[0] = xx.data_ptr()
        d.c[0] = c
        d.cout, d.kh, d.kw, d.stride, d.pad = co, 3, 3, 1, 1
        y = torch.empty(n, h, h, co, device=dev)
        L.call("vdnn_kernel_conv_fprop", C.byref(d), C.c_void_p(wt.data_ptr()), None, C.c_void_p(y.data_ptr()), None)
        wsb = L.lib().vdnn_kernel_conv_wgrad_ws_bytes(C.byref(d))
        ws = torch.empty(max(wsb // 4, 1), device=dev)
        dw = torch.empty_like(wt)
        L.call("vdnn_kernel_conv_wgrad", C.byref(d), C.c_void_p(dy.data_ptr()), C.c_void_p(wt.data_ptr()),
               C.c_float(0.0), C.c_void_p(dw.data_ptr()), C.c_void_p(ws.data_ptr()), C.c_size_t(wsb), None)
        torch.cuda.synchronize()
        outs.append((y, dw))
    assert torch.equal(outs[0][0], outs[1][0])
    assert torch.equal(outs[0][1], outs[1][1])


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


@pytest.mark.parametrize("net,batch", [("alexnet", 16), ("inception_toy", 16)])
def test_tf32_exact_session_bit_identical(net, batch):
    """compress_offload="tf32": maps read in backward only by TF32
    contractions and ReLU masks travel TF32-exact; losses and weights after
    two steps equal the copy-engine run bit for bit, with fewer wire bytes
    than the lossless format."""
    g = V.build_preset(net, batch)
    d = V.static_decision(V.PolicyKind.VdnnAll, V.AlgoMode.MemoryOptimal, g, V.CostModel())
    cap = 8 << 30
    l0, w0, _, _ = _train(g, d, cap, False)
    _, _, t1, _ = _train(g, d, cap, True)
    l2, w2, t2, _ = _train(g, d, cap, "tf32")
    assert l0 == l2
    for a, b in zip(w0, w2):
        assert np.array_equal(a.view(np.int32), b.view(np.int32))
    assert t2["offload_wire"] == t2["prefetch_wire"]
    assert t2["offload_wire"] < t1["offload_wire"]


# ------------------------------------------------------------------ BF16 ----
# BF16 maps (elem_size = 2, kernels/zvc.cu zvcb_*): per 2048-bf16 chunk a
# 256-B mask + 16-B header, then the nonzeros as u16 or -- when their top
# bytes span <= 15 -- one low byte each plus a 4-bit top-byte offset.

def _expected_wire_bf16(bits):
    u = bits.cpu().numpy().view(np.uint16)
    n = u.size
    u = np.concatenate([u, np.zeros((-n) % 2048, dtype=np.uint16)]).reshape(-1, 2048)
    total = 0
    for row in u:
        nzv = row[row != 0]
        nnz = nzv.size
        top = nzv >> 8
        if nnz and int(top.max()) - int(top.min()) <= 15:
            total += 272 + _pad16(nnz) + _pad16((nnz + 1) // 2)
        else:
            total += 272 + _pad16(2 * nnz)
    return total


def _roundtrip_bf16(bits):
    """bits: int16 CUDA tensor of bf16 bit patterns (numel % 8 == 0)."""
    n = bits.numel()
    lib = L.lib()
    slot = lib.vdnn_kernel_zvc_slot_bytes_bf16(C.c_uint64(2 * n))
    host = torch.empty(slot // 4 + 4, dtype=torch.float32).pin_memory()
    host.fill_(float("nan"))
    wire = torch.zeros(2, dtype=torch.int64, device="cuda")
    y = torch.full_like(bits, 0x3F80)
    assert lib.vdnn_kernel_zvc_compress_bf16(C.c_void_p(bits.data_ptr()), C.c_uint64(n), C.c_void_p(host.data_ptr()),
                                             C.c_void_p(wire.data_ptr()), None) == 0, lib.vdnn_last_error()
    assert lib.vdnn_kernel_zvc_decompress_bf16(C.c_void_p(host.data_ptr()), C.c_uint64(n), C.c_void_p(y.data_ptr()),
                                               C.c_void_p(wire.data_ptr() + 8), None) == 0, lib.vdnn_last_error()
    torch.cuda.synchronize()
    assert torch.equal(bits, y), "bf16 round trip not bit-exact"
    w = wire.cpu().tolist()
    assert w[0] == w[1] == _expected_wire_bf16(bits)
    return w[0]


def _relu_bits(n, seed=0):
    g = torch.Generator(device="cuda").manual_seed(seed)
    x = torch.relu(torch.randn(n, device="cuda", generator=g)).to(torch.bfloat16)
    return x.view(torch.int16).contiguous()


@pytest.mark.parametrize("n", [8, 2048, 2056, 2048 * 5 + 16, 1 << 20])
def test_zvc_bf16_roundtrip_relu_like(n):
    w = _roundtrip_bf16(_relu_bits(n, n))
    if n >= 2048:
        assert w < 2 * n * 0.6  # about half zeros: mask + 1.5 B per nonzero


def test_zvc_bf16_special_values_and_modes():
    # -0.0, NaN, Inf, denormals are values (only 0x0000 is a zero); a chunk with
    # a wide exponent span takes the u16 mode, a narrow one the packed mode
    specials = torch.tensor([0x8000, 0x7FC0, 0x7F80, 0xFF80, 0x0001, 0x807F, 0x3F80, 0x0000], dtype=torch.int32)
    specials = (specials - (specials > 32767).to(torch.int32) * 65536).to(torch.int16)
    wide = specials.repeat(2048 // 8 * 3).cuda()
    _roundtrip_bf16(wide)
    narrow = torch.full((4096,), 0x3F81, dtype=torch.int16, device="cuda")
    narrow[::3] = 0
    narrow[1::7] = 0x4000
    _roundtrip_bf16(narrow)
    _roundtrip_bf16(torch.zeros(2048 * 2, dtype=torch.int16, device="cuda"))       # all zero: 272 B a chunk
    _roundtrip_bf16(torch.full((2048 * 2,), 0x4049, dtype=torch.int16, device="cuda"))  # dense, one top byte
    odd = _relu_bits(2048 + 8, 3)
    odd[-1] = 0x3F80  # a chunk whose nonzero count is odd at the end
    _roundtrip_bf16(odd)


def test_zvc_bf16_rejects_bad_arguments():
    lib = L.lib()
    x = torch.zeros(16, dtype=torch.int16, device="cuda")
    assert lib.vdnn_kernel_zvc_compress_bf16(C.c_void_p(x.data_ptr()), C.c_uint64(12), None, None, None) == \
        L.INVALID_ARGUMENT


@pytest.mark.parametrize("net,batch", [("alexnet", 16), ("inception_toy", 16)])
def test_compressed_session_bit_identical_bf16(net, batch):
    """BF16 storage (elem_size = 2) with lossless compressed transfers: losses
    and weights after two steps equal the copy-engine BF16 run bit for bit."""
    g = V.build_preset(net, batch)
    cm = V.CostModel()
    cm.elem_size = 2
    d = V.static_decision(V.PolicyKind.VdnnAll, V.AlgoMode.MemoryOptimal, g, cm)
    cap = 8 << 30

    def run(compress):
        s = V.Session(g, d, cm, cap, compress_offload=compress)
        s.synthetic_batch(7)
        losses = [s.step(0.01) for _ in range(2)]
        ws = [s.get_weights(l.id) for l in g.layers() if l.kind in (V.LayerKind.Conv, V.LayerKind.Fc)]
        return losses, ws, s.transfer_stats()

    l0, w0, t0 = run(False)
    l1, w1, t1 = run(True)
    assert l0 == l1
    for a, b in zip(w0, w1):
        assert np.array_equal(a.view(np.int32), b.view(np.int32))
    assert t1["offload_wire"] == t1["prefetch_wire"]
    assert t1["offload_wire"] < t1["offload_planned"]
    with pytest.raises(V.VdnnError):
        V.Session(g, d, cm, cap, compress_offload="tf32")
