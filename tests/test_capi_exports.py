"""The C ABI library loads on a CPU-only host and exports every symbol that
include/vdnn.h declares (no compute calls: those need a GPU)."""
import ctypes as C
import os
import re
import subprocess

from paper_1602_08124_b200 import _lib as L

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared():
    with open(os.path.join(ROOT, "include", "vdnn.h")) as f:
        src = re.sub(r"/\*.*?\*/", "", f.read(), flags=re.S)
    return sorted(set(re.findall(r"\b(vdnn_[a-z0-9_]+)\s*\(", src)))


def test_every_declared_symbol_is_exported():
    lib = L.lib()
    names = declared()
    assert len(names) > 60
    missing = [n for n in names if not hasattr(lib, n)]
    assert missing == [], missing


def test_only_the_c_abi_is_exported():
    out = subprocess.run(["nm", "-D", "--defined-only", L.LIB_PATH], capture_output=True, text=True).stdout
    syms = [l.split()[-1] for l in out.splitlines() if l.strip()]
    assert syms and all(s.startswith("vdnn_") for s in syms), [s for s in syms if not s.startswith("vdnn_")][:5]


def test_errors_are_status_codes_not_crashes():
    lib = L.lib()
    g = C.c_void_p()
    assert lib.vdnn_preset(b"nope", C.c_uint64(4), C.byref(g)) == L.UNKNOWN_PRESET
    assert b"unknown network preset" in lib.vdnn_last_error()
    assert lib.vdnn_extend_vgg(150, C.c_uint64(4), C.byref(g)) == L.INVALID_DEPTH
    assert lib.vdnn_version().startswith(b"vdnn-b200")


def test_session_option_validation_before_any_device_work():
    """Bad transfer-mode options are rejected up front (no GPU needed): the
    Python mirror raises ValueError, the C ABI returns a CONFIG status."""
    import pytest
    import paper_1602_08124_b200 as V
    g = V.build_preset("alexnet", 4)
    d = V.static_decision(V.PolicyKind.VdnnAll, V.AlgoMode.MemoryOptimal, g, V.CostModel())
    with pytest.raises(ValueError):
        V.Session(g, d, compress_offload="bf16")
    with pytest.raises(ValueError):
        V.Session(g, d, offload_target="nvme")
    opt = L.SessionOptions()
    L.lib().vdnn_session_options_default(C.byref(opt))
    assert opt.compress_offload == 0
    opt.compress_offload = 3
    s = C.c_void_p()
    dd = d._handle(g)
    cm = V.CostModel()._c()
    st = L.lib().vdnn_session_create(g.handle, dd.h, C.byref(cm), C.c_uint64(1 << 30), C.byref(opt), C.byref(s))
    assert st != 0 and b"compress_offload" in L.lib().vdnn_last_error()


def test_kernel_entry_points_reject_bad_arguments_without_a_device():
    """The workspace / TF32-exact kernel entry points validate their
    arguments before touching CUDA: a strided dgrad is UNSUPPORTED, null
    buffers are INVALID_ARGUMENT."""
    lib = L.lib()
    d = L.ConvDesc()
    d.n, d.h, d.w, d.nseg = 2, 8, 8, 1
    d.c[0] = 32
    d.cout, d.kh, d.kw, d.stride, d.pad = 32, 3, 3, 2, 1
    assert lib.vdnn_kernel_conv_dgrad_ws(C.byref(d), None, None, 0, None, C.c_size_t(0), None) == L.UNSUPPORTED
    assert lib.vdnn_kernel_zvc_compress_tf32(None, C.c_uint64(4), None, None, None) == L.INVALID_ARGUMENT
    assert b"null" in lib.vdnn_last_error()
