"""ctypes binding of libvdnn.so (include/vdnn.h).

The shared library is built in-tree (``paper_1602_08124_b200/libvdnn.so``) by
``__graft_entry__.build()`` / ``make -C paper_1602_08124_b200/csrc``. There is
no fallback: if the library is missing every call fails loudly.
"""
from __future__ import annotations

import ctypes as C
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libvdnn.so")

_lib = None


class VdnnError(RuntimeError):
    """Raised for a non-OK vdnn_status; ``status`` holds the code."""

    def __init__(self, status: int, msg: str):
        super().__init__(f"vdnn status {status}: {msg}")
        self.status = status


# Status codes mirror the reference's exception hierarchy (core.hpp:21-32).
OK = 0
ERROR = 1
SHAPE_MISMATCH = 2
UNKNOWN_PRESET = 3
INVALID_DEPTH = 4
OVERFLOW = 5
WRONG_LAYER_KIND = 6
POOL_MISUSE = 7
INVALID_DECISION = 8
CONFIG_ERROR = 9
CUDA_ERROR = 10
NCCL_ERROR = 11
UNSUPPORTED = 12
INVALID_ARGUMENT = 13


class LayerInfo(C.Structure):
    _fields_ = [
        ("id", C.c_int32), ("kind", C.c_int32), ("join", C.c_int32), ("n_inputs", C.c_int32),
        ("inputs", C.c_int32 * 16),
        ("p0", C.c_uint64), ("p1", C.c_uint64), ("p2", C.c_uint64), ("p3", C.c_uint64),
        ("n", C.c_uint64), ("c", C.c_uint64), ("h", C.c_uint64), ("w", C.c_uint64),
        ("refcnt", C.c_int32),
    ]


class CostModelC(C.Structure):
    _fields_ = [
        ("peak_flops", C.c_double), ("dram_bw", C.c_double), ("mem_capacity", C.c_uint64),
        ("compute_efficiency", C.c_double), ("link_effective_bw", C.c_double),
        ("link_nominal_bw", C.c_double), ("link_launch_overhead", C.c_double),
        ("elem_size", C.c_uint64), ("bwd_fwd_ratio", C.c_double),
        ("speed_factor_implicit_gemm", C.c_double), ("speed_factor_gemm_ws", C.c_double),
        ("speed_factor_fft", C.c_double), ("n_overrides", C.c_int32),
        ("override_layer", C.POINTER(C.c_int32)), ("override_fwd_s", C.POINTER(C.c_double)),
        ("override_bwd_s", C.POINTER(C.c_double)),
    ]


class Footprint(C.Structure):
    _fields_ = [(n, C.c_uint64) for n in (
        "weights_bytes", "feature_maps_bytes", "gradient_buffers_bytes", "workspace_bytes",
        "total_bytes", "classifier_bytes")]


class Event(C.Structure):
    _fields_ = [
        ("stream", C.c_int32), ("kind", C.c_int32), ("layer", C.c_int32), ("buffer", C.c_int32),
        ("start_ns", C.c_int64), ("end_ns", C.c_int64), ("bytes", C.c_uint64), ("offset", C.c_uint64),
        ("tag", C.c_char * 4),
    ]


class ReportSummary(C.Structure):
    _fields_ = [
        ("pass_", C.c_int32), ("has_oom", C.c_int32), ("oom_layer", C.c_int32), ("oom_phase", C.c_int32),
        ("oom_fragmented", C.c_int32), ("oom_requested", C.c_uint64), ("oom_tag", C.c_char * 4),
        ("max_mem_bytes", C.c_uint64), ("avg_mem_bytes", C.c_uint64), ("offload_traffic_bytes", C.c_uint64),
        ("prefetch_traffic_bytes", C.c_uint64), ("host_peak_bytes", C.c_uint64),
        ("stall_fwd_offload_ns", C.c_int64), ("stall_bwd_prefetch_ns", C.c_int64), ("total_ns", C.c_int64),
        ("interference_bound", C.c_double), ("n_events", C.c_uint64), ("verdict", C.c_char * 96),
    ]


class PoolTraceRow(C.Structure):
    _fields_ = [
        ("time_ns", C.c_int64), ("op", C.c_char), ("tag", C.c_char * 4), ("offset", C.c_uint64),
        ("bytes", C.c_uint64), ("current", C.c_uint64), ("high_water", C.c_uint64),
    ]


class PassInfo(C.Structure):
    _fields_ = [
        ("phase", C.c_char * 16), ("label", C.c_char * 64), ("pass_", C.c_int32), ("has_oom", C.c_int32),
        ("oom_layer", C.c_int32), ("oom_phase", C.c_int32), ("total_ns", C.c_int64),
        ("max_mem_bytes", C.c_uint64),
    ]


class Violation(C.Structure):
    _fields_ = [("kind", C.c_char * 32), ("detail", C.c_char * 160)]


class SessionOptions(C.Structure):
    _fields_ = [
        ("device", C.c_int32), ("weight_seed", C.c_uint64), ("external_grads", C.c_int32),
        ("record_timeline", C.c_int32), ("host_arena", C.c_int32), ("precise_fp32", C.c_int32),
        ("compress_offload", C.c_int32), ("offload_target", C.c_int32), ("cuda_graph", C.c_int32),
        ("algo_kernels", C.c_int32),
    ]


class ProbeSeg(C.Structure):
    _fields_ = [("what", C.c_int32), ("index", C.c_int32), ("after", C.c_int32), ("pad_", C.c_int32),
                ("offset", C.c_uint64), ("bytes", C.c_uint64)]


PROBE_MAX_SEGS = 40


class ProbeLayout(C.Structure):
    """vdnn_probe_layout: segments of a layer-local probe and the fusions the step applies."""
    _fields_ = [("nseg", C.c_int32), ("relu_fused", C.c_int32), ("accumulate", C.c_int32), ("skip", C.c_int32),
                ("mask_planes", C.c_uint32), ("pad_", C.c_uint32), ("total_bytes", C.c_uint64),
                ("seg", ProbeSeg * PROBE_MAX_SEGS)]


class PeerHandle(C.Structure):
    """vdnn_peer_handle: three CUDA IPC handles + the layout they must agree on."""
    _fields_ = [
        ("arena", C.c_uint8 * 64), ("grads", C.c_uint8 * 64), ("signal", C.c_uint8 * 64),
        ("arena_lo", C.c_uint64), ("arena_bytes", C.c_uint64), ("grads_count", C.c_uint64),
    ]


class ConvDesc(C.Structure):
    _fields_ = [
        ("n", C.c_int32), ("h", C.c_int32), ("w", C.c_int32), ("nseg", C.c_int32),
        ("x", C.c_void_p * 8), ("dx", C.c_void_p * 8), ("c", C.c_int32 * 8),
        ("cout", C.c_int32), ("kh", C.c_int32), ("kw", C.c_int32), ("stride", C.c_int32), ("pad", C.c_int32),
    ]


def lib() -> C.CDLL:
    """Load libvdnn.so (raises if it was not built)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise VdnnError(ERROR, f"{LIB_PATH} missing: run __graft_entry__.build() first")
        _lib = C.CDLL(LIB_PATH)
        _lib.vdnn_last_error.restype = C.c_char_p
        _lib.vdnn_version.restype = C.c_char_p
        _lib.vdnn_kernel_launch_count.restype = C.c_uint64
        _lib.vdnn_kernel_conv_wgrad_ws_bytes.restype = C.c_size_t
        _lib.vdnn_kernel_conv_wgrad_ws_bytes.argtypes = [C.c_void_p]
        _lib.vdnn_kernel_conv_fprop_ws_bytes.restype = C.c_size_t
        _lib.vdnn_kernel_conv_fprop_ws_bytes.argtypes = [C.c_void_p]
        _lib.vdnn_kernel_conv_dgrad_ws_bytes.restype = C.c_size_t
        _lib.vdnn_kernel_conv_dgrad_ws_bytes.argtypes = [C.c_void_p]
        _lib.vdnn_kernel_set_precise.restype = None
        _lib.vdnn_kernel_set_precise.argtypes = [C.c_int32]
        _lib.vdnn_kernel_set_tma.restype = None
        _lib.vdnn_kernel_set_tma.argtypes = [C.c_int32]
        _lib.vdnn_kernel_tf32_peak.argtypes = [C.POINTER(C.c_double)]
        _lib.vdnn_kernel_zvc_slot_bytes.restype = C.c_uint64
        _lib.vdnn_kernel_zvc_slot_bytes.argtypes = [C.c_uint64]
        _lib.vdnn_kernel_zvc_compress.argtypes = [C.c_void_p, C.c_uint64, C.c_void_p, C.c_void_p, C.c_void_p]
        _lib.vdnn_kernel_zvc_compress_tf32.argtypes = [C.c_void_p, C.c_uint64, C.c_void_p, C.c_void_p, C.c_void_p]
        _lib.vdnn_kernel_zvc_decompress.argtypes = [C.c_void_p, C.c_uint64, C.c_void_p, C.c_void_p, C.c_void_p]
        if hasattr(_lib, "vdnn_session_plan"):
            _lib.vdnn_session_plan.restype = C.c_void_p
            _lib.vdnn_session_plan.argtypes = [C.c_void_p]
        for name in ("vdnn_graph_destroy", "vdnn_decision_destroy", "vdnn_report_destroy",
                     "vdnn_dyn_destroy", "vdnn_session_destroy"):
            if hasattr(_lib, name):
                getattr(_lib, name).restype = None
                getattr(_lib, name).argtypes = [C.c_void_p]
        if hasattr(_lib, "vdnn_cost_model_default"):
            _lib.vdnn_cost_model_default.restype = None
    return _lib


def check(status: int) -> None:
    if status != OK:
        raise VdnnError(status, lib().vdnn_last_error().decode(errors="replace"))


def call(name: str, *args) -> None:
    check(getattr(lib(), name)(*args))
