"""ORACLE ONLY: ctypes access to the compiled reference simulator.

The library is built by ``make -C oracle`` from the reference's own headers
(read in place under /root/reference, never copied). It travels to the GPU box
as a prebuilt .so; nothing here reads /root/reference at run time.
"""
from __future__ import annotations

import ctypes as C
import json
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB = os.path.join(_HERE, "_ref", "libvdnnref.so")
_lib = None

TAGS = ["", "W", "dW", "X", "Y", "dX", "WS", "G2"]


def available() -> bool:
    return os.path.exists(LIB)


def lib():
    global _lib
    if _lib is None:
        _lib = C.CDLL(LIB)
        for n in ("vref_run", "vref_preset_spec", "vref_replay", "vref_fuzz", "vref_fuzz_graph"):
            getattr(_lib, n).restype = C.c_void_p
        _lib.vref_free.argtypes = [C.c_void_p]
        _lib.vref_time_plan.restype = C.c_double
        _lib.vref_time_plan.argtypes = [C.c_char_p, C.c_ulonglong, C.c_int]
    return _lib


def _take(p) -> str:
    s = C.cast(p, C.c_char_p).value.decode()
    lib().vref_free(p)
    return s


def preset_spec(name: str, batch: int, extra: int = 0) -> str:
    s = _take(lib().vref_preset_spec(name.encode(), C.c_ulonglong(batch), int(extra)))
    if s.startswith("ERROR:"):
        raise RuntimeError(s)
    return s


def run(graph_spec: str, dec_spec: str, capacity: int, cost_spec: str = "", events: bool = True,
        weight_grads: bool = False) -> dict:
    flags = (1 if events else 0) | (2 if weight_grads else 0)
    out = json.loads(_take(lib().vref_run(graph_spec.encode(), cost_spec.encode(), dec_spec.encode(),
                                          C.c_ulonglong(capacity), flags)))
    if "error" in out:
        raise RuntimeError(out["error"])
    return out


def replay(graph_spec: str, dec_spec: str, capacity: int, events, max_mem: int, avg_mem: int, total_ns: int,
           passed: bool):
    """Reference replay_check over an event list of (stream, kind, layer, start, end, bytes, tag, buffer, offset)."""
    n = len(events)
    arr = (C.c_longlong * (9 * max(n, 1)))()
    for i, e in enumerate(events):
        s, k, l, a, b, by, tag, buf, off = e
        arr[9 * i: 9 * i + 9] = [int(s), int(k), int(l), int(a), int(b), int(by), TAGS.index(tag), int(buf), int(off)]
    out = json.loads(_take(lib().vref_replay(graph_spec.encode(), dec_spec.encode(), C.c_ulonglong(capacity), arr,
                                             C.c_longlong(n), C.c_ulonglong(max_mem), C.c_ulonglong(avg_mem),
                                             C.c_longlong(total_ns), int(passed))))
    if isinstance(out, dict) and "error" in out:
        raise RuntimeError(out["error"])
    return out


def fuzz_graph(seed: int, max_layers: int = 12) -> str:
    """Graph spec of the reference fuzz generator (fuzz.hpp:26-63) for `seed`."""
    s = _take(lib().vref_fuzz_graph(C.c_ulonglong(seed), int(max_layers)))
    if s.startswith("ERROR:"):
        raise RuntimeError(s)
    return s


def fuzz(seed: int, trials: int) -> dict:
    return json.loads(_take(lib().vref_fuzz(C.c_ulonglong(seed), int(trials))))


def time_plan(graph_spec: str, capacity: int, iters: int) -> float:
    """Seconds per reference dynamic_select + simulate (single thread)."""
    return lib().vref_time_plan(graph_spec.encode(), C.c_ulonglong(capacity), int(iters))


# ---- front-end / artefact formats (oracle/_ref/libvdnnref_fmt.so, needs nlohmann) ----
LIB_FMT = os.path.join(_HERE, "_ref", "libvdnnref_fmt.so")
_fmt = None


def fmt_available() -> bool:
    return os.path.exists(LIB_FMT)


def _fmt_lib():
    global _fmt
    if _fmt is None:
        _fmt = C.CDLL(LIB_FMT)
        for n in ("vref_fmt_config", "vref_fmt_graph_to_json", "vref_fmt_graph_from_json", "vref_fmt_report"):
            getattr(_fmt, n).restype = C.c_void_p
        _fmt.vref_fmt_free.argtypes = [C.c_void_p]
    return _fmt


def _fmt_take(p) -> str:
    s = C.cast(p, C.c_char_p).value.decode()
    _fmt_lib().vref_fmt_free(p)
    return s


def fmt_config(path: str) -> dict:
    """Reference load_config(path) + build_network: all fields, graph as a spec (or error)."""
    return json.loads(_fmt_take(_fmt_lib().vref_fmt_config(path.encode())))


def fmt_graph_to_json(graph_spec: str) -> dict:
    return json.loads(_fmt_take(_fmt_lib().vref_fmt_graph_to_json(graph_spec.encode())))


def fmt_graph_from_json(text: str) -> str:
    """Reference graph_from_json -> spec (or a JSON error object string)."""
    return _fmt_take(_fmt_lib().vref_fmt_graph_from_json(text.encode()))


def fmt_report(graph_spec: str, capacity: int) -> dict:
    """Reference decision_to_json + report_to_json of dynamic_select/simulate."""
    return json.loads(_fmt_take(_fmt_lib().vref_fmt_report(graph_spec.encode(), C.c_ulonglong(capacity))))
