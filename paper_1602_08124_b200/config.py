"""INI experiment configs and inline-layer networks: the reference's
front-end (vdnnsim/config.hpp) restated on this package's API.

* ``parse_bytes`` / ``parse_rate`` ........ config.hpp:22-47
* ``ExperimentConfig`` .................... config.hpp:49-63
* ``load_config`` ([network] [device] [link] [latencies] [policy]) .. config.hpp:66-185
* ``parse_inline_layer`` .................. config.hpp:189-234
* ``build_network`` (preset, vggN, inline list, graph .json, nested .conf,
  $VDNN_SIM_EXPERIMENTS lookup) ........... config.hpp:236-269

The result feeds the same planner / B200 session as any hand-built graph.
Parity with the compiled reference is tested in tests/test_formats.py.
"""
from __future__ import annotations

import json
import os
import re
from dataclasses import dataclass, field
from typing import Dict, List, Optional, Tuple

from . import api as V

_NUM = re.compile(r"\s*[+-]?(?:inf(?:inity)?|nan|(?:\d+\.?\d*|\.\d+)(?:[eE][+-]?\d+)?)", re.I)


def _stod(s: str) -> float:
    """std::stod: longest leading decimal number; no number -> error."""
    m = _NUM.match(s)
    if not m:
        raise ValueError(s)
    return float(m.group(0))


def parse_bytes(s: str) -> int:
    """config.hpp:22-44 (decimal KB/MB/GB, binary KiB/MiB/GiB, B, scientific)."""
    if s in ("unlimited", "inf"):
        return V.KUNLIMITED_BYTES
    mult = 1.0
    for suf, m in (("GiB", 1073741824.0), ("MiB", 1048576.0), ("KiB", 1024.0), ("GB", 1e9), ("MB", 1e6),
                   ("KB", 1e3), ("B", 1.0)):
        if s.endswith(suf):
            mult = m
            s = s[: len(s) - len(suf)]
            break
    try:
        return int(_stod(s) * mult)
    except (ValueError, OverflowError):
        raise V.ConfigError(9, f"cannot parse byte size: '{s}'")


def parse_rate(s: str) -> float:
    return float(parse_bytes(s))


@dataclass
class ExperimentConfig:
    network: str = "vgg16"
    batch: int = 64
    policy: str = "baseline"          # baseline|vdnn-all|vdnn-conv|vdnn-dyn|decision-file
    algo_mode: V.AlgoMode = V.AlgoMode.PerfOptimal
    capacity: Optional[int] = None
    decision_file: str = ""
    cost: V.CostModel = field(default_factory=V.CostModel)
    include_weight_grads: bool = False
    seed: int = 0
    inline_layers: List[str] = field(default_factory=list)

    def effective_capacity(self) -> int:
        return self.capacity if self.capacity is not None else self.cost.mem_capacity


def _parse_ini(text: str, where: str) -> Dict[str, List[Tuple[str, str]]]:
    """config.hpp:78-101: '#'/';' comments, [section], key = value."""
    sections: Dict[str, List[Tuple[str, str]]] = {}
    section = ""
    for lineno, line in enumerate(text.splitlines(), 1):
        cut = min([i for i in (line.find("#"), line.find(";")) if i >= 0], default=-1)
        if cut >= 0:
            line = line[:cut]
        line = line.strip(" \t\r\n")
        if not line:
            continue
        if line[0] == "[":
            if line[-1] != "]":
                raise V.ConfigError(9, f"{where}:{lineno}: bad section")
            section = line[1:-1].strip(" \t\r\n")
            continue
        eq = line.find("=")
        if eq < 0:
            raise V.ConfigError(9, f"{where}:{lineno}: expected key = value")
        sections.setdefault(section, []).append((line[:eq].strip(" \t\r\n"), line[eq + 1:].strip(" \t\r\n")))
    return sections


def _device_key(cfg: ExperimentConfig, key: str, val: str) -> None:
    cm = cfg.cost
    if key == "preset":
        if val != "titanx":
            raise V.ConfigError(9, "unknown device preset: " + val)
        d = V.CostModel()
        cm.peak_flops, cm.dram_bw, cm.mem_capacity, cm.compute_efficiency = (
            d.peak_flops, d.dram_bw, d.mem_capacity, d.compute_efficiency)
    elif key == "peak_flops":
        cm.peak_flops = _stod(val)
    elif key == "dram_bw":
        cm.dram_bw = parse_rate(val)
    elif key == "mem_capacity":
        cm.mem_capacity = parse_bytes(val)
    elif key == "compute_efficiency":
        cm.compute_efficiency = _stod(val)
    elif key == "elem_size":
        cm.elem_size = parse_bytes(val)
    elif key == "bwd_fwd_ratio":
        cm.bwd_fwd_ratio = _stod(val)
    elif key == "include_weight_grads":
        cfg.include_weight_grads = val in ("true", "1")
    else:
        raise V.ConfigError(9, "unknown [device] key: " + key)


def _link_key(cm: V.CostModel, key: str, val: str) -> None:
    if key == "preset":
        if val == "pcie3":
            d = V.CostModel()
            cm.link_effective_bw, cm.link_nominal_bw, cm.link_fixed_launch_overhead = (
                d.link_effective_bw, d.link_nominal_bw, d.link_fixed_launch_overhead)
        elif val == "page_migration":  # cost_model.hpp:30
            cm.link_effective_bw, cm.link_nominal_bw, cm.link_fixed_launch_overhead = 200e6, 200e6, 0.0
        else:
            raise V.ConfigError(9, "unknown link preset: " + val)
    elif key == "effective_bw":
        cm.link_effective_bw = parse_rate(val)
    elif key == "nominal_bw":
        cm.link_nominal_bw = parse_rate(val)
    elif key == "launch_overhead":
        cm.link_fixed_launch_overhead = _stod(val)
    else:
        raise V.ConfigError(9, "unknown [link] key: " + key)


def _latency_key(cm: V.CostModel, key: str, val: str) -> None:
    parts = val.split()
    try:
        fwd, bwd = _stod(parts[0]), _stod(parts[1])
    except (IndexError, ValueError):
        raise V.ConfigError(9, "bad [latencies] entry for layer " + key)
    cm.latency_overrides[int(_stod(key))] = (fwd, bwd)


def load_config(path: str) -> ExperimentConfig:
    """config.hpp:137-185. Sections are visited in name order (std::map)."""
    try:
        with open(path) as f:
            text = f.read()
    except OSError:
        raise V.ConfigError(9, "cannot open config file: " + path)
    cfg = ExperimentConfig()
    named = False
    for section in sorted(_parse_ini(text, path).items()):
        name, entries = section
        for key, val in entries:
            if name == "network":
                if key in ("preset", "file"):
                    cfg.network = val
                    named = True
                elif key == "batch":
                    cfg.batch = int(_stod(val))
                elif key.startswith("layer"):
                    cfg.inline_layers.append(val)
                else:
                    raise V.ConfigError(9, "unknown [network] key: " + key)
            elif name == "device":
                _device_key(cfg, key, val)
            elif name == "link":
                _link_key(cfg.cost, key, val)
            elif name == "latencies":
                _latency_key(cfg.cost, key, val)
            elif name == "policy":
                if key == "policy":
                    cfg.policy = val
                elif key == "algo_mode":
                    if val == "perf":
                        cfg.algo_mode = V.AlgoMode.PerfOptimal
                    elif val == "memory":
                        cfg.algo_mode = V.AlgoMode.MemoryOptimal
                    else:
                        raise V.ConfigError(9, "algo_mode must be perf or memory")
                elif key == "capacity":
                    cfg.capacity = parse_bytes(val)
                elif key == "decision":
                    cfg.decision_file = val
                elif key == "seed":
                    cfg.seed = int(_stod(val))
                else:
                    raise V.ConfigError(9, "unknown [policy] key: " + key)
            else:
                raise V.ConfigError(9, f"unknown config section: [{name}]")
    if cfg.inline_layers and not named:
        cfg.network = "custom"
    return cfg


_KINDS = {"input": V.LayerKind.Input, "conv": V.LayerKind.Conv, "actv": V.LayerKind.Actv,
          "pool": V.LayerKind.Pool, "fc": V.LayerKind.Fc, "loss": V.LayerKind.Loss}


def parse_inline_layer(text: str):
    """config.hpp:194-234: '<kind> [inputs=a,b] [join=..] k= s= p= out= window= stride= c= h= w='.
    Returns (kind, inputs, params, join) for NetworkGraph.add_layer."""
    toks = text.split()
    if not toks or toks[0] not in _KINDS:
        raise V.ConfigError(9, "unknown layer kind: " + (toks[0] if toks else ""))
    kind = _KINDS[toks[0]]
    kv: Dict[str, str] = {}
    for tok in toks[1:]:
        eq = tok.find("=")
        if eq < 0:
            raise V.ConfigError(9, "bad layer attribute: " + tok)
        kv[tok[:eq]] = tok[eq + 1:]
    inputs = [int(_stod(x)) for x in kv["inputs"].split(",") if x != ""] if "inputs" in kv else []
    join = V.JoinRule.Elementwise if kv.get("join") == "eltwise" else V.JoinRule.Concat

    def num(key, fallback):
        return int(_stod(kv[key])) if key in kv else fallback

    if kind == V.LayerKind.Conv:
        params = (num("k", 3), num("s", 1), num("p", 0), num("out", 1))
    elif kind == V.LayerKind.Pool:
        params = (num("window", 2), num("stride", 2))
    elif kind == V.LayerKind.Fc:
        params = (num("out", 1),)
    elif kind == V.LayerKind.Input:
        params = (num("c", 1), num("h", 1), num("w", 1))
    else:
        params = ()
    return kind, inputs, params, join


def resolve_path(name: str) -> Optional[str]:
    """config.hpp:236-245: the name itself, else under $VDNN_SIM_EXPERIMENTS."""
    if os.path.exists(name):
        return name
    d = os.environ.get("VDNN_SIM_EXPERIMENTS")
    if d and os.path.exists(os.path.join(d, name)):
        return os.path.join(d, name)
    return None


def build_network(cfg: ExperimentConfig) -> V.NetworkGraph:
    """config.hpp:252-269."""
    if cfg.inline_layers:
        g = V.NetworkGraph(cfg.batch)
        for text in cfg.inline_layers:
            kind, inputs, params, join = parse_inline_layer(text)
            g.add_layer(kind, inputs, params, join)
        return g.finalize()
    name = cfg.network
    if name in ("alexnet", "overfeat", "vgg16", "inception_toy"):
        return V.build_preset(name, cfg.batch)
    if name.startswith("vgg") and len(name) > 3 and name[3].isdigit():
        return V.extend_vgg(int(re.match(r"\d+", name[3:]).group(0)) - 16, cfg.batch)
    path = resolve_path(name)
    if path:
        if len(path) > 5 and path.endswith(".json"):
            from . import formats
            with open(path) as f:
                return formats.graph_from_json(json.load(f))
        nested = load_config(path)
        nested.batch = cfg.batch
        if nested.inline_layers or nested.network != cfg.network:
            return build_network(nested)
        raise V.ConfigError(9, "network config file does not define a network: " + path)
    raise V.UnknownPreset(3, "unknown network: " + name)
