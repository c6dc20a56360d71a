"""INI experiment configs, inline-layer networks and graph/report JSON versus
the compiled reference front-end (vdnnsim/config.hpp, report.hpp via
oracle/_ref/libvdnnref_fmt.so). SURVEY §8(f)3."""
import json
import os

import pytest

import paper_1602_08124_b200 as V
from paper_1602_08124_b200 import config as K
from paper_1602_08124_b200 import formats as F
from oracle import refsim

pytestmark = pytest.mark.skipif(not refsim.fmt_available(), reason="oracle/_ref/libvdnnref_fmt.so not built")

NAMES = ["input", "conv", "actv", "pool", "fc", "loss"]


def norm(spec: str):
    """Graph spec -> comparable tuples (params that matter for the kind, join only for multi-input)."""
    parts = spec.split("|")
    out = [parts[0]]
    for p in parts[1:]:
        kind, ins, a, b, c, d, j = p.split()
        n = {"input": 3, "conv": 4, "pool": 2, "fc": 1}.get(kind, 0)
        prm = [a, b, c, d][:n]
        out.append((kind, ins, tuple(prm), j if ins.count(",") else "0"))
    return out


def ours(path):
    cfg = K.load_config(path)
    try:
        g = K.build_network(cfg)
        gspec, gerr = g.spec(), None
    except V.VdnnError as e:
        gspec, gerr = None, type(e).__name__
    return cfg, gspec, gerr


def check(path):
    ref = refsim.fmt_config(path)
    if "error" in ref:
        with pytest.raises(V.VdnnError):
            ours(path)
        return ref
    cfg, gspec, gerr = ours(path)
    assert cfg.network == ref["network"]
    assert cfg.batch == ref["batch"]
    assert cfg.policy == ref["policy"]
    assert ("perf" if cfg.algo_mode == V.AlgoMode.PerfOptimal else "memory") == ref["algo_mode"]
    assert cfg.capacity == ref["capacity"]
    assert cfg.effective_capacity() == ref["effective_capacity"]
    assert cfg.decision_file == ref["decision_file"]
    assert cfg.include_weight_grads == ref["include_weight_grads"]
    assert cfg.seed == ref["seed"]
    assert cfg.inline_layers == ref["inline_layers"]
    c = ref["cost"]
    assert (cfg.cost.peak_flops, cfg.cost.dram_bw, cfg.cost.mem_capacity, cfg.cost.compute_efficiency,
            cfg.cost.elem_size, cfg.cost.bwd_fwd_ratio) == (c["peak_flops"], c["dram_bw"], c["mem_capacity"],
                                                            c["compute_efficiency"], c["elem_size"],
                                                            c["bwd_fwd_ratio"])
    assert (cfg.cost.link_effective_bw, cfg.cost.link_nominal_bw, cfg.cost.link_fixed_launch_overhead) == (
        c["link_effective_bw"], c["link_nominal_bw"], c["link_launch_overhead"])
    assert {str(k): list(v) for k, v in cfg.cost.latency_overrides.items()} == ref["latency_overrides"]
    if "graph" in ref:
        assert gerr is None, gerr
        assert norm(gspec) == norm(ref["graph"])
    else:
        assert gerr is not None
    return ref


def write(tmp_path, name, text):
    p = tmp_path / name
    p.write_text(text)
    return str(p)


def test_full_config(tmp_path):
    check(write(tmp_path, "a.conf", """
# every section the reference reads
[network]
preset = alexnet        ; trailing comment
batch = 32
[device]
preset = titanx
peak_flops = 1.2e13
dram_bw = 480GB
mem_capacity = 16GiB
compute_efficiency = 0.55
elem_size = 2
bwd_fwd_ratio = 2.5
include_weight_grads = true
[link]
preset = page_migration
effective_bw = 25GB
nominal_bw = 32GB
launch_overhead = 1e-5
[latencies]
1 = 0.001 0.002
5 = 3e-4 6e-4
[policy]
policy = vdnn-dyn
algo_mode = memory
capacity = 8GiB
seed = 7
decision = d.json
"""))


@pytest.mark.parametrize("size", ["12GiB", "12GB", "512MiB", "1.5e9", "3KB", "4096B", "100", "unlimited", "inf",
                                  "7 MB", "2.5KiB"])
def test_byte_sizes(tmp_path, size):
    ref = check(write(tmp_path, "b.conf", f"[policy]\ncapacity = {size}\n"))
    assert K.parse_bytes(size) == ref["capacity"]


def test_inline_layers(tmp_path):
    check(write(tmp_path, "c.conf", """
[network]
batch = 4
layer0 = input c=3 h=32 w=32
layer1 = conv inputs=0 k=3 s=1 p=1 out=16
layer2 = actv inputs=1
layer3 = conv inputs=0 k=1 out=8
layer4 = conv inputs=2,3 join=concat k=3 p=1 out=24
layer5 = conv inputs=4 k=3 p=1 out=24
layer6 = pool inputs=4,5 join=eltwise window=2 stride=2
layer7 = fc inputs=6 out=10
layer8 = loss inputs=7
"""))


def test_vgg_depth_and_presets(tmp_path):
    for net in ("vgg116", "vgg16", "overfeat", "inception_toy"):
        check(write(tmp_path, f"{net}.conf", f"[network]\npreset = {net}\nbatch = 2\n"))


def test_nested_config_and_json_graph(tmp_path, monkeypatch):
    inner = write(tmp_path, "inner.conf", "[network]\nlayer0 = input c=3 h=8 w=8\nlayer1 = fc inputs=0 out=5\n"
                                          "layer2 = loss inputs=1\n")
    g = V.build_preset("alexnet", 3)
    gj = write(tmp_path, "g.json", json.dumps(F.graph_to_json(g)))
    monkeypatch.setenv("VDNN_SIM_EXPERIMENTS", str(tmp_path))
    check(write(tmp_path, "outer.conf", f"[network]\nfile = {os.path.basename(inner)}\nbatch = 6\n"))
    check(write(tmp_path, "outer2.conf", f"[network]\nfile = {os.path.basename(gj)}\nbatch = 9\n"))


@pytest.mark.parametrize("text", [
    "[network\nbatch = 1\n",                      # bad section
    "[network]\nbatch\n",                         # missing '='
    "[network]\ncolour = red\n",                  # unknown key
    "[device]\npreset = h100\n",                  # unknown device preset
    "[link]\npreset = nvlink\n",                  # unknown link preset
    "[policy]\nalgo_mode = fast\n",               # bad algo mode
    "[policy]\ncapacity = lots\n",                # bad byte size
    "[latencies]\n3 = 0.1\n",                     # missing bwd latency
    "[extras]\na = b\n",                          # unknown section
])
def test_config_errors(tmp_path, text):
    ref = refsim.fmt_config(write(tmp_path, "e.conf", text))
    assert "error" in ref and ref["type"] == "ConfigError"
    with pytest.raises(V.ConfigError):
        K.load_config(str(tmp_path / "e.conf"))


@pytest.mark.parametrize("text", [
    "[network]\npreset = resnet\n",                                                     # unknown network
    "[network]\nlayer0 = input c=3 h=8 w=8\nlayer1 = actv inputs=0\nlayer2 = actv inputs=0,1\n",  # ACTV arity
    "[network]\nlayer0 = input c=3 h=8 w=8\nlayer1 = conv inputs=0,0 out=2\n",           # duplicate input
    "[network]\nlayer0 = input c=3 h=8 w=8\nlayer1 = conv inputs=0 k=3 s=2 out=2\n",     # non-divisible conv
    "[network]\nlayer0 = input c=3 h=8 w=8\nlayer1 = blur inputs=0\n",                   # unknown kind
])
def test_network_errors(tmp_path, text):
    ref = refsim.fmt_config(write(tmp_path, "n.conf", text))
    assert "graph_error" in ref or "error" in ref
    with pytest.raises(V.VdnnError):
        K.build_network(K.load_config(str(tmp_path / "n.conf")))


@pytest.mark.parametrize("net,batch", [("alexnet", 8), ("inception_toy", 4), ("vgg16", 2)])
def test_graph_json_matches_reference(net, batch):
    g = V.build_preset(net, batch)
    ref = refsim.fmt_graph_to_json(g.spec())
    assert F.graph_to_json(g) == ref
    back = refsim.fmt_graph_from_json(json.dumps(F.graph_to_json(g)))
    assert norm(back) == norm(g.spec())
    assert norm(F.graph_from_json(ref).spec()) == norm(g.spec())


@pytest.mark.parametrize("net,batch", [("alexnet", 128), ("vgg16", 256)])
def test_report_and_decision_json_match_reference(net, batch):
    cap = 12884901888
    g = V.build_preset(net, batch)
    ref = refsim.fmt_report(g.spec(), cap)
    sel = V.dynamic_select(g, cap, V.CostModel())
    r = V.simulate(g, sel.decision, V.CostModel(), cap)
    assert F.decision_to_json(sel.decision) == ref["decision"]
    assert F.report_to_json(r, True) == ref["report"]
