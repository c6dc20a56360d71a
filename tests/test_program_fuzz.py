"""The executable program the CUDA executor runs, checked on the CPU.

``program_check`` compiles a plan into the executor's form -- every operand of
every FWD/BWD step bound to a pool offset, the incoming gradient planes of a
backward step (after the folds of earlier fork sums), the scratch gap, the
transfers -- and verifies each binding against the plan's own event log: an
operand must lie inside the extent that is live for *that* buffer at *that*
step. A binding to a recycled extent (the stale-fold bug of round 1, where a
folded gradient plane was keyed by address and a later dX reused the address)
is a failure here, without a GPU.
"""
import random

import pytest

import paper_1602_08124_b200 as V
from planner_util import graph_from_spec, vocab_spec


def fork_heavy_spec(rng: random.Random, max_layers: int = 16) -> str:
    """Graphs with forks into 2-3 consumers, ACTV chains on fork outputs,
    concat and elementwise joins, forks of forks."""
    batch = 1 + rng.randrange(3)
    h = rng.choice([8, 16])
    layers = [f"input - {1 + rng.randrange(4)} {h} {h} 0 0"]
    shapes = {0: None}
    prev = 0
    ch = {0: 0}

    def add(s):
        layers.append(s)
        return len(layers) - 1

    c = 4
    prev = add(f"conv 0 3 1 1 {c} 0")
    while len(layers) + 6 < max_layers:
        r = rng.randrange(6)
        if r == 0:
            prev = add(f"actv {prev} 0 0 0 0 0")
        elif r == 1 and h >= 4:
            prev = add(f"pool {prev} 2 2 0 0 0")
            h //= 2
        elif r <= 3:  # fork into 2-3 branches, then concat
            nb = 2 + rng.randrange(2)
            ends = []
            for _ in range(nb):
                b = add(f"conv {prev} {rng.choice([1, 3])} 1 {rng.choice([0, 1]) if False else 0} 0 0")
                # keep shapes: 1x1 pad 0 or 3x3 pad 1
                k = rng.choice([1, 3])
                layers[b] = f"conv {prev} {k} 1 {k // 2} {1 + rng.randrange(4)} 0"
                if rng.randrange(2):
                    b = add(f"actv {b} 0 0 0 0 0")
                ends.append(b)
            c = 0
            prev = add(f"conv {','.join(map(str, ends))} 1 1 0 {2 + rng.randrange(4)} 0")
        elif r == 4:  # elementwise join of two same-shaped branches
            k = rng.choice([1, 3])
            oc = 1 + rng.randrange(4)
            a = add(f"conv {prev} {k} 1 {k // 2} {oc} 0")
            b = add(f"conv {prev} 1 1 0 {oc} 0")
            if rng.randrange(2):
                b = add(f"actv {b} 0 0 0 0 0")
            prev = add(f"conv {a},{b} 3 1 1 {1 + rng.randrange(4)} 1")
        else:  # a fork whose one branch feeds a later join with a deeper path
            a = add(f"actv {prev} 0 0 0 0 0")
            b = add(f"conv {a} 3 1 1 {1 + rng.randrange(3)} 0")
            b = add(f"actv {b} 0 0 0 0 0")
            prev = add(f"conv {a},{b} 1 1 0 {1 + rng.randrange(4)} 0")
    prev = add(f"fc {prev} {2 + rng.randrange(8)} 0 0 0 0")
    add(f"loss {prev} 0 0 0 0 0")
    return f"B={batch}|" + "|".join(layers)


def decisions(g, cm):
    out = []
    for kind in (V.PolicyKind.Baseline, V.PolicyKind.VdnnAll, V.PolicyKind.VdnnConv):
        for mode in (V.AlgoMode.MemoryOptimal, V.AlgoMode.PerfOptimal):
            out.append(V.static_decision(kind, mode, g, cm))
    return out


@pytest.mark.parametrize("seed", range(6))
def test_program_bindings_on_fork_heavy_graphs(seed):
    rng = random.Random(77 + seed)
    cm = V.CostModel()
    checked = 0
    for _ in range(30):
        spec = fork_heavy_spec(rng)
        g = graph_from_spec(spec)
        fp = V.simulate_oracle(g, cm).max_mem_bytes
        for d in decisions(g, cm) + [V.dynamic_select(g, int(fp * rng.uniform(0.4, 1.2)), cm).decision]:
            if d is None:
                continue
            for cap in (int(fp * rng.uniform(0.3, 1.5)), 1 << 40):
                r = V.simulate(g, d, cm, cap)
                if not r.pass_:
                    continue
                bad = V.program_check(g, d, cm, cap)
                assert bad == [], (spec, d.label, cap, bad[:3])
                checked += 1
    assert checked > 50


def test_program_bindings_on_presets():
    cm = V.CostModel()
    cap = 12884901888
    for net, b in (("alexnet", 128), ("overfeat", 128), ("inception_toy", 128), ("vgg16", 256)):
        g = V.build_preset(net, b)
        for d in decisions(g, cm) + [V.dynamic_select(g, cap, cm).decision]:
            c = cap if d.gradient_scheme == V.GradientScheme.PerLayer else 1 << 40
            if V.simulate(g, d, cm, c).pass_:
                assert V.program_check(g, d, cm, c) == [], (net, d.label)


def test_program_bindings_on_full_vocabulary_graphs():
    """Elementwise joins over ReLU chains (shared maps read-only, private
    planes), strided convs, several INPUT and LOSS layers: the compiled
    program binds every operand inside its live extent (private planes sit
    after the arena), and the generator emits every construct."""
    rng = random.Random(4242)
    cm = V.CostModel()
    seen = {"eltwise": 0, "stride": 0, "inputs": 0, "losses": 0, "private": 0}
    for _ in range(60):
        spec = vocab_spec(rng)
        g = graph_from_spec(spec)
        layers = spec.split("|")[1:]
        seen["eltwise"] += any(p.startswith("conv") and p.endswith(" 1") and "," in p.split()[1] for p in layers)
        seen["stride"] += any(p.startswith("conv") and p.split()[3] == "2" for p in layers)
        seen["inputs"] += sum(p.startswith("input") for p in layers) > 1
        seen["losses"] += sum(p.startswith("loss") for p in layers) > 1
        fp = V.simulate_oracle(g, cm).max_mem_bytes
        for d in decisions(g, cm):
            for cap in (int(fp * rng.uniform(0.5, 1.5)), 1 << 40):
                if not V.simulate(g, d, cm, cap).pass_:
                    continue
                assert V.program_check(g, d, cm, cap) == [], (spec, d.label, cap)
    assert all(v > 0 for k, v in seen.items() if k != "private"), seen
