"""Differential fuzzing: planner vs the compiled reference (oracle/_ref).

Random fork/join graphs in the style of the reference campaign
(fuzz.hpp:26-82) x random capacities x {baseline, all, conv}(m|p), dyn, greedy
and fully random decisions; every field of every report must be identical and
replay-clean. Skipped when the oracle library is absent (it is built here by
``make -C oracle`` and travels prebuilt to the GPU box).
"""
import random

import pytest

import paper_1602_08124_b200 as V
from oracle import refsim
from planner_util import compare_case

pytestmark = pytest.mark.skipif(not refsim.available(), reason="oracle/_ref not built")


def random_spec(rng: random.Random, max_layers: int = 12) -> str:
    batch = 1 + rng.randrange(4)
    h = rng.choice([4, 8, 16])
    layers = [f"input - {1 + rng.randrange(4)} {h} {h} 0 0"]
    prev = 0
    fc_seen = False
    while len(layers) + 1 < max_layers:
        budget = max_layers - len(layers) - 1
        pick = rng.randrange(10)
        if fc_seen or pick < 1:
            layers.append(f"fc {prev} {1 + rng.randrange(16)} 0 0 0 0")
            prev = len(layers) - 1
            fc_seen = True
            if rng.randrange(2) == 0 and len(layers) + 1 < max_layers:
                layers.append(f"actv {prev} 0 0 0 0 0")
                prev = len(layers) - 1
            if rng.randrange(2) == 0:
                break
            continue
        if pick < 4:
            k = rng.choice([1, 3])
            layers.append(f"conv {prev} {k} 1 {k // 2} {1 + rng.randrange(8)} 0")
        elif pick < 6:
            layers.append(f"actv {prev} 0 0 0 0 0")
        elif pick < 8 and h >= 4 and h % 2 == 0:
            layers.append(f"pool {prev} 2 2 0 0 0")
            h //= 2
        elif budget >= 3:
            layers.append(f"conv {prev} 1 1 0 {1 + rng.randrange(4)} 0")
            a = len(layers) - 1
            if rng.randrange(2) == 0:
                layers.append(f"actv {prev} 0 0 0 0 0")
            else:
                layers.append(f"conv {prev} 3 1 1 {1 + rng.randrange(4)} 0")
            b = len(layers) - 1
            layers.append(f"conv {a},{b} 1 1 0 {1 + rng.randrange(8)} 0")
        else:
            layers.append(f"actv {prev} 0 0 0 0 0")
        prev = len(layers) - 1
    layers.append(f"loss {prev} 0 0 0 0 0")
    return f"B={batch}|" + "|".join(layers)


def random_decision(rng: random.Random, spec: str) -> str:
    kinds = [l.split()[0] for l in spec.split("|")[1:]]
    off = [str(i) for i, k in enumerate(kinds) if k in ("conv", "pool", "input") and rng.randrange(2) == 0]
    alg = []
    for i, k in enumerate(kinds):
        if k == "conv":
            a = rng.randrange(3)
            alg.append(f"{i}={a}")
    return f"custom:1:fuzz-random:{','.join(off)}:{','.join(alg)}"


DECS = ["static:baseline:m", "static:baseline:p", "static:all:m", "static:all:p", "static:conv:m", "static:conv:p",
        "dyn", "greedy:conv", "greedy:all"]


@pytest.mark.parametrize("seed", range(8))
def test_differential_random_graphs(seed):
    rng = random.Random(1000 + seed)
    for trial in range(40):
        spec = random_spec(rng)
        oracle_run = refsim.run(spec, "oracle", 1 << 62)
        fp = oracle_run["report"]["max_mem_bytes"]
        cap = int(4096 * (2 * fp / 4096) ** rng.random())
        for dec in DECS + [random_decision(rng, spec)]:
            if dec.startswith("custom:"):
                # the reference rejects FFT on strided convs only via cost; random algos are always legal
                ref = refsim.run(spec, dec, cap)
                g = __import__("planner_util").graph_from_spec(spec)
                parts = dec.split(":")
                d = V.PolicyDecision([0] * g.size(), {}, V.GradientScheme.PerLayer, parts[2])
                for i in parts[3].split(","):
                    if i:
                        d.offload[int(i)] = 1
                for kv in parts[4].split(","):
                    if kv:
                        i, a = kv.split("=")
                        d.algos[int(i)] = V.AlgoId(int(a))
                r = V.simulate(g, d, V.CostModel(), cap)
                from planner_util import report_json
                got = report_json(r, g.size())
                for k, v in ref["report"].items():
                    if k != "violations":
                        assert got[k] == v, (spec, dec, cap, k)
                assert [x.kind for x in V.replay_check(r, g, d, cap)] == ref["report"]["violations"] == []
            else:
                case = {"decision_spec": dec, "capacity": cap, "result": refsim.run(spec, dec, cap)}
                compare_case(spec, case)
                if case["result"].get("report"):
                    assert case["result"]["report"]["violations"] == []


def test_reference_fuzz_campaign_clean():
    """The reference's own campaign (fuzz.hpp:89-158) stays violation-free."""
    r = refsim.fuzz(0, 2000)
    assert r["trials"] == 2000 and r["violations"] == 0
