"""Regenerate the golden fixtures from the compiled reference (oracle/_ref).

    make -C oracle && python tests/golden/gen_golden.py

Every fixture is produced by the unmodified reference simulator
(/root/reference/proj/include/vdnnsim, compiled by oracle/Makefile). Capacity
12 GiB = 12,884,901,888 B (cost_model.hpp:18) is the headline; 12e9 B is also
recorded (SURVEY.md §7.3 hard part 8).
"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
from oracle import refsim  # noqa: E402

GIB12 = 12884901888
CAPS = [GIB12, 12_000_000_000]
DECS = ["static:baseline:m", "static:baseline:p", "static:all:m", "static:all:p", "static:conv:m", "static:conv:p",
        "dyn", "oracle", "greedy:conv", "greedy:all"]
NETS = [("alexnet", 128, 0), ("overfeat", 128, 0), ("inception_toy", 128, 0), ("vgg16", 256, 0)]

# Hand graphs from the reference tests (tests/test_simulator.cpp:27-37,93-133; tests/test_policy.cpp:157-172).
SMALL_LINEAR = "B=2|input - 4 16 16 0 0|conv 0 3 1 1 8 0|actv 1 0 0 0 0 0|pool 2 2 2 0 0 0|fc 3 64 0 0 0 0|loss 4 0 0 0 0 0"
FIG8 = "B=1|input - 5 1000 1000 0 0|conv 0 1 1 0 20 0|conv 1 1 1 0 1 0|conv 2 1 1 0 1 0|loss 3 0 0 0 0 0"
FIG8_COST = ("pf=7000000000000.0,bw=336000000000.0,cap=12884901888,eff=0.5,lbw=4000000000.0,lnom=16000000000.0,"
             "lov=0.0,es=4,ratio=2.0,sfi=1.0,sfg=0.8,sff=0.6;ov=1:0.01:0.01,2:0.01:0.01,3:0.01:0.01")
SHRINK = ("B=4|input - 8 16 16 0 0|conv 0 3 1 1 8 0|actv 1 0 0 0 0 0|pool 2 2 2 0 0 0|conv 3 3 1 1 8 0|"
          "actv 4 0 0 0 0 0|pool 5 2 2 0 0 0|conv 6 3 1 1 8 0|actv 7 0 0 0 0 0|fc 8 10 0 0 0 0|loss 9 0 0 0 0 0")


def main():
    out_dir = os.path.dirname(os.path.abspath(__file__))
    for name, batch, extra in NETS:
        spec = refsim.preset_spec(name, batch, extra)
        cases = []
        for cap in CAPS:
            for dec in DECS:
                r = refsim.run(spec, dec, cap)
                cases.append({"decision_spec": dec, "capacity": cap, "result": r})
        with open(os.path.join(out_dir, f"{name}_b{batch}.json"), "w") as f:
            json.dump({"spec": spec, "cases": cases}, f, separators=(",", ":"))
    # VGG-416 b32: no events (7.6k per run) -- summaries, tallies, signatures.
    spec = refsim.preset_spec("vgg16", 32, 400)
    cases = []
    for cap, dec in [(GIB12, "dyn"), (GIB12, "static:all:m"), (GIB12, "static:conv:p"), (180_000_000_000, "dyn"),
                     (GIB12, "oracle")]:
        cases.append({"decision_spec": dec, "capacity": cap, "result": refsim.run(spec, dec, cap, events=False)})
    with open(os.path.join(out_dir, "vgg416_b32.json"), "w") as f:
        json.dump({"spec": spec, "cases": cases}, f, separators=(",", ":"))
    small = []
    for spec, cost, dec, cap in [
        (SMALL_LINEAR, "", "static:baseline:m", 1 << 62), (SMALL_LINEAR, "", "static:all:m", 1 << 62),
        (SMALL_LINEAR, "", "static:all:m", 4096), (FIG8, FIG8_COST, "static:all:m", 1 << 62),
        (SHRINK, "", "greedy:conv", 1 << 40), (SHRINK, "", "greedy:all", 300000), (SHRINK, "", "dyn", 400000),
    ]:
        small.append({"spec": spec, "cost": cost, "decision_spec": dec, "capacity": cap,
                      "result": refsim.run(spec, dec, cap, cost_spec=cost)})
    with open(os.path.join(out_dir, "small_graphs.json"), "w") as f:
        json.dump(small, f, separators=(",", ":"))
    # BF16 storage: elem_size = 2 (cost_model.hpp:69, config.hpp:112), every BASELINE config
    es2 = []
    for name, batch, extra in NETS + [("vgg16", 32, 400)]:
        spec = refsim.preset_spec(name, batch, extra)
        decs = ["dyn", "static:all:m", "static:conv:m", "static:conv:p", "static:baseline:p"]
        for dec in decs:
            r = refsim.run(spec, dec, GIB12, cost_spec="es=2", events=extra == 0)
            es2.append({"spec": spec, "cost": "es=2", "decision_spec": dec, "capacity": GIB12, "result": r})
    with open(os.path.join(out_dir, "es2.json"), "w") as f:
        json.dump(es2, f, separators=(",", ":"))
    print("wrote fixtures to", out_dir)


if __name__ == "__main__":
    main()
