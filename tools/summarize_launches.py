"""Summarise an ncu launch list (gpu__time_duration.sum [+ dram bytes]) of
bench.py / one_step.py: per kernel family, the launch count, summed time,
share of the step and DRAM bytes per launch, over the LAST training step
(the launches after the last tf32 probe / before the end).

    python tools/summarize_launches.py gpurun_out/r01_launches_dyn.csv [--per-step N] [--steps N]
"""
import csv
import re
import sys
from collections import OrderedDict, defaultdict

UNIT = {"ns": 1e-6, "us": 1e-3, "ms": 1.0, "nsecond": 1e-6, "usecond": 1e-3, "msecond": 1.0, "second": 1e3,
        "byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}


def load(path):
    rows = list(csv.reader(open(path)))
    i = [k for k, r in enumerate(rows) if r and r[0] == "ID"][0]
    h = rows[i]
    L = OrderedDict()
    for r in rows[i + 1:]:
        d = dict(zip(h, r))
        k = d["ID"]
        e = L.setdefault(k, {"name": d["Kernel Name"], "grid": d.get("Grid Size", "")})
        v = float(d["Metric Value"].replace(",", "")) * UNIT.get(d["Metric Unit"], 1.0)
        e[d["Metric Name"]] = v
    return list(L.values())


def family(name):
    n = re.sub(r"\(.*", "", name)
    n = re.sub(r"^void ", "", n)
    return re.sub(r"vdnnk::(<unnamed>::)?", "", n)


def main():
    path = sys.argv[1]
    per = int(sys.argv[sys.argv.index("--per-step") + 1]) if "--per-step" in sys.argv else None
    ks = load(path)
    # steps start with the first layer's fprop; take the last complete step
    # (bench.py runs the tf32 probe before the policies: drop it and
    # everything before it)
    probe = [i for i, k in enumerate(ks) if "tf32_peak" in k["name"]]
    ks = ks[probe[-1] + 1:] if probe else ks
    if "--steps" in sys.argv:
        # N identical steps after the synthetic-data fills: the last N-th
        n = int(sys.argv[sys.argv.index("--steps") + 1])
        ks = [k for k in ks if "fill_" not in k["name"]]
        step = ks[len(ks) - len(ks) // n:]
    else:
        first = sys.argv[sys.argv.index("--first") + 1] if "--first" in sys.argv else "c3tc_fprop"
        starts = [i for i, k in enumerate(ks) if first in k["name"]]
        step = ks[starts[-2]:starts[-1]] if len(starts) >= 2 else ks[starts[-1]:]
        if per:
            step = ks[starts[-1]:starts[-1] + per]
    tot = sum(k.get("gpu__time_duration.sum", 0) for k in step)
    agg = defaultdict(lambda: [0, 0.0, 0.0, 0.0])
    for k in step:
        a = agg[family(k["name"])]
        a[0] += 1
        a[1] += k.get("gpu__time_duration.sum", 0)
        a[2] += k.get("dram__bytes_read.sum", 0)
        a[3] += k.get("dram__bytes_write.sum", 0)
    print(f"launches {len(step)}  serialized kernel time {tot:.3f} ms  (ncu: cold-cache, serialised)")
    print(f"{'kernel':58s} {'n':>4s} {'ms':>9s} {'share':>6s} {'DRAM MB/launch':>15s}")
    for name, (n, t, rd, wr) in sorted(agg.items(), key=lambda x: -x[1][1]):
        print(f"{name[:58]:58s} {n:4d} {t:9.3f} {t / tot:6.1%} {(rd + wr) / n / 1e6:15.1f}")
    if "--traffic-json" in sys.argv:
        # DRAM bytes per conv-engine launch (bench.py's roofline "traffic")
        import json
        conv = [k for k in step if "tc_conv" in k["name"] or "tc_wgrad" in k["name"] or "tcb_conv" in k["name"]
                or "c3tc" in k["name"]]
        byt = sum(k.get("dram__bytes_read.sum", 0) + k.get("dram__bytes_write.sum", 0) for k in conv)
        out = {"source": "ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum "
                         "--clock-control none, python bench.py --policies dyn --steps 1 --warmup 3 (last step): "
                         + path.split("/")[-1],
               "conv_launches": len(conv), "conv_dram_bytes_per_launch": byt / max(1, len(conv)),
               "conv_ms_serialized": sum(k.get("gpu__time_duration.sum", 0) for k in conv),
               "step_kernel_ms_serialized": tot}
        with open(sys.argv[sys.argv.index("--traffic-json") + 1], "w") as f:
            json.dump(out, f, indent=1)


if __name__ == "__main__":
    main()
