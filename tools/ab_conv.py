"""Interleaved A/B of conv-engine variants selected by environment variables,
in ONE process per variant pair... (env is read once per process, so each
variant runs in its own subprocess; rounds alternate A, B, A, B, ... and the
best time per op is kept -- robust to the clock droop that makes single runs
swing by +-10%).

    python tools/ab_conv.py VAR=a VAR=b [--rounds 4] [--shapes 56,28,14]
"""
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
args = [a for a in sys.argv[1:] if "=" in a and not a.startswith("--")]
rounds = int(sys.argv[sys.argv.index("--rounds") + 1]) if "--rounds" in sys.argv else 4
best = {}
for r in range(rounds):
    for a in args:
        k, v = a.split("=", 1)
        env = dict(os.environ, **{k: v}, REPS="10")
        out = subprocess.run([sys.executable, "tools/bench_conv.py"], cwd=ROOT, env=env, capture_output=True,
                             text=True, timeout=300).stdout
        for line in out.splitlines():
            shape = line.split(":")[0]
            for op in ("fprop", "dgrad", "wgrad"):
                i = line.index(op)
                ms = float(line[i + len(op):].split("ms")[0])
                key = (a, shape, op)
                best[key] = min(best.get(key, 1e9), ms)
shapes = sorted({k[1] for k in best}, key=lambda s: list(best).index((args[0], s, "fprop")))
for shape in shapes:
    row = [f"{shape:24s}"]
    for op in ("fprop", "dgrad", "wgrad"):
        row.append(op + " " + " / ".join(f"{best[(a, shape, op)]:.3f}" for a in args))
    print(" | ".join(row))
print("columns:", " / ".join(args), "(best ms over", rounds, "rounds)")
