"""Stall-sample breakdown of one ncu report's kernels by SASS region: prints
the top stalled instructions and, for each mbarrier wait, how often its
retry path ran (a wait that spins is the role that waits; the role it waits
for is the limiter). Usage: ncu_warp_roles.py REPORT.ncu-rep [launch index]"""
import csv, io, subprocess, sys

rep = sys.argv[1]
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
blocks = [b for b in out.split('"Kernel Name"') if b.strip()]
for b in blocks[: int(sys.argv[2]) + 1 if len(sys.argv) > 2 else len(blocks)]:
    lines = list(csv.reader(io.StringIO('"Kernel Name"' + b)))
    name = lines[0][1][:90]
    h, rows = lines[1], [r for r in lines[2:] if len(r) == len(lines[1])]
    i_src, i_s, i_e = h.index("Source"), h.index("Warp Stall Sampling (All Samples)"), h.index("Instructions Executed")
    tot = sum(float(r[i_s] or 0) for r in rows) or 1
    print(f"== {name}  samples {int(tot)}")
    for k in sorted(range(len(rows)), key=lambda k: -float(rows[k][i_s] or 0))[:12]:
        r = rows[k]
        print(f"  {float(r[i_s]) / tot * 100:5.1f}% {k:5d} {r[i_src][:64]:64s} <- {rows[k - 1][i_src][:44]}")
    print("  waits (executions):")
    for k, r in enumerate(rows):
        if "TRYWAIT" in r[i_src] or "UTCHMMA" in r[i_src] or "UTMALDG" in r[i_src]:
            if int(r[i_e] or 0) > 0:
                print(f"    {k:5d} {int(r[i_e]):>10d} {r[i_src][:70]}")
