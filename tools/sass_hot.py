"""Hot SASS of one kernel from an ncu report (source page): instructions
executed per SASS line, in address order, with stall samples.

    python tools/sass_hot.py REPORT.ncu-rep [MIN_FRACTION]
"""
import csv
import subprocess
import sys
from collections import Counter

rep = sys.argv[1]
frac = float(sys.argv[2]) if len(sys.argv) > 2 else 0.002
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout.splitlines()
rows = list(csv.DictReader(out[1:]))
tot = sum(int(r["Instructions Executed"] or 0) for r in rows)
samples = sum(int(r["Warp Stall Sampling (All Samples)"] or 0) for r in rows)
print(f"total warp instructions {tot:.4e}, stall samples {samples}")
ops = Counter()
for r in rows:
    n = int(r["Instructions Executed"] or 0)
    op = r["Source"].split()[0] if r["Source"].split() else "?"
    if op.startswith("@"):
        op = r["Source"].split()[1]
    ops[op.split(".")[0]] += n
print("by opcode:", ", ".join(f"{k} {v / tot:.3f}" for k, v in ops.most_common(25)))
for r in rows:
    n = int(r["Instructions Executed"] or 0)
    s = int(r["Warp Stall Sampling (All Samples)"] or 0)
    if n >= frac * tot or s >= 0.004 * samples:
        print(f"{r['Address'][-5:]} {n / tot * 100:6.2f}% st{s / max(samples, 1) * 100:5.1f}%  {r['Source'].strip()}")
