"""Histogram of executed SASS instructions from an `ncu --page source
--print-source sass --csv` export: per opcode, and per basic-block-like run of
equal execution counts (to locate the hot regions)."""
import csv
import re
import sys
from collections import Counter, defaultdict

rows = list(csv.reader(open(sys.argv[1])))
h = rows[1]
iS, iE, iSmp = h.index("Source"), h.index("Instructions Executed"), h.index("Warp Stall Sampling (All Samples)")
ops = Counter()
samples = Counter()
runs = []
tot = 0
for r in rows[2:]:
    if len(r) <= iE:
        continue
    src = r[iS].strip()
    try:
        n = int(r[iE])
        smp = int(r[iSmp])
    except ValueError:
        continue
    op = re.sub(r"^@!?U?P[T0-9]+\s+", "", src).split(" ")[0]
    ops[op] += n
    samples[op] += smp
    tot += n
    if runs and runs[-1][0] == n:
        runs[-1][1] += 1
        runs[-1][2][op] += 1
        runs[-1][3] += smp
    else:
        runs.append([n, 1, Counter({op: 1}), smp])
print(f"total executed warp instructions: {tot:.4g}")
for op, n in ops.most_common(int(sys.argv[2]) if len(sys.argv) > 2 else 25):
    print(f"{n:14d} {100 * n / tot:5.1f}%  samples {samples[op]:7d}  {op}")
print("--- hottest runs (exec count x length)")
for n, L, c, smp in sorted(runs, key=lambda x: -x[0] * x[1])[:25]:
    print(f"{n * L:14d} {100 * n * L / tot:5.1f}%  exec {n:10d} len {L:4d} samples {smp:6d}  {dict(c.most_common(6))}")
