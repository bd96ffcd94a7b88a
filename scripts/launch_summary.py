"""Per-kernel totals of an ncu launch list (--metrics gpu__time_duration.sum --csv)."""
import csv
import collections
import sys

lines = open(sys.argv[1]).read().split("\n")
i = next(k for k, l in enumerate(lines) if l.startswith('"ID"'))
rows = list(csv.reader(lines[i:]))
h = rows[0]
ik, iv, iu = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
tot = collections.defaultdict(float)
cnt = collections.Counter()
for r in rows[1:]:
    if len(r) <= iv:
        continue
    name = r[ik]
    short = name.split("(")[0].replace("void ", "")
    t = float(r[iv]) * {"nsecond": 1e-6, "usecond": 1e-3, "msecond": 1.0}.get(r[iu], 1e-6)
    tot[short] += t
    cnt[short] += 1
T = sum(tot.values())
for k, v in sorted(tot.items(), key=lambda x: -x[1]):
    print(f"{v:10.3f} ms {100 * v / T:5.1f}% n={cnt[k]:4d} avg {v / cnt[k]:8.3f} {k[:90]}")
print(f"total {T:.2f} ms")
