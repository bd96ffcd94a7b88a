"""Per-part V-cycle breakdown of bench lines (files given on the command line)."""
import json
import sys

for f in sys.argv[1:]:
    for line in open(f):
        if not line.startswith("{"):
            continue
        d = json.loads(line)
        b = d.get("breakdown", {})
        parts = " ".join(f"{k} {v['ms_per_step']:.3f}" for k, v in b.items())
        print(f"{f.split('/')[-1]:14s} vcycle {d.get('vcycle_ms', 0):.3f} step {d['ms_per_step']:.3f} | {parts}")
