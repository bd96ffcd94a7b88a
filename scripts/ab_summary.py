"""Summarise the bench lines written by scripts/gpu_ab_old.sh: step, V-cycle, k_l0 launch, frac."""
import json
import sys
import glob
import os

d = sys.argv[1]
for f in sorted(glob.glob(os.path.join(d, "*.json"))):
    for line in open(f):
        line = line.strip()
        if not line.startswith("{"):
            continue
        j = json.loads(line)
        r = j.get("roofline", {})
        print(f"{os.path.basename(f):14s} step {j['ms_per_step']:7.3f}  vcycle {j.get('vcycle_ms', 0):7.3f}  "
              f"k_l0 {r.get('avg_launch_ms', 0):6.3f} ms  frac {r.get('frac', 0):.4f}")
