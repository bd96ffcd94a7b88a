"""Where the bench step goes, call by call (device time per public API call,
synchronised between calls, so overlap between calls is removed).
usage: python scripts/step_split.py [--res 512] [--reps 5]"""
import argparse
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth  # noqa: E402
from paper_2604_26518_b200 import Problem, build  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--res", type=int, default=512)
ap.add_argument("--reps", type=int, default=5)
a = ap.parse_args()
build.build()
n = a.res
s = synth.tpms(n, "gyroid", 0.3)
s_dev = torch.from_numpy(np.ascontiguousarray(s)).cuda()
u0_dev = torch.from_numpy(synth.initial_guess(n, 6, 3, seed=1, material=s, z0=0, nz=n)).cuda()
P = Problem(s_dev, physics="elastic")
st = torch.cuda.ExternalStream(P.stream)
calls = [("set_material", lambda: P.gmt_set_material(s_dev)),
         ("set_initial_guess", lambda: P.gmt_set_initial_guess(u0_dev)),
         ("vcycle", lambda: P.gmt_vcycle(1)),
         ("homogenize", lambda: P.gmt_homogenize())]
tot = {k: [] for k, _ in calls}
for r in range(a.reps + 2):
    for k, f in calls:
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(st)
        f()
        e1.record(st)
        torch.cuda.synchronize()
        if r >= 2:
            tot[k].append(e0.elapsed_time(e1))
for k, v in tot.items():
    print(f"{k:20s} {np.median(v):8.3f} ms  (min {min(v):.3f})")
print(f"{'sum':20s} {sum(np.median(v) for v in tot.values()):8.3f} ms")
