"""Convergence study of the GMG solve at large N (history of max_m r_m)."""
import sys
import numpy as np
sys.path.insert(0, ".")
import synth
from paper_2604_26518_b200 import Problem

n = int(sys.argv[1]) if len(sys.argv) > 1 else 512
for L in [int(v) for v in (sys.argv[2].split(",") if len(sys.argv) > 2 else ["8"])]:
    s = synth.tpms(n, "gyroid", 0.3)
    for pre, post, cs in ((2, 2, 16), (4, 4, 32)):
        with Problem(s, physics="elastic", levels=L, pre_sweeps=pre, post_sweeps=post, coarse_sweeps=cs) as P:
            k, fr, h = P.gmt_solve(1e-6, 120)
            w = h.max(axis=1)
            print(f"n={n} L={L} pre/post={pre}/{post} coarse={cs}: cycles={k} final={fr:.2e} "
                  f"hist[0,1,5,10,20,40,80,120]={[f'{w[i]:.1e}' for i in (0, 1, 5, 10, 20, 40, 80, 120) if i < len(w)]}",
                  flush=True)
