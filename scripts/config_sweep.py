"""Robustness sweep over resolutions / physics / partitions: every config must
solve to 1e-5 (or refine) and give a symmetric positive C^H; the
single-device and slab results must agree."""
import sys
import numpy as np
sys.path.insert(0, ".")
import synth
from paper_2604_26518_b200 import Problem

fails = 0
for n, L in ((36, 0), (48, 0), (96, 0), (100, 0), (120, 4), (160, 0), (200, 0)):
    s = synth.tpms(n, "diamond", 0.25)
    for kind in ("elastic", "thermal"):
        try:
            with Problem(s, physics=kind, levels=L) as P:
                k, fr, _ = P.gmt_solve(1e-5, 200)
                CH = P.gmt_homogenize()
                ok = fr <= 1e-5 and np.allclose(CH, CH.T, atol=1e-12) and np.linalg.eigvalsh(CH).min() > 0
                print(f"n={n} L={P.levels} {kind}: cycles {k} rel {fr:.1e} refine {P.gmt_refinement_active()} "
                      f"C11 {CH[0,0]:.6f} {'OK' if ok else 'FAIL'}", flush=True)
                fails += not ok
        except Exception as e:
            print(f"n={n} {kind}: ERROR {e}", flush=True)
            fails += 1
for n, P_ in ((64, 2), (96, 2), (128, 4), (192, 2)):
    s = synth.stochastic(n, 0.3, seed=1)
    for kind in ("elastic", "thermal"):
        try:
            with Problem(s, physics=kind) as A, Problem(s, physics=kind, slabs=P_) as B:
                for Q in (A, B):
                    Q.gmt_solve(1e-5, 200)
                CA, CB = A.gmt_homogenize(), B.gmt_homogenize()
                err = np.abs(CA - CB).max() / np.abs(CA).max()
                ok = err < 1e-5
                print(f"slabs n={n} P={P_} {kind}: C^H diff {err:.1e} {'OK' if ok else 'FAIL'}", flush=True)
                fails += not ok
        except Exception as e:
            print(f"slabs n={n} P={P_} {kind}: ERROR {e}", flush=True)
            fails += 1
print("FAILS", fails)
