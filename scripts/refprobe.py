import sys; sys.path.insert(0, '.')
import numpy as np, synth
from oracle import fem, gmg
from paper_2604_26518_b200 import Problem
def fg(a):
    M, dpn, n = a.shape[0], a.shape[1], a.shape[2]
    return np.asarray(a, dtype=np.float64).transpose(2, 3, 4, 1, 0).reshape(n ** 3 * dpn, M)
s = synth.truss(32, "bcc", 0.14); ph = fem.Physics("elastic"); H = gmg.Hierarchy(s, ph, 4)
uo, _ = gmg.solve(H, tol=1e-11, max_cycles=600, omega=0.45, pre=2, post=2, coarse=16)
uo = gmg.project_zero_mean(uo, 3, H.active[0].reshape(-1, 3)[:, 0]); CHo = fem.effective_tensor(s, ph, uo)
act = np.repeat(H.active[0][:, None], 6, axis=1)
for mode in (1, 0):
    with Problem(s, physics="elastic", levels=4, omega=0.45) as P:
        P.gmt_set_refinement(mode); k, fr, h = P.gmt_solve(1e-12, 250)
        ug = fg(P.gmt_get_solution(zero_mean=True)); err = np.abs(ug - uo)[act].max() / np.abs(uo[act]).max()
        CH = P.gmt_homogenize()
        print("32 mode", mode, "cycles", k, "fr %.2e err %.2e CHerr %.2e" % (fr, err, np.abs(CH - CHo).max() / np.linalg.norm(CHo)), "hist", [f"{x:.1e}" for x in h.max(1)[::25]], flush=True)
s = synth.tpms(128, "gyroid", 0.3)
for mode in (1, 0):
    with Problem(s, physics="elastic", omega=0.45) as P:
        P.gmt_set_refinement(mode); k, fr, h = P.gmt_solve(1e-12, 120)
        print("128 mode", mode, "cycles", k, "fr %.2e" % fr, [f"{x:.1e}" for x in h.max(1)[::10]], flush=True)
