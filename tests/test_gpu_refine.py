"""Mixed-precision iterative refinement (gmt_set_refinement): the fp32
solution stalls at a relative residual ~ N * 2^-24 because |u| grows like N;
refinement keeps the solution as hi + lo and cycles on the fp32 correction.

* A refinement V-cycle is the same V-cycle in exact arithmetic: per-cycle
  solutions and residual reduction factors match the FP64 oracle (Alg. 1)
  to the tolerances of test_gpu_parity.py.
* A refined solve matches the oracle's converged fp64 solution (5e-7) and
  C^H (1e-7).
* gmt_solve's automatic switch takes a 128^3 problem below its fp32 floor.
"""
import numpy as np
import pytest

import synth
from oracle import fem, gmg

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _lib():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2604_26518_b200 import build
    build.build()


def _problem(s, kind, levels, **kw):
    from paper_2604_26518_b200 import Problem
    kw.setdefault("omega", 0.45 if kind == "elastic" else 0.6)
    return Problem(np.ascontiguousarray(s, dtype=np.float32), physics=kind, levels=levels, **kw)


def from_gpu(a):
    M, dpn, n = a.shape[0], a.shape[1], a.shape[2]
    return np.asarray(a, dtype=np.float64).transpose(2, 3, 4, 1, 0).reshape(n ** 3 * dpn, M)


@pytest.mark.parametrize("kind", ["elastic", "thermal"])
def test_refinement_cycles_match_oracle(kind):
    s = synth.tpms(16, "gyroid", 0.3)
    ph = fem.Physics(kind)
    H = gmg.Hierarchy(s, ph, 3)
    om = 0.45 if kind == "elastic" else 0.6
    u = np.zeros_like(H.f)
    with _problem(s, kind, 3) as P:
        P.gmt_set_refinement(2)
        assert P.gmt_refinement_active()
        r_prev_o = fem.relative_residual(H.K[0], u, H.f)
        r_prev_g, _, _ = P.gmt_residual_norms()
        assert np.allclose(r_prev_g, r_prev_o, rtol=1e-5)
        act = np.repeat(H.active[0][:, None], ph.nrhs, axis=1)
        for cyc in range(4):
            u = gmg.vcycle(H, u, omega=om, pre=2, post=2, coarse=16)
            P.gmt_vcycle(1)
            ug = from_gpu(P.gmt_get_solution())
            err = np.abs(ug - u)[act].max() / np.abs(u[act]).max()
            assert err < 1e-4 * (cyc + 1), f"cycle {cyc}: {err:.2e}"
            r_o = fem.relative_residual(H.K[0], u, H.f)
            r_g, _, _ = P.gmt_residual_norms()
            rho_o, rho_g = r_o / r_prev_o, r_g / r_prev_g
            assert np.all(np.abs(rho_g - rho_o) <= 0.05 * rho_o), (cyc, rho_o, rho_g)
            r_prev_o, r_prev_g = r_o, r_g


def test_refined_solve_matches_converged_oracle():
    """Refined solve of a 32^3 truss against the oracle's converged fp64
    solution: solution to 5e-7 (the fp32 output), C^H to 1e-7."""
    kind, n, L = "elastic", 32, 4
    s = synth.truss(n, "bcc", 0.14)
    ph = fem.Physics(kind)
    H = gmg.Hierarchy(s, ph, L)
    uo, hist = gmg.solve(H, tol=1e-11, max_cycles=600, omega=0.45, pre=2, post=2, coarse=16)
    uo = gmg.project_zero_mean(uo, ph.dpn, H.active[0].reshape(-1, ph.dpn)[:, 0])
    CHo = fem.effective_tensor(s, ph, uo)
    act = np.repeat(H.active[0][:, None], ph.nrhs, axis=1)
    with _problem(s, kind, L) as P:
        P.gmt_set_refinement(2)
        k, fr, h = P.gmt_solve(3e-7, 250)
        assert fr <= 3e-7, (k, fr)
        ug = from_gpu(P.gmt_get_solution(zero_mean=True))
        CH = P.gmt_homogenize()
    err = np.abs(ug - uo)[act].max() / np.abs(uo[act]).max()
    assert err < 5e-7, err
    assert np.abs(CH - CHo).max() / np.linalg.norm(CHo) <= 1e-7


def test_auto_switch_below_fp32_floor():
    """128^3: plain fp32 cycles stall near 1e-5 (~N 2^-24); gmt_solve's
    automatic switch reaches 5e-7 (the floor of the fp32 defect, ~3.5e-7 with
    the sum-factorised level-0 operator, independent of N)."""
    s = synth.tpms(128, "gyroid", 0.3)
    with _problem(s, "elastic", 0) as P:
        P.gmt_set_refinement(1)                   # plain fp32: stalls
        k, fr, _ = P.gmt_solve(3e-7, 60)
        assert fr > 5e-6 and not P.gmt_refinement_active()
        P.gmt_set_initial_guess(None)
        P.gmt_set_refinement(0)                   # auto
        k, fr, h = P.gmt_solve(5e-7, 120)
        assert P.gmt_refinement_active()
        assert fr <= 5e-7, (k, fr)
        # leaving refinement keeps the solution (fp32(hi + lo))
        u_ref = P.gmt_get_solution()
        P.gmt_set_refinement(1)
        assert not P.gmt_refinement_active()
        assert np.array_equal(P.gmt_get_solution(), u_ref)
