"""Slab partition (row A11) on one GPU: gmt_create_slabs runs the partitioned
V-cycle -- ghost-plane halos, region restriction into the first replicated
level + all-gather, summed dot products -- with P virtual slabs, and must
reproduce the single-device problem (itself pinned to the oracle in
test_gpu_parity.py) and the oracle directly.

Per-node arithmetic is identical in both layouts (same kernels, same operand
order), so solutions agree to float rounding of the summed reductions only;
the bound used is 1e-6 relative (fp32 ulp scale), C^H 1e-5 vs the oracle
(north star)."""
import numpy as np
import pytest

import synth
from oracle import fem, gmg

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

OMEGA = {"elastic": 0.45, "thermal": 0.6}


@pytest.fixture(scope="module", autouse=True)
def _lib():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2604_26518_b200 import build
    build.build()


def _problem(s, kind, levels, slabs=1, **kw):
    from paper_2604_26518_b200 import Problem
    kw.setdefault("omega", OMEGA[kind])
    return Problem(np.ascontiguousarray(s, dtype=np.float32), physics=kind, levels=levels, slabs=slabs, **kw)


def from_gpu(a):
    M, dpn, n = a.shape[0], a.shape[1], a.shape[2]
    return np.asarray(a, dtype=np.float64).transpose(2, 3, 4, 1, 0).reshape(n ** 3 * dpn, M)


CASES = [
    ("elastic", "gyroid32-P2", lambda: synth.tpms(32, "gyroid", 0.3), 4, 2),
    ("elastic", "gyroid32-P4", lambda: synth.tpms(32, "gyroid", 0.3), 4, 4),
    ("thermal", "stoch32-P2", lambda: synth.stochastic(32, 0.3, seed=5), 4, 2),
    ("elastic", "octet64-P4", lambda: synth.truss(64, "octet", 0.08), 5, 4),
    ("thermal", "density32-P4", lambda: synth.random_density(32, 1e-3, 1.0, seed=6), 4, 4),
    # non-power-of-2 slab: 24 planes per slab, levels 0-2 partitioned, the
    # replicated level 3 assembled from 3-plane regions
    ("elastic", "gyroid48-P2", lambda: synth.tpms(48, "gyroid", 0.3), 4, 2),
]


@pytest.mark.parametrize("kind,name,gen,L,P", CASES, ids=[c[1] for c in CASES])
def test_slabs_match_single_device(kind, name, gen, L, P):
    s = gen()
    with _problem(s, kind, L) as A, _problem(s, kind, L, slabs=P) as B:
        assert B.num_slabs == P and A.num_slabs == 1
        rA, arA, afA = A.gmt_residual_norms()
        rB, arB, afB = B.gmt_residual_norms()
        assert np.allclose(afB, afA, rtol=1e-6) and np.allclose(rB, rA, rtol=1e-6)
        for cyc in range(3):
            A.gmt_vcycle(1)
            B.gmt_vcycle(1)
            uA, uB = A.gmt_get_solution(), B.gmt_get_solution()
            scale = np.abs(uA).max()
            err = np.abs(uB - uA).max() / scale
            assert err <= 1e-6, f"cycle {cyc}: {err:.2e}"
            rA, _, _ = A.gmt_residual_norms()
            rB, _, _ = B.gmt_residual_norms()
            assert np.allclose(rB, rA, rtol=1e-4), (cyc, rA, rB)
        CA, CB = A.gmt_homogenize(), B.gmt_homogenize()
        assert np.abs(CB - CA).max() <= 1e-6 * np.abs(CA).max()
        zA = A.gmt_get_solution(zero_mean=True)
        zB = B.gmt_get_solution(zero_mean=True)
        assert np.abs(zB - zA).max() <= 1e-6 * np.abs(zA).max()


def test_slabs_vs_oracle_vcycle_and_tensor():
    """Partitioned V-cycles against the FP64 oracle directly (thermal 32^3,
    4 slabs): per-cycle solution and reduction factor, then C^H of a solve."""
    kind, n, L = "thermal", 32, 4
    s = synth.tpms(n, "schwarz_p", 0.35, sheet=True)
    ph = fem.Physics(kind)
    H = gmg.Hierarchy(s, ph, L)
    kw = dict(omega=OMEGA[kind], pre=2, post=2, coarse=16)
    with _problem(s, kind, L, slabs=4) as B:
        u = np.zeros_like(H.f)
        r_prev_o = fem.relative_residual(H.K[0], u, H.f)
        r_prev_g, _, _ = B.gmt_residual_norms()
        act = np.repeat(H.active[0][:, None], ph.nrhs, axis=1)
        for cyc in range(3):
            u = gmg.vcycle(H, u, **kw)
            B.gmt_vcycle(1)
            ug = from_gpu(B.gmt_get_solution())
            err = np.abs(ug - u)[act].max() / np.abs(u[act]).max()
            assert err < 1e-4 * (cyc + 1), f"cycle {cyc}: {err:.2e}"
            r_o = fem.relative_residual(H.K[0], u, H.f)
            r_g, _, _ = B.gmt_residual_norms()
            rho_o, rho_g = r_o / r_prev_o, r_g / r_prev_g
            assert np.all(np.abs(rho_g - rho_o) <= 0.05 * rho_o), (cyc, rho_o, rho_g)
            r_prev_o, r_prev_g = r_o, r_g
        uo, _ = gmg.solve(H, tol=1e-9, max_cycles=400, **kw)
        CHo = fem.effective_tensor(s, ph, uo)
        B.gmt_set_initial_guess(None)
        k, fr, _ = B.gmt_solve(1e-6, 400)
        assert fr <= 1e-6
        CHg = B.gmt_homogenize()
        assert np.abs(CHg - CHo).max() / np.linalg.norm(CHo) <= 1e-5


def test_slabs_graphs_guess_and_material_roundtrip():
    s = synth.tpms(32, "diamond", 0.3)
    s2 = synth.truss(32, "bcc", 0.15)
    rng = np.random.default_rng(7)
    with _problem(s, "elastic", 4, slabs=2) as B, _problem(s, "elastic", 4, slabs=2, use_graphs=False) as C, \
            _problem(s, "elastic", 4) as A:
        g = (1e-2 * rng.standard_normal(A.vec_shape(0))).astype(np.float32)
        for P in (A, B, C):
            P.gmt_set_initial_guess(g)
            P.gmt_vcycle(2)
        uA, uB, uC = (P.gmt_get_solution() for P in (A, B, C))
        assert np.array_equal(uB, uC)                      # graph replay == eager launches
        assert np.abs(uB - uA).max() <= 1e-6 * np.abs(uA).max()
        # device output buffer
        ud = torch.empty(B.vec_shape(0), device="cuda")
        B.gmt_get_solution(out=ud)
        assert np.array_equal(ud.cpu().numpy(), uB)
        # new material (u8 occupancy, from the device): operators rebuilt, solution reset
        for P in (A, B):
            P.gmt_set_material(torch.from_numpy((s2 > 0).astype(np.uint8)).cuda())
            P.gmt_vcycle(2)
        uA, uB = A.gmt_get_solution(), B.gmt_get_solution()
        assert np.abs(uB - uA).max() <= 1e-6 * np.abs(uA).max()
        assert np.abs(B.gmt_homogenize() - A.gmt_homogenize()).max() <= 1e-6 * np.abs(A.gmt_homogenize()).max()


def test_slab_errors():
    from paper_2604_26518_b200 import GmtError
    s = synth.tpms(32, "gyroid", 0.3)
    with _problem(s, "elastic", 4, slabs=2) as B:
        u = torch.zeros(B.vec_shape(0), device="cuda")
        with pytest.raises(GmtError):
            B.gmt_op_apply(0, u, torch.empty_like(u))
        with pytest.raises(GmtError):
            B.gmt_inject_correction(1, np.zeros(B.vec_shape(1), np.float32))
    with pytest.raises(GmtError):            # 16 / 4 = 4 planes: < 3 partitioned levels
        _problem(synth.tpms(16, "gyroid", 0.3), "elastic", 3, slabs=4)


def test_nccl_loads_and_makes_unique_id():
    """The NCCL transport dlopens libnccl.so.2 (torch's copy when torch is
    loaded) and creates the id rank 0 broadcasts to gmt_create_dist."""
    from paper_2604_26518_b200 import gmt
    a, b = gmt.gmt_nccl_unique_id(), gmt.gmt_nccl_unique_id()
    assert len(a) == 128 and a != bytes(128) and a != b


def test_slabs_refinement_matches_single_device():
    """Iterative refinement on 4 slabs (hi / lo ghosts for the defect) equals
    the single-device refinement and solves below the plain fp32 floor."""
    s = synth.tpms(64, "gyroid", 0.3)
    with _problem(s, "elastic", 5) as A, _problem(s, "elastic", 5, slabs=4) as B:
        for P in (A, B):
            P.gmt_set_refinement(2)
            assert P.gmt_refinement_active()
            P.gmt_vcycle(3)
        uA, uB = A.gmt_get_solution(), B.gmt_get_solution()
        assert np.abs(uB - uA).max() <= 1e-6 * np.abs(uA).max()
        rA, _, _ = A.gmt_residual_norms()
        rB, _, _ = B.gmt_residual_norms()
        assert np.allclose(rB, rA, rtol=1e-3)
        for P in (A, B):
            k, fr, _ = P.gmt_solve(3e-7, 120)
            assert fr <= 3e-7, (k, fr)
        CA, CB = A.gmt_homogenize(), B.gmt_homogenize()
        assert np.abs(CB - CA).max() <= 1e-6 * np.abs(CA).max()


def test_gather_level_env_matches_single_device(monkeypatch):
    """GMT_SLAB_MIN_PLANES moves the gather level (first replicated level):
    64^3 on 4 slabs partitions levels 0-3 by default and 0-2 with a minimum
    of 4 planes; both reproduce the single-device V-cycles and C^H."""
    from paper_2604_26518_b200 import gmt
    s = synth.tpms(64, "gyroid", 0.3)
    monkeypatch.setenv("GMT_SLAB_MIN_PLANES", "4")
    assert gmt.gmt_slab_layout(64, 5, 4, 0)["Ld"] == 3
    with _problem(s, "elastic", 5) as A, _problem(s, "elastic", 5, slabs=4) as B:
        A.gmt_vcycle(3)
        B.gmt_vcycle(3)
        uA, uB = A.gmt_get_solution(), B.gmt_get_solution()
        assert np.abs(uB - uA).max() <= 1e-6 * np.abs(uA).max()
        CA, CB = A.gmt_homogenize(), B.gmt_homogenize()
        assert np.abs(CB - CA).max() <= 1e-6 * np.abs(CA).max()


@pytest.mark.parametrize("kind,P", [("elastic", 2), ("thermal", 4)])
def test_halo_overlap_matches_serial_exchange(kind, P, monkeypatch):
    """Level-0 sweeps with the ghost-plane exchange on a second stream while
    each slab's interior planes sweep, boundary planes after it (default),
    against exchange-then-sweep (GMT_HALO_OVERLAP=0): the same per-node
    arithmetic in another z chunking, so the V-cycles agree to fp32 rounding,
    and both stay on the single-device problem."""
    s = synth.tpms(64, "gyroid", 0.3)
    monkeypatch.setenv("GMT_HALO_OVERLAP", "0")
    B0 = _problem(s, kind, 5, slabs=P)
    monkeypatch.delenv("GMT_HALO_OVERLAP")
    with B0, _problem(s, kind, 5, slabs=P) as B1, _problem(s, kind, 5) as A:
        for cyc in range(3):
            for X in (A, B0, B1):
                X.gmt_vcycle(1)
            uA, u0, u1 = A.gmt_get_solution(), B0.gmt_get_solution(), B1.gmt_get_solution()
            scale = np.abs(uA).max()
            assert np.abs(u1 - u0).max() <= 1e-6 * scale, cyc
            assert np.abs(u1 - uA).max() <= 1e-6 * scale, cyc
        CA, C1 = A.gmt_homogenize(), B1.gmt_homogenize()
        assert np.abs(C1 - CA).max() <= 1e-6 * np.abs(CA).max()
