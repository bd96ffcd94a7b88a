"""Pins for oracle/transfer.py, oracle/gmg.py and oracle/fem.effective_tensor:
brute force, closed forms (laminates), bounds and dense direct solves."""
import numpy as np
import pytest

import synth
from oracle import fem, gmg, transfer


# ------------------------------------------------------------------ transfer

def test_stencil_worked_cases():
    """App. E1 by hand: xi = 0 -> single weight 1; xi = (0.5,0,0) -> 0.5/0.5;
    last fine node wraps to coarse node 0."""
    nf = 8
    nc = 4
    I, W = transfer.stencil(nf)

    def row(x, y, z):
        i = x + nf * (y + nf * z)
        return {int(a): float(w) for a, w in zip(I[i], W[i]) if w != 0}

    assert row(0, 0, 0) == {0: 1.0}
    assert row(1, 0, 0) == {0: 0.5, 1: 0.5}
    assert row(nf - 1, 0, 0) == {nc - 1: 0.5, 0: 0.5}
    assert row(1, 1, 1) == {a + nc * (b + nc * c): 0.125 for a in (0, 1) for b in (0, 1) for c in (0, 1)}


def test_prolongation_partition_of_unity_and_hat_functions():
    nf, nc = 8, 4
    P = transfer.prolongation(nf, 1)
    assert np.abs(P @ np.ones(nc ** 3) - 1).max() < 1e-15
    # coarse delta -> trilinear hat function (brute force, periodic distance)
    J = (1, 3, 2)
    e = np.zeros(nc ** 3); e[J[0] + nc * (J[1] + nc * J[2])] = 1
    u = (P @ e).reshape(nf, nf, nf)
    for z in range(nf):
        for y in range(nf):
            for x in range(nf):
                h = 1.0
                for xf, Jc in zip((x, y, z), J):
                    d = abs(xf / 2.0 - Jc)
                    d = min(d, nc - d)
                    h *= max(0.0, 1.0 - d)
                assert abs(u[z, y, x] - h) < 1e-15


def test_restriction_is_transpose_and_full_weighting():
    nf = 8
    P = transfer.prolongation(nf, 3)
    R = transfer.restriction(nf, 3)
    rng = np.random.default_rng(0)
    a, b = rng.standard_normal(P.shape[1]), rng.standard_normal(P.shape[0])
    assert abs((P @ a) @ b - a @ (R @ b)) < 1e-12
    # full weighting: restricting the constant 1 gives 8 (sum of 27 weights)
    Rn = transfer.restriction(nf, 1)
    assert np.abs(Rn @ np.ones(nf ** 3) - 8.0).max() < 1e-14


# ------------------------------------------------------------------ Galerkin

@pytest.mark.parametrize("kind", ["elastic", "thermal"])
def test_galerkin_global_equals_element_local(kind):
    """Sec. 3.2 global R K P (Hierarchy) == Sec. 4.6 Eq. 17 element-local
    R_loc K_patch P_loc, assembled, at levels 1->2 and 2->3."""
    ph = fem.Physics(kind)
    n = 8
    s = synth.random_occupancy(n, 0.4, seed=5)
    H = gmg.Hierarchy(s, ph, 3)
    Kel = gmg.level1_element_matrices(s, ph)
    for l in range(2):
        Kel = gmg.coarse_element_matrices(Kel, H.n[l], ph.dpn)
        Kc = gmg.assemble_from_elements(Kel, H.n[l + 1], ph.dpn)
        assert abs(Kc - H.K[l + 1]).max() < 1e-12 * abs(H.K[l + 1]).max()
    # coarse operator stays symmetric with the translations in its null space
    for K in H.K:
        assert abs(K - K.T).max() < 1e-12
        t = np.zeros(K.shape[0]); t[0::ph.dpn] = 1
        assert np.abs(K @ t).max() < 1e-11


def test_galerkin_single_child_patch():
    """Patch with one active fine element: kernel = P_j^T K_e P_j with P_j
    the rows of P_loc for that child (direct small-matrix product)."""
    ph = fem.Physics("thermal")
    s = np.zeros((2, 2, 2), np.float32); s[1, 0, 1] = 1.0   # child (x=1,y=0,z=1) -> j = 5
    Kel = gmg.coarse_element_matrices(gmg.level1_element_matrices(s, ph), 2, 1)
    Pl = gmg.local_prolongation(1)
    j = 5
    rows = []
    for k in range(8):
        p = fem.CORNERS[j] + fem.CORNERS[k]
        rows.append(p[0] + 3 * p[1] + 9 * p[2])
    Pj = Pl[rows]
    assert np.abs(Kel[0] - Pj.T @ ph.Ke @ Pj).max() < 1e-15


# ------------------------------------------------------------------ smoother / cycle

def _dense_solution(H):
    """Direct dense least-squares solve of K u = f (min-norm), then the
    zero-mean gauge -- independent of the multigrid path."""
    K = H.K[0].toarray()
    dpn = H.phys.dpn
    # gauge: add the translation projectors (null space of a connected
    # periodic structure); fall back to min-norm least squares otherwise
    act = np.diag(K) > 0
    T = np.zeros((K.shape[0], dpn))
    for c in range(dpn):
        T[c::dpn, c] = act[c::dpn]
        T[:, c] /= np.linalg.norm(T[:, c])
    Kr = K + np.abs(K).max() * (T @ T.T + np.diag(~act))
    u = np.linalg.solve(Kr, H.f)
    u[~act] = 0.0
    if np.abs(K @ u - H.f).max() > 1e-10 * max(1.0, np.abs(H.f).max()):
        u, *_ = np.linalg.lstsq(K, H.f, rcond=1e-12)
    return u


@pytest.mark.parametrize("kind", ["elastic", "thermal"])
def test_vcycle_solve_matches_dense_direct_solve(kind):
    """Alg. 1 V-cycles iterated to 1e-10 reproduce the dense direct solve's
    C^H (App. F1/F2) on 4^3 random occupancies (SPEC acceptance 5 analogue)."""
    ph = fem.Physics(kind)
    om = 0.45 if kind == "elastic" else 0.6
    for seed in range(3):
        s = synth.random_occupancy(4, 0.6, seed=seed)
        H = gmg.Hierarchy(s, ph, 2)
        u, hist = gmg.solve(H, tol=1e-10, max_cycles=400, omega=om, coarse=20)
        assert hist[-1].max() <= 1e-10
        ud = _dense_solution(H)
        CH = fem.effective_tensor(s, ph, u)
        CHd = fem.effective_tensor(s, ph, ud)
        assert np.abs(CH - CHd).max() <= 1e-8 * np.abs(CHd).max()
        # the solutions agree up to the null space (compare residual-free parts)
        assert np.abs(H.K[0] @ (u - ud)).max() < 1e-8


def test_jacobi_and_vcycle_fixed_point():
    ph = fem.Physics("elastic")
    s = synth.tpms(8, "gyroid", 0.4)
    H = gmg.Hierarchy(s, ph, 3)
    ud = _dense_solution(H)
    u1 = gmg.jacobi(H.K[0], H.Dinv[0], ud, H.f, 0.45, 3)
    assert np.abs(u1 - ud).max() < 1e-9
    u2 = gmg.vcycle(H, ud, omega=0.45)
    r0 = np.linalg.norm(H.f - H.K[0] @ ud)
    r1 = np.linalg.norm(H.f - H.K[0] @ u2)
    assert r1 <= r0 + 1e-10 * np.linalg.norm(H.f)


def test_vcycle_injection_zero_equals_standard_and_reduces_residual():
    ph = fem.Physics("thermal")
    s = synth.tpms(16, "gyroid", 0.3)
    H = gmg.Hierarchy(s, ph, 3)
    u0 = np.zeros_like(H.f)
    a = gmg.vcycle(H, u0, omega=0.6)
    b = gmg.vcycle(H, u0, omega=0.6, inject={1: np.zeros_like(H.P[0].T @ H.f),
                                              2: np.zeros((H.n[2] ** 3, 3))})
    assert np.array_equal(a, b)
    r = fem.relative_residual(H.K[0], a, H.f)
    assert np.all(r < 0.5)


def test_inactive_dofs_stay_zero():
    """Reading R2: nodes whose 8 voxels are void are outside the active set."""
    ph = fem.Physics("elastic")
    s = synth.laminate(8, axis=0, layers=3)          # x >= 4 nodes fully void
    H = gmg.Hierarchy(s, ph, 2)
    u = gmg.vcycle(H, np.zeros_like(H.f), omega=0.45)
    un = fem.to_node_layout(u, 8, 3)
    assert np.all(un[:, :, 4:8] == 0)
    assert np.any(un[:, :, 1:3] != 0)


# ------------------------------------------------------------------ C^H closed forms

def _laminate_exact(C1, C2, f1, axis):
    """Exact effective stiffness of a two-phase laminate with normal e_axis
    (continuity of tangential strains and normal tractions)."""
    n_idx = {0: [0, 4, 5], 1: [1, 3, 5], 2: [2, 3, 4]}[axis]
    t_idx = [i for i in range(6) if i not in n_idx]
    phases = [(C1, f1), (C2, 1 - f1)]

    def avg(fun):
        return sum(w * fun(C) for C, w in phases)

    inv = np.linalg.inv
    nn = lambda C: C[np.ix_(n_idx, n_idx)]
    nt = lambda C: C[np.ix_(n_idx, t_idx)]
    tn = lambda C: C[np.ix_(t_idx, n_idx)]
    tt = lambda C: C[np.ix_(t_idx, t_idx)]
    Hnn = inv(avg(lambda C: inv(nn(C))))
    Hnt = Hnn @ avg(lambda C: inv(nn(C)) @ nt(C))
    Htt = avg(lambda C: tt(C) - tn(C) @ inv(nn(C)) @ nt(C)) + avg(lambda C: tn(C) @ inv(nn(C))) @ Hnt
    H = np.zeros((6, 6))
    H[np.ix_(n_idx, n_idx)] = Hnn
    H[np.ix_(n_idx, t_idx)] = Hnt
    H[np.ix_(t_idx, n_idx)] = Hnt.T
    H[np.ix_(t_idx, t_idx)] = Htt
    return H


@pytest.mark.parametrize("axis", [0, 2])
def test_elastic_laminate_closed_form_and_bounds(axis):
    ph = fem.Physics("elastic")
    n, layers, s1, s2 = 8, 3, 1.0, float(np.float32(0.2))   # material is stored as float32
    s = synth.laminate(n, axis=axis, layers=layers, s_solid=s1, s_other=s2)
    H = gmg.Hierarchy(s, ph, 2)
    u = _dense_solution(H)
    CH = fem.effective_tensor(s, ph, u)
    f1 = layers / n
    exact = _laminate_exact(s1 * ph.C0, s2 * ph.C0, f1, axis)
    assert np.abs(CH - exact).max() < 1e-10
    voigt = (f1 * s1 + (1 - f1) * s2) * ph.C0
    reuss = np.linalg.inv(f1 * np.linalg.inv(s1 * ph.C0) + (1 - f1) * np.linalg.inv(s2 * ph.C0))
    assert np.linalg.eigvalsh(voigt - CH).min() > -1e-10
    assert np.linalg.eigvalsh(CH - reuss).min() > -1e-10


def test_thermal_laminate_series_parallel():
    ph = fem.Physics("thermal")
    n, layers = 16, 8
    for s_other in (0.0, 0.25):
        s = synth.laminate(n, axis=0, layers=layers, s_solid=1.0, s_other=s_other)
        H = gmg.Hierarchy(s, ph, 3)
        u, hist = gmg.solve(H, tol=1e-11, max_cycles=300, omega=0.6, coarse=30)
        CH = fem.effective_tensor(s, ph, u)
        par = 0.5 * (1.0 + s_other)
        ser = 0.0 if s_other == 0 else 1.0 / (0.5 / 1.0 + 0.5 / s_other)
        assert abs(CH[1, 1] - par) < 1e-8 and abs(CH[2, 2] - par) < 1e-8
        assert abs(CH[0, 0] - ser) < 1e-8
        assert np.abs(CH - np.diag(np.diag(CH))).max() < 1e-8


def test_gyroid_tensor_sanity():
    """SPEC acceptance 13: symmetric, PSD, within the Voigt bound v_f C_0."""
    ph = fem.Physics("elastic")
    s = synth.tpms(8, "gyroid", 0.35)
    H = gmg.Hierarchy(s, ph, 2)
    CH = fem.effective_tensor(s, ph, _dense_solution(H))
    assert np.abs(CH - CH.T).max() < 1e-10 * np.abs(CH).max()
    assert np.linalg.eigvalsh(CH).min() > -1e-10
    vf = synth.volume_fraction(s)
    assert np.linalg.eigvalsh(vf * ph.C0 - CH).min() > -1e-10
