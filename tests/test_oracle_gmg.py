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


# ------------------------------------------------------------------ per-cycle pins (round 2)

def test_jacobi_hand_evaluated_single_voxel_heat():
    """Sec. 4.6 Eq. 16 update u <- u + omega D^-1 (f - K u), evaluated by hand
    on the 2^3 periodic grid holding one solid voxel (heat, kappa = 1).

    Every node is then exactly one corner k of that voxel, so K = K_e^th
    (diagonal 1/3, edge neighbours 0, face and body diagonals -1/12) and
    D = 1/3 at every node.  Load case m (unit gradient e_m, App. F2):
    f_k = int dN_k/dx_m = (2 k_m - 1) / 4.
      sweep 1 from u = 0:  u = omega * 3 * f            -> +-3 omega / 4
      sweep 2:  K f = f / 2 (K_e applied to the corner coordinate k_m / 2 -
                1/4: row sums of the -1/12 entries over the k_m = 1 face),
                u = 3 omega f (2 - 3 omega / 2)          -> +-3 omega / 4 (2 - 1.5 omega)
    With omega = 0.6: 0.45 and 0.495.  A wrong omega, a diagonal from another
    operator or an update from the new iterate changes these numbers."""
    ph = fem.Physics("thermal")
    s = np.zeros((2, 2, 2), np.float32)
    s[0, 0, 0] = 1.0
    H = gmg.Hierarchy(s, ph, 1)
    assert np.allclose(H.K[0].diagonal(), 1.0 / 3.0)
    om = 0.6
    sign = np.zeros((8, 3))
    for node in range(8):
        x, y, z = node & 1, (node >> 1) & 1, (node >> 2) & 1
        sign[node] = [2 * x - 1, 2 * y - 1, 2 * z - 1]
    u1 = gmg.jacobi(H.K[0], H.Dinv[0], np.zeros((8, 3)), H.f, om, 1)
    assert np.abs(u1 - sign * 0.45).max() < 1e-15
    u2 = gmg.jacobi(H.K[0], H.Dinv[0], np.zeros((8, 3)), H.f, om, 2)
    assert np.abs(u2 - sign * 0.495).max() < 1e-15
    u3 = gmg.jacobi(H.K[0], H.Dinv[0], u1, H.f, om, 1)          # sweeps compose
    assert np.abs(u3 - u2).max() < 1e-15


def _dense_cycle_operators(H, omega, pre, post, coarse):
    """Alg. 1 written as matrices instead of a loop.  With S_l = I - omega
    D_l^-1 K_l, W_l = omega D_l^-1 and Q_l(k) = sum_{j<k} S_l^j W_l (k sweeps
    from a zero guess), the cycle from a zero guess at level l is
        B_{L-1} = Q(It_L),
        B_l     = S_l^post [Q_l(pre) + P_l B_{l+1} P_l^T (I - K_l Q_l(pre))] + Q_l(post),
    and the level-l cycle from a guess u is u -> E_l u + B_l f with the
    error propagation E_l = S_l^post (I - P_l B_{l+1} P_l^T K_l) S_l^pre."""
    L = H.L
    K = [k.toarray() for k in H.K]
    P = [p.toarray() for p in H.P]
    S, Wm = [], []
    for l in range(L):
        Wm.append(omega * np.diag(H.Dinv[l]))
        S.append(np.eye(K[l].shape[0]) - Wm[l] @ K[l])

    def Q(l, k):
        out = np.zeros_like(K[l])
        for _ in range(k):
            out = S[l] @ out + Wm[l]
        return out

    mp = np.linalg.matrix_power
    B = [None] * L
    E = [None] * L
    B[L - 1] = Q(L - 1, coarse)
    E[L - 1] = mp(S[L - 1], coarse)
    for l in range(L - 2, -1, -1):
        Qp = Q(l, pre)
        I = np.eye(K[l].shape[0])
        C = P[l] @ B[l + 1] @ P[l].T
        B[l] = mp(S[l], post) @ (Qp + C @ (I - K[l] @ Qp)) + Q(l, post)
        E[l] = mp(S[l], post) @ (I - C @ K[l]) @ mp(S[l], pre)
    return E, B, S, P


@pytest.mark.parametrize("kind,n,L,pre,post,coarse", [("thermal", 8, 3, 2, 2, 5),
                                                      ("elastic", 4, 2, 1, 3, 4),
                                                      ("thermal", 8, 2, 3, 1, 7)])
def test_vcycle_equals_dense_error_propagation(kind, n, L, pre, post, coarse):
    """gmg.vcycle (the loop of Alg. 1) == E_0 u + B_0 f from the matrix
    recursion above, for random u and f.  Dropping post-smoothing,
    restricting before pre-smoothing, a wrong sweep count or a wrong level's
    diagonal all change E_0 or B_0."""
    ph = fem.Physics(kind)
    om = 0.45 if kind == "elastic" else 0.6
    s = synth.random_occupancy(n, 0.6, seed=3)
    H = gmg.Hierarchy(s, ph, L)
    E, B, _, _ = _dense_cycle_operators(H, om, pre, post, coarse)
    rng = np.random.default_rng(1)
    u = rng.standard_normal(H.f.shape)
    f = rng.standard_normal(H.f.shape)
    got = gmg.vcycle(H, u, f1=f, omega=om, pre=pre, post=post, coarse=coarse)
    want = E[0] @ u + B[0] @ f
    assert np.abs(got - want).max() <= 1e-11 * np.abs(want).max()


def test_alg2_injection_equals_dense_coarse_error_propagation():
    """Alg. 2 line 6: the level-1 cycle starts from the injected e_hat instead
    of 0, so vcycle(.., inject={1: e}) - vcycle(..) = S_0^post P_0 E_1 e."""
    ph = fem.Physics("thermal")
    s = synth.random_occupancy(8, 0.6, seed=4)
    H = gmg.Hierarchy(s, ph, 3)
    om, pre, post, coarse = 0.6, 2, 2, 4
    E, B, S, P = _dense_cycle_operators(H, om, pre, post, coarse)
    rng = np.random.default_rng(2)
    e = rng.standard_normal((H.K[1].shape[0], 3))
    f = rng.standard_normal(H.f.shape)
    a = gmg.vcycle(H, np.zeros_like(f), f1=f, omega=om, pre=pre, post=post, coarse=coarse, inject={1: e})
    b = gmg.vcycle(H, np.zeros_like(f), f1=f, omega=om, pre=pre, post=post, coarse=coarse)
    want = np.linalg.matrix_power(S[0], post) @ P[0] @ E[1] @ e
    assert np.abs((a - b) - want).max() <= 1e-11 * np.abs(want).max()


def test_project_zero_mean_worked_example():
    """Sec. 4.5 gauge sum_i u_i = 0 over active nodes, per component and load
    case; inactive nodes are left alone.  Worked by hand: active values
    (1, 2, 6) have mean 3."""
    u = np.array([[1.0], [2.0], [5.0], [6.0]])
    act = np.array([True, True, False, True])
    got = gmg.project_zero_mean(u, 1, act)
    assert np.array_equal(got, np.array([[-2.0], [-1.0], [5.0], [3.0]]))
    # dpn = 2, two load cases: components are separate, constants vanish
    rng = np.random.default_rng(0)
    v = rng.standard_normal((5, 2, 2))
    v -= v.mean(axis=0, keepdims=True)                   # zero mean per (component, case)
    shift = np.array([[3.0, -1.0], [0.5, 7.0]])          # [component, case]
    u = (v + shift[None]).reshape(10, 2)
    got = gmg.project_zero_mean(u, 2)
    assert np.abs(got - v.reshape(10, 2)).max() < 1e-14


def test_relative_residual_closed_form():
    """Sec. 5.2 r = ||f - K u||_2 / ||f||_2 per load case; a zero right-hand
    side reports the absolute norm (hand values)."""
    import scipy.sparse as sp
    K = sp.identity(4, format="csr") * 2.0
    u = np.ones((4, 2))
    f = np.zeros((4, 2))
    f[:, 0] = 3.0                        # r = 1 everywhere: ||r|| = 2, ||f|| = 6
    got = fem.relative_residual(K, u, f)
    assert abs(got[0] - 1.0 / 3.0) < 1e-15
    assert abs(got[1] - 4.0) < 1e-15     # f = 0: ||-2 * 1|| = 4


@pytest.mark.parametrize("kind", ["elastic", "thermal"])
def test_effective_tensor_planes_partition(kind):
    """Plane-restricted App. F1/F2 sums over a partition of the planes add up
    to effective_tensor * N^3 (the definition split over a partition of the
    elements), on a random field and a density material."""
    ph = fem.Physics(kind)
    n = 8
    s = synth.random_density(n, 0.0, 1.0, seed=6)
    s[s < 0.3] = 0.0
    rng = np.random.default_rng(4)
    u = rng.standard_normal((n ** 3 * ph.dpn, ph.nrhs))
    want = fem.effective_tensor(s, ph, u) * n ** 3
    un = fem.to_node_layout(u, n, ph.dpn)                      # [z, y, x, m, c]
    got = sum(fem.effective_tensor_planes(s, ph, lambda z: un[z], a, b) for a, b in ((0, 3), (3, 4), (4, 8)))
    assert np.abs(got - want).max() <= 1e-12 * np.abs(want).max()
