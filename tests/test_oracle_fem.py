"""Pins for oracle/fem.py against closed forms, invariants and brute force.

Each test names the oracle function it pins and the independent truth used.
"""
import json
import os

import numpy as np
import pytest

import synth
from oracle import fem

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def _gold(name):
    with open(os.path.join(GOLD, name)) as fh:
        return json.load(fh)


# ---------------------------------------------------------------- element data

def test_thermal_element_matrix_closed_form():
    """element_matrix_thermal vs the exact-integral closed form (golden)."""
    g = _gold("thermal_element_matrix.json")
    K = fem.element_matrix_thermal(1.0)
    for a in range(8):
        for b in range(8):
            h = int(np.sum(fem.CORNERS[a] != fem.CORNERS[b]))
            assert abs(K[a, b] - g["by_hamming_distance"][str(h)]) < 1e-14
    assert np.allclose(fem.element_matrix_thermal(2.5), 2.5 * K, rtol=0, atol=1e-14)


def _exact_G():
    """G_pq(a,b) = int dN_a/dx_p dN_b/dx_q over the unit cube from exact 1D
    integrals (independent of the Gauss-quadrature B^T C B code path)."""
    def i00(i, j):      # int N_i N_j
        return 1 / 3 if i == j else 1 / 6

    def i10(i, j):      # int N_i' N_j
        return (1 if i else -1) * 0.5

    def i11(i, j):      # int N_i' N_j'
        return (1 if i else -1) * (1 if j else -1)

    G = np.zeros((8, 8, 3, 3))
    for a in range(8):
        for b in range(8):
            ca, cb = fem.CORNERS[a], fem.CORNERS[b]
            for p in range(3):
                for q in range(3):
                    v = 1.0
                    for d in range(3):
                        if d == p and d == q:
                            v *= i11(ca[d], cb[d])
                        elif d == p:
                            v *= i10(ca[d], cb[d])
                        elif d == q:
                            v *= i10(cb[d], ca[d])
                        else:
                            v *= i00(ca[d], cb[d])
                    G[a, b, p, q] = v
    return G


@pytest.mark.parametrize("E,nu", [(1.0, 0.3), (2.0, 0.1), (0.7, 0.45), (1.0, -0.2)])
def test_elastic_element_matrix_vs_exact_bilinear_form(E, nu):
    """element_stiffness_elastic vs the isotropic bilinear form
    K[(a,p),(b,q)] = lam G_pq + mu (delta_pq tr G + G_qp), exact integrals."""
    lam, mu = fem.lame(E, nu)
    G = _exact_G()
    Kx = np.zeros((24, 24))
    for a in range(8):
        for b in range(8):
            for p in range(3):
                for q in range(3):
                    Kx[3 * a + p, 3 * b + q] = (lam * G[a, b, p, q]
                                                + mu * ((p == q) * np.trace(G[a, b]) + G[a, b, q, p]))
    K = fem.element_stiffness_elastic(E, nu)
    assert np.abs(K - Kx).max() < 1e-13 * max(1.0, np.abs(Kx).max())


def test_elastic_element_null_space_is_rigid_motions():
    K = fem.element_stiffness_elastic(1.0, 0.3)
    assert np.abs(K - K.T).max() < 1e-14
    ev = np.linalg.eigvalsh(K)
    assert ev.min() > -1e-12 and int(np.sum(ev > 1e-10)) == 18
    X = fem.CORNERS.astype(float)
    modes = []
    for d in range(3):                     # translations
        t = np.zeros((8, 3)); t[:, d] = 1
        modes.append(t.reshape(-1))
    for axis in np.eye(3):                 # infinitesimal rotations w x x
        modes.append(np.cross(axis, X).reshape(-1))
    for r in modes:
        assert np.abs(K @ r).max() < 1e-13


def test_base_tensor_and_affine_fields_reproduce_C0_golden():
    """C_0 closed form (golden) and x0^T K_e x0 = C_0, K_e x0 = f_e (App. F1)."""
    g = _gold("isotropic_c0.json")
    C = fem.base_elasticity(g["E"], g["nu"])
    assert abs(C[0, 0] - g["C11"]) < 1e-15 and abs(C[0, 1] - g["C12"]) < 1e-15
    assert abs(C[3, 3] - g["C44"]) < 1e-15 and abs(C[5, 5] - g["C44"]) < 1e-15
    ph = fem.Physics("elastic", g["E"], g["nu"])
    assert np.abs(ph.X0.T @ ph.Ke @ ph.X0 - C).max() < 1e-14
    assert np.abs(ph.Ke @ ph.X0 - ph.Fe).max() < 1e-14
    # B x0 is the constant unit strain at any point (rigid check of X0 itself)
    for xi in ([0.1, 0.7, 0.3], [0.9, 0.2, 0.5]):
        assert np.abs(fem.strain_displacement(np.array(xi)) @ ph.X0 - np.eye(6)).max() < 1e-14


def test_thermal_affine_fields():
    ph = fem.Physics("thermal", kappa=1.7)
    assert np.abs(ph.X0.T @ ph.Ke @ ph.X0 - 1.7 * np.eye(3)).max() < 1e-14
    assert np.abs(ph.Ke @ ph.X0 - ph.Fe).max() < 1e-14
    assert np.abs(ph.Ke @ np.ones(8)).max() < 1e-14


# ------------------------------------------------------------- global operator

def test_element_dofs_brute_force():
    n = 3
    d = fem.element_dofs(n, 1)
    e = 2 + n * (0 + n * 1)          # element (2, 0, 1)
    want = []
    for k in range(8):
        kx, ky, kz = fem.CORNERS[k]
        want.append(((2 + kx) % n) + n * (((0 + ky) % n) + n * ((1 + kz) % n)))
    assert list(d[e]) == want
    assert d[e][1] == 0 + n * (0 + n * 1)   # corner x+1 wraps to x = 0


@pytest.mark.parametrize("kind", ["elastic", "thermal"])
def test_assembled_equals_matrix_free_and_sampled(kind):
    """assemble_K (global sparse) == apply_K_ebe (Eq. 14 gather/scatter) ==
    apply_K_at_nodes (per-node loops over the 8 incident elements)."""
    ph = fem.Physics(kind)
    n = 5
    s = synth.random_density(n, 0.0, 1.0, seed=3)
    s[s < 0.3] = 0.0
    rng = np.random.default_rng(0)
    u = rng.standard_normal((n ** 3 * ph.dpn, ph.nrhs))
    K = fem.assemble_K(s, ph)
    y1 = K @ u
    y2 = fem.apply_K_ebe(s, ph, u)
    assert np.abs(y1 - y2).max() < 1e-12 * np.abs(y1).max()
    un = fem.to_node_layout(u, n, ph.dpn)
    nodes = [(0, 0, 0), (4, 4, 4), (2, 3, 1), (4, 0, 2)]
    y3 = fem.apply_K_at_nodes(s, ph, lambda x, y, z: un[z, y, x], nodes)
    yn = fem.to_node_layout(y1, n, ph.dpn)
    for t, (x, y, z) in enumerate(nodes):
        assert np.abs(y3[t] - yn[z, y, x]).max() < 1e-12
    # symmetric, and constants (translations) are in the null space on the torus
    assert abs((K - K.T)).max() < 1e-13
    for c in range(ph.dpn):
        t = np.zeros(n ** 3 * ph.dpn); t[c::ph.dpn] = 1
        assert np.abs(K @ t).max() < 1e-12


@pytest.mark.parametrize("kind", ["elastic", "thermal"])
def test_loads(kind):
    ph = fem.Physics(kind)
    n = 4
    # solid torus: uniform strain is in equilibrium -> f = 0
    assert np.abs(fem.assemble_f(synth.solid(n), ph)).max() < 1e-13
    # single voxel: f = f_e scattered to its 8 corners
    s = np.zeros((n, n, n), np.float32); s[1, 2, 3] = 1.0
    f = fem.assemble_f(s, ph)
    fn = fem.to_node_layout(f, n, ph.dpn)
    for k in range(8):
        kx, ky, kz = fem.CORNERS[k]
        got = fn[(1 + kz) % n, (2 + ky) % n, (3 + kx) % n]        # (M, dpn)
        want = ph.Fe[k * ph.dpn:(k + 1) * ph.dpn, :].T
        assert np.abs(got - want).max() < 1e-15
    assert np.abs(f).sum() - np.abs(ph.Fe).sum() < 1e-12
    # sampled evaluation agrees with assembly
    s = synth.random_occupancy(n, 0.5, seed=1)
    f = fem.to_node_layout(fem.assemble_f(s, ph), n, ph.dpn)
    nodes = [(0, 0, 0), (3, 1, 2)]
    fs = fem.loads_at_nodes(s, ph, nodes)
    for t, (x, y, z) in enumerate(nodes):
        assert np.abs(fs[t] - f[z, y, x]).max() < 1e-14


@pytest.mark.parametrize("kind", ["elastic", "thermal"])
def test_diagonal_at_nodes_matches_assembled(kind):
    """diagonal_at_nodes (per-node element loop) == diag of the assembled K."""
    ph = fem.Physics(kind)
    n = 5
    s = synth.random_density(n, 0.0, 1.0, seed=7)
    s[s < 0.4] = 0.0
    d = fem.to_node_layout(fem.assemble_K(s, ph).diagonal()[:, None], n, ph.dpn)   # (z, y, x, 1, dpn)
    nodes = [(0, 0, 0), (4, 1, 3), (2, 2, 2), (1, 4, 0)]
    got = fem.diagonal_at_nodes(s, ph, nodes)
    for t, (x, y, z) in enumerate(nodes):
        assert np.abs(got[t] - d[z, y, x, 0]).max() < 1e-13


def test_effective_tensor_solid_is_base_tensor():
    for kind in ("elastic", "thermal"):
        ph = fem.Physics(kind, E=1.3, nu=0.25, kappa=0.8)
        n = 4
        u = np.zeros((n ** 3 * ph.dpn, ph.nrhs))
        CH = fem.effective_tensor(synth.solid(n), ph, u)
        assert np.abs(CH - ph.C0).max() < 1e-14
        # constant translation of u leaves C^H unchanged (K_e null space)
        u[0::ph.dpn] += 0.37
        assert np.abs(fem.effective_tensor(synth.solid(n), ph, u) - ph.C0).max() < 1e-13
