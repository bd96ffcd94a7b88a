"""CPU check of the Walsh-basis evaluation used by k_effective_tensor
(k_reduce.cuh): for random trilinear element fields, the kernel's slot layout
(corner Walsh-Hadamard sums, chunk A = constant | s_z modes, chunk B = s_x |
s_y modes, bilinear modes collapsed to (lam + 4 mu)/144) must reproduce the
2x2x2 Gauss-rule energy  sum_g w_g (e_m - eps_g(u^m)) : C_0 : (e_n - eps_g(u^n))
(App. F1, K_e = sum_g w_g B_g^T C_0 B_g).  The Gauss side below is written from
the trilinear shape functions directly; the Walsh side transcribes the
kernel's index mapping, so a wrong slot, sign or weight there fails here.
Pure numpy, fp64; no GPU and no oracle code involved."""
import itertools

import numpy as np

G = [(1 - 1 / np.sqrt(3)) / 2, (1 + 1 / np.sqrt(3)) / 2]
CORNERS = [(k & 1, (k >> 1) & 1, k >> 2) for k in range(8)]   # corner k = (x, y, z)


def grad_trilinear(v, p):
    """gradient of the trilinear interpolant of corner values v[8] at p in [0,1]^3"""
    g = np.zeros(3)
    for k, (cx, cy, cz) in enumerate(CORNERS):
        fx = (p[0] if cx else 1 - p[0], 1.0 if cx else -1.0)
        fy = (p[1] if cy else 1 - p[1], 1.0 if cy else -1.0)
        fz = (p[2] if cz else 1 - p[2], 1.0 if cz else -1.0)
        g[0] += v[k] * fx[1] * fy[0] * fz[0]
        g[1] += v[k] * fx[0] * fy[1] * fz[0]
        g[2] += v[k] * fx[0] * fy[0] * fz[1]
    return g


def c0_voigt(lam, mu):
    C = np.zeros((6, 6))
    C[:3, :3] = lam
    for i in range(3):
        C[i, i] += 2 * mu
    for i in range(3, 6):
        C[i, i] = mu
    return C


def gauss_energy(U, lam, mu):
    """Q_mn, U[m][c][8] corner values of displacement component c, case m"""
    nr = len(U)
    C = c0_voigt(lam, mu)
    Q = np.zeros((nr, nr))
    for p in itertools.product(G, G, G):
        E = []
        for m in range(nr):
            du = np.array([grad_trilinear(U[m][c], p) for c in range(3)])   # du[c][r]
            eps = np.array([du[0, 0], du[1, 1], du[2, 2], du[1, 2] + du[2, 1], du[0, 2] + du[2, 0],
                            du[0, 1] + du[1, 0]])
            e = np.zeros(6)
            e[m] = 1.0
            E.append(e - eps)
        for m in range(nr):
            for n in range(nr):
                Q[m, n] += 0.125 * E[m] @ C @ E[n]
    return Q


def wht(v):
    """the kernel's difference-first sums h_x, h_y, h_z, h_xy, h_xz, h_yz, h_xyz"""
    dx0, dx1, dx2, dx3 = v[1] - v[0], v[3] - v[2], v[5] - v[4], v[7] - v[6]
    a, b, c, d = dx0 + dx1, dx2 + dx3, dx1 - dx0, dx3 - dx2
    p = (v[2] - v[0]) + (v[3] - v[1])
    r = (v[6] - v[4]) + (v[7] - v[5])
    hz = ((v[4] - v[0]) + (v[5] - v[1])) + ((v[6] - v[2]) + (v[7] - v[3]))
    return [a + b, p + r, hz, c + d, b - a, r - p, d - c]


def walsh_energy(U, lam, mu):
    nr = len(U)
    H = []
    for m in range(nr):
        h = [wht(U[m][c]) for c in range(3)]
        S = [(1.0 if m == 0 else 0.0) - 0.25 * h[0][0],
             (1.0 if m == 1 else 0.0) - 0.25 * h[1][1],
             (1.0 if m == 2 else 0.0) - 0.25 * h[2][2],
             (1.0 if m == 3 else 0.0) - 0.25 * (h[1][2] + h[2][1]),
             (1.0 if m == 4 else 0.0) - 0.25 * (h[0][2] + h[2][0]),
             (1.0 if m == 5 else 0.0) - 0.25 * (h[0][1] + h[1][0])]
        for k in range(4):
            for c in range(3):
                S.append(h[c][3 + k])
        H.append(S)
    Q = np.zeros((nr, nr))
    # chunk A lanes: constant mode (weight 1) | s_z mode (1/48)
    A = [[(H[m][0], H[m][9]), (H[m][1], H[m][13]), (H[m][2], 0.0), (H[m][3], H[m][14]),
          (H[m][4], H[m][11]), (H[m][5], H[m][12] + H[m][10])] for m in range(nr)]
    # chunk B lanes: s_x mode | s_y mode (both 1/48)
    B = [[(H[m][7], H[m][6]), (H[m][11], H[m][14]), (H[m][10] + H[m][8], H[m][13]),
          (H[m][9], H[m][12] + H[m][8]), (H[m][6], H[m][7])] for m in range(nr)]
    for lane, wa, wb in ((0, 1.0, 1 / 48), (1, 1 / 48, 1 / 48)):
        for m in range(nr):
            ea = np.array([A[m][i][lane] for i in range(6)])
            tr = ea[:3].sum()
            sa = np.concatenate([wa * (2 * mu * ea[:3] + lam * tr), wa * mu * ea[3:]])
            eb = np.array([B[m][i][lane] for i in range(5)])
            trb = eb[0] + eb[1]
            sb = np.concatenate([wb * (2 * mu * eb[:2] + lam * trb), wb * mu * eb[2:]])
            for n in range(nr):
                Q[m, n] += sa @ np.array([A[n][i][lane] for i in range(6)])
                Q[m, n] += sb @ np.array([B[n][i][lane] for i in range(5)])
    wb = (lam + 4 * mu) / 144
    for m in range(nr):
        for n in range(nr):
            Q[m, n] += wb * sum(H[m][15 + c] * H[n][15 + c] for c in range(3))
    return Q


def test_walsh_form_matches_gauss_rule():
    rng = np.random.default_rng(3)
    lam, mu = 0.577, 0.385
    for _ in range(5):
        U = rng.standard_normal((6, 3, 8)) * rng.uniform(0.1, 3.0)
        np.testing.assert_allclose(walsh_energy(U, lam, mu), gauss_energy(U, lam, mu), rtol=1e-12, atol=1e-12)


def test_walsh_form_affine_field_is_exact():
    """u = the affine field of unit strain m leaves E = 0 for that case."""
    lam, mu = 1.0, 0.5
    U = np.zeros((6, 3, 8))
    for m in range(6):
        eps = np.zeros((3, 3))
        i, j = [(0, 0), (1, 1), (2, 2), (1, 2), (0, 2), (0, 1)][m]
        if i == j:
            eps[i, i] = 1.0
        else:
            eps[i, j] = eps[j, i] = 0.5
        for k, x in enumerate(CORNERS):
            U[m, :, k] = eps @ np.array(x, dtype=float)
    assert np.abs(walsh_energy(U, lam, mu)).max() < 1e-12
    assert np.abs(gauss_energy(U, lam, mu)).max() < 1e-12


def test_walsh_form_heat():
    """the DPN = 1 branch: weights 1 (constant), 2/48 (h_xy, h_xz, h_yz), 3/144 (h_xyz)"""
    rng = np.random.default_rng(5)
    kappa = 1.7
    for _ in range(5):
        U = rng.standard_normal((3, 8))
        Qg = np.zeros((3, 3))
        for p in itertools.product(G, G, G):
            E = [np.eye(3)[m] - grad_trilinear(U[m], p) for m in range(3)]
            for m in range(3):
                for n in range(3):
                    Qg[m, n] += 0.125 * kappa * E[m] @ E[n]
        Qw = np.zeros((3, 3))
        for m in range(3):
            hm = wht(U[m])
            Em = [(1.0 if m == r else 0.0) - 0.25 * hm[r] for r in range(3)]
            for n in range(3):
                hn = wht(U[n])
                En = [(1.0 if n == r else 0.0) - 0.25 * hn[r] for r in range(3)]
                a = sum(Em[r] * En[r] for r in range(3))
                a += (1 / 24) * sum(hm[3 + r] * hn[3 + r] for r in range(3))
                a += (1 / 48) * hm[6] * hn[6]
                Qw[m, n] = kappa * a
        np.testing.assert_allclose(Qw, Qg, rtol=1e-12, atol=1e-12)
