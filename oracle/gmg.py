"""Oracle: Galerkin hierarchy, damped-Jacobi smoother and the GMG V-cycle
(Sec. 3.2 Alg. 1, Sec. 4.4 Alg. 2, Sec. 4.6), FP64.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

Readings:
  R1 smoother: the north star fixes damped Jacobi,
     u <- u + omega D^{-1} (f - K u)  (Sec. 4.6 Eq. 16 update with every node
     updated from the previous iterate), applied It times where Alg. 1 says
     GS(K, u, f; It).
  R2 inactive dofs (zero diagonal: every incident element void) are excluded
     from the active set (Sec. 4.1.1 "sparse voxels"): D^{-1} := 0 there.
  R3 coarsest level: It_L sweeps of the same smoother (Alg. 1 line 8).
  R4 transfer on the active set: App. E2 precomputes the stencil "for each
     active fine node i", so P has zero rows at inactive fine nodes (and
     R = P^T ignores them).  Active = nonzero diagonal (touches an active
     element; Sec. 4.1.2 conservative coarsening keeps parents active).
"""
from __future__ import annotations

import numpy as np
import scipy.sparse as sp

from . import fem, transfer

_P27 = np.array([[a, b, c] for c in range(3) for b in range(3) for a in range(3)], dtype=np.int64)


def default_levels(n: int, coarsest: int = 4) -> int:
    """Depth with coarsest resolution max(coarsest, smallest even divisor chain)."""
    L, m = 1, n
    while m % 2 == 0 and m // 2 >= coarsest:
        m //= 2
        L += 1
    return L


class Hierarchy:
    """Grid hierarchy {Omega_l} (Sec. 3.2 "Grid Hierarchy") with Galerkin
    coarse operators K^{l+1} = R K^l P, R = P^T (Sec. 3.2 "Operator
    Consistency"; Sec. 4.6 Eq. 17), written as the global triple product."""

    def __init__(self, s: np.ndarray, phys: fem.Physics, levels: int):
        n = s.shape[0]
        if n % (1 << (levels - 1)):
            raise ValueError("N_res must be divisible by 2^(L-1)")
        self.phys = phys
        self.s = s
        self.n = [n >> l for l in range(levels)]
        self.K = [fem.assemble_K(s, phys)]
        self.P = []
        self.active = []
        for l in range(levels - 1):
            act = self.K[l].diagonal() > 0                       # R4
            self.active.append(act)
            P = sp.diags(act.astype(np.float64)) @ transfer.prolongation(self.n[l], phys.dpn)
            P = P.tocsr()
            self.P.append(P)
            self.K.append((P.T @ self.K[l] @ P).tocsr())
        self.active.append(self.K[-1].diagonal() > 0)
        self.Dinv = []
        for K in self.K:
            D = K.diagonal()
            self.Dinv.append(np.where(D > 0, 1.0 / np.where(D > 0, D, 1.0), 0.0))
        self.f = fem.assemble_f(s, phys)

    @property
    def L(self):
        return len(self.K)


def jacobi(K, Dinv, u, f, omega: float, sweeps: int):
    """Reading R1: damped Jacobi, u <- u + omega D^{-1} (f - K u), `sweeps` times."""
    u = u.copy()
    for _ in range(sweeps):
        u = u + omega * Dinv[:, None] * (f - K @ u)
    return u


def vcycle(H: Hierarchy, u1, f1=None, omega: float = 0.6, pre: int = 2, post: int = 2,
           coarse: int = 2, inject=None):
    """Alg. 1 (Standard GMG V-Cycle) / Alg. 2 (GMT V-cycle with injected
    coarse corrections e_hat^l).  ``inject`` maps level index (0-based,
    l >= 1) to the injected initial coarse error; missing levels start at 0
    (Alg. 1 line 6)."""
    L = H.L
    u = [None] * L
    f = [None] * L
    u[0] = np.array(u1, dtype=np.float64, copy=True)
    f[0] = H.f if f1 is None else f1
    for l in range(L - 1):
        u[l] = jacobi(H.K[l], H.Dinv[l], u[l], f[l], omega, pre)        # pre-smoothing
        r = f[l] - H.K[l] @ u[l]                                        # residual update
        f[l + 1] = H.P[l].T @ r                                         # f^{l+1} = R r^l
        if inject is not None and (l + 1) in inject:
            u[l + 1] = np.array(inject[l + 1], dtype=np.float64, copy=True)
        else:
            u[l + 1] = np.zeros_like(f[l + 1])                          # u^{l+1} = 0
    u[L - 1] = jacobi(H.K[L - 1], H.Dinv[L - 1], u[L - 1], f[L - 1], omega, coarse)
    for l in range(L - 2, -1, -1):
        u[l] = u[l] + H.P[l] @ u[l + 1]                                  # prolongate, correct
        u[l] = jacobi(H.K[l], H.Dinv[l], u[l], f[l], omega, post)       # post-smoothing
    return u[0]


def solve(H: Hierarchy, u0=None, tol: float = 1e-5, max_cycles: int = 200, **kw):
    """Repeat V-cycles until the Sec. 5.2 relative residual of every load
    case is <= tol.  Returns (u, history) with history[k] = per-load-case
    relative residual after k cycles (history[0] = initial)."""
    u = np.zeros_like(H.f) if u0 is None else np.array(u0, dtype=np.float64, copy=True)
    hist = [fem.relative_residual(H.K[0], u, H.f)]
    for _ in range(max_cycles):
        if np.all(hist[-1] <= tol):
            break
        u = vcycle(H, u, **kw)
        hist.append(fem.relative_residual(H.K[0], u, H.f))
    return u, np.array(hist)


def project_zero_mean(u: np.ndarray, dpn: int, active: np.ndarray | None = None) -> np.ndarray:
    """Sec. 4.5 gauge "sum_i u_i^1 = 0": subtract, per load case and per
    component, the mean over active nodes."""
    nn = u.shape[0] // dpn
    v = u.reshape(nn, dpn, -1).copy()
    mask = np.ones(nn, bool) if active is None else active
    v[mask] -= v[mask].mean(axis=0, keepdims=True)
    return v.reshape(u.shape)


# ---------------------------------------------------------------------------
# Element-local Galerkin (Sec. 4.6 Eq. 17): K_c = R_loc K_patch P_loc
# ---------------------------------------------------------------------------

def local_prolongation(dpn: int) -> np.ndarray:
    """P_loc: the 27 fine patch nodes (positions {0,1,2}^3 in fine units of a
    coarse element, numbered a + 3 b + 9 c) interpolated from the 8 coarse
    corners with the App. E1 weights prod_d (1 - |p_d / 2 - o_d|).
    Shape (27 dpn, 8 dpn)."""
    Pn = np.zeros((27, 8))
    for p in range(27):
        for k in range(8):
            o = fem.CORNERS[k]
            Pn[p, k] = np.prod(1.0 - np.abs(_P27[p] / 2.0 - o))
    return np.kron(Pn, np.eye(dpn))


def coarse_element_matrices(Ke_fine: np.ndarray, n_fine: int, dpn: int) -> np.ndarray:
    """Sec. 4.6 Eq. 17: for every coarse element E, assemble K_patch from its
    2x2x2 fine children (element matrices Ke_fine[e], e numbered
    ex + N(ey + N ez)) on the 27-node patch and return P_loc^T K_patch P_loc.
    Output (n_c^3, 8 dpn, 8 dpn)."""
    nc = n_fine // 2
    Ploc = local_prolongation(dpn)
    nd = 8 * dpn
    out = np.zeros((nc ** 3, nd, nd))
    # patch dof index of child j's local dof (corner k, comp c)
    pidx = np.zeros((8, nd), dtype=np.int64)
    for j in range(8):
        for k in range(8):
            p = fem.CORNERS[j] + fem.CORNERS[k]
            pn = p[0] + 3 * p[1] + 9 * p[2]
            for c in range(dpn):
                pidx[j, k * dpn + c] = pn * dpn + c
    for Z in range(nc):
        for Y in range(nc):
            for X in range(nc):
                Kp = np.zeros((27 * dpn, 27 * dpn))
                for j in range(8):
                    cx, cy, cz = fem.CORNERS[j]
                    e = (2 * X + cx) + n_fine * ((2 * Y + cy) + n_fine * (2 * Z + cz))
                    Kp[np.ix_(pidx[j], pidx[j])] += Ke_fine[e]
                out[X + nc * (Y + nc * Z)] = Ploc.T @ Kp @ Ploc
    return out


def level1_element_matrices(s: np.ndarray, phys: fem.Physics) -> np.ndarray:
    """s_e K_e for every fine element (App. F3 Eq. C_e = scale * C_0)."""
    return s.reshape(-1)[:, None, None].astype(np.float64) * phys.Ke[None]


def assemble_from_elements(Kel: np.ndarray, n: int, dpn: int) -> sp.csr_matrix:
    """K = sum_E A_E^T K_E A_E for per-element matrices at resolution n."""
    dofs = fem.element_dofs(n, dpn)
    nd = 8 * dpn
    rows = np.repeat(dofs, nd, axis=1).reshape(-1)
    cols = np.tile(dofs, (1, nd)).reshape(-1)
    ndof = n ** 3 * dpn
    return sp.csr_matrix((Kel.reshape(-1), (rows, cols)), shape=(ndof, ndof))
