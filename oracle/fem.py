"""Oracle: voxel finite elements, EBE operator, loads and effective tensors (FP64).

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

Conventions:
  * Voxel grid of N^3 unit-cube trilinear hexahedra on the periodic torus
    (Sec. 3.1 Eq. 2 "periodic boundary conditions"; App. F1 "The RVE
    is discretized into N_res^3 eight-node hexahedral elements").  Lengths are
    in voxel units, so |Omega| = N^3 element volumes.
  * Element-local corner k = kx + 2 ky + 4 kz, (kx,ky,kz) in {0,1}^3.
  * Global node n = x + N (y + N z); element e=(ex,ey,ez) has corner k at
    node ((ex+kx) mod N, (ey+ky) mod N, (ez+kz) mod N).
  * Global dof = n * dpn + c (dpn = 3 elasticity, 1 heat); load cases are
    the columns of a (ndof, M) array.
  * Voigt order (11, 22, 33, 23, 13, 12) with engineering shear strains,
    the order App. F1 lists the six unit strain modes in.
  * Material: a per-voxel scale s_e >= 0 multiplying the base tensor
    (binary occupancy s in {0,1}; App. F3 Eq. "C_e(rho_e) = (rho_min +
    rho_e^p) C_0" for densities).
"""
from __future__ import annotations

import numpy as np
import scipy.sparse as sp

CORNERS = np.array([[k & 1, (k >> 1) & 1, (k >> 2) & 1] for k in range(8)], dtype=np.int64)

# 2-point Gauss rule on [0, 1]
_GP = np.array([0.5 - 0.5 / np.sqrt(3.0), 0.5 + 0.5 / np.sqrt(3.0)])
_GW = np.array([0.5, 0.5])


def _shape_grad(xi: np.ndarray) -> np.ndarray:
    """dN_k/dx_d at local point xi in [0,1]^3 for the 8 trilinear shape
    functions N_k(x) = prod_d (x_d if k_d else 1 - x_d).  Returns (8, 3)."""
    g = np.zeros((8, 3))
    for k in range(8):
        f = [xi[d] if CORNERS[k, d] else 1.0 - xi[d] for d in range(3)]
        df = [1.0 if CORNERS[k, d] else -1.0 for d in range(3)]
        g[k, 0] = df[0] * f[1] * f[2]
        g[k, 1] = f[0] * df[1] * f[2]
        g[k, 2] = f[0] * f[1] * df[2]
    return g


def _gauss_points():
    for a in range(2):
        for b in range(2):
            for c in range(2):
                yield np.array([_GP[a], _GP[b], _GP[c]]), _GW[a] * _GW[b] * _GW[c]


def strain_displacement(xi: np.ndarray) -> np.ndarray:
    """App. F1 "epsilon(u)_e = B d_e": the 6x24 strain-displacement matrix B,
    Voigt (11,22,33,23,13,12), engineering shear."""
    g = _shape_grad(xi)
    B = np.zeros((6, 24))
    for k in range(8):
        dx, dy, dz = g[k]
        c = 3 * k
        B[0, c + 0] = dx
        B[1, c + 1] = dy
        B[2, c + 2] = dz
        B[3, c + 1] = dz; B[3, c + 2] = dy
        B[4, c + 0] = dz; B[4, c + 2] = dx
        B[5, c + 0] = dy; B[5, c + 1] = dx
    return B


def lame(E: float, nu: float):
    lam = E * nu / ((1.0 + nu) * (1.0 - 2.0 * nu))
    mu = E / (2.0 * (1.0 + nu))
    return lam, mu


def base_elasticity(E: float = 1.0, nu: float = 0.3) -> np.ndarray:
    """C_0 (Sec. 3.1 Example 1, "the base elasticity tensor"): isotropic,
    Voigt form, engineering shear strains."""
    if not (-1.0 < nu < 0.5) or E <= 0:
        raise ValueError("need E > 0 and -1 < nu < 0.5")
    lam, mu = lame(E, nu)
    C = np.zeros((6, 6))
    C[:3, :3] = lam
    for i in range(3):
        C[i, i] = lam + 2 * mu
        C[3 + i, 3 + i] = mu
    return C


def element_stiffness_elastic(E: float = 1.0, nu: float = 0.3) -> np.ndarray:
    """App. F1: K_e = int_{Omega_e} B^T C_0 B dOmega (24x24), 2x2x2 Gauss
    quadrature on the unit cube (exact for this integrand)."""
    C = base_elasticity(E, nu)
    K = np.zeros((24, 24))
    for xi, w in _gauss_points():
        B = strain_displacement(xi)
        K += w * B.T @ C @ B
    return K


def element_loads_elastic(E: float = 1.0, nu: float = 0.3) -> np.ndarray:
    """App. F1: f_e = int B^T C_0 eps_bar dOmega for the six unit strains
    eps_bar_11 .. eps_bar_12 (columns), shape (24, 6)."""
    C = base_elasticity(E, nu)
    F = np.zeros((24, 6))
    for xi, w in _gauss_points():
        F += w * strain_displacement(xi).T @ C @ np.eye(6)
    return F


def element_matrix_thermal(kappa: float = 1.0) -> np.ndarray:
    """App. F2: K_e^th = int B_th^T kappa_0 B_th dOmega (8x8), B_th = grad N."""
    if kappa <= 0:
        raise ValueError("kappa must be > 0")
    K = np.zeros((8, 8))
    for xi, w in _gauss_points():
        Bt = _shape_grad(xi).T  # (3, 8)
        K += w * kappa * Bt.T @ Bt
    return K


def element_loads_thermal(kappa: float = 1.0) -> np.ndarray:
    """App. F2: F_e^th = int B_th^T kappa_0 I_3 dOmega, shape (8, 3)."""
    F = np.zeros((8, 3))
    for xi, w in _gauss_points():
        F += w * kappa * _shape_grad(xi)
    return F


def affine_nodal_elastic() -> np.ndarray:
    """App. F1: x_0 = the element nodal displacement under the uniform unit
    strain (the affine field u(x) = eps_bar . x at the 8 local corners),
    shape (24, 6).  Engineering shear: eps_23 = gamma_23 / 2, so
    gamma_23 = 1 gives u = (0, z/2, y/2), etc."""
    X = np.zeros((24, 6))
    for k in range(8):
        x, y, z = CORNERS[k].astype(float)
        fields = [
            (x, 0, 0), (0, y, 0), (0, 0, z),
            (0, z / 2, y / 2), (z / 2, 0, x / 2), (y / 2, x / 2, 0),
        ]
        for m, u in enumerate(fields):
            X[3 * k: 3 * k + 3, m] = u
    return X


def affine_nodal_thermal() -> np.ndarray:
    """App. F2: T_0^(i)(x) = e_i . x at the 8 local corners, shape (8, 3)."""
    return CORNERS.astype(float).copy()


class Physics:
    """Element data for one physics (App. F1 elasticity / App. F2 heat)."""

    def __init__(self, kind: str, E: float = 1.0, nu: float = 0.3, kappa: float = 1.0):
        self.kind = kind
        if kind == "elastic":
            self.dpn, self.nrhs = 3, 6
            self.Ke = element_stiffness_elastic(E, nu)
            self.Fe = element_loads_elastic(E, nu)
            self.X0 = affine_nodal_elastic()
            self.C0 = base_elasticity(E, nu)
        elif kind == "thermal":
            self.dpn, self.nrhs = 1, 3
            self.Ke = element_matrix_thermal(kappa)
            self.Fe = element_loads_thermal(kappa)
            self.X0 = affine_nodal_thermal()
            self.C0 = kappa * np.eye(3)
        else:
            raise ValueError(kind)


def element_dofs(n: int, dpn: int) -> np.ndarray:
    """A_e as an index map: (n^3 elements, 8*dpn) global dof numbers of each
    element's local dofs (periodic incidence, Eq. 2)."""
    ez, ey, ex = np.meshgrid(np.arange(n), np.arange(n), np.arange(n), indexing="ij")
    ex, ey, ez = ex.reshape(-1), ey.reshape(-1), ez.reshape(-1)
    cols = []
    for k in range(8):
        kx, ky, kz = CORNERS[k]
        node = ((ex + kx) % n) + n * (((ey + ky) % n) + n * ((ez + kz) % n))
        for c in range(dpn):
            cols.append(node * dpn + c)
    return np.stack(cols, axis=1)


def assemble_K(s: np.ndarray, phys: Physics) -> sp.csr_matrix:
    """Sec. 4.6 Eq. 14: K = sum_e A_e^T (s_e K_e) A_e, assembled explicitly as
    a global sparse matrix (oracle only; the CUDA path never assembles K)."""
    n = s.shape[0]
    dofs = element_dofs(n, phys.dpn)
    se = s.reshape(-1).astype(np.float64)
    act = se != 0
    dofs, se = dofs[act], se[act]
    nd = 8 * phys.dpn
    rows = np.repeat(dofs, nd, axis=1).reshape(-1)
    cols = np.tile(dofs, (1, nd)).reshape(-1)
    vals = (se[:, None, None] * phys.Ke[None]).reshape(-1)
    ndof = n ** 3 * phys.dpn
    return sp.csr_matrix((vals, (rows, cols)), shape=(ndof, ndof))


def assemble_f(s: np.ndarray, phys: Physics) -> np.ndarray:
    """Eq. 3 right-hand side: f = sum_e A_e^T (s_e f_e), one column per
    load case (App. F1 six unit strains / App. F2 three unit gradients)."""
    n = s.shape[0]
    dofs = element_dofs(n, phys.dpn)
    se = s.reshape(-1).astype(np.float64)
    f = np.zeros((n ** 3 * phys.dpn, phys.nrhs))
    contrib = se[:, None, None] * phys.Fe[None]  # (ne, 8dpn, M)
    for j in range(dofs.shape[1]):
        np.add.at(f, dofs[:, j], contrib[:, j, :])
    return f


def apply_K_ebe(s: np.ndarray, phys: Physics, u: np.ndarray) -> np.ndarray:
    """Sec. 4.6 Eq. 14 verbatim: K u = sum_e A_e^T K_e A_e u_e, matrix-free
    (gather element dofs, multiply by s_e K_e, scatter-add)."""
    n = s.shape[0]
    dofs = element_dofs(n, phys.dpn)
    se = s.reshape(-1).astype(np.float64)
    ue = u[dofs]                                  # (ne, 8dpn, M)
    ye = np.einsum("ij,ejm->eim", phys.Ke, ue) * se[:, None, None]
    y = np.zeros_like(u, dtype=np.float64)
    for j in range(dofs.shape[1]):
        np.add.at(y, dofs[:, j], ye[:, j, :])
    return y


def apply_K_at_nodes(s: np.ndarray, phys: Physics, u_node, nodes) -> np.ndarray:
    """Sec. 4.6 Eq. 14 evaluated only at the requested nodes, by looping over
    the 8 elements around each node (for sampled checks at full size).
    ``u_node(x, y, z)`` returns the (M, dpn) nodal values; ``nodes`` is a list
    of (x, y, z).  Returns (len(nodes), M, dpn)."""
    n = s.shape[0]
    dpn = phys.dpn
    out = np.zeros((len(nodes), phys.nrhs, dpn))
    for t, (x, y, z) in enumerate(nodes):
        for k in range(8):  # node is corner k of element (x,y,z) - corner_k
            kx, ky, kz = CORNERS[k]
            ex, ey, ez = (x - kx) % n, (y - ky) % n, (z - kz) % n
            se = float(s[ez, ey, ex])
            if se == 0.0:
                continue
            ue = np.zeros((8 * dpn, phys.nrhs))
            for b in range(8):
                bx, by, bz = CORNERS[b]
                ue[b * dpn:(b + 1) * dpn, :] = np.asarray(
                    u_node((ex + bx) % n, (ey + by) % n, (ez + bz) % n), dtype=np.float64).T
            out[t] += se * (phys.Ke[k * dpn:(k + 1) * dpn, :] @ ue).T
    return out


def loads_at_nodes(s: np.ndarray, phys: Physics, nodes) -> np.ndarray:
    """Eq. 3 load vector evaluated only at the requested nodes; (len, M, dpn)."""
    n = s.shape[0]
    dpn = phys.dpn
    out = np.zeros((len(nodes), phys.nrhs, dpn))
    for t, (x, y, z) in enumerate(nodes):
        for k in range(8):
            kx, ky, kz = CORNERS[k]
            se = float(s[(z - kz) % n, (y - ky) % n, (x - kx) % n])
            out[t] += se * phys.Fe[k * dpn:(k + 1) * dpn, :].T
    return out


def diagonal_at_nodes(s: np.ndarray, phys: Physics, nodes) -> np.ndarray:
    """Sec. 4.6 Eq. 16 smoother diagonal D = diag(K) at the requested nodes:
    sum over the 8 incident elements of s_e K_e[(k,c),(k,c)]; (len, dpn)."""
    n = s.shape[0]
    dpn = phys.dpn
    out = np.zeros((len(nodes), dpn))
    dK = np.diag(phys.Ke)
    for t, (x, y, z) in enumerate(nodes):
        for k in range(8):
            kx, ky, kz = CORNERS[k]
            se = float(s[(z - kz) % n, (y - ky) % n, (x - kx) % n])
            out[t] += se * dK[k * dpn:(k + 1) * dpn]
    return out


def effective_tensor(s: np.ndarray, phys: Physics, u: np.ndarray) -> np.ndarray:
    """App. F1 / F2 "Effective Property Calculation":
        C^H_ij = 1/|Omega| sum_e (x_0^i - u_e^i)^T (s_e K_e) (x_0^j - u_e^j),
    |Omega| = N^3 voxel volumes.  u is (ndof, M)."""
    n = s.shape[0]
    dofs = element_dofs(n, phys.dpn)
    se = s.reshape(-1).astype(np.float64)
    act = se != 0
    d = phys.X0[None, :, :] - u[dofs[act]]              # (ne, 8dpn, M)
    Kd = np.einsum("ij,ejm->eim", phys.Ke, d)
    CH = np.einsum("eim,ein,e->mn", d, Kd, se[act])
    return CH / float(n ** 3)


def relative_residual(K, u: np.ndarray, f: np.ndarray) -> np.ndarray:
    """Sec. 5.2 "Relative Residual": r = ||f - K u||_2 / ||f||_2 per load case."""
    r = f - K @ u
    nf = np.linalg.norm(f, axis=0)
    nr = np.linalg.norm(r, axis=0)
    return np.where(nf > 0, nr / np.where(nf > 0, nf, 1.0), nr)


def to_node_layout(u: np.ndarray, n: int, dpn: int) -> np.ndarray:
    """(ndof, M) oracle layout -> [z, y, x, m, c] (the CUDA path's layout)."""
    M = u.shape[1]
    return u.reshape(n, n, n, dpn, M).transpose(0, 1, 2, 4, 3).copy()


def from_node_layout(a: np.ndarray) -> np.ndarray:
    """[z, y, x, m, c] -> (ndof, M)."""
    n, M, dpn = a.shape[0], a.shape[3], a.shape[4]
    return a.transpose(0, 1, 2, 4, 3).reshape(n ** 3 * dpn, M).astype(np.float64)


def effective_tensor_planes(s: np.ndarray, phys: Physics, u_plane, z0: int, z1: int) -> np.ndarray:
    """The App. F1 / F2 sum of ``effective_tensor`` restricted to the elements
    of voxel planes ez in [z0, z1), NOT divided by |Omega|:
        sum_{e: z0 <= ez < z1} (x_0^i - u_e^i)^T (s_e K_e) (x_0^j - u_e^j).
    Summing it over a partition of the planes and dividing by N^3 gives
    C^H; it exists so that fields too large for the (ndof, M) layout (512^3)
    can be evaluated one plane at a time.  ``u_plane(z)`` returns the nodal
    values of node plane z (periodic) as an array [y, x, m, c]."""
    n = s.shape[0]
    dpn, M = phys.dpn, phys.nrhs
    out = np.zeros((M, M))
    for ez in range(z0, z1):
        se = s[ez % n].astype(np.float64).reshape(-1)           # element (ex, ey) at ey * n + ex
        act = se != 0
        if not act.any():
            continue
        ue = np.zeros((n * n, 8 * dpn, M))
        planes = {kz: np.asarray(u_plane((ez + kz) % n), dtype=np.float64) for kz in (0, 1)}
        for k in range(8):
            kx, ky, kz = CORNERS[k]
            # corner k of element (ex, ey) is node ((ex + kx) mod n, (ey + ky) mod n)
            v = np.roll(planes[kz], shift=(-ky, -kx), axis=(0, 1)).reshape(n * n, M, dpn)
            ue[:, k * dpn:(k + 1) * dpn, :] = v.transpose(0, 2, 1)
        d = phys.X0[None, :, :] - ue[act]                       # (ne, 8dpn, M)
        Kd = np.matmul(phys.Ke[None], d)
        w = se[act][:, None, None]
        out += (d * w).reshape(-1, M).T @ Kd.reshape(-1, M)
    return out
