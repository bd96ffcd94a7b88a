"""Oracle: matrix-free geometric transfer operators written as explicit sparse
matrices (Appendix E "Matrix-Free Geometric Transfer Operators").

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).
"""
from __future__ import annotations

import numpy as np
import scipy.sparse as sp

_OFFS = np.array([[k & 1, (k >> 1) & 1, (k >> 2) & 1] for k in range(8)], dtype=np.int64)


def stencil(n_fine: int):
    """App. E1/E2: for every fine node x_f the stencil tuple (I, W):
    x_c = floor(x_f / 2); rho = x_f mod 2; xi = rho / 2;
    coarse neighbour k: (x_c + o_k) mod N_c; weight
    w_k = prod_d (1 - |xi_d - o_{k,d}|).
    Returns I (n_f^3, 8) coarse node numbers and W (n_f^3, 8) weights, fine
    nodes numbered x + N (y + N z)."""
    if n_fine % 2:
        raise ValueError("fine resolution must be even")
    nc = n_fine // 2
    z, y, x = np.meshgrid(np.arange(n_fine), np.arange(n_fine), np.arange(n_fine), indexing="ij")
    xf = np.stack([x.reshape(-1), y.reshape(-1), z.reshape(-1)], axis=1)
    xc = xf // 2
    xi = (xf % 2) / 2.0
    I = np.zeros((xf.shape[0], 8), dtype=np.int64)
    W = np.zeros((xf.shape[0], 8))
    for k in range(8):
        o = _OFFS[k]
        c = (xc + o) % nc
        I[:, k] = c[:, 0] + nc * (c[:, 1] + nc * c[:, 2])
        W[:, k] = np.prod(1.0 - np.abs(xi - o), axis=1)
    return I, W


def prolongation(n_fine: int, dpn: int) -> sp.csr_matrix:
    """App. E2 "Prolongation": u_f(i) = sum_k W_{i,k} u_c(I_{i,k}), as a sparse
    (n_f^3 dpn) x (n_c^3 dpn) matrix acting componentwise."""
    I, W = stencil(n_fine)
    nf, nc = n_fine ** 3, (n_fine // 2) ** 3
    rows = np.repeat(np.arange(nf), 8)
    cols = I.reshape(-1)
    vals = W.reshape(-1)
    keep = vals != 0
    Pn = sp.csr_matrix((vals[keep], (rows[keep], cols[keep])), shape=(nf, nc))
    return sp.kron(Pn, sp.identity(dpn), format="csr")


def restriction(n_fine: int, dpn: int) -> sp.csr_matrix:
    """App. E2 "Restriction ... strictly defined as the transpose of
    prolongation (R = P^T)"."""
    return prolongation(n_fine, dpn).T.tocsr()
