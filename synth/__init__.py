"""Seeded synthetic voxel microstructures (input generators only).

This module is the ONE piece shared by the oracle tests and the CUDA path
("Input recipe").  It produces material fields -- a float32
array ``s[z, y, x]`` of per-voxel material scales in [0, 1] (0 = void,
1 = base material, intermediate values = SIMP-style density scale) -- and
nothing else.  It holds none of the method's arithmetic: no element
matrices, no operators, no solver steps.

Geometry families follow the paper's datasets (Sec. 5.1 "Training
Datasets", Appendix C "Geometric Profiles"): TPMS level sets, truss lattices
made of cylindrical struts, parametric shell lattices (approximated by thin
TPMS sheets), stochastic microstructures (periodic random fields), plus the
analytic two-phase laminates used as closed-form checks.  Volume fractions
default into the paper's training range v_f in [10%, 30%] (Appendix C,
"V_f is uniformly sampled within the range of [10%, 30%]").

All generators are periodic by construction: voxel centres are sampled at
(i + 1/2)/N of a unit cell and every level-set is 1-periodic.
"""
from __future__ import annotations

import numpy as np

__all__ = [
    "tpms", "truss", "shell_lattice", "stochastic", "laminate",
    "random_occupancy", "solid", "batch_truss_psl", "initial_guess",
    "volume_fraction",
]

_TWO_PI = 2.0 * np.pi


def _axes(n: int, dtype=np.float64):
    return (np.arange(n, dtype=dtype) + 0.5) / n


def _threshold_to_vf(phi: np.ndarray, vf: float, below: bool = True) -> np.ndarray:
    """Solid where phi < t (below) with t chosen so the solid count is
    round(vf * size) exactly (ties broken by index order, deterministic)."""
    flat = phi.reshape(-1)
    k = int(round(vf * flat.size))
    k = min(max(k, 1), flat.size)
    if not below:
        flat = -flat
    idx = np.argpartition(flat, k - 1)[:k]
    out = np.zeros(flat.size, dtype=np.float32)
    out[idx] = 1.0
    return out.reshape(phi.shape)


def _tpms_field(n: int, kind: str, dtype=np.float32) -> np.ndarray:
    t = _axes(n).astype(dtype)
    s = np.sin(_TWO_PI * t).astype(dtype)
    c = np.cos(_TWO_PI * t).astype(dtype)
    # arrays indexed [z, y, x]
    X = (slice(None),)
    sx, cx = s[None, None, :], c[None, None, :]
    sy, cy = s[None, :, None], c[None, :, None]
    sz, cz = s[:, None, None], c[:, None, None]
    del X
    if kind == "gyroid":
        phi = sx * cy + sy * cz
        phi = phi + sz * cx
    elif kind == "schwarz_p":
        phi = cx + cy
        phi = phi + cz
    elif kind == "diamond":
        phi = sx * sy * sz + sx * cy * cz
        phi = phi + cx * sy * cz
        phi = phi + cx * cy * sz
    else:
        raise ValueError(f"unknown TPMS kind {kind!r}")
    return np.ascontiguousarray(np.broadcast_to(phi, (n, n, n)), dtype=dtype)


def tpms(n: int, kind: str = "gyroid", vf: float = 0.3, sheet: bool = False) -> np.ndarray:
    """TPMS lattice (Appendix C (a)): network (phi < t) or sheet (|phi| < t)
    solid, threshold set to hit the requested volume fraction exactly."""
    if n < 2:
        raise ValueError("N_res must be >= 2")
    phi = _tpms_field(n, kind)
    if sheet:
        phi = np.abs(phi)
    return _threshold_to_vf(phi, vf, below=True)


def _periodic_segment_distance(p: np.ndarray, a: np.ndarray, b: np.ndarray, cutoff: float | None = None) -> np.ndarray:
    """Distance from points p (..., 3) in [0,1]^3 to segment a-b on the unit
    torus (minimum over the 27 periodic images of the segment).  With a
    cutoff, images whose bounding box grown by the cutoff misses [0,1]^3 are
    skipped: every point is farther than the cutoff from them, so the answer
    to "distance <= cutoff" is unchanged (only distances above it may be
    overestimated)."""
    best = None
    ab = b - a
    L2 = float(ab @ ab)
    lo, hi = np.minimum(a, b), np.maximum(a, b)
    for ox in (-1, 0, 1):
        for oy in (-1, 0, 1):
            for oz in (-1, 0, 1):
                o = np.array([ox, oy, oz], dtype=p.dtype)
                if cutoff is not None and (np.any(hi + o + cutoff < 0.0) or np.any(lo + o - cutoff > 1.0)):
                    continue
                ap = p - (a + o)
                t = np.clip((ap @ ab) / L2, 0.0, 1.0)
                d = ap - t[..., None] * ab
                dist = np.sqrt(np.einsum("...i,...i->...", d, d))
                best = dist if best is None else np.minimum(best, dist)
    if best is None:
        best = np.full(p.shape[:-1], np.inf, dtype=p.dtype)
    return best


_TRUSS_EDGES = {
    # unit-cell strut lists (endpoints in [0,1]^3); periodic images complete them
    "cubic": [((0, 0, 0), (1, 0, 0)), ((0, 0, 0), (0, 1, 0)), ((0, 0, 0), (0, 0, 1))],
    "bcc": [((0, 0, 0), (1, 1, 1)), ((1, 0, 0), (0, 1, 1)),
            ((0, 1, 0), (1, 0, 1)), ((0, 0, 1), (1, 1, 0))],
    "octet": [((0, 0, 0), (.5, .5, 0)), ((.5, .5, 0), (1, 1, 0)), ((1, 0, 0), (.5, .5, 0)),
              ((.5, .5, 0), (0, 1, 0)), ((0, 0, 0), (.5, 0, .5)), ((.5, 0, .5), (1, 0, 1)),
              ((1, 0, 0), (.5, 0, .5)), ((.5, 0, .5), (0, 0, 1)), ((0, 0, 0), (0, .5, .5)),
              ((0, .5, .5), (0, 1, 1)), ((0, 1, 0), (0, .5, .5)), ((0, .5, .5), (0, 0, 1)),
              ((.5, .5, 0), (.5, 0, .5)), ((.5, 0, .5), (0, .5, .5)), ((0, .5, .5), (.5, .5, 0))],
}


def truss(n: int, kind: str = "bcc", radius: float = 0.08, cells: int = 1,
          extra_struts=None) -> np.ndarray:
    """Truss lattice (Appendix C (b)): cylindrical struts of the given radius
    (unit-cell units) between lattice nodes, repeated ``cells`` times per axis.
    A voxel is solid when its centre lies within ``radius`` of a strut on the
    unit torus.  Each strut is cut into short pieces and every periodic image
    of a piece is tested only on the voxels of its bounding box grown by the
    radius (the union of the pieces' capsules is the strut's capsule)."""
    edges = list(_TRUSS_EDGES[kind]) if kind else []
    if extra_struts:
        edges += list(extra_struts)
    if cells > 1 and n % cells == 0:
        one = truss(n // cells, kind, radius, 1, extra_struts)
        return np.ascontiguousarray(np.tile(one, (cells, cells, cells)))
    if cells > 1:   # cell size not a whole number of voxels: evaluate everywhere
        out = np.zeros((n, n, n), dtype=np.float32)
        t = _axes(n) * cells % 1.0
        chunk = max(1, (1 << 21) // (n * n))
        for z0 in range(0, n, chunk):
            z1 = min(n, z0 + chunk)
            P = np.stack(np.meshgrid(t[z0:z1], t, t, indexing="ij"), axis=-1)[..., ::-1]
            d = None
            for a, b in edges:
                da = _periodic_segment_distance(P, np.asarray(a, float), np.asarray(b, float), cutoff=radius)
                d = da if d is None else np.minimum(d, da)
            out[z0:z1] = (d <= radius).astype(np.float32)
        return out
    solid = np.zeros((n, n, n), dtype=bool)            # [z, y, x]
    t = _axes(n)
    for a, b in edges:
        a, b = np.asarray(a, float), np.asarray(b, float)
        pieces = max(1, int(np.ceil(np.linalg.norm(b - a) / 0.125)))
        for k in range(pieces):
            pa = a + (b - a) * (k / pieces)
            pb = a + (b - a) * ((k + 1) / pieces)
            ab = pb - pa
            L2 = float(ab @ ab)
            lo, hi = np.minimum(pa, pb), np.maximum(pa, pb)
            for ox in (-1, 0, 1):
                for oy in (-1, 0, 1):
                    for oz in (-1, 0, 1):
                        o = np.array([ox, oy, oz], float)
                        blo, bhi = lo + o - radius, hi + o + radius
                        if np.any(bhi < 0.0) or np.any(blo > 1.0):
                            continue
                        # voxel index window (x, y, z) whose centres fall in the box
                        i0 = np.clip(np.floor(blo * n - 0.5).astype(int), 0, n - 1)
                        i1 = np.clip(np.ceil(bhi * n - 0.5).astype(int), 0, n - 1)
                        xs, ys, zs = (t[i0[d]:i1[d] + 1] for d in range(3))
                        P = np.stack(np.meshgrid(zs, ys, xs, indexing="ij"), axis=-1)[..., ::-1]
                        ap = P - (pa + o)
                        tt = np.clip((ap @ ab) / L2, 0.0, 1.0)
                        dv = ap - tt[..., None] * ab
                        near = np.einsum("...i,...i->...", dv, dv) <= radius * radius
                        solid[i0[2]:i1[2] + 1, i0[1]:i1[1] + 1, i0[0]:i1[0] + 1] |= near
    return solid.astype(np.float32)


def shell_lattice(n: int, kind: str = "gyroid", vf: float = 0.15) -> np.ndarray:
    """Stand-in for parametric shell lattices (Appendix C (c)): thin TPMS sheets."""
    return tpms(n, kind=kind, vf=vf, sheet=True)


def stochastic(n: int, vf: float = 0.3, seed: int = 0, corr: float = 0.08,
               sheet: bool = True) -> np.ndarray:
    """Stochastic microstructure (Appendix C (d), Sto-MS-like): a periodic
    Gaussian random field (white noise filtered by a Gaussian kernel in
    Fourier space, hence exactly periodic), thresholded into a band
    (|g| < t, a connected spinodal-like sheet) or a level set (g < t)."""
    rng = np.random.default_rng(seed)
    w = rng.standard_normal((n, n, n)).astype(np.float32)
    k = np.fft.fftfreq(n) * n  # integer wavenumbers
    kz, ky, kx = k[:, None, None], k[None, :, None], k[None, None, :]
    k2 = (kx * kx + ky * ky + kz * kz).astype(np.float32)
    filt = np.exp(-0.5 * (_TWO_PI * corr) ** 2 * k2).astype(np.float32)
    g = np.fft.irfftn(np.fft.rfftn(w) * filt[:, :, : n // 2 + 1], s=(n, n, n), axes=(0, 1, 2)).astype(np.float32)
    if sheet:
        g = np.abs(g)
    return _threshold_to_vf(g, vf, below=True)


def laminate(n: int, axis: int = 0, layers: int = 1, s_solid: float = 1.0,
             s_other: float = 0.0) -> np.ndarray:
    """Two-phase laminate: voxels whose coordinate along ``axis`` (0=x,1=y,2=z)
    is < ``layers`` get scale s_solid, the rest s_other."""
    if not 1 <= layers <= n - 1 and not (s_other > 0 and layers in (0, n)):
        raise ValueError("layers out of range")
    out = np.full((n, n, n), s_other, dtype=np.float32)
    sl = [slice(None)] * 3
    sl[2 - axis] = slice(0, layers)
    out[tuple(sl)] = s_solid
    return out


def random_occupancy(n: int, vf: float = 0.5, seed: int = 0) -> np.ndarray:
    rng = np.random.default_rng(seed)
    out = (rng.random((n, n, n)) < vf).astype(np.float32)
    if out.sum() == 0:
        out[0, 0, 0] = 1.0
    return out


def random_density(n: int, lo: float = 1e-3, hi: float = 1.0, seed: int = 0) -> np.ndarray:
    rng = np.random.default_rng(seed)
    return rng.uniform(lo, hi, (n, n, n)).astype(np.float32)


def solid(n: int, s: float = 1.0) -> np.ndarray:
    return np.full((n, n, n), s, dtype=np.float32)


def batch_truss_psl(n: int, count: int, seed: int = 0):
    """High-throughput screening batch (BASELINE configs[2]): a seeded mix of
    truss lattices (random kind / radius) and shell lattices (random TPMS
    kind / v_f), each a separate unit cell."""
    rng = np.random.default_rng(seed)
    kinds_t = ["cubic", "bcc", "octet"]
    kinds_s = ["gyroid", "schwarz_p", "diamond"]
    out = []
    for i in range(count):
        if i % 2 == 0:
            k = kinds_t[int(rng.integers(len(kinds_t)))]
            r = float(rng.uniform(0.05, 0.1)) if k != "octet" else float(rng.uniform(0.035, 0.06))
            out.append(truss(n, k, r))
        else:
            k = kinds_s[int(rng.integers(len(kinds_s)))]
            out.append(shell_lattice(n, k, float(rng.uniform(0.1, 0.3))))
    return out


def initial_guess(n: int, nrhs: int, dpn: int, seed: int = 0, amp: float = 0.1,
                  material: np.ndarray | None = None, z0: int = 0, nz: int | None = None) -> np.ndarray:
    """A smooth, seeded synthetic warm start u_hat^1 (Alg. 2 line 1 input),
    layout [m, c, z, y, x] float32 (component planes); zero on nodes whose 8
    surrounding voxels are all void when ``material`` (the full N^3 field) is
    given.  Stands in for the network prediction, which is out of scope.
    z0/nz select the planes [z0, z0+nz) of the same field (a rank's slab)."""
    nz = n - z0 if nz is None else nz
    rng = np.random.default_rng(seed)
    t = _axes(n)
    tz = t[z0:z0 + nz]
    out = np.zeros((nrhs, dpn, nz, n, n), dtype=np.float32)
    for m in range(nrhs):
        for c in range(dpn):
            a = rng.standard_normal(3)
            ph = rng.uniform(0, _TWO_PI, 3)
            fx = np.sin(_TWO_PI * t + ph[0]) * a[0]
            fy = np.sin(_TWO_PI * t + ph[1]) * a[1]
            fz = np.sin(_TWO_PI * tz + ph[2]) * a[2]
            out[m, c] = amp * (fz[:, None, None] + fy[None, :, None] + fx[None, None, :])
    if material is not None:
        # node (z, y, x) touches voxels z-1..z, y-1..y, x-1..x (periodic)
        occ = np.take(material > 0, np.arange(z0 - 1, z0 + nz) % n, axis=0)
        act = np.zeros((nz, n, n), dtype=bool)
        for dz in (0, 1):
            for dy in (0, 1):
                for dx in (0, 1):
                    act |= np.roll(occ, shift=(dy, dx), axis=(1, 2))[1 - dz:1 - dz + nz]
        out[:, :, ~act] = 0.0
    return out


def volume_fraction(s: np.ndarray) -> float:
    return float(np.mean(s))
