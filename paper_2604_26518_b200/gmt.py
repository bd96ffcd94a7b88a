"""Thin ctypes binding over libgmt (include/gmt.h).  Argument marshalling only:
every step of the path runs in libgmt's CUDA kernels.  There is no CPU
fallback -- loading fails loudly when libgmt.so is missing.

Arrays: numpy arrays are passed as host buffers (GMT_HOST); torch CUDA
tensors as device buffers (GMT_DEVICE).  Nodal vectors are float32
component planes [m, c, z, y, x] (m = load case, c = component); material
fields float32 or uint8 [z, y, x].
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
# GMT_LIB selects an in-tree build variant for A/B timing (scripts/ab_lib.sh)
LIB_PATH = os.environ.get("GMT_LIB") or os.path.join(_HERE, "libgmt.so")

GMT_OK = 0
PHYSICS = {"elastic": 0, "thermal": 1}
GMT_F32, GMT_U8 = 0, 1
GMT_HOST, GMT_DEVICE = 0, 1


class GmtError(RuntimeError):
    pass


class gmt_config(C.Structure):
    _fields_ = [
        ("physics", C.c_int), ("res", C.c_int), ("levels", C.c_int),
        ("E", C.c_double), ("nu", C.c_double), ("kappa", C.c_double), ("omega", C.c_double),
        ("pre_sweeps", C.c_int), ("post_sweeps", C.c_int), ("coarse_sweeps", C.c_int),
        ("device", C.c_int), ("stream", C.c_void_p), ("use_graphs", C.c_int),
    ]


# name -> (restype, argtypes); mirrors include/gmt.h
_P = C.c_void_p
_FP = C.c_void_p
_DP = C.POINTER(C.c_double)
SIGNATURES = {
    "gmt_default_config": (C.c_int, [C.POINTER(gmt_config), C.c_int, C.c_int]),
    "gmt_create": (C.c_int, [C.POINTER(gmt_config), C.c_void_p, C.c_int, C.c_int, C.POINTER(C.c_void_p)]),
    "gmt_set_material": (C.c_int, [_P, C.c_void_p, C.c_int, C.c_int]),
    "gmt_set_initial_guess": (C.c_int, [_P, _FP, C.c_int]),
    "gmt_inject_correction": (C.c_int, [_P, C.c_int, _FP, C.c_int]),
    "gmt_vcycle": (C.c_int, [_P, C.c_int]),
    "gmt_residual_norms": (C.c_int, [_P, _DP, _DP, _DP]),
    "gmt_solve": (C.c_int, [_P, C.c_double, C.c_int, C.POINTER(C.c_int), _DP, _DP]),
    "gmt_homogenize": (C.c_int, [_P, _DP]),
    "gmt_get_solution": (C.c_int, [_P, _FP, C.c_int, C.c_int]),
    "gmt_num_levels": (C.c_int, [_P]),
    "gmt_level_res": (C.c_int, [_P, C.c_int]),
    "gmt_nrhs": (C.c_int, [_P]),
    "gmt_dpn": (C.c_int, [_P]),
    "gmt_stream": (C.c_void_p, [_P]),
    "gmt_device_bytes": (C.c_size_t, [_P]),
    "gmt_sync": (C.c_int, [_P]),
    "gmt_destroy": (None, [_P]),
    "gmt_last_error": (C.c_char_p, []),
    "gmt_abi_version": (C.c_int, []),
    "gmt_profile_enable": (C.c_int, [_P, C.c_uint]),
    "gmt_profile_collect": (C.c_int, [_P]),
    "gmt_profile_read": (C.c_int, [_P, C.c_int, _DP, C.POINTER(C.c_longlong), C.c_int]),
    "gmt_kernel_launches": (C.c_longlong, [_P]),
    "gmt_op_apply": (C.c_int, [_P, C.c_int, _FP, _FP]),
    "gmt_op_residual": (C.c_int, [_P, C.c_int, _FP, _FP, _FP]),
    "gmt_op_jacobi": (C.c_int, [_P, C.c_int, _FP, _FP, _FP]),
    "gmt_op_restrict": (C.c_int, [_P, C.c_int, _FP, _FP]),
    "gmt_op_prolong_add": (C.c_int, [_P, C.c_int, _FP, _FP]),
    "gmt_op_loads": (C.c_int, [_P, _FP]),
    "gmt_op_diagonal": (C.c_int, [_P, C.c_int, _FP]),
    "gmt_op_stencil": (C.c_int, [_P, C.c_int, _FP]),
    "gmt_op_effective_tensor": (C.c_int, [_P, _FP, _DP]),
    "gmt_slab_layout": (C.c_int, [C.c_int, C.c_int, C.c_int, C.c_int, C.POINTER(C.c_int)]),
    "gmt_halo_schedule": (C.c_int, [C.c_int, C.c_int, C.c_int, C.c_int, C.c_longlong, C.c_longlong, C.c_int, C.c_int,
                                    C.POINTER(C.c_int), C.POINTER(C.c_int), C.POINTER(C.c_longlong),
                                    C.POINTER(C.c_longlong), C.c_int]),
    "gmt_create_slabs": (C.c_int, [C.POINTER(gmt_config), C.c_void_p, C.c_int, C.c_int, C.c_int,
                                   C.POINTER(C.c_void_p)]),
    "gmt_nccl_unique_id": (C.c_int, [C.c_void_p, C.c_size_t]),
    "gmt_create_dist": (C.c_int, [C.POINTER(gmt_config), C.c_void_p, C.c_int, C.c_int, C.c_int, C.c_int,
                                  C.c_void_p, C.POINTER(C.c_void_p)]),
    "gmt_num_slabs": (C.c_int, [_P]),
    "gmt_set_refinement": (C.c_int, [_P, C.c_int]),
    "gmt_active_count": (C.c_longlong, [_P]),
    "gmt_set_level0_kernel": (C.c_int, [_P, C.c_int]),
    "gmt_batch_create": (C.c_int, [C.POINTER(C.c_void_p), C.c_int, C.POINTER(C.c_void_p)]),
    "gmt_batch_vcycle": (C.c_int, [_P, C.c_int]),
    "gmt_batch_homogenize": (C.c_int, [_P, _DP]),
    "gmt_batch_residual_norms": (C.c_int, [_P, _DP]),
    "gmt_batch_destroy": (None, [_P]),
    "gmt_active_nodes": (C.c_int, [_P, C.c_void_p, C.c_int]),
    "gmt_set_initial_guess_compact": (C.c_int, [_P, _FP, C.c_int]),
    "gmt_get_solution_compact": (C.c_int, [_P, _FP, C.c_int, C.c_int]),
    "gmt_refinement_active": (C.c_int, [_P]),
}

_lib = None


def load(path: str = LIB_PATH):
    """Load libgmt.so (raises GmtError if it is missing -- no fallback)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(path):
        raise GmtError(f"libgmt.so not built at {path}; run __graft_entry__.build()")
    lib = C.CDLL(path)
    for name, (res, args) in SIGNATURES.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    if lib.gmt_abi_version() != 1:
        raise GmtError("libgmt ABI mismatch")
    _lib = lib
    return lib


def _check(rc: int, what: str):
    if rc != GMT_OK:
        raise GmtError(f"{what} failed ({rc}): {_lib.gmt_last_error().decode()}")


def _buf(a, dtype=None, writable=False):
    """(pointer, location) of a numpy array (host) or torch CUDA tensor (device)."""
    if a is None:
        return None, GMT_HOST
    if isinstance(a, np.ndarray):
        if dtype is not None and a.dtype != dtype:
            raise TypeError(f"expected {dtype}, got {a.dtype}")
        if not a.flags.c_contiguous:
            raise ValueError("array must be C-contiguous")
        return a.ctypes.data, GMT_HOST
    try:
        import torch
    except ImportError:  # pragma: no cover
        torch = None
    if torch is not None and isinstance(a, torch.Tensor):
        if not a.is_cuda:
            raise ValueError("torch tensors must be CUDA tensors (use numpy for host buffers)")
        if not a.is_contiguous():
            raise ValueError("tensor must be contiguous")
        if dtype is not None and a.dtype != {np.float32: torch.float32, np.uint8: torch.uint8}[dtype]:
            raise TypeError(f"expected {dtype}, got {a.dtype}")
        return a.data_ptr(), GMT_DEVICE
    raise TypeError(f"unsupported buffer type {type(a)}")


def _dptr(a, size=None):
    p, loc = _buf(a, np.float32)
    if loc != GMT_DEVICE:
        raise ValueError("row-level ops take torch CUDA tensors")
    _check_size(a, size)
    return p


def _numel(a) -> int:
    return int(a.size) if isinstance(a, np.ndarray) else int(a.numel())


def _check_size(a, size):
    """libgmt reads/writes exactly `size` elements through the pointer: a
    smaller buffer would be overrun, so refuse it here."""
    if a is not None and size is not None and _numel(a) != size:
        raise ValueError(f"buffer holds {_numel(a)} elements, expected {size}")


def gmt_slab_layout(res: int, levels: int, nslabs: int, rank: int) -> dict:
    """Slab geometry (host only): z0, nz, Ld (partitioned levels), L."""
    lib = load()
    info = (C.c_int * 4)()
    _check(lib.gmt_slab_layout(res, levels, nslabs, rank, info), "gmt_slab_layout")
    return {"z0": info[0], "nz": info[1], "Ld": info[2], "L": info[3]}


def gmt_halo_schedule(nslabs: int, rank: int, nz: int, ncomp: int, cstride: int, plane: int, lo: int,
                      hi: int) -> list:
    """Ghost-plane exchange of one part (host only): [(peer, is_send, offset,
    count)] in issue order, offsets / counts in elements of the view."""
    lib = load()
    n = lib.gmt_halo_schedule(nslabs, rank, nz, ncomp, cstride, plane, lo, hi, None, None, None, None, 0)
    _check(n if n < 0 else 0, "gmt_halo_schedule")
    peer, snd = (C.c_int * max(n, 1))(), (C.c_int * max(n, 1))()
    off, cnt = (C.c_longlong * max(n, 1))(), (C.c_longlong * max(n, 1))()
    lib.gmt_halo_schedule(nslabs, rank, nz, ncomp, cstride, plane, lo, hi, peer, snd, off, cnt, n)
    return [(peer[i], bool(snd[i]), off[i], cnt[i]) for i in range(n)]


def gmt_nccl_unique_id() -> bytes:
    """128-byte NCCL unique id for gmt_create_dist (create on rank 0, broadcast)."""
    lib = load()
    buf = C.create_string_buffer(128)
    _check(lib.gmt_nccl_unique_id(buf, 128), "gmt_nccl_unique_id")
    return buf.raw


class Problem:
    """One periodic cell problem set (all load cases): gmt_create on one GPU,
    gmt_create_slabs (slabs=P: P z-slabs on one GPU with device-copy halos), or
    gmt_create_dist (dist=(rank, nranks, nccl_id): this rank's slab of an
    NCCL job; `material` then holds this rank's N/P planes)."""

    def __init__(self, material, physics: str = "elastic", levels: int = 0, E: float = 1.0,
                 nu: float = 0.3, kappa: float = 1.0, omega: float = 0.0, pre_sweeps: int = 2,
                 post_sweeps: int = 2, coarse_sweeps: int = 16, device: int = 0, stream=None,
                 use_graphs: bool = True, slabs: int = 1, dist=None):
        lib = load()
        n = int(material.shape[1])
        nz = int(material.shape[0])
        if tuple(material.shape[1:]) != (n, n) or (dist is None and nz != n):
            raise ValueError("material must be (N, N, N) (or (N/P, N, N) for dist)")
        cfg = gmt_config()
        _check(lib.gmt_default_config(C.byref(cfg), PHYSICS[physics], n), "gmt_default_config")
        cfg.levels, cfg.E, cfg.nu, cfg.kappa, cfg.omega = levels, E, nu, kappa, omega
        cfg.pre_sweeps, cfg.post_sweeps, cfg.coarse_sweeps = pre_sweeps, post_sweeps, coarse_sweeps
        cfg.device = device
        cfg.stream = stream
        cfg.use_graphs = int(use_graphs)
        ptr, loc, dt = self._material(material)
        h = C.c_void_p()
        if dist is not None:
            rank, nranks, nid = dist
            if nz * nranks != n:
                raise ValueError("dist material must hold N/nranks planes")
            idb = C.create_string_buffer(bytes(nid), 128)
            _check(lib.gmt_create_dist(C.byref(cfg), ptr, dt, loc, rank, nranks, idb, C.byref(h)),
                   "gmt_create_dist")
        elif slabs > 1:
            _check(lib.gmt_create_slabs(C.byref(cfg), ptr, dt, loc, slabs, C.byref(h)), "gmt_create_slabs")
        else:
            _check(lib.gmt_create(C.byref(cfg), ptr, dt, loc, C.byref(h)), "gmt_create")
        self._h = h
        self.nz = nz   # planes held at level 0 (N, or N/P for dist)
        self.lib = lib
        self.physics = physics
        self.n = n
        self.levels = lib.gmt_num_levels(h)
        self.nrhs = lib.gmt_nrhs(h)
        self.dpn = lib.gmt_dpn(h)

    @staticmethod
    def _material(material):
        dt = GMT_U8 if str(material.dtype) in ("uint8", "torch.uint8") else GMT_F32
        ptr, loc = _buf(material, np.uint8 if dt == GMT_U8 else np.float32)
        return ptr, loc, dt

    # -- lifecycle ---------------------------------------------------------
    def close(self):
        if getattr(self, "_h", None):
            self.lib.gmt_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *a):
        self.close()

    # -- shape helpers -----------------------------------------------------
    def level_res(self, level: int) -> int:
        return self.lib.gmt_level_res(self._h, level)

    def vec_shape(self, level: int = 0):
        n = self.level_res(level)
        if level == 0:
            return (self.nrhs, self.dpn, self.nz, n, n)
        return (self.nrhs, self.dpn, n, n, n)

    @property
    def num_slabs(self) -> int:
        return self.lib.gmt_num_slabs(self._h)

    @property
    def stream(self) -> int:
        return self.lib.gmt_stream(self._h)

    @property
    def device_bytes(self) -> int:
        return self.lib.gmt_device_bytes(self._h)

    # -- the boundary --------------------------------------------------------
    def _vsize(self, level: int = 0) -> int:
        return int(np.prod(self.vec_shape(level)))

    def gmt_set_material(self, material):
        if tuple(material.shape) != (self.nz, self.n, self.n):
            raise ValueError(f"material must be {(self.nz, self.n, self.n)}, got {tuple(material.shape)}")
        ptr, loc, dt = self._material(material)
        _check(self.lib.gmt_set_material(self._h, ptr, dt, loc), "gmt_set_material")

    def gmt_set_initial_guess(self, u=None):
        ptr, loc = _buf(u, np.float32)
        _check_size(u, self._vsize(0))
        _check(self.lib.gmt_set_initial_guess(self._h, ptr, loc), "gmt_set_initial_guess")

    def gmt_inject_correction(self, level: int, e=None):
        ptr, loc = _buf(e, np.float32)
        _check_size(e, self._vsize(level) if 0 < level < self.levels else None)
        _check(self.lib.gmt_inject_correction(self._h, level, ptr, loc), "gmt_inject_correction")

    def gmt_vcycle(self, ncycles: int = 1):
        _check(self.lib.gmt_vcycle(self._h, ncycles), "gmt_vcycle")

    def gmt_residual_norms(self):
        rel = (C.c_double * self.nrhs)()
        ar = (C.c_double * self.nrhs)()
        af = (C.c_double * self.nrhs)()
        _check(self.lib.gmt_residual_norms(self._h, rel, ar, af), "gmt_residual_norms")
        return np.array(rel), np.array(ar), np.array(af)

    def gmt_solve(self, rel_tol: float = 1e-5, max_cycles: int = 100):
        hist = (C.c_double * ((max_cycles + 1) * self.nrhs))()
        k = C.c_int()
        fr = C.c_double()
        _check(self.lib.gmt_solve(self._h, rel_tol, max_cycles, C.byref(k), C.byref(fr), hist), "gmt_solve")
        h = np.array(hist).reshape(max_cycles + 1, self.nrhs)[: k.value + 1]
        return k.value, fr.value, h

    def gmt_homogenize(self):
        CH = (C.c_double * (self.nrhs * self.nrhs))()
        _check(self.lib.gmt_homogenize(self._h, CH), "gmt_homogenize")
        return np.array(CH).reshape(self.nrhs, self.nrhs)

    def gmt_get_solution(self, out=None, zero_mean: bool = False):
        if out is None:
            out = np.empty(self.vec_shape(0), dtype=np.float32)
        ptr, loc = _buf(out, np.float32)
        _check_size(out, self._vsize(0))
        _check(self.lib.gmt_get_solution(self._h, ptr, loc, int(zero_mean)), "gmt_get_solution")
        return out

    # -- compact active-node I/O (Sec. 4.1.1) ---------------------------------
    def gmt_active_count(self) -> int:
        n = self.lib.gmt_active_count(self._h)
        if n < 0:
            _check(int(n), "gmt_active_count")
        return int(n)

    def compact_shape(self):
        return (self.nrhs, self.dpn, self.gmt_active_count())

    def gmt_active_nodes(self, out=None):
        if out is None:
            out = np.empty(self.gmt_active_count(), dtype=np.int32)
        if isinstance(out, np.ndarray):
            if out.dtype != np.int32 or not out.flags.c_contiguous:
                raise TypeError("active-node list must be a contiguous int32 array")
            ptr, loc = out.ctypes.data, GMT_HOST
        else:
            if not out.is_cuda or str(out.dtype) != "torch.int32" or not out.is_contiguous():
                raise TypeError("active-node list must be a contiguous int32 CUDA tensor")
            ptr, loc = out.data_ptr(), GMT_DEVICE
        _check_size(out, self.gmt_active_count())
        _check(self.lib.gmt_active_nodes(self._h, ptr, loc), "gmt_active_nodes")
        return out

    def gmt_set_initial_guess_compact(self, u):
        ptr, loc = _buf(u, np.float32)
        _check_size(u, int(np.prod(self.compact_shape())))
        _check(self.lib.gmt_set_initial_guess_compact(self._h, ptr, loc), "gmt_set_initial_guess_compact")

    def gmt_get_solution_compact(self, out=None, zero_mean: bool = False):
        if out is None:
            out = np.empty(self.compact_shape(), dtype=np.float32)
        ptr, loc = _buf(out, np.float32)
        _check_size(out, int(np.prod(self.compact_shape())))
        _check(self.lib.gmt_get_solution_compact(self._h, ptr, loc, int(zero_mean)), "gmt_get_solution_compact")
        return out

    def gmt_set_refinement(self, mode: int):
        """0 auto (default), 1 off, 2 on: mixed-precision iterative refinement."""
        _check(self.lib.gmt_set_refinement(self._h, int(mode)), "gmt_set_refinement")

    def gmt_set_level0_kernel(self, kind: int):
        """0: CUDA-core sum-factorised stencil (default), 1: tcgen05 element contractions."""
        _check(self.lib.gmt_set_level0_kernel(self._h, int(kind)), "gmt_set_level0_kernel")

    def gmt_refinement_active(self) -> bool:
        return bool(self.lib.gmt_refinement_active(self._h))

    def gmt_sync(self):
        _check(self.lib.gmt_sync(self._h), "gmt_sync")

    # -- live profiling ------------------------------------------------------
    PROFILE_CLASSES = ("l0_jacobi", "l0_residual", "l0_prolong", "restrict01", "coarse_levels",
                       "coarsest", "galerkin_setup", "effective_tensor")

    def gmt_profile_enable(self, mask: int):
        _check(self.lib.gmt_profile_enable(self._h, mask), "gmt_profile_enable")

    def gmt_profile_collect(self):
        _check(self.lib.gmt_profile_collect(self._h), "gmt_profile_collect")

    def gmt_profile_read(self, cls: int, reset: bool = False):
        ms = C.c_double()
        cnt = C.c_longlong()
        _check(self.lib.gmt_profile_read(self._h, cls, C.byref(ms), C.byref(cnt), int(reset)), "gmt_profile_read")
        return ms.value, cnt.value

    def gmt_kernel_launches(self) -> int:
        return self.lib.gmt_kernel_launches(self._h)

    # -- row-level entry points (torch CUDA tensors) -------------------------
    def gmt_op_apply(self, level, u, y):
        n = self._vsize(level)
        _check(self.lib.gmt_op_apply(self._h, level, _dptr(u, n), _dptr(y, n)), "gmt_op_apply")

    def gmt_op_residual(self, level, u, f, r):
        n = self._vsize(level)
        fp = None if f is None else _dptr(f, n)
        _check(self.lib.gmt_op_residual(self._h, level, _dptr(u, n), fp, _dptr(r, n)), "gmt_op_residual")

    def gmt_op_jacobi(self, level, u, f, u_out):
        n = self._vsize(level)
        fp = None if f is None else _dptr(f, n)
        _check(self.lib.gmt_op_jacobi(self._h, level, _dptr(u, n), fp, _dptr(u_out, n)), "gmt_op_jacobi")

    def gmt_op_restrict(self, level, r, fc):
        _check(self.lib.gmt_op_restrict(self._h, level, _dptr(r, self._vsize(level)), _dptr(fc, self._vsize(level + 1))),
               "gmt_op_restrict")

    def gmt_op_prolong_add(self, level, e, u):
        _check(self.lib.gmt_op_prolong_add(self._h, level, _dptr(e, self._vsize(level + 1)), _dptr(u, self._vsize(level))),
               "gmt_op_prolong_add")

    def gmt_op_loads(self, f):
        _check(self.lib.gmt_op_loads(self._h, _dptr(f, self._vsize(0))), "gmt_op_loads")

    def gmt_op_diagonal(self, level, d):
        _check(self.lib.gmt_op_diagonal(self._h, level, _dptr(d, self._vsize(level) // self.nrhs)), "gmt_op_diagonal")

    def gmt_op_stencil(self, level, S):
        _check(self.lib.gmt_op_stencil(self._h, level, _dptr(S, 27 * self.dpn * self._vsize(level) // self.nrhs)),
               "gmt_op_stencil")

    def gmt_op_effective_tensor(self, u):
        CH = (C.c_double * (self.nrhs * self.nrhs))()
        _check(self.lib.gmt_op_effective_tensor(self._h, _dptr(u, self._vsize(0)), CH), "gmt_op_effective_tensor")
        return np.array(CH).reshape(self.nrhs, self.nrhs)


class Batch:
    """A batch of independent problems on one GPU (gmt_batch_*): one CUDA-graph
    launch per V-cycle of all of them, C^H / residual norms with one
    synchronisation.  The problems must outlive the batch."""

    def __init__(self, problems):
        lib = load()
        self.lib = lib
        self.problems = list(problems)
        arr = (C.c_void_p * len(self.problems))(*[P._h.value for P in self.problems])
        h = C.c_void_p()
        _check(lib.gmt_batch_create(arr, len(self.problems), C.byref(h)), "gmt_batch_create")
        self._h = h

    def gmt_batch_vcycle(self, ncycles: int = 1):
        _check(self.lib.gmt_batch_vcycle(self._h, ncycles), "gmt_batch_vcycle")

    def gmt_batch_homogenize(self):
        nr = self.problems[0].nrhs
        out = (C.c_double * (len(self.problems) * nr * nr))()
        _check(self.lib.gmt_batch_homogenize(self._h, out), "gmt_batch_homogenize")
        return np.array(out).reshape(len(self.problems), nr, nr)

    def gmt_batch_residual_norms(self):
        nr = self.problems[0].nrhs
        out = (C.c_double * (len(self.problems) * nr))()
        _check(self.lib.gmt_batch_residual_norms(self._h, out), "gmt_batch_residual_norms")
        return np.array(out).reshape(len(self.problems), nr)

    def close(self):
        if getattr(self, "_h", None):
            self.lib.gmt_batch_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *a):
        self.close()

