"""paper_2604_26518_b200 -- B200-native matrix-free voxel GMG hot path of GMT
(arXiv 2604.26518): libgmt (CUDA, sm_100a, C ABI in include/gmt.h) plus this
thin ctypes binding.  See DESIGN.md."""
from .gmt import Batch, GmtError, Problem, load  # noqa: F401

__all__ = ["Problem", "Batch", "GmtError", "load"]
