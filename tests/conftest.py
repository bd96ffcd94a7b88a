import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
# exercise the tiled coarse-level sweep on the small parity grids too
os.environ.setdefault("GMT_COARSE_TILED_MIN", "8")
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA GPU (B200) and the built libgmt")
    config.addinivalue_line("markers", "slow: CPU test taking more than ~20 s")
