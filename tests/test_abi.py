"""CPU-side checks of the C-ABI boundary: libgmt.so builds/loads without a GPU
and exports every symbol include/gmt.h declares; the Python binding declares
exactly those symbols."""
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "gmt.h")


def header_symbols():
    txt = open(HEADER).read()
    return sorted(set(re.findall(r"^GMT_API\s+[\w\s\*]+?\b(gmt_\w+)\s*\(", txt, re.M)))


def test_header_declares_boundary():
    syms = header_symbols()
    for need in ("gmt_create", "gmt_vcycle", "gmt_solve", "gmt_homogenize", "gmt_destroy"):
        assert need in syms
    assert len(syms) >= 25


@pytest.fixture(scope="module")
def lib():
    from paper_2604_26518_b200 import build as b
    b.build()
    from paper_2604_26518_b200 import gmt
    return gmt.load()


def test_library_exports_every_header_symbol(lib):
    import ctypes
    missing = [s for s in header_symbols() if not hasattr(lib, s)]
    assert not missing, missing
    assert lib.gmt_abi_version() == 1


def test_binding_covers_header():
    from paper_2604_26518_b200 import gmt
    assert sorted(gmt.SIGNATURES) == header_symbols()


def test_default_config_and_errors_without_gpu(lib):
    import ctypes
    from paper_2604_26518_b200 import gmt
    cfg = gmt.gmt_config()
    assert lib.gmt_default_config(ctypes.byref(cfg), 0, 64) == 0
    assert (cfg.pre_sweeps, cfg.post_sweeps, abs(cfg.omega - 0.45) < 1e-12) == (2, 2, True)
    assert lib.gmt_default_config(ctypes.byref(cfg), 7, 64) == -1
    assert b"physics" in lib.gmt_last_error()
    assert lib.gmt_default_config(ctypes.byref(cfg), 1, 1) == -1


def test_product_never_imports_oracle():
    """The product and the oracle share no code and neither imports the other."""
    pkg = os.path.join(ROOT, "paper_2604_26518_b200")
    imp_oracle = re.compile(r"^\s*(from\s+oracle|import\s+oracle)", re.M)
    for dp, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".cpp", ".h")):
                txt = open(os.path.join(dp, f)).read()
                assert not imp_oracle.search(txt), f
                assert "oracle/" not in txt, f
    imp_prod = re.compile(r"^\s*(from\s+paper_2604_26518_b200|import\s+paper_2604_26518_b200)", re.M)
    for f in os.listdir(os.path.join(ROOT, "oracle")):
        if f.endswith(".py"):
            assert not imp_prod.search(open(os.path.join(ROOT, "oracle", f)).read()), f
