"""Build libgmt.so in-tree with nvcc for sm_100a (no JIT cache: the built .so
travels with the repo snapshot to the GPU box)."""
from __future__ import annotations

import os
import shutil
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
LIB = os.path.join(HERE, "libgmt.so")

SOURCES = ["gmt_api.cu", "gmt_fem.cpp"]
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ["-std=c++17", "-O3", "-lineinfo", "-Xcompiler", "-fPIC", "-shared",
         "-Xcompiler", "-fvisibility=hidden", "-Xptxas", "-warn-spills"]


def nvcc() -> str:
    for cand in (shutil.which("nvcc"), "/usr/local/cuda/bin/nvcc"):
        if cand and os.path.exists(cand):
            return cand
    raise RuntimeError("nvcc not found")


def sources():
    return [os.path.join(CSRC, s) for s in SOURCES]


def _deps():
    out = []
    for d in (CSRC, os.path.join(ROOT, "include")):
        for f in sorted(os.listdir(d)):
            if f.endswith((".cu", ".cuh", ".h", ".cpp", ".inc")):
                out.append(os.path.join(d, f))
    return out


def up_to_date() -> bool:
    if not os.path.exists(LIB):
        return False
    t = os.path.getmtime(LIB)
    return all(os.path.getmtime(f) <= t for f in _deps())


TABLES = os.path.join(CSRC, "gmt_tables.inc")


def gen_tables(verbose: bool = False):
    """Compile and run gen_tables.cpp (host) -> csrc/gmt_tables.inc."""
    exe = os.path.join(CSRC, ".gen_tables")
    cxx = shutil.which("g++") or shutil.which("c++")
    cmd = [cxx, "-O1", "-std=c++17", "-o", exe, os.path.join(CSRC, "gen_tables.cpp"),
           os.path.join(CSRC, "gmt_fem.cpp")]
    res = subprocess.run(cmd, capture_output=True, text=True)
    if res.returncode != 0:
        raise RuntimeError(f"gen_tables build failed:\n{res.stderr}")
    res = subprocess.run([exe, TABLES + ".tmp"], capture_output=True, text=True)
    if res.returncode != 0:
        raise RuntimeError("gen_tables failed")
    os.replace(TABLES + ".tmp", TABLES)
    os.remove(exe)


def build(force: bool = False, verbose: bool = False) -> str:
    if force or not os.path.exists(TABLES) or \
            os.path.getmtime(TABLES) < max(os.path.getmtime(os.path.join(CSRC, f))
                                           for f in ("gen_tables.cpp", "gmt_fem.cpp", "gmt_fem.h")):
        gen_tables(verbose)
    if not force and up_to_date():
        return LIB
    cmd = [nvcc(), *ARCH, *FLAGS, "-I", os.path.join(ROOT, "include"), "-o", LIB + ".tmp", *sources()]
    if verbose:
        print(" ".join(cmd), file=sys.stderr)
    res = subprocess.run(cmd, capture_output=True, text=True)
    if res.returncode != 0:
        raise RuntimeError(f"nvcc failed ({res.returncode}):\n{res.stderr}")
    if "spill" in res.stderr and "0 bytes spill" not in res.stderr:
        print(res.stderr, file=sys.stderr)
    os.replace(LIB + ".tmp", LIB)
    return LIB


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose=True))
