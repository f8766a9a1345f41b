"""Build and load libfoe.so (the sm_100a CUDA library behind include/foe.h).

The library is built in-tree (``paper_1404_5344_b200/libfoe.so``) with nvcc for
``-gencode arch=compute_100a,code=sm_100a`` only.  There is no CPU fallback: if the
library is missing or cannot be loaded, every call raises.
"""
from __future__ import annotations

import ctypes as C
import glob
import os
import shutil
import subprocess
import threading

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
INCLUDE = os.path.join(ROOT, "include")
SO = os.path.join(PKG, "libfoe.so")
ARCH = "-gencode=arch=compute_100a,code=sm_100a"

_lock = threading.Lock()
_lib = None


def sources():
    return sorted(glob.glob(os.path.join(CSRC, "*.cu")) + glob.glob(os.path.join(CSRC, "*.cuh"))
                  + [os.path.join(INCLUDE, "foe.h")])


def nvcc_path() -> str:
    for cand in (shutil.which("nvcc"), "/usr/local/cuda/bin/nvcc"):
        if cand and os.path.exists(cand):
            return cand
    raise RuntimeError("nvcc not found: cannot build libfoe.so")


def needs_build() -> bool:
    if not os.path.exists(SO):
        return True
    t = os.path.getmtime(SO)
    return any(os.path.getmtime(s) > t for s in sources())


def build(force: bool = False, verbose: bool = False) -> str:
    """Compile csrc/*.cu into libfoe.so for sm_100a (-O3 -lineinfo)."""
    if not force and not needs_build():
        return SO
    cus = sorted(glob.glob(os.path.join(CSRC, "*.cu")))
    tmp = SO + f".tmp{os.getpid()}"
    cmd = [nvcc_path(), ARCH, "-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "-shared",
           "-I" + INCLUDE, "-Xptxas", "-v" if verbose else "-O3", "-o", tmp] + cus
    res = subprocess.run(cmd, capture_output=True, text=True)
    if res.returncode != 0:
        raise RuntimeError("nvcc failed:\n" + " ".join(cmd) + "\n" + res.stdout + res.stderr)
    if verbose:
        print(res.stdout + res.stderr)
    os.replace(tmp, SO)
    return SO


def load():
    """Load libfoe.so (building it first if sources are newer).  Raises if unavailable."""
    global _lib
    with _lock:
        if _lib is None:
            if needs_build():
                build()
            _lib = C.CDLL(SO)
    return _lib
