"""The C-ABI library builds for sm_100a, loads, and exports every symbol include/foe.h
declares (CPU only: no compute calls).  Without a GPU the product path must fail loudly."""
import ctypes as C
import os
import re
import subprocess

import numpy as np
import pytest

import paper_1404_5344_b200 as P
from paper_1404_5344_b200 import _lib

HDR = os.path.join(_lib.ROOT, "include", "foe.h")


def _declared():
    src = open(HDR).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    names = re.findall(r"^\s*(?:const\s+)?(?:(?:unsigned|long|short)\s+)*[A-Za-z_]\w*(?:\s+|\s*\*\s*)([a-z_][a-z0-9_]*)\s*\(",
                       src, flags=re.M)
    return sorted(set(n for n in names if n.startswith(("foe_", "ipiano_"))))


def test_header_declares_the_boundary_calls():
    d = _declared()
    for n in ("foe_model_create", "foe_energy_grad", "ipiano_step", "ipiano_run"):   # BASELINE north_star
        assert n in d


def test_library_exports_every_declared_symbol():
    L = P.lib()
    for n in _declared():
        assert hasattr(L, n), n
    assert sorted(P.EXPORTED) == _declared()


def test_library_is_sm100a_only():
    so = _lib.load()._name
    out = subprocess.run(["cuobjdump", "--list-elf", so], capture_output=True, text=True).stdout
    assert "sm_100a" in out
    assert not re.search(r"sm_(?!100a)\d+", out)


def test_no_cpu_fallback_without_gpu():
    import torch
    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    k = np.zeros((2, 7, 7), np.float32); k[:, 3, 3] = 1
    with pytest.raises(P.FoeError) as e:
        P.foe_model_create(k, [1.0, 1.0], looks=8)
    assert e.value.status == 2  # FOE_ERR_CUDA


def test_argument_validation_before_device_use():
    k = np.zeros((2, 4, 4), np.float32)
    with pytest.raises(P.FoeError) as e:
        P.foe_model_create(k, [1.0, 1.0], looks=8)
    assert e.value.status == 1 and "odd" in e.value.message
    k = np.zeros((2, 7, 7), np.float32)
    with pytest.raises(P.FoeError) as e:
        P.foe_model_create(k, [1.0, 0.0], looks=8)
    assert e.value.status == 1 and "filter 1" in e.value.message
    with pytest.raises(P.FoeError) as e:
        P.foe_model_create(k, [1.0, 1.0], looks=2)
    assert e.value.status == 1
    L = P.lib()
    assert L.foe_status_string(6) == b"FOE_ERR_PROX_NO_CONVERGENCE"
    assert b"sm_100a" in L.foe_version()
