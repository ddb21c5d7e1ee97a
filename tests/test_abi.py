"""The C-ABI library loads and exports every symbol include/sfgpu.h declares;
without a GPU it refuses to run (no CPU fallback)."""
import os
import re

import pytest

from paper_2111_12238_b200 import abi

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def header_symbols():
    text = open(os.path.join(ROOT, "include", "sfgpu.h")).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(sfg_[a-z0-9_]+)\s*\(", text)))


def test_library_exports_every_declared_symbol():
    L = abi.load()
    syms = header_symbols()
    assert len(syms) >= 25
    for s in syms:
        assert hasattr(L, s), s
    assert sorted(abi.EXPORTS) == syms


def test_version():
    assert b"sm_100a" in abi.load().sfg_version()


def test_no_cpu_fallback():
    import paper_2111_12238_b200 as sf
    if abi.device_available():
        pytest.skip("a CUDA device is present")
    M = sf.config_matrix(1, size=4)
    with pytest.raises(sf.NoDeviceError):
        sf.make_state(4, M)


def test_invalid_arguments_rejected_before_device():
    import ctypes as C
    import numpy as np
    L = abi.load()
    h = C.c_void_p()
    cp = np.array([0, 1], np.int32)
    ri = np.array([0], np.int32)
    va = np.array([1.0])
    # combo ids outside 1..8 are rejected; nsys > 1 only for 1 and 8
    for bad in (0, 9):
        assert L.sfg_plan_create(bad, 1, abi.ptr(cp, abi.i32p), abi.ptr(ri, abi.i32p),
                                 abi.ptr(va, abi.f64p), 1, None, 7, C.byref(h)) == abi.SFG_ERR_INVALID_ARGUMENT
    assert L.sfg_plan_create(5, 1, abi.ptr(cp, abi.i32p), abi.ptr(ri, abi.i32p),
                             abi.ptr(va, abi.f64p), 2, None, 7, C.byref(h)) == abi.SFG_ERR_INVALID_ARGUMENT
