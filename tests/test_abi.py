"""CPU: the C-ABI library builds, loads and exports every symbol include/f2lin_gpu.h
declares; without a GPU every compute entry point fails loudly (no CPU fallback)."""
import os
import re

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_symbols():
    src = open(os.path.join(ROOT, "include", "f2lin_gpu.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(f2_[a-z0-9_]+)\s*\(", src)))


def test_header_declares_the_surface():
    syms = declared_symbols()
    for s in ["f2_mmpf_pls", "f2_pls_recursive", "f2_addmul", "f2_mul_m4rm", "f2_trsm_lower_left_unit",
              "f2_matrix_create", "f2_matrix_randomize", "f2_compress_columns", "f2_apply_rows"]:
        assert s in syms


def test_library_exports_every_declared_symbol():
    import ctypes
    import paper_1006_1744_b200 as f2
    L = f2.load_library()
    for s in declared_symbols():
        assert hasattr(L, s), s
        assert isinstance(getattr(L, s), ctypes._CFuncPtr)


def test_no_cpu_fallback_without_device():
    import paper_1006_1744_b200 as f2
    L = f2.load_library()
    if L.f2_device_count() > 0:
        pytest.skip("a GPU is visible")
    with pytest.raises(f2.NoDeviceError):
        f2.DeviceMatrix(4, 4)
    w = np.zeros((4, 1), np.uint64)
    with pytest.raises(f2.NoDeviceError):
        f2.mmpf_pls_host(w, 4)


def test_host_helpers_without_device():
    import paper_1006_1744_b200 as f2
    assert f2.auto_table_bits(4096) == 8
    assert f2.auto_table_bits(15) == 1
    assert f2.default_cutoff_bytes() > 0
    os.environ["F2_L2_BYTES"] = "12345"
    try:
        assert f2.default_cutoff_bytes() == 12345
    finally:
        del os.environ["F2_L2_BYTES"]


def test_argument_checks_before_device():
    """Checks the reference performs before any work (mmpf.cpp:85-90) are reported
    as ValueError/IndexError even without a device only where no device state is
    needed; with no device the library reports NoDeviceError first for creation."""
    import paper_1006_1744_b200 as f2
    with pytest.raises(ValueError):
        f2.set_panel_bits(100)
