"""CPU-side checks of the C ABI: the library loads and exports every symbol
include/dash_b200.h declares (no compute calls -- no GPU here)."""
import re
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]


def header_symbols():
    text = (ROOT / "include" / "dash_b200.h").read_text()
    return sorted(set(re.findall(r"^\s*(?:int|void)\s+\*?\s*(dash_\w+)\s*\(", text, re.M)))


def test_header_declares_the_update_entry_points():
    syms = header_symbols()
    for name in ("dash_update_f64", "dash_group_update_f64", "dash_ridge_solve_f64",
                 "dash_init_helpers_f64", "dash_local_error_f64", "dash_ctx_create"):
        assert name in syms


def test_library_exports_every_declared_symbol():
    from paper_2305_18376_b200 import _native
    from paper_2305_18376_b200.build import build_library
    build_library()
    lib = _native.load_library()
    for name in header_symbols():
        assert hasattr(lib, name), name
    assert set(header_symbols()) == set(_native.SIGNATURES)


def test_product_path_refuses_to_run_without_cuda():
    import torch
    from paper_2305_18376_b200 import _native
    if torch.cuda.is_available():
        pytest.skip("CUDA present")
    with pytest.raises(_native.NativeUnavailable):
        _native.lib()


def test_sm100a_cubin_in_library():
    import subprocess
    from paper_2305_18376_b200.build import build_library
    so = build_library()
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", str(so)],
                         capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_host_row_ptr_helper_on_cpu():
    """dash_host_row_ptr is host-only (no device): prefix sums and bad counts."""
    import ctypes
    import numpy as np
    from paper_2305_18376_b200 import _native
    from paper_2305_18376_b200.build import build_library
    build_library()
    lib = _native.load_library()
    counts = np.array([3, 0, 5, 1, 64, 65], dtype=np.int64)
    rp = np.full(counts.size + 1, -7, dtype=np.int64)
    n = ctypes.c_int64(0)
    assert lib.dash_host_row_ptr(counts.ctypes.data, counts.size, rp.ctypes.data, ctypes.byref(n)) == 0
    assert rp.tolist() == [0, 3, 3, 8, 9, 73, 138] and n.value == 138
    empty = np.zeros(1, dtype=np.int64)
    assert lib.dash_host_row_ptr(0, 0, empty.ctypes.data, ctypes.byref(n)) == 0 and n.value == 0
    bad = np.array([2, -1], dtype=np.int64)
    assert lib.dash_host_row_ptr(bad.ctypes.data, 2, rp.ctypes.data, ctypes.byref(n)) == _native.DASH_E_ARG
