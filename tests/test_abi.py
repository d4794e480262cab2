"""The C-ABI library loads and exports every symbol include/anovafs.h declares
(no compute calls: this runs without a GPU)."""

import ctypes
import os
import re

import pytest

from paper_2111_10140_b200 import _native

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(REPO, "include", "anovafs.h")


def declared_symbols():
    text = open(HEADER).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(afs_[a-z_]+)\s*\(", text)))


def test_header_declares_expected_entry_points():
    assert declared_symbols() == sorted(_native.SIGNATURES)


def test_library_exports_every_declared_symbol():
    if not os.path.exists(_native.LIB_PATH):
        pytest.skip("libanovafs.so not built")
    lib = ctypes.CDLL(_native.LIB_PATH)
    for name in declared_symbols():
        assert hasattr(lib, name), name
    lib.afs_abi_version.restype = ctypes.c_int
    assert lib.afs_abi_version() == 3


def test_struct_layouts_match_header():
    # afs_window_desc: 4 + 12 + 24 + 8 + 8 + 8 = 64 bytes; afs_plan_desc: 80 bytes
    assert ctypes.sizeof(_native.WindowDesc) == 64
    assert ctypes.sizeof(_native.PlanDesc) == 80
    assert ctypes.sizeof(_native.PlanInfo) == 40


def test_status_codes_map_to_reference_exceptions():
    lib = _native.load()
    from paper_2111_10140_b200 import NumericalError, ShapeError, ValidationError
    for code, exc in ((1, ShapeError), (2, ValidationError), (3, NumericalError)):
        with pytest.raises(exc):
            _native.check(code)
    _native.check(0)
    assert lib is not None


def test_plan_create_rejects_bad_descriptor_without_gpu():
    lib = _native.load()
    desc = _native.PlanDesc()
    desc.n_windows = 0
    h = ctypes.c_void_p()
    st = lib.afs_plan_create(ctypes.byref(desc), ctypes.byref(h))
    assert st == _native.AFS_ERR_VALIDATION
    assert b"window" in lib.afs_last_error()
