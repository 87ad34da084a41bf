"""CPU-side checks of the C ABI: the library loads, exports every symbol the
header declares, and validates arguments before touching a device."""

from __future__ import annotations

import ctypes
import os
import re

import pytest

from paper_2003_12726_b200 import _native

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "pxst_b200.h")


@pytest.fixture(scope="module")
def lib():
    if not os.path.exists(_native.LIB_PATH):
        from paper_2003_12726_b200 import build_native
        build_native.build()
    return _native.load_library()


def header_symbols():
    text = open(HEADER).read()
    return sorted(set(re.findall(r"^\s*(?:const\s+)?[a-z_0-9]+\*?\s+\*?(pxst_[a-z_0-9]+)\(", text,
                                 re.M)))


def test_header_symbols_exported(lib):
    syms = header_symbols()
    assert len(syms) >= 13, syms
    for s in syms:
        assert hasattr(lib, s), s
    assert set(syms) == set(_native.EXPORTED)


def test_abi_version(lib):
    assert lib.pxst_abi_version() == _native.ABI_VERSION


def test_null_arguments_rejected_without_device(lib):
    rc = lib.pxst_pixel_map_search(None, None, None, None, None, None, 3, 3, 0.0, 1, None, None,
                                   None, None, None)
    assert rc == _native.PXST_EINVAL
    assert b"NULL" in lib.pxst_last_error()
    rc = lib.pxst_translation_search(None, None, None, None, None, None, 1, 1, 0.0, 0, 0, None,
                                     None, None, None)
    assert rc == _native.PXST_EINVAL
    rc = lib.pxst_error_maps(None, None, None, None, None, None, None, None, None, None, None,
                             None)
    assert rc == _native.PXST_EINVAL
    rc = lib.pxst_object_splat(None, None, None, None, 0, 0, 1, 1, 0, 0, None, None, None)
    assert rc == _native.PXST_EINVAL
    rc = lib.pxst_object_finish(None, 1, None, None, None, None, None)
    assert rc == _native.PXST_EINVAL and b"accumulator" in lib.pxst_last_error()


def test_bad_window_rejected(lib):
    # a structurally valid descriptor with dummy (never dereferenced) pointers
    sc = _native.PxstScan(1, 2, 4, 4, 1, 1, 1, 1, 1, (ctypes.c_int64 * 4)(0, 4, 0, 4))
    st = _native.PxstStats(1, 1, 1, 1)
    ref = _native.PxstRef(1, 1, 8, 8, 0, 0)
    rc = lib.pxst_pixel_map_search(ctypes.byref(sc), ctypes.byref(st), ctypes.byref(ref), 1, 1, 1,
                                   -1, 2, 0.0, 1, None, None, 1, 1, None)
    assert rc == _native.PXST_EINVAL and b"halves" in lib.pxst_last_error()
    rc = lib.pxst_pixel_map_search(ctypes.byref(sc), ctypes.byref(st), ctypes.byref(ref), 1, 1, 1,
                                   2, 2, 1.5, 1, None, None, 1, 1, None)
    assert rc == _native.PXST_EINVAL and b"subpixel" in lib.pxst_last_error()
    bad_roi = _native.PxstScan(1, 2, 4, 4, 1, 1, 1, 1, 1, (ctypes.c_int64 * 4)(2, 2, 0, 4))
    rc = lib.pxst_bbox(ctypes.byref(bad_roi), 1, 1, 1, 1, None)
    assert rc == _native.PXST_EINVAL and b"ROI" in lib.pxst_last_error()


def test_check_maps_codes(lib):
    with pytest.raises(ValueError):
        _native.check(_native.PXST_EINVAL)
    with pytest.raises(RuntimeError):
        _native.check(_native.PXST_ECUDA)
