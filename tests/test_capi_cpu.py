"""CPU-side checks of the C ABI: the library builds, loads and exports every
symbol include/critprob_b200.h declares (no compute calls without a GPU)."""

import ctypes
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "critprob_b200.h")


def _declared():
    txt = open(HEADER).read()
    return sorted(set(re.findall(r"^\s*(?:int|double|const char\*)\s+(cpb_\w+)\s*\(", txt, re.M)))


@pytest.fixture(scope="module")
def lib():
    from paper_2407_18015_b200 import build

    path = build.build()
    return ctypes.CDLL(path)


def test_header_declares_entry_points():
    names = _declared()
    for must in ("cpb_fit", "cpb_classify_closed", "cpb_classify_mc", "cpb_materialize",
                 "cpb_unit_block", "cpb_run_host", "cpb_epsilon", "cpb_read_range"):
        assert must in names


def test_library_exports_every_declared_symbol(lib):
    missing = [n for n in _declared() if not hasattr(lib, n)]
    assert not missing


def test_binding_covers_header():
    from paper_2407_18015_b200 import _lib

    assert sorted(_lib.EXPORTED) == _declared()


def test_pure_host_helpers(lib):
    lib.cpb_abi_version.restype = ctypes.c_int
    assert lib.cpb_abi_version() == 1
    lib.cpb_epsilon.restype = ctypes.c_double
    lib.cpb_epsilon.argtypes = [ctypes.c_double, ctypes.c_double]
    # distributions.py:30-36
    assert lib.cpb_epsilon(0.0, 2.0) == max(1e-12, 1e-9 * 2.0)
    assert lib.cpb_epsilon(1.0, 1.0) == 1e-12
    out = (ctypes.c_size_t * 7)()
    lib.cpb_field_plane_bytes.argtypes = [ctypes.c_int32, ctypes.c_int32, ctypes.c_int32,
                                          ctypes.c_int64, ctypes.c_int64,
                                          ctypes.POINTER(ctypes.c_size_t)]
    assert lib.cpb_field_plane_bytes(2, 5, 64, 10, 20, out) == 0
    assert list(out) == [800, 800, 0, 0, 1000, 65 * 8, 12]
    assert lib.cpb_field_plane_bytes(1, 5, 64, 10, 20, out) == 0
    assert list(out)[:4] == [0, 0, 1600, 1600]
    assert lib.cpb_field_plane_bytes(7, 5, 64, 10, 20, out) == 1


def test_no_oracle_on_product_path():
    """The shipped package never imports the test oracle."""
    pkg = os.path.join(ROOT, "paper_2407_18015_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith(".py"):
                src = open(os.path.join(dirpath, f)).read()
                assert "oracle" not in re.findall(r"^\s*(?:from|import)\s+(\w+)", src, re.M), f
