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


def test_header_compiles_as_c_and_links(lib, tmp_path):
    """A plain C99 program includes the header, links
    libcritprob_b200.so and calls its host-only entry points."""
    import shutil
    import subprocess

    gcc = shutil.which("gcc")
    if gcc is None:
        pytest.skip("gcc not available")
    src = tmp_path / "abi.c"
    src.write_text(
        '#include <stdio.h>\n#include "critprob_b200.h"\n'
        "int main(void) {\n"
        "  cpb_case_batch b = {0};\n  cpb_field f = {0};\n  (void)b; (void)f;\n"
        '  printf("%d %.17g %.17g\\n", cpb_abi_version(), cpb_epsilon(0.0, 10.0), cpb_epsilon(2.0, 2.0));\n'
        "  return cpb_abi_version() == CPB_ABI_VERSION ? 0 : 1;\n}\n")
    libdir = os.path.join(ROOT, "paper_2407_18015_b200")
    exe = tmp_path / "abi"
    subprocess.run([gcc, "-std=c99", "-Wall", "-Werror", "-I", os.path.join(ROOT, "include"), str(src),
                    "-L", libdir, "-lcritprob_b200", "-Wl,-rpath," + libdir, "-o", str(exe)], check=True)
    out = subprocess.run([str(exe)], check=True, capture_output=True, text=True).stdout.split()
    assert out[0] == "1" and float(out[1]) == 1e-8 and float(out[2]) == 1e-12
