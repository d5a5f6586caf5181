"""C-ABI library: builds for sm_100a, loads, and exports every symbol include/hps_b200.h declares."""
import ctypes
import os
import re
import subprocess

from paper_1612_02736_b200 import _ext, build_ext

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_symbols():
    text = open(os.path.join(ROOT, "include", "hps_b200.h")).read()
    return sorted(set(re.findall(r"^\s*(?:int|long long|const char\*)\s+(hps_\w+)\(", text, re.M)))


def test_header_matches_exports():
    decl = declared_symbols()
    assert decl == sorted(_ext.EXPORTS)


def test_library_loads_and_exports():
    path = build_ext.build()
    lib = ctypes.CDLL(path)
    for name in declared_symbols():
        assert hasattr(lib, name), name
    lib.hps_abi_version.restype = ctypes.c_int
    assert lib.hps_abi_version() == _ext.ABI_VERSION
    # workspace queries are host-only arithmetic
    lib.hps_leaf_workspace_bytes.restype = ctypes.c_longlong
    assert lib.hps_leaf_workspace_bytes(4, 16, 15) > 0


def test_sass_is_sm100a_and_uses_dmma():
    path = build_ext.build()
    out = subprocess.run(["cuobjdump", "-sass", path], capture_output=True, text=True).stdout
    assert "sm_100a" in out
    assert "DMMA.8x8x4" in out
