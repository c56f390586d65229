"""The C-ABI library loads and exports every symbol include/*.h declares (no GPU needed)."""

import ctypes
import glob
import os
import re

import pytest

from paper_1308_5467_b200 import _native

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_symbols():
    names = set()
    for h in glob.glob(os.path.join(ROOT, "include", "*.h")):
        text = open(h).read()
        names.update(re.findall(r"SDB_API\s+[\w\s\*]+?\b(sdb_\w+)\s*\(", text))
    return names


def test_header_declares_symbols():
    names = declared_symbols()
    assert "sdb_cheb_moments" in names and "sdb_lanczos" in names and len(names) >= 20


def test_library_exports_every_declared_symbol():
    lib = _native.load()
    missing = [n for n in sorted(declared_symbols()) if not hasattr(lib, n)]
    assert not missing, missing


def test_binding_table_matches_header():
    assert set(_native.SIGNATURES) == declared_symbols()


def test_no_gpu_calls():
    lib = _native.load()
    assert lib.sdb_version() == 1
    assert lib.sdb_block_ldv(64) == 64
    assert lib.sdb_block_ldv(20) == 24
    assert lib.sdb_block_ldv(128) == 128
    assert lib.sdb_block_ldv(1) == 2
    assert lib.sdb_block_ldv(0) == -1
    assert lib.sdb_block_ldv(257) == -1
    for n in range(1, 257):
        assert lib.sdb_block_ldv(n) >= n


def test_invalid_arguments_map_to_value_error():
    lib = _native.load()
    out = ctypes.c_void_p()
    with pytest.raises(ValueError, match="positive"):
        _native.check(lib.sdb_matrix_create_csr(0, 0, 0, None, None, 32, None, None, ctypes.byref(out)))
    assert "dimension" in _native.last_error()


def test_library_is_sm100a():
    """The fatbin carries sm_100a SASS (cuobjdump lists the arch)."""
    import shutil
    import subprocess

    if shutil.which("cuobjdump") is None:
        pytest.skip("cuobjdump not available")
    out = subprocess.run(["cuobjdump", "--list-elf", _native.LIB_PATH], capture_output=True, text=True).stdout
    assert "sm_100a" in out
