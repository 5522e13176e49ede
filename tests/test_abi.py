"""The C-ABI library loads and exports every symbol include/cirr.h declares
(no compute calls: this runs on CPU-only hosts)."""
import ctypes
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIB = os.path.join(ROOT, "paper_2511_01927_b200", "libcirr.so")


def declared():
    text = open(os.path.join(ROOT, "include", "cirr.h")).read()
    return sorted(set(re.findall(r"^(?:int|long long|void)\s+(cirr_\w+)\s*\(", text, re.M)))


@pytest.fixture(scope="module")
def lib():
    if not os.path.exists(LIB):
        subprocess.run(["make", "-C", ROOT], check=True, capture_output=True)
    return ctypes.CDLL(LIB)


def test_header_declares_entries():
    names = declared()
    assert "cirr_zgetrf_batched" in names and "cirr_assemble" in names and len(names) >= 12


def test_every_declared_symbol_exported(lib):
    for name in declared():
        assert hasattr(lib, name), name


def test_binding_table_matches_header():
    from paper_2511_01927_b200 import _lib
    assert set(_lib.SIGNATURES) == set(declared())


def test_no_cpu_work_queries(lib):
    lib.cirr_target_sm.restype = ctypes.c_int
    assert lib.cirr_target_sm() == 100
    lib.cirr_small_eig_ws_bytes.restype = ctypes.c_longlong
    lib.cirr_small_eig_ws_bytes.argtypes = [ctypes.c_int]
    assert lib.cirr_small_eig_ws_bytes(256) > 4 * 256 * 256 * 16


def test_cubins_are_sm100a():
    out = subprocess.run(["cuobjdump", "--list-elf", LIB], capture_output=True, text=True)
    if out.returncode != 0:
        pytest.skip("cuobjdump unavailable")
    assert "sm_100a" in out.stdout


def test_dmma_in_sass():
    out = subprocess.run(["cuobjdump", "-sass", LIB], capture_output=True, text=True)
    if out.returncode != 0:
        pytest.skip("cuobjdump unavailable")
    assert "DMMA.8x8x4" in out.stdout
