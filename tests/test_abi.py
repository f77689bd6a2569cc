"""CPU checks of the drop-in boundary: the product library loads without a
GPU and exports every entry point include/mswave_b200.h declares; the
oracle library is separate and the product does not link it."""
import ctypes
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "mswave_b200.h")
LIB = os.path.join(ROOT, "paper_1604_06750_b200", "libmswave_b200.so")


def declared_symbols():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(msw_[a-z_]+)\s*\(", src)))


def test_header_declares_the_reference_boundary():
    syms = declared_symbols()
    for s in ("msw_create", "msw_make_state", "msw_step", "msw_run", "msw_corner_correct",
              "msw_get_state", "msw_set_state", "msw_fine_leapfrog"):
        assert s in syms


def test_library_exports_every_declared_symbol():
    if not os.path.exists(LIB):
        pytest.fail("libmswave_b200.so not built (run __graft_entry__.build())")
    lib = ctypes.CDLL(LIB)
    for s in declared_symbols():
        assert hasattr(lib, s), s
    out = subprocess.run(["nm", "-D", "--defined-only", LIB], capture_output=True, text=True).stdout
    exported = set(re.findall(r"\bT (msw_\w+)", out))
    assert set(declared_symbols()) <= exported


def test_python_binding_covers_the_header():
    from paper_1604_06750_b200 import _ffi
    assert set(declared_symbols()) == set(_ffi.EXPORTED_SYMBOLS)


def test_product_does_not_link_the_oracle():
    out = subprocess.run(["ldd", LIB], capture_output=True, text=True).stdout
    assert "oracle" not in out
    out = subprocess.run(["nm", "-D", LIB], capture_output=True, text=True).stdout
    assert "oracle_" not in out


def test_kernels_are_sm100a():
    out = subprocess.run(["cuobjdump", "--list-elf", LIB], capture_output=True, text=True).stdout
    assert "sm_100a" in out
