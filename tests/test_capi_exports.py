"""The C-ABI library loads and exports every symbol include/evr.h declares
(CPU only: no compute calls)."""

import ctypes
import os
import re
import subprocess

import pytest

from paper_1607_06283_b200 import _lib

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "evr.h")


def declared_functions():
    text = open(HEADER).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(evr_[a-z0-9_]+)\s*\(", text)))


def test_library_exists_and_loads():
    assert os.path.exists(_lib.LIB_PATH), "build libevr.so first (__graft_entry__.build())"
    _lib.load()


def test_every_header_symbol_is_exported_and_bound():
    lib = ctypes.CDLL(_lib.LIB_PATH)
    names = declared_functions()
    assert len(names) >= 35
    for name in names:
        assert hasattr(lib, name), f"{name} declared in evr.h but not exported"
    assert set(names) == set(_lib.exported_symbols()), "ctypes table out of sync with evr.h"


def test_library_is_sm100a_cuda():
    out = subprocess.run(["cuobjdump", "--list-elf", _lib.LIB_PATH], capture_output=True,
                         text=True).stdout
    assert "sm_100a" in out


def test_version_string_needs_no_device():
    assert b"sm_100a" in _lib.lib().evr_version()


def test_struct_layouts_match_header():
    assert ctypes.sizeof(_lib.Config) == 6 * 8 + 2 * 4 + 2 * 8 + 2 * 4 + 2 * 8
    assert ctypes.sizeof(_lib.SolveInfo) == 16
    assert _lib.EVENT_DTYPE.itemsize == 16
    assert _lib.EVENT_DTYPE.fields["t"][1] == 0 and _lib.EVENT_DTYPE.fields["x"][1] == 8


def test_context_refuses_without_gpu():
    if _lib.device_count() > 0:
        pytest.skip("a GPU is visible")
    with pytest.raises(RuntimeError, match="GPU only"):
        _lib.Context(4, 4)
