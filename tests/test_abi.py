"""The C-ABI library loads without a GPU and exports every symbol that
include/hoi_b200.h declares (no compute calls here)."""

import re
import subprocess
from pathlib import Path

import pytest

from paper_2501_03381_b200 import _build, _native

HEADER = Path(__file__).resolve().parents[1] / "include" / "hoi_b200.h"


def declared():
    text = HEADER.read_text()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(hoi_\w+)\s*\(", text)))


@pytest.fixture(scope="module")
def lib():
    _build.build()
    return _native.load()


def test_header_and_binding_agree():
    assert declared() == sorted(_native.exported_symbols())


def test_library_exports_every_declared_symbol(lib):
    for name in declared():
        assert hasattr(lib, name), name
    out = subprocess.run(["nm", "-D", "--defined-only", str(_build.LIB)], capture_output=True,
                         text=True, check=True).stdout
    exported = set(re.findall(r"\bT (hoi_\w+)", out))
    assert set(declared()) <= exported


def test_host_only_entry_points(lib):
    assert lib.hoi_version() == 100
    assert lib.hoi_launch_count() >= 0
    # argument validation happens on the host and never touches the device
    assert lib.hoi_unrank(0, 1, 1, 0, 1, None, None, None) == _native.INVALID_ARG
    assert b"hoi_unrank" in lib.hoi_last_error()


def test_sm100a_code_object(lib):
    sass = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", str(_build.LIB)],
                          capture_output=True, text=True).stdout
    assert "sm_100a" in sass
