"""The C-ABI library loads and exports every symbol the public header
declares.  No compute calls (CPU only)."""
import re
from pathlib import Path

import pytest

from paper_1204_0556_b200 import _lib

HEADER = Path(__file__).resolve().parents[1] / "include" / "admm_b200.h"


def header_functions():
    text = HEADER.read_text()
    return sorted(set(re.findall(r"^\s*(?:const\s+)?\w+\s*\*?\s*(admm_\w+)\s*\(", text, re.M)))


def test_header_declares_expected_api():
    assert header_functions() == sorted(_lib.EXPORTED)


def test_library_exports_every_declared_symbol():
    if not _lib.LIB_PATH.exists():
        pytest.fail("libadmm_b200.so is not built (run make)")
    lib = _lib.load()
    for name in header_functions():
        assert hasattr(lib, name), name
    assert lib.admm_version() == 1


def test_error_reporting_without_gpu():
    lib = _lib.load()
    rc = lib.admm_project_batch(0, 4, 0, None, None, None)
    assert rc == -1
    assert b"d >= 1" in lib.admm_last_error()
    with pytest.raises(ValueError):
        _lib.check(rc)
