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


def test_header_is_plain_c_and_links(tmp_path):
    """include/admm_b200.h is the drop-in boundary: it must compile as C (no
    C++ or torch types in the signatures) and a C program must link against
    the library through it.  The program only calls entry points that need no
    GPU."""
    import shutil
    import subprocess

    if shutil.which("gcc") is None:
        pytest.skip("no gcc")
    if not _lib.LIB_PATH.exists():
        pytest.fail("libadmm_b200.so is not built (run make)")
    src = tmp_path / "abi_probe.c"
    src.write_text(
        '#include <stdio.h>\n#include <string.h>\n#include "admm_b200.h"\n'
        "int main(void) {\n"
        "  if (admm_version() != 1) return 1;\n"
        "  /* argument validation happens before any CUDA call */\n"
        "  if (admm_project_batch(ADMM_F32, 4, 0, NULL, NULL, NULL) != ADMM_E_ARG) return 2;\n"
        '  if (strstr(admm_last_error(), "d >= 1") == NULL) return 3;\n'
        '  printf("abi ok\\n");\n  return 0;\n}\n')
    exe = tmp_path / "abi_probe"
    lib_dir = _lib.LIB_PATH.parent
    subprocess.run(["gcc", "-std=c99", "-Wall", "-Werror", "-I", str(HEADER.parent), str(src), "-o", str(exe),
                    "-L", str(lib_dir), f"-l:{_lib.LIB_PATH.name}", f"-Wl,-rpath,{lib_dir}"], check=True)
    out = subprocess.run([str(exe)], check=True, capture_output=True, text=True).stdout
    assert "abi ok" in out
