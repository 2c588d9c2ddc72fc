"""CPU-side checks of the C-ABI library: it loads, and exports every symbol the
public header declares (no compute calls: there is no GPU here)."""
import ctypes
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HDR = os.path.join(ROOT, "include", "lgreco.h")


def _declared():
    txt = open(HDR).read()
    txt = re.sub(r"/\*.*?\*/", "", txt, flags=re.S)
    return sorted(set(re.findall(r"\b(lgreco_[a-z0-9_]+)\s*\(", txt)))


def test_header_declares_the_boundary():
    names = _declared()
    for required in ("lgreco_profile", "lgreco_solve", "lgreco_compress_allreduce", "lgreco_ctx_create",
                     "lgreco_ctx_destroy", "lgreco_last_error"):
        assert required in names


def test_library_exports_every_declared_symbol():
    from paper_2210_17357_b200 import lgreco
    lib = lgreco.lib()  # dlopen works without a GPU
    for name in _declared():
        assert hasattr(lib, name), f"{name} declared in lgreco.h but not exported"
    # the binding wraps exactly the declared entry points
    assert set(lgreco.EXPORTED) == set(_declared())
    assert lib.lgreco_version() == 1


def test_library_is_sm100a():
    so = os.path.join(ROOT, "paper_2210_17357_b200", "liblgreco.so")
    out = subprocess.run(["cuobjdump", "--list-elf", so], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_no_oracle_in_product_path():
    # the product package must not import or link the oracle (task rule ③)
    pkg = os.path.join(ROOT, "paper_2210_17357_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".h", ".cpp")):
                src = open(os.path.join(dirpath, f)).read()
                assert not re.search(r"(from|import)\s+oracle|liblgreco_ref|lgreco_ref", src), f
    nm = subprocess.run(["nm", "-D", os.path.join(pkg, "liblgreco.so")], capture_output=True, text=True).stdout
    assert "ref_" not in nm
