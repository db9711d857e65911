"""The C ABI library builds for sm_100a, loads, and exports every entry point that
include/cgks.h declares (no compute calls: runs without a GPU)."""
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _declared():
    src = open(os.path.join(ROOT, "include", "cgks.h")).read()
    return sorted(set(re.findall(r"\b(cgks_[a-z_]+)\s*\(", src)))


def test_header_declares_the_north_star_calls():
    d = _declared()
    for name in ["cgks_create", "cgks_set_state", "cgks_step", "cgks_get_state", "cgks_destroy"]:
        assert name in d


def test_library_exports_every_declared_symbol():
    from paper_2508_19911_b200 import build as b
    lib = b.build()
    out = subprocess.run(["nm", "-D", "--defined-only", lib], capture_output=True, text=True, check=True).stdout
    exported = set(re.findall(r"\bT (cgks_[a-z_]+)\b", out))
    missing = [s for s in _declared() if s not in exported]
    assert not missing, missing


def test_library_is_sm100a_code():
    from paper_2508_19911_b200 import build as b
    lib = b.build()
    out = subprocess.run(["cuobjdump", "--list-elf", lib], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_binding_loads_and_has_no_fallback():
    import paper_2508_19911_b200.binding as bd
    L = bd.load()
    for name in bd.EXPORTS:
        assert hasattr(L, name)
    with pytest.raises(ImportError):
        bd._lib, saved = None, bd._lib
        try:
            bd.load("/nonexistent/libcgks.so")
        finally:
            bd._lib = saved


def test_oracle_and_product_share_no_code():
    # the product package never imports the oracle; the oracle never includes product headers
    pkg = os.path.join(ROOT, "paper_2508_19911_b200")
    for dp, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".cpp", ".h")):
                txt = open(os.path.join(dp, f)).read()
                assert "import oracle" not in txt and "from oracle" not in txt and "cgks_oracle" not in txt, f
    osrc = open(os.path.join(ROOT, "oracle", "cgks_oracle.cpp")).read()
    assert "#include \"" not in osrc
