"""CPU-side checks of the C-ABI library: it is built for sm_100a, loads, and
exports every symbol include/romdot_b200.h declares. No compute (no GPU here)."""
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def so():
    from paper_1602_00138_b200 import build
    return build.build()


def header_symbols():
    txt = open(os.path.join(ROOT, "include", "romdot_b200.h")).read()
    return sorted(set(re.findall(r"\b(rd_[A-Za-z0-9_]+)\s*\(", txt)))


def test_header_declares_expected_surface():
    syms = header_symbols()
    for s in ["rd_ctx_create", "rd_op_apply", "rd_recycled_solve", "rd_basis_refresh", "rd_basis_append",
              "rd_process_system", "rd_rrqr", "rd_smallest_eigenpairs", "rd_initial_solutions"]:
        assert s in syms


def test_library_exports_every_header_symbol(so):
    out = subprocess.run(["nm", "-D", "--defined-only", so], capture_output=True, text=True).stdout
    exported = set(re.findall(r"\bT (rd_[A-Za-z0-9_]+)\b", out))
    missing = [s for s in header_symbols() if s not in exported]
    assert not missing, missing


def test_library_loads_and_python_mirror_binds(so):
    from paper_1602_00138_b200 import romdot
    L = romdot.load_library(so)
    for s in romdot.EXPORTS:
        assert hasattr(L, s)
    assert set(romdot.EXPORTS) == set(header_symbols())


def test_sm100a_cubin_embedded(so):
    out = subprocess.run(["cuobjdump", "--list-elf", so], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_product_never_imports_oracle():
    pkg = os.path.join(ROOT, "paper_1602_00138_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".h", ".cpp")):
                txt = open(os.path.join(dirpath, f)).read()
                assert "liboracle" not in txt and "import oracle" not in txt and "romdot_oracle" not in txt, f
