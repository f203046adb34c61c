"""CPU-side checks of the C-ABI boundary: libkk.so builds for sm_100a, loads,
and exports every entry point include/kk.h declares (no compute calls here)."""
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "kk.h")


def _declared():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(kk_[a-z_0-9]+)\s*\(", src)))


@pytest.fixture(scope="module")
def lib():
    from paper_1309_4349_b200 import build as B
    B.build()
    from paper_1309_4349_b200 import kk
    return kk.load()


def test_header_declares_entry_points():
    names = _declared()
    for must in ["kk_create", "kk_sweep", "kk_energy", "kk_composition", "kk_cluster_histogram"]:
        assert must in names          # north_star's named calls


def test_library_exports_every_declared_symbol(lib):
    for name in _declared():
        assert hasattr(lib, name), name


def test_binding_covers_header():
    from paper_1309_4349_b200 import kk
    assert set(_declared()) == set(kk.SIGNATURES)


def test_sm100a_code_and_no_oracle_linkage(lib):
    so = os.path.join(ROOT, "paper_1309_4349_b200", "libkk.so")
    out = subprocess.run(["cuobjdump", "--list-elf", so], capture_output=True, text=True).stdout
    assert "sm_100a" in out
    syms = subprocess.run(["nm", "-D", so], capture_output=True, text=True).stdout
    assert "kko_" not in syms          # the oracle is never linked into the product


def test_version_and_errors_without_gpu(lib):
    assert b"sm_100a" in lib.kk_version()
    from paper_1309_4349_b200 import kk
    with pytest.raises(kk.KKError):
        kk.Lattice(10, 8, 0.5, 0.5, 1)     # Lx % 4 != 0 -> argument error, before any CUDA call
