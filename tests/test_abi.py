"""The C-ABI library loads without a GPU and exports every symbol that
include/lbfs.h declares; the product never routes through the oracle."""

import re
import subprocess
from pathlib import Path

import pytest

from paper_1604_02844_b200 import _lib

ROOT = Path(__file__).resolve().parent.parent


def declared_symbols():
    text = (ROOT / "include" / "lbfs.h").read_text()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(lbfs_[a-z_0-9]+)\s*\(", text)))


def test_library_loads_and_exports_every_declared_symbol():
    lib = _lib.load()
    names = declared_symbols()
    assert len(names) >= 18
    for name in names:
        assert hasattr(lib, name), name
        assert name in _lib.SIGNATURES, name
    assert set(_lib.SIGNATURES) == set(names)


def test_exported_dynamic_symbols_match_header():
    out = subprocess.run(["nm", "-D", "--defined-only", str(_lib.LIB_PATH)], capture_output=True,
                         text=True, check=True).stdout
    exported = {l.split()[-1] for l in out.splitlines() if " T lbfs_" in l}
    assert exported == set(declared_symbols())


def test_library_carries_sm100a_code():
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", str(_lib.LIB_PATH)],
                         capture_output=True, text=True, check=True).stdout
    assert "sm_100a" in out


def test_last_error_is_callable_without_gpu():
    assert isinstance(_lib.last_error(), str)


def test_product_package_never_imports_the_oracle():
    for p in (ROOT / "paper_1604_02844_b200").rglob("*.py"):
        src = p.read_text()
        assert not re.search(r"^\s*(import|from)\s+oracle\b", src, flags=re.M), p


@pytest.mark.skipif(__import__("conftest").gpu_available(), reason="checks the no-GPU failure path")
def test_device_calls_fail_loudly_without_gpu():
    import numpy as np

    from paper_1604_02844_b200 import CsrGraph, bfs

    g = CsrGraph(3, np.array([1, 0, 2, 1], np.int32), np.array([0, 1, 3, 4], np.int64))
    with pytest.raises((RuntimeError, MemoryError)):
        bfs(g, 0)
