"""The C ABI library loads and exports every symbol include/emhd.h declares (no GPU needed)."""

import ctypes
import os
import re

from conftest import ROOT


def header_symbols():
    with open(os.path.join(ROOT, "include", "emhd.h")) as fh:
        txt = fh.read()
    return sorted(set(re.findall(r"\b(emhd_[a-z_0-9]+)\s*\(", txt)))


def test_library_builds_and_loads():
    from paper_1604_02614_b200 import _native as N
    assert os.path.exists(N.LIB_PATH), "run __graft_entry__.build() first"
    L = N.lib()
    assert L.emhd_version().decode().startswith("emhd-b200")
    assert L.emhd_error_string(3).decode().startswith("non-finite")


def test_every_declared_symbol_is_exported_and_bound():
    from paper_1604_02614_b200 import _native as N
    lib = ctypes.CDLL(N.LIB_PATH)
    syms = header_symbols()
    assert len(syms) >= 20
    for s in syms:
        assert hasattr(lib, s), f"{s} declared in emhd.h but not exported"
    bound = set(N.exported_symbols())
    assert set(syms) == bound, f"ctypes table out of sync: {set(syms) ^ bound}"


def test_no_cuda_means_loud_failure():
    import torch
    if torch.cuda.is_available():
        return
    import pytest
    from paper_1604_02614_b200 import make_rhs, Grid2D, MhdParams, BoundaryPolicy
    with pytest.raises(RuntimeError, match="no CPU fallback"):
        make_rhs(MhdParams(), Grid2D(8, 8, 0, 1, 0, 1), BoundaryPolicy())


def test_sass_is_sm100a():
    import shutil
    import subprocess
    from paper_1604_02614_b200 import _native as N
    tool = shutil.which("cuobjdump") or "/usr/local/cuda/bin/cuobjdump"
    if not os.path.exists(tool):
        return
    out = subprocess.run([tool, "--list-elf", N.LIB_PATH], capture_output=True, text=True).stdout
    assert "sm_100a" in out
