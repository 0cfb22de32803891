"""The C-ABI library loads without a GPU and exports every symbol that
include/ebz200.h declares; the product refuses to run without a device
(no CPU fallback).  CPU only."""

import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_symbols():
    text = open(os.path.join(ROOT, "include", "ebz200.h")).read()
    return sorted(set(re.findall(r"\b(ebz_[a-z_0-9]+)\s*\(", text)))


def test_library_exports_every_declared_symbol():
    from paper_1706_03791_b200 import _native
    lib = _native.load_library()
    names = declared_symbols()
    assert len(names) >= 15
    for name in names:
        assert hasattr(lib, name), name
        assert name in _native.EXPORTS, f"{name} not bound in _native.EXPORTS"
    assert lib.ebz_abi_version() == 1


def test_library_built_for_sm100a():
    import subprocess
    so = os.path.join(ROOT, "paper_1706_03791_b200", "libebz200.so")
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", so],
                         capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_no_cpu_fallback_without_device():
    import torch
    if torch.cuda.is_available():
        pytest.skip("device present")
    from paper_1706_03791_b200 import _native, compress, CompressorConfig, DataGrid, \
        ErrorBoundSpec
    import numpy as np
    with pytest.raises(_native.NativeUnavailable):
        compress(DataGrid((4,), np.zeros(4)), CompressorConfig(ErrorBoundSpec(absolute=0.1)))
