"""The C-ABI library loads and exports every symbol include/pintgpu.h
declares (no compute calls: this runs without a GPU)."""

import ctypes
import os
import re
import subprocess

import pytest

from conftest import ROOT

HEADER = os.path.join(ROOT, "include", "pintgpu.h")


def declared():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(pg_[a-z_]+)\s*\(", src)))


def test_header_declares_the_boundary():
    names = declared()
    for must in ("pg_create", "pg_phi_batch", "pg_restrict", "pg_prolong_add",
                 "pg_c_residual", "pg_fas_rhs", "pg_last_error"):
        assert must in names


def test_library_exports_every_declared_symbol():
    from paper_1912_03106_b200 import build
    path = build.build()
    lib = ctypes.CDLL(path)
    for name in declared():
        assert hasattr(lib, name), name
    out = subprocess.run(["nm", "-D", "--defined-only", path], capture_output=True,
                         text=True).stdout
    exported = set(re.findall(r" T (pg_[a-z_]+)", out))
    assert set(declared()) <= exported


def test_python_binding_covers_the_header():
    from paper_1912_03106_b200 import _lib
    assert set(declared()) == set(_lib.EXPORTS)


def test_no_cpu_fallback_without_gpu():
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    from paper_1912_03106_b200 import GpuFemProblem, PintGpuError, configs
    with pytest.raises(PintGpuError):
        GpuFemProblem(configs.config1(N=8, n_steps=16))
    from paper_1912_03106_b200 import _lib
    lib = _lib.load()
    ctx = ctypes.c_void_p()
    assert lib.pg_create(ctypes.byref(ctx), 0) != 0
