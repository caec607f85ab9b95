"""C-ABI boundary checks that need no GPU: the library loads, exports every
entry point include/rhg_b200.h declares, host-side parameter logic mirrors
the reference (geometry.hpp:14-73) bit for bit, and without a GPU the device
entry points fail loudly (no CPU fallback)."""
import ctypes as C
import os
import re
import subprocess

import pytest
import torch

import paper_1710_07565_b200 as rhg
from paper_1710_07565_b200 import _native

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "rhg_b200.h")


def declared_symbols():
    txt = open(HEADER).read()
    return sorted(set(re.findall(r"^\s*(?:int|void|const char\*)\s+(rhg_\w+)\s*\(", txt, re.M)))


def test_header_declares_expected_entry_points():
    syms = declared_symbols()
    assert set(_native.EXPORTS) == set(syms), syms


def test_library_exports_every_declared_symbol():
    lib = C.CDLL(_native.LIB_PATH)
    for s in declared_symbols():
        assert hasattr(lib, s), s
    out = subprocess.run(["nm", "-D", "--defined-only", _native.LIB_PATH], capture_output=True, text=True).stdout
    for s in declared_symbols():
        assert re.search(rf"\bT {s}$", out, re.M), s


def test_library_is_sm100a():
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", _native.LIB_PATH], capture_output=True,
                         text=True).stdout
    assert "sm_100a" in out, out


def test_abi_version():
    assert _native.lib().rhg_abi_version() == 6


def test_params_mirror_oracle(oracle):
    for g in (2.2, 2.6, 3.0, 7.5):
        assert rhg.alpha_from_gamma(g) == oracle.alpha_from_gamma(g)
    for d, a in [(16.0, 1.0), (64.0, 0.6), (256.0, 1.0), (4.0, 1.0), (16.0, 0.8), (3.3, 0.51)]:
        assert rhg.radial_const_from_avg_degree(d, a) == oracle.radial_const_from_avg_degree(d, a)
    p = rhg.ModelParams.from_avg_degree(1 << 20, 1.0, 16.0, 1, 8)
    L = oracle.layout(p.n, p.alpha, p.C, p.seed, p.chunks)
    assert p.R == L.R == rhg.radius_from_size(p.n, p.C)


@pytest.mark.parametrize("call,match", [
    (lambda: rhg.alpha_from_gamma(2.0), "gamma must be > 2"),
    (lambda: rhg.radial_const_from_avg_degree(4.0, 0.5), "alpha must be > 1/2"),
    (lambda: rhg.radial_const_from_avg_degree(-1.0, 1.0), "average degree must be positive"),
    (lambda: rhg.ModelParams(0, 1.0, 1.0, 1, 1), "n must be >= 1"),
    (lambda: rhg.ModelParams(10, 0.5, 1.0, 1, 1), "alpha must be > 1/2"),
    (lambda: rhg.ModelParams(2, 1.0, -5.0, 1, 1), "must be positive"),
    (lambda: rhg.ModelParams(10, 1.0, 1.0, 1, 0), "chunk count must be >= 1"),
])
def test_invalid_argument_mapping(call, match):
    with pytest.raises(ValueError, match=match):
        call()


@pytest.mark.skipif(torch.cuda.is_available(), reason="checks the no-GPU failure mode")
def test_no_gpu_fails_loudly():
    p = rhg.ModelParams.from_avg_degree(1000, 1.0, 8.0, 1, 2)
    with pytest.raises(rhg.RhgCudaError):
        rhg.generate_stats(p)


def test_multi_context_rejects_duplicates_and_needs_gpus():
    p = rhg.ModelParams.from_avg_degree(1000, 0.8, 8.0, 1, 4)
    with pytest.raises(ValueError, match="twice"):
        rhg.generate_stats(p, rhg.GenOptions(devices=(0, 0)))
    if not torch.cuda.is_available():
        with pytest.raises(rhg.RhgCudaError):
            rhg.generate_stats(p, rhg.GenOptions(devices=(0, 1)))
