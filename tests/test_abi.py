"""CPU-side checks of the C ABI (-m "not gpu"): libpa builds for sm_100a, exports every symbol
include/pa.h declares, and the binding refuses to run without a device (no CPU fallback)."""
import ctypes
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_symbols():
    src = open(os.path.join(ROOT, "include", "pa.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(pa_[a-z_]+)\s*\(", src)) - {"pa_allreduce_fn"})


def test_library_builds_and_exports_every_declared_symbol():
    from paper_2604_09643_b200 import build

    lib_path = build.build()
    lib = ctypes.CDLL(lib_path)
    syms = declared_symbols()
    assert "pa_forward" in syms and "pa_step" in syms and len(syms) >= 10
    for s in syms:
        assert hasattr(lib, s), s
    from paper_2604_09643_b200 import _pa

    assert set(_pa.EXPORTS) == set(syms)
    assert lib.pa_version  # callable without a device
    lib.pa_version.restype = ctypes.c_char_p
    assert b"sm_100a" in lib.pa_version()


def test_sass_is_sm100a():
    import subprocess

    from paper_2604_09643_b200 import build

    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", build.build()], capture_output=True, text=True)
    assert "sm_100a" in out.stdout


def test_no_cpu_fallback():
    import torch

    if torch.cuda.is_available():
        pytest.skip("GPU present")
    from paper_2604_09643_b200 import Context

    with pytest.raises(RuntimeError):
        Context(0)
