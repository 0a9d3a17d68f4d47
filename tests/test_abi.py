"""CPU tests of the C-ABI boundary: the sm_100a library builds in-tree, loads
without a GPU, exports every symbol include/wgpf.h declares, and refuses to
run without a CUDA device (no CPU fallback)."""
import ctypes
import os
import re
import subprocess

import pytest

from conftest import ROOT, have_gpu


def declared_symbols():
    hdr = open(os.path.join(ROOT, "include", "wgpf.h")).read()
    hdr = re.sub(r"/\*.*?\*/", "", hdr, flags=re.S)
    return sorted(set(re.findall(r"\b(wgpf_[a-z_0-9]+)\s*\(", hdr)))


def test_library_builds_and_exports_every_declared_symbol():
    from paper_2505_21661_b200 import _build
    path = _build.build()
    lib = ctypes.CDLL(path)
    syms = declared_symbols()
    assert len(syms) >= 15
    missing = [s for s in syms if not hasattr(lib, s)]
    assert not missing, missing
    assert lib.wgpf_abi_version() == 1


def test_library_is_sm100a():
    from paper_2505_21661_b200 import _build
    out = subprocess.run(["cuobjdump", "--list-elf", _build.LIB],
                         capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_error_categories_match_reference_error_kinds():
    """error.hpp:29-51: status = 1 + ErrorKind."""
    from paper_2505_21661_b200 import _lib as L
    lib = L.lib()
    want = ["parse-error", "validate-error", "instrument-error", "lower-error",
            "capacity-error", "simulation-deadlock", "trace-error",
            "config-error", "io-error"]
    assert [lib.wgpf_error_category(i + 1).decode() for i in range(9)] == want


@pytest.mark.skipif(have_gpu(), reason="checks the no-GPU failure path")
def test_no_cpu_fallback_without_device():
    from paper_2505_21661_b200 import trace as T
    with pytest.raises(RuntimeError, match="no usable CUDA device"):
        T.Context(0)


def test_cxx_shim_compiles():
    """include/wgprof_b200.hpp (reference signatures over the C-ABI) compiles
    as C++20 against the header alone."""
    src = os.path.join(ROOT, "tests", "cxx", "shim_compile.cpp")
    out = os.path.join("/tmp", "wgpf_shim_compile.o")
    res = subprocess.run(["g++", "-std=c++20", "-c", "-I", os.path.join(ROOT, "include"),
                          src, "-o", out], capture_output=True, text=True)
    assert res.returncode == 0, res.stderr
