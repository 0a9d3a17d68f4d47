"""The reference CLI's decode / replay / export commands
(tools/wgprof.cpp:78-126), compiled UNCHANGED against the drop-in header
include/wgprof_b200.hpp (tests/cxx/cli_build.py), run on the GPU and compared
byte for byte with the same commands built against the reference headers
(tests/golden/cli/, tests/golden/gen_cli_golden.py) -- stdout for the
fixtures, stderr and exit status for inputs the reference rejects.  This is
the header-swap drop-in of INTEGRATION.md, end to end.
"""
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.join(ROOT, "tests", "cxx"))
sys.path.insert(0, os.path.join(ROOT, "tests", "golden"))

import cli_build  # noqa: E402
import gen_cli_golden as G  # noqa: E402

GOLD = os.path.join(ROOT, "tests", "golden", "cli")


def _cli():
    if not os.path.exists(cli_build.CLI):
        pytest.skip("tests/cxx/_build/wgprof_b200_cli not built (build() in the "
                    "container with /root/reference)")
    return cli_build.CLI


@pytest.mark.gpu
@pytest.mark.parametrize("name", G.NAMES)
@pytest.mark.parametrize("cmd", ["decode", "replay", "export", "export_1965"])
def test_reference_cli_on_the_shim_byte_identical(name, cmd):
    argv = G.commands(name)[cmd]
    r = subprocess.run([_cli(), *argv], capture_output=True, timeout=300)
    assert r.returncode == 0, r.stderr
    want = open(os.path.join(GOLD, f"{name}_{cmd}.txt"), "rb").read()
    assert r.stdout == want


@pytest.mark.gpu
@pytest.mark.parametrize("tag", ["capacity_mismatch", "truncated", "bad_magic",
                                 "missing_file"])
def test_reference_cli_errors_on_the_shim(tmp_path, tag):
    argv = G.resolve(G.error_cases(str(tmp_path))[tag], str(tmp_path))
    r = subprocess.run([_cli(), *argv], capture_output=True, timeout=300)
    assert r.returncode == 1
    want = open(os.path.join(GOLD, f"error_{tag}.txt"), "rb").read()
    assert r.stderr.replace(str(tmp_path).encode(), b"@") == want


def test_cli_links_libwgpf():
    """CPU check: the shim CLI is built and links the in-tree libwgpf.so."""
    cli = _cli()
    out = subprocess.run(["ldd", cli], capture_output=True, text=True).stdout
    assert "libwgpf.so" in out
