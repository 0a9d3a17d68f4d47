"""Builds the reference's own CLI commands against the drop-in header.

The replay / export / decode commands of the reference CLI
(/root/reference/proj/tools/wgprof.cpp: emit, load_device, load_image,
cmd_decode, cmd_replay, cmd_export) are taken from the reference source AS IS
at build time -- nothing is copied into this repository -- and compiled twice:

  tests/cxx/_build/wgprof_b200_cli   against include/wgprof_b200.hpp, linked
                                     with libwgpf.so (the GPU path)
  oracle/_ref/wgprof_ref_cli         against the reference headers (test
                                     oracle: golden outputs)

Both get the same small main() (the reference's main parses flags with CLI11,
which is not vendored; the argv order here is fixed).  The binaries are
git-ignored and travel to the GPU box with the tree, like oracle/_ref.
Run: python tests/cxx/cli_build.py  (also called by __graft_entry__.build()).
"""
from __future__ import annotations

import os
import re
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
REF = "/root/reference/proj"
TOOL = os.path.join(REF, "tools", "wgprof.cpp")
JSON_DIR = ("/opt/prime-rl/.venv/lib/python3.12/site-packages/include/cudnn_frontend/"
            "thirdparty/nlohmann")
OUT = os.path.join(HERE, "_build")
CLI = os.path.join(OUT, "wgprof_b200_cli")
REF_CLI = os.path.join(ROOT, "oracle", "_ref", "wgprof_ref_cli")

MAIN = r'''
int main(int argc, char** argv) {
  try {
    const std::string cmd = argc > 1 ? argv[1] : "";
    auto arg = [&](int i) { return i < argc ? std::string(argv[i]) : std::string("-"); };
    if (cmd == "decode" && argc >= 4) return cmd_decode(argv[2], argv[3], arg(4));
    if (cmd == "replay" && argc >= 5)
      return cmd_replay(argv[2], argv[3], std::stoull(argv[4]), arg(5));
    if (cmd == "export" && argc >= 6)
      return cmd_export(argv[2], argv[3], std::stoull(argv[4]), std::stod(argv[5]),
                        arg(6));
    std::cerr << "usage: decode <trace> <dev> [out] | replay <trace> <dev> <cost> [out]"
                 " | export <trace> <dev> <cost> <cycles_per_us> [out]\n";
    return 2;
  } catch (const wgprof::Error& e) {
    std::cerr << "error: " << e.category() << ": " << e.what() << "\n";
    return 1;
  } catch (const std::exception& e) {
    std::cerr << "error: internal: " << e.what() << "\n";
    return 1;
  }
}
'''


def extract(src: str) -> str:
    """emit() and load_device() .. cmd_export() from the reference CLI."""
    m = re.search(r"^void emit\(.*?^}\n", src, re.S | re.M)
    a = src.find("wgprof::DeviceProgram load_device(")
    b = src.find("int cmd_model(")
    if not m or a < 0 or b < 0:
        raise RuntimeError("reference CLI layout not recognised")
    return m.group(0) + "\n" + src[a:b]


def source(shim: bool) -> str:
    cmds = extract(open(TOOL).read())
    if shim:
        head = '#include <iostream>\n#include <sstream>\n#include "wgprof_b200.hpp"\n'
    else:
        head = ('#include <iostream>\n#include <sstream>\n'
                '#include "wgprof/lower.hpp"\n#include "wgprof/perfmodel.hpp"\n'
                '#include "wgprof/pipeline.hpp"\n#include "wgprof/trace.hpp"\n')
    return head + "namespace {\n" + cmds + "}  // namespace\n" + MAIN


SHIM_BENCH = os.path.join(OUT, "shim_bench")


def build_shim_bench(verbose: bool = False) -> str:
    """tests/cxx/shim_bench.cpp (the drop-in C++ path, end to end) against
    the shim and libwgpf.so; needs no reference sources."""
    sys.path.insert(0, ROOT)
    from paper_2505_21661_b200 import _build
    lib = _build.build()
    os.makedirs(OUT, exist_ok=True)
    cmd = ["g++", "-std=c++20", "-O2", os.path.join(HERE, "shim_bench.cpp"),
           "-I", os.path.join(ROOT, "include"), "-I", "/usr/local/cuda/include", lib,
           "-L/usr/local/cuda/lib64", "-lcudart", f"-Wl,-rpath,{os.path.dirname(lib)}",
           "-Wl,-rpath,/usr/local/cuda/lib64", "-o", SHIM_BENCH]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"building shim_bench failed:\n{r.stderr[-6000:]}")
    if verbose:
        print("built", SHIM_BENCH)
    return SHIM_BENCH


def build(verbose: bool = False) -> bool:
    build_shim_bench(verbose)
    if not os.path.exists(TOOL):
        return os.path.exists(CLI)
    sys.path.insert(0, ROOT)
    from paper_2505_21661_b200 import _build
    lib = _build.build()
    os.makedirs(OUT, exist_ok=True)
    os.makedirs(os.path.dirname(REF_CLI), exist_ok=True)
    jobs = [
        (source(True), CLI, ["-I", os.path.join(ROOT, "include"), "-I", JSON_DIR, lib,
                             f"-Wl,-rpath,{os.path.dirname(lib)}"]),
        (source(False), REF_CLI, ["-I", os.path.join(REF, "include"), "-I", JSON_DIR]),
    ]
    for text, out, flags in jobs:
        # the source goes through stdin: no file with reference text is left
        cmd = ["g++", "-std=c++20", "-O2", "-x", "c++", "-", "-x", "none", *flags, "-o",
               out]
        r = subprocess.run(cmd, input=text, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"building {out} failed:\n{r.stderr[-6000:]}")
        if verbose:
            print("built", out)
    return True


if __name__ == "__main__":
    build(verbose=True)
