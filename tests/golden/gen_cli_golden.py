"""Golden outputs of the reference CLI's decode / replay / export commands
(/root/reference/proj/tools/wgprof.cpp:78-126, built unchanged against the
reference headers by tests/cxx/cli_build.py into oracle/_ref/wgprof_ref_cli)
on the four fixtures.  tests/test_gpu_cli.py runs the same commands built
against include/wgprof_b200.hpp and compares byte for byte.

Run: python tests/golden/gen_cli_golden.py   (needs /root/reference)
"""
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, os.path.join(ROOT, "tests", "cxx"))
import cli_build  # noqa: E402

FIX = os.path.join(HERE, "fixtures")
OUT = os.path.join(HERE, "cli")
NAMES = ["simple", "gemm_swp", "fa3_vanilla", "fa3_improved"]


def commands(name):
    k, d = os.path.join(FIX, name + ".kpft"), os.path.join(FIX, name + ".dev")
    cost = open(os.path.join(FIX, name + ".cost")).read().split()[0]
    return {"decode": ["decode", k, d], "replay": ["replay", k, d, cost],
            "export": ["export", k, d, cost, "1000"],
            "export_1965": ["export", k, d, cost, "1965"]}


def error_cases(tmp):
    """Inputs the reference rejects: (tag, argv); files written under tmp."""
    k = os.path.join(FIX, "simple.kpft")
    data = open(k, "rb").read()
    trunc = os.path.join(tmp, "trunc.kpft")
    open(trunc, "wb").write(data[:-5])
    badmagic = os.path.join(tmp, "badmagic.kpft")
    open(badmagic, "wb").write(b"XPFT" + data[4:])
    return {
        "capacity_mismatch": ["replay", k, os.path.join(FIX, "fa3_vanilla.dev"), "33"],
        "truncated": ["replay", "@trunc.kpft", os.path.join(FIX, "simple.dev"), "33"],
        "bad_magic": ["export", "@badmagic.kpft", os.path.join(FIX, "simple.dev"), "33",
                      "1000"],
        "missing_file": ["decode", "@absent.kpft", os.path.join(FIX, "simple.dev")],
    }


def resolve(argv, tmp):
    return [os.path.join(tmp, a[1:]) if a.startswith("@") else a for a in argv]


def main():
    import tempfile
    cli_build.build()
    os.makedirs(OUT, exist_ok=True)
    for name in NAMES:
        for tag, argv in commands(name).items():
            r = subprocess.run([cli_build.REF_CLI, *argv], capture_output=True)
            assert r.returncode == 0, r.stderr
            open(os.path.join(OUT, f"{name}_{tag}.txt"), "wb").write(r.stdout)
    with tempfile.TemporaryDirectory() as tmp:
        for tag, argv in error_cases(tmp).items():
            r = subprocess.run([cli_build.REF_CLI, *resolve(argv, tmp)],
                               capture_output=True)
            assert r.returncode == 1, (tag, r.returncode)
            err = r.stderr.replace(tmp.encode(), b"@")
            open(os.path.join(OUT, f"error_{tag}.txt"), "wb").write(err)
    print("wrote", OUT)


if __name__ == "__main__":
    main()
