"""Builds compile-time variants of libwgpf_p1.so into
paper_2505_21661_b200/_lib/ab_p1/ for A/B runs (WGPF_P1_LIB_OVERRIDE).
  python scripts/build_ab_p1.py NAME "-DFOO=1" [NAME2 "..."]"""
import glob
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2505_21661_b200 import _build as B  # noqa: E402

out_dir = os.path.join(B.LIBDIR, "ab_p1")
os.makedirs(out_dir, exist_ok=True)
args = sys.argv[1:]
for name, defs in zip(args[::2], args[1::2]):
    out = os.path.join(out_dir, f"{name}.so")
    cmd = [B._nvcc(), *B.NVCC_FLAGS, *defs.split(), f"-I{B.INCLUDE}", f"-I{B.CSRC}",
           *sorted(glob.glob(os.path.join(B.CSRC_P1, "*.cu"))), "-o", out]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode:
        sys.exit(r.stderr[-4000:])
    print("built", out)
