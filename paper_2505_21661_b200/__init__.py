"""paper_2505_21661_b200 -- B200-native (sm_100a) KPerfIR trace runtime and
post-processor.

The product is the CUDA library libwgpf.so (csrc/, C-ABI in include/wgpf.h);
this package holds its in-tree build and the Python mirror of the reference's
trace API (trace.py).  There is no CPU fallback.
"""
from . import _build  # noqa: F401

__all__ = ["trace", "models", "build"]


def build(force: bool = False) -> str:
    return _build.build(force=force)
