"""Shapes of the synthetic traces of SURVEY.md 8(d) configs 4 and 5, as the
device generator (csrc/k_synth.cuh, C-ABI wgpf_synth_body) writes them.

config 4 ("mixed", flush): stream s -> block s // 16, warp s % 16, slot
  capacity 256, record_count 222 for s < n_long else 221 (2^30 records at full
  size); regions TMA0 TMA0.wait TMA1 TMA1.wait MMA MMA.k EPI EPI.st.
config 5 ("nested", circular): 2^22 streams, capacity 256, 1000 writes each,
  64 regions R00..R63, S0..S63 E63..E0 repeated.
"""
from __future__ import annotations

MIXED, NESTED = 0, 1  # wgpf_synth_body shapes
CAP = 256
STREAMS_PER_BLOCK = 16
MIXED_LABELS = ["TMA0", "TMA0.wait", "TMA1", "TMA1.wait", "MMA", "MMA.k", "EPI",
                "EPI.st"]
NESTED_LABELS = [f"R{i:02d}" for i in range(64)]
MIXED_FULL_STREAMS = 148 * 2048 * 16
MIXED_FULL_LONG = 1966080
NESTED_FULL_STREAMS = 1 << 22
NESTED_WRITES = 1000


def stream_stride(cap: int = CAP) -> int:
    return 16 + 8 * cap


def mixed_long_for(n_streams: int) -> int:
    """Streams with 222 records (the first ones) in an n-stream mixed trace."""
    if n_streams == MIXED_FULL_STREAMS:
        return MIXED_FULL_LONG
    return int(round(n_streams * MIXED_FULL_LONG / MIXED_FULL_STREAMS))


def mixed_records(s0: int, s1: int, n_long: int) -> int:
    """Records of streams [s0, s1) of a mixed trace."""
    nl = max(0, min(s1, n_long) - s0)
    return 222 * nl + 221 * (s1 - s0 - nl)
