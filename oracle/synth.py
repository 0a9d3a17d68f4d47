"""oracle/synth.py -- TEST INFRASTRUCTURE: CPU (numpy) restatement of the
synthetic trace generators that bench.py drives on the GPU
(paper_2505_21661_b200/csrc/synth.cu, C-ABI wgpf_synth_body).

The shapes are SURVEY.md section 8(d) configs 4 and 5:

config 4 ("mixed", flush): S streams, stream s -> block s // 16, warp s % 16,
  slot capacity 256, record_count 222 for s < n_long else 221.
  regions: TMA0 TMA0.wait TMA1 TMA1.wait MMA MMA.k EPI EPI.st
  warps 0-3 (producers) repeat  S(L) E(L) S(L.wait) E(L.wait), L = TMA0 on
  even iterations, TMA1 on odd ones; warps 4-15 (consumers) repeat
  S4 S5 S6 S7 E7 E6 E5 E4.
config 5 ("nested", circular): S streams, capacity 256, 1000 writes each,
  64 regions R00..R63, pattern S0..S63 E63..E0 repeated.

Clocks: splitmix64 seeded 0x5EED ^ s.  record 0 clock = low 32 bits of the
first draw; record i >= 1 adds gap = 1 + draw % 200, except that a producer's
E(L) -> S(L.wait) transition (record index % 4 == 2) uses 1 + draw % 4000.
All arithmetic mod 2^32.  Unwritten slots are zero.
"""
from __future__ import annotations

import numpy as np

M64 = (1 << 64) - 1
MIXED_LABELS = ["TMA0", "TMA0.wait", "TMA1", "TMA1.wait", "MMA", "MMA.k", "EPI",
                "EPI.st"]
NESTED_LABELS = [f"R{i:02d}" for i in range(64)]
CAP = 256
START = 0x80000000

# config 4 full size: 148 SMs x 2048 CTAs x 16 warps, 2^30 records
MIXED_FULL_STREAMS = 148 * 2048 * 16
MIXED_FULL_LONG = 1966080
NESTED_FULL_STREAMS = 1 << 22
NESTED_WRITES = 1000


def mixed_long_for(n_streams: int) -> int:
    """Streams with 222 records so that the full config sums to 2^30."""
    if n_streams == MIXED_FULL_STREAMS:
        return MIXED_FULL_LONG
    return int(round(n_streams * MIXED_FULL_LONG / MIXED_FULL_STREAMS))


def _splitmix_next(state: np.ndarray):
    with np.errstate(over="ignore"):
        state += np.uint64(0x9E3779B97F4A7C15)
        z = state.copy()
        z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
        z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
        z = z ^ (z >> np.uint64(31))
    return z


def mixed_tags(warp: np.ndarray, i: int) -> np.ndarray:
    """Tag of record i for streams with the given warp index."""
    prod = warp < 4
    k = i // 4
    ph = i % 4
    L = np.uint32(0 if k % 2 == 0 else 2)
    # producer: S(L) E(L) S(L.wait) E(L.wait)
    p_region = L + (1 if ph >= 2 else 0)
    p_start = ph in (0, 2)
    ptag = np.uint32((START if p_start else 0) | (int(p_region) << 12))
    j = i % 8
    if j < 4:
        c_region, c_start = 4 + j, True
    else:
        c_region, c_start = 4 + (7 - j), False
    ctag = np.uint32((START if c_start else 0) | (c_region << 12))
    return np.where(prod, ptag, ctag).astype(np.uint32)


def nested_tag(i: int) -> int:
    j = i % 128
    if j < 64:
        return START | (j << 12)
    return (127 - j) << 12


def mixed_body(s0: int, n: int, n_long: int) -> np.ndarray:
    """KPFT body (uint8) of streams [s0, s0 + n) of a mixed trace whose first
    n_long streams (global index) have 222 records."""
    s = np.arange(s0, s0 + n, dtype=np.uint64)
    warp = (s % np.uint64(16)).astype(np.uint32)
    count = np.where(s < np.uint64(n_long), 222, 221).astype(np.uint32)
    stride_words = 4 + 2 * CAP  # u32 words per stream
    out = np.zeros((n, stride_words), np.uint32)
    out[:, 0] = (s // np.uint64(16)).astype(np.uint32)
    out[:, 1] = warp
    out[:, 2] = count
    out[:, 3] = CAP
    state = (np.uint64(0x5EED) ^ s).astype(np.uint64)
    clock = np.zeros(n, np.uint32)
    prod = warp < 4
    for i in range(222):
        z = _splitmix_next(state)
        if i == 0:
            clock = (z & np.uint64(0xFFFFFFFF)).astype(np.uint32)
        else:
            mod = np.where(prod & (i % 4 == 2), np.uint64(4000), np.uint64(200))
            gap = (np.uint64(1) + z % mod).astype(np.uint32)
            with np.errstate(over="ignore"):
                clock = (clock + gap).astype(np.uint32)
        live = i < count
        tag = mixed_tags(warp, i)
        out[:, 4 + 2 * i] = np.where(live, tag, 0)
        out[:, 5 + 2 * i] = np.where(live, clock, 0)
    return out.view(np.uint8).reshape(-1)


def nested_body(s0: int, n: int, writes: int = NESTED_WRITES) -> np.ndarray:
    s = np.arange(s0, s0 + n, dtype=np.uint64)
    stride_words = 4 + 2 * CAP
    out = np.zeros((n, stride_words), np.uint32)
    out[:, 0] = (s // np.uint64(16)).astype(np.uint32)
    out[:, 1] = (s % np.uint64(16)).astype(np.uint32)
    out[:, 2] = writes
    out[:, 3] = CAP
    state = (np.uint64(0x5EED) ^ s).astype(np.uint64)
    clock = np.zeros(n, np.uint32)
    for w in range(writes):
        z = _splitmix_next(state)
        if w == 0:
            clock = (z & np.uint64(0xFFFFFFFF)).astype(np.uint32)
        else:
            gap = (np.uint64(1) + z % np.uint64(200)).astype(np.uint32)
            with np.errstate(over="ignore"):
                clock = (clock + gap).astype(np.uint32)
        if w >= writes - CAP:
            slot = w % CAP
            out[:, 4 + 2 * slot] = nested_tag(w)
            out[:, 5 + 2 * slot] = clock
    return out.view(np.uint8).reshape(-1)


def kpft_v1(body: np.ndarray, n_streams: int) -> bytes:
    assert n_streams <= 0xFFFF
    return b"KPFT" + (1).to_bytes(2, "little") + n_streams.to_bytes(2, "little") + \
        body.tobytes()


def kpft_v2(body: np.ndarray, n_streams: int) -> bytes:
    return b"KPFT" + (2).to_bytes(2, "little") + b"\0\0" + \
        n_streams.to_bytes(8, "little") + body.tobytes()


def stream_stride(cap: int = CAP) -> int:
    return 16 + 8 * cap
