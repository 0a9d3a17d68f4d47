"""Seeded random KPFT images for parity tests (edge cases the reference's
own tests exercise: wrap-around circular buffers, dropped heads, truncated
tails, wait markers / orphans, out-of-table region ids, duplicate labels,
32-bit clock wraps, non-single-stack nesting)."""
from __future__ import annotations

import numpy as np

from oracle import synth as S

LABEL_SETS = [
    ["A", "A.wait", "B", "B.wait", "C"],
    ["X", "X.wait", "X.wait.wait", "Y", "X"],           # duplicate label
    ["region#7", "region#7.wait", "L", "L.wait"],       # collides with id 7
    ["Load K", "Load K.wait", "GEMM", "GEMM.wait", "Softmax", ".wait", "Z.wait"],
]


def _stream_records(rng, n, n_labels, mode, big_gaps):
    """Chronological records of one stream."""
    tags, clocks = [], []
    clock = int(rng.integers(0, 1 << 32))
    open_stack = []
    ids_hi = n_labels + 4  # some out-of-table ids
    while len(tags) < n:
        r = rng.random()
        if mode == "nested":
            # properly nested with canonical async groups
            if open_stack and r < 0.45:
                rid = open_stack.pop()
                tags.append(rid << 12)
            elif r < 0.65 and n_labels >= 2:
                base = int(rng.integers(0, n_labels))
                tags.append(0x80000000 | (base << 12))
                gap_clock = clock
                clocks.append(clock)
                clock = (clock + int(rng.integers(1, 300))) & 0xFFFFFFFF
                if len(tags) >= n:
                    break
                tags.append(base << 12)
                clocks.append(clock)
                clock = (clock + int(rng.integers(0, 50 if rng.random() < 0.5 else 3000))) & 0xFFFFFFFF
                m = min(n_labels - 1, base + 1)
                if len(tags) >= n:
                    break
                tags.append(0x80000000 | (m << 12))
                clocks.append(clock)
                clock = (clock + int(rng.integers(0, 40))) & 0xFFFFFFFF
                if len(tags) >= n:
                    break
                if rng.random() < 0.85:
                    tags.append(m << 12)
                else:
                    open_stack.append(m)
                    continue
                del gap_clock
            else:
                rid = int(rng.integers(0, ids_hi if rng.random() < 0.1 else n_labels))
                tags.append(0x80000000 | (rid << 12))
                open_stack.append(rid)
        else:  # "random": arbitrary start/end sequence (may cross regions)
            rid = int(rng.integers(0, ids_hi if rng.random() < 0.1 else n_labels))
            tags.append((0x80000000 if rng.random() < 0.5 else 0) | (rid << 12) |
                        int(rng.integers(0, 4096)))
        clocks.append(clock)
        if big_gaps and rng.random() < 0.05:
            clock = (clock + int(rng.integers(1 << 30, (1 << 32) - 1))) & 0xFFFFFFFF
        else:
            clock = (clock + int(rng.integers(0, 500))) & 0xFFFFFFFF
    return np.array(tags[:n], np.uint32), np.array(clocks[:n], np.uint32)


def random_image(seed: int, n_streams: int = 8, cap: int = 64,
                 mode: str = "nested", big_gaps: bool = False,
                 labels_idx: int | None = None, per_block: int = 4):
    """Returns (kpft v1 bytes, slots, strategy, labels)."""
    rng = np.random.default_rng(seed)
    labels = LABEL_SETS[labels_idx if labels_idx is not None else
                        int(rng.integers(0, len(LABEL_SETS)))]
    strategy = int(rng.integers(0, 2))
    body = np.zeros((n_streams, 4 + 2 * cap), np.uint32)
    for s in range(n_streams):
        if strategy == 1:
            count = int(rng.integers(0, cap + 1))
            writes = count
        else:
            count = int(rng.integers(0, 3 * cap))
            writes = count
        tags, clocks = _stream_records(rng, writes, len(labels), mode, big_gaps)
        body[s, 0] = s // per_block
        body[s, 1] = s % per_block
        body[s, 2] = count
        body[s, 3] = cap
        for w in range(writes):
            slot = w % cap
            body[s, 4 + 2 * slot] = tags[w]
            body[s, 5 + 2 * slot] = clocks[w]
    data = S.kpft_v1(body.view(np.uint8).reshape(-1), n_streams)
    return data, cap, strategy, labels


DEEP_LABELS = [f"D{i:02d}" for i in range(56)] + [f"D{i:02d}.wait" for i in range(8)]


def _deep_records(rng, writes, depth, big_gaps, violate, level_ids=None, n_base=56):
    """A nesting program `depth` levels deep (labels D00.. by level),
    repeated: START per level going down, at the bottom an async group of an
    eight-label base (S(X) E(X) S(X.wait) E(X.wait)) or a plain scope, then
    the ENDs going up; `violate` swaps one END's region now and then."""
    tags, clocks = [], []
    clock = int(rng.integers(0, 1 << 32))

    def rec(tag):
        nonlocal clock
        tags.append(tag)
        clocks.append(clock)
        if big_gaps and rng.random() < 0.01:
            clock = (clock + int(rng.integers(1 << 29, 1 << 31))) & 0xFFFFFFFF
        else:
            clock = (clock + int(rng.integers(1, 300))) & 0xFFFFFFFF

    while len(tags) < writes:
        d = depth if rng.random() < 0.7 else int(rng.integers(1, depth + 1))
        ids = level_ids if level_ids is not None else list(range(depth))
        for lv in range(d):
            rec(0x80000000 | (ids[lv] << 12))
        x = int(rng.integers(0, 8))
        if rng.random() < 0.5:
            rec(0x80000000 | (x << 12))
            rec(x << 12)
            rec(0x80000000 | ((n_base + x) << 12))
            rec((n_base + x) << 12)
        for lv in reversed(range(d)):
            r = ids[lv]
            if violate and rng.random() < 0.01:
                r = ids[(lv + 1) % d] if d > 1 else (r + 1) % n_base
            rec(r << 12)
    return np.array(tags[:writes], np.uint32), np.array(clocks[:writes], np.uint32)


def deep_image(seed: int, n_streams: int = 64, cap: int = 256, depth: int = 40,
               same_start: bool = True, odd: bool = False, big_gaps: bool = False,
               violate: bool = False, per_block: int = 16):
    """Circular streams of deep nesting (the deep thread-per-stream kernel's
    inputs): every stream wraps (writes > cap); same_start gives all streams
    one write count (one start slot: TMA windows), odd an odd start slot.
    Returns (kpft v1 bytes, slots, strategy, labels)."""
    rng = np.random.default_rng(seed)
    body = np.zeros((n_streams, 4 + 2 * cap), np.uint32)
    base_writes = 3 * cap + (1 if odd else 0) + (0 if odd else 2 * int(rng.integers(0, cap // 2)))
    for s in range(n_streams):
        writes = base_writes if same_start else int(rng.integers(cap + 1, 4 * cap))
        tags, clocks = _deep_records(rng, writes, depth, big_gaps, violate)
        body[s, 0] = s // per_block
        body[s, 1] = s % per_block
        body[s, 2] = writes
        body[s, 3] = cap
        for w in range(writes):
            slot = w % cap
            body[s, 4 + 2 * slot] = tags[w]
            body[s, 5 + 2 * slot] = clocks[w]
    data = S.kpft_v1(body.view(np.uint8).reshape(-1), n_streams)
    return data, cap, 0, list(DEEP_LABELS)


def wide_image(seed: int, n_streams: int = 64, cap: int = 256, depth: int = 20,
               n_labels: int = 200, same_start: bool = True, big_gaps: bool = False,
               violate: bool = False, per_block: int = 16):
    """Circular streams of plans with many labels (the wide thread-per-stream
    kernel's inputs): labels W000.. (n_labels - 8 bases, then ".wait" markers
    of the first eight), every stream nests `depth` levels whose region ids
    are drawn from the whole table (ids >= 64 past the deep kernel).
    Returns (kpft v1 bytes, slots, strategy, labels)."""
    rng = np.random.default_rng(seed)
    n_base = n_labels - 8
    labels = [f"W{i:03d}" for i in range(n_base)] + [f"W{i:03d}.wait" for i in range(8)]
    level_ids = [int(x) for x in rng.choice(np.arange(8, n_base), depth, replace=False)]
    body = np.zeros((n_streams, 4 + 2 * cap), np.uint32)
    base_writes = 3 * cap + 2 * int(rng.integers(0, cap // 2))
    for s in range(n_streams):
        writes = base_writes if same_start else int(rng.integers(cap + 1, 4 * cap))
        tags, clocks = _deep_records(rng, writes, depth, big_gaps, violate, level_ids, n_base)
        body[s, 0] = s // per_block
        body[s, 1] = s % per_block
        body[s, 2] = writes
        body[s, 3] = cap
        for w in range(writes):
            slot = w % cap
            body[s, 4 + 2 * slot] = tags[w]
            body[s, 5 + 2 * slot] = clocks[w]
    data = S.kpft_v1(body.view(np.uint8).reshape(-1), n_streams)
    return data, cap, 0, labels
