"""Seed sweep of the deep / wide thread-per-stream kernels and the random
fuzz images against the oracle (GPU box; not part of the default test run):
python scripts/fuzz_sweep.py [seeds]"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT, os.path.join(ROOT, "tests")]
import numpy as np  # noqa: E402

import fuzz  # noqa: E402
from oracle import oracle as O  # noqa: E402
from paper_2505_21661_b200 import trace as T  # noqa: E402
from test_gpu_parity import DEEP_CASES, WIDE_CASES  # noqa: E402

seeds = int(sys.argv[1]) if len(sys.argv) > 1 else 20
ctx, orc = T.Context(0), O.Oracle()
bad = []
n = 0


def check(tag, data, cap, st, labels):
    global n
    n += 1
    try:
        o, oerr = orc.replay_kpft(data, cap, st, labels, 33), None
    except O.OracleError as e:
        o, oerr = None, (e.category, str(e))
    try:
        r, gerr = ctx.replay_image_bytes(data, T.BufferPlan(cap, T.BufferStrategy(st), labels),
                                         33, flags=0x2), None
    except T.Error as e:
        r, gerr = None, (e.category(), str(e))
    if oerr != gerr:
        bad.append((tag, "error", oerr, gerr))
        return
    if oerr:
        return
    if len(r.events) != len(o.events) or not np.array_equal(r.events, o.events):
        bad.append((tag, "events"))
        return
    if (r.dropped_heads, r.truncated_tails, r.flagged_preconditions, r.malformed_groups) != \
            (o.dropped_heads, o.truncated_tails, o.flagged_preconditions, o.malformed_groups):
        bad.append((tag, "warnings"))
        return
    got = ctx.stats()
    for s in orc.region_stats(o.events, labels):
        g = got[s.label]
        if (g.count, g.min, g.max, g.sum, g.mean, g.first_event, g.warp_group, g.kind,
                g.hist) != (s.count, s.min, s.max, s.sum, s.mean, s.first_event,
                            s.warp_group, s.kind, s.hist):
            bad.append((tag, "stats", s.label))
            return


for case, kw in enumerate(DEEP_CASES):
    for seed in range(seeds):
        check(("deep", case, seed), *fuzz.deep_image(900000 + 1000 * case + seed, **kw))
for case, kw in enumerate(WIDE_CASES):
    for seed in range(seeds):
        check(("wide", case, seed), *fuzz.wide_image(800000 + 1000 * case + seed, **kw))
for seed in range(seeds * 4):
    for mode in ("nested", "random"):
        check(("random", mode, seed),
              *fuzz.random_image(700000 + seed, n_streams=48, cap=64, mode=mode,
                                 big_gaps=seed % 3 == 0))
print(f"fuzz sweep: {n} images, {len(bad)} mismatches")
for b in bad[:20]:
    print(b)
sys.exit(1 if bad else 0)
