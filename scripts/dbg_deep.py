"""Debug: one deep-kernel fuzz case, GPU vs oracle, first differing event."""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT, os.path.join(ROOT, "tests")]
import fuzz  # noqa: E402
from oracle import oracle as O  # noqa: E402
from paper_2505_21661_b200 import trace as T  # noqa: E402

case = dict(n_streams=96, cap=256, depth=64)
if len(sys.argv) > 1:
    case = eval(sys.argv[1])
data, cap, st, labels = fuzz.deep_image(int(os.environ.get("SEED", 31000)), **case)
o = O.Oracle().replay_kpft(data, cap, st, labels, 33)
c = T.Context(0)
r = c.replay_image_bytes(data, T.BufferPlan(cap, T.BufferStrategy(st), labels), 33)
print("n", len(r.events), len(o.events), "prof", c.last_profile())
d = np.nonzero(r.events != o.events)[0]
print("ndiff", len(d))
for i in d[:6]:
    print(i, r.events[i], o.events[i])

# per-stream: which streams differ, their nesting depth
stride = 16 + 8 * cap
body = np.frombuffer(data[8:], np.uint8)
orc = O.Oracle()
pos = 0
bad = []
for s in range(case["n_streams"]):
    one = body[s * stride:(s + 1) * stride]
    oe = orc.replay_body(one, 1, cap, st, labels, 33).events
    h = one[:16].view(np.uint32)
    cnt, start = int(h[2]), int(h[2]) % cap if h[2] > cap else 0
    recs = one[16:].view(np.uint32).reshape(-1, 2)
    tags = np.concatenate([recs[start:, 0], recs[:start, 0]])[:min(cnt, cap)]
    q = np.cumsum(np.where(tags >> 31, 1, -1))
    dmax = int((q - np.minimum.accumulate(np.minimum(q, 0))).max())
    same = np.array_equal(r.events[pos:pos + len(oe)], oe)
    zero = not r.events[pos:pos + len(oe)].view(np.uint64).any()
    if not same:
        bad.append((s, dmax, start, len(oe), zero))
    pos += len(oe)
print("bad streams (s, depth, start, events, all-zero):", bad[:20], len(bad))
