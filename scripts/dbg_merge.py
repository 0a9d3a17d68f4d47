"""Debug helper: stats export / merge round trip on one device."""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from oracle import synth as S  # noqa: E402
from paper_2505_21661_b200 import trace as t  # noqa: E402

n = 40000
plan = t.BufferPlan(S.CAP, t.BufferStrategy(1), list(S.MIXED_LABELS))
body = torch.empty(n * S.stream_stride(), dtype=torch.uint8, device="cuda")
ctx = t.Context(0)
ctx.set_plan(plan)
ctx.synth_body(body.data_ptr(), 0, S.MIXED_FULL_LONG - n // 2, n, S.MIXED_FULL_LONG)
ctx.replay_device(body.data_ptr(), body.numel(), n, 33, 0, 0, 0x1)
whole = ctx.stats()
pb = ctx.stats_packed_bytes()
print("pb", pb, "per", pb // 8)
parts = [t.Context(0), t.Context(0)]
g = torch.zeros(2 * pb, dtype=torch.uint8, device="cuda")
cut = 17003
stride = S.stream_stride()
for r, (a, b) in enumerate([(0, cut), (cut, n)]):
    c = parts[r]
    c.set_plan(plan)
    c.replay_device(body.data_ptr() + a * stride, (b - a) * stride, b - a, 33, 0, 0, 0x1,
                    stream_base=a)
    c.stats_export(g.data_ptr() + r * pb)
torch.cuda.synchronize()
pc = [p.stats() for p in parts]
k0 = S.MIXED_LABELS[0]
for k in whole:
    print(k, whole[k].count, [p[k].count if k in p else 0 for p in pc])
for nr in (1, 2):
    m = t.Context(0)
    m.set_plan(plan)
    m.stats_merge(g.data_ptr(), nr)
    ms = m.stats()
    print("merge", nr, {k: v.count for k, v in ms.items()})
# merge rank 1 alone
m = t.Context(0)
m.set_plan(plan)
m.stats_merge(g.data_ptr() + pb, 1)
print("merge rank1 alone", {k: v.count for k, v in m.stats().items()})
