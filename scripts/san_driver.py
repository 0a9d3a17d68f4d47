"""Small inputs through every hot kernel, for compute-sanitizer
(memcheck / racecheck / synccheck): pass 1 (k_count_tps, TMA and cp.async
windows), k_tps (grouped TMA), k_tpsd (TMA and cp.async windows; deep and
wide geometries), k_exact_mean, k_fast_emit,
the general path, the critical path / overlap kernels (k_cp*), the Chrome
formatter and the alignment kernel."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT, os.path.join(ROOT, "tests")]
import numpy as np  # noqa: E402
import torch  # noqa: E402

import fuzz  # noqa: E402
from paper_2505_21661_b200 import trace as T  # noqa: E402
from paper_2505_21661_b200 import workloads as W  # noqa: E402

ctx = T.Context(0)
# config 4 slice (k_count_tps + k_tps with TMA windows)
ctx.set_plan(T.BufferPlan(W.CAP, T.BufferStrategy.Flush, W.MIXED_LABELS))
n = 4096
body = torch.empty(n * W.stream_stride(), dtype=torch.uint8, device="cuda")
ctx.synth_body(body.data_ptr(), W.MIXED, 0, n, n // 2)
ev = torch.empty(n * 128 * 32, dtype=torch.uint8, device="cuda")
ne, _ = ctx.replay_device(body.data_ptr(), body.numel(), n, 33, ev.data_ptr(), n * 128)
e = ev[:ne * 32].cpu().numpy().view(T.EVENT_DTYPE)
cp = ctx.critical_path(e, [("TMA0.wait", "MMA"), ("MMA", "TMA0")], gate_by_block=True)
ov = ctx.overlap(e, [0] * 4 + [1] * 12)
js = ctx.export_chrome_trace(None, 1000.0, on_device_ptr=ev.data_ptr(), n_events=min(ne, 20000))
# config 5 slice (k_tpsd, TMA windows)
ctx.set_plan(T.BufferPlan(W.CAP, T.BufferStrategy.Circular, W.NESTED_LABELS))
n5 = 1024
b5 = torch.empty(n5 * W.stream_stride(), dtype=torch.uint8, device="cuda")
ctx.synth_body(b5.data_ptr(), W.NESTED, 0, n5, 0)
e5 = torch.empty(n5 * 128 * 32, dtype=torch.uint8, device="cuda")
ctx.replay_device(b5.data_ptr(), b5.numel(), n5, 33, e5.data_ptr(), n5 * 128)
# deep streams with mixed starts (cp.async windows), deep + general streams
for seed, case in enumerate([dict(n_streams=64, cap=256, depth=20, same_start=False),
                             dict(n_streams=64, cap=128, depth=64)]):
    data, cap, st, labels = fuzz.deep_image(77 + seed, **case)
    ctx.replay_image_bytes(data, T.BufferPlan(cap, T.BufferStrategy(st), labels), 33)
# wide streams (k_tpsd<kWide>: > 64 labels), TMA and cp.async windows; the
# exact-mean statistics (k_exact_mean's shared-memory ring) on them
for seed, case in enumerate([dict(n_streams=64, cap=256, depth=20),
                             dict(n_streams=64, cap=256, depth=32, same_start=False)]):
    data, cap, st, labels = fuzz.wide_image(88 + seed, **case)
    ctx.replay_image_bytes(data, T.BufferPlan(cap, T.BufferStrategy(st), labels), 33,
                           flags=0x2)
# random fuzz images: warp-per-stream and general paths, errors
for seed in range(12):
    data, cap, st, labels = fuzz.random_image(500 + seed, n_streams=40, cap=64, mode="random")
    try:
        ctx.replay_image_bytes(data, T.BufferPlan(cap, T.BufferStrategy(st), labels), 33)
    except T.Error:
        pass
torch.cuda.synchronize()
print("san driver ok", ne, cp["period"] if isinstance(cp, dict) and "period" in cp else "", ov["blocks"])
