"""Dump the decoded device trace of the instrumented attention kernel (config
3 shape, fewer heads) for offline inspection: gpurun_out/<tag>/attn_ev_s{1,2}.npy"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2505_21661_b200 import p1  # noqa: E402
from paper_2505_21661_b200 import trace as T  # noqa: E402

out = sys.argv[1] if len(sys.argv) > 1 else "gpurun_out/attn_dump"
os.makedirs(out, exist_ok=True)
BH, S = int(os.environ.get("BH", 8)), 8192
g = torch.Generator(device="cuda").manual_seed(0)
q, k, v = (torch.randn(BH, S, 128, generator=g, device="cuda").to(torch.bfloat16)
           for _ in range(3))
o = torch.empty_like(q)
ctas = BH * S // 256
prof = torch.zeros(p1.attn_profile_bytes(BH, S), dtype=torch.uint8, device="cuda")
timing = torch.zeros(ctas * 32, dtype=torch.uint8, device="cuda")
ctx = T.Context(0)
ctx.set_plan(T.BufferPlan(p1.ATTN_SLOTS, T.BufferStrategy.Circular, p1.ATTN_LABELS))
n_streams = ctas * p1.ATTN_WARPS
ev = torch.empty(n_streams * p1.ATTN_SLOTS * 32, dtype=torch.uint8, device="cuda")
for stages in (1, 2):
    for _ in range(3):
        p1.attention(q.data_ptr(), k.data_ptr(), v.data_ptr(), o.data_ptr(), BH, S,
                     kv_stages=stages, instrument=True, profile_ptr=prof.data_ptr(),
                     timing_ptr=timing.data_ptr())
    torch.cuda.synchronize()
    ne, w = ctx.replay_device(prof.data_ptr(), prof.numel(), n_streams, 0,
                              ev.data_ptr(), n_streams * p1.ATTN_SLOTS)
    np.save(f"{out}/attn_ev_s{stages}.npy", ev[:ne * 32].cpu().numpy().view(T.EVENT_DTYPE))
    np.save(f"{out}/attn_body_s{stages}.npy", prof.cpu().numpy())
    np.save(f"{out}/attn_timing_s{stages}.npy", timing.cpu().numpy())
print("ok", ne)
