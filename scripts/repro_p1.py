"""Instrumented tcgen05 GEMM profile -> GPU decoder vs oracle (debug)."""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from oracle import oracle as O  # noqa: E402
from paper_2505_21661_b200 import p1  # noqa: E402
from paper_2505_21661_b200 import trace as T  # noqa: E402

M = N = K = int(sys.argv[1]) if len(sys.argv) > 1 else 1024
g = torch.Generator(device="cuda").manual_seed(0)
A = torch.randn(M, K, generator=g, device="cuda").to(torch.bfloat16)
B = torch.randn(N, K, generator=g, device="cuda").to(torch.bfloat16)
C1 = torch.empty(M, N, dtype=torch.bfloat16, device="cuda")
ctas = (M // 128) * (N // 256)
prof = torch.zeros(p1.gemm_profile_bytes(M, N), dtype=torch.uint8, device="cuda")
p1.gemm(A.data_ptr(), B.data_ptr(), C1.data_ptr(), M, N, K, True, prof.data_ptr())
torch.cuda.synchronize()
n_streams = ctas * p1.GEMM_WARPS
host = prof.cpu().numpy()
hdr = host[: n_streams * p1.stream_stride(p1.GEMM_SLOTS)].view(np.uint32).reshape(n_streams, -1)[:, :4]
print("streams", n_streams, "count range", hdr[:, 2].min(), hdr[:, 2].max(), "cap", hdr[0, 3])
ctx = T.Context(0)
ctx.set_plan(T.BufferPlan(p1.GEMM_SLOTS, T.BufferStrategy.Circular, p1.GEMM_LABELS))
cap_ev = n_streams * p1.GEMM_SLOTS
ev = torch.empty(cap_ev * 32, dtype=torch.uint8, device="cuda")
ne, w = ctx.replay_device(prof.data_ptr(), prof.numel(), n_streams, 0, ev.data_ptr(), cap_ev)
print("gpu events", ne, w.dropped_heads, w.truncated_tails, w.flagged_preconditions, w.malformed_groups)
orc = O.Oracle()
r = orc.replay_kpft(p1.kpft_v1(host, n_streams) if n_streams < 65536 else p1.kpft_v2(host, n_streams),
                    p1.GEMM_SLOTS, 0, p1.GEMM_LABELS, 0)
print("oracle events", len(r.events))
