"""Throughput of the interval-overlap analyser (K6: wgpf_critical_path,
wgpf_overlap_counters) and of the warp-per-stream fallback kernel
(k_fast_emit) on device-resident inputs; prints one JSON object.

  critical path / overlap: events of config-4 prefixes (2.6 M events, the
  size of the config-3 attention trace, and 33 M / 133 M events), gated per
  (block, warp group); events/s and GB/s of event bytes read (32 B / event).
  k_fast_emit: a trace whose streams use region ids >= 64 (so pass 1 routes
  them to the warp-per-stream kernel): 2^20 streams x 222 records.
"""
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

from paper_2505_21661_b200 import trace as T  # noqa: E402
from paper_2505_21661_b200 import workloads as W  # noqa: E402


def cuda_time(fn, reps=3):
    fn()
    torch.cuda.synchronize()
    best = 1e30
    for _ in range(reps):
        torch.cuda.synchronize()
        a = time.perf_counter()
        fn()
        torch.cuda.synchronize()
        best = min(best, time.perf_counter() - a)
    return best


def main():
    out = {}
    ctx = T.Context(0)
    plan = T.BufferPlan(W.CAP, T.BufferStrategy.Flush, W.MIXED_LABELS)
    ctx.set_plan(plan)
    n = 1 << 20
    body = torch.empty(n * W.stream_stride(), dtype=torch.uint8, device="cuda")
    ctx.synth_body(body.data_ptr(), W.MIXED, 0, n, n // 2)
    ne, _ = ctx.replay_device(body.data_ptr(), body.numel(), n, 33, 0, 0, 0x1 | 0x8)
    ev = torch.empty(ne * 32, dtype=torch.uint8, device="cuda")
    ctx.replay_device(body.data_ptr(), body.numel(), n, 33, ev.data_ptr(), ne)
    edges = [("TMA0.wait", "MMA"), ("TMA1.wait", "MMA"), ("MMA", "TMA0"), ("MMA", "TMA1")]
    roles = [0] * 4 + [1] * 12
    rows = []
    for m in (2_600_000, 33_000_000, ne):
        m = min(m, ne)
        t_cp = cuda_time(lambda: ctx.critical_path(None, edges, on_device_ptr=ev.data_ptr(),
                                                    n_events=m, gate_by_block=True))
        t_ov = cuda_time(lambda: ctx.overlap(None, roles, on_device_ptr=ev.data_ptr(),
                                             n_events=m))
        rows.append({"events": m, "critical_path_s": t_cp, "critical_path_events_per_s": m / t_cp,
                     "critical_path_gbs_event_bytes": 32 * m / t_cp / 1e9,
                     "overlap_s": t_ov, "overlap_events_per_s": m / t_ov,
                     "overlap_gbs_event_bytes": 32 * m / t_ov / 1e9})
    out["k6"] = rows
    del ev, body
    torch.cuda.empty_cache()

    # warp-per-stream fallback: nested scopes over region ids 60..99 (ids >= 64
    # leave the thread-per-stream kernels), 100 labels, flush, 222 records
    labels = [f"W{i:03d}" for i in range(100)]
    nb = 1 << 20
    rec = 222
    tags = np.zeros(rec, np.uint32)
    depth = 20
    pat = [0x80000000 | ((60 + d) << 12) for d in range(depth)] + \
          [((60 + d) << 12) for d in reversed(range(depth))]
    for i in range(rec):
        tags[i] = pat[i % len(pat)]
    rng = np.random.default_rng(1)
    stride_w = 4 + 2 * W.CAP
    host = np.zeros((nb, stride_w), np.uint32)
    host[:, 0] = np.arange(nb) // 16
    host[:, 1] = np.arange(nb) % 16
    host[:, 2] = rec
    host[:, 3] = W.CAP
    clocks = np.cumsum(rng.integers(1, 200, (nb, rec), dtype=np.uint32), axis=1, dtype=np.uint32)
    host[:, 4:4 + 2 * rec:2] = tags
    host[:, 5:5 + 2 * rec:2] = clocks
    wb = torch.from_numpy(host.view(np.uint8).reshape(-1)).cuda()
    ctx.set_plan(T.BufferPlan(W.CAP, T.BufferStrategy.Flush, labels))
    ne, _ = ctx.replay_device(wb.data_ptr(), wb.numel(), nb, 33, 0, 0, 0x1 | 0x8)
    wev = torch.empty(ne * 32, dtype=torch.uint8, device="cuda")
    profs = []
    for _ in range(4):
        ctx.replay_device(wb.data_ptr(), wb.numel(), nb, 33, wev.data_ptr(), ne, 0x10)
        profs.append(ctx.last_profile())
    p = profs[-1]
    alg = 16 * nb + 8 * rec * nb + 32 * ne
    out["k_fast_emit"] = {"streams": nb, "records": rec * nb, "events": ne,
                          "regions": len(labels), "nesting": depth,
                          "emit_ms": p["emit_ms"], "count_ms": p["count_ms"],
                          "records_per_s_emit": rec * nb / (p["emit_ms"] / 1e3),
                          "gbs_algorithmic_emit": alg / (p["emit_ms"] / 1e3) / 1e9}
    print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()
