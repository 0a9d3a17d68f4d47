"""GPU test of the multi-GPU shard-and-reduce path with the product's own
export / merge (pipeline.hpp:69-80 loops streams with no
cross-stream state).

Two processes share cuda:0 (the driver's boxes have one GPU); each owns a
contiguous block range of ONE synthetic trace (shard.stream_range), replays
it on the device (wgpf_replay_device with its global stream base), exports its
packed per-label table (wgpf_stats_export), the tables are all-gathered --
host-staged over gloo, the same bytes NCCL moves in bench.py -- and
wgpf_stats_merge combines them.  The merged table must equal, byte for byte,
the table of one process replaying the whole trace, and bench.stats_digest
must agree.
"""
import os
import queue
import socket

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

pytestmark = pytest.mark.gpu


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _setup(shape, total):
    from paper_2505_21661_b200 import trace as T
    from paper_2505_21661_b200 import workloads as W
    if shape == W.NESTED:
        plan = T.BufferPlan(W.CAP, T.BufferStrategy.Circular, W.NESTED_LABELS)
        n_long = 0
    else:
        plan = T.BufferPlan(W.CAP, T.BufferStrategy.Flush, W.MIXED_LABELS)
        n_long = total // 3
    return plan, n_long


def _replay_range(ctx, shape, s0, s1, n_long):
    import torch
    from paper_2505_21661_b200 import workloads as W
    n = s1 - s0
    body = torch.empty(max(1, n) * W.stream_stride(), dtype=torch.uint8, device="cuda")
    ctx.synth_body(body.data_ptr(), shape, s0, n, n_long)
    ev = torch.empty(max(1, n) * W.CAP * 32, dtype=torch.uint8, device="cuda")
    ne, w = ctx.replay_device(body.data_ptr(), body.numel(), n, 33, ev.data_ptr(),
                              n * W.CAP, 0, stream_base=s0)
    return ne, w


def _rank_main(rank, world, port, shape, total, q):
    import sys
    sys.path.insert(0, ROOT)
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    import torch
    import torch.distributed as dist
    import bench
    from paper_2505_21661_b200 import shard
    from paper_2505_21661_b200 import trace as T
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        plan, n_long = _setup(shape, total)
        ctx = T.Context(0)
        merged = T.Context(0)
        ctx.set_plan(plan)
        merged.set_plan(plan)
        s0, s1 = shard.stream_range(total, 16, world, rank)
        ne, w = _replay_range(ctx, shape, s0, s1, n_long)
        pb = ctx.stats_packed_bytes()
        mine = torch.zeros(pb, dtype=torch.uint8, device="cuda")
        ctx.stats_export(mine.data_ptr())
        host = mine.cpu()
        gathered = torch.empty(pb * world, dtype=torch.uint8)
        dist.all_gather_into_tensor(gathered, host)
        dg = gathered.cuda()
        merged.stats_merge(dg.data_ptr(), world)
        out = torch.zeros(pb, dtype=torch.uint8, device="cuda")
        merged.stats_export(out.data_ptr())
        torch.cuda.synchronize()
        q.put((rank, (out.cpu().numpy().tobytes(), bench.stats_digest(merged.stats()),
                      ne, (w.dropped_heads, w.truncated_tails,
                           w.flagged_preconditions, w.malformed_groups))))
    finally:
        dist.destroy_process_group()


def _run_world(world, shape, total):
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_rank_main, args=(r, world, port, shape, total, q))
             for r in range(world)]
    for p in procs:
        p.start()
    res = {}
    for _ in range(world):
        try:
            k, v = q.get(timeout=300)
        except queue.Empty:
            break
        res[k] = v
    for p in procs:
        p.join(timeout=60)
        if p.is_alive():
            p.kill()
        assert p.exitcode == 0
    assert len(res) == world
    return res


@pytest.mark.parametrize("shape,total", [(0, 16 * 1024), (0, 16 * 101),
                                         (1, 16 * 256)])
def test_two_process_export_merge_equals_single_shot(shape, total):
    import torch
    import bench
    from paper_2505_21661_b200 import trace as T
    res = _run_world(2, shape, total)
    # single shot: the whole trace in one replay
    plan, n_long = _setup(shape, total)
    ctx = T.Context(0)
    ctx.set_plan(plan)
    ne, w = _replay_range(ctx, shape, 0, total, n_long)
    pb = ctx.stats_packed_bytes()
    one = torch.zeros(pb, dtype=torch.uint8, device="cuda")
    ctx.stats_export(one.data_ptr())
    torch.cuda.synchronize()
    single = one.cpu().numpy().tobytes()
    for r in range(2):
        packed, digest, _, _ = res[r]
        assert packed == single, f"rank {r}: merged table != single-shot table"
        assert digest == bench.stats_digest(ctx.stats())
    # events and warnings are sums over the shards
    assert res[0][2] + res[1][2] == ne
    ws = tuple(a + b for a, b in zip(res[0][3], res[1][3]))
    assert ws == (w.dropped_heads, w.truncated_tails, w.flagged_preconditions,
                  w.malformed_groups)


def test_bench_refuses_more_gpus_than_the_box_has():
    """--gpus N on a box with fewer GPUs fails loudly (non-zero exit)."""
    import subprocess
    import sys
    import torch
    n = torch.cuda.device_count() + 1
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus",
                        str(n), "--steps", "1", "--warmup", "0", "--streams", "1024",
                        "--no-e2e", "--no-cpu-baseline", "--no-p1", "--no-config5"],
                       capture_output=True, text=True, timeout=600)
    assert r.returncode != 0
    assert "cannot run here" in (r.stdout + r.stderr)


def test_allreduce_stats_over_nccl_single_rank():
    """wgpf_allreduce_stats (export -> ncclAllGather -> merge) on a one-rank
    NCCL communicator made through libnccl directly (no torch): the C-ABI's
    own collective runs and leaves the statistics unchanged."""
    import ctypes as C
    import torch
    from paper_2505_21661_b200 import trace as T
    from paper_2505_21661_b200 import workloads as W
    torch.cuda.set_device(0)
    nccl = C.CDLL("libnccl.so.2", mode=C.RTLD_GLOBAL)

    class UniqueId(C.Structure):
        _fields_ = [("internal", C.c_char * 128)]
    uid = UniqueId()
    assert nccl.ncclGetUniqueId(C.byref(uid)) == 0
    comm = C.c_void_p()
    assert nccl.ncclCommInitRank(C.byref(comm), 1, uid, 0) == 0
    try:
        plan, n_long = _setup(W.MIXED, 4096)
        ctx = T.Context(0)
        ctx.set_plan(plan)
        _replay_range(ctx, W.MIXED, 0, 4096, n_long)
        pb = ctx.stats_packed_bytes()
        before = torch.zeros(pb, dtype=torch.uint8, device="cuda")
        ctx.stats_export(before.data_ptr())
        torch.cuda.synchronize()
        b = before.cpu().numpy().tobytes()
        st0 = ctx.stats()
        ctx.allreduce_stats(comm.value)
        after = torch.zeros(pb, dtype=torch.uint8, device="cuda")
        ctx.stats_export(after.data_ptr())
        torch.cuda.synchronize()
        assert after.cpu().numpy().tobytes() == b
        st1 = ctx.stats()
        assert {k: (v.count, v.sum, v.min, v.max, v.hist) for k, v in st0.items()} == \
            {k: (v.count, v.sum, v.min, v.max, v.hist) for k, v in st1.items()}
    finally:
        nccl.ncclCommDestroy(comm)


@pytest.mark.parametrize("ranks", [2, 4, 8])
def test_bench_ranks_on_one_gpu_match_one_rank(ranks):
    """The N > 1 path of bench.py itself (self-launch under torchrun, block-
    range shards of one trace, per-step export / all-gather / merge, max-over-
    ranks timing, rank 0's line) on a one-GPU box: WGPF_BENCH_SHARE_GPU=1 puts
    all N ranks on cuda:0 over gloo (host-staged collective, the test mode --
    NCCL cannot share a device).  The merged statistics digest must equal the
    single-rank run's on the same trace."""
    import json
    import subprocess
    import sys
    base = [sys.executable, os.path.join(ROOT, "bench.py"), "--steps", "2", "--warmup", "3",
            "--no-e2e", "--no-cpu-baseline", "--no-p1", "--no-config5", "--streams", "65536"]
    env = dict(os.environ, WGPF_BENCH_SHARE_GPU="1")
    one = subprocess.run(base + ["--gpus", "1"], capture_output=True, text=True, timeout=600,
                         env=env)
    two = subprocess.run(base + ["--gpus", str(ranks)], capture_output=True, text=True,
                         timeout=900, env=env)
    assert one.returncode == 0, one.stderr[-2000:]
    assert two.returncode == 0, two.stderr[-2000:]
    l1 = json.loads([l for l in one.stdout.splitlines() if l.startswith("{")][-1])
    l2 = json.loads([l for l in two.stdout.splitlines() if l.startswith("{")][-1])
    assert l1["n_gpus"] == 1 and l2["n_gpus"] == ranks
    assert l2["config"]["streams_total"] == l1["config"]["streams_total"] == 65536
    assert l2["config"]["streams_per_gpu_rank0"] == 65536 // ranks
    assert l2["stats_digest"] == l1["stats_digest"]
    assert l2["nccl"]["collectives_per_step"] == 1
