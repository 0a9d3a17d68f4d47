"""CPU tests of the multi-GPU path with torch.distributed / gloo, world 2.

Each rank takes its block range of a synthetic trace (shard.stream_range),
computes its per-label table with the CPU oracle in the packed layout that
wgpf_stats_export produces (70 u64 per label: count, sum, min, max, first key,
first warp group, 64 bins), the ranks all-gather the tables (the one
collective), and the merge rule of wgpf_stats_merge (add / min / max /
first-key min with its warp group) must reproduce the single-process table;
the role-overlap counters all-reduced across ranks (shard.allreduce_overlap)
must equal the whole trace's.
"""
import os
import socket

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

WORDS = 70


def pack_table(stats, labels, stream_base, offsets_of_stream):
    """Oracle stats -> packed rows in label-table order (dense classes)."""
    rows = np.zeros((len(labels), WORDS), np.uint64)
    idx = {l: i for i, l in enumerate(labels)}
    for s in stats:
        r = rows[idx[s.label]]
        r[0], r[1], r[2], r[3] = s.count, s.sum, s.min, s.max
        gs, k = offsets_of_stream(s.first_event)
        r[4] = ((stream_base + gs) << 25) | (k << 1) | (1 if s.kind == "wait" else 0)
        r[5] = s.warp_group
        r[6:] = np.array(s.hist, np.uint64)
    return rows


def merge_tables(tables):
    """The wgpf_stats_merge rule (csrc/k_stats.cuh k_stats_merge*)."""
    out = np.zeros_like(tables[0])
    out[:, 2] = np.iinfo(np.uint64).max
    out[:, 4] = np.iinfo(np.uint64).max
    for t in tables:
        live = t[:, 0] > 0
        out[live, 0] += t[live, 0]
        out[live, 1] += t[live, 1]
        out[live, 2] = np.minimum(out[live, 2], t[live, 2])
        out[live, 3] = np.maximum(out[live, 3], t[live, 3])
        out[live, 6:] += t[live, 6:]
        better = live & (t[:, 4] < out[:, 4])
        out[better, 4] = t[better, 4]
        out[better, 5] = t[better, 5]
    return out


def _rank_main(rank, world, port, n_streams, q):
    import sys
    sys.path.insert(0, ROOT)
    import torch
    import torch.distributed as dist
    from oracle import oracle as O
    from oracle import synth as S
    from paper_2505_21661_b200 import shard
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        s0, s1 = shard.stream_range(n_streams, 16, world, rank)
        body = S.mixed_body(s0, s1 - s0, S.MIXED_FULL_LONG - n_streams // 3)
        orc = O.Oracle()
        r = orc.replay_body(body, s1 - s0, S.CAP, 1, S.MIXED_LABELS, 33)
        # event index -> (local stream, index in stream)
        per_stream = []
        stride = S.stream_stride()
        cnt = np.zeros(s1 - s0, np.int64)
        for s in range(s1 - s0):
            one = body[s * stride:(s + 1) * stride]
            cnt[s] = len(orc.replay_body(one, 1, S.CAP, 1, S.MIXED_LABELS, 33).events)
        starts = np.concatenate([[0], np.cumsum(cnt)])

        def locate(e):
            s = int(np.searchsorted(starts, e, side="right") - 1)
            return s, int(e - starts[s])
        del per_stream
        st = orc.region_stats(r.events, S.MIXED_LABELS)
        mine = torch.from_numpy(pack_table(st, S.MIXED_LABELS, s0, locate).view(np.int64))
        out = torch.empty((world * mine.shape[0], mine.shape[1]), dtype=torch.int64)
        dist.all_gather_into_tensor(out, mine)
        tables = [t.numpy().view(np.uint64) for t in out.chunk(world)]
        merged = merge_tables(tables)
        # role-overlap counters: per-rank counters, one all-reduce (sum)
        roles = [0] * 4 + [1] * 12
        ov = shard.allreduce_overlap(orc.overlap(r.events, roles), dist, device="cpu")
        q.put((rank, (merged, ov)))
    finally:
        dist.destroy_process_group()


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def test_block_ranges_partition():
    from paper_2505_21661_b200 import shard
    for n_blocks in (1, 7, 303104):
        for world in (1, 2, 3, 8):
            rs = [shard.block_range(n_blocks, world, r) for r in range(world)]
            assert rs[0][0] == 0 and rs[-1][1] == n_blocks
            assert all(rs[i][1] == rs[i + 1][0] for i in range(world - 1))
            sizes = [b - a for a, b in rs]
            assert max(sizes) - min(sizes) <= 1


def test_gloo_world2_shard_and_merge_equals_single(oracle):
    import torch.multiprocessing as mp
    from oracle import synth as S
    n_streams = 1600
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_rank_main, args=(r, 2, port, n_streams, q))
             for r in range(2)]
    for p in procs:
        p.start()
    import queue
    res = {}
    for _ in range(2):
        try:
            k, v = q.get(timeout=180)
        except queue.Empty:
            break
        res[k] = v
    for p in procs:
        p.join(timeout=60)
        if p.is_alive():
            p.kill()
        assert p.exitcode == 0
    assert len(res) == 2
    assert np.array_equal(res[0][0], res[1][0])
    assert res[0][1] == res[1][1]
    ov_all = oracle.overlap(
        oracle.replay_body(S.mixed_body(0, n_streams, S.MIXED_FULL_LONG - n_streams // 3),
                           n_streams, S.CAP, 1, S.MIXED_LABELS, 33).events,
        [0] * 4 + [1] * 12)
    assert res[0][1] == ov_all
    res = {k: v[0] for k, v in res.items()}
    # single process, whole trace
    body = S.mixed_body(0, n_streams, S.MIXED_FULL_LONG - n_streams // 3)
    r = oracle.replay_body(body, n_streams, S.CAP, 1, S.MIXED_LABELS, 33)
    st = {s.label: s for s in oracle.region_stats(r.events, S.MIXED_LABELS)}
    for i, label in enumerate(S.MIXED_LABELS):
        row = res[0][i]
        s = st[label]
        assert (int(row[0]), int(row[1]), int(row[2]), int(row[3])) == (
            s.count, s.sum, s.min, s.max)
        assert [int(x) for x in row[6:]] == s.hist
        assert int(row[5]) == s.warp_group
        assert int(row[4]) & 1 == (1 if s.kind == "wait" else 0)


def test_bench_self_launches_ranks_for_the_reference_arm():
    """bench.py --gpus 2 outside torchrun re-launches itself with 2 ranks
    (torch.distributed.run); rank 0 alone runs the reference arm and prints
    the one JSON line, the other rank exits 0."""
    import json
    import subprocess
    import sys
    from oracle import oracle as O
    if not O.have_ref():
        pytest.skip("oracle/_ref not built")
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl",
                        "reference", "--gpus", "2", "--steps", "1", "--warmup", "0",
                        "--ref-budget-s", "0.1"],
                       capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [l for l in r.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    assert d["impl"] == "reference" and d["n_gpus"] == 2 and d["value"] > 0
    cb = d["cpu_baseline"]
    assert cb["single_core"]["cores"] == 1 and cb["nproc"] >= 1 and cb["cpu_model"]
    # whole rounds of equal chunks: no half-idle last wave
    assert d["config"]["sample_streams"] % cb["cores"] == 0


def test_bench_world_size_mismatch_fails():
    import subprocess
    import sys
    env = dict(os.environ, WORLD_SIZE="1", RANK="0", LOCAL_RANK="0")
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "2"],
                       capture_output=True, text=True, timeout=120, env=env)
    assert r.returncode == 2 and "WORLD_SIZE=1" in r.stderr
