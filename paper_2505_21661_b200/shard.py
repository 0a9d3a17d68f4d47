"""Multi-GPU shard-and-reduce for replay_image.

Streams (one per (block, warp)) are independent through decode / pair /
replay (pipeline.hpp:69-80), so each rank owns a contiguous range of blocks
-- every CTA's warps stay on one rank -- and decodes it with no data-path
communication.  The one exchange is the per-label statistics table: each rank
exports its packed table (wgpf_stats_export), one NCCL all-gather over NVLink
moves all tables to every rank, and wgpf_stats_merge combines them on the
device (sums / bins add, min / max, first-event key min with its warp group).
"""
from __future__ import annotations

PACKED_WORDS_PER_SLOT = 70  # count, sum, min, max, first, first_wg, hist[64]


def block_range(n_blocks: int, world: int, rank: int) -> tuple[int, int]:
    """Contiguous, balanced block range [b0, b1) of `rank`."""
    base, extra = divmod(n_blocks, world)
    b0 = rank * base + min(rank, extra)
    return b0, b0 + base + (1 if rank < extra else 0)


def stream_range(n_streams: int, streams_per_block: int, world: int,
                 rank: int) -> tuple[int, int]:
    """Streams of the rank's block range (stream s belongs to block
    s // streams_per_block)."""
    n_blocks = (n_streams + streams_per_block - 1) // streams_per_block
    b0, b1 = block_range(n_blocks, world, rank)
    return min(b0 * streams_per_block, n_streams), min(b1 * streams_per_block,
                                                      n_streams)


def allgather_merge(ctx, merged_ctx, dist, world: int, mine=None, gathered=None):
    """Exports ctx's statistics, all-gathers them (one collective) and merges
    them into merged_ctx.  `mine` / `gathered` are reusable device byte
    tensors of ctx.stats_packed_bytes() and world times that size."""
    import torch
    nbytes = ctx.stats_packed_bytes()
    if mine is None:
        mine = torch.empty(nbytes, dtype=torch.uint8, device="cuda")
    if gathered is None:
        gathered = torch.empty(nbytes * world, dtype=torch.uint8, device="cuda")
    ctx.stats_export(mine.data_ptr())
    dist.all_gather_into_tensor(gathered, mine)
    merged_ctx.stats_merge(gathered.data_ptr(), world)
    return merged_ctx.stats()


OVERLAP_FIELDS = ("blocks", "span", "busy0", "busy1", "both", "bubble0", "bubble1")


def allreduce_overlap(counters: dict, dist, device="cuda") -> dict:
    """Role-overlap counters (wgpf_overlap_counters) of every rank combined:
    they are sums over blocks, and blocks never straddle ranks (block-range
    shards), so one all-reduce (sum) gives the whole-trace counters."""
    import torch
    v = [counters["blocks"], counters["span"], counters["busy"][0], counters["busy"][1],
         counters["both"], counters["bubble"][0], counters["bubble"][1]]
    t = torch.tensor(v, dtype=torch.int64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.SUM)
    a = [int(x) for x in t.tolist()]
    return dict(blocks=a[0], span=a[1], busy=[a[2], a[3]], both=a[4], bubble=[a[5], a[6]])
