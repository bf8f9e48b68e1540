"""Host-side multi-GPU plumbing: column sharding with no data-path collective.

Every detector column is an independent filter instance (one partition = one
column), so a flightline [cols][pixels][bands] is
split into contiguous column ranges, one per rank; each rank runs smf_retrieve
on its slice (a contiguous sub-array of the cube, no copy) and writes its
slice of enhancement / albedo. The only communication is the optional gather
of the results for a caller that wants the whole map on one rank -- never part
of the retrieval itself.
"""
from __future__ import annotations


def column_range(cols: int, rank: int, world: int) -> tuple[int, int]:
    """Contiguous, balanced [start, stop) column range of `rank` (sizes differ by <= 1;
    lower ranks take the extra columns)."""
    if cols < 0 or world < 1 or not 0 <= rank < world:
        raise ValueError(f"bad shard request cols={cols} rank={rank} world={world}")
    base, extra = divmod(cols, world)
    start = rank * base + min(rank, extra)
    return start, start + base + (1 if rank < extra else 0)


def all_ranges(cols: int, world: int) -> list[tuple[int, int]]:
    return [column_range(cols, r, world) for r in range(world)]


def gather_columns(local, cols: int, group=None):
    """Gather per-rank column slices (torch tensors [local_cols][...], same trailing
    shape and dtype on every rank) into the full [cols][...] tensor on every rank.
    Uses torch.distributed all_gather on equal-size padded buffers (gloo or nccl)."""
    import torch
    import torch.distributed as dist
    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    ranges = all_ranges(cols, world)
    lo, hi = ranges[rank]
    if local.shape[0] != hi - lo:
        raise ValueError(f"rank {rank}: local slice has {local.shape[0]} columns, expected {hi - lo}")
    width = max(h - l for l, h in ranges)
    pad = torch.zeros((width,) + tuple(local.shape[1:]), dtype=local.dtype, device=local.device)
    pad[: hi - lo] = local
    bufs = [torch.empty_like(pad) for _ in range(world)]
    dist.all_gather(bufs, pad, group=group)
    return torch.cat([b[: h - l] for b, (l, h) in zip(bufs, ranges)], dim=0)
