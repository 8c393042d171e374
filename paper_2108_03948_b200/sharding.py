"""Batch sharding across ranks (one process per GPU).

Every trace is independent: FFT, CZT and zoom have no cross-trace coupling and the
only shared state (plan tables, X_ref) is read-only and rebuilt on each device. A batch is split
into contiguous row blocks, one per rank, with no data-path collective. `gather_rows` is the
optional final collect of results on every rank (NCCL over NVLink on the GPU box, gloo in the CPU
tests); it is not part of the timed hot path.
"""
from __future__ import annotations


def shard_bounds(batch: int, rank: int, world: int) -> tuple[int, int]:
    """[begin, end) rows of `batch` owned by `rank`; sizes differ by at most one row."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError(f"bad rank {rank} for world {world}")
    q, r = divmod(batch, world)
    begin = rank * q + min(rank, r)
    return begin, begin + q + (1 if rank < r else 0)


def gather_rows(local, batch: int, group=None):
    """All-gather the per-rank row blocks (torch tensors, rank order) into the full batch."""
    import torch
    import torch.distributed as dist
    world = dist.get_world_size(group)
    sizes = [shard_bounds(batch, r, world) for r in range(world)]
    width = max(e - b for b, e in sizes)
    pad = torch.zeros((width,) + tuple(local.shape[1:]), dtype=local.dtype, device=local.device)
    pad[: local.shape[0]] = local
    parts = [torch.empty_like(pad) for _ in range(world)]
    dist.all_gather(parts, pad, group=group)
    return torch.cat([p[: e - b] for p, (b, e) in zip(parts, sizes)])
