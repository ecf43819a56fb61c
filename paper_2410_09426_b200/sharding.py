"""Token (data) sharding of the hot path across GPUs -- SURVEY.md §8(e).

Every token is independent (per-token transform, per-token scale, GEMM rows), so the prefill
batch is split into contiguous token blocks, one per rank, with P1, P2, alpha, Q_w and s_w
replicated.  The timed path has no collective; `gather_rows` (an all-gather of the output
rows) exists only for verification.  The same logic runs on gloo (CPU tests) and NCCL.
"""
from __future__ import annotations

import torch
import torch.distributed as dist


def shard_range(T: int, rank: int, world: int) -> tuple[int, int]:
    """Contiguous block [lo, hi) of the T tokens owned by `rank` (sizes differ by <= 1)."""
    if world < 1 or not (0 <= rank < world) or T < 0:
        raise ValueError("bad shard arguments")
    base, extra = divmod(T, world)
    lo = rank * base + min(rank, extra)
    hi = lo + base + (1 if rank < extra else 0)
    return lo, hi


def gather_rows(local: torch.Tensor, T: int, group=None) -> torch.Tensor:
    """All-gather the per-rank row blocks produced by `shard_range` into the full [T, ...] tensor
    (verification only; handles uneven blocks by padding to the largest block)."""
    world = dist.get_world_size(group)
    sizes = [shard_range(T, r, world) for r in range(world)]
    maxrows = max(hi - lo for lo, hi in sizes)
    pad = torch.zeros((maxrows,) + tuple(local.shape[1:]), dtype=local.dtype, device=local.device)
    pad[: local.shape[0]] = local
    bufs = torch.empty((world * maxrows,) + tuple(local.shape[1:]), dtype=local.dtype, device=local.device)
    dist.all_gather_into_tensor(bufs, pad, group=group)
    parts = [bufs[r * maxrows: r * maxrows + (hi - lo)] for r, (lo, hi) in enumerate(sizes)]
    return torch.cat(parts, dim=0)
