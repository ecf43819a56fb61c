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


def max_over_ranks(value: float, device, group=None) -> float:
    """The slowest rank's value (bench.py: the step time is the max over ranks)."""
    if not dist.is_initialized() or dist.get_world_size(group) == 1:
        return float(value)
    t = torch.tensor([float(value)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX, group=group)
    return float(t.item())


def rank_table(fields: list[float], device, group=None) -> list[list[float]]:
    """Every rank's row of numbers (rank, tokens, ms, ...), gathered to all ranks."""
    mine = torch.tensor([float(f) for f in fields], dtype=torch.float64, device=device)
    if not dist.is_initialized() or dist.get_world_size(group) == 1:
        return [mine.tolist()]
    rows = [torch.empty_like(mine) for _ in range(dist.get_world_size(group))]
    dist.all_gather(rows, mine, group=group)
    return [r.tolist() for r in rows]


def verify_gather(local: torch.Tensor, total_rows: int, recompute_last, group=None) -> bool:
    """Untimed multi-GPU check: all-gather every rank's output rows and compare, bit for bit,
    (a) each rank's own block of the gathered tensor with what it computed and (b) on rank 0 the
    LAST rank's block with rank 0's own recompute of that shard (`recompute_last(lo, hi)` returns
    the rows [lo, hi) computed locally).  All ranks get the same verdict."""
    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    full = gather_rows(local, total_rows, group=group)
    lo, hi = shard_range(total_rows, rank, world)
    ok = bool(torch.equal(full[lo:hi], local))
    if rank == 0:
        rlo, rhi = shard_range(total_rows, world - 1, world)
        ok = ok and bool(torch.equal(full[rlo:rhi], recompute_last(rlo, rhi)))
    flag = torch.tensor([1 if ok else 0], dtype=torch.int32, device=local.device)
    dist.all_reduce(flag, op=dist.ReduceOp.MIN, group=group)
    return bool(flag.item() == 1)
