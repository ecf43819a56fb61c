"""Multi-process (world size 2, gloo, CPU) tests of the token-sharding host logic
(DESIGN.md §9): the shard ranges partition the tokens, the verification
all-gather reassembles them in order (even and uneven splits), and the max-over-ranks
timing reduction bench.py uses picks the slowest rank.  The per-shard computation itself is
per-token independent, which the oracle pins below make explicit: transform+quant of a shard
equals the same rows of the full batch bit for bit."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle as O
import synth
from paper_2410_09426_b200.sharding import gather_rows, shard_range


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def test_shard_range_partitions_tokens():
    for T in [0, 1, 7, 2048, 32768, 32769]:
        for world in [1, 2, 3, 4, 8]:
            spans = [shard_range(T, r, world) for r in range(world)]
            assert spans[0][0] == 0 and spans[-1][1] == T
            for (a, b), (c, d) in zip(spans, spans[1:]):
                assert b == c
            sizes = [b - a for a, b in spans]
            assert max(sizes) - min(sizes) <= 1
    with pytest.raises(ValueError):
        shard_range(10, 2, 2)


def _worker(rank, world, port, T, results):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        lo, hi = shard_range(T, rank, world)
        full = torch.arange(T * 3, dtype=torch.int32).reshape(T, 3)
        local = full[lo:hi].clone()
        got = gather_rows(local, T)
        ok_gather = bool(torch.equal(got, full))
        # bench.py's max-over-ranks timing: the slowest rank's time wins
        t = torch.tensor([10.0 + rank])
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ok_max = float(t.item()) == 10.0 + world - 1
        # per-token independence of a1-a5 (oracle): shard rows == the same rows of the full batch
        x = synth.activations(T, 64, seed=5)
        p1 = synth.well_conditioned(8, seed=5, tag="p1")
        p2 = synth.well_conditioned(8, seed=5, tag="p2")
        q_full, s_full, _ = O.transform_quant(x, p1, p2, 0.9)
        q_sh, s_sh, _ = O.transform_quant(x[lo:hi], p1, p2, 0.9)
        ok_indep = bool(np.array_equal(q_full[lo:hi], q_sh) and np.array_equal(s_full[lo:hi], s_sh))
        # the gathered shard outputs equal the single-process result
        qg = gather_rows(torch.from_numpy(q_sh.astype(np.int8)), T).numpy()
        ok_gather_q = bool(np.array_equal(qg, q_full))
        results[rank] = (ok_gather, ok_max, ok_indep, ok_gather_q)
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("T", [64, 37])            # even and uneven splits
def test_gloo_world2_gather_and_timing(T):
    world = 2
    port = _free_port()
    with mp.Manager() as m:
        results = m.dict()
        mp.spawn(_worker, args=(world, port, T, results), nprocs=world, join=True)
        res = dict(results)
    assert sorted(res) == [0, 1]
    for r, flags in res.items():
        assert all(flags), f"rank {r}: {flags}"


def _bench_helpers_worker(rank, world, port, results):
    """bench.py's multi-GPU helpers on gloo: max over ranks, the per-rank table, and the gather
    verification (passes on correct shards, fails on a corrupted one, same verdict everywhere)."""
    from paper_2410_09426_b200 import sharding
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        dev = torch.device("cpu")
        T = 37
        full = torch.arange(T * 5, dtype=torch.float32).reshape(T, 5) * 0.5
        lo, hi = sharding.shard_range(T, rank, world)
        mx = sharding.max_over_ranks(3.0 + rank, dev)
        tab = sharding.rank_table([rank, hi - lo, 1.5 * rank], dev)
        good = sharding.verify_gather(full[lo:hi].clone(), T, lambda a, b: full[a:b].clone())
        bad_local = full[lo:hi].clone()
        if rank == world - 1:
            bad_local[0, 0] += 1.0                   # the last shard is wrong
        bad = sharding.verify_gather(bad_local, T, lambda a, b: full[a:b].clone())
        results[rank] = (mx == 3.0 + world - 1, [int(r[0]) for r in tab] == list(range(world)),
                         sum(int(r[1]) for r in tab) == T, good, not bad)
    finally:
        dist.destroy_process_group()


def test_gloo_world2_bench_helpers():
    world = 2
    port = _free_port()
    with mp.Manager() as m:
        results = m.dict()
        mp.spawn(_bench_helpers_worker, args=(world, port, results), nprocs=world, join=True)
        res = dict(results)
    assert sorted(res) == [0, 1]
    for r, flags in res.items():
        assert all(flags), f"rank {r}: {flags}"
