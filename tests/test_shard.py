"""Multi-rank host logic on CPU (gloo, world size 2): frame sharding covers a
batch exactly once, per-rank seeds are distinct, and the timing reduction is
the max over ranks -- the N>1 path of bench.py without a GPU."""

from __future__ import annotations

import os
import socket

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2103_06644_b200.shard import frame_range, max_over_ranks, rank_seed_base


def test_frame_range_partition():
    for total in (0, 1, 7, 64, 1024, 1025):
        for world in (1, 2, 3, 4, 8):
            ranges = [frame_range(total, world, r) for r in range(world)]
            covered = [f for a, b in ranges for f in range(a, b)]
            assert covered == list(range(total))
            sizes = [b - a for a, b in ranges]
            assert max(sizes) - min(sizes) <= 1
    with pytest.raises(ValueError):
        frame_range(10, 2, 2)


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        start, stop = frame_range(64, world, rank)
        mine = torch.zeros(64, dtype=torch.int64)
        mine[start:stop] = 1
        dist.all_reduce(mine)
        seeds = torch.tensor([rank_seed_base(2, rank)], dtype=torch.int64)
        all_seeds = [torch.zeros(1, dtype=torch.int64) for _ in range(world)]
        dist.all_gather(all_seeds, seeds)
        elapsed = 10.0 + 5.0 * rank  # per-rank "device time"
        dist.barrier()
        worst = max_over_ranks(elapsed, world)
        q.put((rank, mine.tolist(), [int(s) for s in all_seeds], worst))
    finally:
        dist.destroy_process_group()


def test_gloo_world2_sharding_and_max_timing():
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    results = [q.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for rank, mine, seeds, worst in results:
        assert mine == [1] * 64              # every frame fitted exactly once
        assert len(set(seeds)) == world      # weak scaling: distinct per-rank batches
        assert worst == 15.0                 # max over ranks
