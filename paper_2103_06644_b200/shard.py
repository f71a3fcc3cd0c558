"""Frame sharding across ranks (one process per GPU).

Frames are independent, so the data path has no collective: each rank fits a
contiguous range of frames of a batch (strong sharding of a fixed batch, the
BASELINE C4/C5 setting) or its own batch (weak scaling, bench.py).  The only
collectives are the host-side barrier and the max-over-ranks reduction of the
measured time, both outside the data path.
"""

from __future__ import annotations

import torch


def frame_range(total: int, world: int, rank: int) -> tuple[int, int]:
    """Contiguous frame range [start, stop) of `rank`; sizes differ by at most one."""
    if world <= 0 or not (0 <= rank < world):
        raise ValueError(f"bad rank {rank} for world size {world}")
    if total < 0:
        raise ValueError(f"negative frame count {total}")
    base, extra = divmod(total, world)
    start = rank * base + min(rank, extra)
    return start, start + base + (1 if rank < extra else 0)


def rank_seed_base(config_index: int, rank: int) -> int:
    """Seed of frame 0 of a rank's own batch (weak scaling): 1000*config + 100000*rank."""
    return 1000 * int(config_index) + 100000 * int(rank)


def max_over_ranks(value: float, world: int, device: str | torch.device = "cpu") -> float:
    """Max of a per-rank scalar (e.g. elapsed ms) over all ranks."""
    if world == 1:
        return float(value)
    import torch.distributed as dist

    t = torch.tensor([float(value)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())
