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


def fit_frames_sharded(depth, intrinsics, window: int, formulations=None, devices=None, chunk_frames: int = 8):
    """Fit a host batch of frames across several GPUs of this process: contiguous frame ranges
    (frame_range) per device, each streamed through its own HostPipeline (H2D, tile kernels,
    D2H on its own streams and PCIe link) from its own host thread, straight into one pinned
    host output per formulation.  No collective: frames are independent.

    depth: host tensor [B, H, W] (float32 / float64 metres or uint16 mm); intrinsics: the
    camera (CameraIntrinsics); devices: CUDA device indices (default: every visible device; a
    device may repeat).  Returns {formulation: PixelFits} of pinned host tensors."""
    import threading

    from .pixels import PIXEL_FORMULATIONS, HostPipeline, PixelFits, compute_tan_maps

    formulations = PIXEL_FORMULATIONS if formulations is None else (
        (formulations,) if isinstance(formulations, str) else tuple(formulations))
    if depth.is_cuda or depth.dim() != 3:
        raise ValueError("fit_frames_sharded takes a host batch [B, H, W]")
    devices = list(range(torch.cuda.device_count())) if devices is None else [int(d) for d in devices]
    if not devices:
        raise ValueError("no CUDA device to shard over (the sm_100a path has no CPU fallback)")
    B, H, W = depth.shape
    pin = dict(pin_memory=True)
    out = {f: PixelFits(torch.empty((B, H, W, 3), **pin), torch.empty((B, H, W), **pin),
                        torch.empty((B, H, W), **pin), torch.empty((B, H, W), **pin),
                        torch.empty((B, H, W), dtype=torch.uint8, **pin)) for f in formulations}
    src = depth.contiguous()
    errors = []

    def work(rank: int, dev: int):
        try:
            start, stop = frame_range(B, len(devices), rank)
            if stop == start:
                return
            with torch.cuda.device(dev):
                maps = compute_tan_maps(intrinsics, dev)
                pipe = HostPipeline(maps, window, formulations, chunk_frames=chunk_frames)
                view = {f: PixelFits(*(getattr(out[f], k)[start:stop] for k in
                                       ("normal", "offset", "residual", "curvature", "status")))
                        for f in formulations}
                pipe.run(src[start:stop], out=view)
        except BaseException as e:  # surfaced in the caller's thread
            errors.append(e)

    threads = [threading.Thread(target=work, args=(k, d)) for k, d in enumerate(devices)]
    for t in threads:
        t.start()
    for t in threads:
        t.join()
    if errors:
        raise errors[0]
    return out
