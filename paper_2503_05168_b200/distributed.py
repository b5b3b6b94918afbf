"""Frame-sharded trajectory rendering over the GPUs of one node.

The scene (and its cluster table) is replicated on every GPU -- 3M splats are
~0.7 GB of 180 GB HBM -- and a camera trajectory shards by frame:
frame f goes to rank f mod N.  No scene data crosses
GPUs; the only collective is an optional gather of the rendered frames
(uint8, quantised like io.quantize_image, io.py:428-434) and of each frame's
FrameStats counters to rank 0 over NCCL / NVLink.  One process per GPU,
``torch.distributed`` for the plumbing; the render itself is the
single-GPU path.
"""
from __future__ import annotations

from dataclasses import dataclass, field
from typing import Callable, Sequence

import numpy as np
import torch
import torch.distributed as dist

from . import _native


def frames_for_rank(rank: int, world: int, n_frames: int, steps: int | None = None) -> list[int]:
    """Frames of a trajectory owned by ``rank``: f = rank + world * k.

    With ``steps`` the trajectory wraps around (k < steps), so every rank
    renders exactly ``steps`` frames (weak scaling)."""
    if not 0 <= rank < world:
        raise ValueError(f"rank {rank} outside world of {world}")
    if steps is None:
        return list(range(rank, n_frames, world))
    return [(rank + world * k) % n_frames for k in range(steps)]


def quantize(image: torch.Tensor) -> torch.Tensor:
    """io.quantize_image on the device: clamp to [0, 1], x 255, round half up."""
    return torch.floor(image.clamp(0.0, 1.0) * 255.0 + 0.5).to(torch.uint8)


@dataclass
class ShardedResult:
    frames: list[int]                           # frames rendered by this rank
    stats: np.ndarray                           # [len(frames), STAT_COUNT] int64 device counters
    gathered_frames: list[int] | None = None     # rank 0: every frame index, in trajectory order
    gathered_images: np.ndarray | None = None    # rank 0: [F, H, W, 3] uint8
    gathered_stats: np.ndarray | None = None     # rank 0: [F, STAT_COUNT]
    extras: dict = field(default_factory=dict)


def render_trajectory(render_one: Callable[[int], tuple[torch.Tensor, torch.Tensor]], n_frames: int,
                      *, gather: bool = False, device=None, group=None, to_host: bool = True) -> ShardedResult:
    """Render this rank's share of an ``n_frames`` trajectory.

    ``render_one(f) -> (image [H,W,3] float32, stats [STAT_COUNT] int64)`` renders
    frame f on this rank's device (e.g. ResidentRenderer.render_device), without
    host synchronisation.  Each frame is quantised on the device into a
    preallocated [rounds, H, W, 3] uint8 buffer (rounds = ceil(n_frames / world);
    ranks with fewer frames leave zero padding and stats rows of -1).  With
    ``gather`` ONE all_gather_into_tensor of the images and one of the stats
    (NCCL over NVLink, or gloo) assemble every frame on every rank, in
    trajectory order: row r * world + src holds frame r * world + src.  There
    is no per-frame host copy; with ``to_host`` the results are read back once
    at the end (rank 0 for the gathered set).
    """
    rank = dist.get_rank(group) if dist.is_initialized() else 0
    world = dist.get_world_size(group) if dist.is_initialized() else 1
    mine = frames_for_rank(rank, world, n_frames)
    rounds = -(-n_frames // world)
    imgs = sts = None
    dev = torch.device(device) if device is not None else None
    for r, f in enumerate(mine):
        img, st = render_one(f)
        if imgs is None:
            dev = dev or img.device
            imgs = torch.zeros((rounds,) + tuple(img.shape), dtype=torch.uint8, device=dev)
            sts = torch.full((rounds, _native.STAT_COUNT), -1, dtype=torch.int64, device=dev)
        imgs[r].copy_(quantize(img))
        sts[r].copy_(st)
    if dev is None:  # this rank rendered nothing: the collective still needs a device
        if dist.is_initialized() and dist.get_backend(group) == "nccl":
            dev = torch.device("cuda", torch.cuda.current_device())
        else:
            dev = torch.device("cpu")
    local_stats = sts[:len(mine)] if sts is not None else torch.zeros((0, _native.STAT_COUNT), dtype=torch.int64)
    out = ShardedResult(frames=mine, stats=local_stats.cpu().numpy() if to_host else local_stats)
    if not gather:
        return out
    if world > 1:
        shape_t = torch.tensor(list(imgs.shape[1:]) if imgs is not None else [0, 0, 0], dtype=torch.int64,
                               device=dev)
        dist.all_reduce(shape_t, op=dist.ReduceOp.MAX, group=group)
        shape = tuple(int(v) for v in shape_t.tolist())
        if imgs is None:
            imgs = torch.zeros((rounds,) + shape, dtype=torch.uint8, device=dev)
            sts = torch.full((rounds, _native.STAT_COUNT), -1, dtype=torch.int64, device=dev)
        all_imgs = torch.empty((world * rounds,) + shape, dtype=torch.uint8, device=dev)
        all_sts = torch.empty((world * rounds, _native.STAT_COUNT), dtype=torch.int64, device=dev)
        dist.all_gather_into_tensor(all_imgs, imgs, group=group)
        dist.all_gather_into_tensor(all_sts, sts, group=group)
        # [src, round] -> frame round * world + src
        all_imgs = all_imgs.view((world, rounds) + shape).transpose(0, 1).reshape((world * rounds,) + shape)
        all_sts = all_sts.view(world, rounds, -1).transpose(0, 1).reshape(world * rounds, -1)
    else:
        all_imgs, all_sts = imgs, sts
    out.extras["device_images"] = all_imgs[:n_frames] if all_imgs is not None else None
    out.extras["device_stats"] = all_sts[:n_frames] if all_sts is not None else None
    if rank == 0:
        out.gathered_frames = list(range(n_frames))
        if to_host:
            out.gathered_images = all_imgs[:n_frames].cpu().numpy() if all_imgs is not None else None
            out.gathered_stats = all_sts[:n_frames].cpu().numpy() if all_sts is not None else None
    return out


def shard_summary(frame_counts: Sequence[int]) -> dict:
    """Load balance of a frame sharding (max / mean frames per rank)."""
    arr = np.asarray(frame_counts, dtype=np.float64)
    return {"ranks": len(arr), "max": int(arr.max()), "mean": float(arr.mean()),
            "imbalance": float(arr.max() / arr.mean()) if arr.mean() else 0.0}
