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
                      *, gather: bool = False, device=None, group=None) -> ShardedResult:
    """Render this rank's share of an ``n_frames`` trajectory.

    ``render_one(f) -> (image [H,W,3] float32, stats [STAT_COUNT] int64)`` renders
    frame f on this rank's device (e.g. ResidentRenderer.render_device).  With
    ``gather`` the quantised images and the stats of every frame are collected
    on rank 0 in trajectory order (one all_gather of fixed-size buffers per
    round of frames; ranks with fewer frames contribute padding).
    """
    rank = dist.get_rank(group) if dist.is_initialized() else 0
    world = dist.get_world_size(group) if dist.is_initialized() else 1
    mine = frames_for_rank(rank, world, n_frames)
    stats, images = [], []
    for f in mine:
        img, st = render_one(f)
        stats.append(st.detach().to("cpu", torch.int64).numpy().copy())
        if gather:
            images.append(quantize(img))
    out = ShardedResult(frames=mine, stats=np.stack(stats) if stats else np.zeros((0, _native.STAT_COUNT), np.int64))
    if not gather:
        return out
    if world == 1:
        out.gathered_frames = list(mine)
        out.gathered_images = torch.stack(images).cpu().numpy() if images else None
        out.gathered_stats = out.stats
        return out
    rounds = -(-n_frames // world)
    shape = images[0].shape if images else None
    shape_t = torch.tensor(list(shape) if shape else [0, 0, 0], dtype=torch.int64, device=device)
    dist.all_reduce(shape_t, op=dist.ReduceOp.MAX, group=group)
    h, w, c = (int(v) for v in shape_t.tolist())
    all_imgs, all_stats, order = [], [], []
    for r in range(rounds):
        f_local = r * world + rank
        has = f_local < n_frames
        img = images[r] if has else torch.zeros((h, w, c), dtype=torch.uint8, device=device)
        st = torch.as_tensor(out.stats[r] if has else np.full(_native.STAT_COUNT, -1, np.int64), device=device)
        imgs = [torch.empty_like(img) for _ in range(world)]
        sts = [torch.empty_like(st) for _ in range(world)]
        dist.all_gather(imgs, img.contiguous(), group=group)
        dist.all_gather(sts, st.contiguous(), group=group)
        if rank == 0:
            for src in range(world):
                f = r * world + src
                if f < n_frames:
                    order.append(f)
                    all_imgs.append(imgs[src].cpu().numpy())
                    all_stats.append(sts[src].cpu().numpy())
    if rank == 0:
        out.gathered_frames = order
        out.gathered_images = np.stack(all_imgs)
        out.gathered_stats = np.stack(all_stats)
    return out


def shard_summary(frame_counts: Sequence[int]) -> dict:
    """Load balance of a frame sharding (max / mean frames per rank)."""
    arr = np.asarray(frame_counts, dtype=np.float64)
    return {"ranks": len(arr), "max": int(arr.max()), "mean": float(arr.mean()),
            "imbalance": float(arr.max() / arr.mean()) if arr.mean() else 0.0}
