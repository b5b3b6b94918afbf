"""Frame sharding across ranks (host logic) with the gloo backend, world size 2.

The render call is a deterministic stand-in: these tests cover the sharding
and the gather (no GPU here); the per-frame render path is covered by the GPU
parity tests."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2503_05168_b200 import _native
from paper_2503_05168_b200.distributed import frames_for_rank, quantize, render_trajectory, shard_summary


def test_frames_partition_trajectory():
    for world in (1, 2, 3, 4, 8):
        got = sorted(f for r in range(world) for f in frames_for_rank(r, world, 120))
        assert got == list(range(120))
        counts = [len(frames_for_rank(r, world, 120)) for r in range(world)]
        assert shard_summary(counts)["imbalance"] <= 1.1
    assert frames_for_rank(1, 4, 120, steps=5) == [1, 5, 9, 13, 17]
    assert frames_for_rank(3, 8, 120, steps=16)[-1] == (3 + 8 * 15) % 120
    with pytest.raises(ValueError):
        frames_for_rank(2, 2, 10)


def test_quantize_matches_reference_rule():
    x = torch.tensor([-0.5, 0.0, 0.5 / 255.0, 1.0 / 255.0, 0.5, 1.0, 2.0])
    want = np.floor(np.clip(x.numpy().astype(np.float64), 0, 1) * 255 + 0.5).astype(np.uint8)
    assert quantize(x).numpy().tolist() == want.tolist()


def _fake_render(f: int):
    img = torch.full((4, 6, 3), (f % 7) / 7.0, dtype=torch.float32)
    st = torch.arange(_native.STAT_COUNT, dtype=torch.int64) + 1000 * f
    return img, st


def _worker(rank, world, port, n_frames, out_path):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        res = render_trajectory(_fake_render, n_frames, gather=True)
        assert res.frames == frames_for_rank(rank, world, n_frames)
        if rank == 0:
            np.savez(out_path, frames=np.array(res.gathered_frames), images=res.gathered_images,
                     stats=res.gathered_stats)
        dist.barrier()
    finally:
        dist.destroy_process_group()


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


@pytest.mark.parametrize("n_frames", [10, 9])
def test_gather_world2_gloo(tmp_path, n_frames):
    out = tmp_path / "gathered.npz"
    mp.spawn(_worker, args=(2, _free_port(), n_frames, str(out)), nprocs=2, join=True)
    z = np.load(out)
    assert z["frames"].tolist() == list(range(n_frames))
    for k, f in enumerate(z["frames"]):
        img, st = _fake_render(int(f))
        np.testing.assert_array_equal(z["images"][k], quantize(img).numpy())
        np.testing.assert_array_equal(z["stats"][k], st.numpy())
