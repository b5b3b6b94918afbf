"""Frame-sharded trajectory rendering with the real per-frame render, world
size 2: two processes share GPU 0 (one box has one GPU here),
each renders its frames f = rank + 2k of a clustered orbit through
ResidentRenderer.render_device, quantises them on the device, and the gloo
backend gathers every frame and its FrameStats counters on the host
(distributed.render_trajectory with device="cpu" buffers; NCCL needs one GPU
per rank).  Rank 0's gathered images and stats must equal a single-process
render of the whole trajectory."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu

N_FRAMES = 9  # odd: one rank renders one frame fewer (padding path)


def _setup():
    from paper_2503_05168_b200.clusters import build_cluster_table
    from paper_2503_05168_b200.container import container_from_table
    from paper_2503_05168_b200.synthetic import orbit, synth

    scene = synth(40_000, 3)
    poses = orbit(N_FRAMES, 256, 144)
    table = build_cluster_table(scene, poses, n_clusters=6, neighbors=1, beta=1.0, seed=0, device="cuda")
    return container_from_table(table, scene), poses


def _worker(rank, world, port, out_path):
    from paper_2503_05168_b200 import EngineConfig, FrameRenderer
    from paper_2503_05168_b200.distributed import render_trajectory
    from paper_2503_05168_b200.residency import ResidentRenderer

    torch.cuda.set_device(0)
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        container, poses = _setup()
        rr = ResidentRenderer(container, m=1)
        r = FrameRenderer()
        cfg = EngineConfig(engine="cr", group_w=2)

        def render_one(f):
            out = rr.render_device(poses[f], cfg, renderer=r)
            return out.image, out.stats.clone()

        res = render_trajectory(render_one, N_FRAMES, gather=True, device="cpu")
        if rank == 0:
            np.savez(out_path, frames=np.array(res.gathered_frames), images=res.gathered_images,
                     stats=res.gathered_stats, mine=np.array(res.frames))
        dist.barrier()
    finally:
        dist.destroy_process_group()


def test_two_ranks_real_render_gather(tmp_path):
    from paper_2503_05168_b200 import EngineConfig
    from paper_2503_05168_b200.distributed import quantize
    from paper_2503_05168_b200.residency import ResidentRenderer

    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    out = tmp_path / "gathered.npz"
    mp.spawn(_worker, args=(2, port, str(out)), nprocs=2, join=True)
    z = np.load(out)
    assert z["frames"].tolist() == list(range(N_FRAMES))
    assert z["mine"].tolist() == list(range(0, N_FRAMES, 2))
    container, poses = _setup()
    rr = ResidentRenderer(container, m=1)
    cfg = EngineConfig(engine="cr", group_w=2)
    for f in range(N_FRAMES):
        want = rr.render_frame(poses[f], cfg)
        np.testing.assert_array_equal(z["images"][f], quantize(torch.as_tensor(want.image.astype(np.float32))).numpy())
        assert z["stats"][f][0] == want.stats.alpha_eval_steps
        assert z["stats"][f][3] == want.stats.warp_steps
