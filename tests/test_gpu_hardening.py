"""GPU regressions for round-1 review findings:

* the streaming slot pool with evict_policy="lru" and prefetch on, a
  container of 12 clusters and a trajectory that jumps across the orbit
  (one frame can add 1 + m stalls and 1 + m prefetches before eviction runs);
* caller-supplied output buffers are validated (shape, dtype, device,
  contiguity) before any kernel writes through them, and a trajectory whose
  cameras change size is rejected;
* distributed.render_trajectory driven by the real render on a one-rank NCCL
  group: device-side quantisation into the gather buffer and the collective.
"""
import os
import socket

import numpy as np
import pytest
import torch

from paper_2503_05168_b200 import DeviceScene, EngineConfig, FrameRenderer
from paper_2503_05168_b200.clusters import build_cluster_table
from paper_2503_05168_b200.container import container_from_table
from paper_2503_05168_b200.errors import InvalidArgumentError
from paper_2503_05168_b200.residency import ResidentRenderer
from paper_2503_05168_b200.streaming import StreamingRenderer
from paper_2503_05168_b200.synthetic import make_camera, orbit, orbit_pose, random_scene, synth

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def twelve_clusters():
    scene = synth(60_000, 5)
    poses = orbit(120, 320, 180)
    table = build_cluster_table(scene, poses, n_clusters=12, neighbors=1, beta=1.0, seed=0, device="cuda")
    return container_from_table(table, scene), poses


def test_lru_prefetch_jumping_trajectory(twelve_clusters):
    container, poses = twelve_clusters
    assert container.num_clusters >= 10
    traj = [poses[i] for i in (0, 40, 80, 5, 45, 85, 20, 60, 100, 0, 119, 59)]
    cfg = EngineConfig(engine="cr", group_w=2)
    resident = ResidentRenderer(container, m=1)
    with StreamingRenderer(container, m=1, prefetch=True, evict=True, evict_policy="lru") as sr:
        for i, cam in enumerate(traj):
            res = sr.render_frame(cam, cfg)
            full = resident.render_frame(cam, cfg)
            np.testing.assert_array_equal(res.contrib_count, full.contrib_count, err_msg=str(i))
            np.testing.assert_array_equal(res.image, full.image, err_msg=str(i))
        assert sr.stall_count > 0


def test_output_buffers_are_validated():
    cam = make_camera(64, 48)
    scene = random_scene(np.random.default_rng(1), 500, sh_degree=1, camera=cam)
    ds = DeviceScene.from_arrays(scene)
    r = FrameRenderer()
    cfg = EngineConfig()
    dev = r.device
    bad = [
        dict(image=torch.empty((48, 64, 3), dtype=torch.float64, device=dev)),
        dict(image=torch.empty((32, 64, 3), dtype=torch.float32, device=dev)),
        dict(image=torch.empty((64, 48, 3), dtype=torch.float32, device=dev).transpose(0, 1)),
        dict(image=torch.empty((48, 64, 3), dtype=torch.float32)),
        dict(contrib=torch.empty((48, 63), dtype=torch.int32, device=dev)),
        dict(contrib=torch.empty((48, 64), dtype=torch.int64, device=dev)),
        dict(stats=torch.empty(3, dtype=torch.int64, device=dev)),
    ]
    for kw in bad:
        with pytest.raises(InvalidArgumentError):
            r.render(ds, cam, cfg, **kw)
    out = r.render(ds, cam, cfg, image=torch.empty((48, 64, 3), dtype=torch.float32, device=dev))
    torch.cuda.synchronize()
    assert out.image.shape == (48, 64, 3)


def test_trajectory_rejects_mixed_sizes(twelve_clusters):
    container, poses = twelve_clusters
    rr = ResidentRenderer(container, m=1)
    cams = [poses[0], orbit_pose(1, width=640, height=360)]
    with pytest.raises(InvalidArgumentError):
        list(rr.render_trajectory(cams, EngineConfig()))


def test_distributed_trajectory_one_rank_nccl(twelve_clusters):
    import torch.distributed as dist

    from paper_2503_05168_b200.distributed import quantize, render_trajectory

    container, poses = twelve_clusters
    rr = ResidentRenderer(container, m=1)
    cfg = EngineConfig(engine="cr", group_w=2)
    r = FrameRenderer()
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
    try:
        def render_one(f):
            out = rr.render_device(poses[f], cfg, renderer=r, image=torch.empty((180, 320, 3), device="cuda"))
            return out.image, out.stats.clone()

        res = render_trajectory(render_one, 10, gather=True)
    finally:
        dist.destroy_process_group()
    assert res.gathered_frames == list(range(10))
    for f in (0, 7):
        want = rr.render_frame(poses[f], cfg)
        np.testing.assert_array_equal(res.gathered_images[f], quantize(torch.as_tensor(want.image.astype(np.float32))).numpy())
        assert res.gathered_stats[f][0] >= 0
