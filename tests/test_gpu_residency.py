"""GPU: device cluster lookup (K0) and clustered rendering (select -> range
table -> render without a host round trip) against reference vectors and the
oracle on the reference-order assembled working set."""
import numpy as np
import pytest

from helpers import STAT_KEYS, load, psnr
from oracle import oracle as O
from paper_2503_05168_b200.clusters import build_cluster_table
from paper_2503_05168_b200.container import load_clustered_scene, write_clustered_scene
from paper_2503_05168_b200.errors import InvalidArgumentError
from paper_2503_05168_b200.model import CameraPose
from paper_2503_05168_b200.render import EngineConfig
from paper_2503_05168_b200.residency import ResidentRenderer, select_clusters
from paper_2503_05168_b200.synthetic import make_camera, orbit, orbit_pose, synth

pytestmark = pytest.mark.gpu


def test_device_select_matches_reference():
    g = load("clusters_orbit")
    norm = (g["norm_mean"], float(g["norm_scale"][0]))
    for i in range(120):
        p = orbit_pose(i)
        cam = CameraPose(p.position, p.orientation, p.fov_x, p.fov_y, p.width, p.height)
        assert select_clusters(cam, g["centroids"], 4, 1.0, norm) == g["selections"][i].tolist()
    base = orbit_pose(0)
    for probe, want in zip(g["probes"], g["probe_selections"]):
        cam = CameraPose(probe[:3], probe[3:], base.fov_x, base.fov_y, base.width, base.height)
        assert select_clusters(cam, g["centroids"], 4, 1.0, norm) == want.tolist()
    with pytest.raises(InvalidArgumentError):
        select_clusters(base, g["centroids"], 24, 1.0, norm)


def test_resident_renderer_two_sided(tmp_path):
    g = load("clusters_two_sided")
    for key in g:
        if key.startswith("file:"):
            (tmp_path / key[5:]).write_bytes(g[key].tobytes())
    rr = ResidentRenderer(str(tmp_path), m=0)
    cfg = EngineConfig(engine="cr", group_w=2)
    for i, sel in enumerate(g["selections"]):
        pose = g[f"pose{i}"]
        cam = make_camera(64, 64, position=pose[:3], orientation=pose[3:])
        assert rr.select(cam) == sel.tolist()
        res = rr.render_frame(cam, cfg)
        assert [getattr(res.stats, k) for k in STAT_KEYS] == g[f"stats{i}"].tolist()
        assert float(np.abs(res.image - g["images"][i]).max()) <= 1e-3


@pytest.fixture(scope="module")
def synthetic_container(tmp_path_factory):
    scene = synth(200_000, 3)
    poses = orbit(120, 640, 360)
    table = build_cluster_table(scene, poses, n_clusters=24, neighbors=4)
    d = tmp_path_factory.mktemp("c3small")
    write_clustered_scene(table, scene, d)
    return d, poses


@pytest.mark.parametrize("frame", [0, 45, 91])
def test_clustered_render_vs_oracle(synthetic_container, frame):
    d, poses = synthetic_container
    rr = ResidentRenderer(str(d))
    cam = poses[frame]
    sel = rr.select(cam)
    ws = rr.assemble(sel)
    for eng in (dict(engine="ref"), dict(engine="cr", group_w=2)):
        cfg = EngineConfig(**eng)
        want = O.render(ws, cam, cfg)
        res = rr.render_frame(cam, cfg)
        np.testing.assert_array_equal(res.contrib_count, want["contrib"])
        assert [getattr(res.stats, k) for k in STAT_KEYS] == [want["stats"][k] for k in STAT_KEYS]
        assert float(np.abs(res.image - want["image"]).max()) <= 1e-3
        assert psnr(res.image, want["image"]) >= 50.0


def test_working_set_is_reference_order(synthetic_container):
    d, poses = synthetic_container
    c = load_clustered_scene(d)
    rr = ResidentRenderer(c)
    sel = rr.select(poses[10])
    np.testing.assert_array_equal(rr.working_set_ids(sel), rr.assemble(sel).ids)
    assert len(sel) == 1 + c.m


@pytest.mark.parametrize("depth", [1, 2, 3])
def test_trajectory_pipeline_matches_serial(synthetic_container, depth):
    """Frames in flight on separate streams (FramePipeline / render_trajectory)
    give exactly the per-frame results of the serial path."""
    d, poses = synthetic_container
    rr = ResidentRenderer(str(d))
    cfg = EngineConfig(engine="cr", group_w=2)
    frames = [3, 17, 40, 41, 77, 100, 119]
    want = {}
    for f in frames:
        res = rr.render_frame(poses[f], cfg, output="numpy32")
        want[f] = (res.image.copy(), res.contrib_count.copy(), [getattr(res.stats, k) for k in STAT_KEYS])
    got = 0
    for i, img, cnt, st in rr.render_trajectory([poses[f] for f in frames], cfg, depth=depth,
                                                pair_capacity=4_000_000):
        w_img, w_cnt, w_st = want[frames[i]]
        np.testing.assert_array_equal(img, w_img)
        np.testing.assert_array_equal(cnt, w_cnt)
        assert [int(st[k]) for k in range(len(STAT_KEYS))] == w_st
        got += 1
    assert got == len(frames)


def test_partitioned_pipeline_matches_serial(synthetic_container):
    """FramePipeline on an SM partition (plan stages and rasters on disjoint
    green-context SM sets, seele_partition_create) gives exactly the per-frame
    results of the serial path."""
    import torch

    from paper_2503_05168_b200.pipeline import FramePipeline

    d, poses = synthetic_container
    rr = ResidentRenderer(str(d))
    cfg = EngineConfig(engine="cr", group_w=2)
    frames = [5, 29, 30, 64, 118]
    w, h = poses[0].width, poses[0].height
    pipe = FramePipeline(rr, w, h, depth=2, pair_capacity=4_000_000, partition=32)
    assert pipe.partition is not None and pipe.partition[0] >= 32 and sum(pipe.partition) <= 148 * 2
    for f in frames:
        want = rr.render_frame(poses[f], cfg, output="numpy32")
        k = pipe.slot_of_next()
        out = pipe.submit(poses[f], cfg)
        pipe.output_stream(k).synchronize()
        np.testing.assert_array_equal(out.image.cpu().numpy(), want.image)
        np.testing.assert_array_equal(out.contrib.cpu().numpy(), want.contrib_count)
        got = out.stats.cpu().numpy()
        assert [int(got[i]) for i in range(len(STAT_KEYS))] == [getattr(want.stats, s) for s in STAT_KEYS]
    torch.cuda.synchronize()
