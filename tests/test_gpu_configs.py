"""GPU parity at the BASELINE configurations the smaller tests do not reach,
against the CPU fp64 oracle (oracle/seele_oracle.c, all host cores):

* C4: synth(6M, 0) at 3840x2160, orbit frame 0, flat -- 123M sorted tile
  pairs over 32,400 tiles (sorting.py:32-54 at scale), engines ref and cr2;
* C5 "HP off": synth(3M, 0) flat at 1080p with the plain 3-sigma extents
  (opacity_aware_filter=False, preprocess.py:68-71), engines ref and cr2;
* C3 as benchmarked: the 3M scene with its 24-cluster table, every one of the
  120 orbit frames -- device cluster lookup (K0) vs the reference selection
  rule and the whole plan (the (tile, splat) sequence and the tile ranges) vs
  the oracle on the reference-order working set (residency.py:217-220) -- and
  full rasters of three frames.

Bar (north_star): (tile, id) sequence, ranges, contributor counts and all
seven FrameStats integers bit-exact; image max-abs <= 1e-3 per channel and
PSNR >= 50 dB against the oracle image.
"""
import ctypes

import numpy as np
import pytest
import torch

from helpers import STAT_KEYS, psnr
from oracle import oracle as O
from paper_2503_05168_b200 import DeviceScene, EngineConfig, _native, render_frame
from paper_2503_05168_b200.clusters import build_cluster_table
from paper_2503_05168_b200.container import container_from_table
from paper_2503_05168_b200.render import FrameRenderer, TileGrid
from paper_2503_05168_b200.residency import ResidentRenderer
from paper_2503_05168_b200.synthetic import orbit, orbit_pose, synth

pytestmark = pytest.mark.gpu
IMAGE_TOL = 1e-3
ENGINES = (dict(engine="ref"), dict(engine="cr", group_w=2))


def _check_frame(res, want):
    np.testing.assert_array_equal(res.contrib_count, want["contrib"])
    assert [getattr(res.stats, k) for k in STAT_KEYS] == [want["stats"][k] for k in STAT_KEYS]
    err = float(np.abs(res.image - want["image"]).max())
    assert err <= IMAGE_TOL, err
    assert psnr(res.image, want["image"]) >= 50.0


def _device_plan(renderer: FrameRenderer, host_stats: np.ndarray) -> tuple[np.ndarray, np.ndarray, np.ndarray]:
    """(pair tile, pair assembled position, per-tile [start, end)) of the renderer's last frame."""
    k = int(host_stats[_native.STAT_TILE_PAIRS])
    w, h = renderer.size
    d = renderer.device
    tiles = TileGrid.for_image(w, h).tile_count
    pair_pos = torch.empty(max(k, 1), dtype=torch.int32, device=d)
    pair_tile = torch.empty(max(k, 1), dtype=torch.int32, device=d)
    ranges = torch.empty((tiles, 2), dtype=torch.int32, device=d)
    view = _native.PlanView(pair_pos.data_ptr(), pair_tile.data_ptr(), ranges.data_ptr(), None, None, None, None,
                            None, None, None)
    _native.check(renderer.lib.seele_plan_export(renderer.workspace.data_ptr(), renderer.n_max,
                                                 renderer.pair_capacity, w, h, 0, k, ctypes.byref(view),
                                                 torch.cuda.current_stream(d).cuda_stream))
    return pair_tile.cpu().numpy()[:k], pair_pos.cpu().numpy()[:k], ranges.cpu().numpy()


def _check_plan(tile, pos, ranges, pl):
    assert len(tile) == pl["tile_pairs"]
    np.testing.assert_array_equal(tile, pl["pair_tile"])
    np.testing.assert_array_equal(pos.astype(np.int64), pl["index"][pl["pair_ref"]])
    np.testing.assert_array_equal(ranges[:, 0], pl["range_start"])
    np.testing.assert_array_equal(ranges[:, 1], pl["range_end"])


def _flat_case(n, cam, opacity_aware):
    scene = synth(n, 0)
    dscene = DeviceScene.from_arrays(scene, layout="planes")
    host = dscene.host_arrays()
    del scene
    pl = O.plan(host, cam, EngineConfig(opacity_aware_filter=opacity_aware))
    r = FrameRenderer()
    r.reserve(dscene.n, cam.width, cam.height, pair_capacity=pl["tile_pairs"] + 4096)
    for eng in ENGINES:
        cfg = EngineConfig(opacity_aware_filter=opacity_aware, **eng)
        out, host_stats = r.render_checked(dscene, cam, cfg)
        assert int(host_stats[_native.STAT_TILE_PAIRS]) == pl["tile_pairs"]
        _check_plan(*_device_plan(r, host_stats), pl)
        want = O.raster(pl, cfg)
        res = render_frame(dscene, cam, cfg)
        _check_frame(res, want)
    return pl


def test_c4_6m_4k_vs_oracle():
    """C4: 6M splats, 3840x2160, 123,359,184 tile pairs."""
    pl = _flat_case(6_000_000, orbit_pose(0, width=3840, height=2160), True)
    assert pl["tile_pairs"] > 120_000_000  # (123,359,184 for the fp64 arrays; the container's fp32 values differ)


def test_c5_hp_off_3m_vs_oracle():
    """C5 'HP off': the flat 3M scene with plain 3-sigma extents (24,222,172 pairs at frame 0)."""
    pl = _flat_case(3_000_000, orbit_pose(0), False)
    assert pl["tile_pairs"] > 24_000_000


@pytest.fixture(scope="module")
def c3():
    """The benchmark's C3 workload (bench.py build_workload): synth(3M, 0), 24-cluster table, M = 4."""
    scene = synth(3_000_000, 0)
    poses = orbit(120, 1920, 1080)
    table = build_cluster_table(scene, poses, n_clusters=24, neighbors=4, beta=1.0, seed=0, device="cuda")
    container = container_from_table(table, scene)
    del scene
    rr = ResidentRenderer(container)
    r = FrameRenderer()
    r.reserve(rr.n_max, 1920, 1080, pair_capacity=40_000_000)
    return rr, r, poses


def _c3_plan_frames(c3, frames):
    rr, r, poses = c3
    cfg = EngineConfig(engine="cr", group_w=2)
    for f in frames:
        cam = poses[f]
        sel = rr.select(cam)  # K0 on the device
        assert sel == O.select_clusters(cam, rr.container.centroids, rr.m, rr.beta, rr.normalization), f
        rr.select_async(cam)
        out, host_stats = r.render_checked(rr.scene, cam, cfg, ranges=rr.ranges, n_ranges=rr.m + 2, n_max=rr.n_max)
        ws = rr.assemble(sel)
        assert int(host_stats[_native.STAT_WORKING_SET]) == len(ws.positions)
        pl = O.plan(ws, cam, cfg)
        assert [int(host_stats[_native.STAT_CULLED_NEAR]), int(host_stats[_native.STAT_DROPPED_DEGENERATE])] == \
            [pl["culled_near"], pl["dropped_degenerate"]], f
        _check_plan(*_device_plan(r, host_stats), pl)


@pytest.mark.parametrize("part", range(4))
def test_c3_trajectory_plans_vs_oracle(c3, part):
    """All 120 C3 frames (30 per part): selection, working-set size, near/degenerate counts, the full
    (tile, position) pair sequence and every tile range, bit-exact."""
    _c3_plan_frames(c3, range(part, 120, 4))


@pytest.mark.parametrize("frame", [0, 45, 97])
def test_c3_frames_vs_oracle(c3, frame):
    """Full C3 frames as benchmarked (clustered working set, HP + CR w=2 and the ref engine)."""
    rr, _, poses = c3
    cam = poses[frame]
    ws = rr.assemble(rr.select(cam))
    pl = O.plan(ws, cam, EngineConfig())
    for eng in ENGINES:
        cfg = EngineConfig(**eng)
        _check_frame(rr.render_frame(cam, cfg), O.raster(pl, cfg))
