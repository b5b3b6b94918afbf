"""GPU parity: the CUDA path (through the C-ABI) against the reference's golden
vectors and the CPU oracle.

Bar (BASELINE.json north_star): sort order, ranges, per-pixel contributor
counts and FrameStats bit-exact; images max-abs <= 1e-3 per channel and
PSNR >= 50 dB.  Both raster precisions ("fast" fp32 with guarded fp64
re-decision, "exact" fp64) must meet it.
"""
import numpy as np
import pytest
import torch

from helpers import (SMALL_CASES, STAT_KEYS, camera_from, config_for, engines_in, golden_ranges, load, psnr,
                     scene_from, sha)
from oracle import oracle as O
from paper_2503_05168_b200 import DeviceScene, EngineConfig, FrameRenderer, _native, plan_frame, render_frame
from paper_2503_05168_b200.synthetic import config1_scene, make_camera, orbit_pose, random_scene, synth

pytestmark = pytest.mark.gpu
IMAGE_TOL = 1e-3


def _stats(res):
    return [getattr(res.stats, k) for k in STAT_KEYS]


def _check_frame(res, contrib, stats, image):
    np.testing.assert_array_equal(res.contrib_count, contrib)
    assert _stats(res) == list(stats)
    err = float(np.abs(res.image - image).max())
    assert err <= IMAGE_TOL, err
    assert psnr(res.image, image) >= 50.0


@pytest.mark.parametrize("precision", ["fast", "exact"])
@pytest.mark.parametrize("name", SMALL_CASES)
def test_small_cases_vs_reference(name, precision):
    g = load(name)
    cam, scene = camera_from(g), scene_from(g)
    dscene = DeviceScene.from_arrays(scene)
    for tag in engines_in(g):
        res = render_frame(dscene, cam, config_for(g, tag, precision=precision))
        _check_frame(res, g[f"{tag}_contrib"], g[f"{tag}_stats"], g[f"{tag}_image"])


@pytest.mark.parametrize("name", SMALL_CASES)
def test_small_plan_vs_reference(name):
    g = load(name)
    cam, scene = camera_from(g), scene_from(g)
    plan = plan_frame(scene, cam, config_for(g, "ref"))
    np.testing.assert_array_equal(plan.ids, g["plan_ids"])
    np.testing.assert_array_equal(plan.sorted_pairs["tile_id"], g["pair_tile"])
    np.testing.assert_array_equal(plan.sorted_pairs["gaussian_ref"], g["pair_ref"])
    got = np.array([(r.tile_id, r.start, r.end) for r in plan.ranges], dtype=np.int64).reshape(-1, 3)
    np.testing.assert_array_equal(got, g["ranges"])
    assert [plan.culled_near, plan.dropped_degenerate] == g["plan_counts"].tolist()
    np.testing.assert_array_equal(plan.depths, g["plan_depths"])  # the sort key: bit-exact
    np.testing.assert_allclose(plan.conics, g["plan_conics"], rtol=1e-11, atol=1e-12)
    np.testing.assert_allclose(plan.means, g["plan_means"], rtol=1e-12, atol=1e-9)
    np.testing.assert_allclose(plan.colors, g["plan_colors"], atol=1e-6)


@pytest.mark.parametrize("layout", ["f64", "planes"])
@pytest.mark.parametrize("seed", [0, 1, 2])
def test_random_scenes_vs_oracle(seed, layout):
    rng = np.random.default_rng(100 + seed)
    w, h = [(64, 64), (200, 120), (333, 177)][seed]
    cam = make_camera(w, h, position=rng.normal(0, 0.1, 3), orientation=(1.0, *rng.normal(0, 0.05, 3)))
    scene = random_scene(rng, 3000, sh_degree=3, camera=cam, scale_range=(0.005, 0.3), opacity_range=(0.004, 0.99))
    dscene = DeviceScene.from_arrays(scene, layout=layout)
    host = dscene.host_arrays()
    for eng in ("ref", "cr1", "cr2", "cr4"):
        kw = {"engine": "ref"} if eng == "ref" else {"engine": "cr", "group_w": int(eng[2])}
        cfg = EngineConfig(background=(0.2, 0.1, 0.05), **kw)
        want = O.render(host, cam, cfg)
        res = render_frame(dscene, cam, cfg)
        _check_frame(res, want["contrib"], [want["stats"][k] for k in STAT_KEYS], want["image"])


@pytest.mark.parametrize("layout", ["f64", "planes"])
def test_high_opacity_clamp_vs_oracle(layout):
    """Opacities up to 1: alpha = min(o exp(-q/2), 0.99) clamps near the centres
    (rasterize.py:146-151), the FAST raster's rare path for o > 0.99."""
    rng = np.random.default_rng(77)
    cam = make_camera(160, 96)
    scene = random_scene(rng, 2500, sh_degree=3, camera=cam, scale_range=(0.01, 0.2), opacity_range=(0.97, 1.0))
    assert (scene.opacities > 0.99).sum() > 500
    dscene = DeviceScene.from_arrays(scene, layout=layout)
    host = dscene.host_arrays()
    for eng in ("ref", "cr2", "cr4"):
        kw = {"engine": "ref"} if eng == "ref" else {"engine": "cr", "group_w": int(eng[2])}
        cfg = EngineConfig(background=(0.1, 0.2, 0.3), **kw)
        want = O.render(host, cam, cfg)
        res = render_frame(dscene, cam, cfg)
        _check_frame(res, want["contrib"], [want["stats"][k] for k in STAT_KEYS], want["image"])


def test_fast_equals_exact_discrete():
    cam = make_camera(256, 256)
    scene = random_scene(np.random.default_rng(9), 20000, sh_degree=3, camera=cam, opacity_range=(0.3, 0.99))
    dscene = DeviceScene.from_arrays(scene)
    for kw in ({"engine": "ref"}, {"engine": "cr", "group_w": 2}, {"engine": "cr", "group_w": 4}):
        fast = render_frame(dscene, cam, EngineConfig(precision="fast", **kw))
        exact = render_frame(dscene, cam, EngineConfig(precision="exact", **kw))
        np.testing.assert_array_equal(fast.contrib_count, exact.contrib_count)
        assert _stats(fast) == _stats(exact)
        assert float(np.abs(fast.image - exact.image).max()) <= 1e-4


def test_deterministic_across_runs():
    scene, cam = config1_scene()
    dscene = DeviceScene.from_arrays(scene)
    cfg = EngineConfig(engine="cr", group_w=2)
    a = render_frame(dscene, cam, cfg)
    b = render_frame(dscene, cam, cfg)
    np.testing.assert_array_equal(a.image, b.image)
    np.testing.assert_array_equal(a.contrib_count, b.contrib_count)
    assert _stats(a) == _stats(b)


def test_config1_vs_reference():
    """BASELINE config 1 (100K SH3 @256x256), reference golden hashes + counts."""
    g = load("config1")
    scene, cam = config1_scene()
    dscene = DeviceScene.from_arrays(scene)
    plan = plan_frame(dscene, cam, EngineConfig())
    pair_ids = np.stack([plan.sorted_pairs["tile_id"], plan.ids[plan.sorted_pairs["gaussian_ref"]]], axis=1)
    assert sha(pair_ids.astype(np.int64)) == str(g["pairs_sha"][0])
    d32 = plan.sorted_pairs["depth"].astype(np.float32).view(np.uint32).astype(np.uint64)
    keys = (plan.sorted_pairs["tile_id"].astype(np.uint64) << np.uint64(32)) | d32
    assert sha(keys) == str(g["keys_sha"][0])
    got = np.array([(r.tile_id, r.start, r.end) for r in plan.ranges], dtype=np.int64)
    np.testing.assert_array_equal(got, g["ranges"])
    for tag in ("ref", "cr2"):
        for precision in ("fast", "exact"):
            res = render_frame(dscene, cam, config_for(g, tag, precision=precision))
            _check_frame(res, g[f"{tag}_contrib"], g[f"{tag}_stats"], g[f"{tag}_image_f32"].astype(np.float64))


@pytest.mark.parametrize("frame", [0, 37])
def test_synth_1080p_vs_reference(frame):
    g = load(f"synth20k_f{frame}")
    scene = synth(20_000, 0)
    cam = camera_from(g)
    dscene = DeviceScene.from_arrays(scene)
    plan = plan_frame(dscene, cam, EngineConfig())
    pair_ids = np.stack([plan.sorted_pairs["tile_id"], plan.ids[plan.sorted_pairs["gaussian_ref"]]], axis=1)
    assert sha(pair_ids.astype(np.int64)) == str(g["pairs_sha"][0])
    rs, re = golden_ranges(g, plan.grid.tile_count)
    got = np.array([(r.tile_id, r.start, r.end) for r in plan.ranges], dtype=np.int64)
    np.testing.assert_array_equal(got, g["ranges"])
    for tag in ("ref", "cr2"):
        res = render_frame(dscene, cam, config_for(g, tag))
        np.testing.assert_array_equal(res.contrib_count, g[f"{tag}_contrib"])
        assert _stats(res) == g[f"{tag}_stats"].tolist()
        idx = g[f"{tag}_sample_idx"]
        assert float(np.abs(res.image.reshape(-1, 3)[idx] - g[f"{tag}_sample_rgb"]).max()) <= IMAGE_TOL


@pytest.mark.parametrize("n,frame", [(1_000_000, 0), (3_000_000, 30)])
def test_large_synth_vs_oracle(n, frame):
    """BASELINE configs 2/3 geometry (1M / 3M @1080p, container layout) vs the fp64 oracle."""
    scene = synth(n, 0)
    cam = orbit_pose(frame)
    dscene = DeviceScene.from_arrays(scene, layout="planes")
    host = dscene.host_arrays()
    cfg = EngineConfig(engine="cr", group_w=2)
    pl = O.plan(host, cam, cfg)
    plan = plan_frame(dscene, cam, cfg)
    np.testing.assert_array_equal(plan.sorted_pairs["tile_id"], pl["pair_tile"])
    np.testing.assert_array_equal(plan.ids[plan.sorted_pairs["gaussian_ref"]], pl["ids"][pl["pair_ref"]])
    for eng in (dict(engine="ref"), dict(engine="cr", group_w=2)):
        c = EngineConfig(**eng)
        want = O.raster(pl, c)
        res = render_frame(dscene, cam, c)
        _check_frame(res, want["contrib"], [want["stats"][k] for k in STAT_KEYS], want["image"])


def test_overflow_grows_workspace():
    cam = make_camera(128, 128)
    scene = random_scene(np.random.default_rng(3), 4000, sh_degree=1, camera=cam, scale_range=(0.1, 0.5))
    dscene = DeviceScene.from_arrays(scene)
    r = FrameRenderer()
    r.reserve(len(scene), 128, 128, pair_capacity=1000)
    first = r.render(dscene, cam, EngineConfig()).stats.cpu().numpy()
    assert first[_native.STAT_OVERFLOW] == 1
    out, host = r.render_checked(dscene, cam, EngineConfig())
    want = O.render(scene, cam, EngineConfig())
    np.testing.assert_array_equal(out.contrib.cpu().numpy(), want["contrib"])
    assert host[_native.STAT_TILE_PAIRS] == want["stats"]["tile_pairs"] > 1000
    assert r.pair_capacity >= host[_native.STAT_TILE_PAIRS]


def test_native_library_is_loaded():
    import paper_2503_05168_b200._native as nat
    assert nat._lib is not None or nat.load() is not None
    assert torch.cuda.is_available()
