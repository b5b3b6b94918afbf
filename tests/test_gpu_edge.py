"""GPU edge cases of the sort / binning / raster path against the oracle:
long runs of equal (and nearly equal) depths (the depth sort's exact fp64
fix-up, including the CTA path for runs longer than 32), very wide splats
(row entries split into 3-column segments), many tile rows and columns, runs
of ties of every length 2..40 crossing the fix-up's 256-position blocks,
near-opaque splats (the 0.99 alpha clamp), and a frame with no binned splat."""
import numpy as np
import pytest

from helpers import STAT_KEYS, psnr
from oracle import oracle as O
from paper_2503_05168_b200 import DeviceScene, EngineConfig, plan_frame, render_frame
from paper_2503_05168_b200.model import SceneArrays
from paper_2503_05168_b200.synthetic import make_camera, random_scene

pytestmark = pytest.mark.gpu


def _check(scene, cam, cfgs):
    dscene = DeviceScene.from_arrays(scene)
    for cfg in cfgs:
        want = O.render(scene, cam, cfg)
        res = render_frame(dscene, cam, cfg)
        np.testing.assert_array_equal(res.contrib_count, want["contrib"])
        assert [getattr(res.stats, k) for k in STAT_KEYS] == [want["stats"][k] for k in STAT_KEYS]
        assert float(np.abs(res.image - want["image"]).max()) <= 1e-3
        assert psnr(res.image, want["image"]) >= 50.0


CFGS = (EngineConfig(engine="ref"), EngineConfig(engine="cr", group_w=2), EngineConfig(engine="cr", group_w=4))


def _with_depths(scene, cam, depths):
    """Move each splat along its view ray to the given camera depth."""
    r = cam.rotation_matrix()
    view = (r.T @ (scene.positions - cam.position).T).T
    view = view * (depths / view[:, 2])[:, None]
    pos = (r @ view.T).T + cam.position
    return SceneArrays(pos, scene.log_scales, scene.rotations, scene.opacities, scene.sh, scene.ids)


def test_equal_and_nearly_equal_depths():
    cam = make_camera(160, 96)
    rng = np.random.default_rng(21)
    n = 6000
    scene = random_scene(rng, n, sh_degree=2, camera=cam, opacity_range=(0.05, 0.7))
    d = rng.uniform(2.0, 6.0, size=n)
    d[:1500] = 3.0                                        # one long run of identical depths (> 32: CTA path)
    d[1500:2500] = 4.0 + 1e-13 * rng.integers(0, 50, 1000)  # distinct depths inside one quantisation step
    d[2500:2600] = d[2600:2700]                           # scattered pairs of exact ties
    _check(_with_depths(scene, cam, d), cam, CFGS)


def test_tie_runs_of_every_length():
    # depths drawn from a small set so that equal-key runs of every length 2..40 occur at many offsets
    # relative to the fix-up's 256-position blocks (runs > 32 take the CTA path)
    cam = make_camera(192, 128)
    rng = np.random.default_rng(8)
    lengths = np.tile(np.arange(2, 41), 14)
    rng.shuffle(lengths)
    n = int(lengths.sum())
    scene = random_scene(rng, n, sh_degree=1, camera=cam, opacity_range=(0.05, 0.6))
    levels = np.sort(rng.uniform(2.0, 6.0, size=lengths.size))
    d = np.repeat(levels, lengths)[rng.permutation(n)]
    _check(_with_depths(scene, cam, d), cam, CFGS[:2])


def test_near_opaque_splats():
    # opacities above 0.99: alpha = min(o exp(-q/2), 0.99) clamps near the centres
    cam = make_camera(128, 96)
    rng = np.random.default_rng(13)
    scene = random_scene(rng, 3000, sh_degree=2, camera=cam, opacity_range=(0.97, 0.9999))
    _check(scene, cam, CFGS)


def test_wide_splats_and_many_tiles():
    cam = make_camera(1000, 720)  # 63 x 45 tiles
    rng = np.random.default_rng(5)
    scene = random_scene(rng, 4000, sh_degree=1, camera=cam, scale_range=(0.02, 0.9), opacity_range=(0.02, 0.8))
    _check(scene, cam, CFGS[:2])
    plan = plan_frame(DeviceScene.from_arrays(scene), cam, EngineConfig())
    want = O.plan(scene, cam, EngineConfig())
    np.testing.assert_array_equal(plan.sorted_pairs["tile_id"], want["pair_tile"])


def test_no_binned_splat():
    cam = make_camera(64, 48)
    rng = np.random.default_rng(2)
    scene = random_scene(rng, 50, camera=cam, opacity_range=(0.0005, 0.003))  # all below alpha_theta: r^2 = 0
    _check(scene, cam, CFGS[:1])


# ---- binning (binning.cu) geometry edges ----------------------------------------------------------------

def _plan_check(scene, cam, cfg):
    """The GPU plan's (tile, id) sequence and ranges against the oracle's sort_intersections."""
    plan = plan_frame(DeviceScene.from_arrays(scene), cam, cfg)
    want = O.plan(scene, cam, cfg)
    pairs = plan.sorted_pairs
    assert len(pairs) == want["tile_pairs"]
    np.testing.assert_array_equal(pairs["tile_id"], want["pair_tile"])
    np.testing.assert_array_equal(pairs["gaussian_ref"], want["pair_ref"])
    got_r = {r.tile_id: (r.start, r.end) for r in plan.ranges}
    for t in np.flatnonzero(want["range_end"] > want["range_start"]):
        assert got_r[int(t)] == (int(want["range_start"][t]), int(want["range_end"][t]))


def test_max_tile_axis_and_partial_super_tiles():
    # 4096 x 200 px: 256 tile columns (the 8-bit packed rect at its limit, 64 super-tile columns), 13 tile rows
    # (the last super-tile row holds one tile row); splats of every size down to single tiles
    cam = make_camera(4096, 200)
    rng = np.random.default_rng(44)
    scene = random_scene(rng, 30_000, sh_degree=1, camera=cam, scale_range=(0.002, 0.3))
    _plan_check(scene, cam, EngineConfig())
    _check(scene, cam, (EngineConfig(engine="cr", group_w=2),))


def test_odd_size_super_tile_edges():
    # 1000 x 600 px: 63 x 38 tiles, partial super-tiles on the right and bottom edges
    cam = make_camera(1000, 600)
    rng = np.random.default_rng(45)
    scene = random_scene(rng, 40_000, sh_degree=1, camera=cam, scale_range=(0.005, 0.25))
    _plan_check(scene, cam, EngineConfig())


def test_large_splats_beyond_the_head():
    # screen-covering splats at every depth (not only the nearest ranks, which the per-tile head pass takes):
    # their super-tile entries span the whole grid in every chunk
    cam = make_camera(640, 384)
    rng = np.random.default_rng(46)
    scene = random_scene(rng, 20_000, sh_degree=1, camera=cam, scale_range=(0.01, 0.1))
    big = rng.choice(len(scene.positions), 400, replace=False)
    ls = scene.log_scales.copy()
    ls[big] = np.log(rng.uniform(0.8, 2.5, size=(400, 3)))
    op = scene.opacities.copy()
    op[big] = rng.uniform(0.02, 0.08, size=400)  # faint, so the pixels behind them still blend
    scene = SceneArrays(scene.positions, ls, scene.rotations, op, scene.sh, scene.ids)
    _plan_check(scene, cam, EngineConfig())
    _check(scene, cam, (EngineConfig(), EngineConfig(engine="cr", group_w=2)))
