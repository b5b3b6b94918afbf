"""GPU depth order (csrc/depth.cu) under adversarial depth distributions,
against the CPU oracle's np.lexsort((ref, depth, tile)) order
(sorting.py:32-54): every path of the bucket sort is driven --

* a wall of splats at one exact depth (all ties: order by position; one
  bucket far beyond a CTA's shared memory -> the global merge sort);
* a dense band (thousands of splats per depth bucket -> the shared-memory
  bitonic sort) plus far outliers (the round-1 quantised key collapsed such a
  band into long equal-key runs);
* depths beyond the bucket range (all in the last, clamped bucket).

Bar: the (tile, position) pair sequence, tile ranges, contributor counts and
FrameStats bit-exact, image within 1e-3.
"""
import numpy as np
import pytest

from helpers import STAT_KEYS
from oracle import oracle as O
from paper_2503_05168_b200 import DeviceScene, EngineConfig, render_frame
from paper_2503_05168_b200.model import SceneArrays
from paper_2503_05168_b200.render import FrameRenderer
from paper_2503_05168_b200.synthetic import make_camera, random_scene
from test_gpu_configs import _check_plan, _device_plan

pytestmark = pytest.mark.gpu


def _run(scene, cam):
    dscene = DeviceScene.from_arrays(scene)
    cfg = EngineConfig(engine="cr", group_w=2)
    pl = O.plan(scene, cam, cfg)
    r = FrameRenderer()
    out, host = r.render_checked(dscene, cam, cfg)
    _check_plan(*_device_plan(r, host), pl)
    for c in (cfg, EngineConfig(engine="ref")):
        want = O.raster(pl, c)
        res = render_frame(dscene, cam, c)
        np.testing.assert_array_equal(res.contrib_count, want["contrib"])
        assert [getattr(res.stats, k) for k in STAT_KEYS] == [want["stats"][k] for k in STAT_KEYS]
        assert float(np.abs(res.image - want["image"]).max()) <= 1e-3


def _with_depths(scene: SceneArrays, z: np.ndarray) -> SceneArrays:
    """Move every splat along its view ray (identity camera at the origin) to depth z."""
    p = scene.positions.copy()
    p *= (z / p[:, 2])[:, None]
    p[:, 2] = z
    return SceneArrays(p, scene.log_scales, scene.rotations, scene.opacities, scene.sh, scene.ids)


def test_wall_of_equal_depths():
    cam = make_camera(320, 240)
    rng = np.random.default_rng(11)
    scene = random_scene(rng, 12000, camera=cam, scale_range=(0.005, 0.03), opacity_range=(0.02, 0.6))
    _run(_with_depths(scene, np.full(len(scene.positions), 5.0)), cam)


def test_dense_band_and_far_outliers():
    cam = make_camera(320, 240)
    rng = np.random.default_rng(12)
    n = 20000
    scene = random_scene(rng, n, camera=cam, scale_range=(0.005, 0.04), opacity_range=(0.02, 0.6))
    z = rng.uniform(4.0, 4.004, size=n)  # ~3000 splats per depth bucket
    z[:8] = [1e4, 2e4, 5e3, 3e4, 1e5, 7e3, 9e3, 4e4]
    z[8:40] = 4.002  # exact ties inside the band
    _run(_with_depths(scene, z), cam)


def test_depths_beyond_bucket_range():
    cam = make_camera(256, 192)
    rng = np.random.default_rng(13)
    n = 3000
    scene = random_scene(rng, n, camera=cam, scale_range=(100.0, 800.0), opacity_range=(0.3, 0.9))
    z = rng.uniform(2.0e4, 9.0e4, size=n)  # > near * 2^16: one clamped bucket
    _run(_with_depths(scene, z), cam)
