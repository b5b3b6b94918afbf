"""Pin the CPU oracle (oracle/seele_oracle.c) to the reference's own outputs.

The golden vectors were produced by the reference Python package
(tests/golden/make_golden.py).  Discrete outputs must match bit for bit;
floating outputs to 1e-9 (numpy's BLAS/SIMD exp differ from glibc by ulps).
"""
import numpy as np
import pytest

from helpers import (ENGINES, SMALL_CASES, STAT_KEYS, base_cfg, camera_from, config_for, engines_in, golden_ranges,
                     load, scene_from, sha)
from oracle import oracle as O
from paper_2503_05168_b200.model import CameraPose
from paper_2503_05168_b200.synthetic import config1_scene, orbit_pose, synth


@pytest.mark.parametrize("name", SMALL_CASES)
def test_oracle_small_cases(name):
    g = load(name)
    cam, scene = camera_from(g), scene_from(g)
    first = True
    for tag in engines_in(g):
        cfg = config_for(g, tag)
        out = O.render(scene, cam, cfg)
        pl = out["plan"]
        if first:
            np.testing.assert_array_equal(pl["ids"], g["plan_ids"])
            np.testing.assert_array_equal(pl["pair_tile"], g["pair_tile"])
            np.testing.assert_array_equal(pl["pair_ref"], g["pair_ref"])
            rs, re = golden_ranges(g, pl["tiles_x"] * pl["tiles_y"])
            np.testing.assert_array_equal(pl["range_start"], rs)
            np.testing.assert_array_equal(pl["range_end"], re)
            assert [pl["culled_near"], pl["dropped_degenerate"]] == g["plan_counts"].tolist()
            np.testing.assert_allclose(pl["means"], g["plan_means"], rtol=1e-12, atol=1e-9)
            np.testing.assert_allclose(pl["conics"], g["plan_conics"], rtol=1e-11, atol=1e-12)
            np.testing.assert_allclose(pl["colors"], g["plan_colors"], rtol=0, atol=1e-13)
            np.testing.assert_array_equal(pl["depths"], g["plan_depths"])  # bit-exact: the sort key (tools/blas_order.py)
            first = False
        np.testing.assert_array_equal(out["contrib"], g[f"{tag}_contrib"])
        assert [out["stats"][k] for k in STAT_KEYS] == g[f"{tag}_stats"].tolist(), tag
        np.testing.assert_allclose(out["image"], g[f"{tag}_image"], rtol=0, atol=1e-9)


def test_edge_case_fixture_exercises_rejects():
    g = load("edges80x48")
    culled, dropped = g["plan_counts"].tolist()
    assert culled == 3 and dropped >= 1


def _check_big(g, scene, cam, tags, image_mode):
    pl = O.plan(scene, cam, config_for(g, "ref"))
    pair_ids = np.stack([pl["pair_tile"].astype(np.int64), pl["ids"][pl["pair_ref"]]], axis=1)
    assert sha(pair_ids) == str(g["pairs_sha"][0])
    assert sha(O.spec_keys(pl)) == str(g["keys_sha"][0])
    assert sha(pl["ids"]) == str(g["ids_sha"][0])
    counts = g["plan_counts"].tolist()
    assert [pl["culled_near"], pl["dropped_degenerate"], pl["tile_pairs"], len(pl["ids"])] == counts
    rs, re = golden_ranges(g, pl["tiles_x"] * pl["tiles_y"])
    np.testing.assert_array_equal(pl["range_start"], rs)
    np.testing.assert_array_equal(pl["range_end"], re)
    for tag in tags:
        out = O.raster(pl, config_for(g, tag))
        np.testing.assert_array_equal(out["contrib"], g[f"{tag}_contrib"])
        assert [out["stats"][k] for k in STAT_KEYS] == g[f"{tag}_stats"].tolist(), tag
        if image_mode == "f32":
            np.testing.assert_allclose(out["image"], g[f"{tag}_image_f32"], rtol=0, atol=1e-6)
        else:
            h, w = cam.height, cam.width
            idx = g[f"{tag}_sample_idx"]
            np.testing.assert_allclose(out["image"].reshape(-1, 3)[idx], g[f"{tag}_sample_rgb"], atol=1e-9)
            pad = np.zeros((-(-h // 16) * 16, -(-w // 16) * 16, 3))
            pad[:h, :w] = out["image"]
            sums = pad.reshape(pad.shape[0] // 16, 16, pad.shape[1] // 16, 16, 3).sum(axis=(1, 3))
            np.testing.assert_allclose(sums, g[f"{tag}_tile_sums"], atol=1e-7)


@pytest.mark.slow
def test_oracle_config1():
    """BASELINE config 1: 100K SH3 @256x256 (2,276,235 pairs), both engines."""
    g = load("config1")
    scene, cam = config1_scene()
    got = [sha(scene.positions), sha(scene.log_scales), sha(scene.rotations), sha(scene.opacities), sha(scene.sh)]
    assert got == [str(v) for v in g["scene_sha"]], "synthetic.random_scene no longer reproduces the reference scene"
    _check_big(g, scene, cam, ("ref", "cr2"), "f32")


@pytest.mark.slow
@pytest.mark.parametrize("frame", [0, 37])
def test_oracle_synth_1080p(frame):
    """SURVEY Appendix C scene (20K sample) on the 1080p orbit: partial bottom tile row."""
    g = load(f"synth20k_f{frame}")
    scene = synth(20_000, 0)
    got = [sha(scene.positions), sha(scene.log_scales), sha(scene.rotations), sha(scene.opacities), sha(scene.sh)]
    assert got == [str(v) for v in g["scene_sha"]]
    cam = camera_from(g)  # the reference re-normalised orbit_pose's quaternion
    np.testing.assert_allclose(cam.orientation, orbit_pose(frame).orientation, rtol=0, atol=1e-15)
    _check_big(g, scene, cam, ("ref", "cr2"), "summary")


def test_oracle_select_clusters_orbit():
    g = load("clusters_orbit")
    norm = (g["norm_mean"], float(g["norm_scale"][0]))
    for i in range(120):
        p = orbit_pose(i)
        cam = CameraPose(p.position, p.orientation, p.fov_x, p.fov_y, p.width, p.height)
        assert O.select_clusters(cam, g["centroids"], 4, 1.0, norm) == g["selections"][i].tolist()
    base = orbit_pose(0)
    for probe, want in zip(g["probes"], g["probe_selections"]):
        cam = CameraPose(position=probe[:3], orientation=probe[3:], fov_x=base.fov_x, fov_y=base.fov_y,
                         width=base.width, height=base.height)
        assert O.select_clusters(cam, g["centroids"], 4, 1.0, norm) == want.tolist()


def test_oracle_engine_table_complete():
    assert set(ENGINES) == {"ref", "cr1", "cr2", "cr4"}
    assert base_cfg({})["sh_degree"] == 3
