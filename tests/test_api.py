"""CPU-side checks: API surface, validation/error behaviour of the reference
(render.py:45-51, model.py validators), container encode/decode, and the
C-ABI library (loads, exports every symbol of include/seele_b200.h, rejects
bad arguments with the documented status codes before touching a GPU)."""
import ctypes
import math
import re
from pathlib import Path

import numpy as np
import pytest

import paper_2503_05168_b200 as pkg
from paper_2503_05168_b200 import _native
from paper_2503_05168_b200.device import decode_planes, encode_planes, validate_arrays
from paper_2503_05168_b200.errors import DataError, InvalidArgumentError, SeeleError, UserInputError
from paper_2503_05168_b200.model import CameraPose, Gaussian3D, PixelGroup, SceneArrays
from paper_2503_05168_b200.render import EngineConfig
from paper_2503_05168_b200.synthetic import make_camera, random_scene

ROOT = Path(__file__).resolve().parent.parent
REFERENCE_EXPORTS = ["ALPHA_THRESHOLD", "GAMMA_THRESHOLD", "TILE_SIZE", "CameraPose", "EngineConfig", "Gaussian3D",
                     "PixelGroup", "ProjectedGaussian", "RenderResult", "SceneArrays", "covariance3d", "render_frame",
                     "sh_to_color", "__version__"]


def test_reference_exports_present():
    for name in REFERENCE_EXPORTS:
        assert hasattr(pkg, name), name


@pytest.mark.parametrize("kw", [dict(engine="gpu"), dict(group_w=3), dict(threads=0), dict(precision="half"),
                                dict(sh_degree=4), dict(tile_size=8)])
def test_engine_config_rejects(kw):
    with pytest.raises(InvalidArgumentError):
        EngineConfig(**kw)


def test_error_hierarchy():
    assert issubclass(InvalidArgumentError, UserInputError) and issubclass(InvalidArgumentError, ValueError)
    assert issubclass(DataError, SeeleError)


def test_camera_validation():
    with pytest.raises(DataError):
        make_camera(8, 64)
    with pytest.raises(DataError):
        CameraPose(position=np.zeros(3), orientation=np.zeros(4), fov_x=0.8, fov_y=0.8, width=64, height=64)
    with pytest.raises(DataError):
        make_camera(fov=math.pi)
    cam = make_camera(64, 64, orientation=(2.0, 0, 0, 0))
    np.testing.assert_array_equal(cam.orientation, [1.0, 0, 0, 0])


def test_gaussian_and_group_validation():
    with pytest.raises(DataError):
        Gaussian3D(np.zeros(3), np.zeros(3), np.array([1.0, 0, 0, 0]), 1.0, np.zeros((3, 16)))
    with pytest.raises(InvalidArgumentError):
        PixelGroup((1, 0), 2)


def test_scene_validation_catches_bad_splats():
    scene = random_scene(np.random.default_rng(0), 10)
    validate_arrays(scene)
    bad = SceneArrays(scene.positions.copy(), scene.log_scales.copy(), scene.rotations.copy(),
                      scene.opacities.copy(), scene.sh.copy(), scene.ids)
    bad.opacities[3] = 1.0
    with pytest.raises(DataError, match="splat 3"):
        validate_arrays(bad)
    bad.opacities[3] = 0.5
    bad.rotations[5] = 0.0
    with pytest.raises(DataError, match="splat 5"):
        validate_arrays(bad)
    bad.rotations[5] = scene.rotations[5]
    bad.log_scales[2, 1] = 800.0
    with pytest.raises(DataError, match="overflows"):
        validate_arrays(bad)


def test_planes_roundtrip_matches_container_decode():
    """encode_planes/decode_planes == io._encode_chunk/_decode_chunk semantics."""
    scene = random_scene(np.random.default_rng(1), 257, sh_degree=3)
    planes = encode_planes(scene)
    assert planes.shape == (15, 257, 4) and planes.dtype == np.float32
    dec = decode_planes(planes, scene.ids)
    np.testing.assert_array_equal(dec.positions, scene.positions.astype(np.float32).astype(np.float64))
    np.testing.assert_array_equal(dec.sh, scene.sh.astype(np.float32).astype(np.float64))
    np.testing.assert_allclose(dec.opacities, scene.opacities, rtol=1e-6)
    np.testing.assert_allclose(np.linalg.norm(dec.rotations, axis=1), 1.0, rtol=1e-15)


# ---- C-ABI -----------------------------------------------------------------

def _header_symbols():
    text = (ROOT / "include" / "seele_b200.h").read_text()
    return sorted(set(re.findall(r"^\s*(?:int|int32_t|int64_t|size_t|const char \*)\s*(seele_\w+)\s*\(", text, re.M)))


def test_library_exports_header_symbols():
    lib = _native.load()
    declared = _header_symbols()
    assert set(declared) == set(_native.EXPORTED_SYMBOLS)
    for name in declared:
        assert hasattr(lib, name), name
    assert lib.seele_abi_version() == _native.ABI_VERSION


def test_workspace_bytes_monotone():
    lib = _native.load()
    a = lib.seele_workspace_bytes(1000, 10000, 256, 256)
    b = lib.seele_workspace_bytes(2000, 10000, 256, 256)
    c = lib.seele_workspace_bytes(2000, 20000, 1920, 1080)
    assert 0 < a < b < c


def _render_status(cfg=None, cam=None, n_ranges=1):
    lib = _native.load()
    cfg = cfg or EngineConfig()
    cam = cam or make_camera()
    sc = _native.Scene()
    sc.layout, sc.n = _native.LAYOUT_F64, 0
    cfgc = _native.config_struct(cfg)
    camc = _native.camera_struct(cam)
    return cfgc, camc, sc, lib


def test_render_rejects_bad_arguments_without_gpu():
    cfgc, camc, sc, lib = _render_status()
    dummy = ctypes.c_void_p(16)
    cfgc.engine = 7
    rc = lib.seele_render(ctypes.byref(sc), dummy, 1, ctypes.byref(camc), ctypes.byref(cfgc), dummy, 1 << 30, 10, 10,
                          dummy, None, dummy, None)
    assert rc == 1 and b"engine" in lib.seele_last_error()
    cfgc.engine, cfgc.group_w = 1, 3
    rc = lib.seele_render(ctypes.byref(sc), dummy, 1, ctypes.byref(camc), ctypes.byref(cfgc), dummy, 1 << 30, 10, 10,
                          dummy, None, dummy, None)
    assert rc == 1 and b"group width" in lib.seele_last_error()
    cfgc.group_w = 2
    camc.width = 8
    rc = lib.seele_render(ctypes.byref(sc), dummy, 1, ctypes.byref(camc), ctypes.byref(cfgc), dummy, 1 << 30, 10, 10,
                          dummy, None, dummy, None)
    assert rc == 2
    camc.width = 64
    rc = lib.seele_render(ctypes.byref(sc), dummy, 0, ctypes.byref(camc), ctypes.byref(cfgc), dummy, 1 << 30, 10, 10,
                          dummy, None, dummy, None)
    assert rc == 1
    rc = lib.seele_render(ctypes.byref(sc), dummy, 1, ctypes.byref(camc), ctypes.byref(cfgc), dummy, 16, 10, 10,
                          dummy, None, dummy, None)
    assert rc == 1 and b"workspace too small" in lib.seele_last_error()


def test_select_rejects_m_ge_n():
    lib = _native.load()
    camc = _native.camera_struct(make_camera())
    dummy = ctypes.c_void_p(16)
    mean = (ctypes.c_double * 3)(0, 0, 0)
    rc = lib.seele_select_clusters(ctypes.byref(camc), dummy, 4, 4, 1.0, mean, 1.0, dummy, dummy, dummy, None)
    assert rc == 1 and b"m must be" in lib.seele_last_error()


def test_warp_cost_and_tile_intersection_mirror_the_reference():
    """rasterize.py:36-70 (WarpCost, FrameStats.add_cost), preprocess.py:59-65 (TileIntersection),
    rasterize.py:154-156 (_check_sorted)."""
    import numpy as np
    import pytest

    from paper_2503_05168_b200 import FrameStats, TileIntersection, WarpCost
    from paper_2503_05168_b200.errors import ContractViolationError
    from paper_2503_05168_b200.render import INTERSECTION_DTYPE, check_sorted_depths

    total = WarpCost()
    total.add(WarpCost(alpha_eval_steps=3, blend_steps=2, leader_eval_steps=1, warp_steps=4))
    total.add(WarpCost(alpha_eval_steps=1, blend_steps=1, leader_eval_steps=0, warp_steps=2))
    st = FrameStats(tile_pairs=7)
    st.add_cost(total)
    assert (st.alpha_eval_steps, st.blend_steps, st.leader_eval_steps, st.warp_steps, st.tile_pairs) == (4, 3, 1, 6, 7)
    rec = np.zeros(1, dtype=INTERSECTION_DTYPE)
    rec[0] = (5, 11, 2.5)
    ti = TileIntersection.from_record(rec[0])
    assert ti == TileIntersection(tile_id=5, gaussian_ref=11, depth=2.5)
    with pytest.raises(Exception):
        ti.depth = 1.0  # frozen like the reference's
    check_sorted_depths(np.array([1.0, 1.0, 2.0]))
    with pytest.raises(ContractViolationError):
        check_sorted_depths(np.array([2.0, 1.0]))
