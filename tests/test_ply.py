"""PLY ingest (io.py:36-152) against the reference's own
load_ply on the same files (tests/golden/ply.npz, from
tests/golden/make_ply.py): decoded arrays and error classes; and the
device planes path against the arrays."""
import numpy as np
import pytest

from helpers import GOLDEN
from paper_2503_05168_b200 import errors
from paper_2503_05168_b200.device import decode_planes
from paper_2503_05168_b200.plyio import load_ply, ply_to_planes


@pytest.fixture(scope="module")
def golden():
    with np.load(GOLDEN / "ply.npz") as z:
        return {k: z[k] for k in z.files}


def _write(tmp_path, g, name):
    f = tmp_path / f"{name}.ply"
    f.write_bytes(g[f"{name}_bytes"].tobytes())
    return f


def test_arrays_match_reference(golden, tmp_path):
    for name in (str(n) for n in golden["names"]):
        if f"{name}_error" in golden:
            continue
        sf = load_ply(_write(tmp_path, golden, name))
        a = sf.arrays()
        assert sf.sh_degree == int(golden[f"{name}_degree"])
        np.testing.assert_array_equal(a.positions, golden[f"{name}_positions"], err_msg=name)
        np.testing.assert_array_equal(a.log_scales, golden[f"{name}_log_scales"], err_msg=name)
        np.testing.assert_array_equal(a.opacities, golden[f"{name}_opacities"], err_msg=name)
        np.testing.assert_array_equal(a.sh, golden[f"{name}_sh"], err_msg=name)
        np.testing.assert_allclose(a.rotations, golden[f"{name}_rotations"], rtol=0, atol=2e-16, err_msg=name)


def test_errors_match_reference(golden, tmp_path):
    for name in (str(n) for n in golden["names"]):
        if f"{name}_error" not in golden:
            continue
        cls = getattr(errors, str(golden[f"{name}_error"]))
        with pytest.raises(cls):
            load_ply(_write(tmp_path, golden, name))
        with pytest.raises(cls):
            ply_to_planes(_write(tmp_path, golden, name))


def test_planes_decode_to_the_same_scene(golden, tmp_path):
    # the device layout holds the file's float32 values; decoded the container way they give load_ply's scene
    for name in ("deg0", "deg45", "mixed"):
        planes, ids, _ = ply_to_planes(_write(tmp_path, golden, name))
        dec = decode_planes(planes, ids)
        a = load_ply(_write(tmp_path, golden, name)).arrays()
        np.testing.assert_array_equal(dec.positions, a.positions)
        np.testing.assert_array_equal(dec.log_scales, a.log_scales)
        np.testing.assert_array_equal(dec.sh, a.sh)
        np.testing.assert_allclose(dec.opacities, a.opacities, rtol=1e-6)  # (mixed: the double logit is stored as float32)
        np.testing.assert_allclose(dec.rotations, a.rotations, rtol=0, atol=2e-16)


@pytest.mark.gpu
def test_device_ingest_renders_like_the_arrays(golden, tmp_path):
    from paper_2503_05168_b200 import DeviceScene, EngineConfig, render_frame
    from paper_2503_05168_b200.synthetic import make_camera

    f = _write(tmp_path, golden, "deg45")
    cam = make_camera(96, 64)
    cfg = EngineConfig(engine="cr", group_w=2)
    a = render_frame(load_ply(f).arrays(), cam, cfg)
    b = render_frame(DeviceScene.from_ply(f), cam, cfg)
    np.testing.assert_array_equal(a.contrib_count, b.contrib_count)
    assert float(np.abs(a.image - b.image).max()) <= 1e-6
