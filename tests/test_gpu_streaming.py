"""Streaming residency (residency.py:57-264) against the
reference's ResidentRenderer on the same container files and trajectory
(tests/golden/streaming.npz, from tests/golden/make_streaming.py): per-frame
stalls and prefetch hits for four policies, resident bytes where the
reference is timing-independent (no prefetch), and images / contributor
counts identical to the fully resident renderer."""
import json

import numpy as np
import pytest

from helpers import GOLDEN
from paper_2503_05168_b200 import EngineConfig
from paper_2503_05168_b200.container import load_clustered_scene
from paper_2503_05168_b200.model import CameraPose
from paper_2503_05168_b200.residency import ResidentRenderer
from paper_2503_05168_b200.streaming import StreamingRenderer, predict_pose

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def setup(tmp_path_factory):
    with np.load(GOLDEN / "streaming.npz") as z:
        g = {k: z[k] for k in z.files}
    d = tmp_path_factory.mktemp("container")
    for name in (str(f) for f in g["files"]):
        (d / name).write_bytes(g["file_" + name].tobytes())
    traj = [CameraPose(position=g["traj_position"][i], orientation=g["traj_orientation"][i], fov_x=1.0,
                       fov_y=0.75, width=64, height=48) for i in range(len(g["traj_position"]))]
    return g, d, traj


@pytest.mark.parametrize("name", ["imm_pf", "imm_nopf", "lru3_nopf", "noevict_nopf"])
def test_policy_counters_match_reference(setup, name):
    g, d, traj = setup
    kw = json.loads(str(g["configs"]))[name]
    want = g["stats_" + name]
    cfg = EngineConfig(sh_degree=1)
    resident = ResidentRenderer(load_clustered_scene(d))
    with StreamingRenderer(load_clustered_scene(d), **kw) as sr:
        for i, cam in enumerate(traj):
            res = sr.render_frame(cam, cfg)
            assert [res.stats.stalls, res.stats.prefetch_hits] == want[i][:2].tolist(), (name, i)
            if "nopf" in name:
                assert res.stats.resident_bytes == int(want[i][2]), (name, i)
            if i % 5 == 0:  # same working set, same order: identical frames
                full = resident.render_frame(cam, cfg)
                np.testing.assert_array_equal(res.contrib_count, full.contrib_count)
                np.testing.assert_array_equal(res.image, full.image)


def test_predict_pose_extrapolates():
    a = CameraPose(position=np.zeros(3), orientation=np.array([1.0, 0, 0, 0]), fov_x=1.0, fov_y=0.8, width=32,
                   height=32)
    q = np.array([np.cos(0.05), 0.0, np.sin(0.05), 0.0])
    b = CameraPose(position=np.array([0.1, 0, 0]), orientation=q, fov_x=1.0, fov_y=0.8, width=32, height=32)
    p = predict_pose(a, b)
    np.testing.assert_allclose(p.position, [0.2, 0, 0])
    np.testing.assert_allclose(p.orientation, [np.cos(0.1), 0.0, np.sin(0.1), 0.0], atol=1e-12)
