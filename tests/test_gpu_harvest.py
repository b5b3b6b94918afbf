"""GPU contribution harvest (compiler.py:196-311) against
the reference's own harvests (tests/golden/harvest.npz, from
tests/golden/make_harvest.py): per-cluster top-k sets for k = 1, 4, 32 with
both engines, and a full compile (clusters, harvest, partition)."""
import numpy as np
import pytest

from helpers import GOLDEN
from paper_2503_05168_b200 import EngineConfig
from paper_2503_05168_b200.clusters import PoseCluster, compile_table, harvest_top_contributors
from paper_2503_05168_b200.errors import InvalidArgumentError
from paper_2503_05168_b200.model import CameraPose, SceneArrays

pytestmark = pytest.mark.gpu


def _load():
    with np.load(GOLDEN / "harvest.npz") as z:
        g = {k: z[k] for k in z.files}
    scene = SceneArrays(g["positions"], g["log_scales"], g["rotations"], g["opacities"], g["sh"], g["ids"])
    poses = [CameraPose(position=g["pose_position"][i], orientation=g["pose_orientation"][i],
                        fov_x=float(g["pose_fov"][i][0]), fov_y=float(g["pose_fov"][i][1]),
                        width=int(g["pose_size"][i][0]), height=int(g["pose_size"][i][1]),
                        near_clip=float(g["pose_fov"][i][2])) for i in range(len(g["pose_size"]))]
    return g, scene, poses


def test_cluster_harvests_match_reference():
    g, scene, poses = _load()
    for name in (str(c) for c in g["cases"]):
        k = int(name.split("_")[0][1:])
        eng = name.split("_")[1]
        members = [int(c) for c in name.split("_")[2][1:]]
        cfg = EngineConfig(engine="ref") if eng == "ref" else EngineConfig(engine="cr", group_w=2)
        spec = PoseCluster(np.zeros(6), members, [poses[i] for i in members])
        got = harvest_top_contributors(spec, scene, k, cfg)
        np.testing.assert_array_equal(got, g["h_" + name], err_msg=name)


def test_compile_matches_reference():
    g, scene, poses = _load()
    t = compile_table(scene, poses, n_clusters=3, neighbors=1, top_k=8, cfg=EngineConfig(sh_degree=3))
    np.testing.assert_allclose(t.centroids, g["c_centroids"], rtol=0, atol=1e-12)
    np.testing.assert_array_equal(t.pose_assignments, g["c_assign"])
    np.testing.assert_array_equal(t.shared_ids, g["c_shared"])
    np.testing.assert_array_equal(t.discarded_ids, g["c_discarded"])
    for c, ex in enumerate(t.exclusive_ids):
        np.testing.assert_array_equal(ex, g[f"c_exclusive{c}"])


def test_argument_checks():
    g, scene, poses = _load()
    spec = PoseCluster(np.zeros(6), [0], [poses[0]])
    with pytest.raises(InvalidArgumentError):
        harvest_top_contributors(spec, scene, 0)
    with pytest.raises(InvalidArgumentError):
        harvest_top_contributors(PoseCluster(np.zeros(6), [], []), scene, 4)
