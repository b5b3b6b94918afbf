"""Golden vectors for the contribution harvest (compiler.py:196-311) from the
REFERENCE implementation (build container only, like make_golden.py):

    python tests/golden/make_harvest.py

Small random scenes seen by a short orbit: per-cluster harvests for several
k (1, 4, 32) and both engines, and one full compile_scene (clusters,
harvest, partition).  Writes tests/golden/harvest.npz; nothing here runs at
test time.
"""
import sys
from pathlib import Path

import numpy as np

REF = Path("/root/reference/pkg")
sys.path[:0] = [str(REF / "src"), str(REF / "tests")]
HERE = Path(__file__).resolve().parent

from seele.compiler import ClusterSpec, CompileParams, compile_scene, harvest_top_contributors  # noqa: E402
from seele.model import CameraPose  # noqa: E402
from seele.render import EngineConfig  # noqa: E402
from support import make_camera, random_scene  # noqa: E402


def orbit(n, w, h, r=3.0):
    poses = []
    for i in range(n):
        a = 2.0 * np.pi * i / n
        pos = np.array([r * np.sin(a), -0.3, -r * np.cos(a) + 4.0])
        # look at (0, 0, 4): camera +z toward the scene centre; yaw about y
        yaw = -a
        q = np.array([np.cos(yaw / 2.0), 0.0, np.sin(yaw / 2.0), 0.0])
        poses.append(CameraPose(position=pos, orientation=q, fov_x=1.0, fov_y=0.75, width=w, height=h))
    return poses


out = {}
cam = make_camera(80, 64)
scene = random_scene(np.random.default_rng(77), 600, sh_degree=2, camera=cam, scale_range=(0.01, 0.15),
                     opacity_range=(0.05, 0.95))
poses = [cam] + orbit(6, 80, 64)
out.update(positions=scene.positions, log_scales=scene.log_scales, rotations=scene.rotations,
           opacities=scene.opacities, sh=scene.sh, ids=scene.ids)
out["pose_position"] = np.stack([p.position for p in poses])
out["pose_orientation"] = np.stack([p.orientation for p in poses])
out["pose_fov"] = np.array([[p.fov_x, p.fov_y, p.near_clip] for p in poses])
out["pose_size"] = np.array([[p.width, p.height] for p in poses], dtype=np.int64)
cases = []
for k in (1, 4, 32):
    for eng in ("ref", "cr2"):
        cfg = EngineConfig(engine="ref") if eng == "ref" else EngineConfig(engine="cr", group_w=2)
        for members in ((0,), (0, 1, 2), (3, 4, 5, 6)):
            spec = ClusterSpec(centroid=np.zeros(6), member_indices=list(members),
                               member_poses=[poses[i] for i in members])
            ids = harvest_top_contributors(spec, scene, k, cfg)
            name = f"k{k}_{eng}_m{''.join(map(str, members))}"
            out["h_" + name] = ids
            cases.append(name)
            print(name, len(ids))
out["cases"] = np.array(cases)
cs = compile_scene(scene, poses, CompileParams(num_clusters=3, neighbors=1, top_k=8), seed=0)
out["c_shared"] = cs.shared_ids
out["c_discarded"] = cs.discarded_ids
for c, ex in enumerate(cs.exclusive_ids):
    out[f"c_exclusive{c}"] = ex
out["c_centroids"] = cs.centroids
out["c_assign"] = cs.pose_assignments
print("compile:", len(cs.shared_ids), [len(e) for e in cs.exclusive_ids], len(cs.discarded_ids))
np.savez_compressed(HERE / "harvest.npz", **out)
