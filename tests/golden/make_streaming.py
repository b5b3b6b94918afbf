"""Golden vectors for streaming residency (residency.py:57-264) from the
REFERENCE implementation (build container only):

    python tests/golden/make_streaming.py

Compiles a small scene into 6 clusters (the reference's compile_scene over a
24-pose orbit), writes the container with the reference's writer, and runs
its ResidentRenderer over a trajectory (the orbit, then a jump back) with
several residency policies, recording per frame the cumulative stalls and
prefetch hits, and -- for the timing-independent configurations (no
prefetch) -- the resident bytes.  The container files go into the .npz so the
test reads exactly these bytes.  Writes tests/golden/streaming.npz.
"""
import json
import sys
import tempfile
from pathlib import Path

import numpy as np

REF = Path("/root/reference/pkg")
sys.path[:0] = [str(REF / "src"), str(REF / "tests")]
HERE = Path(__file__).resolve().parent

from seele import io as sio  # noqa: E402
from seele.compiler import CompileParams, compile_scene  # noqa: E402
from seele.model import CameraPose  # noqa: E402
from seele.render import EngineConfig  # noqa: E402
from seele.residency import ResidentRenderer  # noqa: E402
from support import make_camera, random_scene  # noqa: E402


def orbit(n, w, h, r=3.0):
    poses = []
    for i in range(n):
        a = 2.0 * np.pi * i / n
        pos = np.array([r * np.sin(a), -0.3, -r * np.cos(a) + 4.0])
        q = np.array([np.cos(-a / 2.0), 0.0, np.sin(-a / 2.0), 0.0])
        poses.append(CameraPose(position=pos, orientation=q, fov_x=1.0, fov_y=0.75, width=w, height=h))
    return poses


cam = make_camera(64, 48)
scene = random_scene(np.random.default_rng(31), 1500, sh_degree=1, camera=cam, scale_range=(0.01, 0.12),
                     opacity_range=(0.05, 0.95))
poses = orbit(24, 64, 48)
cs = compile_scene(scene, poses, CompileParams(num_clusters=6, neighbors=1, top_k=4, sh_degree=1), seed=0)
traj = poses + poses[:6][::-1] + poses[12:18]
out = {}
with tempfile.TemporaryDirectory() as d:
    sio.write_clustered_scene(cs, scene, d)
    files = sorted(p.name for p in Path(d).iterdir())
    for name in files:
        out["file_" + name] = np.frombuffer((Path(d) / name).read_bytes(), dtype=np.uint8)
    out["files"] = np.array(files)
    configs = {"imm_pf": dict(prefetch=True, evict=True, evict_policy="immediate"),
               "imm_nopf": dict(prefetch=False, evict=True, evict_policy="immediate"),
               "lru3_nopf": dict(prefetch=False, evict=True, evict_policy="lru", lru_capacity=3),
               "noevict_nopf": dict(prefetch=False, evict=False)}
    cfg = EngineConfig(sh_degree=1)
    for name, kw in configs.items():
        rr = ResidentRenderer(sio.load_clustered_scene(d), **kw)
        rows = []
        for cam_i in traj:
            st = rr.render_frame(cam_i, cfg).stats
            rows.append([st.stalls, st.prefetch_hits, st.resident_bytes])
        rr.close()
        out["stats_" + name] = np.array(rows, dtype=np.int64)
        print(name, out["stats_" + name][-1].tolist())
out["traj_position"] = np.stack([p.position for p in traj])
out["traj_orientation"] = np.stack([p.orientation for p in traj])
out["configs"] = np.array(json.dumps({k: v for k, v in configs.items()}))
np.savez_compressed(HERE / "streaming.npz", **out)
