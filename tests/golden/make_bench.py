"""Golden rows of the reference's comparative benchmark harness
(metrics.bench_compare, pkg/src/seele/metrics.py:172-243, and its CSV / JSON
writer write_report, :246-266) from the REFERENCE implementation:

    python tests/golden/make_bench.py

Same compiled scene as make_streaming.py (1500 SH1 splats, 6 clusters, the
reference's writer); the harness runs the four engine x scene configurations
over 8 orbit poses.  Stored: the container files, the poses, every row
(wall_ms excluded: a clock), and the CSV / JSON text write_report emits for
those rows with wall_ms set to 0.  Writes tests/golden/bench.npz.
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
from seele import metrics as smet  # noqa: E402
from seele.compiler import CompileParams, compile_scene  # noqa: E402
from seele.model import CameraPose  # noqa: E402
from seele.render import EngineConfig  # noqa: E402
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
traj = poses[::3]
configs = [{"engine": "ref", "scene": "flat"}, {"engine": "cr", "scene": "flat"},
           {"engine": "ref", "scene": "clustered"}, {"engine": "cr", "scene": "clustered"}]
base = EngineConfig(sh_degree=1, group_w=2)
out = {}
with tempfile.TemporaryDirectory() as d:
    sio.write_clustered_scene(cs, scene, d)
    files = sorted(p.name for p in Path(d).iterdir())
    for name in files:
        out["file_" + name] = np.frombuffer((Path(d) / name).read_bytes(), dtype=np.uint8)
    out["files"] = np.array(files)
    rows = smet.bench_compare(configs, traj, flat_scene=scene, clustered=sio.load_clustered_scene(d), base_cfg=base)
    for r in rows:
        r["wall_ms"] = 0.0
    csv_path = Path(d) / "report.csv"
    smet.write_report(rows, csv_path)
    out["report_csv"] = np.array(csv_path.read_text())
    out["report_json"] = np.array(csv_path.with_suffix(".json").read_text())
    keys = [c for c in smet.REPORT_COLUMNS if c not in ("config", "lpips")]
    out["columns"] = np.array(keys)
    out["rows"] = np.array([[float(r[k]) for k in keys] for r in rows])
    out["row_config"] = np.array([r["config"] for r in rows])
    for r in rows:
        print(r)
for k in ("positions", "log_scales", "rotations", "opacities", "sh"):
    out["scene_" + k] = np.asarray(getattr(scene, k))
out["scene_ids"] = np.asarray(scene.ids)
out["traj_position"] = np.stack([p.position for p in traj])
out["traj_orientation"] = np.stack([p.orientation for p in traj])
out["configs"] = np.array(json.dumps(configs))
np.savez_compressed(HERE / "bench.npz", **out)
