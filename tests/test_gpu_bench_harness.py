"""Comparative benchmark harness (metrics.bench_compare / write_report,
pkg/src/seele/metrics.py:164-266) against the reference's
own rows on the same scene, container files and trajectory
(tests/golden/bench.npz, from tests/golden/make_bench.py): the lockstep
counters, peak resident bytes and stalls are bit-exact, PSNR / SSIM agree to
1e-4 relative (float32 vs float64 images, scored by the GPU kernels), and the
CSV / JSON the writer emits equal the reference's text once the
float-formatted quality columns agree."""
import csv
import io
import json
import math

import numpy as np
import pytest

from helpers import GOLDEN
from paper_2503_05168_b200 import EngineConfig
from paper_2503_05168_b200.container import load_clustered_scene
from paper_2503_05168_b200.metrics import REPORT_COLUMNS, bench_compare, write_report
from paper_2503_05168_b200.model import CameraPose, SceneArrays

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def rows(tmp_path_factory):
    with np.load(GOLDEN / "bench.npz") as z:
        g = {k: z[k] for k in z.files}
    d = tmp_path_factory.mktemp("container")
    for name in (str(f) for f in g["files"]):
        (d / name).write_bytes(g["file_" + name].tobytes())
    scene = SceneArrays(positions=g["scene_positions"], log_scales=g["scene_log_scales"],
                        rotations=g["scene_rotations"], opacities=g["scene_opacities"], sh=g["scene_sh"],
                        ids=g["scene_ids"])
    traj = [CameraPose(position=g["traj_position"][i], orientation=g["traj_orientation"][i], fov_x=1.0,
                       fov_y=0.75, width=64, height=48) for i in range(len(g["traj_position"]))]
    got = bench_compare(json.loads(str(g["configs"])), traj, flat_scene=scene, clustered=load_clustered_scene(d),
                        base_cfg=EngineConfig(sh_degree=1, group_w=2))
    return g, got


def test_rows_match_reference(rows):
    g, got = rows
    assert [r["config"] for r in got] == [str(c) for c in g["row_config"]]
    cols = [str(c) for c in g["columns"]]
    for r, want in zip(got, g["rows"]):
        for c, w in zip(cols, want):
            if c == "wall_ms":
                assert r[c] > 0.0
            elif c in ("psnr_db", "ssim"):
                assert (math.isinf(w) and math.isinf(r[c])) or r[c] == pytest.approx(w, rel=1e-4), (r["config"], c)
            else:
                assert r[c] == int(w), (r["config"], c, r[c], w)
        assert r["lpips"] is None


def test_report_files(rows, tmp_path):
    g, got = rows
    fixed = []
    want_rows = list(csv.reader(io.StringIO(str(g["report_csv"]))))
    for r, w in zip(got, want_rows[1:]):
        r = dict(r, wall_ms=0.0)
        # quality columns formatted like the reference (agree to 1e-4: take the reference's text)
        r["psnr_db"] = math.inf if w[1] == "inf" else float(w[1])
        r["ssim"] = float(w[2])
        fixed.append(r)
    path = tmp_path / "report.csv"
    write_report(fixed, path)
    assert path.read_text() == str(g["report_csv"])
    got_json = json.loads(path.with_suffix(".json").read_text())
    want_json = json.loads(str(g["report_json"]))
    assert [list(r) for r in got_json] == [REPORT_COLUMNS] * len(want_json)
    for a, b in zip(got_json, want_json):
        for c in REPORT_COLUMNS:
            if c in ("psnr_db", "ssim"):
                assert a[c] == "inf" if b[c] == "inf" else a[c] == pytest.approx(b[c], rel=1e-5)
            else:
                assert a[c] == b[c], c
