"""Certify the C oracle against the Python reference on one full C2 frame
(SURVEY 8(c)): synth(1_000_000, 0), orbit frame 0 at 1920x1080, Seele engine
(cr w=2).  Runs only in the build container (imports /root/reference read-only);
writes profiles/r02/c2_oracle_vs_reference.json.

    python tools/certify_c2.py
"""
from __future__ import annotations

import hashlib
import json
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
REF = Path("/root/reference/pkg")
sys.path[:0] = [str(REF / "src"), str(ROOT)]

from seele.model import CameraPose, SceneArrays  # noqa: E402
from seele.render import EngineConfig as RefConfig  # noqa: E402
from seele.render import plan_frame, render_frame  # noqa: E402

from oracle import oracle as O  # noqa: E402
from paper_2503_05168_b200.render import EngineConfig  # noqa: E402
from paper_2503_05168_b200.synthetic import orbit_pose, synth  # noqa: E402

STATS = ("alpha_eval_steps", "blend_steps", "leader_eval_steps", "warp_steps", "tile_pairs", "culled_near",
         "dropped_degenerate")


def sha(a) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def main() -> None:
    mine = synth(1_000_000, 0)
    p = orbit_pose(0)
    scene = SceneArrays(mine.positions, mine.log_scales, mine.rotations, mine.opacities, mine.sh, mine.ids)
    cam = CameraPose(position=p.position, orientation=p.orientation, fov_x=p.fov_x, fov_y=p.fov_y,
                     width=p.width, height=p.height, near_clip=p.near_clip)
    out = {"config": "C2: synth(1_000_000, 0), orbit frame 0, 1920x1080, engine cr w=2"}

    t0 = time.perf_counter()
    oo = O.render(mine, p, EngineConfig(engine="cr", group_w=2))
    out["oracle_seconds"] = time.perf_counter() - t0
    opl = oo["plan"]

    t0 = time.perf_counter()
    rplan = plan_frame(scene, cam, RefConfig(engine="cr", group_w=2))
    out["reference_plan_seconds"] = time.perf_counter() - t0
    t0 = time.perf_counter()
    rres = render_frame(scene, cam, RefConfig(engine="cr", group_w=2))
    out["reference_render_seconds"] = time.perf_counter() - t0

    ref_pairs = np.stack([rplan.sorted_pairs["tile_id"], rplan.ids[rplan.sorted_pairs["gaussian_ref"]]], 1)
    ora_pairs = np.stack([opl["pair_tile"], opl["ids"][opl["pair_ref"]]], 1)
    out["pairs"] = int(len(ref_pairs))
    out["pairs_equal"] = bool(ref_pairs.shape == ora_pairs.shape and np.array_equal(ref_pairs.astype(np.int64),
                                                                                    ora_pairs.astype(np.int64)))
    out["pairs_sha_reference"] = sha(ref_pairs.astype(np.int64))
    out["ids_equal"] = bool(np.array_equal(np.asarray(rplan.ids, np.int64), np.asarray(opl["ids"], np.int64)))
    rs = np.zeros(opl["tiles_x"] * opl["tiles_y"], np.int64)
    re = np.zeros_like(rs)
    for r in rplan.ranges:
        rs[r.tile_id], re[r.tile_id] = r.start, r.end
    out["ranges_equal"] = bool(np.array_equal(rs, np.asarray(opl["range_start"], np.int64))
                               and np.array_equal(re, np.asarray(opl["range_end"], np.int64)))
    rstats = rres.stats.as_dict()
    out["stats_reference"] = {k: int(rstats[k]) for k in STATS}
    out["stats_oracle"] = {k: int(oo["stats"][k]) for k in STATS}
    out["stats_equal"] = out["stats_reference"] == out["stats_oracle"]
    img_r = np.asarray(rres.image, np.float64)
    img_o = np.asarray(oo["image"], np.float64).reshape(img_r.shape)
    out["image_max_abs"] = float(np.abs(img_r - img_o).max())
    out["pass"] = bool(out["pairs_equal"] and out["ids_equal"] and out["ranges_equal"] and out["stats_equal"]
                       and out["image_max_abs"] <= 1e-9)
    dst = ROOT / "profiles" / "r02" / "c2_oracle_vs_reference.json"
    dst.write_text(json.dumps(out, indent=1) + "\n")
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
