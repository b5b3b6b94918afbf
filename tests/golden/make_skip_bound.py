"""Golden vectors for frame_skip_bound (render.py:236-256, rasterize.py:325-377)
from the REFERENCE implementation (build container only, like make_golden.py):

    python tests/golden/make_skip_bound.py

Scenes: the reference's own test_error_bounded_by_skip_bound scenes
(test_rasterize.py:219-232: 48 splats, scale 0.01-0.2, default camera) for a
few seeds, two denser 96x64 scenes (group widths 2 and 4) and a dense one on
which the reference's own bound is exceeded at a few pixels.  Writes
tests/golden/skipbound.npz; nothing here runs at test time.
"""
import sys
from pathlib import Path

import numpy as np

REF = Path("/root/reference/pkg")
sys.path[:0] = [str(REF / "src"), str(REF / "tests")]
HERE = Path(__file__).resolve().parent

from seele.render import EngineConfig, frame_skip_bound, render_frame  # noqa: E402
from support import make_camera, random_scene  # noqa: E402

out = {}
cases = []
cam0 = make_camera()
for seed in (0, 3, 7, 11):
    cases.append((f"t{seed}", random_scene(np.random.default_rng(seed + 400), 48, scale_range=(0.01, 0.2)), cam0, 2))
cam1 = make_camera(96, 64)
for seed, w in ((1, 2), (2, 4)):
    cases.append((f"d{seed}", random_scene(np.random.default_rng(900 + seed), 400, sh_degree=2, camera=cam1,
                                           scale_range=(0.01, 0.12), opacity_range=(0.05, 0.9)), cam1, w))
# a dense scene on which the reference's bound is itself exceeded (by <= 1.6e-5 at 3 pixels): the GPU must
# reproduce the reference's values, not a tighter or looser bound
cases.append(("v3000", random_scene(np.random.default_rng(42), 3000, sh_degree=2, camera=cam1,
                                    scale_range=(0.005, 0.1), opacity_range=(0.05, 0.95)), cam1, 2))
names = []
for name, sc, cam, w in cases:
    cfg = EngineConfig(engine="cr", group_w=w)
    bound = frame_skip_bound(sc, cam, cfg)
    img_ref = render_frame(sc, cam, EngineConfig(engine="ref")).image
    img_cr = render_frame(sc, cam, cfg).image
    over = int((np.abs(img_cr - img_ref).max(axis=2) > bound + 1e-12).sum())
    p = name + "_"
    out.update({p + "positions": sc.positions, p + "log_scales": sc.log_scales, p + "rotations": sc.rotations,
                p + "opacities": sc.opacities, p + "sh": sc.sh, p + "ids": sc.ids,
                p + "cam_position": cam.position, p + "cam_orientation": cam.orientation,
                p + "cam_fov": np.array([cam.fov_x, cam.fov_y, cam.near_clip]),
                p + "cam_size": np.array([cam.width, cam.height], dtype=np.int64),
                p + "group_w": np.array(w), p + "bound": bound})
    names.append(name)
    out[p + "violations"] = np.array(over)
    print(name, bound.shape, float(bound.max()), int((bound > 0).sum()), "pixels over the bound:", over)
out["names"] = np.array(names)
np.savez_compressed(HERE / "skipbound.npz", **out)
