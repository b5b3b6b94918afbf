"""Golden vectors for the GPU image metrics (metrics.py:44-112) from the
REFERENCE implementation (build container only):

    python tests/golden/make_metrics.py

Pairs of (H, W, 3) images -- random, smooth, nearly equal, and a rendered
frame pair (reference vs contribution-aware engine) -- with the reference's
psnr and ssim.  Writes tests/golden/metrics.npz; nothing runs at test time.
"""
import sys
from pathlib import Path

import numpy as np

REF = Path("/root/reference/pkg")
sys.path[:0] = [str(REF / "src"), str(REF / "tests")]
HERE = Path(__file__).resolve().parent

from seele.metrics import psnr, ssim  # noqa: E402
from seele.render import EngineConfig, render_frame  # noqa: E402
from support import make_camera, random_scene  # noqa: E402

rng = np.random.default_rng(5)
pairs = []
a = rng.random((37, 53, 3))
pairs.append(("random", a, rng.random((37, 53, 3))))
yy, xx = np.mgrid[0:64, 0:96]
s = np.stack([np.sin(xx / 7.0), np.cos(yy / 5.0), np.sin((xx + yy) / 11.0)], axis=2) * 0.5 + 0.5
pairs.append(("smooth", s, np.clip(s + 0.01 * rng.standard_normal(s.shape), 0, 1)))
pairs.append(("near", s, s + 1e-7 * rng.standard_normal(s.shape)))
cam = make_camera(64, 48)
scene = random_scene(np.random.default_rng(9), 800, camera=cam, opacity_range=(0.05, 0.95))
r = render_frame(scene, cam, EngineConfig(engine="ref")).image
c = render_frame(scene, cam, EngineConfig(engine="cr", group_w=4)).image
pairs.append(("render", r, c))
out = {}
for name, x, y in pairs:
    out[name + "_a"], out[name + "_b"] = x, y
    out[name + "_psnr"] = np.array(psnr(x, y))
    out[name + "_ssim"] = np.array(ssim(x, y))
    print(name, float(out[name + "_psnr"]), float(out[name + "_ssim"]))
out["names"] = np.array([p[0] for p in pairs])
np.savez_compressed(HERE / "metrics.npz", **out)
