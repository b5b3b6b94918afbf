"""Golden vectors for ``render_frame(record_contributions=True)`` and its two
reference callers, from the REFERENCE implementation:

    python tests/golden/make_contrib.py

For scenes already pinned in tests/golden (their arrays and cameras are read
from the committed .npz files), runs the reference's
``render.render_frame(..., record_contributions=True)`` (render.py:172-233),
``metrics.contribution_cdf`` (metrics.py:115-161) and
``compiler.top_contributors_per_pixel`` (compiler.py:196-213) for several
engines and records:

* the dense contribution matrix, stored sparsely (row, column, value of
  every non-zero; rows are plan refs, columns pixels) plus its shape;
* ``contribution_ids``;
* the ContributionCurve fields (aggregate, per-pixel totals, fraction for
  99 %, and the per-pixel curves flattened with their lengths -- lengths
  only for the largest case);
* the top-k sets for k in (1, 4, 32).

Writes tests/golden/contrib.npz.  Nothing here runs at test time.
"""
from __future__ import annotations

import sys
from pathlib import Path

import numpy as np

REF = Path("/root/reference/pkg")
sys.path[:0] = [str(REF / "src"), str(REF / "tests")]
HERE = Path(__file__).resolve().parent

from seele.compiler import top_contributors_per_pixel  # noqa: E402
from seele.metrics import contribution_cdf  # noqa: E402
from seele.model import CameraPose, SceneArrays  # noqa: E402
from seele.render import EngineConfig, render_frame  # noqa: E402

CASES = ["rand64_s0", "rand64_s2", "accept_003", "edges80x48", "odd100x70"]
ENGINES = {"ref": dict(engine="ref"), "cr2": dict(engine="cr", group_w=2), "cr4": dict(engine="cr", group_w=4)}
KS = (1, 4, 32)


def main():
    out = {"cases": np.array(CASES), "engines": np.array(list(ENGINES)), "ks": np.array(KS)}
    for name in CASES:
        with np.load(HERE / f"{name}.npz") as z:
            g = {k: z[k] for k in z.files}
        scene = SceneArrays(g["positions"], g["log_scales"], g["rotations"], g["opacities"], g["sh"], g["ids"])
        fov = g["cam_fov"]
        w, h = (int(v) for v in g["cam_size"])
        cam = CameraPose(position=g["cam_position"], orientation=g["cam_orientation"], fov_x=float(fov[0]),
                         fov_y=float(fov[1]), width=w, height=h, near_clip=float(fov[2]))
        flags = g.get("cfg_flags", np.array([1, 3]))
        bg = tuple(float(v) for v in g.get("cfg_background", np.zeros(3)))
        for tag, kw in ENGINES.items():
            cfg = EngineConfig(background=bg, opacity_aware_filter=bool(flags[0]), sh_degree=int(flags[1]), **kw)
            res = render_frame(scene, cam, cfg, record_contributions=True)
            m = res.contributions
            r, c = np.nonzero(m)
            p = f"{name}:{tag}:"
            out[p + "shape"] = np.array(m.shape, dtype=np.int64)
            out[p + "rows"] = r.astype(np.int32)
            out[p + "cols"] = c.astype(np.int32)
            out[p + "vals"] = m[r, c]
            out[p + "ids"] = np.asarray(res.contribution_ids, dtype=np.int64)
            cur = contribution_cdf(scene, cam, cfg, keep_per_pixel=True)
            out[p + "aggregate"] = cur.aggregate
            out[p + "totals"] = cur.per_pixel_totals
            out[p + "frac99"] = np.array([cur.fraction_for_99])
            out[p + "curve_len"] = np.array([len(v) for v in cur.per_pixel_curves], dtype=np.int64)
            if name != "odd100x70":  # (the largest case keeps only the curve lengths: file size)
                out[p + "curves"] = np.concatenate(cur.per_pixel_curves) if cur.per_pixel_curves else np.zeros(0)
            for k in KS:
                out[p + f"top{k}"] = top_contributors_per_pixel(m, res.contribution_ids, k)
            print(name, tag, m.shape, len(r), cur.fraction_for_99)
    np.savez_compressed(HERE / "contrib.npz", **out)


if __name__ == "__main__":
    main()
