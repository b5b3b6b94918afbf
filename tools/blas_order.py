"""Which operation order does the REFERENCE's `world_to_view @ (position -
cam.position)` (preprocess.py:100) round to in this container?

numpy sends the 3x3 @ 3 product to OpenBLAS dgemv (DYNAMIC_ARCH; the
Haswell kernel on this Xeon), so the rounding is a property of the BLAS
kernel, not of the formula.  This script evaluates candidate orders exactly
(fractions) against numpy on the Appendix-C scene's fp32 positions for a few
orbit cameras.  Result here: t[r] = fma(w[r][2], d[2], fma(w[r][1], d[1],
w[r][0] * d[0])) for every component of every splat tested; the plain
left-to-right sum differs for ~25 % of depths.  The oracle and K1 use the
fma order.  Build-container tool only (imports the reference read-only).

    python tools/blas_order.py
"""
import sys
from fractions import Fraction
from pathlib import Path

import numpy as np

sys.path[:0] = ["/root/reference/pkg/src", str(Path(__file__).resolve().parent.parent)]
from seele.model import CameraPose  # noqa: E402

from paper_2503_05168_b200.synthetic import orbit, synth  # noqa: E402


def fma(a, b, c):
    return float(Fraction(a) * Fraction(b) + Fraction(c))


def main(n: int = 2000):
    poses = orbit(120, 1920, 1080)
    pos = synth(20000, 0).positions.astype(np.float32).astype(np.float64)
    for f in (0, 37, 90):
        c = poses[f]
        cam = CameraPose(c.position, c.orientation, c.fov_x, c.fov_y, c.width, c.height)
        w = cam.rotation_matrix().T
        hits = {"fma_left_to_right": 0, "plain_left_to_right": 0}
        for i in range(n):
            d = pos[i] - cam.position
            t = w @ d
            for r in range(3):
                hits["fma_left_to_right"] += t[r] == fma(w[r][2], d[2], fma(w[r][1], d[1], w[r][0] * d[0]))
                hits["plain_left_to_right"] += t[r] == (w[r][0] * d[0] + w[r][1] * d[1]) + w[r][2] * d[2]
        print(f"orbit frame {f}: of {3 * n} components", {k: int(v) for k, v in hits.items()})


if __name__ == "__main__":
    main()
