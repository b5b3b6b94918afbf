"""GPU image metrics (metrics.py:44-112) against the
reference's own psnr / ssim values (tests/golden/metrics.npz, from
tests/golden/make_metrics.py), and the reference's argument checks."""
import math

import numpy as np
import pytest

from helpers import GOLDEN
from paper_2503_05168_b200.errors import InvalidArgumentError
from paper_2503_05168_b200.metrics import psnr, ssim

pytestmark = pytest.mark.gpu


def test_match_reference_values():
    with np.load(GOLDEN / "metrics.npz") as z:
        g = {k: z[k] for k in z.files}
    for name in (str(n) for n in g["names"]):
        a, b = g[name + "_a"], g[name + "_b"]
        assert psnr(a, b) == pytest.approx(float(g[name + "_psnr"]), rel=1e-12), name
        assert ssim(a, b) == pytest.approx(float(g[name + "_ssim"]), rel=1e-12, abs=1e-14), name


def test_identical_and_errors():
    a = np.random.default_rng(0).random((20, 30, 3))
    assert math.isinf(psnr(a, a))
    assert ssim(a, a) == pytest.approx(1.0, abs=1e-12)
    with pytest.raises(InvalidArgumentError):
        psnr(a, a[:10])
    with pytest.raises(InvalidArgumentError):
        ssim(a[:8, :8], a[:8, :8])
