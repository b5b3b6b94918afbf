"""render_frame(..., record_contributions=True) on the GPU (render.py:172-193,
229-233) and the reference's two callers of it -- metrics.contribution_cdf
(metrics.py:115-161) and compiler.top_contributors_per_pixel
(compiler.py:196-213) -- run against the drop-in, compared with the
reference's own outputs on the same scenes (tests/golden/contrib.npz, made by
tests/golden/make_contrib.py).

Bar: the set of (splat, pixel) blends (the non-zero pattern of the dense
matrix), the ids and the top-k sets bit-exact; weights, cumulative curves and
totals within 1e-12 relative (fp64 exp of the device vs numpy); the 99 %
ranks exact (fraction_for_99 to 1e-12)."""
import numpy as np
import pytest

from helpers import GOLDEN, camera_from, config_for, load, scene_from
from paper_2503_05168_b200 import render
from paper_2503_05168_b200.clusters import top_contributors_per_pixel
from paper_2503_05168_b200.errors import InvalidArgumentError
from paper_2503_05168_b200.metrics import contribution_cdf
from paper_2503_05168_b200.render import render_frame

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def golden():
    with np.load(GOLDEN / "contrib.npz") as z:
        return {k: z[k] for k in z.files}


def _cases(g):
    return [(str(c), str(e)) for c in g["cases"] for e in g["engines"]]


def _setup(name, tag):
    s = load(name)
    return scene_from(s), camera_from(s), config_for(s, tag)


def test_contribution_matrix_vs_reference(golden):
    for name, tag in _cases(golden):
        scene, cam, cfg = _setup(name, tag)
        p = f"{name}:{tag}:"
        res = render_frame(scene, cam, cfg, record_contributions=True)
        m = res.contributions
        assert m.shape == tuple(golden[p + "shape"]), (name, tag)
        np.testing.assert_array_equal(res.contribution_ids, golden[p + "ids"])
        r, c = np.nonzero(m)
        np.testing.assert_array_equal(r, golden[p + "rows"])
        np.testing.assert_array_equal(c, golden[p + "cols"])
        np.testing.assert_allclose(m[r, c], golden[p + "vals"], rtol=1e-12, atol=0)
        # the per-pixel contributor count is the column's non-zero count
        np.testing.assert_array_equal((m > 0).sum(0).reshape(cam.height, cam.width), res.contrib_count)


def test_contribution_cdf_vs_reference(golden):
    for name, tag in _cases(golden):
        scene, cam, cfg = _setup(name, tag)
        p = f"{name}:{tag}:"
        cur = contribution_cdf(scene, cam, cfg, keep_per_pixel=True)
        np.testing.assert_allclose(cur.aggregate, golden[p + "aggregate"], rtol=1e-12, atol=1e-15)
        np.testing.assert_allclose(cur.per_pixel_totals, golden[p + "totals"], rtol=1e-12, atol=0)
        assert cur.fraction_for_99 == pytest.approx(float(golden[p + "frac99"][0]), rel=1e-12)
        np.testing.assert_array_equal([len(v) for v in cur.per_pixel_curves], golden[p + "curve_len"])
        if p + "curves" in golden:
            got = np.concatenate(cur.per_pixel_curves) if cur.per_pixel_curves else np.zeros(0)
            np.testing.assert_allclose(got, golden[p + "curves"], rtol=1e-12, atol=0)


def test_top_contributors_vs_reference(golden):
    for name, tag in _cases(golden):
        scene, cam, cfg = _setup(name, tag)
        p = f"{name}:{tag}:"
        res = render_frame(scene, cam, cfg, record_contributions=True)
        for k in golden["ks"]:
            got = top_contributors_per_pixel(res.contributions, res.contribution_ids, int(k))
            np.testing.assert_array_equal(got, golden[p + f"top{int(k)}"], err_msg=f"{name} {tag} k={k}")


def test_contributions_memory_cap(monkeypatch):
    scene, cam, cfg = _setup("odd100x70", "ref")
    monkeypatch.setattr(render, "CONTRIB_MAX_BYTES", 1 << 20)
    with pytest.raises(InvalidArgumentError):
        render_frame(scene, cam, cfg, record_contributions=True)
