"""Image quality metrics on the GPU (drop-in for metrics.psnr / metrics.ssim,
pkg/src/seele/metrics.py:44-112): fp64 kernels in csrc/metrics.cu behind
``seele_psnr`` / ``seele_ssim``, so a rendered trajectory can be scored on the
device.  Inputs are (H, W, 3) arrays (numpy, or torch tensors on the device);
results are Python floats like the reference's."""
from __future__ import annotations

import csv
import json
import math
import time
from dataclasses import dataclass, replace
from pathlib import Path

import numpy as np

from . import _native
from .errors import InvalidArgumentError

SSIM_WINDOW = 11


def _device_pair(img_a, img_b):
    import torch

    def dev(x):
        if isinstance(x, torch.Tensor):
            return x.to(device="cuda", dtype=torch.float64).contiguous()
        return torch.as_tensor(np.ascontiguousarray(np.asarray(x, dtype=np.float64)), device="cuda")

    a, b = dev(img_a), dev(img_b)
    if tuple(a.shape) != tuple(b.shape):
        raise InvalidArgumentError(f"image shapes differ: {tuple(a.shape)} vs {tuple(b.shape)}")
    return a, b


def psnr(img_a, img_b) -> float:
    """metrics.py:44-54: peak signal-to-noise ratio in dB for unit-range
    images; identical inputs give +inf."""
    import torch

    a, b = _device_pair(img_a, img_b)
    lib = _native.load()
    scratch = torch.empty(1024, dtype=torch.float64, device=a.device)
    out = torch.empty(1, dtype=torch.float64, device=a.device)
    _native.check(lib.seele_psnr(a.data_ptr(), b.data_ptr(), a.numel(), scratch.data_ptr(), out.data_ptr(),
                                 torch.cuda.current_stream(a.device).cuda_stream))
    return float(out.item())


def ssim(img_a, img_b) -> float:
    """metrics.py:72-112: mean structural similarity over the BT.601
    luminance, Gaussian 11x11 windows (sigma 1.5) where they fit."""
    import torch

    a, b = _device_pair(img_a, img_b)
    if a.dim() != 3 or a.shape[2] != 3:
        raise InvalidArgumentError("ssim expects (H, W, 3) images")
    h, w = int(a.shape[0]), int(a.shape[1])
    if min(h, w) < SSIM_WINDOW:
        raise InvalidArgumentError(f"images must be at least {SSIM_WINDOW} pixels per side for SSIM")
    lib = _native.load()
    scratch = torch.empty(int(lib.seele_metrics_scratch_doubles(w, h)), dtype=torch.float64, device=a.device)
    out = torch.empty(1, dtype=torch.float64, device=a.device)
    _native.check(lib.seele_ssim(a.data_ptr(), b.data_ptr(), w, h, scratch.data_ptr(), out.data_ptr(),
                                 torch.cuda.current_stream(a.device).cuda_stream))
    return float(out.item())


@dataclass
class ContributionCurve:
    """metrics.py:104-112."""

    aggregate: np.ndarray         # (p,) mean cumulative weight of the k strongest splats
    per_pixel_totals: np.ndarray  # (h*w,) total blended weight
    fraction_for_99: float        # mean fraction of a pixel's splats covering 99 %
    per_pixel_curves: list | None = None


def contribution_cdf(scene, cam, cfg=None, *, keep_per_pixel: bool = False) -> ContributionCurve:
    """metrics.py:115-161 on the GPU: the dense contribution matrix comes from
    render_frame(record_contributions=True) (seele_contributions, reference
    schedule in fp64) and stays on the device; every pixel's weights are
    sorted in descending order and accumulated column by column (a sequential
    scan per pixel, the same association as numpy's cumsum), and the 99 %
    rank is searchsorted(cumulative, 0.99 total - 1e-15) + 1 as a count of
    cumulative values below the target."""
    import torch

    from .render import EngineConfig, render_frame

    cfg = cfg or EngineConfig()
    result = render_frame(scene, cam, cfg, record_contributions=True, output="torch")
    matrix = result.contributions
    n_pixels = int(matrix.shape[1]) if matrix is not None else 0
    if matrix is None or matrix.numel() == 0:
        return ContributionCurve(aggregate=np.zeros(0), per_pixel_totals=np.zeros(n_pixels), fraction_for_99=0.0,
                                 per_pixel_curves=[] if keep_per_pixel else None)
    sorted_desc = torch.sort(matrix, dim=0, descending=True).values
    cumulative = torch.cumsum(sorted_desc, dim=0)  # (p, n_pixels), outer-dimension scan: sequential per column
    totals = cumulative[-1]
    counts = (sorted_desc > 0.0).sum(dim=0)
    target = 0.99 * totals - 1e-15
    rank = (cumulative < target[None, :]).sum(dim=0) + 1
    has = counts > 0
    fractions = rank[has].to(torch.float64) / counts[has].to(torch.float64)
    fraction_for_99 = float(fractions.cpu().numpy().mean()) if int(has.sum()) else 0.0
    curves = None
    if keep_per_pixel:
        cum_h, cnt_h = cumulative.cpu().numpy(), counts.cpu().numpy()
        curves = [cum_h[:max(int(c), 1), pix] if c else np.zeros(0) for pix, c in enumerate(cnt_h)]
    return ContributionCurve(aggregate=cumulative.mean(dim=1).cpu().numpy(), per_pixel_totals=totals.cpu().numpy(),
                             fraction_for_99=fraction_for_99, per_pixel_curves=curves)


# ---- comparative benchmark harness (metrics.py:164-266) -------------------------------------------------

REPORT_COLUMNS = ["config", "psnr_db", "ssim", "lpips", "warp_steps", "alpha_evals", "blend_steps",
                  "leader_evals", "peak_resident_bytes", "stalls", "wall_ms"]


def _fmt(value) -> str:
    if isinstance(value, float):
        return "inf" if math.isinf(value) else f"{value:.6f}"
    return "" if value is None else str(value)


def bench_compare(configs: list[dict], poses: list, *, flat_scene=None, clustered=None, base_cfg=None,
                  m: int | None = None) -> list[dict]:
    """metrics.bench_compare (metrics.py:172-243) on the GPU: render a
    trajectory under each configuration ({"engine": "ref"|"cr", "scene":
    "flat"|"clustered"}) and report quality (GPU PSNR / SSIM against the flat
    scene under the reference engine, rendered once up front) and the
    lockstep cost counters.  Clustered configurations stream the container
    through :class:`~.streaming.StreamingRenderer` (the reference
    ResidentRenderer's state machine: its stall count and peak resident bytes,
    same defaults).  ``wall_ms`` is this host's wall clock."""
    from .container import BYTES_PER_GAUSSIAN
    from .render import EngineConfig, render_frame
    from .streaming import StreamingRenderer

    base_cfg = base_cfg or EngineConfig()
    if flat_scene is None:
        raise InvalidArgumentError("bench requires the flat scene for the baseline")
    baseline_cfg = replace(base_cfg, engine="ref")
    baseline = [render_frame(flat_scene, pose, baseline_cfg, output="torch").image for pose in poses]
    flat_bytes = len(flat_scene) * BYTES_PER_GAUSSIAN

    def score(res, base, totals, psnrs, ssims):
        st = res.stats
        totals["warp"] += st.warp_steps
        totals["alpha"] += st.alpha_eval_steps
        totals["blend"] += st.blend_steps
        totals["leader"] += st.leader_eval_steps
        psnrs.append(psnr(res.image, base))
        ssims.append(ssim(res.image, base))

    rows = []
    for entry in configs:
        engine, scene_mode = entry["engine"], entry["scene"]
        cfg = replace(base_cfg, engine=engine)
        t0 = time.perf_counter()
        totals = {"warp": 0, "alpha": 0, "blend": 0, "leader": 0, "stalls": 0}
        peak_bytes = flat_bytes
        psnrs, ssims = [], []
        if scene_mode == "clustered":
            if clustered is None:
                raise InvalidArgumentError("no clustered scene supplied for a clustered config")
            with StreamingRenderer(clustered, m) as renderer:
                for pose, base in zip(poses, baseline):
                    score(renderer.render_frame(pose, cfg, output="torch"), base, totals, psnrs, ssims)
                peak_bytes = renderer.peak_resident_bytes
                totals["stalls"] = renderer.stall_count
        else:
            for pose, base in zip(poses, baseline):
                score(render_frame(flat_scene, pose, cfg, output="torch"), base, totals, psnrs, ssims)
        wall_ms = (time.perf_counter() - t0) * 1000.0
        finite = [v for v in psnrs if not math.isinf(v)]
        rows.append({
            "config": f"{engine}:{scene_mode}",
            "psnr_db": math.inf if not finite else float(np.mean(finite)),
            "ssim": float(np.mean(ssims)),
            "lpips": None,
            "warp_steps": totals["warp"],
            "alpha_evals": totals["alpha"],
            "blend_steps": totals["blend"],
            "leader_evals": totals["leader"],
            "peak_resident_bytes": peak_bytes,
            "stalls": totals["stalls"],
            "wall_ms": wall_ms,
        })
    return rows


def write_report(rows: list[dict], csv_path) -> None:
    """metrics.write_report (metrics.py:246-266): the table as CSV plus a JSON
    mirror next to it (same columns, number formatting and "inf" spelling)."""
    csv_path = Path(csv_path)
    with csv_path.open("w", newline="") as fh:
        writer = csv.writer(fh)
        writer.writerow(REPORT_COLUMNS)
        for row in rows:
            writer.writerow([_fmt(row[c]) for c in REPORT_COLUMNS])
    json_rows = []
    for row in rows:
        json_rows.append({c: ("inf" if isinstance(row[c], float) and math.isinf(row[c]) else row[c])
                          for c in REPORT_COLUMNS})
    csv_path.with_suffix(".json").write_text(json.dumps(json_rows, indent=1))
