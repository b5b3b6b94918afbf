"""Shared test helpers: golden fixture loading and scene/camera/config builders."""
from __future__ import annotations

import hashlib
from pathlib import Path

import numpy as np

from paper_2503_05168_b200.model import CameraPose, SceneArrays
from paper_2503_05168_b200.render import EngineConfig

GOLDEN = Path(__file__).resolve().parent / "golden"
STAT_KEYS = ("alpha_eval_steps", "blend_steps", "leader_eval_steps", "warp_steps", "tile_pairs",
             "culled_near", "dropped_degenerate")
ENGINES = {
    "ref": dict(engine="ref"),
    "cr1": dict(engine="cr", group_w=1),
    "cr2": dict(engine="cr", group_w=2),
    "cr4": dict(engine="cr", group_w=4),
}
SMALL_CASES = ["rand64_s0", "rand64_s1", "rand64_s2", "rand64_s3", "accept_000", "accept_003", "accept_010",
               "accept_017", "odd100x70", "plain3sigma", "edges80x48", "shdeg0", "shdeg1", "shdeg2"]


def sha(a: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def load(name: str) -> dict:
    with np.load(GOLDEN / f"{name}.npz") as z:
        return {k: z[k] for k in z.files}


def camera_from(g: dict) -> CameraPose:
    fov = g["cam_fov"]
    w, h = (int(v) for v in g["cam_size"])
    return CameraPose(position=g["cam_position"], orientation=g["cam_orientation"], fov_x=float(fov[0]),
                      fov_y=float(fov[1]), width=w, height=h, near_clip=float(fov[2]))


def scene_from(g: dict) -> SceneArrays:
    return SceneArrays(g["positions"], g["log_scales"], g["rotations"], g["opacities"], g["sh"], g["ids"])


def base_cfg(g: dict) -> dict:
    flags = g.get("cfg_flags", np.array([1, 3]))
    bg = g.get("cfg_background", np.zeros(3))
    return dict(background=tuple(float(v) for v in bg), opacity_aware_filter=bool(flags[0]),
                sh_degree=int(flags[1]))


def engines_in(g: dict) -> list[str]:
    return [t for t in ENGINES if f"{t}_stats" in g]


def config_for(g: dict, tag: str, **extra) -> EngineConfig:
    return EngineConfig(**base_cfg(g), **ENGINES[tag], **extra)


def golden_ranges(g: dict, n_tiles: int) -> tuple[np.ndarray, np.ndarray]:
    rs = np.zeros(n_tiles, dtype=np.int64)
    re = np.zeros(n_tiles, dtype=np.int64)
    for t, s, e in g["ranges"]:
        rs[t], re[t] = s, e
    return rs, re


def psnr(a: np.ndarray, b: np.ndarray, peak: float = 1.0) -> float:
    """metrics.psnr (metrics.py:44-54): 10 log10(peak^2 / mse)."""
    mse = float(np.mean((np.asarray(a, dtype=np.float64) - np.asarray(b, dtype=np.float64)) ** 2))
    return float("inf") if mse == 0.0 else 10.0 * np.log10(peak * peak / mse)
