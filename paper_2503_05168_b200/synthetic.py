"""Deterministic synthetic scenes and camera trajectories for the BASELINE configs.

``synth`` and ``orbit`` follow SURVEY.md Appendix C exactly (the numpy call
sequence is part of the spec: the calibrated visible / binned / pair counts
of the survey depend on it).  ``random_scene`` / ``make_camera`` restate the
reference test builders (pkg/tests/support.py:15-83) so config 1
(100K SH3 @ 256x256) can be produced without the reference on the GPU box.

Scenes come back as plain numpy arrays in a :class:`~.model.SceneArrays`.
"""
from __future__ import annotations

import math

import numpy as np

from .model import CameraPose, SceneArrays


def synth(n: int, seed: int = 0) -> SceneArrays:
    """SURVEY.md Appendix C scene: 70 % object blob + 30 % background shell."""
    rng = np.random.default_rng(seed)
    n_obj = int(0.7 * n)
    n_bg = n - n_obj
    obj = rng.normal(0, 0.6, size=(n_obj, 3))
    d = rng.normal(size=(n_bg, 3))
    d /= np.linalg.norm(d, axis=1, keepdims=True)
    bg = d * rng.uniform(4.0, 10.0, size=(n_bg, 1))
    positions = np.concatenate([obj, bg])
    log_scales = np.concatenate([rng.normal(np.log(0.008), 0.5, size=(n_obj, 3)),
                                 rng.normal(np.log(0.04), 0.5, size=(n_bg, 3))])
    q = rng.normal(size=(n, 4))
    rotations = q / np.linalg.norm(q, axis=1, keepdims=True)
    opacities = np.where(rng.random(n) < 0.3, rng.uniform(0.005, 0.1, n), rng.uniform(0.1, 0.99, n))
    rs = np.random.default_rng(seed + 7)
    sh = np.zeros((n, 3, 16))
    sh[:, :, 0] = rs.normal(0, 0.3, size=(n, 3))
    sh[:, :, 1:] = rs.normal(0, 0.05, size=(n, 3, 15))
    return SceneArrays(positions, log_scales, rotations, opacities, sh, ids=np.arange(n, dtype=np.int64))


def _matrix_to_quat(r: np.ndarray) -> np.ndarray:
    """Rotation matrix -> (w, x, y, z) via the trace / copysign formula."""
    w = math.sqrt(max(0.0, 1.0 + r[0, 0] + r[1, 1] + r[2, 2])) / 2.0
    x = math.copysign(math.sqrt(max(0.0, 1.0 + r[0, 0] - r[1, 1] - r[2, 2])) / 2.0, r[2, 1] - r[1, 2])
    y = math.copysign(math.sqrt(max(0.0, 1.0 - r[0, 0] + r[1, 1] - r[2, 2])) / 2.0, r[0, 2] - r[2, 0])
    z = math.copysign(math.sqrt(max(0.0, 1.0 - r[0, 0] - r[1, 1] + r[2, 2])) / 2.0, r[1, 0] - r[0, 1])
    return np.array([w, x, y, z])


def orbit_pose(i: int, frames: int = 120, width: int = 1920, height: int = 1080,
               radius: float = 3.0, height_offset: float = -0.3, fov_x: float = 1.0) -> CameraPose:
    """Frame ``i`` of the SURVEY.md Appendix C orbit, looking at the origin."""
    theta = 2.0 * math.pi * i / frames
    c = np.array([radius * math.sin(theta), height_offset, -radius * math.cos(theta)])
    f = -c / np.linalg.norm(c)
    r = np.cross(np.array([0.0, 1.0, 0.0]), f)
    r /= np.linalg.norm(r)
    u = np.cross(f, r)
    rot = np.column_stack([r, u, f])
    fx = width / (2.0 * math.tan(fov_x / 2.0))
    fov_y = 2.0 * math.atan(height / (2.0 * fx))
    return CameraPose(position=c, orientation=_matrix_to_quat(rot), fov_x=fov_x, fov_y=fov_y,
                      width=width, height=height, near_clip=0.2)


def orbit(frames: int = 120, width: int = 1920, height: int = 1080) -> list[CameraPose]:
    return [orbit_pose(i, frames, width, height) for i in range(frames)]


# -- reference test builders (pkg/tests/support.py) ---------------------------

DEFAULT_FOV = 0.8


def make_camera(width: int = 64, height: int = 64, position=(0.0, 0.0, 0.0),
                orientation=(1.0, 0.0, 0.0, 0.0), fov: float = DEFAULT_FOV) -> CameraPose:
    """support.py:15-29."""
    return CameraPose(position=np.asarray(position, dtype=np.float64),
                      orientation=np.asarray(orientation, dtype=np.float64),
                      fov_x=fov, fov_y=fov, width=width, height=height)


def random_scene(rng: np.random.Generator, n: int, *, depth_range=(2.0, 6.0), scale_range=(0.03, 0.2),
                 opacity_range=(0.05, 0.95), sh_degree: int = 1, camera: CameraPose | None = None) -> SceneArrays:
    """support.py:45-83 (same numpy call sequence, so seeds reproduce)."""
    cam = camera or make_camera()
    z = rng.uniform(*depth_range, size=n)
    lateral = 0.8 * np.tan(cam.fov_x / 2.0)
    x = rng.uniform(-lateral, lateral, size=n) * z
    y = rng.uniform(-lateral, lateral, size=n) * z
    view = np.stack([x, y, z], axis=1)
    r = cam.rotation_matrix()
    positions = (r @ view.T).T + cam.position
    log_scales = np.log(rng.uniform(*scale_range, size=(n, 3)))
    rotations = np.stack([_unit_quat(rng) for _ in range(n)])
    opacities = rng.uniform(*opacity_range, size=n)
    sh = np.zeros((n, 3, 16))
    sh[:, :, 0] = rng.normal(0.0, 0.3, size=(n, 3))
    if sh_degree > 0:
        bands = (sh_degree + 1) ** 2 - 1
        sh[:, :, 1:1 + bands] = rng.normal(0.0, 0.05, size=(n, 3, bands))
    return SceneArrays(positions=positions, log_scales=log_scales, rotations=rotations,
                       opacities=opacities, sh=sh, ids=np.arange(n, dtype=np.int64))


def _unit_quat(rng: np.random.Generator) -> np.ndarray:
    q = rng.normal(size=4)
    return q / np.linalg.norm(q)


def config1_scene() -> tuple[SceneArrays, CameraPose]:
    """BASELINE config 1: random_scene(default_rng(0), 100_000, sh_degree=3) @ 256x256."""
    cam = make_camera(256, 256)
    return random_scene(np.random.default_rng(0), 100_000, sh_degree=3, camera=cam), cam
