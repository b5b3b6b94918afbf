"""Scenes resident in HBM.

A :class:`DeviceScene` is the B200-side replacement of the per-frame
``SceneArrays`` hand-off of the reference (render.py:94-108 rebuilds a
``Gaussian3D`` per splat every frame).  The scene is validated once on upload
with the reference's rules (``Gaussian3D.__post_init__``, model.py:111-129)
and then stays in HBM; frames only pass a camera.

Two layouts (include/seele_b200.h):

* ``"f64"`` -- the ``SceneArrays`` fields as given, float64.  Exact drop-in
  for any caller-built scene (e.g. BASELINE config 1, ``random_scene``).
* ``"planes"`` -- the cluster-container record (io.py:22-25: 59 float32 per
  splat) transposed into 15 float4 planes, 240 B per splat, fully coalesced
  ``float4`` loads.  Opacity stays a float32 logit and is decoded on device
  with the container's ``clip(sigmoid(x))`` (io.py:33-34); the rotation is
  normalised like ``_decode_chunk`` + ``Gaussian3D``.  This is what a
  compiled / streamed scene looks like, and what the benchmark renders.
"""
from __future__ import annotations

import numpy as np
import torch

from . import _native
from .errors import DataError, InvalidArgumentError
from .model import SceneArrays, sigmoid

N_PLANES = 15
_OPACITY_EPS = 1e-12


def validate_arrays(scene: SceneArrays) -> None:
    """Vectorised Gaussian3D validation (model.py:111-129); raises DataError."""
    n = len(scene)
    shapes = {"positions": (n, 3), "log_scales": (n, 3), "rotations": (n, 4), "opacities": (n,), "sh": (n, 3, 16)}
    for name, shape in shapes.items():
        arr = np.asarray(getattr(scene, name))
        if arr.shape != shape:
            raise DataError(f"{name} must have shape {shape}, got {arr.shape}")
        bad = ~np.isfinite(arr.reshape(n, -1)).all(axis=1) if n else np.zeros(0, bool)
        if bad.any():
            raise DataError(f"splat {int(np.flatnonzero(bad)[0])}: {name} contains non-finite values")
    with np.errstate(over="ignore"):
        bad = ~np.isfinite(np.exp(np.asarray(scene.log_scales))).all(axis=1)
    if bad.any():
        raise DataError(f"splat {int(np.flatnonzero(bad)[0])}: exp(scale) overflows")
    norms = np.linalg.norm(np.asarray(scene.rotations), axis=1)
    if (norms < 1e-8).any():
        raise DataError(f"splat {int(np.flatnonzero(norms < 1e-8)[0])}: quaternion norm too small to normalize")
    o = np.asarray(scene.opacities)
    bad = ~((o > 0.0) & (o < 1.0))
    if bad.any():
        raise DataError(f"splat {int(np.flatnonzero(bad)[0])}: opacity must lie in (0, 1), got {o[bad][0]}")
    if np.asarray(scene.ids).shape != (n,):
        raise DataError("ids must have shape (n,)")


def encode_planes(scene: SceneArrays) -> np.ndarray:
    """Container encoding (io.py:198-208) laid out as [15, n, 4] float32."""
    n = len(scene)
    planes = np.zeros((N_PLANES, n, 4), dtype=np.float32)
    planes[0, :, :3] = scene.positions
    with np.errstate(divide="ignore"):
        planes[0, :, 3] = np.log(scene.opacities) - np.log1p(-np.asarray(scene.opacities))
    planes[1, :, :3] = scene.log_scales
    planes[2] = scene.rotations
    sh = np.asarray(scene.sh, dtype=np.float32)
    for ch in range(3):
        for k in range(4):
            planes[3 + 4 * ch + k] = sh[:, ch, 4 * k:4 * k + 4]
    return planes


def decode_planes(planes: np.ndarray, ids: np.ndarray) -> SceneArrays:
    """What the reference sees after loading the container (io.py:211-234)."""
    n = planes.shape[1]
    p = planes.astype(np.float64)
    sh = np.zeros((n, 3, 16))
    for ch in range(3):
        for k in range(4):
            sh[:, ch, 4 * k:4 * k + 4] = p[3 + 4 * ch + k]
    rot = p[2]
    rot = rot / np.linalg.norm(rot, axis=1, keepdims=True)
    opac = np.clip(sigmoid(p[0, :, 3]), _OPACITY_EPS, 1.0 - _OPACITY_EPS)
    return SceneArrays(positions=p[0, :, :3].copy(), log_scales=p[1, :, :3].copy(), rotations=rot,
                       opacities=opac, sh=sh, ids=np.asarray(ids, dtype=np.int64).copy())


class DeviceScene:
    """A validated scene resident in HBM (one copy per GPU; nothing streams)."""

    def __init__(self, layout: str, n: int, tensors: dict, ids: torch.Tensor, host_ids: np.ndarray):
        self.layout = layout
        self.n = int(n)
        self.tensors = tensors
        self.ids = ids
        self.host_ids = host_ids
        self.device = ids.device

    # -- construction ----------------------------------------------------------
    @classmethod
    def from_arrays(cls, scene: SceneArrays, device=None, layout: str = "f64") -> "DeviceScene":
        if layout not in ("f64", "planes"):
            raise InvalidArgumentError(f"unknown scene layout '{layout}'")
        validate_arrays(scene)
        dev = torch.device(device or "cuda")
        host_ids = np.ascontiguousarray(np.asarray(scene.ids, dtype=np.int64))
        if layout == "planes":
            return cls.from_planes(encode_planes(scene), host_ids, dev)
        t = {name: torch.from_numpy(np.ascontiguousarray(np.asarray(getattr(scene, name), dtype=np.float64)))
             .to(dev) for name in ("positions", "log_scales", "rotations", "opacities", "sh")}
        return cls("f64", len(scene), t, torch.from_numpy(host_ids).to(dev), host_ids)

    @classmethod
    def from_planes(cls, planes: np.ndarray, ids, device=None) -> "DeviceScene":
        planes = np.ascontiguousarray(planes, dtype=np.float32)
        if planes.ndim != 3 or planes.shape[0] != N_PLANES or planes.shape[2] != 4:
            raise DataError(f"planes must have shape (15, n, 4), got {planes.shape}")
        n = planes.shape[1]
        if not np.isfinite(planes).all():
            raise DataError("scene planes contain non-finite values")
        if n and (np.linalg.norm(planes[2].astype(np.float64), axis=1) < 1e-8).any():
            raise DataError("degenerate rotation record")
        dev = torch.device(device or "cuda")
        host_ids = np.ascontiguousarray(np.asarray(ids, dtype=np.int64))
        return cls("planes", n, {"planes": torch.from_numpy(planes).to(dev)}, torch.from_numpy(host_ids).to(dev),
                   host_ids)

    # -- C-ABI view --------------------------------------------------------------
    @classmethod
    def from_ply(cls, path, device=None) -> "DeviceScene":
        """A trained-scene PLY straight into the planes layout (plyio.ply_to_planes)."""
        from .plyio import ply_to_planes

        planes, ids, _ = ply_to_planes(path)
        return cls.from_planes(planes, ids, device)

    def struct(self) -> _native.Scene:
        s = _native.Scene()
        s.n = self.n
        s.ids = self.ids.data_ptr()
        if self.layout == "planes":
            s.layout = _native.LAYOUT_PLANES
            s.planes = self.tensors["planes"].data_ptr()
            s.plane_stride = self.n
        else:
            s.layout = _native.LAYOUT_F64
            for name in ("positions", "log_scales", "rotations", "opacities", "sh"):
                setattr(s, name, self.tensors[name].data_ptr())
        return s

    def host_arrays(self) -> SceneArrays:
        """The fp64 scene the reference would render for this resident scene."""
        if self.layout == "planes":
            return decode_planes(self.tensors["planes"].cpu().numpy(), self.host_ids)
        t = {k: v.cpu().numpy() for k, v in self.tensors.items()}
        return SceneArrays(t["positions"], t["log_scales"], t["rotations"], t["opacities"], t["sh"],
                           self.host_ids.copy())

    def nbytes(self) -> int:
        return sum(t.numel() * t.element_size() for t in self.tensors.values()) + self.ids.numel() * 8

    def __len__(self) -> int:
        return self.n
