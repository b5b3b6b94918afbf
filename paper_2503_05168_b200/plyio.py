"""Trained-scene PLY ingest (io.py:36-152), vectorised.

``load_ply`` is the drop-in for the reference's per-record Python loop: the
vertex block is decoded with one numpy view and validated with the
reference's rules and messages (binary little-endian only, no list
properties, f_rest count 0 / 9 / 24 / 45, required properties, truncation,
non-finite values, degenerate quaternions -- reported at the first bad
record in file order).  ``ply_to_planes`` / ``DeviceScene.from_ply`` go from
the file straight to the device layout ([15, n, 4] float32 planes: the file's
float32 values, opacity logit and raw quaternion, decoded in the preprocess
kernel exactly as for the container).
"""
from __future__ import annotations

from dataclasses import dataclass
from pathlib import Path

import numpy as np

from .errors import DataError, SchemaError
from .model import Gaussian3D, SceneArrays, sigmoid

_PLY_NUMPY_TYPES = {
    "float": "<f4", "float32": "<f4", "double": "<f8", "float64": "<f8",
    "uchar": "u1", "uint8": "u1", "char": "i1", "int8": "i1",
    "ushort": "<u2", "uint16": "<u2", "short": "<i2", "int16": "<i2",
    "uint": "<u4", "uint32": "<u4", "int": "<i4", "int32": "<i4",
}
_REST_COUNT_TO_DEGREE = {0: 0, 9: 1, 24: 2, 45: 3}
_OPACITY_EPS = 1e-12


def _parse_header(raw: bytes, path: Path):
    """io.py:62-90."""
    end = raw.find(b"end_header\n")
    if not raw.startswith(b"ply") or end < 0:
        raise SchemaError(f"{path}: not a PLY file")
    header = raw[:end].decode("ascii", errors="replace").splitlines()
    count, props, in_vertex, fmt_ok = None, [], False, False
    for line in header:
        parts = line.split()
        if not parts:
            continue
        if parts[0] == "format":
            fmt_ok = parts[1] == "binary_little_endian"
        elif parts[0] == "element":
            in_vertex = parts[1] == "vertex"
            if in_vertex:
                count = int(parts[2])
        elif parts[0] == "property" and in_vertex:
            if parts[1] == "list":
                raise SchemaError(f"{path}: list properties are not supported")
            props.append((parts[1], parts[2]))
    if not fmt_ok:
        raise SchemaError(f"{path}: only binary little-endian PLY is supported")
    if count is None:
        raise SchemaError(f"{path}: no vertex element")
    return count, props, end + len(b"end_header\n")


def _read_records(path):
    """Header rules + one structured view of the vertex block (io.py:93-121)."""
    path = Path(path)
    raw = path.read_bytes()
    count, props, offset = _parse_header(raw, path)
    if count <= 0:
        raise DataError(f"{path}: scene has no gaussians")
    names = [n for _, n in props]
    rest = sum(1 for n in names if n.startswith("f_rest_"))
    if rest not in _REST_COUNT_TO_DEGREE:
        raise SchemaError(f"{path}: unsupported f_rest count {rest}")
    required = ["x", "y", "z", "f_dc_0", "f_dc_1", "f_dc_2", "opacity", "scale_0", "scale_1", "scale_2",
                "rot_0", "rot_1", "rot_2", "rot_3"] + [f"f_rest_{i}" for i in range(rest)]
    for name in required:
        if name not in names:
            raise SchemaError(f"{path}: missing vertex property '{name}'")
    dtype = np.dtype([(n, _PLY_NUMPY_TYPES[k]) for k, n in props])
    body = memoryview(raw)[offset:]
    if len(body) < count * dtype.itemsize:
        raise DataError(f"{path}: truncated vertex data")
    rec = np.frombuffer(body, dtype=dtype, count=count)
    return path, rec, count, rest


def _columns(rec, count, rest):
    """(fields[n, 11] = x y z opacity scale rot, sh[n, 3, 16]) as float64, the reference's promotion."""
    cols = ["x", "y", "z", "opacity", "scale_0", "scale_1", "scale_2", "rot_0", "rot_1", "rot_2", "rot_3"]
    fields = np.stack([rec[c].astype(np.float64) for c in cols], axis=1)
    sh = np.zeros((count, 3, 16), dtype=np.float64)
    per = rest // 3
    for ch in range(3):
        sh[:, ch, 0] = rec[f"f_dc_{ch}"]
        for j in range(per):
            sh[:, ch, 1 + j] = rec[f"f_rest_{ch * per + j}"]
    return fields, sh


def _validate(path, fields, sh):
    """The first bad record in file order, with the reference's error (io.py:133-148, model.py:61-67)."""
    finite = np.isfinite(fields).all(axis=1) & np.isfinite(sh.reshape(len(sh), -1)).all(axis=1)
    qn = np.sqrt(np.einsum("ij,ij->i", fields[:, 7:11], fields[:, 7:11]))
    bad_q = finite & (qn < 1e-8)
    first_nf = int(np.argmin(finite)) if not finite.all() else None
    first_q = int(np.argmax(bad_q)) if bad_q.any() else None
    if first_nf is not None and (first_q is None or first_nf < first_q):
        raise DataError(f"{path}: non-finite value at record {first_nf}")
    if first_q is not None:
        raise DataError("quaternion norm too small to normalize")


@dataclass
class SceneFile:
    """io.py:50-59: a parsed trained scene (arrays first; Gaussian3D objects on demand)."""

    scene: SceneArrays
    source_path: str
    sh_degree: int

    def arrays(self) -> SceneArrays:
        return self.scene

    @property
    def gaussians(self) -> list:
        s = self.scene
        return [Gaussian3D(position=s.positions[i], scale=s.log_scales[i], rotation=s.rotations[i],
                           opacity=float(s.opacities[i]), sh_coeffs=s.sh[i]) for i in range(len(s))]


def load_ply(path) -> SceneFile:
    """io.py:93-152: parse a trained scene in the de-facto splat PLY layout."""
    path, rec, count, rest = _read_records(path)
    fields, sh = _columns(rec, count, rest)
    _validate(path, fields, sh)
    rot = fields[:, 7:11]
    rot = rot / np.linalg.norm(rot, axis=1, keepdims=True)  # Gaussian3D.__post_init__ (model.py:122)
    opac = np.clip(sigmoid(fields[:, 3]), _OPACITY_EPS, 1.0 - _OPACITY_EPS)  # _decode_opacity (io.py:33-34)
    scene = SceneArrays(positions=fields[:, 0:3].copy(), log_scales=fields[:, 4:7].copy(), rotations=rot,
                        opacities=opac, sh=sh, ids=np.arange(count, dtype=np.int64))
    return SceneFile(scene=scene, source_path=str(path), sh_degree=_REST_COUNT_TO_DEGREE[rest])


def ply_to_planes(path) -> tuple[np.ndarray, np.ndarray, int]:
    """The file straight to the device layout: ([15, n, 4] float32 planes, ids, sh degree)."""
    from .device import N_PLANES

    path, rec, count, rest = _read_records(path)
    fields, sh = _columns(rec, count, rest)
    _validate(path, fields, sh)
    planes = np.zeros((N_PLANES, count, 4), dtype=np.float32)
    for k, c in enumerate(("x", "y", "z", "opacity")):
        planes[0, :, k] = rec[c]
    for k in range(3):
        planes[1, :, k] = rec[f"scale_{k}"]
    for k in range(4):
        planes[2, :, k] = rec[f"rot_{k}"]
    sh32 = sh.astype(np.float32)
    for ch in range(3):
        for k in range(4):
            planes[3 + 4 * ch + k] = sh32[:, ch, 4 * k:4 * k + 4]
    return planes, np.arange(count, dtype=np.int64), _REST_COUNT_TO_DEGREE[rest]
