"""ctypes front end of the CPU fp64 oracle (``seele_oracle.c``).

TEST INFRASTRUCTURE ONLY.  This module is the checker the CUDA path is
compared against; it is imported solely by ``tests/``,
``__graft_entry__.smoke()`` and the ``cpu_baseline`` / ``--impl reference``
legs of ``bench.py``.  The product package never imports it.

Parity of this restatement with the reference Python package is pinned by
``tests/golden/`` (vectors produced by the reference itself, see
``tests/golden/make_golden.py``) and checked in ``tests/test_oracle.py``.

Inputs are duck-typed: any scene with ``positions, log_scales, rotations,
opacities, sh, ids`` arrays, any camera with ``position, orientation,
fov_x, fov_y, width, height, near_clip`` and any config with ``engine,
group_w, background, alpha_theta, gamma_threshold, sh_degree,
opacity_aware_filter`` works -- the reference's own ``SceneArrays`` /
``CameraPose`` / ``EngineConfig`` as well as this repo's mirrors.
"""
from __future__ import annotations

import ctypes
import os
import subprocess
from pathlib import Path

import numpy as np

_HERE = Path(__file__).resolve().parent
_LIB_PATH = _HERE / "_build" / "libseele_oracle.so"
TILE = 16

_lib = None


class _Camera(ctypes.Structure):
    _fields_ = [
        ("position", ctypes.c_double * 3),
        ("orientation", ctypes.c_double * 4),
        ("fov_x", ctypes.c_double),
        ("fov_y", ctypes.c_double),
        ("near_clip", ctypes.c_double),
        ("width", ctypes.c_int32),
        ("height", ctypes.c_int32),
    ]


class _Config(ctypes.Structure):
    _fields_ = [
        ("engine", ctypes.c_int32),
        ("group_w", ctypes.c_int32),
        ("sh_degree", ctypes.c_int32),
        ("opacity_aware", ctypes.c_int32),
        ("alpha_theta", ctypes.c_double),
        ("gamma_threshold", ctypes.c_double),
        ("background", ctypes.c_double * 3),
    ]


def build() -> Path:
    """Compile the oracle shared library (gcc, -ffp-contract=off)."""
    subprocess.run(["make", "-s", "-C", str(_HERE)], check=True)
    return _LIB_PATH


def lib():
    global _lib
    if _lib is None:
        if not _LIB_PATH.exists():
            build()
        _lib = ctypes.CDLL(str(_LIB_PATH))
        P = ctypes.c_void_p
        _lib.oracle_preprocess.argtypes = [ctypes.c_int64] + [P] * 14
        _lib.oracle_preprocess.restype = None
        _lib.oracle_sort_pairs.argtypes = [ctypes.c_int64, P, P, ctypes.c_int32, ctypes.c_int32, P, P, P, P]
        _lib.oracle_sort_pairs.restype = ctypes.c_int64
        _lib.oracle_raster_frame.argtypes = [ctypes.c_int32, ctypes.c_int32] + [P] * 8 + [ctypes.c_int32, P, P, P]
        _lib.oracle_raster_frame.restype = None
        _lib.oracle_select_clusters.argtypes = [P, P, ctypes.c_int32, ctypes.c_int32, ctypes.c_double, P,
                                                ctypes.c_double, P]
        _lib.oracle_select_clusters.restype = ctypes.c_int
    return _lib


def _ptr(a: np.ndarray):
    return a.ctypes.data_as(ctypes.c_void_p)


def _c64(a, shape=None) -> np.ndarray:
    out = np.ascontiguousarray(np.asarray(a, dtype=np.float64))
    if shape is not None:
        out = out.reshape(shape)
    return out


def camera_struct(cam) -> _Camera:
    c = _Camera()
    c.position[:] = [float(v) for v in np.asarray(cam.position, dtype=np.float64)]
    c.orientation[:] = [float(v) for v in np.asarray(cam.orientation, dtype=np.float64)]
    c.fov_x = float(cam.fov_x)
    c.fov_y = float(cam.fov_y)
    c.near_clip = float(cam.near_clip)
    c.width = int(cam.width)
    c.height = int(cam.height)
    return c


def config_struct(cfg) -> _Config:
    c = _Config()
    c.engine = 0 if cfg.engine == "ref" else 1
    c.group_w = int(cfg.group_w)
    c.sh_degree = int(cfg.sh_degree)
    c.opacity_aware = 1 if cfg.opacity_aware_filter else 0
    c.alpha_theta = float(cfg.alpha_theta)
    c.gamma_threshold = float(cfg.gamma_threshold)
    c.background[:] = [float(v) for v in cfg.background]
    return c


def plan(scene, cam, cfg) -> dict:
    """plan_frame (render.py:90-141) restated: project, bin, sort, ranges."""
    L = lib()
    n = len(scene.positions)
    pos = _c64(scene.positions, (n, 3))
    ls = _c64(scene.log_scales, (n, 3))
    rot = _c64(scene.rotations, (n, 4))
    op = _c64(scene.opacities, (n,))
    sh = _c64(scene.sh, (n, 48))
    status = np.zeros(n, dtype=np.int8)
    mean = np.zeros((n, 2))
    conic = np.zeros((n, 3))
    depth = np.zeros(n)
    color = np.zeros((n, 3))
    r2 = np.zeros(n)
    rect = np.zeros((n, 4), dtype=np.int32)
    camc, cfgc = camera_struct(cam), config_struct(cfg)
    L.oracle_preprocess(n, _ptr(pos), _ptr(ls), _ptr(rot), _ptr(op), _ptr(sh), ctypes.byref(camc),
                        ctypes.byref(cfgc), _ptr(status), _ptr(mean), _ptr(conic), _ptr(depth),
                        _ptr(color), _ptr(r2), _ptr(rect))
    keep = np.flatnonzero(status == 0)
    tiles_x = -(-int(cam.width) // TILE)
    tiles_y = -(-int(cam.height) // TILE)
    p_rect = np.ascontiguousarray(rect[keep])
    p_depth = np.ascontiguousarray(depth[keep])
    k = L.oracle_sort_pairs(len(keep), _ptr(p_rect), _ptr(p_depth), tiles_x, tiles_y, None, None, None, None)
    pair_tile = np.zeros(k, dtype=np.int32)
    pair_ref = np.zeros(k, dtype=np.int32)
    rs = np.zeros(tiles_x * tiles_y, dtype=np.int64)
    re = np.zeros(tiles_x * tiles_y, dtype=np.int64)
    L.oracle_sort_pairs(len(keep), _ptr(p_rect), _ptr(p_depth), tiles_x, tiles_y, _ptr(pair_tile),
                        _ptr(pair_ref), _ptr(rs), _ptr(re))
    return {
        "width": int(cam.width),
        "height": int(cam.height),
        "tiles_x": tiles_x,
        "tiles_y": tiles_y,
        "index": keep.astype(np.int64),  # assembled position of each ref
        "ids": np.asarray(scene.ids, dtype=np.int64)[keep],
        "means": np.ascontiguousarray(mean[keep]),
        "conics": np.ascontiguousarray(conic[keep]),
        "colors": np.ascontiguousarray(color[keep]),
        "opacities": np.ascontiguousarray(op[keep]),
        "depths": p_depth,
        "r2": np.ascontiguousarray(r2[keep]),
        "rects": p_rect,
        "pair_tile": pair_tile,
        "pair_ref": pair_ref,
        "range_start": rs,
        "range_end": re,
        "culled_near": int((status == 1).sum()),
        "dropped_degenerate": int((status == 2).sum()),
        "tile_pairs": int(k),
    }


def raster(pl: dict, cfg, threads: int = 0) -> dict:
    """render_frame's tile loop (render.py:194-233) restated for one engine."""
    L = lib()
    w, h = pl["width"], pl["height"]
    image = np.zeros((h, w, 3))
    contrib = np.zeros((h, w), dtype=np.int32)
    cost = np.zeros(4, dtype=np.int64)
    cfgc = config_struct(cfg)
    L.oracle_raster_frame(w, h, _ptr(pl["pair_ref"]), _ptr(pl["range_start"]), _ptr(pl["range_end"]),
                          _ptr(pl["means"]), _ptr(pl["conics"]), _ptr(pl["colors"]), _ptr(pl["opacities"]),
                          ctypes.byref(cfgc), int(threads), _ptr(image), _ptr(contrib), _ptr(cost))
    stats = {
        "alpha_eval_steps": int(cost[0]),
        "blend_steps": int(cost[1]),
        "leader_eval_steps": int(cost[2]),
        "warp_steps": int(cost[3]),
        "tile_pairs": pl["tile_pairs"],
        "culled_near": pl["culled_near"],
        "dropped_degenerate": pl["dropped_degenerate"],
    }
    return {"image": image, "contrib": contrib, "stats": stats}


def render(scene, cam, cfg, threads: int = 0) -> dict:
    pl = plan(scene, cam, cfg)
    out = raster(pl, cfg, threads)
    out["plan"] = pl
    return out


def select_clusters(cam, centroids, m: int, beta: float, normalization) -> list[int]:
    """select_clusters (residency.py:38-54) restated."""
    L = lib()
    cent = _c64(centroids)
    n = cent.shape[0]
    mean = _c64(normalization[0], (3,))
    out = np.zeros(m + 1, dtype=np.int32)
    camc = camera_struct(cam)
    rc = L.oracle_select_clusters(ctypes.byref(camc), _ptr(cent), n, int(m), float(beta), _ptr(mean),
                                  float(normalization[1]), _ptr(out))
    if rc != 0:
        raise ValueError(f"invalid selection arguments (m={m}, n={n})")
    return [int(v) for v in out]


def sorted_pair_ids(pl: dict) -> np.ndarray:
    """(tile_id, global id) sequence of the sorted pairs; invariant to ref numbering."""
    return np.stack([pl["pair_tile"].astype(np.int64), pl["ids"][pl["pair_ref"]]], axis=1)


def spec_keys(pl: dict) -> np.ndarray:
    """SPEC key layout tile<<32 | float32_bits(depth) along the sorted order."""
    d32 = pl["depths"][pl["pair_ref"]].astype(np.float32).view(np.uint32).astype(np.uint64)
    return (pl["pair_tile"].astype(np.uint64) << np.uint64(32)) | d32
