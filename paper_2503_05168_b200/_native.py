"""ctypes binding of ``libseele_b200.so`` (include/seele_b200.h).

The library is built in-tree by ``__graft_entry__.build()`` (csrc/Makefile,
nvcc -gencode arch=compute_100a,code=sm_100a).  There is no fallback: if the
library is missing or no CUDA device is present, every render call raises
:class:`~.errors.DeviceError`.
"""
from __future__ import annotations

import ctypes
import os
from pathlib import Path

from .errors import DeviceError, raise_for_status

# SEELE_LIB: development override (A/B builds of the same library)
LIB_PATH = Path(os.environ.get("SEELE_LIB") or Path(__file__).resolve().parent / "libseele_b200.so")
ABI_VERSION = 1

# enum indices of the device stats vector (seele_b200.h)
STAT_ALPHA_EVAL = 0
STAT_BLEND = 1
STAT_LEADER_EVAL = 2
STAT_WARP_STEPS = 3
STAT_TILE_PAIRS = 4
STAT_CULLED_NEAR = 5
STAT_DROPPED_DEGENERATE = 6
STAT_PROJECTED = 7
STAT_BINNED = 8
STAT_WORKING_SET = 9
STAT_OVERFLOW = 10
STAT_SKIPPED_PIXEL_STEPS = 11
STAT_ALPHA_REDECIDE = 12
STAT_T_AMBIGUOUS = 13
STAT_LIVE_PIXEL_STEPS = 14
STAT_PIXEL_BLENDS = 15
STAT_COUNT = 16

LAYOUT_F64 = 0
LAYOUT_PLANES = 1
PRECISION_FAST = 0
PRECISION_EXACT = 1
KEEP_UNBINNED = 0x100  # SEELE_KEEP_UNBINNED, OR-ed into precision
MAX_RANGES = 64

EXPORTED_SYMBOLS = (
    "seele_workspace_bytes",
    "seele_render",
    "seele_render_split",
    "seele_partition_create",
    "seele_select_clusters",
    "seele_plan_export",
    "seele_skip_bound",
    "seele_contributions",
    "seele_harvest_topk",
    "seele_psnr",
    "seele_ssim",
    "seele_metrics_scratch_doubles",
    "seele_profile_enable",
    "seele_profile_read",
    "seele_last_error",
    "seele_abi_version",
    "seele_launch_count",
)


class Camera(ctypes.Structure):
    _fields_ = [
        ("position", ctypes.c_double * 3),
        ("orientation", ctypes.c_double * 4),
        ("fov_x", ctypes.c_double),
        ("fov_y", ctypes.c_double),
        ("near_clip", ctypes.c_double),
        ("width", ctypes.c_int32),
        ("height", ctypes.c_int32),
    ]


class Config(ctypes.Structure):
    _fields_ = [
        ("engine", ctypes.c_int32),
        ("group_w", ctypes.c_int32),
        ("sh_degree", ctypes.c_int32),
        ("opacity_aware", ctypes.c_int32),
        ("alpha_theta", ctypes.c_double),
        ("gamma_threshold", ctypes.c_double),
        ("background", ctypes.c_double * 3),
        ("precision", ctypes.c_int32),
        ("tile_size", ctypes.c_int32),
    ]


class Scene(ctypes.Structure):
    _fields_ = [
        ("layout", ctypes.c_int32),
        ("_pad", ctypes.c_int32),
        ("n", ctypes.c_int64),
        ("positions", ctypes.c_void_p),
        ("log_scales", ctypes.c_void_p),
        ("rotations", ctypes.c_void_p),
        ("opacities", ctypes.c_void_p),
        ("sh", ctypes.c_void_p),
        ("planes", ctypes.c_void_p),
        ("plane_stride", ctypes.c_int64),
        ("ids", ctypes.c_void_p),
    ]


class PlanView(ctypes.Structure):
    _fields_ = [(name, ctypes.c_void_p) for name in
                ("pair_pos", "pair_tile", "ranges", "status", "depth", "rect", "mean", "conic", "opacity", "color")]


_lib = None


def load(required: bool = True):
    """Load the native library once; raise DeviceError if it is missing."""
    global _lib
    if _lib is not None:
        return _lib
    if not LIB_PATH.exists():
        if not required:
            return None
        raise DeviceError(f"{LIB_PATH} is missing; run __graft_entry__.build() (no CPU fallback exists)")
    lib = ctypes.CDLL(str(LIB_PATH))
    P, I32, I64 = ctypes.c_void_p, ctypes.c_int32, ctypes.c_int64
    lib.seele_workspace_bytes.argtypes = [I64, I64, I32, I32]
    lib.seele_workspace_bytes.restype = ctypes.c_size_t
    lib.seele_render.argtypes = [P, P, I32, P, P, P, ctypes.c_size_t, I64, I64, P, P, P, P]
    lib.seele_render.restype = ctypes.c_int
    lib.seele_render_split.argtypes = [P, P, I32, P, P, P, ctypes.c_size_t, I64, I64, P, P, P, P, P]
    lib.seele_partition_create.restype = I32
    lib.seele_partition_create.argtypes = [I32, I32, P, P, P, P]
    lib.seele_render_split.restype = ctypes.c_int
    lib.seele_select_clusters.argtypes = [P, P, I32, I32, ctypes.c_double, P, ctypes.c_double, P, P, P, P]
    lib.seele_select_clusters.restype = ctypes.c_int
    lib.seele_plan_export.argtypes = [P, I64, I64, I32, I32, I64, I64, P, P]
    lib.seele_plan_export.restype = ctypes.c_int
    lib.seele_skip_bound.argtypes = [P, I64, I64, P, P, P, P]
    lib.seele_skip_bound.restype = ctypes.c_int
    lib.seele_contributions.argtypes = [P, I64, I64, P, P, I64, P, P, P]
    lib.seele_contributions.restype = ctypes.c_int
    lib.seele_harvest_topk.argtypes = [P, I64, I64, P, P, P, I32, P, P]
    lib.seele_harvest_topk.restype = ctypes.c_int
    lib.seele_psnr.argtypes = [P, P, I64, P, P, P]
    lib.seele_psnr.restype = ctypes.c_int
    lib.seele_ssim.argtypes = [P, P, I32, I32, P, P, P]
    lib.seele_ssim.restype = ctypes.c_int
    lib.seele_metrics_scratch_doubles.argtypes = [I32, I32]
    lib.seele_metrics_scratch_doubles.restype = I64
    lib.seele_profile_enable.argtypes = [I32]
    lib.seele_profile_enable.restype = ctypes.c_int
    lib.seele_profile_read.argtypes = [P, I32]
    lib.seele_profile_read.restype = ctypes.c_int
    lib.seele_last_error.argtypes = []
    lib.seele_last_error.restype = ctypes.c_char_p
    lib.seele_abi_version.argtypes = []
    lib.seele_abi_version.restype = I32
    lib.seele_launch_count.argtypes = []
    lib.seele_launch_count.restype = I64
    if lib.seele_abi_version() != ABI_VERSION:
        raise DeviceError(f"libseele_b200 ABI {lib.seele_abi_version()} != expected {ABI_VERSION}; rebuild")
    _lib = lib
    return lib


def check(code: int) -> None:
    if code != 0:
        msg = _lib.seele_last_error().decode() if _lib is not None else ""
        raise_for_status(code, msg)


def camera_struct(cam) -> Camera:
    c = Camera()
    c.position[:] = [float(v) for v in cam.position]
    c.orientation[:] = [float(v) for v in cam.orientation]
    c.fov_x, c.fov_y, c.near_clip = float(cam.fov_x), float(cam.fov_y), float(cam.near_clip)
    c.width, c.height = int(cam.width), int(cam.height)
    return c


def config_struct(cfg, keep_unbinned: bool = False) -> Config:
    c = Config()
    c.engine = 0 if cfg.engine == "ref" else 1
    c.group_w = int(cfg.group_w)
    c.sh_degree = int(cfg.sh_degree)
    c.opacity_aware = 1 if cfg.opacity_aware_filter else 0
    c.alpha_theta = float(cfg.alpha_theta)
    c.gamma_threshold = float(cfg.gamma_threshold)
    c.background[:] = [float(v) for v in cfg.background]
    c.precision = PRECISION_EXACT if getattr(cfg, "precision", "fast") == "exact" else PRECISION_FAST
    if keep_unbinned:  # plan export: every projected splat's record, not only the binned ones
        c.precision |= KEEP_UNBINNED
    c.tile_size = int(cfg.tile_size)
    return c
