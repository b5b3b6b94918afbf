"""Frame API of the reference (pkg/src/seele/render.py) on the B200 path.

``render_frame(scene, cam, cfg)`` keeps the reference signature
(render.py:172-179) and returns ``RenderResult(image, stats)``; ``plan_frame``
(render.py:90) returns the same ``FramePlan`` fields, read back from the GPU
plan.  Both drive the single native backend (``libseele_b200.so``): no
engine registry, no CPU fallback.

Throughput callers keep everything on the device with :class:`FrameRenderer`
and a :class:`~.device.DeviceScene`; the drop-in functions below add the
host<->device copies the reference API implies (numpy in, numpy out).
"""
from __future__ import annotations

import ctypes
import time
from dataclasses import dataclass, field

import numpy as np
import torch

from . import _native
from .device import DeviceScene
from .errors import ContractViolationError, DeviceError, InvalidArgumentError
from .model import ALPHA_THRESHOLD, GAMMA_THRESHOLD, TILE_SIZE, CameraPose, SceneArrays

ENGINES = ("ref", "cr")
PRECISIONS = ("fast", "exact")


@dataclass(frozen=True)
class EngineConfig:
    """render.py:31-51, plus ``precision`` ("fast": fp32 with guarded fp64
    re-decision, "exact": fp64 raster; identical discrete results)."""

    engine: str = "ref"
    group_w: int = 2
    background: tuple = (0.0, 0.0, 0.0)
    alpha_theta: float = ALPHA_THRESHOLD
    gamma_threshold: float = GAMMA_THRESHOLD
    sh_degree: int = 3
    tile_size: int = TILE_SIZE
    opacity_aware_filter: bool = True
    threads: int = 1
    precision: str = "fast"

    def __post_init__(self):
        if self.engine not in ENGINES:
            raise InvalidArgumentError(f"unknown engine '{self.engine}'")
        if self.group_w not in (1, 2, 4):
            raise InvalidArgumentError(f"group width must be 1, 2 or 4, got {self.group_w}")
        if self.threads < 1:
            raise InvalidArgumentError("threads must be >= 1")
        if self.precision not in PRECISIONS:
            raise InvalidArgumentError(f"unknown precision '{self.precision}'")
        if not 0 <= int(self.sh_degree) <= 3:
            raise InvalidArgumentError(f"SH degree must lie in [0, 3], got {self.sh_degree}")
        if self.tile_size != TILE_SIZE:
            raise InvalidArgumentError(f"tile size must be {TILE_SIZE}, got {self.tile_size}")


@dataclass
class WarpCost:
    """Lockstep step counters, summed over warps (rasterize.py:36-48).  The
    GPU raster produces them per frame (FrameStats); this mirrors the
    reference's accumulator for callers that sum costs themselves."""

    alpha_eval_steps: int = 0
    blend_steps: int = 0
    leader_eval_steps: int = 0
    warp_steps: int = 0

    def add(self, other: "WarpCost") -> None:
        self.alpha_eval_steps += other.alpha_eval_steps
        self.blend_steps += other.blend_steps
        self.leader_eval_steps += other.leader_eval_steps
        self.warp_steps += other.warp_steps


@dataclass
class FrameStats:
    """Per-frame counters (rasterize.py:51-86)."""

    alpha_eval_steps: int = 0
    blend_steps: int = 0
    leader_eval_steps: int = 0
    warp_steps: int = 0
    tile_pairs: int = 0
    culled_near: int = 0
    dropped_degenerate: int = 0
    resident_bytes: int = 0
    stalls: int = 0
    prefetch_hits: int = 0
    wall_ms: float = 0.0

    def add_cost(self, cost: WarpCost) -> None:
        """rasterize.py:66-70."""
        self.alpha_eval_steps += cost.alpha_eval_steps
        self.blend_steps += cost.blend_steps
        self.leader_eval_steps += cost.leader_eval_steps
        self.warp_steps += cost.warp_steps

    def as_dict(self) -> dict:
        return {k: getattr(self, k) for k in (
            "alpha_eval_steps", "blend_steps", "leader_eval_steps", "warp_steps", "tile_pairs", "culled_near",
            "dropped_degenerate", "resident_bytes", "stalls", "prefetch_hits", "wall_ms")}

    @classmethod
    def from_device(cls, stats: np.ndarray) -> "FrameStats":
        s = [int(v) for v in stats]
        return cls(alpha_eval_steps=s[_native.STAT_ALPHA_EVAL], blend_steps=s[_native.STAT_BLEND],
                   leader_eval_steps=s[_native.STAT_LEADER_EVAL], warp_steps=s[_native.STAT_WARP_STEPS],
                   tile_pairs=s[_native.STAT_TILE_PAIRS], culled_near=s[_native.STAT_CULLED_NEAR],
                   dropped_degenerate=s[_native.STAT_DROPPED_DEGENERATE])


@dataclass
class RenderResult:
    """render.py:82-87.  ``contrib_count`` (H, W) is the per-pixel number of
    blended splats; ``device_stats`` the raw int64 counter vector."""

    image: object
    stats: FrameStats
    contributions: np.ndarray | None = None
    contribution_ids: np.ndarray | None = None
    contrib_count: object = None
    device_stats: np.ndarray | None = None


@dataclass(frozen=True)
class TileGrid:
    """preprocess.py:30-56."""

    tile_size: int
    tiles_x: int
    tiles_y: int
    width: int
    height: int

    @classmethod
    def for_image(cls, width: int, height: int, tile_size: int = TILE_SIZE) -> "TileGrid":
        return cls(tile_size, -(-width // tile_size), -(-height // tile_size), width, height)

    @property
    def tile_count(self) -> int:
        return self.tiles_x * self.tiles_y

    def tile_origin(self, tile_id: int) -> tuple[int, int]:
        ty, tx = divmod(tile_id, self.tiles_x)
        return tx * self.tile_size, ty * self.tile_size


@dataclass(frozen=True)
class SortedTileRange:
    """sorting.py:16-22."""

    tile_id: int
    start: int
    end: int


INTERSECTION_DTYPE = np.dtype([("tile_id", "<i8"), ("gaussian_ref", "<i8"), ("depth", "<f8")])


@dataclass(frozen=True)
class TileIntersection:
    """One (tile, splat) pair surviving the binning test (preprocess.py:59-65);
    ``FramePlan.sorted_pairs`` holds them as INTERSECTION_DTYPE records."""

    tile_id: int
    gaussian_ref: int
    depth: float

    @classmethod
    def from_record(cls, rec) -> "TileIntersection":
        return cls(int(rec["tile_id"]), int(rec["gaussian_ref"]), float(rec["depth"]))


@dataclass
class FramePlan:
    """render.py:54-79, read back from the GPU workspace, plus the device-only
    extras (tile rects, assembled position of each ref)."""

    grid: TileGrid
    ids: np.ndarray
    means: np.ndarray
    conics: np.ndarray
    colors: np.ndarray
    opacities: np.ndarray
    depths: np.ndarray
    sorted_pairs: np.ndarray
    ranges: list
    culled_near: int
    dropped_degenerate: int
    rects: np.ndarray = field(default=None)
    positions: np.ndarray = field(default=None)

    def tile_gaussians(self, start: int, end: int) -> dict:
        refs = self.sorted_pairs["gaussian_ref"][start:end]
        return {"ids": self.ids[refs], "means": self.means[refs], "conics": self.conics[refs],
                "colors": self.colors[refs], "opacities": self.opacities[refs], "depths": self.depths[refs]}


@dataclass
class FrameOutput:
    """Device-side result of one frame (no host synchronisation implied)."""

    image: torch.Tensor          # (H, W, 3) float32
    contrib: torch.Tensor | None  # (H, W) int32
    stats: torch.Tensor          # (16,) int64
    n_ws: int | None = None


class FrameRenderer:
    """Owns the HBM workspace of one device and issues frames on a stream.

    The workspace is sized for ``n_max`` assembled splats and
    ``pair_capacity`` tile pairs; a frame that needs more pairs reports
    overflow in its stats and :meth:`render_checked` grows the workspace and
    re-renders.  Nothing is allocated per frame otherwise.
    """

    def __init__(self, device=None, pair_capacity: int | None = None):
        self.lib = _native.load()
        if not torch.cuda.is_available():
            raise DeviceError("no CUDA device: the B200 render path has no CPU fallback")
        dev = torch.device(device or "cuda")
        self.device = torch.device("cuda", torch.cuda.current_device()) if dev.index is None else dev
        self.pair_capacity = int(pair_capacity) if pair_capacity else 0
        self.n_max = 0
        self.size = (0, 0)
        self.workspace = None
        self.stats = torch.zeros(_native.STAT_COUNT, dtype=torch.int64, device=self.device)
        self._ranges = torch.zeros((_native.MAX_RANGES, 2), dtype=torch.int64, device=self.device)

    def reserve(self, n_max: int, width: int, height: int, pair_capacity: int | None = None) -> None:
        """Size the workspace; an explicit ``pair_capacity`` is used as given."""
        explicit = pair_capacity is not None
        cap = int(pair_capacity) if explicit else (self.pair_capacity or max(16 * max(n_max, 1), 1 << 16))
        same = (int(width), int(height)) == self.size
        if self.workspace is not None and n_max <= self.n_max and same and \
                (cap == self.pair_capacity or (not explicit and cap <= self.pair_capacity)):
            return
        n_max = max(int(n_max), self.n_max if same else 0, 1)
        nbytes = int(self.lib.seele_workspace_bytes(n_max, cap, int(width), int(height)))
        self.workspace = None
        torch.cuda.empty_cache()
        self.workspace = torch.zeros(nbytes, dtype=torch.uint8, device=self.device)  # look-back words must start zeroed
        self.n_max, self.pair_capacity, self.size = n_max, cap, (int(width), int(height))

    def render(self, scene: DeviceScene, cam: CameraPose, cfg: EngineConfig, *, ranges: torch.Tensor | None = None,
               n_ranges: int = 1, n_max: int | None = None, image: torch.Tensor | None = None,
               contrib: torch.Tensor | bool = True, stats: torch.Tensor | None = None,
               stream: torch.cuda.Stream | None = None,
               raster_stream: torch.cuda.Stream | None = None, keep_unbinned: bool = False) -> FrameOutput:
        """Asynchronous frame on ``stream`` (default: current stream); with
        ``raster_stream`` the raster is issued there after the plan stages."""
        w, h = int(cam.width), int(cam.height)
        n_max = int(n_max or scene.n)
        self.reserve(n_max, w, h)
        if ranges is None:
            self._ranges[0, 0] = 0
            self._ranges[0, 1] = scene.n
            ranges, n_ranges = self._ranges, 1
        if image is None:
            image = torch.empty((h, w, 3), dtype=torch.float32, device=self.device)
        else:
            _check_output("image", image, (h, w, 3), torch.float32, self.device)
        if contrib is True:
            contrib = torch.empty((h, w), dtype=torch.int32, device=self.device)
        elif contrib is False:
            contrib = None
        else:
            _check_output("contrib", contrib, (h, w), torch.int32, self.device)
        if stats is None:
            stats = self.stats
        else:
            _check_output("stats", stats, (_native.STAT_COUNT,), torch.int64, self.device)
        if ranges is not None:
            _check_output("ranges", ranges, (ranges.shape[0], 2), torch.int64, self.device)
            if not 1 <= n_ranges <= ranges.shape[0]:
                raise InvalidArgumentError(f"n_ranges {n_ranges} out of [1, {ranges.shape[0]}]")
        st = stream if stream is not None else torch.cuda.current_stream(self.device)
        sc = scene.struct()
        camc = _native.camera_struct(cam)
        cfgc = _native.config_struct(cfg, keep_unbinned)
        _native.check(self.lib.seele_render_split(
            ctypes.byref(sc), ranges.data_ptr(), int(n_ranges), ctypes.byref(camc), ctypes.byref(cfgc),
            self.workspace.data_ptr(), self.workspace.numel(), self.n_max, self.pair_capacity, image.data_ptr(),
            contrib.data_ptr() if contrib is not None else None, stats.data_ptr(), st.cuda_stream,
            raster_stream.cuda_stream if raster_stream is not None else None))
        return FrameOutput(image=image, contrib=contrib, stats=stats)

    def render_checked(self, scene: DeviceScene, cam: CameraPose, cfg: EngineConfig, *, before_sync=None,
                       **kw) -> tuple[FrameOutput, np.ndarray]:
        """Render, synchronise, and re-render with a larger workspace on overflow.
        ``before_sync()`` runs once, after the first render is issued and before
        the host waits for it (host work that overlaps the frame)."""
        for _ in range(4):
            out = self.render(scene, cam, cfg, **kw)
            if before_sync is not None:
                before_sync()
                before_sync = None
            host = out.stats.cpu().numpy()
            if not host[_native.STAT_OVERFLOW]:
                out.n_ws = int(host[_native.STAT_WORKING_SET])
                return out, host
            need = int(host[_native.STAT_TILE_PAIRS])
            self.reserve(self.n_max, self.size[0], self.size[1], pair_capacity=int(need * 1.25) + 1024)
        raise DeviceError("tile-pair workspace could not be grown enough")

    def render_to_host(self, scene: DeviceScene, cam: CameraPose, cfg: EngineConfig, *, before_sync=None, **kw):
        """Render and download image (float32), contributor counts and stats
        into pinned host buffers with one synchronisation; grows the workspace
        and re-renders on overflow.  The returned arrays are views into a
        two-deep ring of pinned buffers: valid until two more calls."""
        w, h = int(cam.width), int(cam.height)
        ring = getattr(self, "_ring", None)
        if ring is None or ring[0][0].shape[:2] != (h, w):
            ring = self._ring = [(torch.empty((h, w, 3), dtype=torch.float32, pin_memory=True),
                                  torch.empty((h, w), dtype=torch.int32, pin_memory=True),
                                  torch.empty(_native.STAT_COUNT, dtype=torch.int64, pin_memory=True))
                                 for _ in range(2)]
            self._ring_i = 0
        img_h, cnt_h, st_h = ring[self._ring_i]
        self._ring_i ^= 1
        for _ in range(4):
            out = self.render(scene, cam, cfg, **kw)
            st_h.copy_(out.stats, non_blocking=True)
            img_h.copy_(out.image, non_blocking=True)
            cnt_h.copy_(out.contrib, non_blocking=True)
            if before_sync is not None:
                before_sync()
                before_sync = None
            torch.cuda.current_stream(self.device).synchronize()
            host = st_h.numpy()
            if not host[_native.STAT_OVERFLOW]:
                return img_h.numpy(), cnt_h.numpy(), host.copy()
            need = int(host[_native.STAT_TILE_PAIRS])
            self.reserve(self.n_max, w, h, pair_capacity=int(need * 1.25) + 1024)
        raise DeviceError("tile-pair workspace could not be grown enough")

    def export_plan(self, scene: DeviceScene, cam: CameraPose, host_stats: np.ndarray,
                    working_ids: np.ndarray | None = None) -> FramePlan:
        """FramePlan of the last frame rendered by this renderer (synchronises)."""
        n_ws = int(host_stats[_native.STAT_WORKING_SET])
        k = int(host_stats[_native.STAT_TILE_PAIRS])
        w, h = self.size
        grid = TileGrid.for_image(w, h)
        d = self.device
        pair_pos = torch.empty(max(k, 1), dtype=torch.int32, device=d)
        pair_tile = torch.empty(max(k, 1), dtype=torch.int32, device=d)
        ranges = torch.empty((grid.tile_count, 2), dtype=torch.int32, device=d)
        status = torch.empty(max(n_ws, 1), dtype=torch.int8, device=d)
        depth = torch.empty(max(n_ws, 1), dtype=torch.float64, device=d)
        rect = torch.empty((max(n_ws, 1), 4), dtype=torch.int32, device=d)
        mean = torch.empty((max(n_ws, 1), 2), dtype=torch.float64, device=d)
        conic = torch.empty((max(n_ws, 1), 3), dtype=torch.float64, device=d)
        opac = torch.empty(max(n_ws, 1), dtype=torch.float64, device=d)
        color = torch.empty((max(n_ws, 1), 3), dtype=torch.float32, device=d)
        view = _native.PlanView(pair_pos.data_ptr(), pair_tile.data_ptr(), ranges.data_ptr(), status.data_ptr(),
                                depth.data_ptr(), rect.data_ptr(), mean.data_ptr(), conic.data_ptr(),
                                opac.data_ptr(), color.data_ptr())
        _native.check(self.lib.seele_plan_export(self.workspace.data_ptr(), self.n_max, self.pair_capacity, w, h,
                                                 n_ws, k, ctypes.byref(view),
                                                 torch.cuda.current_stream(d).cuda_stream))
        status = status.cpu().numpy()[:n_ws]
        ok = np.flatnonzero(status == 0)
        ref_of_pos = np.full(max(n_ws, 1), -1, dtype=np.int64)
        ref_of_pos[ok] = np.arange(len(ok))
        pp = pair_pos.cpu().numpy()[:k].astype(np.int64)
        pairs = np.empty(k, dtype=INTERSECTION_DTYPE)
        pairs["tile_id"] = pair_tile.cpu().numpy()[:k]
        pairs["gaussian_ref"] = ref_of_pos[pp]
        depth = depth.cpu().numpy()[:n_ws]
        pairs["depth"] = depth[pp]
        rg = ranges.cpu().numpy()
        ids_ws = working_ids if working_ids is not None else scene.host_ids[:n_ws]
        return FramePlan(
            grid=grid, ids=np.asarray(ids_ws)[ok], means=mean.cpu().numpy()[:n_ws][ok],
            conics=conic.cpu().numpy()[:n_ws][ok], colors=color.cpu().numpy()[:n_ws][ok].astype(np.float64),
            opacities=opac.cpu().numpy()[:n_ws][ok], depths=depth[ok], sorted_pairs=pairs,
            ranges=[SortedTileRange(int(t), int(s), int(e)) for t, (s, e) in enumerate(rg) if e > s],
            culled_near=int((status == 1).sum()), dropped_degenerate=int((status == 2).sum()),
            rects=rect.cpu().numpy()[:n_ws][ok], positions=ok)


def _check_output(name: str, t, shape: tuple, dtype, device) -> None:
    """Caller-supplied device buffers must match the frame exactly: the kernels
    write ``shape`` elements through the raw pointer."""
    if not isinstance(t, torch.Tensor):
        raise InvalidArgumentError(f"{name} must be a torch.Tensor, got {type(t).__name__}")
    if tuple(t.shape) != tuple(shape) or t.dtype != dtype or not t.is_contiguous() or t.device != device:
        raise InvalidArgumentError(
            f"{name} must be a contiguous {dtype} tensor of shape {tuple(shape)} on {device}, got "
            f"{t.dtype} {tuple(t.shape)} on {t.device}{'' if t.is_contiguous() else ' (non-contiguous)'}")


_renderers: dict = {}


def get_renderer(device=None) -> FrameRenderer:
    dev = torch.device(device or "cuda")
    if dev.index is None:
        dev = torch.device("cuda", torch.cuda.current_device())
    r = _renderers.get(dev)
    if r is None:
        r = _renderers[dev] = FrameRenderer(dev)
    return r


def _as_device_scene(scene) -> DeviceScene:
    if isinstance(scene, DeviceScene):
        return scene
    if isinstance(scene, SceneArrays) or hasattr(scene, "positions"):
        return DeviceScene.from_arrays(scene)
    raise InvalidArgumentError(f"cannot render a {type(scene).__name__}")


def render_frame(scene, cam: CameraPose, cfg: EngineConfig, *, record_contributions: bool = False,
                 plan: FramePlan | None = None, output: str = "numpy") -> RenderResult:
    """Drop-in for render.render_frame (render.py:172-233).

    ``scene`` is a ``SceneArrays`` (uploaded for this call) or a resident
    :class:`~.device.DeviceScene`.  ``plan`` is accepted for API
    compatibility; the GPU recomputes its plan (bit-equal discrete fields).
    ``output="numpy"`` returns the image as (H, W, 3) float64 like the
    reference; ``"numpy32"`` returns float32 views of pinned host buffers
    (valid until two more renders on this device; the fast host path);
    ``"torch"`` leaves image and counts on the device (float32 / int32).
    """
    t0 = time.perf_counter()
    dscene = _as_device_scene(scene)
    renderer = get_renderer(dscene.device)
    res = _finish(renderer, lambda **kw: renderer.render_checked(dscene, cam, cfg, **kw),
                  lambda **kw: renderer.render_to_host(dscene, cam, cfg, **kw), output, t0, {})
    if record_contributions:
        matrix, ids = contributions(renderer, dscene, cam, cfg, res.device_stats)
        res.contributions = matrix if output == "torch" else matrix.cpu().numpy()
        res.contribution_ids = ids
        res.stats.wall_ms = (time.perf_counter() - t0) * 1000.0
    return res


CONTRIB_MAX_BYTES = 4 << 30  # cap of the dense P x H*W fp64 contribution matrix (record_contributions)


def contributions(renderer: FrameRenderer, scene: DeviceScene, cam: CameraPose, cfg: EngineConfig,
                  host_stats: np.ndarray) -> tuple[torch.Tensor, np.ndarray]:
    """Dense per-splat, per-pixel blend weights T * alpha of the frame last
    rendered by ``renderer`` (render.py:186-193, 226-233): a (P, H*W) float64
    device tensor, row r = plan ref r (``plan.ids`` order), computed on the
    GPU with the reference schedule (seele_contributions), and the plan ids.
    Raises InvalidArgumentError when the matrix would exceed CONTRIB_MAX_BYTES
    (the reference allocates it in host memory; this path serves parity-size
    frames -- trajectory-scale harvests use clusters.harvest_top_contributors)."""
    n_ws = int(host_stats[_native.STAT_WORKING_SET])
    plan = renderer.export_plan(scene, cam, host_stats)
    p, n_pix = len(plan.ids), int(cam.width) * int(cam.height)
    if p * n_pix * 8 > CONTRIB_MAX_BYTES:
        raise InvalidArgumentError(f"record_contributions needs a {p} x {n_pix} float64 matrix "
                                   f"({p * n_pix * 8 / 2**30:.1f} GiB > {CONTRIB_MAX_BYTES / 2**30:.0f} GiB cap)")
    d = renderer.device
    out = torch.zeros((p, n_pix), dtype=torch.float64, device=d)
    row_of_pos = torch.empty(max(n_ws, 1), dtype=torch.int32, device=d)
    camc = _native.camera_struct(cam)
    cfgc = _native.config_struct(cfg)
    _native.check(renderer.lib.seele_contributions(
        renderer.workspace.data_ptr(), renderer.n_max, renderer.pair_capacity, ctypes.byref(camc),
        ctypes.byref(cfgc), n_ws, row_of_pos.data_ptr(), out.data_ptr(), torch.cuda.current_stream(d).cuda_stream))
    return out, plan.ids


def _finish(renderer, checked, to_host, output: str, t0: float, kw: dict) -> RenderResult:
    if output == "torch":
        out, host = checked(**kw)
        image, count = out.image, out.contrib
    elif output in ("numpy", "numpy32"):
        image, count, host = to_host(**kw)
        if output == "numpy":
            image, count = image.astype(np.float64), count.copy()
    else:
        raise InvalidArgumentError(f"unknown output '{output}'")
    stats = FrameStats.from_device(host)
    stats.wall_ms = (time.perf_counter() - t0) * 1000.0
    return RenderResult(image=image, stats=stats, contrib_count=count, device_stats=host)


def plan_frame(scene, cam: CameraPose, cfg: EngineConfig) -> FramePlan:
    """Drop-in for render.plan_frame (render.py:90-141), computed on the GPU."""
    dscene = _as_device_scene(scene)
    renderer = get_renderer(dscene.device)
    _, host = renderer.render_checked(dscene, cam, cfg, keep_unbinned=True)
    return renderer.export_plan(dscene, cam, host)


def frame_skip_bound(scene, cam: CameraPose, cfg: EngineConfig, plan: FramePlan | None = None) -> np.ndarray:
    """Drop-in for render.frame_skip_bound (render.py:236-256): per-pixel
    certified error bound (H, W) float64 of the group-gated engine with group
    width ``cfg.group_w`` (skipped_contribution_bound, rasterize.py:325-377),
    computed on the GPU in fp64 over the GPU's own plan.  ``plan`` is
    accepted for API compatibility (the GPU plan is bit-equal on the pairs)."""
    dscene = _as_device_scene(scene)
    renderer = get_renderer(dscene.device)
    renderer.render_checked(dscene, cam, cfg)  # plan (pairs, ranges, fp64 splats) into the workspace
    w, h = renderer.size
    d = renderer.device
    bound = torch.empty((h, w), dtype=torch.float64, device=d)
    camc = _native.camera_struct(cam)
    cfgc = _native.config_struct(cfg)
    _native.check(renderer.lib.seele_skip_bound(renderer.workspace.data_ptr(), renderer.n_max, renderer.pair_capacity,
                                                ctypes.byref(camc), ctypes.byref(cfgc), bound.data_ptr(),
                                                torch.cuda.current_stream(d).cuda_stream))
    return bound.cpu().numpy()


def check_sorted_depths(depths: np.ndarray) -> None:
    """_check_sorted (rasterize.py:154-156) for caller-supplied tile lists."""
    if len(depths) > 1 and np.any(np.diff(depths) < 0):
        raise ContractViolationError("tile gaussians are not in front-to-back order")


STAGES = ("preprocess", "depth_rank", "binning_sort", "raster")


def enable_stage_timing(on: bool = True) -> None:
    """Record CUDA events at the stage boundaries of every frame on this thread."""
    lib = _native.load()
    _native.check(lib.seele_profile_enable(1 if on else 0))


def read_stage_timing() -> dict:
    """Stage times (ms) of the most recent frame (synchronises on its last event)."""
    lib = _native.load()
    buf = (ctypes.c_float * 4)()
    _native.check(lib.seele_profile_read(buf, 4))
    return {name: float(buf[i]) for i, name in enumerate(STAGES)}
