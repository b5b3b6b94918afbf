"""Runtime cluster selection and working-set assembly (residency.py drop-in).

``select_clusters`` (residency.py:38-54) runs on the GPU (kernel K0 in
csrc/preprocess.cu).  ``ResidentRenderer`` keeps the reference constructor
and its ``select`` / ``assemble`` / ``render_frame`` methods, but B200-first:
the whole compiled container lives in HBM (a 3M-splat scene is ~0.7 GB of
180 GB), so there is nothing to stream, prefetch or evict.  A frame is

    K0 select (device) -> working-set range table (device) -> K1..K9 render

with no host round trip in between: the assembled working set of the
reference (``SceneArrays.concatenate([shared, sel_0, ..., sel_M])``,
residency.py:217-220) is a list of chunk ranges of the resident scene, in the
same order, so splat positions and the depth tie-break are the reference's.
The ``prefetch`` / ``evict`` / ``lru_capacity`` / ``loader_delay`` arguments
are accepted for API compatibility and have no effect.
"""
from __future__ import annotations

import ctypes
import time
from pathlib import Path

import numpy as np
import torch

from . import _native
from .container import ClusteredContainer, load_clustered_scene
from .errors import InvalidArgumentError
from .model import CameraPose, SceneArrays
from .render import EngineConfig, RenderResult, _finish, get_renderer


def _select_on_device(cam: CameraPose, centroids: torch.Tensor, m: int, beta: float, normalization,
                      chunks: torch.Tensor, out_ids: torch.Tensor, ranges: torch.Tensor, stream=None) -> None:
    lib = _native.load()
    mean = (ctypes.c_double * 3)(*[float(v) for v in np.asarray(normalization[0], dtype=np.float64)])
    camc = _native.camera_struct(cam)
    st = stream if stream is not None else torch.cuda.current_stream(centroids.device)
    _native.check(lib.seele_select_clusters(ctypes.byref(camc), centroids.data_ptr(), int(centroids.shape[0]), int(m),
                                            float(beta), mean, float(normalization[1]), chunks.data_ptr(),
                                            out_ids.data_ptr(), ranges.data_ptr(), st.cuda_stream))


def select_clusters(cam: CameraPose, centroids, m: int, beta: float, normalization) -> list[int]:
    """residency.py:38-54 on the GPU: nearest cluster plus its m next-nearest."""
    cent = np.ascontiguousarray(np.asarray(centroids, dtype=np.float64))
    n = cent.shape[0]
    if m >= n:
        raise InvalidArgumentError(f"m must be < {n}, got {m}")
    if float(normalization[1]) <= 0.0:
        raise InvalidArgumentError("normalization scale must be positive")
    dev = torch.device("cuda", torch.cuda.current_device())
    cent_d = torch.from_numpy(cent).to(dev)
    chunks = torch.zeros((n + 1, 2), dtype=torch.int64, device=dev)
    out = torch.empty(m + 1, dtype=torch.int32, device=dev)
    ranges = torch.empty((m + 2, 2), dtype=torch.int64, device=dev)
    _select_on_device(cam, cent_d, m, beta, normalization, chunks, out, ranges)
    return [int(v) for v in out.cpu().numpy()]


class ResidentRenderer:
    """Renders a compiled (clustered) scene held entirely in HBM."""

    def __init__(self, handle, m: int | None = None, *, prefetch: bool = True, evict: bool = True,
                 evict_policy: str = "immediate", lru_capacity: int | None = None, loader_delay=None,
                 device=None):
        if evict_policy not in ("immediate", "lru"):
            raise InvalidArgumentError(f"unknown evict policy '{evict_policy}'")
        if isinstance(handle, (str, Path)):
            handle = load_clustered_scene(handle)
        if not isinstance(handle, ClusteredContainer):
            raise InvalidArgumentError(f"expected a container directory or ClusteredContainer, got {type(handle)}")
        self.container = handle
        self.m = handle.m if m is None else int(m)
        if self.m >= handle.num_clusters:
            raise InvalidArgumentError(f"m must be < {handle.num_clusters}, got {self.m}")
        self.beta = handle.beta
        self.normalization = handle.normalization
        self.device = torch.device("cuda", torch.cuda.current_device()) if device is None else torch.device(device)
        self.scene = handle.upload(self.device)
        self.centroids = torch.from_numpy(np.ascontiguousarray(handle.centroids)).to(self.device)
        self.chunks = torch.from_numpy(np.ascontiguousarray(handle.chunks)).to(self.device)
        self.sel_ids = torch.empty(self.m + 1, dtype=torch.int32, device=self.device)
        self.ranges = torch.empty((self.m + 2, 2), dtype=torch.int64, device=self.device)
        counts = handle.chunks[1:, 1]
        # upper bound of any working set: shared + the (1 + m) largest clusters
        self.n_max = int(handle.chunks[0, 1] + np.sort(counts)[::-1][:self.m + 1].sum())
        self.resident_bytes = handle.total_bytes

    # -- reference API -----------------------------------------------------------
    def select(self, cam: CameraPose) -> list[int]:
        self.select_async(cam)
        return [int(v) for v in self.sel_ids.cpu().numpy()]

    def select_async(self, cam: CameraPose, stream=None) -> torch.Tensor:
        """K0 on the device; fills self.sel_ids and the working-set range table."""
        _select_on_device(cam, self.centroids, self.m, self.beta, self.normalization, self.chunks, self.sel_ids,
                          self.ranges, stream)
        return self.ranges

    def assemble(self, selection) -> SceneArrays:
        """Host copy of the working set, in the reference order (shared, then the
        selection): residency.py:217-220.  The render path never calls this; it
        renders the same order from the device range table."""
        parts = [self.container.chunk_arrays(-1)] + [self.container.chunk_arrays(int(c)) for c in selection]
        return SceneArrays.concatenate(parts)

    def working_set_ids(self, selection) -> np.ndarray:
        ch = self.container.chunks
        idx = [np.arange(ch[0, 0], ch[0, 0] + ch[0, 1])] + \
              [np.arange(ch[c + 1, 0], ch[c + 1, 0] + ch[c + 1, 1]) for c in selection]
        return self.container.ids[np.concatenate(idx)]

    def render_device(self, cam: CameraPose, cfg: EngineConfig, renderer=None, stream=None, **kw):
        """Select + render without leaving the device (no host synchronisation)."""
        r = renderer or get_renderer(self.device)
        self.select_async(cam, stream)
        return r.render(self.scene, cam, cfg, ranges=self.ranges, n_ranges=self.m + 2, n_max=self.n_max,
                        stream=stream, **kw)

    def render_frame(self, cam: CameraPose, cfg: EngineConfig, output: str = "numpy") -> RenderResult:
        """residency.py:222-264 minus streaming: select + render of the resident
        working set; ``output`` as in render.render_frame."""
        t0 = time.perf_counter()
        r = get_renderer(self.device)
        self.select_async(cam)
        kw = dict(ranges=self.ranges, n_ranges=self.m + 2, n_max=self.n_max)
        res = _finish(r, lambda **k: r.render_checked(self.scene, cam, cfg, **k),
                      lambda **k: r.render_to_host(self.scene, cam, cfg, **k), output, t0, kw)
        res.stats.resident_bytes = self.resident_bytes
        return res

    def render_trajectory(self, cams, cfg: EngineConfig, *, depth: int = 2, pair_capacity: int | None = None):
        """Render a camera trajectory with ``depth`` frames in flight (B200
        extension of render_frame for trajectories): yields ``(index, image
        float32 (H,W,3), contributor counts int32 (H,W), stats int64)`` host
        views, valid until the next item is requested.  Frames
        whose tile pairs overflow ``pair_capacity`` are reported through
        their stats (``SEELE_STAT_OVERFLOW``); size the capacity first."""
        from .pipeline import TrajectoryRenderer
        cams = list(cams)
        if not cams:
            return
        w, h = int(cams[0].width), int(cams[0].height)
        for i, c in enumerate(cams):  # every slot's outputs and workspace are sized once, from the first camera
            if (int(c.width), int(c.height)) != (w, h):
                raise InvalidArgumentError(f"camera {i} is {c.width}x{c.height}, the trajectory is {w}x{h}")
        key = (w, h, int(depth), pair_capacity)
        tr = getattr(self, "_trajectory", None)
        if tr is None or tr[0] != key:  # workspaces and pinned buffers are kept across calls
            self._trajectory = None
            tr = self._trajectory = (key, TrajectoryRenderer(self, w, h, depth=depth, pair_capacity=pair_capacity))
        yield from tr[1].run(cams, cfg)

    def close(self) -> None:
        pass

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()
