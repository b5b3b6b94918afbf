"""Streaming residency (residency.py:57-264): render a
compiled scene that need not fit in HBM.

The shared chunk stays resident; clusters live in fixed-size device slots
filled from pinned host memory by ``cudaMemcpyAsync`` on a dedicated copy
stream (the paper's "dedicated GPU stream").  Per frame, exactly the
reference's state machine:

* select the clusters of the pose; a selected cluster that is resident or
  already in flight is a prefetch hit, anything else is a stall and is
  loaded now (the render stream waits on its copy event, the host does not);
* render the working set [shared, selection...] from the slots through the
  device range table (the same kernels as the resident path, so images,
  contributor counts and counters are identical to it);
* predict the next pose (constant velocity, slerp-extrapolated orientation,
  residency.py:57-95), prefetch its clusters on the copy stream;
* evict outside (current selection + prediction): "immediate" drops all of
  them, "lru" keeps up to ``lru_capacity`` clusters (least recently used
  dropped first, ties by id; a prefetch counts as loaded).  A freed slot is
  rewritten only after the last render that read it (the copy stream waits
  on that render's event).

Counters: ``stalls`` and ``prefetch_hits`` follow the reference exactly for
a loader that finishes a prefetch within a frame (the reference's own runs:
its loader thread is faster than a frame); ``resident_bytes`` counts a
prefetch from the moment it is issued (the reference counts it when its
loader thread finishes -- timing-dependent).
"""
from __future__ import annotations

import math
import time
from pathlib import Path

import numpy as np
import torch

from .container import BYTES_PER_GAUSSIAN, ClusteredContainer, load_clustered_scene
from .device import N_PLANES, DeviceScene
from .errors import InvalidArgumentError
from .model import CameraPose
from .render import EngineConfig, RenderResult, _finish, get_renderer
from .residency import _select_on_device


def _slerp_extrapolate(q0: np.ndarray, q1: np.ndarray) -> np.ndarray:
    """residency.py:57-74: slerp(q0, q1, t = 2), renormalised."""
    q0 = np.asarray(q0, dtype=np.float64)
    q1 = np.asarray(q1, dtype=np.float64)
    dot = float(q0 @ q1)
    if dot < 0.0:
        q1, dot = -q1, -dot
    if dot < 1e-6 or dot > 1.0 - 1e-12:
        return q1 / np.linalg.norm(q1)
    math.acos(min(dot, 1.0))  # (the reference evaluates theta; the closed form below does not need it)
    out = -q0 + 2.0 * dot * q1
    return out / np.linalg.norm(out)


def predict_pose(prev: CameraPose, curr: CameraPose) -> CameraPose:
    """residency.py:77-95: constant-velocity extrapolation of position and orientation."""
    position = curr.position + (curr.position - prev.position)
    dot = float(prev.orientation @ curr.orientation)
    orientation = curr.orientation if abs(dot) < 1e-6 else _slerp_extrapolate(prev.orientation, curr.orientation)
    return CameraPose(position=position, orientation=orientation, fov_x=curr.fov_x, fov_y=curr.fov_y,
                      width=curr.width, height=curr.height, near_clip=curr.near_clip)


class StreamingRenderer:
    """residency.ResidentRenderer (residency.py:98-264) with the clusters
    streamed through device slots (see the module docstring)."""

    def __init__(self, handle, m: int | None = None, *, prefetch: bool = True, evict: bool = True,
                 evict_policy: str = "immediate", lru_capacity: int | None = None, device=None):
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
        self.prefetch_enabled, self.evict_enabled, self.evict_policy = prefetch, evict, evict_policy
        self.lru_capacity = 2 * (1 + self.m) if lru_capacity is None else int(lru_capacity)
        self.device = torch.device("cuda", torch.cuda.current_device()) if device is None else torch.device(device)
        ch = handle.chunks
        self.shared_count = int(ch[0, 1])
        self.slot_size = int(ch[1:, 1].max()) if len(ch) > 1 else 0
        # resident clusters at most: the kept set (lru capacity / current + predicted) plus, before eviction
        # runs, one frame's stalls (1 + m), the prefetches still in flight (1 + m) and the new ones (1 + m)
        keep = max(self.lru_capacity, 2 * (1 + self.m)) if evict_policy == "lru" else 2 * (1 + self.m)
        self.n_slots = handle.num_clusters if not evict else min(handle.num_clusters, keep + 3 * (1 + self.m))
        cap = self.shared_count + self.n_slots * self.slot_size
        self.host_planes = torch.from_numpy(np.ascontiguousarray(handle.planes)).pin_memory()
        self.host_ids = torch.from_numpy(np.ascontiguousarray(handle.ids)).pin_memory()
        planes = torch.zeros((N_PLANES, max(cap, 1), 4), dtype=torch.float32, device=self.device)
        ids = torch.zeros(max(cap, 1), dtype=torch.int64, device=self.device)
        host_ids = np.zeros(max(cap, 1), dtype=np.int64)
        self.scene = DeviceScene("planes", cap, {"planes": planes}, ids, host_ids)
        self.copy_stream = torch.cuda.Stream(self.device)
        self._last_render = torch.cuda.Event()
        self._copy(0, int(ch[0, 0]), self.shared_count)  # the shared chunk, once
        torch.cuda.current_stream(self.device).wait_stream(self.copy_stream)
        self.free_slots = list(range(self.n_slots))
        self.slot_busy: dict[int, torch.cuda.Event] = {}  # slot -> the last render that read it
        self.slot_of: dict[int, int] = {}
        self.ready: dict[int, torch.cuda.Event] = {}
        self.resident: set[int] = set()
        self.inflight: set[int] = set()
        self.last_used: dict[int, int] = {}
        self.clock = 0
        self.prev_pose: CameraPose | None = None
        self.stall_count = self.prefetch_hit_count = 0
        self.resident_bytes = self.peak_resident_bytes = 0
        self._recount()
        counts = ch[1:, 1]
        self.n_max = int(self.shared_count + np.sort(counts)[::-1][:self.m + 1].sum())
        self.ranges = torch.empty((self.m + 2, 2), dtype=torch.int64, device=self.device)
        self._rows_h = torch.empty((self.m + 2, 2), dtype=torch.int64).pin_memory()
        # K0 state: centroids resident once, fixed buffers, its own stream
        if self.m >= handle.num_clusters:
            raise InvalidArgumentError(f"m must be < {handle.num_clusters}, got {self.m}")
        self.sel_stream = torch.cuda.Stream(self.device)
        self.sel_centroids = torch.from_numpy(np.ascontiguousarray(handle.centroids, dtype=np.float64)).to(self.device)
        self.sel_chunks = torch.zeros((handle.num_clusters + 1, 2), dtype=torch.int64, device=self.device)
        self.sel_ids = torch.empty(self.m + 1, dtype=torch.int32, device=self.device)
        self.sel_ranges = torch.empty((self.m + 2, 2), dtype=torch.int64, device=self.device)
        self.sel_host = torch.empty(self.m + 1, dtype=torch.int32).pin_memory()

    # -- residency ---------------------------------------------------------------
    def _copy(self, dst: int, src: int, count: int) -> None:
        if count <= 0:
            return
        with torch.cuda.stream(self.copy_stream):
            self.scene.tensors["planes"][:, dst:dst + count].copy_(self.host_planes[:, src:src + count],
                                                                   non_blocking=True)
            self.scene.ids[dst:dst + count].copy_(self.host_ids[src:src + count], non_blocking=True)
        self.scene.host_ids[dst:dst + count] = self.container.ids[src:src + count]

    def _load(self, cid: int) -> None:
        if not self.free_slots:
            raise InvalidArgumentError("no free cluster slot: lru_capacity too large for the slot pool")
        slot = self.free_slots.pop(0)
        start, count = (int(v) for v in self.container.chunks[cid + 1])
        if slot in self.slot_busy:  # the slot's previous cluster is no longer read
            self.copy_stream.wait_event(self.slot_busy.pop(slot))
        self._copy(self.shared_count + slot * self.slot_size, start, count)
        ev = torch.cuda.Event()
        ev.record(self.copy_stream)
        self.slot_of[cid], self.ready[cid] = slot, ev

    def _cluster_bytes(self, cid: int) -> int:
        return int(self.container.chunks[cid + 1, 1]) * BYTES_PER_GAUSSIAN

    def _recount(self) -> None:
        total = self.shared_count * BYTES_PER_GAUSSIAN + sum(self._cluster_bytes(c) for c in self.resident | self.inflight)
        self.resident_bytes = total
        self.peak_resident_bytes = max(self.peak_resident_bytes, total)

    def _ensure_resident(self, needed) -> None:
        """residency.py:199-217."""
        for cid in needed:
            if cid in self.resident or cid in self.inflight:
                self.prefetch_hit_count += 1
                self.inflight.discard(cid)
                self.resident.add(cid)
                continue
            self.stall_count += 1
            self._load(cid)
            self.resident.add(cid)
        self._recount()

    # -- reference API -----------------------------------------------------------
    def select(self, cam: CameraPose) -> list[int]:
        """select_clusters (residency.py:38-54) by K0 on the device, on a stream of its own: the host needs
        the ids to drive the copies, and the read-back must not wait for a frame rendering meanwhile."""
        with torch.cuda.stream(self.sel_stream):
            _select_on_device(cam, self.sel_centroids, self.m, self.beta, self.normalization, self.sel_chunks,
                              self.sel_ids, self.sel_ranges, self.sel_stream)
            self.sel_host.copy_(self.sel_ids, non_blocking=True)
        self.sel_stream.synchronize()
        return [int(v) for v in self.sel_host.numpy()]

    def render_frame(self, cam: CameraPose, cfg: EngineConfig, output: str = "numpy") -> RenderResult:
        """residency.py:222-264."""
        t0 = time.perf_counter()
        # prefetches issued by earlier frames have landed by now (the reference's loader thread keeps up
        # with a frame): from here on they are resident, and evictable
        self.resident |= self.inflight
        self.inflight.clear()
        needed = self.select(cam)
        self._ensure_resident(needed)
        st = torch.cuda.current_stream(self.device)
        rows = [[0, self.shared_count]] + [[self.shared_count + self.slot_of[c] * self.slot_size,
                                            int(self.container.chunks[c + 1, 1])] for c in needed]
        rows_h = self._rows_h
        rows_h[:len(rows)] = torch.tensor(rows, dtype=torch.int64)
        self.ranges[:len(rows)].copy_(rows_h[:len(rows)], non_blocking=True)  # (reused after this frame's sync)
        for c in needed:
            st.wait_event(self.ready[c])
        r = get_renderer(self.device)

        def after_issue():
            # prediction, prefetch and eviction on the host while the GPU renders the frame
            self._last_render = torch.cuda.Event()
            self._last_render.record(st)
            self._advance(cam, needed)

        kw = dict(ranges=self.ranges, n_ranges=len(rows), n_max=self.n_max, before_sync=after_issue)
        res = _finish(r, lambda **k: r.render_checked(self.scene, cam, cfg, **k),
                      lambda **k: r.render_to_host(self.scene, cam, cfg, **k), output, t0, kw)
        self._recount()
        res.stats.resident_bytes = self.resident_bytes
        res.stats.stalls = self.stall_count
        res.stats.prefetch_hits = self.prefetch_hit_count
        return res

    def _advance(self, cam: CameraPose, needed) -> None:
        """residency.py:241-259: prefetch the clusters of the predicted next pose, evict the rest."""
        predicted = self.select(predict_pose(self.prev_pose if self.prev_pose is not None else cam, cam))
        self.prev_pose = cam
        if self.prefetch_enabled:
            for cid in predicted:
                if cid not in self.resident and cid not in self.inflight:
                    self._load(cid)
                    self.inflight.add(cid)
        if self.evict_enabled:
            keep = set(needed) | set(predicted)
            self.clock += 1
            for cid in needed:
                self.last_used[cid] = self.clock
            if self.evict_policy == "immediate":
                victims = [c for c in self.resident if c not in keep]
            else:  # (this frame's prefetches are still in flight: not counted, like the reference's)
                overflow = len(self.resident) - self.lru_capacity
                cand = sorted((c for c in self.resident if c not in keep), key=lambda c: (self.last_used.get(c, 0), c))
                victims = cand[:max(overflow, 0)]
            for cid in victims:
                self.resident.discard(cid)
                self.last_used.pop(cid, None)
                slot = self.slot_of.pop(cid)
                self.slot_busy[slot] = self._last_render
                self.free_slots.append(slot)
                self.ready.pop(cid, None)

    def close(self) -> None:
        pass

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()
