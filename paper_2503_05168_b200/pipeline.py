"""Frame pipelining over CUDA streams for trajectory rendering.

Frames of a camera trajectory are independent (the scene is read-only and
every frame owns its workspace and outputs), so a trajectory renders with
``depth`` frames in flight: slot ``k % depth`` issues frame ``k`` on its own
stream with its own workspace, range table and output buffers.  The
latency-bound stages of one frame (cluster lookup, radix passes, scans) then
overlap the compute-bound raster of another on the same GPU, with no
synchronisation between slots.  Each slot's stream orders reuse of its
buffers; a slot's outputs stay valid until the slot is used again
(``depth`` submissions later).
"""
from __future__ import annotations

import ctypes
from dataclasses import dataclass

import torch

from . import _native
from .model import CameraPose
from .render import EngineConfig, FrameOutput, FrameRenderer
from .residency import ResidentRenderer, _select_on_device


_PARTITIONS: dict = {}


def partition_streams(device: torch.device, plan_sms: int, n: int):
    """``n`` plan streams on a partition of ``plan_sms`` SMs and ``n`` raster
    streams on the device's other SMs (seele_partition_create: green
    contexts, which live for the process; one partition per (device,
    plan_sms), its streams shared by every pipeline that asks).  Returns
    (plan streams, raster streams, plan SMs, raster SMs)."""
    key = (torch.device(device).index or 0, int(plan_sms))
    part = _PARTITIONS.get(key)
    if part is None or len(part[0]) < n:
        lib = _native.load()
        k = max(int(n), 4)
        ps, rs = (ctypes.c_void_p * k)(), (ctypes.c_void_p * k)()
        po, ro = ctypes.c_int32(), ctypes.c_int32()
        with torch.cuda.device(device):
            _native.check(lib.seele_partition_create(int(plan_sms), k, ps, rs, ctypes.byref(po), ctypes.byref(ro)))
        part = ([torch.cuda.ExternalStream(ps[i], device=device) for i in range(k)],
                [torch.cuda.ExternalStream(rs[i], device=device) for i in range(k)], po.value, ro.value)
        _PARTITIONS[key] = part
    return part[0][:n], part[1][:n], part[2], part[3]


@dataclass
class _Slot:
    renderer: FrameRenderer
    stream: torch.cuda.Stream          # plan stages (high priority)
    raster_stream: torch.cuda.Stream   # raster (low priority)
    free: torch.cuda.Event             # the slot's last raster finished
    sel_ids: torch.Tensor
    ranges: torch.Tensor
    image: torch.Tensor
    contrib: torch.Tensor
    stats: torch.Tensor
    done: torch.cuda.Event
    outs: list = None          # extra output buffer sets (image, contrib, stats, free event), alternated
    out_next: int = 0


class FramePipeline:
    """Renders frames of a resident (clustered) scene ``depth`` at a time."""

    def __init__(self, rr: ResidentRenderer, width: int, height: int, *, depth: int = 2,
                 pair_capacity: int | None = None, contrib: bool = True, split: bool = False,
                 raster_priority: bool = False, out_buffers: int = 1, partition: int | None = None):
        if depth < 1:
            raise ValueError("depth must be >= 1")
        self.rr = rr
        self.device = rr.device
        self.size = (int(width), int(height))
        self.slots: list[_Slot] = []
        # partition = N: plan stages on N SMs, rasters on the rest (green contexts), so one frame's plan
        # runs beside another frame's raster instead of waiting for its CTAs to drain
        self.partition = None
        if partition:
            split = True
            pstreams, rstreams, psms, rsms = partition_streams(self.device, partition, depth)
            self.partition = (psms, rsms)
        for k in range(depth):
            r = FrameRenderer(self.device)
            r.reserve(rr.n_max, width, height, pair_capacity=pair_capacity)
            least, greatest = torch.cuda.Stream.priority_range()  # lower number = higher priority
            plan_pri, raster_pri = (least, greatest) if raster_priority else (greatest, least)
            self.slots.append(_Slot(
                renderer=r,
                stream=pstreams[k] if partition else torch.cuda.Stream(self.device, priority=plan_pri if split else 0),
                raster_stream=rstreams[k] if partition else torch.cuda.Stream(self.device,
                                                                              priority=raster_pri if split else 0),
                free=torch.cuda.Event(),
                sel_ids=torch.empty(rr.m + 1, dtype=torch.int32, device=self.device),
                ranges=torch.empty((rr.m + 2, 2), dtype=torch.int64, device=self.device),
                image=torch.empty((height, width, 3), dtype=torch.float32, device=self.device),
                contrib=torch.empty((height, width), dtype=torch.int32, device=self.device) if contrib else None,
                stats=torch.zeros(_native.STAT_COUNT, dtype=torch.int64, device=self.device),
                done=torch.cuda.Event()))
            s = self.slots[-1]
            s.outs = [(s.image, s.contrib, s.stats, torch.cuda.Event())]
            for _ in range(out_buffers - 1):  # more output sets: a consumer may still be reading the last one
                s.outs.append((torch.empty_like(s.image), torch.empty_like(s.contrib) if contrib else None,
                               torch.zeros_like(s.stats), torch.cuda.Event()))
        self._next = 0
        self.split = split

    @property
    def depth(self) -> int:
        return len(self.slots)

    def wait_for(self, stream: torch.cuda.Stream) -> None:
        """Make every slot stream wait for the work already queued on ``stream``."""
        ev = torch.cuda.Event()
        ev.record(stream)
        for s in self.slots:
            s.stream.wait_event(ev)
            s.raster_stream.wait_event(ev)

    def join(self, stream: torch.cuda.Stream) -> None:
        """Make ``stream`` wait for every frame submitted so far."""
        for s in self.slots:
            s.done.record(s.raster_stream if self.split else s.stream)
            stream.wait_event(s.done)

    def output_stream(self, k: int) -> torch.cuda.Stream:
        """Stream on which slot k's outputs are complete."""
        s = self.slots[k]
        return s.raster_stream if self.split else s.stream

    def slot_of_next(self) -> int:
        return self._next

    def submit(self, cam: CameraPose, cfg: EngineConfig) -> FrameOutput:
        """Queue one frame (cluster lookup + render) on the next slot; returns
        its device outputs without synchronising."""
        s = self.slots[self._next]
        self._next = (self._next + 1) % len(self.slots)
        rr = self.rr
        image, contrib, stats, free = s.outs[s.out_next]
        s.out_next = (s.out_next + 1) % len(s.outs)
        if len(s.outs) > 1:  # this output set is rewritten only after its consumer released it
            s.stream.wait_event(free)
        if self.split:  # the slot's workspace and outputs are reused: wait for its previous raster
            s.stream.wait_event(s.free)
        _select_on_device(cam, rr.centroids, rr.m, rr.beta, rr.normalization, rr.chunks, s.sel_ids, s.ranges,
                          s.stream)
        out = s.renderer.render(rr.scene, cam, cfg, ranges=s.ranges, n_ranges=rr.m + 2, n_max=rr.n_max,
                                image=image, contrib=contrib if contrib is not None else False,
                                stats=stats, stream=s.stream,
                                raster_stream=s.raster_stream if self.split else None)
        if self.split:
            s.free.record(s.raster_stream)
        out.release = free  # record on the consumer's stream once done with the outputs
        return out


class TrajectoryRenderer:
    """Host-facing trajectory rendering: frames are pipelined on the device
    (FramePipeline, two output sets per slot) and each frame's image,
    contributor counts and stats are copied into pinned host buffers on a
    dedicated copy stream, so a frame's device->host transfer overlaps the
    rendering of the following frames without holding its slot.  ``run``
    yields ``(index, image, contrib, stats)`` numpy views into pinned
    buffers; they stay valid until the next item is requested."""

    def __init__(self, rr: ResidentRenderer, width: int, height: int, *, depth: int = 2,
                 pair_capacity: int | None = None):
        self.pipe = FramePipeline(rr, width, height, depth=depth, pair_capacity=pair_capacity, out_buffers=2)
        self.copy_stream = torch.cuda.Stream(rr.device)
        self.n_host = 2 * depth
        self.host = [(torch.empty((height, width, 3), dtype=torch.float32, pin_memory=True),
                      torch.empty((height, width), dtype=torch.int32, pin_memory=True),
                      torch.empty(_native.STAT_COUNT, dtype=torch.int64, pin_memory=True),
                      torch.cuda.Event()) for _ in range(self.n_host)]

    def run(self, cams, cfg: EngineConfig):
        pending = []  # (index, host buffer)
        nxt = 0
        for i, cam in enumerate(cams):
            if len(pending) == self.n_host:  # the oldest host buffer must be consumed before it is reused
                j, hb = pending.pop(0)
                img, cnt, st, ev = self.host[hb]
                ev.synchronize()
                yield j, img.numpy(), cnt.numpy(), st.numpy()
            k = self.pipe.slot_of_next()
            out = self.pipe.submit(cam, cfg)
            rendered = torch.cuda.Event()
            rendered.record(self.pipe.output_stream(k))
            img, cnt, st, ev = self.host[nxt]
            with torch.cuda.stream(self.copy_stream):
                self.copy_stream.wait_event(rendered)
                st.copy_(out.stats, non_blocking=True)
                img.copy_(out.image, non_blocking=True)
                cnt.copy_(out.contrib, non_blocking=True)
                ev.record(self.copy_stream)
                out.release.record(self.copy_stream)
            pending.append((i, nxt))
            nxt = (nxt + 1) % self.n_host
        for j, hb in pending:
            img, cnt, st, ev = self.host[hb]
            ev.synchronize()
            yield j, img.numpy(), cnt.numpy(), st.numpy()
