"""Throughput of the C3 trajectory with 1..3 frames in flight (FramePipeline)."""
import sys, time
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch
import bench
from paper_2503_05168_b200 import _native
from paper_2503_05168_b200.pipeline import FramePipeline
from paper_2503_05168_b200.render import FrameRenderer
from paper_2503_05168_b200.residency import ResidentRenderer

args = bench.parse()
dev = torch.device("cuda", 0)
torch.cuda.set_device(dev)
scene, poses, table, container, _ = bench.build_workload(args, dev)
rr = ResidentRenderer(container, device=dev)
cfg = bench.engine_cfg(args.engine)
probe = FrameRenderer(dev)
probe.reserve(rr.n_max, args.width, args.height, pair_capacity=16 * rr.n_max)
need = 0
for f in range(0, 120, 3):
    rr.select_async(poses[f])
    _, host = probe.render_checked(rr.scene, poses[f], cfg, ranges=rr.ranges, n_ranges=rr.m + 2, n_max=rr.n_max)
    need = max(need, int(host[_native.STAT_TILE_PAIRS]))
del probe
cap = int(need * 1.05) + 4096
main = torch.cuda.current_stream(dev)
for depth, split, rp in ((3, False, False), (3, True, True), (2, True, True), (4, True, True), (3, True, False)):
    pipe = FramePipeline(rr, args.width, args.height, depth=depth, pair_capacity=cap, split=split, raster_priority=rp)
    for k in range(6):
        pipe.submit(poses[k], cfg)
    pipe.join(main)
    torch.cuda.synchronize()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ev0.record(main)
    pipe.wait_for(main)
    K = args.steps
    for k in range(K):
        pipe.submit(poses[k % 120], cfg)
    pipe.join(main)
    ev1.record(main)
    torch.cuda.synchronize()
    ms = ev0.elapsed_time(ev1)
    ov = max(int(s.stats[_native.STAT_OVERFLOW].item()) for s in pipe.slots)
    print(f"depth {depth} split {split} raster-first {rp}: {K / (ms / 1e3):.1f} frames/s  ({ms / K:.3f} ms/frame) overflow={ov}", flush=True)
    del pipe
    torch.cuda.empty_cache()
