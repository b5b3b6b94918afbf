"""Throughput of the C3 trajectory replayed as one CUDA graph (FramePipeline, 3 frames in flight)
versus the same submissions issued eagerly."""
import sys, time
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch
import bench
from paper_2503_05168_b200 import _native
from paper_2503_05168_b200.pipeline import FramePipeline
from paper_2503_05168_b200.residency import ResidentRenderer

sys.argv = sys.argv[:1]
args = bench.parse()
dev = torch.device("cuda", 0)
torch.cuda.set_device(dev)
scene, poses, table, container, _ = bench.build_workload(args, dev)
rr = ResidentRenderer(container, device=dev)
cfg = bench.engine_cfg(args.engine)
pipe = FramePipeline(rr, args.width, args.height, depth=3, pair_capacity=24_000_000)
side = torch.cuda.Stream(dev)
F = 120
with torch.cuda.stream(side):
    for k in range(9):
        pipe.wait_for(side)
        pipe.submit(poses[k], cfg)
        pipe.join(side)
torch.cuda.synchronize()


def eager(K):
    s = torch.cuda.current_stream(dev)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(s)
    pipe.wait_for(s)
    for k in range(K):
        pipe.submit(poses[k % F], cfg)
    pipe.join(s)
    e1.record(s)
    torch.cuda.synchronize()
    return K / (e0.elapsed_time(e1) / 1e3)


print(f"eager: {eager(F * 2):.1f} frames/s", flush=True)
g = torch.cuda.CUDAGraph()
with torch.cuda.graph(g, stream=side):
    cs = torch.cuda.current_stream(dev)
    pipe.wait_for(cs)
    for k in range(F):
        pipe.submit(poses[k], cfg)
    pipe.join(cs)
torch.cuda.synchronize()
for _ in range(2):
    g.replay()
torch.cuda.synchronize()
s = torch.cuda.current_stream(dev)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
R = 3
e0.record(s)
for _ in range(R):
    g.replay()
e1.record(s)
torch.cuda.synchronize()
print(f"graph: {R * F / (e0.elapsed_time(e1) / 1e3):.1f} frames/s", flush=True)
print(f"eager again: {eager(F * 2):.1f} frames/s", flush=True)
