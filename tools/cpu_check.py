import sys, time
sys.path.insert(0, '/root/repo')
import torch, bench
from paper_2503_05168_b200 import _native
from paper_2503_05168_b200.pipeline import FramePipeline
from paper_2503_05168_b200.render import FrameRenderer
from paper_2503_05168_b200.residency import ResidentRenderer
sys.argv=['x']
args = bench.parse()
dev = torch.device("cuda", 0); torch.cuda.set_device(dev)
scene, poses, table, container, _ = bench.build_workload(args, dev)
rr = ResidentRenderer(container, device=dev)
cfg = bench.engine_cfg(args.engine)
cap = 24_000_000
pipe = FramePipeline(rr, args.width, args.height, depth=3, pair_capacity=cap)
main = torch.cuda.current_stream(dev)
for k in range(6): pipe.submit(poses[k], cfg)
pipe.join(main); torch.cuda.synchronize()
for K in (60, 240):
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ev0.record(main); pipe.wait_for(main)
    t0 = time.perf_counter()
    for k in range(K): pipe.submit(poses[k % 120], cfg)
    t1 = time.perf_counter()
    pipe.join(main); ev1.record(main); torch.cuda.synchronize()
    t2 = time.perf_counter()
    print(f"K={K}: cpu enqueue {1e3*(t1-t0)/K:.3f} ms/frame, gpu {ev0.elapsed_time(ev1)/K:.3f} ms/frame, wall {1e3*(t2-t0)/K:.3f}")
