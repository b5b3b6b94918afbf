"""Debug: warp-step phase counts of the raster (library built with -DSEELE_RASTER_PROFILE)."""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch
import bench
from paper_2503_05168_b200 import _native
from paper_2503_05168_b200.render import FrameRenderer
from paper_2503_05168_b200.residency import ResidentRenderer
args = bench.parse()
dev = torch.device("cuda", 0)
scene, poses, table, container, _ = bench.build_workload(args, dev)
rr = ResidentRenderer(container, device=dev)
r = FrameRenderer(dev)
r.reserve(rr.n_max, args.width, args.height, pair_capacity=16 * rr.n_max)
cfg = bench.engine_cfg(args.engine)
for f in (0, 40, 80):
    rr.select_async(poses[f])
    _, h = r.render_checked(rr.scene, poses[f], cfg, ranges=rr.ranges, n_ranges=rr.m + 2, n_max=rr.n_max)
    print(f"frame {f} {args.engine}: relevant warp-steps={h[11]} no-leader/no-pass={h[12]} no-blend={h[13]} "
          f"ambiguous={h[14]} death-branch={h[15]} pairs={h[4]} alpha_eval={h[0]} blend={h[1]} leader={h[2]}")
