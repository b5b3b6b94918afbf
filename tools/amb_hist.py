"""Debug: histogram of the relative transmittance bound D / T at the raster's
T-ambiguous events (library built with -DSEELE_AMB_PROFILE), C3 and C4 frames."""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch
import bench
from paper_2503_05168_b200.render import FrameRenderer
from paper_2503_05168_b200.residency import ResidentRenderer
args = bench.parse()
dev = torch.device("cuda", 0)
scene, poses, table, container, _ = bench.build_workload(args, dev)
rr = ResidentRenderer(container, device=dev)
r = FrameRenderer(dev)
r.reserve(rr.n_max, args.width, args.height, pair_capacity=40 * rr.n_max)
cfg = bench.engine_cfg(args.engine)
for f in (0, 40):
    rr.select_async(poses[f])
    _, h = r.render_checked(rr.scene, poses[f], cfg, ranges=rr.ranges, n_ranges=rr.m + 2, n_max=rr.n_max)
    print(f"{args.width}x{args.height} frame {f}: T-ambiguous D/T histogram <1e-5 {h[11]}, <1e-4 {h[12]}, <1e-3 {h[13]}, "
          f"<1e-2 {h[14]}, >=1e-2 {h[15]} (pairs {h[4]}, blends from stats n/a)")
