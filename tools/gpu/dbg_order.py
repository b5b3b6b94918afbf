"""Debug: where does the GPU (tile, position) order differ from the oracle's at C3 frame 0?"""
import ctypes, sys
import numpy as np, torch
sys.path[:0] = ["/root/repo", "/root/repo/tests"]
from oracle import oracle as O
from paper_2503_05168_b200 import EngineConfig, _native
from paper_2503_05168_b200.clusters import build_cluster_table
from paper_2503_05168_b200.container import container_from_table
from paper_2503_05168_b200.render import FrameRenderer
from paper_2503_05168_b200.residency import ResidentRenderer
from paper_2503_05168_b200.synthetic import orbit, synth
from test_gpu_configs import _device_plan

scene = synth(3_000_000, 0)
poses = orbit(120, 1920, 1080)
table = build_cluster_table(scene, poses, n_clusters=24, neighbors=4, beta=1.0, seed=0, device="cuda")
container = container_from_table(table, scene)
rr = ResidentRenderer(container)
r = FrameRenderer()
r.reserve(rr.n_max, 1920, 1080, pair_capacity=40_000_000)
cfg = EngineConfig(engine="cr", group_w=2)
for f in (0, 2):
    cam = poses[f]
    sel = rr.select(cam)
    rr.select_async(cam)
    out, hs = r.render_checked(rr.scene, cam, cfg, ranges=rr.ranges, n_ranges=rr.m + 2, n_max=rr.n_max)
    ws = rr.assemble(sel)
    pl = O.plan(ws, cam, cfg)
    tile, pos, rg = _device_plan(r, hs)
    plan = r.export_plan(rr.scene, cam, hs)
    gpu_depth_pos = np.zeros(len(ws.positions)); gpu_depth_pos[plan.positions] = plan.depths
    ora_depth_pos = np.zeros(len(ws.positions)); ora_depth_pos[pl["index"]] = pl["depths"]
    want = pl["index"][pl["pair_ref"]]
    bad = np.flatnonzero(pos.astype(np.int64) != want)
    print("frame", f, "mismatches", len(bad))
    dd = gpu_depth_pos[plan.positions] - ora_depth_pos[plan.positions]
    print("  depth differs for", int((dd != 0).sum()), "of", len(plan.positions), "max", float(np.abs(dd).max()))
    for i in bad[:12]:
        a, b = int(pos[i]), int(want[i])
        print(f"  pair {i} tile {tile[i]}: gpu pos {a} (gz {gpu_depth_pos[a]!r} oz {ora_depth_pos[a]!r}) "
              f"oracle pos {b} (gz {gpu_depth_pos[b]!r} oz {ora_depth_pos[b]!r})")
