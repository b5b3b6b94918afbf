"""Time the GPU contribution harvest + compile on the C3 scene (3M splats, the 120-pose 1080p orbit,
24 clusters, top-32): the table the reference's dense harvest cannot build at this scale."""
import sys, time
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np
import torch
from paper_2503_05168_b200.clusters import compile_table
from paper_2503_05168_b200.synthetic import orbit_pose, synth

scene = synth(3_000_000, 0)
poses = [orbit_pose(i) for i in range(120)]
torch.cuda.synchronize()
t0 = time.time()
t = compile_table(scene, poses, n_clusters=24, neighbors=4, top_k=32)
torch.cuda.synchronize()
dt = time.time() - t0
sizes = [len(e) for e in t.exclusive_ids]
print(f"compile_table C3: {dt:.2f} s for 120 poses ({1e3 * dt / 120:.1f} ms/pose); shared {len(t.shared_ids)}, "
      f"exclusive {min(sizes)}..{max(sizes)} (sum {sum(sizes)}), discarded {len(t.discarded_ids)}")
