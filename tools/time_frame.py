"""Quick device timing of one configuration (development aid, not the bench)."""
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch  # noqa: E402

from paper_2503_05168_b200 import DeviceScene, EngineConfig, FrameRenderer  # noqa: E402
from paper_2503_05168_b200.render import enable_stage_timing, read_stage_timing  # noqa: E402
from paper_2503_05168_b200.synthetic import orbit_pose, synth  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 3_000_000
modes = sys.argv[2].split(",") if len(sys.argv) > 2 else ["ref:fast", "ref:exact", "cr2:fast", "cr2:exact"]
t0 = time.time()
scene = synth(n, 0)
print(f"synth {time.time() - t0:.1f}s", flush=True)
ds = DeviceScene.from_arrays(scene, layout="planes")
r = FrameRenderer()
for mode in modes:
    eng, prec = mode.split(":")
    kw = dict(engine="ref") if eng == "ref" else dict(engine="cr", group_w=int(eng[2]))
    cfg = EngineConfig(precision=prec, **kw)
    out, host = r.render_checked(ds, orbit_pose(0), cfg)
    torch.cuda.synchronize()
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
    K = 10
    ev[0].record()
    for i in range(K):
        r.render(ds, orbit_pose(i), cfg)
    ev[1].record()
    torch.cuda.synchronize()
    ms = ev[0].elapsed_time(ev[1]) / K
    enable_stage_timing(True)
    r.render(ds, orbit_pose(0), cfg)
    st = read_stage_timing()
    enable_stage_timing(False)
    h = r.stats.cpu().numpy()
    print(f"{mode}: {ms:.3f} ms/frame  stages={ {k: round(v, 3) for k, v in st.items()} }  pairs={h[4]} "
          f"binned={h[8]} fixup_warps={h[11]} alpha_redecide={h[12]} t_ambiguous={h[13]} overflow={h[10]}",
          flush=True)
