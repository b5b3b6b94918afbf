"""Runs bench.py over the BASELINE configs (C1-C5) and writes profiles/r02/configs.json."""
import json
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
RUNS = {
    "C1 100K SH3 256x256 (single view)": ["--c1"],
    "C2 1M 1080p orbit (flat)": ["--n", "1000000", "--flat"],
    "C3 3M 1080p clustered (HP + CR w=2)": [],
    "C4 6M 3840x2160 (flat)": ["--n", "6000000", "--width", "3840", "--height", "2160", "--flat", "--steps", "30",
                               "--depth", "2"],
    "C5 HP off + ref (baseline 3DGS raster)": ["--flat", "--no-opacity-aware", "--engine", "ref"],
    "C5 HP off + CR w=2": ["--flat", "--no-opacity-aware", "--engine", "cr2"],
    "C5 HP on + ref": ["--engine", "ref"],
    "C5 HP on + CR w=2 (Seele)": ["--engine", "cr2"],
}
out = {}
for name, extra in RUNS.items():
    cmd = [sys.executable, str(ROOT / "bench.py"), "--steps", "60", "--warmup", "3", "--no-cpu-baseline",
           "--e2e-steps", "20"] + extra
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=900)
    try:
        d = json.loads(r.stdout.strip().splitlines()[-1])
    except Exception:
        out[name] = {"error": r.stderr[-500:]}
        continue
    out[name] = {"frames_per_s": round(d["value"], 1), "frames_per_s_serial": round(d["value_serial"], 1),
                 "e2e_frames_per_s": round(d["e2e"]["value"], 1), "stages_ms": {k: v["ms"] for k, v in d["stages"].items()},
                 "work": d["work"], "config": d["config"]["workload"]}
    print(name, out[name]["frames_per_s"], out[name]["frames_per_s_serial"], flush=True)
(ROOT / "gpurun_out").mkdir(exist_ok=True)
(ROOT / "gpurun_out" / "configs.json").write_text(json.dumps(out, indent=1))
