#!/usr/bin/env python
"""Benchmark of the B200 Seele render path (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

Workload (BASELINE config 3): the SURVEY.md Appendix C synthetic 3M-Gaussian
scene at 1920x1080 on the 120-frame orbit, with view-dependent cluster tables
(24 pose clusters, M = 4 neighbours; built with the reference's clustering +
partition rules, clusters.py) and the Seele engine (hybrid preprocessing +
contribution-aware raster, w = 2).  A step is one frame per GPU: device
cluster lookup -> preprocess -> depth rank -> binning/sort -> raster, image
left in HBM.  Frames are sharded f = rank + N k (mod 120) with no data-path
collective ("weak": per-GPU work fixed).  ``value`` = frames/s of the whole
job (N K / max-over-ranks device time).  ``e2e`` = the same through the public
API (ResidentRenderer.render_frame, float32 image + contributor counts + stats
downloaded to pinned host memory every frame).

``--impl reference`` times the reference algorithm on the host CPU: the C
fp64 restatement of the reference (oracle/, OpenMP over tiles, all cores) on
the same scene, cluster selection and frames; rank 0 only.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import tempfile
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

import numpy as np  # noqa: E402
import torch  # noqa: E402

METRIC = "frames/sec @1920x1080, 3M Gaussians (1/2/4/8 B200); ms/frame per stage"
N_FRAMES = 120


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=int(os.environ.get("WORLD_SIZE", "1")))
    ap.add_argument("--steps", type=int, default=240)
    ap.add_argument("--warmup", type=int, default=10)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--n", type=int, default=3_000_000)
    ap.add_argument("--width", type=int, default=1920)
    ap.add_argument("--height", type=int, default=1080)
    ap.add_argument("--engine", default="cr2", choices=["ref", "cr1", "cr2", "cr4"])
    ap.add_argument("--flat", action="store_true", help="no cluster tables (whole scene every frame)")
    ap.add_argument("--c1", action="store_true", help="BASELINE config 1 (100K random scene, one 256x256 view)")
    ap.add_argument("--no-opacity-aware", action="store_true", help="plain 3-sigma binning (C5 'HP off')")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--e2e-steps", type=int, default=120, help="frames of the e2e run (120 = the whole orbit)")
    ap.add_argument("--depth", type=int, default=3, help="frames in flight (streams)")
    ap.add_argument("--raster-first", action="store_true",
                    help="raster on a high-priority stream, the plan stages of the frames in flight below it")
    ap.add_argument("--plan-first", action="store_true",
                    help="plan stages on a high-priority stream, the raster of the frames in flight below it")
    ap.add_argument("--partition", type=int, default=0,
                    help="SMs for the plan stages (green-context partition; rasters on the rest); 0 = shared")
    ap.add_argument("--gather", action="store_true",
                    help="also time the run with an NCCL all-gather of every frame (uint8) + stats inside the timed "
                         "region (value_gather)")
    ap.add_argument("--no-exact", action="store_true", help="skip the all-fp64 precision='exact' timing")
    return ap.parse_args()


def engine_cfg(name: str, precision: str = "fast", opacity_aware: bool = True):
    from paper_2503_05168_b200.render import EngineConfig
    if name == "ref":
        return EngineConfig(engine="ref", precision=precision, opacity_aware_filter=opacity_aware)
    return EngineConfig(engine="cr", group_w=int(name[2]), precision=precision, opacity_aware_filter=opacity_aware)


def build_workload(args, device):
    from paper_2503_05168_b200.clusters import ClusterTable, build_cluster_table
    from paper_2503_05168_b200.container import container_from_table
    from paper_2503_05168_b200.synthetic import orbit, synth
    t0 = time.time()
    if args.c1:  # BASELINE config 1: support.random_scene(default_rng(0), 100K, SH3) seen by make_camera(256, 256)
        from paper_2503_05168_b200.synthetic import config1_scene
        scene, cam = config1_scene()
        args.n, args.width, args.height, args.flat = len(scene.positions), cam.width, cam.height, True
        poses = [cam] * N_FRAMES
    else:
        scene = synth(args.n, 0)
        poses = orbit(N_FRAMES, args.width, args.height)
    if args.flat:
        table = ClusterTable(shared_ids=np.arange(args.n), exclusive_ids=[np.zeros(0, np.int64)] * 2,
                             discarded_ids=np.zeros(0, np.int64), centroids=np.zeros((2, 6)), beta=1.0, neighbors=0,
                             position_mean=np.zeros(3), position_scale=1.0)
    else:
        table = build_cluster_table(scene, poses, n_clusters=24, neighbors=4, beta=1.0, seed=0, device=device)
    container = container_from_table(table, scene)
    return scene, poses, table, container, time.time() - t0


def world():
    rank = int(os.environ.get("RANK", "0"))
    size = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, size, local


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    FIELDS = ("uuid,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, device):
        self.uuid = None
        try:
            self.uuid = str(torch.cuda.get_device_properties(device).uuid)
        except Exception:  # pragma: no cover
            pass
        self.file = tempfile.NamedTemporaryFile("w+", suffix=".csv", delete=False)
        self.proc = None

    def start(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                                          "-lms", "20"], stdout=self.file, stderr=subprocess.DEVNULL)
        except FileNotFoundError:
            self.proc = None
        time.sleep(0.3)

    def stop(self) -> dict:
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.1)
        self.proc.terminate()
        self.proc.wait(timeout=5)
        self.file.flush()
        rows = [r.split(", ") for r in Path(self.file.name).read_text().splitlines() if r.strip()]
        mine = [r for r in rows if self.uuid is None or self.uuid.replace("GPU-", "") in r[0]] or rows
        sm = [float(r[1]) for r in mine if r[1].replace(".", "").isdigit()]
        mx = [float(r[2]) for r in mine if r[2].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[k] for r in mine for k in range(4) if len(r) > 5 + k and r[5 + k].strip() == "Active"})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(mine)}


def load_peaks() -> dict:
    p = ROOT / "MEASURED_PEAKS.json"
    return json.loads(p.read_text()) if p.exists() else {}


def profile_traffic() -> dict:
    p = ROOT / "profiles" / "traffic.json"
    return json.loads(p.read_text()) if p.exists() else {}


def cpu_baseline(container, rr, poses, cfg, frame: int = 0) -> dict:
    """One full frame of the reference algorithm (C fp64 oracle) on all host cores."""
    from oracle import oracle as O
    cam = poses[frame]
    sel = rr.select(cam)
    ws = rr.assemble(sel)
    threads = os.cpu_count() or 1
    t0 = time.perf_counter()
    O.render(ws, cam, cfg, threads=threads)
    dt = time.perf_counter() - t0
    return {"value": 1.0 / dt, "unit": "frames/s", "cores": threads, "kind": "port",
            "sample": f"1 full frame (orbit frame {frame}, {len(ws)} splats in the working set), "
                      f"oracle/seele_oracle.c fp64, {dt:.1f} s"}


def run_reference(args):
    rank, size, local = world()
    if rank != 0:
        return
    from oracle import oracle as O
    from paper_2503_05168_b200.residency import ResidentRenderer
    device = torch.device("cuda", local) if torch.cuda.is_available() else None
    scene, poses, table, container, _ = build_workload(args, device)
    cfg = engine_cfg(args.engine, opacity_aware=not args.no_opacity_aware)
    # host-side cluster selection + assembly (residency.py:38-54, 217-220), no GPU involved
    from paper_2503_05168_b200.clusters import pose_feature
    norm = container.normalization

    def select(cam):
        f = pose_feature(cam, container.beta, norm)
        d2 = np.sum((container.centroids - f[None, :]) ** 2, axis=1)
        return [int(i) for i in np.lexsort((np.arange(len(d2)), d2))[:1 + container.m]]

    from paper_2503_05168_b200.model import SceneArrays

    def assemble(sel):
        return SceneArrays.concatenate([container.chunk_arrays(-1)] + [container.chunk_arrays(c) for c in sel])

    threads = os.cpu_count() or 1
    steps, warm = max(1, min(args.steps, 3)), min(args.warmup, 1)
    frames = [(k * 7) % N_FRAMES for k in range(warm + steps)]
    times = []
    for k, f in enumerate(frames):
        cam = poses[f]
        t0 = time.perf_counter()
        O.render(assemble(select(cam)), cam, cfg, threads=threads)
        if k >= warm:
            times.append(time.perf_counter() - t0)
    value = steps / sum(times)
    out = {
        "metric": METRIC, "value": value, "unit": "frames/s", "n_gpus": args.gpus, "steps": steps, "warmup": warm,
        "ms_per_step": 1000.0 * sum(times) / steps, "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
        "dtype": "fp64", "data": "synthetic", "impl": "reference",
        "config": {**workload_config(args, container), "parallelism": f"frame-sharded x{args.gpus}"},
        "cpu_baseline": {"value": value, "unit": "frames/s", "cores": threads, "kind": "port",
                         "sample": f"{steps} full frames of the reference algorithm (C fp64 restatement, "
                                   f"OpenMP over tiles) incl. host cluster selection + assembly"},
        "e2e": {"value": value, "unit": "frames/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(out))


def workload_config(args, container) -> dict:
    return {
        "workload": ("C3: synthetic 3M-Gaussian scene (SURVEY App. C synth(3e6, 0)), 1920x1080, 120-frame orbit, "
                     "view-dependent cluster tables (24 clusters, M=4, beta=1), Seele engine (HP + CR w=2)")
        if not args.flat and args.n == 3_000_000 and not args.no_opacity_aware
        else ("C1: support.random_scene(default_rng(0), 100K, SH3), one 256x256 view" if args.c1 else
              f"synth({args.n}) {args.width}x{args.height} {'flat' if args.flat else 'clustered'}"
              f"{' 3-sigma' if args.no_opacity_aware else ''}"),
        "gaussians": args.n, "width": args.width, "height": args.height, "engine": args.engine,
        "clusters": container.num_clusters, "neighbors": container.m,
        "shared_splats": int(container.chunks[0, 1]),
        "frames": "f = rank + N*k mod 120",
        "l2": "inputs larger than L2 (resident scene 720 MB vs 126 MB L2); no flush",
    }


def run_ours(args):
    rank, size, local = world()
    if not torch.cuda.is_available():
        raise SystemExit("bench.py needs a GPU (the render path has no CPU fallback)")
    device = torch.device("cuda", local)
    torch.cuda.set_device(device)
    if size > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=device)
    from paper_2503_05168_b200 import _native
    from paper_2503_05168_b200.pipeline import FramePipeline
    from paper_2503_05168_b200.render import FrameRenderer, enable_stage_timing, read_stage_timing
    from paper_2503_05168_b200.residency import ResidentRenderer

    scene, poses, table, container, setup_s = build_workload(args, device)
    rr = ResidentRenderer(container, device=device)
    renderer = FrameRenderer(device)
    cfg = engine_cfg(args.engine, opacity_aware=not args.no_opacity_aware)
    lib = _native.load()
    my_frames = [(rank + size * k) % N_FRAMES for k in range(args.warmup + args.steps)]

    # size the tile-pair workspace for every frame this rank renders (untimed)
    renderer.reserve(rr.n_max, args.width, args.height, pair_capacity=16 * rr.n_max)
    need = 0
    for f in sorted(set(my_frames)):
        rr.select_async(poses[f])
        _, host = renderer.render_checked(rr.scene, poses[f], cfg, ranges=rr.ranges, n_ranges=rr.m + 2, n_max=rr.n_max)
        need = max(need, int(host[_native.STAT_TILE_PAIRS]))
    renderer.reserve(rr.n_max, args.width, args.height, pair_capacity=int(need * 1.02) + 1024)

    stream = torch.cuda.current_stream(device)
    cap = renderer.pair_capacity

    def timed_serial():
        for f in my_frames[:args.warmup]:
            rr.render_device(poses[f], cfg, renderer=renderer)
        torch.cuda.synchronize(device)
        if size > 1:
            torch.distributed.barrier()
        ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        ev0.record(stream)
        for f in my_frames[args.warmup:]:
            rr.render_device(poses[f], cfg, renderer=renderer)
        ev1.record(stream)
        torch.cuda.synchronize(device)
        return ev0.elapsed_time(ev1)

    def timed_pipelined(pipe):
        for f in my_frames[:args.warmup]:
            pipe.submit(poses[f], cfg)
        pipe.join(stream)
        torch.cuda.synchronize(device)
        if size > 1:
            torch.distributed.barrier()
        ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        ev0.record(stream)
        pipe.wait_for(stream)
        for f in my_frames[args.warmup:]:
            pipe.submit(poses[f], cfg)
        pipe.join(stream)
        ev1.record(stream)
        torch.cuda.synchronize(device)
        return ev0.elapsed_time(ev1)

    serial_ms = timed_serial()
    pipe = FramePipeline(rr, args.width, args.height, depth=args.depth, pair_capacity=cap,
                         split=args.raster_first or args.plan_first, raster_priority=args.raster_first,
                         partition=args.partition or None)
    clocks = ClockSampler(device) if rank == 0 else None
    if clocks:
        clocks.start()
    launches0 = lib.seele_launch_count()
    ms = timed_pipelined(pipe)
    launches = lib.seele_launch_count() - launches0
    clock_info = clocks.stop() if clocks else None
    last = pipe.slots[0].stats.cpu().numpy()
    overflow = max(int(s.stats[_native.STAT_OVERFLOW].item()) for s in pipe.slots)
    del pipe
    torch.cuda.empty_cache()
    ms_t = torch.tensor([ms, serial_ms], dtype=torch.float64, device=device)
    if size > 1:
        torch.distributed.all_reduce(ms_t, op=torch.distributed.ReduceOp.MAX)
        torch.distributed.barrier()
    max_ms, max_serial_ms = float(ms_t[0].item()), float(ms_t[1].item())
    value = size * args.steps / (max_ms / 1000.0)
    value_serial = size * args.steps / (max_serial_ms / 1000.0)

    # per-stage breakdown + work counters on a sample of this rank's frames (instrumented, untimed above)
    enable_stage_timing(True)
    sample = my_frames[args.warmup:args.warmup + min(8, args.steps)] or my_frames[:1]
    st_acc, ctr = {}, []
    for f in sample:
        rr.render_device(poses[f], cfg, renderer=renderer)
        for k, v in read_stage_timing().items():
            st_acc[k] = st_acc.get(k, 0.0) + v / len(sample)
        ctr.append(renderer.stats.cpu().numpy().copy())
    enable_stage_timing(False)
    ctr = np.mean(np.stack(ctr), axis=0)

    # end to end through the public API: ResidentRenderer.render_trajectory, host image + contributor counts +
    # stats of every frame in pinned memory (device->host copies overlap the next frames' rendering)
    e2e_frames = [(rank + size * k) % N_FRAMES for k in range(max(1, args.e2e_steps))]  # independent of --steps
    for _ in rr.render_trajectory([poses[f] for f in e2e_frames[:4]], cfg, depth=args.depth, pair_capacity=cap):
        pass
    torch.cuda.synchronize(device)
    if size > 1:
        torch.distributed.barrier()
    t0 = time.perf_counter()
    e2e_overflow = 0
    for _, img, cnt, st in rr.render_trajectory([poses[f] for f in e2e_frames], cfg, depth=args.depth,
                                                pair_capacity=cap):
        e2e_overflow |= int(st[_native.STAT_OVERFLOW])
    e2e_s = torch.tensor([time.perf_counter() - t0], dtype=torch.float64, device=device)
    if size > 1:
        torch.distributed.all_reduce(e2e_s, op=torch.distributed.ReduceOp.MAX)
    e2e_value = size * len(e2e_frames) / float(e2e_s.item())
    d2h = args.width * args.height * (3 * 4 + 4) + 8 * _native.STAT_COUNT

    # the all-fp64 raster (precision="exact": same discrete results) on the same frames, serial
    exact_ms = None
    if not args.no_exact:
        cfg_exact = engine_cfg(args.engine, precision="exact", opacity_aware=not args.no_opacity_aware)
        ex_frames = my_frames[args.warmup:args.warmup + min(args.steps, 24)] or my_frames[:1]
        rr.render_device(poses[ex_frames[0]], cfg_exact, renderer=renderer)
        torch.cuda.synchronize(device)
        ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        ev0.record(stream)
        for f in ex_frames:
            rr.render_device(poses[f], cfg_exact, renderer=renderer)
        ev1.record(stream)
        torch.cuda.synchronize(device)
        exact_ms = ev0.elapsed_time(ev1) / len(ex_frames)
        ex_t = torch.tensor([exact_ms], dtype=torch.float64, device=device)
        if size > 1:
            torch.distributed.all_reduce(ex_t, op=torch.distributed.ReduceOp.MAX)
        exact_ms = float(ex_t.item())

    gather_info = None
    if args.gather:
        gather_info = timed_gather(args, rr, poses, cfg, my_frames, cap, device, stream, rank, size)

    if rank == 0:
        peaks = load_peaks()
        hbm = float(peaks.get("hbm_gbs", 6650.0))
        sm_mhz = float(peaks.get("sm_max_mhz", 1965.0))
        fp32_tflops = 148 * 128 * 2 * sm_mhz * 1e6 / 1e12  # nominal FFMA peak at max clock
        # raster work model: FP32-pipe instructions ~ 8 per live (pixel, splat) step + 6 per blend
        live, blends = float(ctr[_native.STAT_LIVE_PIXEL_STEPS]), float(ctr[_native.STAT_PIXEL_BLENDS])
        r_ms = st_acc.get("raster", float("nan"))
        r_tflops = 2.0 * (8.0 * live + 6.0 * blends) / (r_ms * 1e-3) / 1e12
        traffic = profile_traffic()
        n_ws, binned, pairs = float(ctr[_native.STAT_WORKING_SET]), float(ctr[_native.STAT_BINNED]), \
            float(ctr[_native.STAT_TILE_PAIRS])
        # algorithmic bytes: preprocess 240 B in per assembled splat + 52 B out per projected;
        # depth rank 12 B read + 4 B written per binned splat; binning: 8 B emitted per pair
        # (4 B tile key + 4 B splat index) + one read+write of both per stable sort pass
        pre_bytes = n_ws * 240 + float(ctr[_native.STAT_PROJECTED]) * 52
        rank_bytes = binned * 16
        sort_bytes = pairs * (8 + 16)
        stages = {
            k: {"ms": round(v, 4)} for k, v in st_acc.items()
        }
        for k, b in (("preprocess", pre_bytes), ("depth_rank", rank_bytes), ("binning_sort", sort_bytes)):
            if k in stages and stages[k]["ms"] > 0:
                gbs = b / (stages[k]["ms"] * 1e-3) / 1e9
                stages[k].update({"bound": "hbm", "algorithmic_bytes": int(b), "achieved_gbs": round(gbs, 1),
                                  "frac": round(gbs / hbm, 4)})
        stages["raster"].update({"bound": "fp32", "achieved_tflops": round(r_tflops, 2),
                                 "frac": round(r_tflops / fp32_tflops, 4)})
        out = {
            "metric": METRIC, "value": value, "unit": "frames/s", "n_gpus": size, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": max_ms / args.steps, "higher_is_better": True, "scaling": "weak",
            "value_serial": value_serial, "frames_in_flight": args.depth, "frames_per_rank": args.steps,
            "vs_baseline": None, "dtype": "fp64+fp32", "data": "synthetic",
            "config": {**workload_config(args, container), "parallelism": f"frame-sharded x{size}"},
            "roofline": {"kernel": "k_raster_quad (raster stage)", "bound": "fp32",
                         "achieved": round(r_tflops, 3), "peak": round(fp32_tflops, 1), "unit": "TFLOP/s",
                         "frac": round(r_tflops / fp32_tflops, 4),
                         "peak_source": f"nominal 148 SM x 128 FP32 lanes x 2 x {sm_mhz:.0f} MHz (no FP32 peak in "
                                        f"MEASURED_PEAKS.json)",
                         "work_model": "2 x (8 x live pixel-splat steps + 6 x blends) per frame (SURVEY 8d)",
                         "traffic": traffic.get("k_raster_quad")},
            "stages": stages,
            "work": {"working_set": int(n_ws), "binned": int(binned), "tile_pairs": int(pairs),
                     "live_pixel_steps": int(live), "blends": int(blends),
                     "skipped_pixel_steps": int(ctr[_native.STAT_SKIPPED_PIXEL_STEPS]),
                     "alpha_redecide": int(ctr[_native.STAT_ALPHA_REDECIDE]),
                     "t_ambiguous": int(ctr[_native.STAT_T_AMBIGUOUS])},
            "e2e": {"value": e2e_value, "unit": "frames/s", "h2d_bytes_per_step": 96, "d2h_bytes_per_step": d2h,
                    "frames": len(e2e_frames), "overflow": e2e_overflow,
                    "api": f"ResidentRenderer.render_trajectory(cams, cfg, depth={args.depth}): float32 image + "
                           f"contributor counts + stats to pinned host memory per frame"},
            "value_exact_serial": (size / (exact_ms / 1000.0)) if exact_ms else None,
            "exact_note": "precision='exact': all-fp64 raster (reference operation order), identical discrete "
                          "results; frames/s one frame at a time (compare value_serial)",
            "gather": gather_info,
            "gpu_launches": int(launches),
            "clocks": clock_info,
            "overflow": overflow,
            "setup_s": round(setup_s, 1),
        }
        if not args.no_cpu_baseline and size == 1:
            out["cpu_baseline"] = cpu_baseline(container, rr, poses, cfg)
        print(json.dumps(out))
    if size > 1:
        torch.distributed.destroy_process_group()


def timed_gather(args, rr, poses, cfg, my_frames, cap, device, stream, rank, size) -> dict:
    """The pipelined run again, each frame quantised (io.quantize_image rule) into a preallocated uint8 buffer
    and, inside the timed region, ONE NCCL all_gather_into_tensor of every rank's frames + stats (the
    north_star's optional gather over NVLink)."""
    import torch.distributed as dist
    from paper_2503_05168_b200 import _native
    from paper_2503_05168_b200.distributed import quantize
    from paper_2503_05168_b200.pipeline import FramePipeline
    steps = args.steps
    pipe = FramePipeline(rr, args.width, args.height, depth=args.depth, pair_capacity=cap)
    frames_u8 = torch.zeros((steps, args.height, args.width, 3), dtype=torch.uint8, device=device)
    stats = torch.zeros((steps, _native.STAT_COUNT), dtype=torch.int64, device=device)
    all_u8 = torch.empty((size * steps, args.height, args.width, 3), dtype=torch.uint8, device=device)
    all_st = torch.empty((size * steps, _native.STAT_COUNT), dtype=torch.int64, device=device)

    def one_pass(frames, timed):
        for k, f in enumerate(frames):
            slot = pipe.slot_of_next()
            out = pipe.submit(poses[f], cfg)
            st = pipe.output_stream(slot)
            with torch.cuda.stream(st):
                frames_u8[k].copy_(quantize(out.image))
                stats[k].copy_(out.stats)
                out.release.record(st)
        pipe.join(stream)
        if timed and size > 1:
            dist.all_gather_into_tensor(all_u8, frames_u8)
            dist.all_gather_into_tensor(all_st, stats)

    one_pass(my_frames[:args.warmup], False)
    torch.cuda.synchronize(device)
    if size > 1:
        dist.barrier()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ev0.record(stream)
    pipe.wait_for(stream)
    one_pass(my_frames[args.warmup:], True)
    ev1.record(stream)
    torch.cuda.synchronize(device)
    ms = torch.tensor([ev0.elapsed_time(ev1)], dtype=torch.float64, device=device)
    if size > 1:
        dist.all_reduce(ms, op=dist.ReduceOp.MAX)
    ms = float(ms.item())
    frame_bytes = args.height * args.width * 3 + 8 * _native.STAT_COUNT
    del pipe
    return {"value_gather": size * steps / (ms / 1000.0), "ms_per_step": ms / steps,
            "collective": "all_gather_into_tensor (NCCL) of uint8 frames + int64 stats, once per timed run"
            if size > 1 else "none (1 GPU: frames quantised into the gather buffer only)",
            "bytes_per_frame": frame_bytes,
            "nvlink_bytes_per_frame_per_rank": frame_bytes * (size - 1) if size > 1 else 0}


def spawn_ranks(n: int) -> int:
    """``bench.py --gpus N`` outside torchrun: re-launch this script as N ranks (one per GPU) under
    torch.distributed.run on 127.0.0.1; rank 0 prints the JSON line."""
    import socket
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr", "127.0.0.1", "--master-port", str(port), str(Path(__file__).resolve())] + sys.argv[1:]
    return subprocess.call(cmd)


def main():
    args = parse()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        raise SystemExit(spawn_ranks(args.gpus))
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
