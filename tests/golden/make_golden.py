"""Generate the golden parity vectors from the REFERENCE implementation.

Run in the build container (the only place /root/reference exists):

    python tests/golden/make_golden.py            # all cases
    python tests/golden/make_golden.py small      # only the small ones

It imports the reference package read-only (pkg/src/seele) plus its test
builders (pkg/tests/support.py) and writes ``tests/golden/*.npz``.  The
vectors pin the CPU oracle (tests/test_oracle.py) and, through it, the GPU
path.  Per-pixel contributor counts come from the reference's tile-level API
(``rasterize_*(contrib_out=rows)`` -> ``(rows > 0).sum(0)``), the route
SURVEY.md Appendix B validated against ``brute_force_image``.

Nothing here runs at test time; tests only read the committed .npz files.
"""
from __future__ import annotations

import hashlib
import math
import sys
import time
from pathlib import Path

import numpy as np

REF = Path("/root/reference/pkg")
sys.path[:0] = [str(REF / "src"), str(REF / "tests")]
HERE = Path(__file__).resolve().parent
sys.path.insert(0, str(HERE.parent.parent))

from seele import io as sio  # noqa: E402
from seele.compiler import CompileParams, cluster_poses, compile_scene, compute_pose_normalization  # noqa: E402
from seele.model import CameraPose, SceneArrays  # noqa: E402
from seele.rasterize import make_tile_context, rasterize_contribution_aware, rasterize_reference  # noqa: E402
from seele.render import EngineConfig, plan_frame, render_frame  # noqa: E402
from seele.residency import ResidentRenderer, select_clusters  # noqa: E402
from support import make_camera, random_scene, two_sided_scene  # noqa: E402

ENGINES = {
    "ref": dict(engine="ref"),
    "cr1": dict(engine="cr", group_w=1),
    "cr2": dict(engine="cr", group_w=2),
    "cr4": dict(engine="cr", group_w=4),
}
STAT_KEYS = ("alpha_eval_steps", "blend_steps", "leader_eval_steps", "warp_steps", "tile_pairs",
             "culled_near", "dropped_degenerate")


def sha(a: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def contrib_counts(plan, cfg, width, height) -> np.ndarray:
    out = np.zeros(width * height, dtype=np.int32)
    for r in plan.ranges:
        ctx = make_tile_context(plan.grid, r.tile_id)
        tg = plan.tile_gaussians(r.start, r.end)
        rows = np.zeros((r.end - r.start, ctx.centers.shape[0]))
        if cfg.engine == "ref":
            rasterize_reference(ctx, tg, contrib_out=rows)
        else:
            rasterize_contribution_aware(ctx, tg, cfg.group_w, contrib_out=rows)
        v = ctx.valid
        out[ctx.pixel_index[v]] = (rows > 0).sum(axis=0)[v]
    return out.reshape(height, width)


def cam_arrays(cam: CameraPose) -> dict:
    return {
        "cam_position": np.asarray(cam.position),
        "cam_orientation": np.asarray(cam.orientation),
        "cam_fov": np.array([cam.fov_x, cam.fov_y, cam.near_clip]),
        "cam_size": np.array([cam.width, cam.height], dtype=np.int64),
    }


def scene_arrays(scene: SceneArrays) -> dict:
    return {
        "positions": scene.positions, "log_scales": scene.log_scales, "rotations": scene.rotations,
        "opacities": scene.opacities, "sh": scene.sh, "ids": scene.ids,
    }


def plan_arrays(plan) -> dict:
    ranges = np.array([(r.tile_id, r.start, r.end) for r in plan.ranges], dtype=np.int64).reshape(-1, 3)
    return {
        "plan_ids": plan.ids, "plan_means": plan.means, "plan_conics": plan.conics,
        "plan_colors": plan.colors, "plan_opacities": plan.opacities, "plan_depths": plan.depths,
        "pair_tile": plan.sorted_pairs["tile_id"].astype(np.int32),
        "pair_ref": plan.sorted_pairs["gaussian_ref"].astype(np.int32),
        "ranges": ranges,
        "plan_counts": np.array([plan.culled_near, plan.dropped_degenerate], dtype=np.int64),
    }


def engine_outputs(scene, cam, plan, tag, overrides, full_image=True) -> dict:
    cfg = EngineConfig(**overrides)
    res = render_frame(scene, cam, cfg, plan=plan)
    out = {f"{tag}_stats": np.array([getattr(res.stats, k) for k in STAT_KEYS], dtype=np.int64),
           f"{tag}_contrib": contrib_counts(plan, cfg, cam.width, cam.height).astype(np.int16)}
    if full_image is True:
        out[f"{tag}_image"] = res.image
    elif full_image == "f32":
        out[f"{tag}_image_f32"] = res.image.astype(np.float32)
    else:  # summary: per-tile channel means + a fixed pixel sample (keeps 1080p fixtures small)
        h, w = cam.height, cam.width
        ts = 16
        pad = np.zeros((-(-h // ts) * ts, -(-w // ts) * ts, 3))
        pad[:h, :w] = res.image
        out[f"{tag}_tile_sums"] = pad.reshape(pad.shape[0] // ts, ts, pad.shape[1] // ts, ts, 3).sum(axis=(1, 3))
        idx = np.random.default_rng(123).choice(h * w, size=4096, replace=False)
        out[f"{tag}_sample_idx"] = idx
        out[f"{tag}_sample_rgb"] = res.image.reshape(-1, 3)[idx]
    return out


def small_case(name, scene, cam, engines=ENGINES, background=(0.0, 0.0, 0.0), aware=True, sh_degree=3):
    base = dict(background=background, opacity_aware_filter=aware, sh_degree=sh_degree)
    plan = plan_frame(scene, cam, EngineConfig(**base))
    data = {**scene_arrays(scene), **cam_arrays(cam), **plan_arrays(plan),
            "cfg_background": np.asarray(background, dtype=np.float64),
            "cfg_flags": np.array([int(aware), sh_degree], dtype=np.int64)}
    for tag, ov in engines.items():
        data.update(engine_outputs(scene, cam, plan, tag, {**base, **ov}))
    np.savez_compressed(HERE / f"{name}.npz", **data)
    print(f"  {name}: {len(scene)} splats, {len(plan.sorted_pairs)} pairs")


def _pixel_to_world(cam, px, py, z):
    fx, fy = cam.focal()
    cx, cy = cam.principal_point()
    return np.array([(px + 0.5 - cx) * z / fx, (py + 0.5 - cy) * z / fy, z])


def acceptance_scene(i: int, cam) -> SceneArrays:
    """test_acceptance.py:73-112 scene builder (low-opacity wide splat every 10th,
    sub-threshold tail every 7th starting at 3)."""
    rng = np.random.default_rng(1000 + i)
    n = int(rng.integers(8, 62))
    scene = random_scene(rng, n)
    extra = []
    if i % 10 == 0:
        extra.append(SceneArrays(positions=np.array([[0.1, -0.1, 3.0]]),
                                 log_scales=np.full((1, 3), math.log(0.45)),
                                 rotations=np.array([[1.0, 0, 0, 0]]), opacities=np.array([0.008]),
                                 sh=np.zeros((1, 3, 16)), ids=np.zeros(1, dtype=np.int64)))
    if i % 7 == 3:
        z = 8.0
        fx = cam.focal()[0]
        pts = [(17, 17), (33, 21), (9, 41)]
        tails = SceneArrays(positions=np.stack([_pixel_to_world(cam, px, py, z) for px, py in pts]),
                            log_scales=np.full((3, 3), math.log(0.3 * z / fx)),
                            rotations=np.tile(np.array([1.0, 0, 0, 0]), (3, 1)), opacities=np.full(3, 0.5),
                            sh=np.zeros((3, 3, 16)), ids=np.zeros(3, dtype=np.int64))
        tails.sh[:, :, 0] = 0.8
        extra.append(tails)
    if extra:
        scene = SceneArrays.concatenate([scene, *extra])
        scene.ids = np.arange(len(scene), dtype=np.int64)
    return scene


def edge_scene() -> tuple[SceneArrays, CameraPose]:
    """Near-culled, degenerate (scale +250), needle (scale -30) and exact
    tile-edge splats (test_preprocess.py:31-75) mixed into a random scene."""
    cam = make_camera(80, 48)
    rng = np.random.default_rng(77)
    scene = random_scene(rng, 60, sh_degree=2, camera=cam)
    fx, fy = cam.focal()
    extra_pos = [
        [0.0, 0.0, 0.1], [0.0, 0.0, 0.2], [0.3, 0.1, -2.0],          # near-culled (z <= 0.2)
        [0.0, 0.0, 3.0], [0.05, 0.05, 2.0],                          # degenerate / needle
        list(_pixel_to_world(cam, 15.5, 7.5, 2.5)),                  # mean exactly on tile edge x=16
        list(_pixel_to_world(cam, 31.5, 31.5, 4.0)),                 # mean on a tile corner
    ]
    k = len(extra_pos)
    ls = np.full((k, 3), math.log(0.05))
    ls[3] = 250.0
    ls[4] = -30.0
    extra = SceneArrays(positions=np.array(extra_pos), log_scales=ls,
                        rotations=np.tile(np.array([1.0, 0, 0, 0]), (k, 1)),
                        opacities=np.linspace(0.2, 0.9, k), sh=np.zeros((k, 3, 16)),
                        ids=np.zeros(k, dtype=np.int64))
    extra.sh[:, :, 0] = 0.5
    scene = SceneArrays.concatenate([scene, extra])
    scene.ids = np.arange(len(scene), dtype=np.int64) * 3 + 7  # non-trivial global ids
    return scene, cam


def make_small():
    print("small cases")
    cam64 = make_camera()
    for seed in range(4):
        small_case(f"rand64_s{seed}", random_scene(np.random.default_rng(seed), 48), cam64, sh_degree=1)
    for i in (0, 3, 10, 17):
        small_case(f"accept_{i:03d}", acceptance_scene(i, cam64), cam64, sh_degree=3)
    cam_odd = make_camera(100, 70, position=(0.1, -0.2, 0.3), orientation=(0.98, 0.05, 0.1, -0.03))
    small_case("odd100x70", random_scene(np.random.default_rng(11), 400, sh_degree=3, camera=cam_odd), cam_odd,
               background=(0.1, 0.2, 0.3))
    small_case("plain3sigma", random_scene(np.random.default_rng(12), 64, opacity_range=(0.006, 0.9)), cam64,
               engines={"ref": ENGINES["ref"], "cr2": ENGINES["cr2"]}, aware=False, sh_degree=1)
    s, c = edge_scene()
    small_case("edges80x48", s, c, sh_degree=2)
    # degree sweep on one scene
    sc = random_scene(np.random.default_rng(21), 120, sh_degree=3)
    for deg in (0, 1, 2):
        small_case(f"shdeg{deg}", sc, cam64, engines={"ref": ENGINES["ref"]}, sh_degree=deg)


def big_case(name, scene, cam, tags, full_image):
    t0 = time.perf_counter()
    plan = plan_frame(scene, cam, EngineConfig())
    t_plan = time.perf_counter() - t0
    pair_ids = np.stack([plan.sorted_pairs["tile_id"], plan.ids[plan.sorted_pairs["gaussian_ref"]]], axis=1)
    d32 = plan.sorted_pairs["depth"].astype(np.float32).view(np.uint32).astype(np.uint64)
    keys = (plan.sorted_pairs["tile_id"].astype(np.uint64) << np.uint64(32)) | d32
    ranges = np.array([(r.tile_id, r.start, r.end) for r in plan.ranges], dtype=np.int64)
    data = {
        "scene_sha": np.array([sha(scene.positions), sha(scene.log_scales), sha(scene.rotations),
                               sha(scene.opacities), sha(scene.sh)]),
        **cam_arrays(cam),
        "pairs_sha": np.array([sha(pair_ids.astype(np.int64))]),
        "keys_sha": np.array([sha(keys)]),
        "ranges": ranges,
        "ids_sha": np.array([sha(plan.ids.astype(np.int64))]),
        "depths_sha": np.array([sha(plan.depths)]),
        "plan_counts": np.array([plan.culled_near, plan.dropped_degenerate, len(plan.sorted_pairs),
                                 len(plan.ids)], dtype=np.int64),
        "plan_seconds": np.array([t_plan]),
    }
    for tag in tags:
        t1 = time.perf_counter()
        data.update(engine_outputs(scene, cam, plan, tag, ENGINES[tag], full_image=full_image))
        data[f"{tag}_seconds"] = np.array([time.perf_counter() - t1])
    np.savez_compressed(HERE / f"{name}.npz", **data)
    print(f"  {name}: {len(scene)} splats, {len(plan.sorted_pairs)} pairs, plan {t_plan:.1f}s")


def make_config1():
    print("config 1 (100K SH3 @256x256, random_scene seed 0)")
    cam = make_camera(256, 256)
    scene = random_scene(np.random.default_rng(0), 100_000, sh_degree=3, camera=cam)
    big_case("config1", scene, cam, ("ref", "cr2"), full_image="f32")


def make_1080():
    print("synthetic 1080p sample (Appendix C synth(20000), orbit frames 0 and 37)")
    from paper_2503_05168_b200.synthetic import orbit_pose, synth
    mine = synth(20_000, 0)
    scene = SceneArrays(mine.positions, mine.log_scales, mine.rotations, mine.opacities, mine.sh, mine.ids)
    for frame in (0, 37):
        p = orbit_pose(frame)
        cam = CameraPose(position=p.position, orientation=p.orientation, fov_x=p.fov_x, fov_y=p.fov_y,
                         width=p.width, height=p.height, near_clip=p.near_clip)
        big_case(f"synth20k_f{frame}", scene, cam, ("ref", "cr2"), full_image="summary")


def make_clusters():
    print("cluster selection + clustered render (two_sided_scene, orbit centroid table)")
    import tempfile
    scene, poses, _ = two_sided_scene()
    params = CompileParams(num_clusters=2, top_k=32, neighbors=0)
    part = compile_scene(scene, poses, params, seed=0)
    with tempfile.TemporaryDirectory() as tmp:
        sio.write_clustered_scene(part, scene, tmp)
        handle = sio.load_clustered_scene(tmp)
        rr = ResidentRenderer(handle, m=0)
        data = {"centroids": handle.centroids,
                "norm_mean": np.asarray(handle.manifest["position_mean"]),
                "norm_scale": np.array([handle.manifest["position_scale"]]),
                "shared_ids": np.asarray(part.shared_ids), "beta": np.array([handle.manifest["beta"]])}
        for k, ex in enumerate(part.exclusive_ids):
            data[f"exclusive_{k}"] = np.asarray(ex)
        sels, images, contribs = [], [], []
        for i, cam in enumerate(poses):
            sel = rr.select(cam)
            sels.append(sel)
            asm = rr.assemble(sel)
            res = render_frame(asm, cam, EngineConfig(engine="cr", group_w=2))
            images.append(res.image)
            data[f"pose{i}"] = np.concatenate([cam.position, cam.orientation])
            data[f"assembled_ids{i}"] = asm.ids
            data[f"stats{i}"] = np.array([getattr(res.stats, k) for k in STAT_KEYS], dtype=np.int64)
        rr.close()
        data["selections"] = np.array(sels, dtype=np.int64)
        data["images"] = np.stack(images)
        # chunk files exactly as the reference wrote them (small): the device loader must decode them
        for f in sorted(Path(tmp).iterdir()):
            data[f"file:{f.name}"] = np.frombuffer(f.read_bytes(), dtype=np.uint8)
    np.savez_compressed(HERE / "clusters_two_sided.npz", **data)
    print("  two_sided: selections", data["selections"].ravel().tolist())

    from paper_2503_05168_b200.synthetic import orbit_pose
    poses = []
    for i in range(120):
        p = orbit_pose(i)
        poses.append(CameraPose(position=p.position, orientation=p.orientation, fov_x=p.fov_x, fov_y=p.fov_y,
                                width=p.width, height=p.height))
    norm = compute_pose_normalization(poses)
    specs = cluster_poses(poses, 24, beta=1.0, seed=0, normalization=norm)
    cent = np.stack([s.centroid for s in specs])
    members = np.full(120, -1, dtype=np.int64)
    for c, s in enumerate(specs):
        members[s.member_indices] = c
    sel = np.array([select_clusters(p, cent, 4, 1.0, norm) for p in poses], dtype=np.int64)
    # off-trajectory probes (jittered poses) exercise ties/ordering away from centroids
    rng = np.random.default_rng(5)
    probes, probe_sel = [], []
    for i in range(64):
        p = poses[int(rng.integers(120))]
        q = p.orientation + rng.normal(0, 0.2, 4)
        cam = CameraPose(position=p.position + rng.normal(0, 0.8, 3), orientation=q, fov_x=p.fov_x,
                         fov_y=p.fov_y, width=p.width, height=p.height)
        probes.append(np.concatenate([cam.position, cam.orientation]))
        probe_sel.append(select_clusters(cam, cent, 4, 1.0, norm))
    np.savez_compressed(HERE / "clusters_orbit.npz", centroids=cent, members=members, selections=sel,
                        norm_mean=norm[0], norm_scale=np.array([norm[1]]), probes=np.array(probes),
                        probe_selections=np.array(probe_sel, dtype=np.int64))
    print("  orbit: 24 centroids, selection of frame 0:", sel[0].tolist())


if __name__ == "__main__":
    which = set(sys.argv[1:]) or {"small", "config1", "1080", "clusters"}
    if "small" in which:
        make_small()
    if "clusters" in which:
        make_clusters()
    if "config1" in which:
        make_config1()
    if "1080" in which:
        make_1080()
