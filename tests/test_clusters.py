"""Cluster tables and the container format (CPU): pose clustering and the
partition restate compiler.py; the container is byte-compatible with io.py.
Pinned by reference-generated vectors in tests/golden/clusters_*.npz."""
import numpy as np
import pytest

from helpers import STAT_KEYS, load
from oracle import oracle as O
from paper_2503_05168_b200.clusters import ClusterTable, cluster_poses, compute_pose_normalization, partition
from paper_2503_05168_b200.container import encode_records, load_clustered_scene, write_clustered_scene
from paper_2503_05168_b200.errors import CorruptionError, SchemaError
from paper_2503_05168_b200.model import CameraPose
from paper_2503_05168_b200.render import EngineConfig
from paper_2503_05168_b200.synthetic import make_camera, orbit


def test_cluster_poses_reproduces_reference_centroids():
    g = load("clusters_orbit")
    # the golden poses went through the reference CameraPose once more (q / |q| again)
    poses = [CameraPose(p.position, p.orientation, p.fov_x, p.fov_y, p.width, p.height) for p in orbit(120)]
    norm = compute_pose_normalization(poses)
    np.testing.assert_array_equal(norm[0], g["norm_mean"])
    assert norm[1] == float(g["norm_scale"][0])
    specs = cluster_poses(poses, 24, beta=1.0, seed=0, normalization=norm)
    np.testing.assert_array_equal(np.stack([s.centroid for s in specs]), g["centroids"])
    members = np.full(120, -1)
    for c, s in enumerate(specs):
        members[s.member_indices] = c
    np.testing.assert_array_equal(members, g["members"])


def test_partition_rules():
    sets = [np.array([0, 1, 2]), np.array([2, 3]), np.array([5])]
    shared, exclusive, discarded = partition(sets, np.arange(7), share_threshold=2)
    assert shared.tolist() == [2]
    assert [e.tolist() for e in exclusive] == [[0, 1], [3], [5]]
    assert discarded.tolist() == [4, 6]


def _two_sided_dir(tmp_path):
    g = load("clusters_two_sided")
    for key in g:
        if key.startswith("file:"):
            (tmp_path / key[5:]).write_bytes(g[key].tobytes())
    return g


def test_container_loads_reference_files(tmp_path):
    g = _two_sided_dir(tmp_path)
    c = load_clustered_scene(tmp_path)
    assert c.num_clusters == 2 and c.m == 0
    np.testing.assert_array_equal(c.centroids, g["centroids"])
    for i, sel in enumerate(g["selections"]):
        ids = np.concatenate([c.chunk_arrays(-1).ids] + [c.chunk_arrays(int(s)).ids for s in sel])
        np.testing.assert_array_equal(ids, g[f"assembled_ids{i}"])


def test_container_writer_is_byte_identical(tmp_path):
    g = _two_sided_dir(tmp_path)
    c = load_clustered_scene(tmp_path)
    # rebuild the source scene from the decoded chunks (ids index the source)
    n = int(c.ids.max()) + 1
    parts = [c.chunk_arrays(-1)] + [c.chunk_arrays(k) for k in range(c.num_clusters)]
    from paper_2503_05168_b200.model import SceneArrays
    allp = SceneArrays.concatenate(parts)
    order = np.argsort(allp.ids)
    src = allp.take(order)
    assert len(src) <= n
    table = ClusterTable(shared_ids=g["shared_ids"], exclusive_ids=[g["exclusive_0"], g["exclusive_1"]],
                         discarded_ids=np.setdiff1d(np.arange(n), src.ids), centroids=g["centroids"],
                         beta=float(g["beta"][0]), neighbors=0, position_mean=g["norm_mean"],
                         position_scale=float(g["norm_scale"][0]))
    # ids index into the source: build a dense source covering ids 0..n-1
    dense = SceneArrays(np.zeros((n, 3)), np.zeros((n, 3)), np.tile([1.0, 0, 0, 0], (n, 1)), np.full(n, 0.5),
                        np.zeros((n, 3, 16)), np.arange(n))
    for name in ("positions", "log_scales", "rotations", "opacities", "sh"):
        getattr(dense, name)[src.ids] = getattr(src, name)
    out = tmp_path / "rewritten"
    write_clustered_scene(table, dense, out)
    for f in ("shared.bin", "cluster_000.bin", "cluster_001.bin"):
        assert (out / f).read_bytes() == (tmp_path / f).read_bytes(), f


def test_container_corruption_detected(tmp_path):
    _two_sided_dir(tmp_path)
    raw = (tmp_path / "cluster_000.bin").read_bytes()
    (tmp_path / "cluster_000.bin").write_bytes(raw[:-4])
    with pytest.raises(CorruptionError):
        load_clustered_scene(tmp_path)
    with pytest.raises(SchemaError):
        load_clustered_scene(tmp_path / "nowhere")


def test_oracle_on_assembled_working_set_matches_reference(tmp_path):
    g = _two_sided_dir(tmp_path)
    c = load_clustered_scene(tmp_path)
    from paper_2503_05168_b200.model import SceneArrays
    cfg = EngineConfig(engine="cr", group_w=2)
    for i, sel in enumerate(g["selections"]):
        pose = g[f"pose{i}"]
        cam = make_camera(64, 64, position=pose[:3], orientation=pose[3:])
        ws = SceneArrays.concatenate([c.chunk_arrays(-1)] + [c.chunk_arrays(int(s)) for s in sel])
        out = O.render(ws, cam, cfg)
        assert [out["stats"][k] for k in STAT_KEYS] == g[f"stats{i}"].tolist()
        np.testing.assert_allclose(out["image"], g["images"][i], atol=1e-9)


def test_encode_records_layout():
    from paper_2503_05168_b200.synthetic import random_scene
    s = random_scene(np.random.default_rng(0), 5, sh_degree=3)
    raw = encode_records(s)
    assert len(raw) == 5 * 240
    rec = np.frombuffer(raw, dtype="<f4", count=5 * 59).reshape(5, 59)
    np.testing.assert_array_equal(rec[:, 3:6], s.sh[:, :, 0].astype(np.float32))
