"""Compiled cluster container: manifest.json + raw chunk files (io.py:198-404).

Byte-compatible with the reference's format (io.py:22-25, 266-314): each
chunk is n records of 59 little-endian float32
``x y z | f_dc[3] | f_rest[45] | opacity logit | scale[3] | rot[4]`` followed
by n uint32 ids, ids ascending inside a chunk.

The loader is the ingest fast path: every chunk is decoded with vectorised
numpy straight into the device layout (``DeviceScene`` "planes": float4
planes, shared chunk first, then clusters 0..N-1), validated with the
reference's rules (``CorruptionError`` / ``SchemaError``), and uploaded once.
Nothing streams afterwards: the whole container stays resident in HBM and a
frame's working set is a list of chunk ranges (see residency.py).
"""
from __future__ import annotations

import json
from dataclasses import dataclass
from pathlib import Path

import numpy as np

from .device import N_PLANES, DeviceScene, decode_planes
from .errors import CorruptionError, SchemaError
from .model import SceneArrays, logit

FLOATS_PER_GAUSSIAN = 59
BYTES_PER_GAUSSIAN = FLOATS_PER_GAUSSIAN * 4 + 4


def encode_records(scene: SceneArrays) -> bytes:
    """io.py:198-208 record encoding."""
    n = len(scene)
    rec = np.empty((n, FLOATS_PER_GAUSSIAN), dtype="<f4")
    rec[:, 0:3] = scene.positions
    rec[:, 3:6] = np.asarray(scene.sh)[:, :, 0]
    rec[:, 6:51] = np.asarray(scene.sh)[:, :, 1:].reshape(n, 45)
    rec[:, 51] = logit(scene.opacities)
    rec[:, 52:55] = scene.log_scales
    rec[:, 55:59] = scene.rotations
    return rec.tobytes() + np.asarray(scene.ids).astype("<u4").tobytes()


def records_to_planes(raw: bytes, count: int, label: str) -> tuple[np.ndarray, np.ndarray]:
    """Decode one chunk straight into [15, count, 4] float32 planes + ids."""
    if len(raw) != count * BYTES_PER_GAUSSIAN:
        raise CorruptionError(f"chunk {label}: expected {count * BYTES_PER_GAUSSIAN} bytes, found {len(raw)}")
    rec = np.frombuffer(raw, dtype="<f4", count=count * FLOATS_PER_GAUSSIAN).reshape(count, FLOATS_PER_GAUSSIAN)
    ids = np.frombuffer(raw, dtype="<u4", offset=count * FLOATS_PER_GAUSSIAN * 4, count=count).astype(np.int64)
    if count and (np.linalg.norm(rec[:, 55:59].astype(np.float64), axis=1) < 1e-8).any():
        raise CorruptionError(f"chunk {label}: degenerate rotation record")
    planes = np.zeros((N_PLANES, count, 4), dtype=np.float32)
    planes[0, :, :3] = rec[:, 0:3]
    planes[0, :, 3] = rec[:, 51]
    planes[1, :, :3] = rec[:, 52:55]
    planes[2] = rec[:, 55:59]
    sh = np.empty((count, 3, 16), dtype=np.float32)
    sh[:, :, 0] = rec[:, 3:6]
    sh[:, :, 1:] = rec[:, 6:51].reshape(count, 3, 15)
    for ch in range(3):
        for k in range(4):
            planes[3 + 4 * ch + k] = sh[:, ch, 4 * k:4 * k + 4]
    return planes, ids


def write_clustered_scene(table, source: SceneArrays, directory) -> dict:
    """io.py:266-314: chunk files (ids ascending) + manifest; returns the manifest."""
    directory = Path(directory)
    directory.mkdir(parents=True, exist_ok=True)
    def chunk(ids):  # partition ids index into `source` (io.py:275-276)
        return source.take(np.sort(np.asarray(ids, dtype=np.int64)))

    shared = chunk(table.shared_ids)
    (directory / "shared.bin").write_bytes(encode_records(shared))
    clusters = []
    for c, ids in enumerate(table.exclusive_ids):
        part = chunk(ids)
        name = f"cluster_{c:03d}.bin"
        (directory / name).write_bytes(encode_records(part))
        clusters.append({"centroid": [float(v) for v in table.centroids[c]], "count": len(part), "file": name})
    manifest = {
        "version": 1, "num_clusters": len(table.exclusive_ids), "k": table.top_k, "beta": table.beta,
        "group_w": table.group_w, "M": table.neighbors, "alpha_theta": table.alpha_theta,
        "shared": {"count": len(shared), "file": "shared.bin"}, "clusters": clusters,
        "discarded_count": int(len(table.discarded_ids)), "share_threshold": table.share_threshold,
        "position_mean": [float(v) for v in table.position_mean], "position_scale": float(table.position_scale),
        "sh_degree": table.sh_degree,
    }
    (directory / "manifest.json").write_text(json.dumps(manifest, indent=1, sort_keys=True))
    return manifest


@dataclass
class ClusteredContainer:
    """A loaded container: planes of all chunks (shared first) and the table."""

    manifest: dict
    planes: np.ndarray          # [15, n_total, 4] float32
    ids: np.ndarray             # [n_total] int64
    chunks: np.ndarray          # [(1 + N), 2] int64 (start, count); row 0 = shared
    centroids: np.ndarray       # [N, 6] fp64

    @property
    def num_clusters(self) -> int:
        return int(self.manifest["num_clusters"])

    @property
    def beta(self) -> float:
        return float(self.manifest["beta"])

    @property
    def m(self) -> int:
        return int(self.manifest["M"])

    @property
    def normalization(self) -> tuple[np.ndarray, float]:
        return np.asarray(self.manifest["position_mean"], dtype=np.float64), float(self.manifest["position_scale"])

    @property
    def total_bytes(self) -> int:
        return int(self.chunks[:, 1].sum()) * BYTES_PER_GAUSSIAN

    def chunk_arrays(self, index: int) -> SceneArrays:
        """Decoded fp64 arrays of one chunk (-1 = shared), as io._decode_chunk returns them."""
        start, count = (int(v) for v in self.chunks[index + 1])
        return decode_planes(self.planes[:, start:start + count], self.ids[start:start + count])

    def upload(self, device=None) -> DeviceScene:
        return DeviceScene.from_planes(self.planes, self.ids, device)


def container_from_table(table, source: SceneArrays) -> ClusteredContainer:
    """The container ``write_clustered_scene`` + ``load_clustered_scene`` would
    produce, built in memory (same chunk order, ids ascending per chunk, same
    float32 record values)."""
    from .device import encode_planes
    chunk_ids = [np.sort(np.asarray(table.shared_ids, dtype=np.int64))] + \
        [np.sort(np.asarray(e, dtype=np.int64)) for e in table.exclusive_ids]
    planes, ids, chunks, start = [], [], [], 0
    for idx in chunk_ids:
        part = source.take(idx)
        planes.append(encode_planes(part))
        ids.append(np.asarray(part.ids, dtype=np.int64).astype(np.uint32).astype(np.int64))
        chunks.append((start, len(idx)))
        start += len(idx)
    manifest = {
        "version": 1, "num_clusters": len(table.exclusive_ids), "k": table.top_k, "beta": table.beta,
        "group_w": table.group_w, "M": table.neighbors, "alpha_theta": table.alpha_theta,
        "shared": {"count": int(chunks[0][1]), "file": "shared.bin"},
        "clusters": [{"centroid": [float(v) for v in table.centroids[c]], "count": int(chunks[c + 1][1]),
                      "file": f"cluster_{c:03d}.bin"} for c in range(len(table.exclusive_ids))],
        "discarded_count": int(len(table.discarded_ids)), "share_threshold": table.share_threshold,
        "position_mean": [float(v) for v in table.position_mean], "position_scale": float(table.position_scale),
        "sh_degree": table.sh_degree,
    }
    return ClusteredContainer(manifest=manifest, planes=np.concatenate(planes, axis=1), ids=np.concatenate(ids),
                              chunks=np.asarray(chunks, dtype=np.int64),
                              centroids=np.asarray(table.centroids, dtype=np.float64).reshape(-1, 6))


def load_clustered_scene(directory) -> ClusteredContainer:
    """io.py:387-404 checks, then every chunk decoded into planes."""
    directory = Path(directory)
    path = directory / "manifest.json"
    if not path.exists():
        raise SchemaError(f"{directory}: no manifest.json")
    manifest = json.loads(path.read_text())
    if manifest.get("version") != 1:
        raise SchemaError(f"{path}: unsupported version {manifest.get('version')}")
    clusters = manifest.get("clusters", [])
    if len(clusters) != int(manifest.get("num_clusters", -1)):
        raise CorruptionError(f"{path}: cluster descriptor count {len(clusters)} does not match num_clusters "
                              f"{manifest.get('num_clusters')}")
    for i, entry in enumerate(clusters):
        if len(entry.get("centroid", [])) != 6:
            raise CorruptionError(f"{path}: cluster {i} centroid is not a 6-vector")
    entries = [("shared", manifest["shared"])] + [(str(i), e) for i, e in enumerate(clusters)]
    planes, ids, chunks, start = [], [], [], 0
    for label, entry in entries:
        f = directory / entry["file"]
        if not f.exists():
            raise CorruptionError(f"chunk {label}: missing file {f}")
        count = int(entry["count"])
        p, i = records_to_planes(f.read_bytes(), count, label)
        planes.append(p)
        ids.append(i)
        chunks.append((start, count))
        start += count
    centroids = np.asarray([e["centroid"] for e in clusters], dtype=np.float64).reshape(len(clusters), 6)
    return ClusteredContainer(manifest=manifest, planes=np.concatenate(planes, axis=1), ids=np.concatenate(ids),
                              chunks=np.asarray(chunks, dtype=np.int64), centroids=centroids)
