"""Golden vectors for the PLY ingest (io.py:36-152) from the REFERENCE
implementation (build container only):

    python tests/golden/make_ply.py

Builds small binary PLY files (SH degrees 0-3, extra normal properties, a
double-typed property, shuffled property order) and error cases, runs the
reference's load_ply on each, and stores the file bytes with the decoded
arrays (or the exception class).  Writes tests/golden/ply.npz.
"""
import sys
import tempfile
from pathlib import Path

import numpy as np

REF = Path("/root/reference/pkg")
sys.path[:0] = [str(REF / "src"), str(REF / "tests")]
HERE = Path(__file__).resolve().parent

from seele.io import load_ply  # noqa: E402


def ply_bytes(props, cols, n, fmt="binary_little_endian"):
    head = ["ply", f"format {fmt} 1.0", f"element vertex {n}"] + [f"property {k} {p}" for k, p in props]
    head.append("end_header")
    dtype = np.dtype([(p, {"float": "<f4", "double": "<f8", "uchar": "u1"}[k]) for k, p in props])
    rec = np.zeros(n, dtype=dtype)
    for p in cols:
        if p in rec.dtype.names:
            rec[p] = cols[p]
    return ("\n".join(head) + "\n").encode() + rec.tobytes()


def gauss_cols(rng, n, rest, normals=True):
    cols = {"x": rng.normal(size=n), "y": rng.normal(size=n), "z": rng.uniform(2, 6, n),
            "opacity": rng.normal(0, 3, n), "scale_0": rng.normal(-3, 1, n), "scale_1": rng.normal(-3, 1, n),
            "scale_2": rng.normal(-3, 1, n)}
    for k in range(4):
        cols[f"rot_{k}"] = rng.normal(size=n)
    for c in range(3):
        cols[f"f_dc_{c}"] = rng.normal(0, 0.5, n)
    for i in range(rest):
        cols[f"f_rest_{i}"] = rng.normal(0, 0.1, n)
    if normals:
        for c in "xyz":
            cols["n" + c] = np.zeros(n)
    return cols


rng = np.random.default_rng(3)
cases = {}
for rest in (0, 9, 24, 45):
    cols = gauss_cols(rng, 50, rest)
    names = ["x", "y", "z", "nx", "ny", "nz"] + [f"f_dc_{c}" for c in range(3)] + [f"f_rest_{i}" for i in range(rest)] \
        + ["opacity", "scale_0", "scale_1", "scale_2", "rot_0", "rot_1", "rot_2", "rot_3"]
    cases[f"deg{rest}"] = ply_bytes([("float", p) for p in names], cols, 50)
cols = gauss_cols(rng, 30, 9, normals=False)
props = [("double" if p == "opacity" else "float", p) for p in
         ["rot_0", "rot_1", "rot_2", "rot_3", "opacity"] + [f"f_rest_{i}" for i in range(9)] +
         ["x", "y", "z", "f_dc_0", "f_dc_1", "f_dc_2", "scale_0", "scale_1", "scale_2"]] + [("uchar", "flag")]
cols["flag"] = np.ones(30)
cases["mixed"] = ply_bytes(props, cols, 30)
# error cases
base = [("float", p) for p in ["x", "y", "z", "f_dc_0", "f_dc_1", "f_dc_2", "opacity", "scale_0", "scale_1", "scale_2",
                               "rot_0", "rot_1", "rot_2", "rot_3"]]
c = gauss_cols(rng, 10, 0, normals=False)
cases["err_ascii"] = ply_bytes(base, c, 10, fmt="ascii")
cases["err_missing"] = ply_bytes(base[:-1], c, 10)
cases["err_rest"] = ply_bytes(base + [("float", "f_rest_0")], dict(c, f_rest_0=np.zeros(10)), 10)
cases["err_trunc"] = ply_bytes(base, c, 10)[:-20]
c2 = dict(c)
c2["x"] = c["x"].copy()
c2["x"][6] = np.nan
c2["rot_0"] = c["rot_0"].copy()
c2["rot_1"] = c["rot_1"].copy()
c2["rot_2"] = c["rot_2"].copy()
c2["rot_3"] = c["rot_3"].copy()
for k in range(4):
    c2[f"rot_{k}"][4] = 0.0
cases["err_quat_first"] = ply_bytes(base, c2, 10)  # quaternion at 4 before the NaN at 6
c3 = dict(c)
c3["x"] = c["x"].copy()
c3["x"][2] = np.inf
cases["err_nonfinite"] = ply_bytes(base, c3, 10)
cases["err_empty"] = ply_bytes(base, {}, 0)

out = {}
with tempfile.TemporaryDirectory() as d:
    for name, raw in cases.items():
        f = Path(d) / f"{name}.ply"
        f.write_bytes(raw)
        out[f"{name}_bytes"] = np.frombuffer(raw, dtype=np.uint8)
        try:
            sf = load_ply(f)
            a = sf.arrays()
            out[f"{name}_positions"], out[f"{name}_log_scales"] = a.positions, a.log_scales
            out[f"{name}_rotations"], out[f"{name}_opacities"], out[f"{name}_sh"] = a.rotations, a.opacities, a.sh
            out[f"{name}_degree"] = np.array(sf.sh_degree)
            print(name, "ok", len(a.positions), sf.sh_degree)
        except Exception as e:  # noqa: BLE001
            out[f"{name}_error"] = np.array(type(e).__name__)
            print(name, type(e).__name__, e)
out["names"] = np.array(list(cases))
np.savez_compressed(HERE / "ply.npz", **out)
