"""write_report (metrics.py:246-266) on the reference's own benchmark rows
(tests/golden/bench.npz): the CSV and its JSON mirror are the reference's
text byte for byte (host logic, no GPU)."""
import csv
import io
import json
import math

import numpy as np

from helpers import GOLDEN
from paper_2503_05168_b200.metrics import REPORT_COLUMNS, write_report


def test_write_report_matches_reference(tmp_path):
    with np.load(GOLDEN / "bench.npz") as z:
        g = {k: z[k] for k in z.files}
    cols = [str(c) for c in g["columns"]]
    rows = []
    for name, vals in zip(g["row_config"], g["rows"]):
        r = {"config": str(name), "lpips": None}
        for c, v in zip(cols, vals):
            r[c] = float(v) if c in ("psnr_db", "ssim", "wall_ms") else int(v)
        rows.append(r)
    path = tmp_path / "report.csv"
    write_report(rows, path)
    assert path.read_text() == str(g["report_csv"])
    assert json.loads(path.with_suffix(".json").read_text()) == json.loads(str(g["report_json"]))
    header = next(csv.reader(io.StringIO(path.read_text())))
    assert header == REPORT_COLUMNS
    assert any(math.isinf(r["psnr_db"]) for r in rows)  # the "inf" spelling is exercised
