"""Full SASS listings of the hot kernels of the built library (cuobjdump -sass),
one file per kernel under profiles/<round>/sass/, encodings stripped:

    python tools/sass_listings.py profiles/r02/sass
"""
import re
import subprocess
import sys
from pathlib import Path

LIB = Path(__file__).resolve().parents[1] / "paper_2503_05168_b200" / "libseele_b200.so"
HOT = ["k_preprocessILi1E", "k_select", "k_bucket_scan", "k_bucket_scatter", "k_bucket_sort", "k_bin_count",
       "k_bin_scan", "k_bin_splitILi8E", "k_bin_head", "k_bin_expand", "k_raster_quadILi0E", "k_raster_quadILi2E"]

out = Path(sys.argv[1])
out.mkdir(parents=True, exist_ok=True)
text = subprocess.run(["cuobjdump", "-sass", str(LIB)], capture_output=True, text=True, check=True).stdout
funcs = re.split(r"\n\s*Function : ", text)
for f in funcs[1:]:
    name = f.split("\n", 1)[0].strip()
    tag = next((h for h in HOT if h in name), None)
    if tag is None:
        continue
    lines = []
    for ln in f.split("\n"):
        m = re.match(r"\s*/\*([0-9a-f]{4,})\*/\s*(.*?);?\s*/\*.*\*/\s*$", ln)
        if m:
            lines.append(f"{m.group(1)}  {m.group(2).rstrip(' ;')}")
        elif ln.strip().startswith(".") or "Function" in ln:
            lines.append(ln.strip())
    short = re.sub(r"ILi(\d+)E", r"_\1", tag)
    (out / f"{short}.sass").write_text(f"// {name}\n// {len(lines)} lines, cuobjdump -sass {LIB.name}\n" + "\n".join(lines) + "\n")
    print(short, len(lines))
