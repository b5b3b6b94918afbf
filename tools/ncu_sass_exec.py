"""SASS of one kernel of a .ncu-rep in address order with executed-instruction counts and stall samples
(the loop bodies show up as runs of equal counts).

    python tools/ncu_sass_exec.py report.ncu-rep <kernel-regex> [min_exec]
"""
import csv
import subprocess
import sys

rep, pat = sys.argv[1], sys.argv[2]
lo = int(sys.argv[3]) if len(sys.argv) > 3 else 0
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass", "--kernel-name",
                      f"regex:{pat}"], capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
hdr = next(r for r in rows if r and r[0] == "Address")
idx = {h: i for i, h in enumerate(hdr)}
for r in rows:
    if len(r) < len(hdr) - 1 or not r[0].startswith("0x"):
        continue
    ex = int(r[idx["Instructions Executed"]] or 0)
    if ex < lo:
        continue
    st = r[idx["Warp Stall Sampling (All Samples)"]]
    print(f"{r[0][-5:]} {ex:9d} {st:>6s}  {r[1].strip()}")
