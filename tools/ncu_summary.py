"""Print the key ncu --set full metrics of a .ncu-rep (first kernel)."""
import csv
import subprocess
import sys

KEYS = ("Duration", "Elapsed Cycles", "DRAM Throughput", "Memory Throughput", "Compute (SM) Throughput",
        "Executed Ipc Active", "Issue Slots Busy", "Achieved Occupancy", "Theoretical Occupancy",
        "Registers Per Thread", "L2 Hit Rate", "L1/TEX Hit Rate", "Warp Cycles Per Issued Instruction",
        "Avg. Active Threads Per Warp", "Executed Instructions", "Grid Size", "Block Size")
out = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "details", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
hdr = rows[0]
seen = set()
for r in rows[1:]:
    d = dict(zip(hdr, r))
    k = d.get("Metric Name")
    if k in KEYS and k not in seen:
        seen.add(k)
        print(f"  {k:36s} {d.get('Metric Value'):>16s} {d.get('Metric Unit')}")
raw = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rr = list(csv.reader(raw.splitlines()))
d = dict(zip(rr[0], rr[2] if len(rr) > 2 else rr[1]))
tot = 0
for k in ("dram__bytes_read.sum", "dram__bytes_write.sum"):
    v = d.get(k)
    print(f"  {k:36s} {v:>16s}")
stalls = {k.replace("smsp__pcsamp_warps_issue_stalled_", ""): float(v.replace(",", "")) for k, v in d.items()
          if k.startswith("smsp__pcsamp_warps_issue_stalled_") and not k.endswith("not_issued") and v.replace(",", "").replace(".", "").isdigit()}
top = sorted(stalls.items(), key=lambda kv: -kv[1])[:6]
print("  top stalls:", ", ".join(f"{k}={int(v)}" for k, v in top))
