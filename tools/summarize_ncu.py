"""Per-kernel summary of an `ncu --set full` report (first launch of each kernel)."""
import csv
import subprocess
import sys

rep, outdir = sys.argv[1], sys.argv[2]
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(raw.splitlines()))
hdr, units = rows[0], rows[1]
seen = set()
KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__inst_executed.avg.per_cycle_active", "smsp__inst_executed.sum", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "launch__registers_per_thread", "launch__grid_size", "launch__block_size", "launch__occupancy_limit_registers",
        "launch__occupancy_limit_shared_mem", "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active", "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active", "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
        "lts__t_bytes.sum", "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum"]
for vals in rows[2:]:
    d = dict(zip(hdr, vals))
    u = dict(zip(hdr, units))
    name = d["Kernel Name"]
    short = name.split("(")[0].split("::")[-1].replace("<", "_").replace(">", "").replace(" ", "")
    if short in seen:
        continue
    seen.add(short)
    st = {k: v for k, v in d.items() if "pcsamp_warps_issue_stalled" in k and not k.endswith("not_issued")}
    tot = sum(float(v.replace(",", "") or 0) for v in st.values()) or 1.0
    with open(f"{outdir}/ncu_{short}.txt", "w") as f:
        f.write(f"# ncu --set full --clock-control none, C3 frame (bench.py --depth 1): {name[:120]}\n")
        for k in KEYS:
            if k in d:
                f.write(f"  {k:62s} {d[k]:>16s} {u.get(k, '')}\n")
        top = sorted(st.items(), key=lambda kv: -float(kv[1].replace(",", "") or 0))[:8]
        f.write("  top stalls: " + ", ".join(
            f"{k.replace('smsp__pcsamp_warps_issue_stalled_', '')}={float(v.replace(',', '')) / tot * 100:.0f}%" for k, v in top) + "\n")
    print("wrote", short)
