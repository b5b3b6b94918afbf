"""Key ncu --set full metrics of EVERY kernel in a .ncu-rep (one block per launch).

    python tools/ncu_kernels.py report.ncu-rep [name-substring]
"""
import csv
import re
import subprocess
import sys

KEYS = ("Duration", "DRAM Throughput", "Memory Throughput", "Compute (SM) Throughput", "Executed Ipc Active",
        "Issue Slots Busy", "Achieved Occupancy", "Theoretical Occupancy", "Registers Per Thread", "L2 Hit Rate",
        "L1/TEX Hit Rate", "Warp Cycles Per Issued Instruction", "Avg. Active Threads Per Warp",
        "Executed Instructions", "Grid Size", "Block Size", "Shared Memory Configuration Size")
RAW = ("dram__bytes_read.sum", "dram__bytes_write.sum", "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum")


def main(path, filt=""):
    det = subprocess.run(["ncu", "-i", path, "--page", "details", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(det.splitlines()))
    hdr = rows[0]
    kern = {}
    for r in rows[1:]:
        d = dict(zip(hdr, r))
        kid = d.get("ID")
        k = kern.setdefault(kid, {"name": d.get("Kernel Name", ""), "m": {}})
        if d.get("Metric Name") in KEYS and d["Metric Name"] not in k["m"]:
            k["m"][d["Metric Name"]] = f"{d.get('Metric Value')} {d.get('Metric Unit')}"
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rr = list(csv.reader(raw.splitlines()))
    rh = rr[0]
    stall_cols = [i for i, h in enumerate(rh) if re.match(r"smsp__average_warp_latency_issue_stalled_(\w+)\.ratio$", h)
                  or re.match(r"smsp__pcsamp_warps_issue_stalled_(\w+)$", h)]
    for r in rr[2:]:
        d = dict(zip(rh, r))
        kid = d.get("ID")
        if kid not in kern:
            continue
        for m in RAW:
            if m in d:
                kern[kid]["m"][m] = d[m]
        st = []
        for i in stall_cols:
            name = re.sub(r"^smsp__(average_warp_latency_issue_stalled_|pcsamp_warps_issue_stalled_)", "", rh[i])
            name = name.replace(".ratio", "")
            try:
                v = float(r[i].replace(",", ""))
            except ValueError:
                continue
            if "not_issued" in name:
                continue
            st.append((v, name))
        st.sort(reverse=True)
        kern[kid]["stalls"] = ", ".join(f"{n}={v:g}" for v, n in st[:7])
    for kid, k in kern.items():
        if filt and filt not in k["name"]:
            continue
        short = re.search(r"(k_\w+)(<[^>(]*>)?", k["name"])
        print(f"[{kid}] {short.group(0) if short else k['name'][:60]}")
        for key in KEYS + RAW:
            if key in k["m"]:
                print(f"    {key:36s} {k['m'][key]}")
        if k.get("stalls"):
            print(f"    stalls: {k['stalls']}")


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2] if len(sys.argv) > 2 else "")
