"""Summarise an ncu --set full report (one or more launches) into the fields the bench's
roofline uses: duration, DRAM bytes and throughput, registers, occupancy, issue activity,
L1/L2 throughput and the top warp-stall reasons.  python tools/ncu_summary.py in.ncu-rep out.txt [note]"""
import csv
import io
import subprocess
import sys

src, dst = sys.argv[1], sys.argv[2]
note = sys.argv[3] if len(sys.argv) > 3 else ""
raw = subprocess.run(["ncu", "-i", src, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
hdr = rows[0]
keys = ["Kernel Name", "Grid Size", "Block Size", "gpu__time_duration.sum", "dram__bytes_read.sum",
        "dram__bytes_write.sum", "dram__throughput.avg.pct_of_peak_sustained_elapsed",
        "launch__registers_per_thread", "launch__occupancy_limit_registers",
        "sm__warps_active.avg.pct_of_peak_sustained_active",
        "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "l1tex__throughput.avg.pct_of_peak_sustained_active", "lts__throughput.avg.pct_of_peak_sustained_elapsed"]
with open(dst, "w") as f:
    f.write(f"# ncu --set full --clock-control none summary of {src.split('/')[-1]} {note}\n")
    for r in rows[2:]:
        if len(r) < len(hdr):
            continue
        f.write("---\n")
        for k in keys:
            if k in hdr:
                f.write(f"{k:60s} {r[hdr.index(k)]}\n")
        stalls = []
        for i, h in enumerate(hdr):
            if "smsp__pcsamp_warps_issue_stalled" in h and not h.endswith("_not_issued"):
                try:
                    stalls.append((float(r[i].replace(",", "")), h.replace("smsp__pcsamp_warps_issue_stalled_", "")))
                except ValueError:
                    pass
        tot = sum(v for v, _ in stalls) or 1.0
        f.write("top stalls: " + ", ".join(f"{n} {100 * v / tot:.0f}%" for v, n in sorted(stalls, reverse=True)[:5]) + "\n")
print(open(dst).read())
