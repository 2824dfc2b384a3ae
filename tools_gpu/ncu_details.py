"""Print key metrics of every kernel in an ncu report (ncu -i ... --page details --csv)."""
import csv
import subprocess
import sys

WANT = ["Duration", "Registers Per Thread", "Achieved Occupancy", "Compute (SM) Throughput", "Memory Throughput",
        "DRAM Throughput", "Executed Ipc Active", "Issue Slots Busy", "Grid Size", "Block Size",
        "Warp Cycles Per Issued Instruction", "L2 Hit Rate"]
out = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "details", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
hdr = rows[0]
ki, mi, vi, ui, ii = (hdr.index(x) for x in ("Kernel Name", "Metric Name", "Metric Value", "Metric Unit", "ID"))
cur = None
for r in rows[1:]:
    if r[mi] in WANT:
        key = (r[ii], r[ki].split("(")[0])
        if key != cur:
            print("==", key)
            cur = key
        print(f"    {r[mi]:38s} {r[vi]} {r[ui]}")
