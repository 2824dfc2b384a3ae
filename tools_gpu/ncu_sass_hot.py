"""Hot SASS ranges of an ncu report: python tools_gpu/ncu_sass_hot.py rep.ncu-rep [top]"""
import csv
import subprocess
import sys

out = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
hdr = rows[1]
ai, si, wi, ei = (hdr.index(x) for x in ("Address", "Source", "Warp Stall Sampling (All Samples)",
                                        "Instructions Executed"))
data = [(r[ai], r[si].strip(), int(r[wi] or 0), int(r[ei] or 0)) for r in rows[2:] if len(r) > ei]
tot_s = sum(d[2] for d in data) or 1
tot_e = sum(d[3] for d in data) or 1
print(f"samples {tot_s}  inst {tot_e}")
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
for i, d in enumerate(data):
    if d[2] / tot_s > 0.01 or d[3] / tot_e > 0.02:
        print(f"{i:5d} {d[2] / tot_s:6.3f} {d[3] / tot_e:6.3f}  {d[1][:90]}")
if "--ranges" in sys.argv:
    W = 40
    for s in range(0, len(data), W):
        e = sum(d[3] for d in data[s:s + W])
        smp = sum(d[2] for d in data[s:s + W])
        if e / tot_e > 0.02 or smp / tot_s > 0.03:
            print(f"[{s}-{s + W}) inst {e / tot_e:.3f} samples {smp / tot_s:.3f}")
