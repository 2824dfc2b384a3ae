"""Summarise an ncu --metrics gpu__time_duration.sum CSV launch list per kernel."""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr, data = None, []
for r in rows:
    if "Kernel Name" in r:
        hdr = r
        continue
    if hdr and len(r) == len(hdr):
        data.append(dict(zip(hdr, r)))
agg = collections.defaultdict(lambda: [0, 0.0])
for d in data:
    nm = d["Kernel Name"].split("(")[0]
    v = float(d["Metric Value"].replace(",", ""))
    u = d["Metric Unit"]
    v = v / 1e3 if u in ("ns", "nsecond") else v * 1e3 if u in ("ms", "msecond") else v
    agg[nm][0] += 1
    agg[nm][1] += v
tot = sum(v[1] for v in agg.values())
print(f"# launches: {len(data)}   sum of kernel time: {tot / 1e3:.1f} ms")
print("kernel,launches,total_ms,avg_us,share")
for k, v in sorted(agg.items(), key=lambda x: -x[1][1]):
    print(f"{k},{v[0]},{v[1] / 1e3:.2f},{v[1] / v[0]:.1f},{v[1] / tot:.4f}")
