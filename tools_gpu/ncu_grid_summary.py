"""Summarise an ncu CSV (metrics gpu__time_duration.sum, launch__grid_size) per (kernel, grid size)."""
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
per = collections.defaultdict(dict)
for d in data:
    per[d["ID"]]["name"] = d["Kernel Name"].split("(")[0]
    v = float(d["Metric Value"].replace(",", ""))
    if d["Metric Name"] == "gpu__time_duration.sum":
        u = d["Metric Unit"]
        per[d["ID"]]["us"] = v / 1e3 if u in ("ns", "nsecond") else v * 1e3 if u in ("ms", "msecond") else v
    else:
        per[d["ID"]]["grid"] = int(v)
agg = collections.defaultdict(lambda: [0, 0.0])
byname = collections.defaultdict(lambda: [0, 0.0])
for k in per.values():
    g = k.get("grid", 0)
    b = 1 << max(0, (g - 1).bit_length()) if g else 0
    agg[(k["name"], b)][0] += 1
    agg[(k["name"], b)][1] += k.get("us", 0.0)
    byname[k["name"]][0] += 1
    byname[k["name"]][1] += k.get("us", 0.0)
tot = sum(v[1] for v in byname.values())
print(f"# launches: {len(per)}   sum of kernel time: {tot / 1e3:.1f} ms")
print("kernel,launches,total_ms,avg_us,share")
for k, v in sorted(byname.items(), key=lambda x: -x[1][1]):
    print(f"{k},{v[0]},{v[1] / 1e3:.2f},{v[1] / v[0]:.1f},{v[1] / tot:.4f}")
print("\nkernel,grid<=,launches,total_ms,avg_us")
for k, v in sorted(agg.items(), key=lambda x: -x[1][1])[:40]:
    print(f"{k[0]},{k[1]},{v[0]},{v[1] / 1e3:.2f},{v[1] / v[0]:.1f}")
