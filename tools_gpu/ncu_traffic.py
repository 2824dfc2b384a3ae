"""Aggregate an ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum CSV
(recompression kernels of one projector step) into profiles/ncu_trunc_traffic_rNN.json."""
import collections
import csv
import json
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr, data = None, []
for r in rows:
    if "Kernel Name" in r:
        hdr = r
        continue
    if hdr and len(r) == len(hdr):
        data.append(dict(zip(hdr, r)))
unit = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ns": 1e-6, "us": 1e-3, "ms": 1.0, "usecond": 1e-3,
        "nsecond": 1e-6, "msecond": 1.0}
agg = collections.defaultdict(lambda: {"launches": set(), "dram_bytes": 0.0, "ms": 0.0})
for d in data:
    k = d["Kernel Name"].split("(")[0].replace("spg::", "")
    v = float(d["Metric Value"].replace(",", "")) * unit.get(d["Metric Unit"], 1.0)
    agg[k]["launches"].add(d["ID"])
    if d["Metric Name"].startswith("dram__bytes"):
        agg[k]["dram_bytes"] += v
    else:
        agg[k]["ms"] += v
per = {k: {"launches": len(v["launches"]), "dram_bytes": v["dram_bytes"], "ms": v["ms"]} for k, v in agg.items()}
batches = per.get("k_core_any", {}).get("launches", 1)
algo = float(sys.argv[2]) if len(sys.argv) > 2 else None
tot = sum(v["dram_bytes"] for v in per.values())
out = {"what": "DRAM traffic of the recompression class (k_tsqr + k_core_w/k_core_any + k_apply) over one headline "
               "projector step",
       "per_kernel": per, "dram_bytes_total": tot, "recompression_batches_per_step": batches,
       "dram_bytes_per_batch": tot / batches}
if algo:
    out["algorithmic_bytes_per_step"] = algo
    out["algorithmic_bytes_per_batch"] = algo / batches
    out["traffic_over_algorithmic"] = tot / algo
print(json.dumps(out, indent=1))
