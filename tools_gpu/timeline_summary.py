"""Summarise a profile-mode batch timeline (SPG_PROF_TIMELINE=path, one row per timed batch:
op, class, stream (-1 main), start/end ms from the first batch).
python tools_gpu/timeline_summary.py timeline.csv"""
import collections
import csv
import sys

rows = list(csv.DictReader(open(sys.argv[1])))
for r in rows:
    r["t0"], r["t1"] = float(r["t0"]), float(r["t1"])
span = max(r["t1"] for r in rows) - min(r["t0"] for r in rows)
print(f"batches {len(rows)}, span {span:.1f} ms")


def union(iv):
    iv = sorted(iv)
    tot, cur = 0.0, None
    for a, b in iv:
        if cur is None or a > cur[1]:
            if cur:
                tot += cur[1] - cur[0]
            cur = [a, b]
        else:
            cur[1] = max(cur[1], b)
    return tot + (cur[1] - cur[0] if cur else 0.0)


by_stream = collections.defaultdict(list)
for r in rows:
    by_stream[int(r["stream"])].append((r["t0"], r["t1"]))
for s in sorted(by_stream):
    print(f"stream {s:3d}: batches {len(by_stream[s]):6d} busy {union(by_stream[s]):8.1f} ms")
print(f"any stream busy: {union([(r['t0'], r['t1']) for r in rows]):.1f} ms")

# per op: span on the main stream, busy time per class, and main-stream idle gaps
ops = collections.OrderedDict()
for r in rows:
    ops.setdefault(r["op"], []).append(r)
for op, rs in ops.items():
    main = sorted((r for r in rs if r["stream"] == "-1"), key=lambda r: r["t0"])
    cls = collections.defaultdict(float)
    for r in rs:
        cls[r["cls"]] += r["t1"] - r["t0"]
    gaps = sum(max(0.0, b["t0"] - a["t1"]) for a, b in zip(main, main[1:]))
    busy_main = union([(r["t0"], r["t1"]) for r in main])
    print(f"op {op}: batches {len(rs)} main-busy {busy_main:.1f} ms main-gaps {gaps:.1f} ms; "
          + " ".join(f"{k}={v:.1f}" for k, v in sorted(cls.items())))
# main-stream busy by class
cls = collections.defaultdict(float)
for r in rows:
    if r["stream"] == "-1":
        cls[r["cls"]] += r["t1"] - r["t0"]
print("main stream by class:", " ".join(f"{k}={v:.1f}" for k, v in sorted(cls.items())))
