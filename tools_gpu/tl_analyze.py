"""Analyse a CUPTI kernel timeline (tools_gpu/timeline.py).  Graph replays run on the
graph's own streams, so the analysis is by time: how long exactly c kernels were running,
and which kernel names own the time when one kernel runs alone (the latency chain).
    python tools_gpu/tl_analyze.py timeline.csv.gz [t0_ms t1_ms]"""
import collections, csv, gzip, sys
rows = list(csv.DictReader(gzip.open(sys.argv[1], "rt")))
for r in rows:
    r["a"], r["b"] = float(r["start_us"]) / 1e3, float(r["end_us"]) / 1e3
t0 = float(sys.argv[2]) if len(sys.argv) > 2 else 0.0
t1 = float(sys.argv[3]) if len(sys.argv) > 3 else max(r["b"] for r in rows)
rows = [r for r in rows if r["b"] > t0 and r["a"] < t1]
print("window %.1f..%.1f ms, kernels %d" % (t0, t1, len(rows)))
ev = []
for i, r in enumerate(rows):
    ev.append((max(r["a"], t0), 1, i)); ev.append((min(r["b"], t1), -1, i))
ev.sort()
active = set(); last = t0
conc = collections.defaultdict(float); alone = collections.defaultdict(float); pair = collections.defaultdict(float)
for t, d, i in ev:
    dt = t - last
    if dt > 0:
        c = len(active); conc[min(c, 8)] += dt
        if c == 1: alone[rows[next(iter(active))]["name"]] += dt
        elif c == 2: pair[tuple(sorted(rows[j]["name"] for j in active))] += dt
    last = t
    if d > 0: active.add(i)
    else: active.discard(i)
print("time with c kernels running:", " ".join("%d:%.1f" % (c, conc[c]) for c in sorted(conc)))
tot = collections.defaultdict(lambda: [0.0, 0])
for r in rows:
    tot[r["name"]][0] += r["b"] - r["a"]; tot[r["name"]][1] += 1
print("kernel: launches, summed ms, avg us, ms running alone")
for k, e in sorted(tot.items(), key=lambda kv: -alone[kv[0]]):
    print("  %-44s n %6d sum %8.2f avg %7.1f alone %8.2f" % (k[:44], e[1], e[0], 1e3 * e[0] / e[1], alone[k]))
print("top pairs:")
for k, v in sorted(pair.items(), key=lambda kv: -kv[1])[:8]:
    print("  %.2f ms  %s" % (v, " + ".join(x[:30] for x in k)))
