"""Concurrent identical projectors with SPG_DBG_DUMP=2: the first (iterate, matrix) whose checksum
is not the same in every projector."""
import os, subprocess, sys, collections
root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
code = ("import sys; sys.path.insert(0, %r)\n"
        "import paper_1608_01164_b200 as S\n"
        "from paper_1608_01164_b200.configs import CONFIGS, make_input\n"
        "c = CONFIGS['smallgap']; A = make_input(c)\n"
        "for i in range(%d):\n"
        "    rs = S.hqdwh_shifts(A, [0.0] * %d, c['nmin'], c['eps'], max_concurrent=%d)\n"
        "    [r.close() for r in rs]\n") % (root, int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[2]))
env = {**os.environ, "SPG_DBG_DUMP": "2"}
out = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, env=env)
seen = collections.OrderedDict()
for ln in out.stderr.splitlines():
    if ln.startswith("DUMP"):
        t = ln.split()
        seen.setdefault((t[1], t[2]), collections.Counter())[t[-1] + t[-2]] += 1
order = ["Z", "W", "Y", "V", "X"]
for (k, name), cnt in sorted(seen.items(), key=lambda kv: (int(kv[0][0].split("=")[1]) if kv[0][0] != "k=-1" else 99, order.index(kv[0][1]))):
    print(k, name, "distinct", len(cnt), dict(cnt.most_common(3)) if len(cnt) > 1 else "")
