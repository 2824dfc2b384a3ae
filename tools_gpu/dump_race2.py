"""Which nodes of W differ in the first differing Cholesky (SPG_DBG_DUMP=3)."""
import os, subprocess, sys, collections
root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
code = ("import sys; sys.path.insert(0, %r)\n"
        "import paper_1608_01164_b200 as S\n"
        "from paper_1608_01164_b200.configs import CONFIGS, make_input\n"
        "c = CONFIGS[%r]; A = make_input(c)\n"
        "for i in range(%d):\n"
        "    if i %% 3 == 0: S.load_library().spg_release_plan_cache()\n"
        "    sys.stderr.write('RUN %%d\\n' %% i); sys.stderr.flush()\n"
        "    S.hqdwh(A, c['nmin'], c['eps']).close()\n") % (root, sys.argv[1], int(sys.argv[2]))
out = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, env={**os.environ, "SPG_DBG_DUMP": "4"})
runs, cur = [], None
for ln in out.stderr.splitlines():
    if ln.startswith("RUN"):
        cur = []; runs.append(cur)
    elif ln.startswith("NODE") and cur is not None:
        cur.append(ln)
ref = collections.Counter(tuple(r) for r in runs).most_common(1)[0][0]
print("runs", len(runs))
for i, r in enumerate(runs):
    if tuple(r) != ref:
        d = [(a, b) for a, b in zip(r, ref) if a != b]
        print("run", i, "differing nodes", len(d))
        import re
        def key(ln):
            m = re.search(r"level=(\d+) leaf=(\d) begin=(\d+) size=(\d+)", ln)
            return (int(m.group(3)), -int(m.group(1)))
        ks = [int(re.search(r"k=(-?\d+)", a).group(1)) for a, b in d]
        k0 = min(k for k in ks if k >= 0)
        ids = sorted((a for (a, b), k in zip(d, ks) if k == k0), key=key)
        print("   first differing iterate", k0, "nodes", len(ids))
        for a in ids[:10]:
            print("   ", a.rsplit(" ", 1)[0])
