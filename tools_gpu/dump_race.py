"""Which matrix of which iterate differs first between runs (SPG_DBG_DUMP=2 checksums)."""
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
out = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, env={**os.environ, "SPG_DBG_DUMP": "2"})
runs, cur = [], None
for ln in out.stderr.splitlines():
    if ln.startswith("RUN"):
        cur = []; runs.append(cur)
    elif ln.startswith("DUMP") and cur is not None:
        t = ln.split()
        cur.append((t[1], t[2], t[-1], t[-2]))
ref = collections.Counter(tuple(r) for r in runs).most_common(1)[0][0]
print("runs", len(runs), "entries per run", len(ref))
for i, r in enumerate(runs):
    if tuple(r) != ref:
        first = next((a for a, b in zip(r, ref) if a != b), None)
        print("run", i, "first difference at", first[:2] if first else None, "ranks differ" if first and first[3] != [b for a, b in zip(r, ref) if a != b][0][3] else "")
