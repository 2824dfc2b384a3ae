"""First intermediate result of the deferred H-Cholesky that differs between runs (SPG_DBG_HASHLOG=1:
checksums of X, m12.V, G, P1, W12, cascade outputs and leaves, queued on the producing streams)."""
import os, subprocess, sys, collections
root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
code = ("import sys; sys.path.insert(0, %r)\n"
        "import paper_1608_01164_b200 as S\n"
        "from paper_1608_01164_b200.configs import CONFIGS, make_input\n"
        "c = CONFIGS['smallgap']; A = make_input(c)\n"
        "for dl in (0.3, 0.1, 3e-2, 1e-2, 3e-3, 1e-3, 1e-4, 1e-6, 1e-8):\n"
        "    r = S.hqdwh(A, c['nmin'], c['eps'], dl)\n"
        "    if r.iterations >= 3: break\n"
        "    r.close()\n"
        "X = r.U; r.close()\n"
        "ctx = S.HodlrContext(c['n'], c['nmin'], c['eps'], 6)\n"
        "ctx.upload(0, X); ctx.op('multiply_upper', 1, 0, 0); ctx.op('scale_shift', 1, alpha=4.175, beta=1.0)\n"
        "sys.stderr.write('BEGIN\\n')\n"
        "for i in range(%d):\n"
        "    sys.stderr.write('RUN\\n'); sys.stderr.flush()\n"
        "    ctx.op('cholesky_deferred', 3, 1); W = ctx.download(3)\n"
        "ctx.close()\n") % (root, int(sys.argv[1]))
out = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, env={**os.environ, "SPG_DBG_HASHLOG": "1"})
runs, cur, on = [], None, False
for ln in out.stderr.splitlines():
    if ln == "BEGIN":
        on = True
    elif ln == "RUN" and on:
        cur = []; runs.append(cur)
    elif ln.startswith("HL ") and cur is not None:
        t = ln.split()
        cur.append((" ".join(t[2:-1]), t[-1]))
print("runs", len(runs), "log entries", [len(r) for r in runs][:3])
if not runs or not runs[0]:
    print(out.stderr[-2000:])
    sys.exit(1)
ref = collections.Counter(tuple(r) for r in runs).most_common(1)[0][0]
nd = 0
for i, r in enumerate(runs):
    if tuple(r) != ref:
        nd += 1
        d = [j for j, (a, b) in enumerate(zip(r, ref)) if a != b]
        print("run", i, "differs in", len(d), "entries; first:", [r[j][0] for j in d[:6]])
print("differing runs", nd)
