"""A/B of the banded l0 estimate against a variant selected by env AB_ENV (default SPG_L0_WINDOW:
the windowed kernel; SPG_HAGER_BAND_SEQ: the single-warp Hager solves)."""
import os
import subprocess
import sys

sys.path.insert(0, ".")
if len(sys.argv) > 1 and sys.argv[1] == "child":
    import paper_1608_01164_b200 as S
    from paper_1608_01164_b200.configs import CONFIGS, make_input
    for name in sys.argv[2:]:
        if name.startswith("dim"):
            n, b = map(int, name[3:].split("_"))
            A, nmin, eps = S.dimer_chain(n, 1.0, 0.8, 0.0, 11, b=b, s=0.05 / (2 * b + 1)), 128, 1e-10
        elif name.startswith("rand"):
            n, b = map(int, name[4:].split("_"))
            A, nmin, eps = S.random_banded(n, b, 7), 64, 1e-10
        else:
            c = CONFIGS[name]
            A, nmin, eps = make_input(name), c["nmin"], c["eps"]
        r = S.hqdwh(A, nmin, eps)
        print(name, repr(r.l0), r.iterations, round(r.info["ms_setup"], 2), flush=True)
    sys.exit(0)
names = sys.argv[1:]
ra = subprocess.run([sys.executable, __file__, "child", *names], capture_output=True, text=True)
print(ra.stderr[-2000:])
a = ra.stdout.split("\n")
b = subprocess.run([sys.executable, __file__, "child", *names], capture_output=True, text=True,
                   env={**os.environ, os.environ.get("AB_ENV", "SPG_L0_WINDOW"): "1"}).stdout.split("\n")
for x, y in zip(a, b):
    if not x:
        continue
    nx, lx, ix, tx = x.split()
    ny, ly, iy, ty = y.split()
    print(f"{nx}: l0 new {lx} old {ly} rel {abs(float(lx) - float(ly)) / abs(float(ly)):.2e} iters {ix}/{iy} "
          f"setup ms {tx} / {ty}")
