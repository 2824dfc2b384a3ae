"""Kernel micro-benchmarks: python tests/gpu_micro.py chol N.. | trunc P..  (phase breakdowns)."""
import sys

sys.path.insert(0, ".")
import paper_1608_01164_b200 as S  # noqa: E402

mode = sys.argv[1] if len(sys.argv) > 1 else "chol"
sizes = [int(a) for a in sys.argv[2:]] or [256]
for n in sizes:
    if mode == "chol":
        o = S.micro_kernel(0, n, 20)
        print(f"leaf_chol n={n}: {o[0]:.1f} us/launch; cycles/panel: tasks {o[1]:.0f} wait {o[2]:.0f} reduce {o[3]:.0f} "
              f"diag {o[4]:.0f} solve {o[5]:.0f} gap {o[6]:.0f}; status {int(o[7])}", flush=True)
    elif mode == "trunc":
        for g, which in ((1, 1), (2, 6)):
            o = S.micro_kernel(which, n, 20)
            print(f"trunc p={n} groups={g}: {o[0]:.1f} us/trunc (tsqr {o[1]:.1f} core {o[2]:.1f} apply {o[3]:.1f}); "
                  f"core cycles C {o[4]:.0f} QRCP {o[5]:.0f} spill {o[6]:.0f} Jacobi {o[7]:.0f} fin {o[8]:.0f}; "
                  f"sweeps {o[9]:.0f} r' {o[10]:.0f} k {o[11]:.0f} rank {o[12]:.0f}", flush=True)
if mode == "trunck":   # python tests/gpu_micro.py trunck P K..
    p = sizes[0]
    for k in sizes[1:]:
        o = S.micro_kernel(100 + k, p, 20)
        print(f"trunc p={p} k={k}: {o[0]:.1f} us/trunc (tsqr {o[1]:.1f} core {o[2]:.1f} apply {o[3]:.1f}); "
              f"core cycles C {o[4]:.0f} QRCP {o[5]:.0f} spill {o[6]:.0f} Jacobi {o[7]:.0f} fin {o[8]:.0f}; "
              f"sweeps {o[9]:.0f} r' {o[10]:.0f} k {o[11]:.0f} rank {o[12]:.0f}", flush=True)
if mode == "lat":
    o = S.micro_kernel(4, 0, 0)
    names = ["dfma", "dmul", "shfl", "lds", "rcp.approx", "rsqrt.approx", "rcp_nr", "bar384", "syncwarp", "dmma",
             "div", "sqrt", "syncwarp_int", "bar.warp.sync", "sts-syncwarp-lds"]
    print("latency cycles:", ", ".join(f"{n}={o[i]:.1f}" for i, n in enumerate(names)))
