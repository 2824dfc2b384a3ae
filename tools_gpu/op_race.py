"""Bit-determinism of each HODLR operation (component API, plan mode) under concurrent memory
traffic: python tools_gpu/op_race.py reps"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1608_01164_b200 as S  # noqa: E402

reps = int(sys.argv[1])
n, nmin, b = 4096, 256, 24
rng = np.random.default_rng(3)
bands = [rng.uniform(-1, 1, n - d) * (0.5 ** d if d else 1.0) for d in range(b + 1)]
bands[0] += 2 * b
A = S.BandedSymmetric(n, b, bands)
ctx = S.HodlrContext(n, nmin, 1e-10, 6)
ctx.from_banded(0, A)
ctx.op("scale_shift", 0, alpha=1.0 / (4 * b), beta=0.0)
side = torch.cuda.Stream()
a = torch.empty(1 << 27, dtype=torch.float32, device="cuda")
c = torch.empty_like(a)


def hog():
    with torch.cuda.stream(side):
        for _ in range(3):
            c.copy_(a)


def run(name, fn, slot):
    ref, bad = None, 0
    for i in range(reps):
        hog()
        fn()
        rk, d = ctx.download(slot).to_flat()
        cur = (rk.copy(), d.copy())
        if ref is None:
            ref = cur
        elif not (np.array_equal(cur[0], ref[0]) and np.array_equal(cur[1], ref[1])):
            bad += 1
    print(f"{name}: {bad}/{reps - 1} differ (max rank {ctx.download(slot).diagnostics()[0]})", flush=True)


run("multiply", lambda: ctx.op("multiply", 1, 0, 0), 1)
run("multiply_upper", lambda: ctx.op("multiply_upper", 2, 0, 0), 2)
ctx.op("multiply", 1, 0, 0)
ctx.op("scale_shift", 1, alpha=3.0, beta=1.0)
run("cholesky(ref order)", lambda: ctx.op("cholesky", 3, 1), 3)
run("cholesky(deferred)", lambda: ctx.op("cholesky_deferred", 4, 1), 4)
ctx.op("cholesky", 3, 1)
run("solve_upper_right", lambda: ctx.op("solve_upper_right", 5, 0, 3), 5)
run("solve_upperT_right", lambda: ctx.op("solve_upperT_right", 2, 5, 3), 2)
run("axpby", lambda: ctx.op("axpby", 2, 0, 5, 0.5, 0.25), 2)
torch.cuda.synchronize()
