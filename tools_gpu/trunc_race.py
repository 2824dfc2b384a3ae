"""Bit-determinism of single tall truncations under concurrent memory traffic"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1608_01164_b200 as S  # noqa: E402

side = torch.cuda.Stream()
a = torch.empty(1 << 27, dtype=torch.float32, device="cuda")
c = torch.empty_like(a)
rng = np.random.default_rng(0)
for p, k in [(8192, 34), (4096, 34), (8192, 70), (2048, 84), (512, 40)]:
    U = rng.standard_normal((p, k)) * np.logspace(0, -20, k)
    V = rng.standard_normal((p, k))
    ref, bad = None, 0
    for i in range(int(sys.argv[1])):
        with torch.cuda.stream(side):
            for _ in range(2):
                c.copy_(a)
        u, v = S.truncate(U, V, 1e-10)
        if ref is None:
            ref = (u, v)
        elif not (u.shape == ref[0].shape and np.array_equal(u, ref[0]) and np.array_equal(v, ref[1])):
            bad += 1
    print(f"p={p} k={k}: rank {ref[0].shape[1]}, {bad} differ", flush=True)
torch.cuda.synchronize()
