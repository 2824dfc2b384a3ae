"""Bit-determinism of the leaf Cholesky kernel under concurrent memory traffic:
python tools_gpu/leafchol_race.py reps"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1608_01164_b200 as S  # noqa: E402

reps = int(sys.argv[1])
n = 256
rng = np.random.default_rng(0)
B = rng.standard_normal((n, n))
M = B @ B.T / n + np.eye(n)
T = S.PartitionTree(n, n)
H = S.HodlrMatrix(T)
H.dense[0] = M
ctx = S.HodlrContext(n, n, 1e-10, 3)
ctx.upload(0, H)
side = torch.cuda.Stream()
a = torch.empty(1 << 28, dtype=torch.float32, device="cuda")
b = torch.empty_like(a)
ref = None
bad = 0
for i in range(reps):
    with torch.cuda.stream(side):
        for _ in range(4):
            b.copy_(a)       # ~2 GB of traffic in flight while the Cholesky runs
    ctx.op("cholesky", 1, 0)
    W = ctx.download(1).dense[0].copy()
    if ref is None:
        ref = W
    elif not np.array_equal(W, ref):
        bad += 1
        print(f"rep {i}: max diff {np.abs(W - ref).max():.3e}", flush=True)
torch.cuda.synchronize()
print(f"leaf chol n={n}: {reps} reps, {bad} differ; residual {np.abs(ref.T @ ref - M).max():.2e}")
