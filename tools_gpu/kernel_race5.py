"""GEMM-only path (spg_result_apply: leaf products, coefficient GEMMs with split-K, accumulations)
repeated on a fixed projector in several threads (one projector per thread): bit-stable?"""
import os, sys, threading, hashlib
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1608_01164_b200 as S
from paper_1608_01164_b200.configs import CONFIGS, make_input
NT, REPS = int(sys.argv[1]), int(sys.argv[2])
c = CONFIGS["smallgap"]
A = make_input(c)
X = np.random.default_rng(0).standard_normal((c["n"], 40))
rs = [S.hqdwh(A, c["nmin"], c["eps"]) for _ in range(NT)]
out = [set() for _ in range(NT)]


def worker(i):
    for _ in range(REPS):
        y = rs[i].apply(X)
        out[i].add(hashlib.sha1(y.tobytes()).hexdigest()[:12])


th = [threading.Thread(target=worker, args=(i,)) for i in range(NT)]
for t in th: t.start()
for t in th: t.join()
print("apply: distinct outputs per thread", [len(o) for o in out])
