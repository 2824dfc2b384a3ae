"""Find inputs whose ranks pass the narrow capacity (56) and run them through the wide fallback."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_1608_01164_b200 as S
for n, b, t2, nmin, eps in [(8192, 4, 0.999, 256, 1e-14), (4096, 4, 0.999, 128, 1e-14), (4096, 8, 0.999, 128, 1e-15), (4096, 16, 0.99, 128, 1e-14), (4096, 8, 0.9995, 128, 1e-14)]:
    A = S.dimer_chain(n, 1.0, t2, 0.0, 1, b=b, s=0.05 / (2 * b + 1)) if b > 1 else S.dimer_chain(n, 1.0, t2, 0.0, 1)
    t0 = time.time()
    try:
        r = S.hqdwh(A, nmin, eps)
        i = r.info
        print(n, b, t2, nmin, eps, "ok iters", r.iterations, "max_rank", i["max_rank"], "kcap", i["kcap"],
              "per-iter", [d.max_rank for d in r.per_iteration], "trace", i["trace"], "ms", round(i["ms_total"], 1),
              "wall", round(time.time() - t0, 2), flush=True)
        r.close()
    except Exception as e:
        print(n, b, t2, nmin, eps, type(e).__name__, str(e)[:200], flush=True)
