"""Timing of hqdwh on BASELINE configs (graph mode, no profiling): python tests/gpu_time.py cfg [cfg...]"""
import json
import sys
import time

sys.path.insert(0, ".")
import paper_1608_01164_b200 as S  # noqa: E402
from paper_1608_01164_b200.configs import CONFIGS, make_input  # noqa: E402

for name in sys.argv[1:]:
    c = CONFIGS[name]
    A = make_input(name)
    for rep in range(2):   # the second call replays the cached plan and graphs of the first
        if rep:
            r.close()
        t0 = time.time()
        r = S.hqdwh(A, c["nmin"], c["eps"])
        w = time.time() - t0
    I = r.info
    print(json.dumps({"config": name, "wall_s": round(w, 4), "ms_total": round(I["ms_total"], 2),
                      "iters": I["iterations"], "trace": I["trace"], "max_rank": I["max_rank"],
                      "launches": I["launches"], "graph": I["graph_used"], "graph_nodes": I["graph_nodes"],
                      "ms_setup": round(I["ms_setup"], 1), "ms_first": round(I["ms_first"], 1),
                      "per_iter_ms": [round(d.wall_ms, 1) for d in r.per_iteration]}), flush=True)
    r.close()
