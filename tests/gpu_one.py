"""One hqdwh projector on a BASELINE config (production graph mode): python tests/gpu_one.py cfg"""
import json
import sys

sys.path.insert(0, ".")
import paper_1608_01164_b200 as S  # noqa: E402
from paper_1608_01164_b200.configs import CONFIGS, make_input  # noqa: E402

name = sys.argv[1]
c = CONFIGS[name]
r = S.hqdwh(make_input(name), c["nmin"], c["eps"])
print(json.dumps({"config": name, "ms_total": round(r.info["ms_total"], 2), "iters": r.info["iterations"],
                  "launches": r.info["launches"]}))
