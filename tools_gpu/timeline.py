"""Kernel timeline of one projector (GPU box tool): CUPTI activity records through
torch.profiler (graph-launched kernels included), one row per kernel:
name, stream, start_us, end_us (relative to the first kernel).

    python tools_gpu/timeline.py [config] [out.csv.gz]
"""
import gzip
import json
import os
import sys
import tempfile

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402
from torch.profiler import ProfilerActivity, profile  # noqa: E402

import paper_1608_01164_b200 as S  # noqa: E402
from paper_1608_01164_b200.configs import CONFIGS, HEADLINE, make_input  # noqa: E402


def main():
    name = sys.argv[1] if len(sys.argv) > 1 else HEADLINE
    out = sys.argv[2] if len(sys.argv) > 2 else os.path.join(ROOT, "gpurun_out", f"timeline_{name}.csv.gz")
    c = CONFIGS[name]
    A = make_input(c)
    torch.cuda.init()
    for _ in range(2):
        S.hqdwh(A, c["nmin"], c["eps"]).close()
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        r = S.hqdwh(A, c["nmin"], c["eps"])
        torch.cuda.synchronize()
    info = r.info
    r.close()
    tmp = tempfile.mktemp(suffix=".json")
    prof.export_chrome_trace(tmp)
    ev = json.load(open(tmp))["traceEvents"]
    ks = [e for e in ev if e.get("cat") == "kernel"]
    ks.sort(key=lambda e: e["ts"])
    t0 = ks[0]["ts"] if ks else 0
    os.makedirs(os.path.dirname(out), exist_ok=True)
    with gzip.open(out, "wt") as f:
        f.write("name,stream,start_us,end_us\n")
        for e in ks:
            nm = e["name"].split("(")[0].replace(",", ";")
            f.write(f"{nm},{e.get('args', {}).get('stream', -1)},{e['ts'] - t0:.3f},{e['ts'] - t0 + e['dur']:.3f}\n")
    phases = {k: info[k] for k in ("ms_total", "ms_setup", "ms_first", "ms_multiply", "ms_cholesky", "ms_solve",
                                   "ms_solveT", "ms_axpby_sym")}
    print(json.dumps({"config": name, "kernels": len(ks), "span_ms": (ks[-1]["ts"] + ks[-1]["dur"] - t0) / 1e3,
                      "busy_ms": sum(e["dur"] for e in ks) / 1e3, **phases}))


if __name__ == "__main__":
    main()
