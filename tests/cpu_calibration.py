"""GPU-box host: times the reference hqdwh (oracle/_ref) on the CPU-baseline sample
(n=8192) and on the full headline (n=65536), same dimer-chain family, 1 core,
default FP environment and FTZ|DAZ.  Writes the measured ratio used
by bench.py to scale the bounded sample to the headline."""
import json
import os
import sys
import time

sys.path.insert(0, ".")
import paper_1608_01164_b200 as S  # noqa: E402
from oracle import ref as R  # noqa: E402
from paper_1608_01164_b200.configs import CONFIGS, HEADLINE  # noqa: E402

RL = R.RefLib()
out = {"cpu": open("/proc/cpuinfo").read().split("model name")[1].split("\n")[0].strip(": "),
       "host_cores": os.cpu_count()}
for tag, n in (("sample", 8192), ("headline", 65536)):
    c = dict(CONFIGS[HEADLINE], n=n)
    A = S.dimer_chain(n, c["t1"], c["t2"], c["eps_dis"], c["seed"])
    for ftz in ([0, 1] if tag == "sample" else [0]):
        RL.L.ref_set_ftz_daz(ftz)
        t0 = time.time()
        res = RL.hqdwh(A.bands, c["nmin"], c["eps"])
        out[f"{tag}_ftz{ftz}_s"] = res["wall_ms"] / 1e3
        out[f"{tag}_iters"] = res["iterations"]
        out[f"{tag}_max_rank"] = RL.L.ref_hodlr_max_rank(res["P"])
        out[f"{tag}_trace"] = RL.L.ref_hodlr_trace(res["P"])
        RL.L.ref_result_free(res["handle"])
        print(tag, ftz, out[f"{tag}_ftz{ftz}_s"], flush=True)
        RL.L.ref_set_ftz_daz(0)
out["ratio"] = out["headline_ftz0_s"] / out["sample_ftz0_s"]
json.dump(out, open("gpurun_out/cpu_calibration_r01.json", "w"), indent=1)
print(json.dumps(out))
