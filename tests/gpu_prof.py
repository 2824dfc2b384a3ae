"""Profiled single run: per-kernel-class device times (CUDA events per batch)."""
import json
import sys

sys.path.insert(0, ".")
import paper_1608_01164_b200 as S  # noqa: E402
from paper_1608_01164_b200.configs import CONFIGS, make_input  # noqa: E402

name = sys.argv[1]
c = CONFIGS[name]
A = make_input(name)
S.set_profile(True)
r = S.hqdwh(A, c["nmin"], c["eps"])
I = r.info
keys = ["ms_total", "ms_setup", "ms_first", "ms_multiply", "ms_cholesky", "ms_solve", "ms_solveT", "ms_axpby_sym",
        "launches", "trunc_bytes", "gemm_flops", "trunc_tasks", "prof_ms_trunc", "prof_ms_gemm", "prof_ms_hsolve",
        "prof_ms_leaf", "prof_batches_trunc", "prof_batches_gemm", "prof_batches_hsolve", "prof_batches_leaf"]
print(json.dumps({k: I[k] for k in keys}, indent=1))
print("DMMA peak TFLOP/s", S.measure_dmma_tflops())
