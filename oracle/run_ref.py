"""TEST INFRASTRUCTURE: run the reference hqdwh (oracle/_ref) on one BASELINE config.

    python -m oracle.run_ref <config> --out DIR [--patched] [--ftz] [--save-p] [--probes M --probe-seed S]

* input: the config's dimer chain generated on the oracle side (ref_make_dimer_chain),
  so this process never loads the product library;
* the call is the reference's public ``specproj::hqdwh`` (qdwh.hpp:196-241), timed with
  steady_clock around the call exactly like tools/specproj.cpp:71-80;
* ``--patched`` uses the memory-patched build (oracle/patch_memory.py; bitwise equal,
  frees assemble_q's auxiliary columns), ``--ftz`` sets FTZ|DAZ in MXCSR first;
* writes DIR/<config>.json (iterations, alpha, l0, per-iteration c / max rank, trace,
  per-level max ranks, wall time), and optionally DIR/<config>_P.npz (the flat
  preorder export of P: ranks, data) and DIR/<config>_probe.npz (P_ref @ Omega with
  Omega = default_rng(S).standard_normal((n, M))).

Used by tests/parity_big.py (GPU box) and bench.py's reference arm.
"""
import argparse
import json
import os
import resource
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from oracle import ref as R  # noqa: E402
from paper_1608_01164_b200.configs import CONFIGS  # noqa: E402  (config table only; no library load)


def level_max_ranks(ranks, n, n_min, RL):
    """max off-diagonal rank per tree depth (1 = root blocks) from the flat preorder ranks"""
    nn = len(ranks) // 2
    begin = np.zeros(nn, dtype=np.int32); size = np.zeros(nn, dtype=np.int32)
    left = np.zeros(nn, dtype=np.int32); right = np.zeros(nn, dtype=np.int32)
    dep = np.zeros(1, dtype=np.int32)
    RL.L.ref_tree(n, n_min, R._i(begin), R._i(size), R._i(left), R._i(right), R._i(dep))
    depth = np.zeros(nn, dtype=np.int32)
    out = {}
    for i in range(nn):           # preorder: parents before children
        if left[i] >= 0:
            depth[left[i]] = depth[right[i]] = depth[i] + 1
            d = int(depth[i]) + 1
            out[d] = max(out.get(d, 0), int(ranks[2 * i]), int(ranks[2 * i + 1]))
    return [out[d] for d in sorted(out)]


def run(name, outdir, patched=False, ftz=False, save_p=False, probes=0, probe_seed=123, seed_offset=0):
    c = CONFIGS[name]
    RL = R.RefLib(R.REF_PATCHED_SO if patched else R.REF_SO)
    bands = RL.config_bands(c, seed_offset)
    if ftz:
        RL.L.ref_set_ftz_daz(1)
    t0 = time.time()
    ref = RL.hqdwh(bands, c["nmin"], c["eps"])
    wall_s = time.time() - t0
    h = ref["P"]
    n = c["n"]
    nn = RL.L.ref_hodlr_nnodes(h)
    ranks = np.zeros(2 * nn, dtype=np.int32)
    data = np.zeros(RL.L.ref_hodlr_flat_size(h))
    RL.L.ref_hodlr_export(h, R._i(ranks), R._d(data))
    meta = {
        "config": name, **c, "seed_offset": seed_offset, "patched": RL.patched, "ftz_daz": bool(ftz),
        "iterations": ref["iterations"], "alpha": ref["alpha"], "l0": ref["l0"],
        "wall_ms": ref["wall_ms"], "wall_s_process": wall_s,
        "per_iteration": [{"k": int(d[0]), "l": d[1], "c": d[2], "max_rank": int(d[3]), "memory_bytes": int(d[4]),
                           "wall_ms": d[5]} for d in ref["diag"]],
        "trace": RL.L.ref_hodlr_trace(h), "max_rank": RL.L.ref_hodlr_max_rank(h),
        "memory_bytes": RL.L.ref_hodlr_memory(h),
        "level_max_ranks": level_max_ranks(ranks, n, c["nmin"], RL),
        "peak_rss_gb": resource.getrusage(resource.RUSAGE_SELF).ru_maxrss / 2 ** 20,
        "host_cores_used": 1,
    }
    os.makedirs(outdir, exist_ok=True)
    if save_p:
        np.savez(os.path.join(outdir, f"{name}_P.npz"), ranks=ranks, data=data)
    if probes:
        Om = np.random.default_rng(probe_seed).standard_normal((n, probes))
        np.savez(os.path.join(outdir, f"{name}_probe.npz"), PrefOm=RL.apply(h, Om), seed=probe_seed,
                 trace=meta["trace"], iterations=meta["iterations"])
        meta["probes"] = {"m": probes, "seed": probe_seed}
    RL.L.ref_result_free(ref["handle"])
    with open(os.path.join(outdir, f"{name}.json"), "w") as f:
        json.dump(meta, f, indent=1)
    return meta


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("config", choices=sorted(CONFIGS))
    ap.add_argument("--out", required=True)
    ap.add_argument("--patched", action="store_true")
    ap.add_argument("--ftz", action="store_true")
    ap.add_argument("--save-p", action="store_true")
    ap.add_argument("--probes", type=int, default=0)
    ap.add_argument("--probe-seed", type=int, default=123)
    a = ap.parse_args()
    m = run(a.config, a.out, a.patched, a.ftz, a.save_p, a.probes, a.probe_seed)
    print(json.dumps({k: m[k] for k in ("config", "iterations", "wall_ms", "trace", "max_rank", "patched",
                                        "ftz_daz", "peak_rss_gb")}))


if __name__ == "__main__":
    main()
