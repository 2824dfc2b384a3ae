"""Parity of the CUDA projector against the reference at BASELINE sizes (GPU box tool).

    python tests/parity_big.py --configs sweep0.999,banded --ref-dir /tmp/parity_ref \
        [--run-ref] [--patched-above 40000] [--ftz CFG,...] [--tag NAME] [--out FILE]

Not collected by pytest (it runs the reference for minutes per config).  For each config:

* the CUDA path (``paper_1608_01164_b200.hqdwh`` through the C-ABI) on the config's input;
* the reference ``specproj::hqdwh`` (oracle/_ref, qdwh.hpp:196-241) on the SAME input,
  run by ``oracle.run_ref`` in its own process (``--run-ref``; one host core each, several
  configs concurrently), or read from ``--ref-dir`` when it ran elsewhere;
* north_star's gate: ||P_gpu - P_ref||_2 by power iteration on E = P_gpu - P_ref (>= 40
  steps, P_gpu applied on the device, P_ref applied to its flat export on the host), the
  Halko bound 10 sqrt(2/pi) max_i ||E w_i|| over 16 Gaussian probes (Halko, Martinsson &
  Tropp 2011, Lemma 4.1: holds with probability >= 1 - 10^-16), ||P^2 - P||_2 by power
  iteration, trace, iterations, and the per-level max ranks next to the reference's.

Writes one JSON (``--out``, default gpurun_out/parity_<tag>.json).
"""
import argparse
import json
import os
import subprocess
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import paper_1608_01164_b200 as S  # noqa: E402
from paper_1608_01164_b200.configs import CONFIGS, make_input  # noqa: E402

HALKO = 10.0 * np.sqrt(2.0 / np.pi)


def power_norm(apply, n, iters=40, seed=0):
    """largest |eigenvalue| of a symmetric operator by power iteration (returns the last Rayleigh norm)"""
    x = np.random.default_rng(seed).standard_normal((n, 1))
    x /= np.linalg.norm(x)
    lam = 0.0
    for _ in range(iters):
        y = apply(x)
        lam = float(np.linalg.norm(y))
        if lam == 0.0:
            return 0.0
        x = y / lam
    return lam


def level_max_ranks(H):
    t = H.tree
    depth = np.zeros(len(t), dtype=np.int32)
    out = {}
    for i in range(len(t)):
        if not t.leaf(i):
            depth[t.left[i]] = depth[t.right[i]] = depth[i] + 1
            U, _ = H.upper[i]
            Ul, _ = H.lower[i]
            out[int(depth[i]) + 1] = max(out.get(int(depth[i]) + 1, 0), U.shape[1], Ul.shape[1])
    return [out[d] for d in sorted(out)]


def spawn_refs(names, ref_dir, patched_above, ftz):
    procs = []
    ncpu = os.cpu_count() or 2
    for j, name in enumerate(names):
        c = CONFIGS[name]
        cmd = [sys.executable, "-m", "oracle.run_ref", name, "--out", ref_dir, "--save-p", "--probes", "16"]
        if c["n"] >= patched_above:
            cmd.append("--patched")
        if name in ftz:
            cmd.append("--ftz")
        core = (j + 1) % ncpu
        log = open(os.path.join(ref_dir, f"{name}.log"), "w")
        procs.append(subprocess.Popen(["taskset", "-c", str(core)] + cmd, cwd=ROOT, stdout=log, stderr=subprocess.STDOUT))
    return procs


def wait_ref(ref_dir, name, procs, timeout):
    js = os.path.join(ref_dir, f"{name}.json")
    t0 = time.time()
    while not os.path.exists(js):
        if time.time() - t0 > timeout:
            return None
        if procs and all(p.poll() is not None for p in procs) and not os.path.exists(js):
            return None
        time.sleep(2.0)
    time.sleep(1.0)
    return json.load(open(js))


def compare(name, r, ref_meta, ref_dir):
    c = CONFIGS[name]
    n = c["n"]
    tree = S.PartitionTree(n, c["nmin"])
    f = np.load(os.path.join(ref_dir, f"{name}_P.npz"))
    Pref = S.HodlrMatrix.from_flat(tree, f["ranks"], f["data"])
    gpu = lambda x: r.apply(x, 0)                       # noqa: E731
    ref = lambda x: Pref.matmat(x)                      # noqa: E731
    t0 = time.time()
    diff = power_norm(lambda x: gpu(x) - ref(x), n, iters=40)
    Om = np.random.default_rng(123).standard_normal((n, 16))
    E_om = gpu(Om) - ref(Om)
    halko = HALKO * float(np.max(np.linalg.norm(E_om, axis=0)))
    idem = power_norm(lambda x: gpu(gpu(x)) - gpu(x), n, iters=40)
    idem_ref = power_norm(lambda x: ref(ref(x)) - ref(x), n, iters=40)
    Pg = r.P
    out = {
        "config": name, "n": n, "b": c["b"], "n_min": c["nmin"], "eps": c["eps"], "gate": 100 * c["eps"],
        "diff_2norm_power": diff, "diff_2norm_halko_bound": halko, "idem_2norm": idem, "idem_2norm_ref": idem_ref,
        "trace_gpu": r.info["trace"], "trace_ref": ref_meta["trace"], "nu": n // 2,
        "iterations_gpu": r.iterations, "iterations_ref": ref_meta["iterations"],
        "alpha_gpu": r.alpha, "alpha_ref": ref_meta["alpha"], "l0_gpu": r.l0, "l0_ref": ref_meta["l0"],
        "c_gpu": [d.c for d in r.per_iteration], "c_ref": [d["c"] for d in ref_meta["per_iteration"]],
        "iter_max_rank_gpu": [d.max_rank for d in r.per_iteration],
        "iter_max_rank_ref": [d["max_rank"] for d in ref_meta["per_iteration"]],
        "level_max_ranks_gpu": level_max_ranks(Pg), "level_max_ranks_ref": ref_meta["level_max_ranks"],
        "max_rank_gpu": r.info["max_rank"], "max_rank_ref": ref_meta["max_rank"],
        "gpu_ms_device": r.info["ms_total"], "ref_wall_ms": ref_meta["wall_ms"],
        "ref_patched": ref_meta["patched"], "ref_ftz_daz": ref_meta["ftz_daz"],
        "env": {k: v for k, v in os.environ.items() if k.startswith("SPG_")},
        "check_s": time.time() - t0,
    }
    g = out["gate"]
    out["pass"] = bool(diff <= g and halko <= g and idem <= g and round(out["trace_gpu"]) == n // 2
                       and out["iterations_gpu"] == out["iterations_ref"])
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--configs", required=True)
    ap.add_argument("--ref-dir", default="/tmp/parity_ref")
    ap.add_argument("--run-ref", action="store_true")
    ap.add_argument("--patched-above", type=int, default=1 << 30)
    ap.add_argument("--ftz", default="")
    ap.add_argument("--tag", default="r02")
    ap.add_argument("--out", default=None)
    ap.add_argument("--ref-timeout", type=float, default=7200.0)
    a = ap.parse_args()
    names = a.configs.split(",")
    os.makedirs(a.ref_dir, exist_ok=True)
    procs = spawn_refs(names, a.ref_dir, a.patched_above, set(a.ftz.split(","))) if a.run_ref else []
    results = {}
    for name in names:            # GPU first: all projectors while the references run
        c = CONFIGS[name]
        S.hqdwh(make_input(c), c["nmin"], c["eps"]).close()        # first call of the shape builds the plan
        results[name] = S.hqdwh(make_input(c), c["nmin"], c["eps"])
        print(f"gpu {name}: {results[name].info['ms_total']:.1f} ms, {results[name].iterations} iterations",
              flush=True)
    out = {"tag": a.tag, "host_cpus": os.cpu_count(), "results": []}
    path = a.out or os.path.join(ROOT, "gpurun_out", f"parity_{a.tag}.json")
    os.makedirs(os.path.dirname(path), exist_ok=True)
    for name in names:
        meta = wait_ref(a.ref_dir, name, procs, a.ref_timeout)
        if meta is None:
            out["results"].append({"config": name, "error": "reference did not finish"})
            continue
        res = compare(name, results[name], meta, a.ref_dir)
        print(json.dumps(res), flush=True)
        out["results"].append(res)
        results[name].close()
        with open(path, "w") as f:
            json.dump(out, f, indent=1)
    for p in procs:
        p.wait()
    with open(path, "w") as f:
        json.dump(out, f, indent=1)


if __name__ == "__main__":
    main()
