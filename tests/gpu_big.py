"""GPU-box driver for the BASELINE configs (not collected by pytest).

python tests/gpu_big.py <config> [--ref] [--probes FILE]
  config: pr1 | smallgap | banded | sweep0.5 | sweep0.9 | sweep0.99 | sweep0.999 | large
  --ref : also run the reference (oracle/_ref) and report ||P - P_ref||_2 by power iteration
"""
import json
import sys
import time

import numpy as np

sys.path.insert(0, ".")
import paper_1608_01164_b200 as S  # noqa: E402

CONFIGS = {
    "pr1": dict(n=2048, b=1, t1=1.0, t2=0.5, eps_dis=0.1, s=0.0, nmin=128, eps=1e-10, seed=1),
    "sg4096": dict(n=4096, b=1, t1=1.0, t2=0.999, eps_dis=2e-4, s=0.0, nmin=256, eps=1e-10, seed=2),
    "smallgap": dict(n=16384, b=1, t1=1.0, t2=0.999, eps_dis=2e-4, s=0.0, nmin=256, eps=1e-10, seed=2),
    "banded": dict(n=32768, b=8, t1=1.0, t2=0.8, eps_dis=0.0, s=0.05 / 17, nmin=256, eps=1e-10, seed=3),
    "sweep0.5": dict(n=65536, b=1, t1=1.0, t2=0.5, eps_dis=0.1, s=0.0, nmin=256, eps=1e-10, seed=40),
    "sweep0.9": dict(n=65536, b=1, t1=1.0, t2=0.9, eps_dis=0.02, s=0.0, nmin=256, eps=1e-10, seed=41),
    "sweep0.99": dict(n=65536, b=1, t1=1.0, t2=0.99, eps_dis=0.002, s=0.0, nmin=256, eps=1e-10, seed=42),
    "sweep0.999": dict(n=65536, b=1, t1=1.0, t2=0.999, eps_dis=2e-4, s=0.0, nmin=256, eps=1e-10, seed=43),
    "large": dict(n=131072, b=16, t1=1.0, t2=0.95, eps_dis=0.0, s=0.02 / 33, nmin=512, eps=1e-8, seed=5),
}


def make_input(c):
    return S.dimer_chain(c["n"], c["t1"], c["t2"], c["eps_dis"], c["seed"], b=c["b"], s=c["s"])


def power_norm(apply, n, iters=40, seed=0):
    rng = np.random.default_rng(seed)
    x = rng.standard_normal((n, 1))
    x /= np.linalg.norm(x)
    lam = 0.0
    for _ in range(iters):
        y = apply(x)
        lam = np.linalg.norm(y)
        if lam == 0:
            return 0.0
        x = y / lam
    return lam


def main():
    name = sys.argv[1]
    c = CONFIGS[name]
    A = make_input(c)
    out = {"config": name, **c}
    t0 = time.time()
    r = S.hqdwh(A, c["nmin"], c["eps"])
    out["gpu_wall_s"] = time.time() - t0
    out["info"] = r.info
    out["per_iteration"] = [d.__dict__ for d in r.per_iteration]
    # warm run timing
    t0 = time.time()
    r2 = S.hqdwh(A, c["nmin"], c["eps"])
    out["gpu_wall_s_warm"] = time.time() - t0
    out["info_warm"] = r2.info
    r2.close()
    n = c["n"]
    Pap = lambda x: r.apply(x, 0)  # noqa: E731
    out["idem"] = power_norm(lambda x: Pap(Pap(x)) - Pap(x), n)
    print(json.dumps(out, indent=1, default=float), flush=True)
    if "--ref" in sys.argv:
        from oracle import ref as R
        RL = R.RefLib()
        t0 = time.time()
        ref = RL.hqdwh(A.bands, c["nmin"], c["eps"])
        res = {"ref_wall_s": time.time() - t0, "ref_iters": ref["iterations"], "ref_alpha": ref["alpha"],
               "ref_l0": ref["l0"], "ref_trace": RL.L.ref_hodlr_trace(ref["P"]),
               "ref_max_rank": RL.L.ref_hodlr_max_rank(ref["P"])}
        Rap = lambda x: RL.apply(ref["P"], x)  # noqa: E731
        res["diff_2norm"] = power_norm(lambda x: Pap(x) - Rap(x), n)
        res["ref_diag"] = RL_diag = ref["diag"].tolist()
        rng = np.random.default_rng(123)
        Om = rng.standard_normal((n, 8))
        np.savez_compressed(f"gpurun_out/probe_{name}.npz", PrefOm=Rap(Om), seed=123, trace=res["ref_trace"])
        print(json.dumps(res, indent=1, default=float), flush=True)


if __name__ == "__main__":
    main()
