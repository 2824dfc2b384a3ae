"""Generates the golden fixtures of tests/golden/ by running the REFERENCE itself
(oracle/_ref/libspecproj_ref.so, built from /root/reference by oracle/Makefile).

    python tests/golden/make_golden.py          # in the build container (needs oracle/_ref)

Inputs come from the product's input generator (std::mt19937_64 +
uniform_real_distribution); the fixtures store the bands
themselves so the checks never depend on the generator.
"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

import paper_1608_01164_b200 as S  # noqa: E402  (host helpers only: generator, no GPU)
from oracle import ref as R  # noqa: E402

OUT = os.path.dirname(os.path.abspath(__file__))

# (name, n, b, n_min, eps, generator args)
CASES = [
    ("dimer_n128_b1", 128, 1, 16, 1e-10, ("dimer", 1.0, 0.5, 0.1, 0.0, 11)),
    ("dimer_n256_b1_gap", 256, 1, 32, 1e-10, ("dimer", 1.0, 0.95, 0.01, 0.0, 12)),
    ("rand_n200_b3", 200, 3, 24, 1e-10, ("random", 13)),
    ("dimer_n777_b3", 777, 3, 50, 1e-10, ("dimer", 1.0, 0.8, 0.0, 0.05 / 7, 14)),
    ("dimer_n512_b8", 512, 8, 64, 1e-10, ("dimer", 1.0, 0.8, 0.0, 0.05 / 17, 15)),
    # the reference tests' own spectra (synth.hpp, test_qdwh.cpp:122-139)
    ("synth_n512_gap1e1", 512, 1, 250, 1e-10, ("synth", 1e-1, 4)),
    ("synth_n512_b8_gap1e4", 512, 8, 500, 1e-10, ("synth", 1e-4, 5)),
    ("pr1", 2048, 1, 128, 1e-10, ("dimer", 1.0, 0.5, 0.1, 0.0, 1)),
    ("smallgap", 16384, 1, 256, 1e-10, ("dimer", 1.0, 0.999, 2e-4, 0.0, 2)),
]
DENSE_MAX = 256      # store the dense projector up to this n
PROBES = 4           # P @ Omega probes (Omega ~ seeded normal) for larger n


def make_bands(RL, n, b, gen):
    if gen[0] == "dimer":
        _, t1, t2, eps_dis, s, seed = gen
        return S.dimer_chain(n, t1, t2, eps_dis, seed, b=b, s=s)
    if gen[0] == "synth":
        return S.BandedSymmetric(n, b, RL.synth_banded(n, b, gen[1], gen[2]))
    return S.random_banded(n, b, gen[1])


def main(only=None):
    RL = R.RefLib()
    # Hqdwh.PropagatesCholeskyFailure (test_qdwh.cpp:184-190): the reference throws
    # NotPositiveDefiniteError on this input with eps = 1e-2, n_min = 32.
    bands = RL.synth_banded(256, 1, 1e-8, 19)
    try:
        RL.hqdwh(bands, 32, 1e-2)
        raise SystemExit("expected NotPositiveDefiniteError from the reference")
    except R.RefError as e:
        assert "status 1" in str(e), e
    np.savez_compressed(os.path.join(OUT, "npd_case.npz"), bands=R.pack_bands(bands), n=256, b=1, n_min=32, eps=1e-2)
    print("npd_case: reference raises NotPositiveDefiniteError")
    for name, n, b, nmin, eps, gen in CASES:
        if only and name not in only:
            continue
        A = make_bands(RL, n, b, gen)
        res = RL.hqdwh(A.bands, nmin, eps)
        h = res["P"]
        out = dict(n=n, b=b, n_min=nmin, eps=eps, bands=A.packed(), alpha=res["alpha"], l0=res["l0"],
                   iterations=res["iterations"], diag=res["diag"][:, :5], trace=RL.L.ref_hodlr_trace(h),
                   max_rank=RL.L.ref_hodlr_max_rank(h), memory=RL.L.ref_hodlr_memory(h), ref_wall_ms=res["wall_ms"])
        if n <= DENSE_MAX:
            out["P_dense"] = RL.to_dense(h, n)
        rng = np.random.default_rng(1000 + n)
        Om = rng.standard_normal((n, PROBES))
        out["omega_seed"] = 1000 + n
        out["P_omega"] = RL.apply(h, Om)
        np.savez_compressed(os.path.join(OUT, f"{name}.npz"), **out)
        RL.L.ref_result_free(res["handle"])
        print(f"{name}: iters {res['iterations']} trace {out['trace']:.6f} max_rank {out['max_rank']} "
              f"wall {res['wall_ms']:.0f} ms", flush=True)

    # kernel-level KATs: Givens R of the stacked QR (fast_qr.hpp:83-232) and estimates
    kat = {}
    for n, b, seed in [(64, 1, 21), (50, 3, 22), (33, 2, 23)]:
        A = S.random_banded(n, b, seed)
        p = R.pack_bands(A.bands)
        rd = np.zeros((2 * b + 1) * n)
        nrot = RL.L.ref_reduce(n, b, R._d(p), R._d(rd))
        st = np.zeros(1, dtype=np.int32)
        alpha = RL.L.ref_estimate_2norm(n, b, R._d(p))
        l0 = RL.L.ref_estimate_l0(n, b, R._d(p), alpha, R._i(st))
        kat[f"reduce_n{n}_b{b}_bands"] = p
        kat[f"reduce_n{n}_b{b}_R"] = rd
        kat[f"reduce_n{n}_b{b}_nrot"] = nrot
        kat[f"est_n{n}_b{b}"] = np.array([alpha, l0])
    for l in [1.0, 0.5, 0.1, 1e-3, 1e-6]:
        abc = np.zeros(3)
        RL.L.ref_qdwh_params(l, R._d(abc))
        kat[f"params_{l:g}"] = abc
    np.savez_compressed(os.path.join(OUT, "kat.npz"), **kat)
    print("kat.npz written")


if __name__ == "__main__":
    main(sys.argv[1:] or None)
