"""BASELINE.json configs (SURVEY.md §8d conventions): seeded dimer chains.

Bond i (0-based) is t1 for even i and t2 for odd i (both chain ends strong, so
nu = n/2); diagonal disorder eps_dis * U(-1,1); band perturbation s * U(-1,1)
for |i-j| <= b; std::mt19937_64(seed) + uniform_real_distribution(-1, 1).
Seeds: PR1 = 1, small-gap = 2, banded = 3, sweep = 40 + j, large = 5.
"""
CONFIGS = {
    "pr1": dict(n=2048, b=1, t1=1.0, t2=0.5, eps_dis=0.1, s=0.0, nmin=128, eps=1e-10, seed=1),
    "sg4096": dict(n=4096, b=1, t1=1.0, t2=0.999, eps_dis=2e-4, s=0.0, nmin=256, eps=1e-10, seed=2),  # profiling
    "smallgap": dict(n=16384, b=1, t1=1.0, t2=0.999, eps_dis=2e-4, s=0.0, nmin=256, eps=1e-10, seed=2),
    "banded": dict(n=32768, b=8, t1=1.0, t2=0.8, eps_dis=0.0, s=0.05 / 17, nmin=256, eps=1e-10, seed=3),
    "sweep0.5": dict(n=65536, b=1, t1=1.0, t2=0.5, eps_dis=0.1, s=0.0, nmin=256, eps=1e-10, seed=40),
    "sweep0.9": dict(n=65536, b=1, t1=1.0, t2=0.9, eps_dis=0.02, s=0.0, nmin=256, eps=1e-10, seed=41),
    "sweep0.99": dict(n=65536, b=1, t1=1.0, t2=0.99, eps_dis=0.002, s=0.0, nmin=256, eps=1e-10, seed=42),
    "sweep0.999": dict(n=65536, b=1, t1=1.0, t2=0.999, eps_dis=2e-4, s=0.0, nmin=256, eps=1e-10, seed=43),
    "large": dict(n=131072, b=16, t1=1.0, t2=0.95, eps_dis=0.0, s=0.02 / 33, nmin=512, eps=1e-8, seed=5),
    # parity-only stress case (not a BASELINE config): t2 = 0.9999 puts c0 above 1e8, where a
    # Cholesky-based first iterate would lose accuracy
    "stress0.9999": dict(n=16384, b=1, t1=1.0, t2=0.9999, eps_dis=2e-5, s=0.0, nmin=256, eps=1e-10, seed=6),
}
HEADLINE = "sweep0.999"


def make_input(name_or_cfg, seed_offset=0):
    from . import dimer_chain
    c = CONFIGS[name_or_cfg] if isinstance(name_or_cfg, str) else name_or_cfg
    return dimer_chain(c["n"], c["t1"], c["t2"], c["eps_dis"], c["seed"] + seed_offset, b=c["b"], s=c["s"])
