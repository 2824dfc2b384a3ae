"""Benchmark of the B200 hQDWH spectral-projector path (driver contract).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--config NAME]

One "step" = one complete hqdwh projector (qdwh.hpp:196-241) on the BASELINE
headline workload (n = 65536 tridiagonal dimer chain, t2 = 0.999, leaf 256,
eps 1e-10, FP64).  Metric: projector time in seconds (lower is better).

* value  : device time of the projector (CUDA events on the engine stream, from
           the bands' H2D (1 MB) to P complete in HBM; production path = CUDA-graph
           replay of the iteration plan), mean over K steps; for N replicas (one
           independent projector per GPU, weak scaling) the whole-job time per
           projector = max-over-ranks total / (K * N).
* e2e    : the same metric through the public API with host buffers: H2D of the
           bands from pinned memory + projector + D2H of P and host assembly.
* roofline: recompression (the north_star HBM-bound kernel class: TSQR + core
           SVD + Q application), algorithmic bytes 8 (p+s)(k_in+k_out) per
           truncation / its device time, from CUDA events around
           every recompression batch in one profiled step run after the timed
           steps (profile mode disables graph replay, so it is kept out of the
           timed region); a second entry gives the FP64 GEMM class against the
           measured DMMA peak.
* cpu_baseline: the reference (oracle/_ref, compiled from the reference sources)
           on a bounded sample of the same workload family, 1 host core.
"""
import argparse
import json
import os
import statistics
import subprocess
import sys
import tempfile
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

from paper_1608_01164_b200.configs import CONFIGS, HEADLINE  # noqa: E402

# Bounded CPU sample of the same workload family (t2 = 0.999 dimer chain) and the
# factor that scales its time to the headline n.  The factor is the measured ratio
# reference(n=65536) / reference(n=8192) from profiles/cpu_calibration_r01.json when
# present, else the complexity model n log^2(n / n_min).
CPU_SAMPLE = dict(CONFIGS[HEADLINE], n=8192)


def cpu_scale_factor():
    path = os.path.join(ROOT, "profiles", "cpu_calibration_r01.json")
    if os.path.exists(path):
        d = json.load(open(path))
        return float(d["ratio"]), f"measured ratio {d['ratio']:.2f} (profiles/cpu_calibration_r01.json)"
    import math
    big, small = CONFIGS[HEADLINE], CPU_SAMPLE
    f = (big["n"] * math.log2(big["n"] / big["nmin"]) ** 2) / (small["n"] * math.log2(small["n"] / small["nmin"]) ** 2)
    return f, f"model n*log2(n/n_min)^2 ratio {f:.2f}"


def metric_name(cfg):
    """The BASELINE metric (projector wall time) on the configuration being run."""
    kind = "tridiagonal dimer chain" if cfg["b"] == 1 else f"banded b={cfg['b']}"
    return f"hqdwh projector time (n={cfg['n']} {kind}, t2={cfg['t2']})"


def dist_init():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if ws > 1:
        import torch
        import torch.distributed as dist
        backend = "nccl" if torch.cuda.is_available() else "gloo"
        if backend == "nccl":
            torch.cuda.set_device(local)
        dist.init_process_group(backend=backend)
    return rank, ws, local


def barrier(ws):
    if ws > 1:
        import torch.distributed as dist
        dist.barrier()


def allreduce_max(x, ws):
    if ws == 1:
        return x
    import torch
    import torch.distributed as dist
    dev = "cuda" if dist.get_backend() == "nccl" else "cpu"
    t = torch.tensor([float(x)], dtype=torch.float64, device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def replica_value(total_max_s, steps, ws):
    """Whole-job time per projector for N independent replicas: the max-over-ranks
    total device time of the K timed steps divided by the K * N projectors done."""
    return total_max_s / (steps * ws)


class ClockSampler:
    """nvidia-smi clocks/throttle sampling during the timed region (B200_PROFILING.md)."""
    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index):
        self.f = tempfile.NamedTemporaryFile("w+", suffix=".csv", delete=False)
        self.gpu = gpu_index
        self.p = None

    def start(self):
        try:
            self.p = subprocess.Popen(["nvidia-smi", f"--id={self.gpu}", f"--query-gpu={self.Q}",
                                       "--format=csv,noheader,nounits", "-lms", "200"], stdout=self.f,
                                      stderr=subprocess.DEVNULL)
        except OSError:
            self.p = None

    def stop(self):
        if not self.p:
            return None
        self.p.terminate()
        try:
            self.p.wait(timeout=5)
        except subprocess.TimeoutExpired:
            self.p.kill()
        self.f.flush()
        rows = [r.split(",") for r in open(self.f.name).read().strip().splitlines() if r.strip()]
        sm, mx, reasons = [], 0.0, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for r in rows:
            try:
                sm.append(float(r[1])); mx = max(mx, float(r[2]))
                for nm, v in zip(names, r[5:9]):
                    if v.strip().lower() == "active":
                        reasons.add(nm)
            except (ValueError, IndexError):
                continue
        if not sm:
            return None
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": mx, "reasons": sorted(reasons), "samples": len(sm)}


def measured_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        d = json.load(open(p))
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


def run_cpu_reference(sample, steps, warmup):
    """Reference hqdwh (unmodified headers, oracle/_ref) on the bounded sample; 1 core."""
    from oracle import ref as R
    import paper_1608_01164_b200 as S
    if not R.ref_available():
        return None
    RL = R.RefLib()
    A = S.dimer_chain(sample["n"], sample["t1"], sample["t2"], sample["eps_dis"], sample["seed"], b=sample["b"],
                      s=sample["s"])
    times = []
    for i in range(warmup + steps):
        res = RL.hqdwh(A.bands, sample["nmin"], sample["eps"])
        if i >= warmup:
            times.append(res["wall_ms"] / 1e3)
        RL.L.ref_result_free(res["handle"])
    return times


def bench_reference(args, cfg):
    rank, ws, _ = dist_init()
    if rank != 0:
        return 0
    fac, how = cpu_scale_factor()
    times = run_cpu_reference(CPU_SAMPLE, args.steps, args.warmup)
    if times is None:
        print(json.dumps({"impl": "reference", "unavailable": "oracle/_ref not built (reference sources absent)"}))
        return 0
    v = statistics.mean(times) * fac
    sample = (f"reference hqdwh (unmodified /root/reference headers, oracle/_ref) on the same dimer-chain family "
              f"at n={CPU_SAMPLE['n']} (t2={CPU_SAMPLE['t2']}, leaf {CPU_SAMPLE['nmin']}, eps {CPU_SAMPLE['eps']}): "
              f"mean {statistics.mean(times):.2f} s over {len(times)} runs, scaled to n={cfg['n']} by {how}")
    out = {"metric": metric_name(cfg), "value": v, "unit": "s",
           "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup, "ms_per_step": v * 1e3,
           "higher_is_better": False, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
           "data": "synthetic (seeded dimer chain, SURVEY.md §8d)", "impl": "reference",
           "config": {"workload": f"hqdwh {args.config}", **{k: cfg[k] for k in ("n", "b", "nmin", "eps", "t2")}},
           "cpu_baseline": {"value": v, "unit": "s", "cores": 1, "kind": "reference", "sample": sample},
           "e2e": {"value": v, "unit": "s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(out))
    return 0


def bench_ours(args, cfg):
    import paper_1608_01164_b200 as S
    rank, ws, local = dist_init()
    import torch
    if torch.cuda.is_available():
        torch.cuda.set_device(local)
    S.load_library()
    A = S.dimer_chain(cfg["n"], cfg["t1"], cfg["t2"], cfg["eps_dis"], cfg["seed"] + rank, b=cfg["b"], s=cfg["s"])
    packed = A.packed()
    pinned = torch.empty(packed.size, dtype=torch.float64, pin_memory=torch.cuda.is_available())
    pinned_np = pinned.numpy()
    pinned_np[:] = packed
    h2d = packed.size * 8

    S.set_profile(False)   # timed steps: the production path (CUDA-graph replay of the iteration plan)
    for _ in range(args.warmup):   # (warms the pinned export pool too)
        r = S.hqdwh(A, cfg["nmin"], cfg["eps"], packed=pinned_np)
        P = r.P
        del P
        r.close()
    clocks = ClockSampler(local)
    barrier(ws)
    torch.cuda.synchronize()
    clocks.start()
    dev_s, e2e_s, infos, d2h = [], [], [], 0
    for _ in range(args.steps):
        t0 = time.perf_counter()
        r = S.hqdwh(A, cfg["nmin"], cfg["eps"], packed=pinned_np)
        P = r.P                              # D2H of the flat P + host HodlrMatrix assembly
        t1 = time.perf_counter()
        e2e_s.append(t1 - t0)
        dev_s.append(r.info["ms_total"] / 1e3)
        infos.append(r.info)
        ranks, data = P.to_flat()
        d2h = data.nbytes + ranks.nbytes
        del P, ranks, data   # the export buffer goes back to the pool before the next step
        r.close()
    torch.cuda.synchronize()
    barrier(ws)
    ck = clocks.stop()
    tot_dev = allreduce_max(sum(dev_s), ws)
    tot_e2e = allreduce_max(sum(e2e_s), ws)
    K = args.steps
    value = replica_value(tot_dev, K, ws)
    e2e = replica_value(tot_e2e, K, ws)
    # one further step in profile mode (CUDA events around every kernel batch on the
    # engine stream; graph replay off) for the per-class device times of the roofline
    pinfo = None
    if not args.no_profile:
        S.set_profile(True)
        r = S.hqdwh(A, cfg["nmin"], cfg["eps"], packed=pinned_np)
        pinfo = r.info
        r.close()
        S.set_profile(False)
    if rank != 0:
        return 0
    I0 = infos[-1]
    peak_hbm, peak_src = measured_peaks()
    roof = None
    roof_gemm = None
    if pinfo and pinfo.get("profiled"):
        infos_p = [pinfo]
        Kp = 1
        tb = sum(i["trunc_bytes"] for i in infos_p) / Kp
        tms = sum(i["prof_ms_trunc"] for i in infos_p) / Kp
        nb = sum(i["prof_batches_trunc"] for i in infos_p) / Kp
        ach = tb / (tms * 1e-3) / 1e9
        traffic = None
        tpath = os.path.join(ROOT, "profiles", "ncu_trunc_traffic_r01.json")
        if os.path.exists(tpath):   # DRAM bytes per recompression batch from the committed ncu capture
            traffic = json.load(open(tpath)).get("dram_bytes_per_batch")
        roof = {"bound": "hbm", "achieved": ach, "peak": peak_hbm, "unit": "GB/s", "frac": ach / peak_hbm,
                "traffic": traffic, "traffic_source": "profiles/ncu_trunc_traffic_r01.json (ncu dram__bytes_read"
                                                      "+write per batch)" if traffic else None, "kernel": "recompression (k_tsqr + k_core + k_apply, lowrank.hpp:67-86)",
                "algorithmic_bytes_per_launch": tb / max(nb, 1), "avg_launch_ms": tms / max(nb, 1),
                "launches_per_step": nb, "peak_source": peak_src,
                "share_of_step": tms / (pinfo["ms_total"]),
                "measured": "CUDA events around each recompression batch in one profiled step after the timed steps"}
        try:
            dmma = S.measure_dmma_tflops()
        except Exception:
            dmma = None
        gf = sum(i["gemm_flops"] for i in infos_p) / Kp
        gms = sum(i["prof_ms_gemm"] for i in infos_p) / Kp
        if dmma:
            a = gf / (gms * 1e-3) / 1e12
            roof_gemm = {"bound": "tensor", "achieved": a, "peak": dmma, "unit": "TFLOP/s", "frac": a / dmma,
                         "kernel": "k_gemm (mma.sync m8n8k4 f64 -> DMMA)", "peak_source": "measured DMMA probe",
                         "share_of_step": gms / pinfo["ms_total"]}
        phase = {k: pinfo[k] for k in ("prof_ms_trunc", "prof_ms_gemm", "prof_ms_hsolve", "prof_ms_leaf")}
        phase["profiled_step_ms"] = pinfo["ms_total"]
    else:
        phase = {}
    cpu = None
    if ws == 1 and not args.no_cpu_baseline:
        fac, how = cpu_scale_factor()
        times = run_cpu_reference(CPU_SAMPLE, 1, 0)
        if times:
            cpu = {"value": times[0] * fac, "unit": "s", "cores": 1, "kind": "reference",
                   "sample": f"reference hqdwh (oracle/_ref) on the n={CPU_SAMPLE['n']} t2={CPU_SAMPLE['t2']} "
                             f"dimer chain: {times[0]:.2f} s on 1 host core, scaled by {how}"}
    out = {
        "metric": metric_name(cfg),
        "value": value, "unit": "s", "n_gpus": ws, "steps": K, "warmup": args.warmup,
        "ms_per_step": value * 1e3, "higher_is_better": False, "scaling": "weak", "vs_baseline": None,
        "dtype": "f64", "data": "synthetic (seeded dimer chain, SURVEY.md §8d)",
        "config": {"workload": f"hqdwh {args.config}: BASELINE config 4 headline", "n": cfg["n"], "b": cfg["b"],
                   "n_min": cfg["nmin"], "eps": cfg["eps"], "t2": cfg["t2"], "replicas": ws,
                   "l2": "no flush: working set (7 HODLR matrices, ~4 GB) >> 126 MB L2"},
        "e2e": {"value": e2e, "unit": "s", "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h},
        "gpu_launches": int(sum(i["launches"] for i in infos)),
        "roofline": roof, "roofline_gemm": roof_gemm, "cpu_baseline": cpu, "clocks": ck,
        "iterations": I0["iterations"], "trace": I0["trace"], "max_rank": I0["max_rank"],
        "phases_ms": {k: I0[k] for k in ("ms_setup", "ms_first", "ms_multiply", "ms_cholesky", "ms_solve",
                                          "ms_solveT", "ms_axpby_sym")},
        "kernel_class_ms": phase,
        "graph_replay": bool(I0.get("graph_used")),
    }
    print(json.dumps(out))
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default=HEADLINE, choices=sorted(CONFIGS))
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-profile", action="store_true")
    args = ap.parse_args()
    cfg = CONFIGS[args.config]
    if args.impl == "reference":
        return bench_reference(args, cfg)
    return bench_ours(args, cfg)


if __name__ == "__main__":
    sys.exit(main())
