"""Benchmark of the B200 hQDWH spectral-projector path (driver contract).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--config NAME]

One "step" = one complete hqdwh projector (qdwh.hpp:196-241) on the BASELINE
headline workload (config 4: n = 65536 tridiagonal dimer chain, t2 = 0.999, leaf 256,
eps 1e-10, FP64).  Metric: projector time in seconds (lower is better).

ours (default):
* value  : device time of the projector (CUDA events on the engine stream, from the bands'
           H2D (1 MB) to P complete in HBM; production path = CUDA-graph replay), mean over
           K steps; for N replicas (one independent projector per GPU, weak scaling) the
           whole-job time per projector = max-over-ranks total / (K * N).
* e2e    : the same metric through the public API with host buffers: H2D of the bands from
           pinned memory + projector + D2H of P and host HodlrMatrix assembly.
* phases : per-phase device times of the timed (graph-replay) steps with each phase's
           algorithmic work (device counters, SURVEY.md §8d units) and its roofline:
           time_roof = max(flops / FP64 tensor peak, bytes / HBM peak).
* roofline: the dominant kernel class (recompression: TSQR + core SVD + Q application) --
           algorithmic bytes 8 (p+s)(k_in+k_out) per batch / its CUDA-event time from one
           profiled step after the timed steps, against the measured HBM peak.
* cpu_baseline: the reference hqdwh (oracle/_ref, the unmodified reference headers) on the
           SAME config and input, one host core, run concurrently with the GPU steps on a
           core the GPU process does not use.

--impl reference: the reference's own CPU implementation (oracle/_ref) through its public
specproj::hqdwh on the same config, timed with steady_clock around the call exactly like
tools/specproj.cpp:71-80, input generated on the oracle side (this process never loads the
product library); one run in the default FP environment (the baseline) and one with
FTZ|DAZ beside it (x86 subnormal stalls).  A run takes minutes, so the arm
runs the count that fits (1 each) and reports it as `steps`.
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

from paper_1608_01164_b200.configs import CONFIGS, HEADLINE  # noqa: E402  (no library load)

PHASES = ("setup", "first", "multiply", "cholesky", "solve", "solveT", "axpby_sym")
PHASE_MS = ("ms_setup", "ms_first", "ms_multiply", "ms_cholesky", "ms_solve", "ms_solveT", "ms_axpby_sym")


def metric_name(cfg):
    """The BASELINE metric (projector wall time) on the configuration being run."""
    kind = "tridiagonal dimer chain" if cfg["b"] == 1 else f"banded b={cfg['b']}"
    return f"hqdwh projector time (n={cfg['n']} {kind}, t2={cfg['t2']})"


def workload(name, cfg):
    tag = {"sweep0.999": "BASELINE config 4 headline"}.get(name, "BASELINE config")
    return {"workload": f"hqdwh {name}: {tag}", "n": cfg["n"], "b": cfg["b"], "n_min": cfg["nmin"],
            "eps": cfg["eps"], "t2": cfg["t2"]}


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


def fp64_peak(S):
    """FP64 tensor-pipe peak: MEASURED_PEAKS.json has no FP64 entry, so the larger of the
    in-library DMMA probe (k_dmma_peak: mma.sync m8n8k4 f64 back to back on every SM) and
    cuBLAS DGEMM (torch.matmul float64, 8192^3, best of 5) measured here."""
    out = {}
    try:
        out["dmma_probe"] = S.measure_dmma_tflops()
    except Exception:   # noqa: BLE001
        pass
    try:
        import torch
        a = torch.randn(8192, 8192, dtype=torch.float64, device="cuda")
        b = torch.randn(8192, 8192, dtype=torch.float64, device="cuda")
        best = 1e9
        for _ in range(6):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            torch.matmul(a, b)
            e1.record()
            torch.cuda.synchronize()
            best = min(best, e0.elapsed_time(e1) / 1e3)
        out["cublas_dgemm"] = 2 * 8192.0 ** 3 / best / 1e12
        del a, b
    except Exception:   # noqa: BLE001
        pass
    peak = max(out.values()) if out else 40.0
    return peak, out


def ref_core():
    """the host core the concurrent CPU baseline runs on (the GPU process keeps the others)"""
    try:
        cores = sorted(os.sched_getaffinity(0))
    except AttributeError:
        return None
    return cores[-1] if len(cores) > 1 else None


def avail_ram_gb():
    try:
        for line in open("/proc/meminfo"):
            if line.startswith("MemAvailable:"):
                return int(line.split()[1]) / 2 ** 20
    except OSError:
        pass
    return 0.0


def ref_cmd(name, outdir, ftz=False):
    """oracle.run_ref on the config; the memory-patched oracle (bitwise equal, labelled)
    only when the host lacks the unpatched build's ~16 n^2 bytes"""
    n = CONFIGS[name]["n"]
    need_gb = 16.0 * n * n / 2 ** 30 * 1.1 + 4.0
    cmd = [sys.executable, "-m", "oracle.run_ref", name, "--out", outdir]
    if avail_ram_gb() < need_gb:
        cmd.append("--patched")
    if ftz:
        cmd.append("--ftz")
    return cmd


def start_cpu_baseline(name):
    from oracle import ref as R
    if not R.ref_available():
        return None
    core = ref_core()
    outdir = tempfile.mkdtemp(prefix="spg_cpu_")
    cmd = ref_cmd(name, outdir)
    if core is not None:
        cmd = ["taskset", "-c", str(core)] + cmd
        os.sched_setaffinity(0, set(os.sched_getaffinity(0)) - {core})
    log = open(os.path.join(outdir, "log"), "w")
    p = subprocess.Popen(cmd, cwd=ROOT, stdout=log, stderr=subprocess.STDOUT)
    return p, outdir, core


def finish_cpu_baseline(h, name, timeout=1800):
    if h is None:
        return None
    p, outdir, core = h
    try:
        p.wait(timeout=timeout)
    except subprocess.TimeoutExpired:
        p.kill()
        return None
    js = os.path.join(outdir, f"{name}.json")
    if not os.path.exists(js):
        return None
    m = json.load(open(js))
    ncpu = len(os.sched_getaffinity(0)) + (1 if core is not None else 0)
    return {"value": m["wall_ms"] / 1e3, "unit": "s", "cores": 1, "kind": "reference", "same_config": True,
            "sample": f"reference hqdwh (unmodified /root/reference headers, oracle/_ref"
                      f"{', memory-patched' if m['patched'] else ''}) on the same {name} input (n={m['n']}, "
                      f"b={m['b']}, leaf {m['nmin']}, eps {m['eps']}), 1 run, steady_clock around the call "
                      f"(tools/specproj.cpp:71-80), 1 of {ncpu} host cores (core {core}), concurrently with "
                      f"the GPU steps; iterations {m['iterations']}, trace {m['trace']:.6f}, max rank {m['max_rank']}",
            "iterations": m["iterations"], "trace": m["trace"], "max_rank": m["max_rank"]}


def bench_reference(args, cfg):
    """--impl reference: the reference's CPU implementation on the same config (rank 0 only)."""
    rank, ws, _ = dist_init()
    if rank != 0:
        return 0
    from oracle import ref as R
    if not R.ref_available():
        print(json.dumps({"impl": "reference", "unavailable": "oracle/_ref not built (reference sources absent)"}))
        return 0
    outdir = tempfile.mkdtemp(prefix="spg_ref_")
    cores = sorted(os.sched_getaffinity(0))
    n = cfg["n"]
    # the default-FP run and the FTZ|DAZ run side by side on two cores when the host has the
    # RAM for two unpatched oracles (16 n^2 bytes each), one after the other otherwise
    both = avail_ram_gb() > 2 * (16.0 * n * n / 2 ** 30 * 1.1 + 4.0) and len(cores) >= 2
    t0 = time.time()
    procs = []
    for j, ftz in enumerate((False, True)):
        d = os.path.join(outdir, "ftz" if ftz else "default")
        os.makedirs(d)
        cmd = ["taskset", "-c", str(cores[j % len(cores)])] + ref_cmd(args.config, d, ftz)
        p = subprocess.Popen(cmd, cwd=ROOT, stdout=open(os.path.join(d, "log"), "w"), stderr=subprocess.STDOUT)
        if not both:
            p.wait()
        procs.append((p, d))
    res = {}
    for (p, d), key in zip(procs, ("default", "ftz")):
        p.wait()
        js = os.path.join(d, f"{args.config}.json")
        res[key] = json.load(open(js)) if os.path.exists(js) else None
    wall = time.time() - t0
    m = res["default"]
    if m is None:
        print(json.dumps({"impl": "reference", "unavailable": "reference run failed: " +
                          open(os.path.join(procs[0][1], "log")).read()[-300:]}))
        return 0
    v = m["wall_ms"] / 1e3
    ftz = res["ftz"]
    sample = (f"reference hqdwh (unmodified /root/reference headers, oracle/_ref"
              f"{', memory-patched' if m['patched'] else ''}) on the {args.config} input (n={n}, b={cfg['b']}, "
              f"leaf {cfg['nmin']}, eps {cfg['eps']}): 1 run in the default FP environment (steady_clock "
              f"around specproj::hqdwh, tools/specproj.cpp:71-80), 1 of {len(cores)} host cores; the FTZ|DAZ "
              f"run {'beside it on another core' if both else 'after it'}; {m['iterations']} iterations, "
              f"trace {m['trace']:.6f}, max rank {m['max_rank']}")
    out = {"metric": metric_name(cfg), "value": v, "unit": "s",
           "n_gpus": args.gpus, "steps": 1, "warmup": 0, "steps_requested": args.steps,
           "warmup_requested": args.warmup, "ms_per_step": v * 1e3,
           "higher_is_better": False, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
           "data": "synthetic (seeded dimer chain, SURVEY.md §8d)", "impl": "reference",
           "config": workload(args.config, cfg),
           "cpu_baseline": {"value": v, "unit": "s", "cores": 1, "kind": "reference", "sample": sample},
           "ftz_daz": {"value": ftz["wall_ms"] / 1e3 if ftz else None, "unit": "s",
                       "note": "same binary with MXCSR FTZ|DAZ set (SURVEY.md §6: assemble_q subnormal stalls)"},
           "e2e": {"value": v, "unit": "s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
           "arm_wall_s": wall, "iterations": m["iterations"], "trace": m["trace"], "max_rank": m["max_rank"],
           "per_iteration_ms": [d["wall_ms"] for d in m["per_iteration"]]}
    print(json.dumps(out))
    return 0


def phase_roofline(infos, peak_fp64, peak_hbm):
    """per-phase device time (mean over the timed steps) with its algorithmic work and roofline"""
    out = {}
    K = len(infos)
    tot_f = tot_b = tot_ms = 0.0
    for i, (ph, key) in enumerate(zip(PHASES, PHASE_MS)):
        ms = sum(x[key] for x in infos) / K
        tb = sum(x["ph_trunc_bytes"][i] for x in infos) / K
        qr = sum(x["ph_qr_flops"][i] for x in infos) / K
        core = sum(x["ph_core_flops"][i] for x in infos) / K
        gemm = sum(x["ph_gemm_flops"][i] for x in infos) / K
        leaf = sum(x["ph_leaf_flops"][i] for x in infos) / K
        fl = qr + core + gemm + leaf
        t_f = fl / (peak_fp64 * 1e12) * 1e3
        t_b = tb / (peak_hbm * 1e9) * 1e3
        out[ph] = {"ms": ms, "trunc_bytes": tb, "flops": fl,
                   "flops_split": {"qr": qr, "trunc_core": core, "gemm": gemm, "leaf_chol": leaf},
                   "tflops": fl / (ms * 1e-3) / 1e12 if ms > 0 else None,
                   "gbs_recompression": tb / (ms * 1e-3) / 1e9 if ms > 0 else None,
                   "frac_fp64": (fl / (ms * 1e-3) / 1e12) / peak_fp64 if ms > 0 else None,
                   "frac_hbm": (tb / (ms * 1e-3) / 1e9) / peak_hbm if ms > 0 else None,
                   "roofline_ms": max(t_f, t_b), "frac_roofline": max(t_f, t_b) / ms if ms > 0 else None}
        tot_f += fl
        tot_b += tb
        tot_ms += ms
    out["total"] = {"ms": tot_ms, "flops": tot_f, "trunc_bytes": tot_b, "tflops": tot_f / (tot_ms * 1e-3) / 1e12,
                    "frac_fp64": tot_f / (tot_ms * 1e-3) / 1e12 / peak_fp64,
                    "roofline_ms": max(tot_f / (peak_fp64 * 1e12), tot_b / (peak_hbm * 1e9)) * 1e3}
    out["total"]["frac_roofline"] = out["total"]["roofline_ms"] / tot_ms
    return out


def bench_ours(args, cfg):
    import paper_1608_01164_b200 as S
    from paper_1608_01164_b200.configs import make_input
    rank, ws, local = dist_init()
    import torch
    if torch.cuda.is_available():
        torch.cuda.set_device(local)
    S.load_library()
    cpu_h = start_cpu_baseline(args.config) if (ws == 1 and not args.no_cpu_baseline) else None
    A = make_input(cfg, seed_offset=rank)
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
    peak_fp64, fp64_src = fp64_peak(S)
    roof = None
    if pinfo and pinfo.get("profiled"):
        tb = pinfo["trunc_bytes"]
        tms = pinfo["prof_ms_trunc"]
        nb = pinfo["prof_batches_trunc"]
        ach = tb / (tms * 1e-3) / 1e9
        traffic = None
        tpath = os.path.join(ROOT, "profiles", "ncu_trunc_traffic_r02.json")
        if os.path.exists(tpath):   # DRAM bytes per recompression batch from the committed ncu capture
            traffic = json.load(open(tpath)).get("dram_bytes_per_batch")
        roof = {"bound": "hbm", "achieved": ach, "peak": peak_hbm, "unit": "GB/s", "frac": ach / peak_hbm,
                "traffic": traffic,
                "traffic_source": "profiles/ncu_trunc_traffic_r02.json (ncu dram__bytes_read+write per batch)"
                                  if traffic else None,
                "kernel": "recompression (k_tsqr + k_core + k_apply, lowrank.hpp:67-86)",
                "algorithmic_bytes_per_launch": tb / max(nb, 1), "avg_launch_ms": tms / max(nb, 1),
                "launches_per_step": nb, "peak_source": peak_src,
                # share of the summed kernel-class time (what the ncu launch list's share measures:
                # profiles/ncu_launches_r02_summary.txt, k_tsqr + k_core_any + k_apply = 0.551 of the
                # summed kernel time there; the event brackets here also hold the gaps inside a batch)
                "share_of_step": tms / max(1e-9, sum(pinfo[k] for k in ("prof_ms_trunc", "prof_ms_gemm",
                                                                        "prof_ms_hsolve", "prof_ms_leaf"))),
                "share_of_span": tms / pinfo["ms_total"],
                "measured": "CUDA events around each recompression batch in one profiled step after the timed steps"}
        kcls = {k: pinfo[k] for k in ("prof_ms_trunc", "prof_ms_gemm", "prof_ms_hsolve", "prof_ms_leaf")}
        kcls["profiled_step_ms"] = pinfo["ms_total"]
    else:
        kcls = {}
    phases = phase_roofline(infos, peak_fp64, peak_hbm)
    cpu = finish_cpu_baseline(cpu_h, args.config)
    out = {
        "metric": metric_name(cfg),
        "value": value, "unit": "s", "n_gpus": ws, "steps": K, "warmup": args.warmup,
        "ms_per_step": value * 1e3, "higher_is_better": False, "scaling": "weak", "vs_baseline": None,
        "dtype": "f64", "data": "synthetic (seeded dimer chain, SURVEY.md §8d)",
        "config": {**workload(args.config, cfg), "replicas": ws,
                   "l2": "no flush: working set (7 HODLR matrices, ~4 GB) >> 126 MB L2"},
        "e2e": {"value": e2e, "unit": "s", "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h},
        "gpu_launches": int(sum(i["launches"] for i in infos)),
        "roofline": roof, "cpu_baseline": cpu, "clocks": ck,
        "phases": phases,
        "peaks": {"hbm_gbs": peak_hbm, "hbm_source": peak_src, "fp64_tflops": peak_fp64,
                  "fp64_source": "max of the measured probes (MEASURED_PEAKS.json has no FP64 entry)",
                  "fp64_probes": fp64_src},
        "iterations": I0["iterations"], "trace": I0["trace"], "max_rank": I0["max_rank"],
        "kernel_class_ms": kcls,
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
