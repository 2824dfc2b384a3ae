"""Key metrics of ncu --set full reports (one launch each): python tools_gpu/ncu_full_summary.py rep... > json"""
import csv, json, subprocess, sys
WANT = {
    "gpu__time_duration.sum": "duration",
    "launch__grid_size": "grid", "launch__block_size": "block",
    "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active": "fp64_pipe_pct_active",
    "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active": "fp64_pipe_cycles_pct_active",
    "sm__inst_executed_pipe_tensor_subpipe_dmma.avg.pct_of_peak_sustained_active": "dmma_pipe_pct_active(avg active SM)",
    "SM_C.TriageCompute.smsp__pipe_tensor_subpipe_dmma_cycles_active.avg": "dmma_subpipe_cycles_active(avg SMSP)",
    "TPC.TriageCompute.sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed": "tensor_pipe_pct_elapsed(chip)",
    "TPC.TriageCompute.sm__pipe_fp64_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed": "fp64_pipe_pct_elapsed(chip)",
    "sm__warps_active.avg.pct_of_peak_sustained_active": "achieved_occupancy_pct",
    "dram__bytes_read.sum": "dram_read", "dram__bytes_write.sum": "dram_write",
    "lts__t_sector_hit_rate.pct": "l2_hit_pct",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed": "sm_throughput_pct",
    "gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed": "mem_throughput_pct",
    "launch__registers_per_thread": "regs", "launch__shared_mem_per_block_dynamic": "dyn_smem",
    "smsp__cycles_active.avg": "smsp_cycles_active", "sm__cycles_elapsed.max": "sm_cycles_elapsed",
    "smsp__inst_executed.sum": "warp_instructions",
}
out = {}
for rep in sys.argv[1:]:
    txt = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(txt.splitlines()))
    if len(rows) < 3:
        continue
    hdr, units, vals = rows[0], rows[1], rows[2]
    name = vals[hdr.index("Kernel Name")].split("(")[0].replace("spg::", "")
    d = {}
    for m, nick in WANT.items():
        if m in hdr:
            i = hdr.index(m)
            d[nick] = (vals[i] + " " + units[i]).strip()
    out[name] = d
print(json.dumps(out, indent=1))
