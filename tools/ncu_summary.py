"""Key metrics of an ncu --set full report (first kernel) for profiles/."""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
raw = subprocess.check_output(["ncu", "-i", rep, "--page", "raw", "--csv"], text=True, stderr=subprocess.DEVNULL)
r = csv.reader(io.StringIO(raw))
hdr, units, vals = next(r), next(r), next(r)
want = ["Kernel Name", "gpu__time_duration.sum", "sm__cycles_elapsed.avg.per_second", "launch__registers_per_thread",
        "launch__grid_size", "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
        "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
        "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
        "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed",
        "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
        "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "dram__throughput.avg.pct_of_peak_sustained_elapsed", "lts__t_sector_hit_rate.pct",
        "smsp__sass_thread_inst_executed_op_dfma_pred_on.sum", "smsp__sass_thread_inst_executed_op_ffma_pred_on.sum",
        "sm__warps_active.avg.pct_of_peak_sustained_active"]
for w in want:
    for h, u, v in zip(hdr, units, vals):
        if h == w:
            print(f"{h:80s} {u:12s} {v}")
stalls = [(float(v.replace(",", "")), h) for h, u, v in zip(hdr, units, vals)
          if h.startswith("smsp__average_warp_latency_issue_stalled") and h.endswith(".ratio") and v]
for v, h in sorted(stalls, reverse=True)[:8]:
    print(f"stall {h:74s} {v:.3f}")
