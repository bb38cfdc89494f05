"""Summarise an ncu report (details page) into key lines (development aid)."""
import csv, subprocess, sys
keys = ["Duration", "Elapsed Cycles", "Compute (SM) Throughput", "Memory Throughput", "DRAM Throughput",
        "Executed Ipc Active", "Issue Slots Busy", "Registers Per Thread", "Theoretical Occupancy",
        "Achieved Occupancy", "Achieved Active Warps Per SM", "Avg. Active Threads Per Warp",
        "Avg. Not Predicated Off Threads Per Warp", "Warp Cycles Per Issued Instruction",
        "Eligible Warps Per Scheduler", "No Eligible", "Branch Efficiency", "L1/TEX Hit Rate",
        "L2 Hit Rate", "Executed Instructions", "Grid Size", "Block Size", "Stack Size",
        "Local Memory Spilling Requests", "Shared Memory Configuration Size"]
rep = sys.argv[1]
out = subprocess.run(["ncu", "-i", rep, "--page", "details", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
hdr = rows[0]
seen = {}
for r in rows[1:]:
    d = dict(zip(hdr, r))
    k = d.get("Metric Name", "")
    kid = d.get("ID", "")
    if k in keys:
        seen.setdefault(kid + " " + d.get("Kernel Name", "")[:40], []).append(f"{k}={d.get('Metric Value')} {d.get('Metric Unit')}")
for k, v in seen.items():
    print(k)
    for x in v:
        print("   ", x)
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(raw.splitlines()))
hdr = rows[0]
want = ["sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
        "smsp__thread_inst_executed_per_inst_executed.ratio", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "smsp__sass_thread_inst_executed_op_dfma_pred_on.sum", "smsp__sass_thread_inst_executed_op_dmul_pred_on.sum",
        "smsp__sass_thread_inst_executed_op_dadd_pred_on.sum", "sm__sass_thread_inst_executed_op_dfma_pred_on.sum",
        "sm__sass_thread_inst_executed_op_dmul_pred_on.sum", "sm__sass_thread_inst_executed_op_dadd_pred_on.sum",
        "smsp__pcsamp_warps_issue_stalled_long_scoreboard", "gpu__time_duration.sum",
        "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_elapsed"]
for r in rows[2:]:
    d = dict(zip(hdr, r))
    print("RAW", d.get("ID"), d.get("Kernel Name", "")[:30])
    for w in want:
        for h in hdr:
            if h.startswith(w):
                print("    ", h, d[h])
