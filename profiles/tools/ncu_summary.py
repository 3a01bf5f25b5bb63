import csv, subprocess, sys
rep = sys.argv[1]
out = subprocess.run(["ncu", "-i", rep, "--page", "details", "--csv"], capture_output=True, text=True).stdout
r = list(csv.reader(out.splitlines()))
h = r[0]
want = ["Duration", "Executed Ipc Active", "Issue Slots Busy", "Achieved Occupancy", "Registers Per Thread",
        "Executed Instructions", "Warp Cycles Per Issued Instruction", "Avg. Active Threads Per Warp",
        "L2 Hit Rate", "L1/TEX Hit Rate", "SM Active Cycles", "Elapsed Cycles", "Theoretical Occupancy",
        "Eligible Warps Per Scheduler", "No Eligible", "DRAM Throughput"]
for row in r[1:]:
    d = dict(zip(h, row))
    if d["Metric Name"] in want:
        print(d["Kernel Name"][:30], d["Metric Name"].ljust(40), d["Metric Unit"].ljust(14), d["Metric Value"])
out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
r = list(csv.reader(out.splitlines()))
h, u = r[0], r[1]
for v in r[2:]:
    for name, unit, val in zip(h, u, v):
        if ("warp_issue_stalled" in name or "average_warps_issue_stalled" in name) and name.endswith("per_issue_active.ratio"):
            try:
                if float(val) > 0.05: print("  stall", name.split("stalled_")[1].split("_per")[0], val)
            except ValueError: pass
        if name.startswith("sm__inst_executed_pipe_") and name.endswith(".avg.pct_of_peak_sustained_active"):
            try:
                if float(val) > 1: print("  pipe", name[len("sm__inst_executed_pipe_"):].split(".")[0], val)
            except ValueError: pass
        if name in ("dram__bytes_read.sum", "dram__bytes_write.sum", "smsp__sass_thread_inst_executed_op_ffma_pred_on.sum",
                    "smsp__sass_thread_inst_executed_op_fadd_pred_on.sum", "smsp__sass_thread_inst_executed_op_fmul_pred_on.sum",
                    "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active", "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active",
                    "sm__pipe_fmaheavy_cycles_active.avg.pct_of_peak_sustained_active", "sm__pipe_xu_cycles_active.avg.pct_of_peak_sustained_active",
                    "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", "sm__pipe_shared_cycles_active.avg.pct_of_peak_sustained_active"):
            print("  ", name, unit, val)
