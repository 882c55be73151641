"""Print key raw metrics of an ncu report (first kernel in it)."""
import csv, subprocess, sys, json
rep = sys.argv[1]
txt = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(txt.splitlines()))
hdr, units, vals = rows[0], rows[1], rows[2]
want = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "lts__t_bytes.sum", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed.sum", "sm__inst_executed.avg.per_cycle_active",
        "smsp__inst_executed.avg.per_cycle_active", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "launch__registers_per_thread", "launch__occupancy_limit_registers",
        "launch__occupancy_limit_shared_mem", "sm__maximum_warps_per_active_cycle_pct",
        "smsp__thread_inst_executed_per_inst_executed.ratio", "launch__grid_size",
        "launch__block_size", "sm__cycles_elapsed.avg", "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
        "smsp__issue_active.avg.pct_of_peak_sustained_active", "launch__shared_mem_per_block_dynamic",
        "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "smsp__warps_eligible.avg.per_cycle_active",
        "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active"]
out = {}
for i, h in enumerate(hdr):
    if h in want:
        print(f"{h:70s} {units[i]:12s} {vals[i]}")
        out[h] = (vals[i], units[i])
if len(sys.argv) > 2:
    json.dump(out, open(sys.argv[2], "w"), indent=1)
