"""Summarise an ncu capture + launch list into profiles/ (tracked).

usage: python tools/make_profile_summary.py <tag> [bench_json]
Reads gpurun_out/full_<tag>.ncu-rep, gpurun_out/full_<tag>.so, gpurun_out/launches_<tag>.csv.
Writes profiles/ncu_c2_summary.json (read by bench.py for roofline.traffic) and
profiles/<tag>_summary.md.
"""
import csv, json, os, subprocess, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
tag = sys.argv[1]
rep = os.path.join(ROOT, "gpurun_out", f"full_{tag}.ncu-rep")
so = os.path.join(ROOT, "gpurun_out", f"full_{tag}.so")
txt = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(txt.splitlines()))
hdr, units, vals = rows[0], rows[1], rows[2]
raw = {h: (vals[i], units[i]) for i, h in enumerate(hdr)}
def num(name):
    v, u = raw[name]
    v = float(v.replace(",", ""))
    scale = {"Gbyte": 1e9, "Mbyte": 1e6, "Kbyte": 1e3, "byte": 1, "ms": 1e-3, "us": 1e-6, "ns": 1e-9, "s": 1}.get(u, 1)
    return v * scale
keys = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "sm__inst_executed.avg.per_cycle_active", "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "smsp__warps_eligible.avg.per_cycle_active",
        "smsp__thread_inst_executed_per_inst_executed.ratio", "launch__registers_per_thread",
        "launch__shared_mem_per_block_dynamic", "launch__grid_size", "launch__block_size",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "sm__inst_executed.sum"]
summary = {"tag": tag, "kernel": "gs_sim_kernel<Hot<64,12,4>>",
           "command": "ncu --set full --clock-control none --import-source on -k regex:gs_sim_kernel -c 1 python bench.py --steps 1 --warmup 0 --no-cpu-baseline --no-e2e",
           "metrics": {k: raw[k][0] + (" " + raw[k][1] if raw[k][1] else "") for k in keys if k in raw}}
summary["dram_bytes_per_launch"] = num("dram__bytes_read.sum") + num("dram__bytes_write.sum")
summary["kernel_seconds_under_ncu"] = num("gpu__time_duration.sum")
# launch list share
launches = []
with open(os.path.join(ROOT, "gpurun_out", f"launches_{tag}.csv")) as fh:
    lines = [l for l in fh if l.startswith('"')]
for r in csv.reader(lines[1:]):
    launches.append((r[4], float(r[-1])))
tot = sum(t for _, t in launches)
mine = sum(t for n, t in launches if "gs_sim_kernel" in n)
summary["launch_list"] = {"launches": len(launches), "gs_sim_kernel_launches": sum(1 for n, _ in launches if "gs_sim_kernel" in n),
                          "gs_sim_kernel_share": mine / tot if tot else None,
                          "note": "cold-cache serialised ncu times; the L2-flush fill kernels are bench.py's, outside the timed region"}
stall = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "ncu_hot.py"), rep, "0"], capture_output=True, text=True).stdout
lines_out = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "ncu_lines.py"), rep, so, "25"], capture_output=True, text=True).stdout
funcs_out = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "ncu_funcs.py"), rep, so, "HotILi64", "30"], capture_output=True, text=True).stdout
regions_out = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "ncu_regions.py"), rep, so, "HotILi64", "0"], capture_output=True, text=True).stdout
os.makedirs(os.path.join(ROOT, "profiles"), exist_ok=True)
with open(os.path.join(ROOT, "profiles", "ncu_c2_summary.json"), "w") as fh:
    json.dump(summary, fh, indent=1)
bench = ""
if len(sys.argv) > 2 and os.path.exists(sys.argv[2]):
    bench = open(sys.argv[2]).read().strip()
with open(os.path.join(ROOT, "profiles", f"{tag}_summary.md"), "w") as fh:
    fh.write(f"# ncu summary {tag}: scenario megakernel on C2 (9472 runs x 300 windows)\n\n")
    fh.write("```\n" + json.dumps(summary, indent=1) + "\n```\n\n## stall reasons\n\n```\n" + stall + "```\n\n")
    fh.write("## code regions (quantum-step subroutine vs window/epoch code)\n\n```\n" + regions_out + "```\n\n")
    fh.write("## per function (samples / executed instructions)\n\n```\n" + funcs_out + "```\n\n")
    fh.write("## hottest source lines (samples / executed instructions)\n\n```\n" + lines_out + "```\n")
    if bench:
        fh.write("\n## bench.py line of the same round\n\n```\n" + bench + "\n```\n")
print(json.dumps(summary, indent=1))
