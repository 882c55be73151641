"""Summarise ncu --set full captures into one tracked JSON (profiles/).

usage: python tools/ncu_summary.py <out.json> <label>=<report.ncu-rep>:<runs>:<command> ...
Per capture: the key raw metrics (time, DRAM bytes, IPC, issue-active, warps
active/eligible, SIMT efficiency, registers, shared memory, grid), the stall
reason shares from the SASS source page (not-issued samples folded into their
reason), and the DRAM bytes per run (so a bench batch of another size can scale
it).  Reads the reports with `ncu -i`; needs no GPU.
"""
import collections
import csv
import json
import subprocess
import sys

KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "sm__inst_executed.sum", "sm__inst_executed.avg.per_cycle_active",
        "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "sm__warps_active.avg.pct_of_peak_sustained_active",
        "smsp__warps_eligible.avg.per_cycle_active",
        "smsp__thread_inst_executed_per_inst_executed.ratio", "launch__registers_per_thread",
        "launch__shared_mem_per_block_dynamic", "launch__grid_size", "launch__block_size",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed"]
SCALE = {"Gbyte": 1e9, "Mbyte": 1e6, "Kbyte": 1e3, "byte": 1, "ms": 1e-3, "us": 1e-6,
         "ns": 1e-9, "s": 1}


def raw(rep):
    txt = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(txt.splitlines()))
    hdr, units, vals = rows[0], rows[1], rows[2]
    return {h: (vals[i], units[i]) for i, h in enumerate(hdr)}


def num(r, k):
    v, u = r[k]
    return float(v.replace(",", "")) * SCALE.get(u, 1)


def stalls(rep):
    txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source=sass"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(txt.splitlines()[1:]))
    hdr, data = rows[0], rows[1:]
    ix = {h: i for i, h in enumerate(hdr)}
    agg = collections.Counter()
    for r in data:
        for h in hdr:
            if h.startswith("stall_"):
                agg[h.split(" (")[0][6:]] += int(r[ix[h]] or 0)
    tot = sum(agg.values()) or 1
    return {k: round(v / tot, 4) for k, v in agg.most_common(10)}


def main():
    out, caps = sys.argv[1], sys.argv[2:]
    res = {}
    for c in caps:
        label, rest = c.split("=", 1)
        rep, runs, cmd = rest.split(":", 2)
        r = raw(rep)
        dram = num(r, "dram__bytes_read.sum") + num(r, "dram__bytes_write.sum")
        res[label] = {"report": rep.split("/")[-1], "command": cmd, "runs_in_capture": int(runs),
                      "metrics": {k: (r[k][0] + (" " + r[k][1] if r[k][1] else ""))
                                  for k in KEYS if k in r},
                      "stall_share": stalls(rep),
                      "dram_bytes_per_launch": dram,
                      "dram_bytes_per_run": dram / int(runs),
                      "kernel_seconds_under_ncu": num(r, "gpu__time_duration.sum")}
    json.dump(res, open(out, "w"), indent=1)
    print(json.dumps(res, indent=1)[:3000])


if __name__ == "__main__":
    main()
