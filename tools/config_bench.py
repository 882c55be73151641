"""Per-config table at the configs' full sizes (GPU box).

bench.py's ``per_config`` block runs C1/C3/C4/C5 at bounded sizes so the
default bench finishes in minutes (C4 at 600 windows); this tool runs the
same measurement (bench.measure_config: device value, state-touch fraction,
oracle CPU baseline on a bounded prefix, record-by-record parity sample of
that prefix) on the full configurations, one JSON line per config:

  C1  4736 copies of the 1-node scenario (one wave of XS warps), both policies
  C2  21312 runs x 300 windows (the headline workload)
  C3  1024 bursty traces x both policies
  C4  148 runs x 3600 windows (one compressed day; one XL CTA per SM)
  C5  the 100k sweep's 12.5k-run shard of one GPU

usage: python tools/config_bench.py [--only C2,C4] > gpurun_out/configs.jsonl
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import bench  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--only", default="C1,C2,C3,C4,C5")
    ap.add_argument("--c4-windows", type=int, default=3600)
    a = ap.parse_args()
    import torch
    from paper_2309_00558_b200 import workloads as wl
    flush = torch.empty(256 * 1024 * 1024, dtype=torch.uint8, device="cuda")
    threads = os.cpu_count() or 1
    peak, _ = bench.load_peak()
    only = set(a.only.split(","))
    work = []
    if "C2" in only:
        work.append(("C2", "4 nodes, 10 functions, Poisson, autoscaling + model sharing, 300 windows",
                     bench.c2_seq(range(21312), 300), ["fast"] * 21312))
    work += bench.config_workloads(only & {"C1", "C3", "C4", "C5"}, windows_c4=a.c4_windows)
    for name, desc, scen, pols in sorted(work):
        rec = bench.measure_config(name, desc, scen, pols, flush=flush, threads=threads, peak=peak)
        print(json.dumps(rec), flush=True)


if __name__ == "__main__":
    main()
