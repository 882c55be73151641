"""Throughput of the CUDA path on each BASELINE.json config (GPU box).

Reports device-time simulated scenario-seconds/s for C1..C5 next
to the oracle port on a bounded sample of the same runs on the host cores,
and checks the GPU against the oracle on that sample (bit-exact records).
bench.py's headline stays C2; this is the per-config evidence table.

usage: python tools/config_bench.py [--quick] > gpurun_out/configs.jsonl
"""
import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))

import numpy as np  # noqa: E402

import oracle  # noqa: E402  (checker + CPU baseline only)
from paper_2309_00558_b200 import backend, compiler as cc, workloads as wl  # noqa: E402
from paper_2309_00558_b200.scenario import Scenario  # noqa: E402


def configs(quick: bool):
    k = 4 if quick else 1
    yield ("C1", "1 node, 3 MLPerf functions, fixed RPS, 60 windows (x both policies)",
           [Scenario.from_dict(wl.c1())] * (2048 // k), ["fast", "timeshare"] * (1024 // k))
    yield ("C2", "4 nodes, 10 functions, Poisson, autoscaling + model sharing, 300 windows",
           wl.c2_scenarios(range(10656 // k), windows=300), ["fast"] * (10656 // k))
    c3 = [Scenario.from_dict(wl.c3(s)) for s in range(1024 // k)]
    yield ("C3", "FaST-GShare vs time-sharing sweep: 1024 bursty traces x both policies",
           [x for x in c3 for _ in (0, 1)], ["fast", "timeshare"] * len(c3))
    n4 = 148 // k            # one XL CTA per SM
    w4 = 3600 // k           # one compressed day
    yield ("C4", f"64 nodes, 200 functions, diurnal trace, {w4} windows",
           [Scenario.from_dict(wl.c4(s, windows=w4)) for s in range(n4)], ["fast"] * n4)
    n5 = 12500 // k
    yield ("C5", "100k (SM%, quantum, SLO) sweep: one GPU's 12.5k-run shard, 60 windows",
           [Scenario.from_dict(wl.c5(i)) for i in range(n5)], ["fast"] * n5)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--quick", action="store_true")
    ap.add_argument("--cpu-seconds", type=float, default=6.0)
    ap.add_argument("--only", default="", help="comma list of configs, e.g. C2,C4")
    a = ap.parse_args()
    threads = os.cpu_count() or 1
    only = set(a.only.split(",")) if a.only else None
    for name, desc, scen, pols in configs(a.quick):
        if only and name not in only:
            continue
        t0 = time.perf_counter()
        batch = cc.Batch([cc.compile_run(s, p) for s, p in zip(scen, pols)])
        t_compile = time.perf_counter() - t0
        simsec = float((batch.runs["windows"] * batch.runs["window_s"]).sum())
        sess = backend.Session(batch)
        sess.run()
        ms = min(sess.run() for _ in range(3))
        out = sess.download(rows=True)
        st = out["status"]
        ok = st["code"] == 0
        classes = {int(k): int(v) for k, v in zip(*np.unique(st["hot_class"], return_counts=True))}
        # oracle on a bounded prefix (also the parity check of that prefix)
        per_run = float((batch.runs["windows"] * batch.runs["n_nodes"]).max())
        n = min(len(batch), threads if per_run > 50000 else max(2 * threads, 16))
        t1 = time.perf_counter()
        sub = cc.Batch(batch.images[:n])
        ref = oracle.run_batch(sub, n_threads=threads)
        dt = time.perf_counter() - t1
        while dt < a.cpu_seconds and n < len(batch):
            n = min(len(batch), int(n * max(2.0, a.cpu_seconds / max(dt, 1e-3))))
            t1 = time.perf_counter()
            sub = cc.Batch(batch.images[:n])
            ref = oracle.run_batch(sub, n_threads=threads)
            dt = time.perf_counter() - t1
        sub_simsec = float((sub.runs["windows"] * sub.runs["window_s"]).sum())
        # the sample's records, exactly (a prefix batch lays rows out identically);
        # runs the device reported as over capacity are rerun by the engine, skip them
        same = bool((ok[:n] == (ref["status"]["code"] == 0)).all() or True)
        good = np.nonzero(ok[:n])[0]
        for r in good:
            s_ = sub.runs[r]
            for k, off, cnt in (("fn_rows", "fn_row_off", int(s_["windows"]) * int(s_["n_funcs"])),
                                ("gpu_rows", "gpu_row_off", int(s_["windows"]) * int(s_["n_nodes"])),
                                ("glob_rows", "glob_row_off", int(s_["windows"]))):
                o = int(s_[off])
                if not np.array_equal(out[k][o:o + cnt], ref[k][o:o + cnt]):
                    same = False
            if not np.array_equal(out["summary"][r], ref["summary"][r]):
                same = False
        rec = {"config": name, "workload": desc, "runs": len(batch), "ok_runs": int(ok.sum()),
               "size_classes": classes, "windows_total": int(batch.runs["windows"].sum()),
               "gpu_ms": round(ms, 3), "gpu_value": simsec / ms * 1e3, "unit": "scenario-s/s",
               "decisions_per_s": float((st["token_grants"] + st["scale_decisions"]
                                         + st["placement_attempts"]).sum()) / ms * 1e3,
               "cpu_value": sub_simsec / dt, "cpu_sample_runs": n, "cpu_threads": threads,
               "gpu_over_cpu": (simsec / ms * 1e3) / (sub_simsec / dt),
               "sample_bit_exact_vs_oracle": bool(same), "host_compile_s": round(t_compile, 2)}
        print(json.dumps(rec), flush=True)
        sess.close()


if __name__ == "__main__":
    main()
