"""Compile one BASELINE config and launch the megakernel on it (GPU box).

A minimal, deterministic target for ncu / compute-sanitizer captures of one
size class at a time:

    python tools/launch_config.py C4 --runs 148 --windows 600 [--launches 1]
    compute-sanitizer --tool racecheck python tools/launch_config.py C5 --runs 8

Prints the size-class histogram, the device time per launch and the status
codes; with --check, also compares the records with the oracle (exit 1 on a
mismatch) -- the check runs after the launches, so it is outside any capture
filtered to gs_sim_kernel*.
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def scenarios(cfg, runs, windows):
    from paper_2309_00558_b200 import workloads as wl
    if cfg == "C1":
        return wl.ScenarioSeq(lambda i: wl.c1(), runs), ["fast", "timeshare"] * (runs // 2) + ["fast"] * (runs % 2)
    if cfg == "C2":
        return wl.ScenarioSeq(lambda i: wl.c2(i, windows=windows or 300), runs), ["fast"] * runs
    if cfg == "C3":
        return wl.ScenarioSeq(lambda i: wl.c3(i // 2), runs), ["fast", "timeshare"] * (runs // 2) + ["fast"] * (runs % 2)
    if cfg == "C4":
        return wl.ScenarioSeq(lambda i: wl.c4(i, windows=windows or 600), runs), ["fast"] * runs
    if cfg == "C5":
        return wl.ScenarioSeq(wl.c5, runs), ["fast"] * runs
    if cfg == "MIX":      # every per-warp class + XL in one launch
        def make(i):
            k = i % 5
            if k == 0:
                return wl.c2(i, windows=windows or 20, n_funcs=3, fleet=2)
            if k == 1:
                return wl.c2(i, windows=windows or 20)
            if k == 2:
                return wl.c2(i, windows=windows or 20, n_funcs=20, fleet=8)
            if k == 3:
                return wl.c2(i, windows=windows or 12, n_funcs=48, fleet=24)
            return wl.c4(i, windows=windows or 8, n_funcs=80, fleet=40)
        return wl.ScenarioSeq(make, runs), ["fast", "timeshare"] * (runs // 2) + ["fast"] * (runs % 2)
    raise SystemExit(f"unknown config {cfg}")


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("config")
    ap.add_argument("--runs", type=int, default=148)
    ap.add_argument("--windows", type=int, default=0)
    ap.add_argument("--launches", type=int, default=1)
    ap.add_argument("--check", action="store_true")
    a = ap.parse_args()
    import numpy as np
    from paper_2309_00558_b200 import backend, compiler as cc
    sc, pols = scenarios(a.config, a.runs, a.windows)
    batch, _, errors = cc.compile_batch(sc, pols)
    assert not errors, errors
    sess = backend.Session(batch)
    ms = [sess.run() for _ in range(a.launches)]
    out = sess.download(rows=True)
    st = out["status"]
    rec = {"config": a.config, "runs": len(batch), "ms": ms,
           "classes": {int(k): int(v) for k, v in zip(*np.unique(st["hot_class"], return_counts=True))},
           "codes": {int(k): int(v) for k, v in zip(*np.unique(st["code"], return_counts=True))}}
    if a.check:
        sys.path.insert(0, os.path.join(ROOT, "oracle"))
        sys.path.insert(0, ROOT)
        import oracle
        import bench
        ref = oracle.run_batch(batch, n_threads=os.cpu_count() or 1)
        rec["parity"] = bench.parity_sample(batch, out, ref)
    sess.close()
    print(json.dumps(rec), flush=True)
    if a.check and rec["parity"]["runs"] != rec["parity"]["bit_exact"]:
        sys.exit(1)


if __name__ == "__main__":
    main()
