"""Time split of the drop-in API path on the GPU box (engine.run_batch):
host compile, the one-shot C-ABI call (pageable vs page-locked outputs),
summaries and CSV rendering.  usage: python tools/api_probe.py [runs]"""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2309_00558_b200 import backend, compiler as cc, engine, report, workloads as wl

n = int(sys.argv[1]) if len(sys.argv) > 1 else 3552
scen = wl.c2_scenarios(range(n), windows=300)
simsec = n * 300.0
engine.run_batch(scen[:64])                      # warm up CUDA + pool
T = {}
t = time.perf_counter(); batch, idx, err = cc.compile_batch(scen, ["fast"] * n); T["compile"] = time.perf_counter() - t
t = time.perf_counter(); out = backend.run_batch(batch, rows=True); T["run_pageable"] = time.perf_counter() - t
t = time.perf_counter(); pout = batch.alloc_outputs(rows=True, pinned=True); T["alloc_pinned"] = time.perf_counter() - t
t = time.perf_counter(); backend.run_batch(batch, out=pout); T["run_pinned"] = time.perf_counter() - t
t = time.perf_counter(); backend.run_batch(batch, out=pout); T["run_pinned_2"] = time.perf_counter() - t
t = time.perf_counter(); s = report.summaries(batch, pout); T["summaries"] = time.perf_counter() - t
t = time.perf_counter(); c = report.csv_texts(batch, pout); T["csv_all"] = time.perf_counter() - t
T["csv_MB"] = sum(len(x) for x in c) / 1e6
t = time.perf_counter(); reps = engine.run_batch(scen); sums = [r.summary() for r in reps]; T["api_total"] = time.perf_counter() - t
T["api_value"] = simsec / T["api_total"]
print({k: round(v, 4) for k, v in T.items()})
