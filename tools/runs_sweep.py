"""Throughput vs batch size (tail effect of the persistent kernel).
usage: python tools/runs_sweep.py [windows] runs..."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2309_00558_b200 import backend, compiler as cc, workloads as wl
windows = int(sys.argv[1])
for runs in map(int, sys.argv[2:]):
    batch = cc.Batch([cc.compile_run(s, "fast") for s in wl.c2_scenarios(range(runs), windows=windows)])
    simsec = float((batch.runs["windows"] * batch.runs["window_s"]).sum())
    s = backend.Session(batch)
    s.run()
    ms = min(s.run() for _ in range(3))
    print(f"runs {runs:6d}: {ms:8.2f} ms  {simsec / ms * 1e3 / 1e6:6.3f} M sim-s/s")
    s.close()
