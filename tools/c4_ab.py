"""C4 (XL class) device time for several builds: python tools/c4_ab.py [--windows W] a.so b.so ..."""
import argparse, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_2309_00558_b200 import backend, compiler as cc, workloads as wl
from paper_2309_00558_b200.scenario import Scenario
ap = argparse.ArgumentParser()
ap.add_argument("libs", nargs="+")
ap.add_argument("--windows", type=int, default=600)
ap.add_argument("--runs", type=int, default=148)
a = ap.parse_args()
b, _, _ = cc.compile_batch(wl.ScenarioSeq(lambda s: wl.c4(s, windows=a.windows), a.runs), ["fast"] * a.runs)
simsec = float((b.runs["windows"] * b.runs["window_s"]).sum())
ref = None
for path in a.libs:
    backend._lib = None
    backend.LIB_PATH = os.path.abspath(path)
    s = backend.Session(b)
    s.run()
    ms = min(s.run() for _ in range(2))
    out = s.download(rows=False)["summary"].tobytes()
    ref = ref or out
    print(f"{os.path.basename(path):12s} {ms:9.1f} ms  {simsec / ms:9.0f} k sim-s/s  same={out == ref}", flush=True)
    s.close()
