"""Time the current library at several launch shapes (warps/CTA, CTAs/SM).
usage: python tools/launch_sweep.py --runs 9472 --windows 100 4,0 4,5 4,6 2,12"""
import argparse, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2309_00558_b200 import backend, compiler as cc, workloads as wl
ap = argparse.ArgumentParser()
ap.add_argument("shapes", nargs="+")
ap.add_argument("--runs", type=int, default=9472)
ap.add_argument("--windows", type=int, default=100)
a = ap.parse_args()
batch = cc.Batch([cc.compile_run(s, "fast") for s in wl.c2_scenarios(range(a.runs), windows=a.windows)])
simsec = float((batch.runs["windows"] * batch.runs["window_s"]).sum())
s = backend.Session(batch)
for shape in a.shapes:
    w, b = (int(x) for x in shape.split(","))
    backend.set_launch(w, b)
    s.run()
    ms = min(s.run() for _ in range(3))
    print(f"warps/CTA {w} CTAs/SM {b or 'auto'}: {ms:8.2f} ms  {simsec / ms * 1e3 / 1e6:6.3f} M sim-s/s")
