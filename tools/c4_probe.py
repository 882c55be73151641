"""One XL launch on C4 runs (ncu target): python tools/c4_probe.py [runs] [windows]"""
import sys; sys.path.insert(0, "/root/repo")
from paper_2309_00558_b200 import backend, compiler as cc, workloads as wl
from paper_2309_00558_b200.scenario import Scenario
n = int(sys.argv[1]) if len(sys.argv) > 1 else 64
w = int(sys.argv[2]) if len(sys.argv) > 2 else 40
b = cc.Batch([cc.compile_run(Scenario.from_dict(wl.c4(s, windows=w)), "fast") for s in range(n)])
s = backend.Session(b); print(s.run())
