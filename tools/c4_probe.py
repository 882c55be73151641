import sys; sys.path.insert(0, "/root/repo")
from paper_2309_00558_b200 import backend, compiler as cc, workloads as wl
from paper_2309_00558_b200.scenario import Scenario
b = cc.Batch([cc.compile_run(Scenario.from_dict(wl.c4(s, windows=40)), "fast") for s in range(64)])
s = backend.Session(b); print(s.run())
