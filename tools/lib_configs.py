"""Device time of C1 / C5 (small runs) for several builds: python tools/lib_configs.py a.so b.so ..."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_2309_00558_b200 import backend, compiler as cc, workloads as wl
from paper_2309_00558_b200.scenario import Scenario
sets = {
    "C1": ([Scenario.from_dict(wl.c1())] * 4096, ["fast", "timeshare"] * 2048),
    "C5": ([Scenario.from_dict(wl.c5(i)) for i in range(12500)], ["fast"] * 12500),
    "C3": ([Scenario.from_dict(wl.c3(s)) for s in range(1024) for _ in (0, 1)], ["fast", "timeshare"] * 1024),
}
batches = {k: cc.Batch([cc.compile_run(s, p) for s, p in zip(*v)]) for k, v in sets.items()}
ref = {}
for path in sys.argv[1:]:
    backend._lib = None
    backend.LIB_PATH = os.path.abspath(path)
    for k, b in batches.items():
        s = backend.Session(b)
        s.run()
        ms = min(s.run() for _ in range(3))
        out = s.download(rows=False)
        summ = out["summary"].tobytes()
        same = ref.setdefault(k, summ) == summ
        simsec = float((b.runs["windows"] * b.runs["window_s"]).sum())
        print(f"{os.path.basename(path):12s} {k}: {ms:8.2f} ms  {simsec / ms / 1e3:7.3f} M sim-s/s  same={same}", flush=True)
        s.close()
