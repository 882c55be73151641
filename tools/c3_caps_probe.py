import sys, numpy as np
sys.path.insert(0, "/root/repo")
from paper_2309_00558_b200 import backend, compiler as cc, workloads as wl
from paper_2309_00558_b200.scenario import Scenario
sc = [Scenario.from_dict(wl.c3(s)) for s in range(1024)]
b = cc.Batch([cc.compile_run(x, p) for x in sc for p in ("fast", "timeshare")])
s = backend.Session(b); s.run(); st = s.download(rows=False)["status"]
bad = st[st["code"] != 0]
print("codes", np.unique(bad["code"], return_counts=True), "details", np.unique(bad["detail"], return_counts=True))
print("caps of bad", np.unique(b.runs["cap_pods"][st["code"] != 0], return_counts=True), "peak", bad["peak_pods"][:10], "arg0", bad["arg0"][:10])
