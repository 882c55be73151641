"""Probe: C2 with fixed initial pods, with and without epochs (icache study).
usage: python tools/noepoch_probe.py <epoch_windows> [runs]"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2309_00558_b200 import backend, compiler as cc, workloads as wl
from paper_2309_00558_b200.scenario import Scenario
E = int(sys.argv[1]); runs = int(sys.argv[2]) if len(sys.argv) > 2 else 9472
PODS = {"resnet": [(12, 0.4)] * 4, "rnnt": [(24, 0.4)] * 4, "bert": [(50, 0.6)] * 2}
sc = []
for s in range(runs):
    d = wl.c2(s, windows=100); d["epoch_windows"] = E
    for fn in d["functions"]:
        kind = fn["function_id"][:-2]
        fn["initial_pods"] = [{"sm": a, "quota": q} for a, q in PODS[kind]]
    sc.append(Scenario.from_dict(d))
batch = cc.Batch([cc.compile_run(x, "fast") for x in sc])
sess = backend.Session(batch); sess.run()
ms = min(sess.run() for _ in range(3))
st = sess.download(rows=False)["status"]
ps = float(st["pod_steps"].sum())
print(f"epoch_windows={E}: {ms:.1f} ms  pod-steps {ps:.3g}  ns/pod-step {ms*1e6/max(ps,1):.4f}  "
      f"run-steps/s {runs*100*50/ms*1e3:.3g}  bad {(st['code'] != 0).sum()}")
